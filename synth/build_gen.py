"""Compile synth/_gen.c (OpenMP) to synth/libsynthgen.so."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libsynthgen.so")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "_gen.c")
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(src):
        return LIB
    subprocess.run(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", "-o", LIB, src, "-lm"], check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
