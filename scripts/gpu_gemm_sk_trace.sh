python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include scripts/gemm_bench.cu -o /tmp/gemm_bench -Lpaper_2601_23278_b200 -lfocus -Xlinker -rpath=$PWD/paper_2601_23278_b200 2>/dev/null || exit 1
FOCUS_GEMM_PSK=1 GEMM_TRACE=1 timeout 60 /tmp/gemm_bench 428 2>&1 | grep -E "o\(|down|gu\(sw"
python - <<'PY'
import numpy as np, glob
for fn in sorted(glob.glob("gpurun_out/gemm_trace_M428_o(add).bin")):
    t = np.fromfile(fn, dtype=np.int64).reshape(148, 3, 256)
    for b in (0, 1, 2, 3, 64, 65, 146, 147):
        t0 = t[b, 0, 0]
        prod = t[b, 0, 1:][t[b, 0, 1:] > 0] - t0
        mma = t[b, 1, 1:][t[b, 1, 1:] > 0] - t0
        epi = t[b, 2, 1:][t[b, 2, 1:] > 0] - t0
        print(b, "prod n", len(prod), "first/last", prod[:1], prod[-1:], "mma n", len(mma), mma[:1], mma[-1:], "epi", epi)
PY
