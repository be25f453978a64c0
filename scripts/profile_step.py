"""Run a workload to decode step `warm`, then run ONE step between cudaProfilerStart/Stop so that
`ncu --profile-from-start off` (or nsys-like tools) capture exactly one decode step.
Usage: python scripts/profile_step.py [C3] [warm_steps] [logit_scale]"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_23278_b200 import FocusContext, make_config  # noqa: E402
from synth import get_config  # noqa: E402
from synth.gen import prompt_tokens  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 260
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
run = get_config(name)
run = run.with_(model=dataclasses.replace(run.model, logit_scale=scale))
ctx = FocusContext(make_config(run))
rids = list(range(run.n_requests))
for r in rids:
    ctx.focus_kv_append(r, prompt_tokens(r, run.prompt_len, run.model.vocab), run.gen_len)
for _ in range(warm):
    ctx.focus_step_block(rids)
    ctx.focus_commit(rids)
ctx.focus_sync()
torch.cuda.profiler.start()
ctx.focus_step_block(rids)
ctx.focus_commit(rids)
ctx.focus_sync()
torch.cuda.profiler.stop()
c = ctx.counters()
print(f"profiled step {warm + 1}: M_P {c[0]} M_S {c[1]} M_L {c[2]}")
