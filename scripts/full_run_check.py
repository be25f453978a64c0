"""Full C3 generation (every request to its 512th token) through the C ABI: all tokens committed,
no invariant flag, and a digest of the committed tokens (compare FOCUS_GRAPH=0 vs 1 runs)."""
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2601_23278_b200 import FocusContext, make_config  # noqa: E402
from paper_2601_23278_b200.runner import generate  # noqa: E402
from synth import get_config  # noqa: E402
from synth.gen import prompt_tokens  # noqa: E402

run = get_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
ctx = FocusContext(make_config(run))
rids = list(range(run.n_requests))
for r in rids:
    ctx.focus_kv_append(r, prompt_tokens(r, run.prompt_len, run.model.vocab), run.gen_len)
torch.cuda.synchronize()
t0 = time.time()
log = generate(ctx, rids, keep_log=False)
ctx.focus_sync()
dt = time.time() - t0
h = hashlib.sha256()
n = 0
for r in rids:
    t = ctx.focus_get_tokens(r)
    assert len(t) == run.gen_len, (r, len(t))
    n += len(t)
    h.update(str(list(map(int, t))).encode())
print(f"{run.name}: {log.steps} steps, {n} tokens ({log.decoded} decoded), {dt:.2f} s wall, digest {h.hexdigest()[:16]}")
