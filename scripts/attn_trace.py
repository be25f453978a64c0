"""Record the clock64 event trace of one tensor-core attention launch (layer L of a C3 decode step)
and save it to gpurun_out/attn_trace.npz (debug tool; see FOCUS_DBG_ATTN_TRACE)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
layer = int(sys.argv[1]) if len(sys.argv) > 1 else 10
os.environ["FOCUS_ATTN_TRACE_LAYER"] = str(layer)
import torch  # noqa: E402
from paper_2601_23278_b200 import FocusContext, make_config  # noqa: E402
from synth import get_config  # noqa: E402
from synth.gen import prompt_tokens  # noqa: E402

run = get_config(sys.argv[2] if len(sys.argv) > 2 else "C3")
ctx = FocusContext(make_config(run))
rids = list(range(run.n_requests))
for r in rids:
    ctx.focus_kv_append(r, prompt_tokens(r, run.prompt_len, run.model.vocab), run.gen_len)
for _ in range(4):
    ctx.focus_step_block(rids)
    ctx.focus_commit(rids)
ctx.focus_sync()
raw = np.frombuffer(ctx.focus_debug_export("ATTN_TRACE", cap=1 << 26), dtype=np.uint64)
sms = torch.cuda.get_device_properties(0).multi_processor_count
np.savez(os.path.join(ROOT, "gpurun_out", "attn_trace.npz"), trace=raw.reshape(sms, 8, 512))
print("saved", raw.size)
