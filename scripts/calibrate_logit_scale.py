"""Decoded tokens per request-step of C3 at several power-of-two LM-head scales (focus_config::
logit_scale): picks the "calibrated" regime of SURVEY 8(d) (mean decoded / step ~ 0.1 B, the
fig:decoding_stats regime).  Usage: python scripts/calibrate_logit_scale.py [C3] [n_req] [steps]"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_23278_b200 import FocusContext, make_config  # noqa: E402
from synth import get_config  # noqa: E402
from synth.gen import prompt_tokens  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
n_req = int(sys.argv[2]) if len(sys.argv) > 2 else 16
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 34
base = get_config(name)
for scale in (1.0, 8.0, 16.0, 32.0, 64.0):
    run = base.with_(model=dataclasses.replace(base.model, logit_scale=scale), n_requests=n_req)
    ctx = FocusContext(make_config(run))
    rids = list(range(n_req))
    for r in rids:
        ctx.focus_kv_append(r, prompt_tokens(r, run.prompt_len, run.model.vocab), run.gen_len)
    dec = nonflush = 0
    live = list(rids)
    for _ in range(steps):
        ctx.focus_step_block(live)
        st = ctx.states()
        nonflush += sum(1 for r in live if not st[r].flush)
        res = ctx.commit_results(live)
        dec += sum(x["n_new"] for x in res)
        live = [x["req_id"] for x in res if not x["finished"]]
    print(json.dumps({"scale": scale, "decoded_per_request_step": round(dec / max(nonflush, 1), 3),
                      "B": run.method.block_size, "steps": steps, "requests": n_req}), flush=True)
    del ctx
    torch.cuda.empty_cache()
