"""GPU parity of the MoE FFN (LLaDA2.0-mini-shaped workload; readings A-M5, A-M6) through
the C ABI, against the oracle's MoE (oracle/moe.py, pinned in tests/test_oracle_moe.py).

- Stage parity at an MoE layer (taps): the routing of every row, recomputed by the oracle from the GPU's
  bf16 RMSNorm rows and router weights, equals the GPU's except where two logits tie within fp32
  accumulation noise; the layer's residual update matches the oracle's MoE at relative L2 <= 1e-3.
- The FOCUS rules stay bit-exact on an MoE model (resynced protocol) and the committed tokens of a small
  MoE model agree >= 90 % with the oracle (free running: discrete routing / selection decisions within
  fp32 noise diverge for any GEMM accumulation order, profiles/r2_moe_free_running_agreement.txt).
"""
import dataclasses

import numpy as np
import pytest

from oracle import moe as MOE
from oracle.engine import request_prompts
from oracle.model import Backbone, OracleWeights
from oracle.numerics import f32
from synth import get_config
from synth.configs import MethodConfig, ModelConfig

from gpu_helpers import rel_l2

pytestmark = pytest.mark.gpu

# layer 0 dense, layers 1-2 MoE (16 experts of width 128, top-4, one shared expert); head_dim 128
MOE_TC = ModelConfig(n_layers=3, d_model=256, n_q_heads=8, n_kv_heads=2, head_dim=128, d_ff=256, vocab=61,
                     rope_theta=1e4, n_experts=16, top_k=4, d_expert=128, n_shared_experts=1, n_dense_layers=1)


def _ctx(run, **kw):
    from paper_2601_23278_b200 import FocusContext, make_config
    return FocusContext(make_config(run, **kw))


@pytest.mark.parametrize("nreq,B", [(3, 16), (20, 16)])
def test_moe_layer_stage(nreq, B):
    run = get_config("C3").with_(model=MOE_TC, method=MethodConfig(block_size=B), n_requests=nreq, prompt_len=40,
                                 gen_len=2 * B)
    ctx = _ctx(run, debug_taps=True)
    prompts = request_prompts(run)
    for r in range(nreq):
        ctx.focus_kv_append(r, prompts[r], run.gen_len)
    live = list(range(nreq))
    ctx.focus_step_block(live)
    ctx.commit_results(live)
    W = OracleWeights(MOE_TC, run.weight_seed)
    bb = Backbone(MOE_TC, W, "gpu")
    d = MOE_TC.d_model
    for l in (1, 2):
        ctx.focus_set_tap(l)
        ctx.focus_step_block(live)
        ctx.focus_sync()
        MS = int(ctx.counters()[1])
        x_mid = ctx.export_f32("TAP_X_MID", (MS, d)).astype(np.float64)
        h2 = ctx.export_bf16("TAP_H2", (MS, d))
        x_out = ctx.export_f32("TAP_X_OUT", (MS, d)).astype(np.float64)
        w = W.layer(l)
        if l == MOE_TC.n_layers - 1:
            # routing of the last MoE layer: the oracle's selection from the GPU's bf16 normalised rows
            # (fp32 logits) equals the GPU's, order included, except in the tie band at the selection
            # boundary (two logits within fp32 accumulation noise); weights within 1e-5
            K = MOE_TC.top_k
            sel = np.frombuffer(ctx.focus_debug_export("MOE_SEL"), np.int32).reshape(MS, K)
            wt = np.frombuffer(ctx.focus_debug_export("MOE_WT"), np.float32).reshape(MS, K)
            z = f32(h2 @ w["router"].T)
            checked = 0
            for n in range(MS):
                srt = np.sort(z[n])[::-1]
                gaps = np.abs(np.diff(srt[:K + 1]))
                if np.min(gaps) < 1e-5 * max(1.0, abs(srt[0])):
                    continue
                r = MOE.route(z[n], K)
                assert [e for e, _ in r] == list(sel[n]), (n, r, sel[n])
                assert np.max(np.abs(np.array([v for _, v in r]) - wt[n])) <= 1e-5
                checked += 1
            assert checked >= 0.9 * MS
        # the layer's residual update against the oracle's MoE on the GPU's input rows
        want = bb.moe(l, x_mid)
        err = rel_l2(x_out - x_mid, want - x_mid)
        assert err <= 1e-3, (l, err)        # measured <= 2e-7 (profiles/r2_moe_free_running_agreement.txt)
        ctx.commit_results(live)
    ctx.focus_set_tap(-1)
    ctx.focus_sync()


def test_moe_end_to_end_small():
    from paper_2601_23278_b200.runner import generate, prefill_all
    from oracle.engine import run_to_completion
    run = get_config("C1").with_(model=MOE_TC, method=MethodConfig(block_size=8), n_requests=3, prompt_len=24,
                                 gen_len=16)
    ctx = _ctx(run)
    rids = prefill_all(ctx, request_prompts(run), run.gen_len)
    generate(ctx, rids, keep_log=False)
    ctx.focus_sync()
    eng, _ = run_to_completion(run, "gpu")
    tot = agree = 0
    for r in rids:
        g, o = ctx.focus_get_tokens(r), eng.req[r].output
        assert len(g) == run.gen_len
        tot += len(o)
        agree += sum(int(a == b) for a, b in zip(g, o))
    # MoE free running: >= 90 % (discrete routing / selection decisions within fp32 noise diverge for
    # either GEMM path: profiles/r2_moe_free_running_agreement.txt); the rules are exact (resynced test)
    assert agree >= 0.90 * tot, (agree, tot)


def test_moe_resynced_rules_bit_exact():
    from test_gpu_parity import _resync
    mdl = dataclasses.replace(MOE_TC, logit_scale=16.0)
    run = get_config("C1").with_(model=mdl, method=MethodConfig(block_size=16), n_requests=5, prompt_len=40,
                                 gen_len=32, page_size=16)
    st = _resync(run, [40] * 5)
    assert st["steps"] > 0
