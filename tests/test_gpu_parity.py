"""GPU parity of the CUDA path (libfocus.so through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star / DESIGN.md "numerics contract"):
  - selection, compaction indices, committed token ids, decisions and state: bit-exact when the
    oracle is fed the GPU's importance and confidence values;
  - importance: per-element relative error <= 1e-3 (denominator floored at 1e-6 * |P| * Hq);
  - attention output: relative L2 <= 1e-2 at bf16;
  - confidence: |conf_gpu - conf_oracle| <= 1e-5 * conf_oracle, argmax token bit-exact;
  - end-to-end committed tokens on the small config: >= 99 % agreement (free running).
"""
import ctypes as C
import dataclasses

import numpy as np
import pytest

from oracle import focus as F
from oracle.engine import OracleEngine, request_prompts, run_to_completion
from synth import get_config
from synth.configs import (CACHE_DC, CACHE_DC_PLUS, CACHE_NONE, PLACEHOLDER_ALL_MASKED, STRATEGY_FIXED_BOTTOM,
                           STRATEGY_FIXED_RANDOM, STRATEGY_FIXED_TOP, STRATEGY_NONE, MethodConfig, ModelConfig)

from gpu_helpers import bits, gpu_importance_sums, oracle_state_from_gpu

pytestmark = pytest.mark.gpu


def _ctx(run, **kw):
    from paper_2601_23278_b200 import FocusContext, make_config
    return FocusContext(make_config(run, **kw))


def _e2e(run):
    from paper_2601_23278_b200.runner import generate, prefill_all
    ctx = _ctx(run)
    prompts = request_prompts(run)
    rids = prefill_all(ctx, prompts, run.gen_len)
    generate(ctx, rids, keep_log=False)
    ctx.focus_sync()
    eng, _ = run_to_completion(run, "gpu")
    tot = agree = 0
    for r in rids:
        g, o = ctx.focus_get_tokens(r), eng.req[r].output
        assert len(g) == run.gen_len
        tot += len(o)
        agree += sum(int(a == b) for a, b in zip(g, o))
    return agree, tot, ctx


def test_c1_end_to_end():
    agree, tot, _ = _e2e(get_config("C1"))
    assert agree >= 0.99 * tot, (agree, tot)


@pytest.mark.parametrize("meth", [
    MethodConfig(block_size=4),
    MethodConfig(block_size=4, cache_mode=CACHE_DC),
    MethodConfig(block_size=4, cache_mode=CACHE_NONE, strategy=STRATEGY_NONE),
    MethodConfig(block_size=8, placeholder_mode=PLACEHOLDER_ALL_MASKED, alpha_num=6, alpha_den=5),
    MethodConfig(block_size=8, strategy=STRATEGY_FIXED_TOP, fixed_k=2),
    MethodConfig(block_size=8, strategy=STRATEGY_FIXED_BOTTOM, fixed_k=2),
    MethodConfig(block_size=8, strategy=STRATEGY_FIXED_RANDOM, fixed_k=3),
])
def test_small_end_to_end_variants(meth):
    run = get_config("C1").with_(method=meth, n_requests=4, gen_len=2 * meth.block_size)
    agree, tot, ctx = _e2e(run)
    assert agree >= 0.99 * tot, (agree, tot)
    ctx.focus_sync()          # no invariant flag


GQA_TINY = ModelConfig(n_layers=3, d_model=128, n_q_heads=8, n_kv_heads=2, head_dim=16, d_ff=256, vocab=61,
                       rope_theta=1e4)
# head_dim 128: the tensor-core (tcgen05) attention path; GQA_TINY (head_dim 16) runs the SIMT one
GQA_TC = ModelConfig(n_layers=3, d_model=256, n_q_heads=8, n_kv_heads=2, head_dim=128, d_ff=256, vocab=61,
                     rope_theta=1e4)


def _resync(run, prompt_lens, max_steps=1 << 30):
    """Drive the GPU step by step; before each step the oracle is re-synced to the GPU state, fed the
    GPU's importance partial sums and confidences, and must reproduce P/M, S, K, N_sigma, K_hist, R',
    the compaction row maps, the decisions and the whole post-commit state bit for bit.  The oracle's
    own argmax / confidence from the GPU's fp32 logits must match (argmax exact, conf <= 1e-5
    relative, c.7), and so must its own decisions wherever no confidence lies in the 1e-5 guard band
    around tau (or ties the fallback's best).  Returns counters of the regimes exercised."""
    B, m = run.method.block_size, run.model
    tau32 = float(np.float32(run.method.conf_threshold))
    nreq = run.n_requests
    ctx = _ctx(run, debug_taps=True)          # the fp32 logits are stored only with taps (fused vocab stats)
    prompts = request_prompts(run)
    for r in range(nreq):
        ctx.focus_kv_append(r, prompts[r], run.gen_len)
    eng = OracleEngine(run, "gpu")
    eng.script = {}
    live = list(range(nreq))
    steps = 0
    outputs = {r: [] for r in range(nreq)}
    stats = dict(steps=0, multi=0, above_tau=0, fallback=0, neighbour_same_step=0, guard=0, evicted=0, rows_L=0)
    while live and steps < max_steps:
        pre = ctx.states()
        ctx.focus_step_block(live)
        ctx.focus_sync()
        mid = ctx.states()
        cnt = ctx.counters()
        Pm = [mid[r].P for r in live]
        I0 = gpu_importance_sums(np.frombuffer(ctx.focus_debug_export("I0"), np.float32), cnt, Pm, m.n_kv_heads, B)
        I1 = gpu_importance_sums(np.frombuffer(ctx.focus_debug_export("I1"), np.float32), cnt, Pm, m.n_kv_heads, B)
        rowsS, rowsL = ctx.rows("S"), ctx.rows("L")
        res = ctx.commit_results(live)
        post = ctx.states()
        tc = np.frombuffer(ctx.focus_debug_export("TOKCONF"), dtype=np.dtype([("tok", "<i4"), ("conf", "<f4")]))
        logits = ctx.export_f32("LOGITS", (len(tc), m.vocab))
        stats["rows_L"] += len(tc)
        expS, expL = [], []
        lrow = 0
        for i, r in enumerate(live):
            eng.req[r] = oracle_state_from_gpu(pre[r], r, B, prompt_lens[r])
            g = mid[r]
            rec_pos = [j for j in range(B) if j not in eng.req[r].committed]
            Mpos = [j for j in rec_pos if eng.req[r].dstep[j] is None]
            # logit rows of this request (S cap M, ascending j) -> GPU conf / tok (fed to the oracle)
            nl = bin(g.S & g.M).count("1")
            conf = {int(rowsL[lrow + k][1]): float(tc["conf"][lrow + k]) for k in range(nl)}
            tok = {int(rowsL[lrow + k][1]): int(tc["tok"][lrow + k]) for k in range(nl)}
            # oracle's own confidence from the GPU's logits: argmax exact, conf within 1e-5
            own = {}
            for k in range(nl):
                z = logits[lrow + k].astype(np.float64).copy()
                z[m.mask_token_id] = -np.inf
                t_o, c_o = F.confidence(z)
                assert t_o == tc["tok"][lrow + k], (steps, r, k)
                assert abs(c_o - tc["conf"][lrow + k]) <= 1e-5 * c_o, (steps, r, k, c_o, tc["conf"][lrow + k])
                own[int(rowsL[lrow + k][1])] = c_o
            lrow += nl
            if own:
                vals = sorted(own.values(), reverse=True)
                band = any(abs(c - tau32) <= 1e-5 * tau32 for c in vals) or \
                    (len(vals) > 1 and vals[0] < tau32 and vals[1] >= vals[0] * (1 - 2e-5))
                if band:
                    stats["guard"] += 1
                else:
                    assert F.decide(own, tau32) == F.decide(conf, tau32), (steps, r)
            eng.script[(r, pre[r].t + 1)] = {"I0": I0[i].astype(np.float64), "I1": I1[i].astype(np.float64),
                                             "conf": conf, "tok": tok}
            rec = eng.step_one(r)
            assert bits(g.P, B) == rec.P and bits(g.M, B) == Mpos == rec.M
            assert bits(g.S, B) == rec.S, (steps, r)
            assert g.R_new == rec.R_new
            if not rec.flush:
                assert (g.K, g.n_sigma, g.k_hist) == (rec.sel.K, rec.sel.n_sigma, rec.sel.k_hist)
                stats["evicted"] += len(rec.P) - len(rec.S)
            com = eng.commit_one(r)
            o = eng.req[r]
            p = post[r]
            outputs[r] += o.output
            assert res[i]["pos"] == com.decoded and res[i]["tok"] == com.tokens
            assert bits(p.committed, B) == sorted(o.committed) or (com.block_done and p.committed == 0)
            assert (p.R, p.token_sum, p.total_steps, p.s, p.b, bool(p.finished)) == \
                (o.R, o.token_sum, o.total_steps, o.s, o.b, o.finished)
            if not o.finished:
                assert list(p.tok[:B]) == o.tok
            if not rec.flush:
                n_above = sum(1 for c in conf.values() if c >= tau32)
                stats["above_tau"] += n_above
                stats["fallback"] += int(n_above == 0)
                stats["multi"] += int(len(com.decoded) >= 2)
                t = pre[r].t + 1
                # DC+ commits whose right neighbour was decoded in this very step (A-DC3)
                stats["neighbour_same_step"] += sum(
                    1 for j in com.new_committed if j < B - 1 and (j + 1) in com.decoded and o.dstep[j] is not None
                    and o.dstep[j] < t)
            expS += [(r, j) for j in rec.S]
            expL += [(r, j) for j in rec.logit_rows]
        assert [(int(a), int(b)) for a, b in rowsS[:, :2]] == expS          # compaction row maps
        assert [(int(a), int(b)) for a, b in rowsL[:, :2]] == expL
        live = [x["req_id"] for x in res if not x["finished"]]
        steps += 1
    stats["steps"] = steps
    ctx.focus_sync()
    if not live:
        for r in range(nreq):
            assert ctx.focus_get_tokens(r) == outputs[r]
    return stats


@pytest.mark.parametrize("model", [GQA_TINY, GQA_TC], ids=["simt", "tc"])
@pytest.mark.parametrize("B,nreq,prompt", [(8, 6, 13), (16, 5, 40), (32, 3, 70), (64, 2, 9), (5, 7, 1)])
def test_resynced_rules_bit_exact(B, nreq, prompt, model):
    run = get_config("C1").with_(model=model, method=MethodConfig(block_size=B), n_requests=nreq,
                                 prompt_len=prompt, gen_len=2 * B, page_size=16)
    _resync(run, [prompt] * nreq)


@pytest.mark.parametrize("model", [GQA_TINY, GQA_TC], ids=["simt", "tc"])
@pytest.mark.parametrize("cache", [CACHE_DC_PLUS, CACHE_DC], ids=["dcplus", "dc"])
@pytest.mark.parametrize("B,nreq,prompt", [(8, 6, 13), (16, 40, 40)])
def test_resynced_threshold_regime(B, nreq, prompt, cache, model):
    """logit_scale 16 puts the max softmax probability above tau = 0.9 for about a third of the logit
    rows (oracle calibration at V = 61): the conf >= tau branch of Decode_and_Verify (Alg.1 P:658,
    P:140) commits several positions per step, DC+ commits positions whose right neighbour was decoded
    in the same step (A-DC3), and 40 requests exceed the 32-lane warp loops of selection and commit."""
    mdl = dataclasses.replace(model, logit_scale=16.0)
    run = get_config("C1").with_(model=mdl, method=MethodConfig(block_size=B, cache_mode=cache), n_requests=nreq,
                                 prompt_len=prompt, gen_len=2 * B, page_size=16)
    st = _resync(run, [prompt] * nreq)
    assert st["above_tau"] > 0 and st["multi"] > 0 and st["fallback"] > 0, st
    if cache == CACHE_DC_PLUS:
        assert st["neighbour_same_step"] > 0, st


# SDAR-8B layer shapes (d 4096, GQA 32/8, d_ff 12288, V 151936) with 4 layers: the full-vocab commit
# path (16 vocab chunks per row, fixed-order combine) and 64 requests (two warp rounds)
SDAR8B_4L = ModelConfig(n_layers=4, d_model=4096, n_q_heads=32, n_kv_heads=8, head_dim=128, d_ff=12288,
                        vocab=151936, rope_theta=1e6)


@pytest.mark.parametrize("scale", [1.0, 32.0], ids=["fallback", "calibrated"])
def test_resynced_full_vocab_64_requests(scale):
    """C3's commit shapes: 64 requests x B = 16 at V = 151936.  At logit_scale 1 every step decodes by
    the fallback; the calibrated scale makes conf >= tau fire on part of the rows."""
    mdl = dataclasses.replace(SDAR8B_4L, logit_scale=scale)
    run = get_config("C3").with_(model=mdl, n_requests=64, prompt_len=48, gen_len=16)
    st = _resync(run, [48] * 64)
    assert st["rows_L"] > 64 * 16, st
    if scale == 1.0:
        assert st["above_tau"] == 0 and st["multi"] == 0, st
    else:
        assert st["above_tau"] > 0 and st["multi"] > 0, st


# d_ff = 8192: the down projection (K = 8192) takes the ordered split-K path of the GEMM
GQA_TC_DEEPFF = ModelConfig(n_layers=3, d_model=256, n_q_heads=8, n_kv_heads=2, head_dim=128, d_ff=8192, vocab=61,
                            rope_theta=1e6)


@pytest.mark.parametrize("model", [GQA_TINY, GQA_TC, GQA_TC_DEEPFF], ids=["simt", "tc", "tc_splitk"])
def test_determinism_and_batch_invariance(model):
    from paper_2601_23278_b200.runner import generate, prefill_all
    run = get_config("C1").with_(model=model, method=MethodConfig(block_size=8), n_requests=5, gen_len=16)
    prompts = request_prompts(run)
    outs = []
    for _ in range(2):
        ctx = _ctx(run)
        rids = prefill_all(ctx, prompts, run.gen_len)
        generate(ctx, rids, keep_log=False)
        outs.append([ctx.focus_get_tokens(r) for r in rids])
    assert outs[0] == outs[1]
    ctx = _ctx(run)
    ctx.focus_kv_append(3, prompts[3], run.gen_len)
    generate(ctx, [3], keep_log=False)
    assert ctx.focus_get_tokens(3) == outs[0][3]


@pytest.mark.parametrize("model", [GQA_TINY, GQA_TC], ids=["simt", "tc"])
def test_prefill_kv_matches_dense_causal_recompute(model):
    run = get_config("C1").with_(model=model, method=MethodConfig(block_size=8), n_requests=2, prompt_len=45,
                                 gen_len=16, page_size=16)
    ctx = _ctx(run, max_prefill_chunk=32)            # two prefill chunks
    prompts = request_prompts(run)
    ctx.focus_kv_append(1, prompts[1], run.gen_len)
    eng = OracleEngine(run, "gpu")
    eng.kv_append(1, prompts[1], run.gen_len)
    m = run.model
    for l in range(m.n_layers):
        for what, ref in (("KV_K", eng.K[1][l]), ("KV_V", eng.V[1][l])):
            g = ctx.export_bf16(what, (45 + 8, m.n_kv_heads, m.head_dim), req_id=1, layer=l)[:45]
            want = ref[:45]
            err = np.linalg.norm(g - want) / np.linalg.norm(want)
            assert err < 1e-2, (l, what, err)
            if l == 0:                                   # layer 0 K/V: same bf16 rounding almost everywhere
                assert np.mean(g == want) > 0.95, (l, what)


@pytest.mark.parametrize("model", [GQA_TINY, GQA_TC], ids=["simt", "tc"])
def test_committed_kv_slots_never_rewritten(model):
    from paper_2601_23278_b200.runner import prefill_all
    run = get_config("C1").with_(model=model, method=MethodConfig(block_size=8), n_requests=2, gen_len=16)
    ctx = _ctx(run)
    prompts = request_prompts(run)
    prefill_all(ctx, prompts, run.gen_len)
    m = run.model
    n = run.prompt_len + run.gen_len
    frozen = {}
    live = [0, 1]
    while live:
        ctx.focus_step_block(live)
        res = ctx.commit_results(live)
        for r in live:
            st = ctx.states()[r]
            if st.finished:
                continue
            for l in range(m.n_layers):
                K = ctx.export_bf16("KV_K", (min(st.s + 8, n), m.n_kv_heads, m.head_dim), req_id=r, layer=l)
                for (rr, ll, p), v in frozen.items():
                    if rr == r and ll == l:
                        assert np.array_equal(K[p], v), (r, l, p)
                for j in bits(st.committed, 8):
                    frozen.setdefault((r, l, st.s + j), K[st.s + j].copy())
                for p in range(run.prompt_len):
                    frozen.setdefault((r, l, p), K[p].copy())
        live = [x["req_id"] for x in res if not x["finished"]]


@pytest.mark.parametrize("model", [GQA_TC, GQA_TC_DEEPFF], ids=["tc", "tc_splitk"])
def test_sharding_invariance_batch_invariant(model):
    """SURVEY 8(e) / tier T5: with batch_invariant = 1, LPT-sharding a mixed-length batch over world
    sizes 1, 2 and 4 (each shard its own context, as on its own GPU) gives every request exactly the
    same committed tokens (logit_scale 16: multi-token commits, so block phases differ by request)."""
    from paper_2601_23278_b200 import dist as D
    from paper_2601_23278_b200.runner import generate
    mdl = dataclasses.replace(model, logit_scale=16.0)
    run = get_config("C1").with_(model=mdl, method=MethodConfig(block_size=16), n_requests=8, prompt_len=20,
                                 prompt_len_hi=300, gen_len=32, page_size=64)
    prompts = request_prompts(run)
    costs = [len(p) + run.gen_len / 2 for p in prompts]
    outs = {}
    for world in (1, 2, 4):
        toks = {}
        for rank in range(world):
            mine = D.shard_requests(run.n_requests, world, rank, costs)
            ctx = _ctx(run, max_requests=len(mine), batch_invariant=True)
            for slot, g in enumerate(mine):
                ctx.focus_kv_append(slot, prompts[g], run.gen_len)
            generate(ctx, list(range(len(mine))), keep_log=False)
            for slot, g in enumerate(mine):
                toks[g] = ctx.focus_get_tokens(slot)
            del ctx
        outs[world] = toks
    assert outs[1] == outs[2] == outs[4]


@pytest.mark.parametrize("swap", ["1", "0"], ids=["swap_ab", "cta_pair"])
def test_resynced_swap_ab_gemm(monkeypatch, swap):
    """The whole step with the swap-AB decode GEMM (48 rows; the default at this row count) and with
    the CTA-pair GEMM: rules bit-exact in the resynced protocol, including the threshold regime."""
    monkeypatch.setenv("FOCUS_GEMM_SWAP", swap)
    mdl = dataclasses.replace(GQA_TC, logit_scale=16.0)
    run = get_config("C1").with_(model=mdl, method=MethodConfig(block_size=8), n_requests=6, prompt_len=13,
                                 gen_len=16, page_size=16)
    st = _resync(run, [13] * 6)
    assert st["above_tau"] > 0, st
