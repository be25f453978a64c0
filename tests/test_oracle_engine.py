"""End-to-end pins of the oracle engine (CPU, -m "not gpu").

- No-eviction equivalence: strategy NONE + cache NONE reproduces a dense
  block-causal recompute of the whole sequence at every step (exact KV cache semantics of
  block diffusion), to 1e-10 in binary64.
- Step invariants: masked -> decoded only, evicted positions stay masked, at
  least one decode per non-flush step, R non-decreasing within a block and -1 after a reset,
  committed KV never rewritten (asserted inside the engine), deterministic replay.
"""
import numpy as np
import pytest

from oracle.engine import OracleEngine, request_prompts, run_to_completion
from oracle.model import Backbone
from oracle.numerics import attend
from synth import get_config
from synth.configs import CACHE_NONE, STRATEGY_NONE, MethodConfig, ModelConfig


def _dense_block_causal_logits(bb: Backbone, cfg, tokens, prompt_len, B):
    """Recompute every position from scratch with the block-causal mask: prompt position p sees
    [0, p]; a generated position in block b sees [0, s_b + B)."""
    n = len(tokens)
    lim = [p + 1 if p < prompt_len else prompt_len + ((p - prompt_len) // B + 1) * B for p in range(n)]
    x = bb.embed(tokens)
    pos = np.arange(n)
    for l in range(cfg.n_layers):
        q, k, v = bb.qkv(l, x, pos)
        o = np.empty((n, cfg.n_q_heads, cfg.head_dim))
        for i in range(n):
            for h in range(cfg.n_q_heads):
                g = h // cfg.group
                o[i, h] = attend(q[i:i + 1, h], k[:lim[i], g], v[:lim[i], g])[0]
        x = bb.mlp(l, bb.o_proj(l, x, o.reshape(n, -1)))
    return bb.logits(x)


@pytest.mark.parametrize("layers,B,heads", [(2, 4, (4, 4)), (3, 3, (4, 2)), (4, 5, (2, 1))])
def test_no_eviction_equivalence(layers, B, heads):
    model = ModelConfig(n_layers=layers, d_model=32, n_q_heads=heads[0], n_kv_heads=heads[1], head_dim=8,
                        d_ff=64, vocab=29, rope_theta=1e4)
    run = get_config("C1").with_(model=model, method=MethodConfig(block_size=B, strategy=STRATEGY_NONE,
                                                                 cache_mode=CACHE_NONE),
                                 prompt_len=7, gen_len=2 * B)
    eng = OracleEngine(run, "ref")
    prompt = request_prompts(run)[0]
    eng.kv_append(0, prompt, run.gen_len)
    st = eng.req[0]
    steps = 0
    while not st.finished:
        rec = eng.step_one(0)
        assert rec.P == list(range(B)) and rec.S == rec.P
        if rec.M:
            toks = list(prompt) + st.output + list(st.tok)
            dense = _dense_block_causal_logits(eng.bb, model, np.array(toks), len(prompt), B)
            want = dense[[st.s + j for j in rec.logit_rows]]
            fin = np.isfinite(want)
            assert np.array_equal(fin, np.isfinite(rec.logits))
            assert np.max(np.abs(want[fin] - rec.logits[fin])) < 1e-10
        eng.commit_one(0)
        steps += 1
    assert len(st.output) == run.gen_len


def test_c1_invariants_and_determinism():
    run = get_config("C1")
    eng, log = run_to_completion(run, "ref")
    eng2, _ = run_to_completion(run, "ref")
    assert eng.req[0].output == eng2.req[0].output                      # deterministic replay
    assert len(eng.req[0].output) == run.gen_len
    mask = run.model.mask_token_id
    prevR, prev_s = -1, None
    for recs, coms in log:
        rec, com = recs[0], coms[0]
        if rec.flush:
            assert not com.decoded
        else:
            assert len(com.decoded) >= 1                                # progress
            assert set(com.decoded) <= set(rec.M) & set(rec.S)          # masked -> decoded, evicted stay masked
            assert all(t != mask for t in com.tokens)
        assert rec.R_new >= prevR                                       # R monotone in a block
        prevR = -1 if com.block_done else rec.R_new
    assert mask not in eng.req[0].output


def test_batch_invariance_and_modes():
    run = get_config("C1").with_(n_requests=3)
    eng_all, _ = run_to_completion(run, "gpu")
    for r in range(3):
        eng_one, _ = run_to_completion(run, "gpu", rids=[r])
        assert eng_one.req[r].output == eng_all.req[r].output
