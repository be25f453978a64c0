"""Masking pin of the oracle engine (SURVEY c.9 "masking oracle"; PAPER.md
P:300 "referable KV states", "evicted tokens serve as fixed reference KV states", "fill the
KV states ... before the token eviction in Layer 1").

An evicting FOCUS run of `OracleEngine` is recomputed step by step by a brute-force forward written
here, independently of `engine.py`: an explicit per-layer store {absolute position: (k, v)} written by
the rules, explicit key-position lists per layer, and attention as plain loops over those lists.

  layer 0        queries P, K/V written for P,          keys ctx + every block slot
  layer 1        queries P (prefix) then S (suffix),    K/V written for ALL of P before eviction,
                                                        keys ctx + every block slot
  layers >= 2    queries S, K/V written for S only,     keys ctx + block slots 0..R' -- slots of
                                                        evicted positions hold the K/V of their last
                                                        processing (stale), slots > R' are never read

The trace is checked to exercise both distinctions (a step with R' < B-1, a stale slot read at layers
>= 2), and the recomputation is shown to be sensitive to them: reading extent B (unwritten slots as the
zeros of a fresh pool) or refreshed K/V for evicted slots changes the logits.
"""
import numpy as np

from oracle import focus as F
from oracle.engine import OracleEngine, request_prompts
from synth import get_config
from synth.configs import MethodConfig, ModelConfig

MODEL = ModelConfig(n_layers=4, d_model=32, n_q_heads=4, n_kv_heads=2, head_dim=8, d_ff=64, vocab=29,
                    rope_theta=1e4)


def _attend_list(q, keys, vals, dh):
    """One query head against an explicit list of key/value vectors: plain loops."""
    sc = [float(np.dot(q, k)) / np.sqrt(dh) for k in keys]
    mx = max(sc)
    w = [np.exp(a - mx) for a in sc]
    tot = sum(w)
    out = np.zeros(dh)
    for wi, v in zip(w, vals):
        out += (wi / tot) * v
    return out


def _attn(bb, cfg, q, store, positions):
    """q [n, Hq, dh]; store {pos: (k [Hkv, dh], v [Hkv, dh])}; every row sees `positions`."""
    out = np.zeros((q.shape[0], cfg.n_q_heads, cfg.head_dim))
    for i in range(q.shape[0]):
        for h in range(cfg.n_q_heads):
            g = h // cfg.group
            out[i, h] = _attend_list(q[i, h], [store[p][0][g] for p in positions],
                                     [store[p][1][g] for p in positions], cfg.head_dim)
    return out.reshape(q.shape[0], -1)


def _brute_step(eng, rid, rec, store, variant="paper"):
    """Recompute the logits of one step from explicit key sets.  `store[l]` is updated in place
    (variant "paper" only).  variant "extent_B": layers >= 2 read every block slot (unwritten ones
    as zeros); "fresh_evicted": evicted slots at layers >= 2 hold this step's recomputed K/V."""
    cfg, bb = eng.cfg, eng.bb
    st = eng.req[rid]
    s, B, P, S = st.s, st.B, rec.P, rec.S
    if variant != "paper":
        store = {l: dict(v) for l, v in store.items()}
    ctx = list(range(s))
    whole = ctx + [s + j for j in range(B)]
    x = bb.embed([st.tok[j] for j in P])
    pos = np.array([s + j for j in P])
    # layer 0 on P
    q, k, v = bb.qkv(0, x, pos)
    for n, j in enumerate(P):
        store[0][s + j] = (k[n], v[n])
    x = bb.mlp(0, bb.o_proj(0, x, _attn(bb, cfg, q, store[0], whole)))
    # layer 1: K/V of all of P stored before eviction; queries of S only after it
    q1, k1, v1 = bb.qkv(1, x, pos)
    for n, j in enumerate(P):
        store[1][s + j] = (k1[n], v1[n])
    idx = [P.index(j) for j in S]
    xs = x[idx]
    xs = bb.mlp(1, bb.o_proj(1, xs, _attn(bb, cfg, q1[idx], store[1], whole)))
    xp = x                                   # all of P, only for the "fresh_evicted" variant
    if variant == "fresh_evicted":
        xp = bb.mlp(1, bb.o_proj(1, x, _attn(bb, cfg, q1, store[1], whole)))
    R_new = max(st.R, max(S))
    for l in range(2, cfg.n_layers):
        qs, ks, vs = bb.qkv(l, xs, np.array([s + j for j in S]))
        for n, j in enumerate(S):
            store[l][s + j] = (ks[n], vs[n])
        if variant == "fresh_evicted":
            qp, kp, vp = bb.qkv(l, xp, pos)
            for n, j in enumerate(P):
                if j not in S:
                    store[l][s + j] = (kp[n], vp[n])
        if variant == "extent_B":
            keys = whole
            zero = (np.zeros((cfg.n_kv_heads, cfg.head_dim)), np.zeros((cfg.n_kv_heads, cfg.head_dim)))
            for p in keys:
                store[l].setdefault(p, zero)
        else:
            keys = ctx + [s + j for j in range(R_new + 1)]
        for p in keys:
            assert p in store[l], f"layer {l} position {p} read before written"
        xs = bb.mlp(l, bb.o_proj(l, xs, _attn(bb, cfg, qs, store[l], keys)))
        if variant == "fresh_evicted":
            xp = bb.mlp(l, bb.o_proj(l, xp, _attn(bb, cfg, qp, store[l], keys)))
    rows = [n for n, j in enumerate(S) if j in set(rec.M)]
    return bb.logits(xs[rows]) if rows else np.zeros((0, cfg.vocab))


def test_masking_oracle_explicit_key_sets():
    run = get_config("C1").with_(model=MODEL, method=MethodConfig(block_size=8), prompt_len=7, gen_len=24)
    eng = OracleEngine(run, "ref")
    prompt = request_prompts(run)[0]
    eng.kv_append(0, prompt, run.gen_len)
    # the explicit store starts from the prompt's exact KV (prefill is pinned by KV exactness)
    store = {l: {p: (eng.K[0][l][p].copy(), eng.V[0][l][p].copy()) for p in range(len(prompt))}
             for l in range(MODEL.n_layers)}
    written_at = {}                          # (layer, pos) -> step of last write, for layers >= 2
    seen = dict(short_extent=0, stale_read=0, extent_sensitive=0, stale_sensitive=0)
    st = eng.req[0]
    while not st.finished:
        s_before, t_next = st.s, st.t + 1
        rec = eng.step_one(0)
        # the engine has already advanced its own state; recompute from the request state of the step
        st_saved = (st.s, st.R, list(st.tok))
        R_before = st.R
        if rec.M:
            alt_B = _brute_step(eng, 0, rec, store, "extent_B")
            alt_fresh = _brute_step(eng, 0, rec, store, "fresh_evicted")
        got = _brute_step(eng, 0, rec, store, "paper")
        assert st_saved == (st.s, st.R, list(st.tok))
        fin = np.isfinite(got)
        assert np.array_equal(fin, np.isfinite(rec.logits))
        if got.size:
            assert np.max(np.abs(got[fin] - rec.logits[fin])) < 1e-10
        # what the step exercised
        stale = [j for j in rec.P if j not in rec.S and j <= rec.R_new]
        if rec.M and rec.R_new < st.B - 1:
            seen["short_extent"] += 1
            if np.max(np.abs(alt_B[fin] - rec.logits[fin])) > 1e-6:
                seen["extent_sensitive"] += 1
        if rec.M and any((2, s_before + j) in written_at for j in stale):
            seen["stale_read"] += 1
            if np.max(np.abs(alt_fresh[fin] - rec.logits[fin])) > 1e-6:
                seen["stale_sensitive"] += 1
        for j in rec.S:
            written_at[(2, s_before + j)] = t_next
        assert R_before == st.R
        com = eng.commit_one(0)
        # evicted positions stay masked (north_star invariant)
        assert set(com.decoded) <= set(rec.S) & set(rec.M)
    assert seen["short_extent"] > 0 and seen["extent_sensitive"] > 0, seen
    assert seen["stale_read"] > 0 and seen["stale_sensitive"] > 0, seen
