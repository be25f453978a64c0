"""Pins for the CPU oracle against values the paper/SPEC print, hand-worked examples,
closed forms, invariants and brute force (CPU only, -m "not gpu").

Each pin targets a plausible mistake: dropped pooling, wrong softmax range, wrong
sign in the delta, sample-vs-population sigma, FP budget rounding, wrong tie
order, transposed predecessor rule, off-by-one in the DC+ neighbour rule ...
"""
import json
import math
import os
import random

import numpy as np
import pytest
import scipy.ndimage
import scipy.special

from oracle import focus as F
from oracle.numerics import attend, bf16_round, maxpool1d_same, rms_norm, rope, softmax
from synth.configs import (CACHE_DC, CACHE_DC_PLUS, CACHE_NONE, PLACEHOLDER_ALL_MASKED,
                           PLACEHOLDER_UNPROCESSED_ONLY, STRATEGY_FIXED_TOP, STRATEGY_NONE)

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


# ----------------------------------------------------------------- primitives
def test_softmax_pins():
    p = G["softmax_0444"]
    np.testing.assert_allclose(softmax(np.array(p["in"], float)), p["out"], atol=p["tol"])
    p = G["softmax_big"]
    np.testing.assert_allclose(softmax(np.array(p["in"], float)), p["out"], atol=p["tol"])


def test_maxpool_pins():
    p = G["maxpool_k3"]
    assert maxpool1d_same(np.array(p["in"], float), 3).tolist() == p["out"]
    v = np.random.default_rng(0).normal(size=9)
    assert np.array_equal(maxpool1d_same(v, 1), v)                       # k=1 identity
    assert maxpool1d_same(np.array([5.0]), 3).tolist() == [5.0]
    with pytest.raises(ValueError):
        maxpool1d_same(v, 2)
    # library routine with -inf padding (independent implementation)
    for k in (3, 5):
        ref = scipy.ndimage.maximum_filter1d(v, size=k, mode="constant", cval=-np.inf)
        assert np.array_equal(maxpool1d_same(v, k), ref)


def test_rope_properties():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(3, 2, 8))
    assert np.allclose(rope(x, [0, 0, 0], 1e4), x, atol=1e-15)           # position 0 identity
    y = rope(x, [5, 17, 1234], 1e4)
    n_in = x[..., :4] ** 2 + x[..., 4:] ** 2
    n_out = y[..., :4] ** 2 + y[..., 4:] ** 2
    assert np.allclose(n_in, n_out, atol=1e-10)                           # pair norm
    q, k = rng.normal(size=(1, 8)), rng.normal(size=(1, 8))
    d1 = (rope(q, [3], 1e4) @ rope(k, [1], 1e4).T).item()
    d2 = (rope(q, [7], 1e4) @ rope(k, [5], 1e4).T).item()
    assert abs(d1 - d2) < 1e-10                                           # relative offset
    # rotate-half pairing: pair (0, d/2) rotated by pos*theta^0 = pos radians
    e = np.zeros((1, 8)); e[0, 0] = 1.0
    r = rope(e, [1], 1e4)
    assert abs(r[0, 0] - math.cos(1.0)) < 1e-15 and abs(r[0, 4] - math.sin(1.0)) < 1e-15


def test_rmsnorm_pins():
    assert np.allclose(rms_norm(np.ones((1, 4)), 1.0, 1e-6), np.ones((1, 4)), atol=1e-3)
    assert np.array_equal(rms_norm(np.zeros((1, 4)), 1.0, 1e-6), np.zeros((1, 4)))
    x = np.random.default_rng(2).normal(size=(4, 8))
    y = rms_norm(x, 1.0, 0.0)
    for i in range(4):                                                    # scalar-loop oracle
        ms = sum(float(t) * float(t) for t in x[i]) / 8
        assert np.allclose(y[i], [float(t) / math.sqrt(ms) for t in x[i]], atol=1e-12)


def test_bf16_round():
    assert bf16_round(1.0) == 1.0
    assert bf16_round(1.0 + 2 ** -8) == 1.0                 # tie -> even (mantissa 0)
    assert bf16_round(1.0 + 3 * 2 ** -8) == 1.0 + 2 ** -6   # tie -> even (round up)
    assert bf16_round(1.0 + 2 ** -7) == 1.0 + 2 ** -7       # representable
    assert bf16_round(-(1.0 + 1.5 * 2 ** -7)) == -(1.0 + 2 ** -6)


def test_attention_brute_force():
    rng = np.random.default_rng(3)
    q, K, V = rng.normal(size=(3, 4)), rng.normal(size=(5, 4)), rng.normal(size=(5, 4))
    out = attend(q, K, V)
    for i in range(3):
        s = [sum(q[i, t] * K[j, t] for t in range(4)) / 2.0 for j in range(5)]
        m = max(s)
        e = [math.exp(v - m) for v in s]
        z = sum(e)
        ref = [sum(e[j] / z * V[j, t] for j in range(5)) for t in range(4)]
        assert np.allclose(out[i], ref, atol=1e-12)
    assert np.allclose(attend(q, K[:1], V[:1]), np.repeat(V[:1], 3, 0))  # single key -> its value
    assert np.allclose(attend(np.zeros((1, 4)), K, V), V.mean(0, keepdims=True))


# ----------------------------------------------------------------- Eq.2 importance
def test_importance_single_row_spec():
    p = G["importance_single_row"]
    sc = np.zeros((1, 4, 4)); sc[0, 0] = p["row"]
    I = F.importance_from_scores(sc, range(4), p["k"], rows=[0])
    np.testing.assert_allclose(I, p["out"], atol=p["tol"])


def test_importance_4x4_hand():
    p = G["importance_4x4"]
    I = F.importance_from_scores(np.array([p["scores"]], float), range(4), p["k"])
    np.testing.assert_allclose(I, p["out"], atol=p["tol"])
    assert abs(I.sum() - 4.0) < 1e-12


def test_importance_committed_column():
    p = G["importance_committed_col"]
    sc = np.zeros((1, 4, 4)); sc[0, 0] = p["row"]
    I = F.importance_from_scores(sc, p["P"], p["k"], rows=[0])
    np.testing.assert_allclose(I, p["out"], atol=p["tol"])


def _importance_library(scores, P, k):
    """Independent implementation from library routines (scipy filter + softmax)."""
    H, B, _ = scores.shape
    mask = np.full(B, -np.inf); mask[list(P)] = 0.0
    I = np.zeros(B)
    for h in range(H):
        a = scores[h][list(P)] + mask[None, :]
        p = scipy.ndimage.maximum_filter1d(a, size=k, axis=1, mode="constant", cval=-np.inf)
        p[:, mask == -np.inf] = -np.inf
        I += scipy.special.softmax(p, axis=1).sum(0)
    return I


def test_importance_brute_force_and_invariants():
    rng = np.random.default_rng(4)
    for trial in range(60):
        H, B = 4, 8
        sc = rng.normal(size=(H, B, B)) * 3
        P = sorted(rng.choice(B, size=rng.integers(1, B + 1), replace=False).tolist())
        for k in (1, 3, 5):
            I = F.importance_from_scores(sc, P, k)
            np.testing.assert_allclose(I, _importance_library(sc, P, k), atol=1e-9)
            assert abs(I.sum() - len(P) * H) < 1e-9
            assert all(I[j] == 0 for j in range(B) if j not in P)
        one = np.repeat(sc[:1], H, 0)                                  # H identical heads -> xH
        np.testing.assert_allclose(F.importance_from_scores(one, P, 3),
                                   H * F.importance_from_scores(sc[:1], P, 3), atol=1e-9)
    # k=1 reduces to column sums of a plain row softmax over P (textbook special case)
    sc = rng.normal(size=(2, 6, 6)); P = [0, 1, 3, 4]
    ref = sum(scipy.special.softmax(sc[h][np.ix_(P, P)], axis=1).sum(0) for h in range(2))
    np.testing.assert_allclose(F.importance_from_scores(sc, P, 1)[P], ref, atol=1e-12)


def test_block_scores_gqa():
    rng = np.random.default_rng(5)
    q, k = rng.normal(size=(3, 4, 8)), rng.normal(size=(3, 2, 8))
    s = F.block_scores(q, k, 2)
    for h in range(4):
        for i in range(3):
            for j in range(3):
                assert abs(s[h, i, j] - sum(q[i, h, t] * k[j, h // 2, t] for t in range(8)) / math.sqrt(8)) < 1e-12


# ----------------------------------------------------------------- Eq.3-5
def test_delta_pin():
    p = G["delta"]
    assert F.delta(p["l0"], p["l1"]) == p["out"]
    assert F.delta([0.3, 0.7], [0.3, 0.7]) == [0.0, 0.0]


def test_n_sigma_pins():
    p = G["n_sigma"]
    ns, mu, sg = F.n_sigma(p["delta"], range(4))
    assert (ns, mu) == (p["count"], p["mu"]) and abs(sg * sg - p["sigma2"]) < 1e-15
    assert F.n_sigma([0.5] * 5, range(5))[0] == 5                         # sigma = 0
    assert F.n_sigma([0.5, 9.0], [1])[0] == 1                             # single masked
    assert F.n_sigma([9.0, 1.0, 2.0, 3.0], [1, 2, 3])[0] == 1             # masked only (A-S2)
    # population (not sample) sigma: [0, 1]: pop sigma 0.5 -> 1 >= 1.0 counts; sample 0.707 -> 1 < 1.207
    assert F.n_sigma([0.0, 1.0], [0, 1])[0] == 1
    rng = random.Random(6)                                                # brute force
    for _ in range(2000):
        n = rng.randint(1, 12)
        v = [rng.choice([-1.0, -0.5, 0.0, 0.25, 1.0, rng.uniform(-1, 1)]) for _ in range(n)]
        mu = math.fsum(v) / n
        sd = math.sqrt(math.fsum((x - mu) ** 2 for x in v) / n)
        ref = sum(1 for x in v if x >= mu + sd)
        ns = F.n_sigma(v, range(n))[0]
        assert abs(ns - ref) <= sum(1 for x in v if abs(x - (mu + sd)) < 1e-12)


def test_budget_pins():
    for p in G["budget"]:
        K, _ = F.budget(p["alpha"][0], p["alpha"][1], p["token_sum"], p["total_steps"], p["n_sigma"], p["B"])
        assert K == p["K"], p
    rng = random.Random(7)
    from fractions import Fraction
    for _ in range(10000):                                                # exact one-line oracle
        an, ad = rng.randint(2, 40), rng.randint(1, 20)
        if an <= ad:
            continue
        T, N, ns, B = rng.randint(0, 500), rng.randint(0, 100), rng.randint(0, 64), rng.randint(1, 64)
        nb = Fraction(T, N) if N else Fraction(1)
        ref = min(B, max(math.ceil(Fraction(an, ad) * nb), ns))
        assert F.budget(an, ad, T, N, ns, B)[0] == ref


def test_stats_mean_pin():
    p = G["stats_mean"]
    T, N = sum(p["yields"]), len(p["yields"])
    assert F.k_hist(1, 1, T, N) == math.ceil(p["mean"]) and T / N == p["mean"]


# ----------------------------------------------------------------- Alg.1 selection
def test_select_spec_trace():
    p = G["select_spec_trace"]
    d = [0.0] * p["B"]; d[p["top1"]] = 1.0
    sel = F.select(d, p["M"], p["U"], set(p["committed"]), p["R"], 0, 0, p["B"],
                   strategy=STRATEGY_FIXED_TOP, fixed_k=1)
    assert sorted(sel.S) == p["S"]
    assert sel.provenance[6] == "topk" and sel.provenance[4] == "uncached_decoded"


def test_select_hand():
    p = G["select_hand"]
    d = [0.0] * p["B"]
    for j, v in p["delta"].items():
        d[int(j)] = v
    sel = F.select(d, p["M"], p["U"], set(p["committed"]), p["R"], p["token_sum"], p["total_steps"], p["B"],
                   p["alpha"][0], p["alpha"][1])
    assert sel.mu == p["mu"] and abs(sel.sigma ** 2 - p["var"]) < 1e-15
    assert (sel.n_sigma, sel.k_hist, sel.K) == (p["n_sigma"], p["k_hist"], p["K"])
    assert sel.candidates == p["C"] and sorted(sel.S) == p["S"] and max(sel.S) == p["R_new"]
    # all_masked placeholder mode adds every masked j < max(S) (Alg.1 literal)
    sel2 = F.select(d, p["M"], p["U"], set(p["committed"]), p["R"], p["token_sum"], p["total_steps"], p["B"],
                    p["alpha"][0], p["alpha"][1], placeholder_mode=PLACEHOLDER_ALL_MASKED)
    assert sorted(sel2.S) == p["S"]


def test_select_limits():
    d = [0.1 * j for j in range(8)]
    sel = F.select(d, [0, 2, 3, 5, 6, 7], [1, 4], set(), 4, 0, 0, 8, strategy=STRATEGY_NONE)
    assert sorted(sel.S) == list(range(8))                          # K >= |M| => S = P
    sel = F.select([0.0], [0], [], set(), -1, 0, 0, 1, strategy=STRATEGY_FIXED_TOP, fixed_k=1)
    assert sorted(sel.S) == [0]
    # ties: lower index first; +0 and -0 are equal (A-E1)
    sel = F.select([0.0, -0.0, 0.0, 0.5], [0, 1, 2, 3], [], set(), -1, 0, 0, 4, strategy=STRATEGY_FIXED_TOP, fixed_k=2)
    assert sel.candidates == [3, 0]
    sel = F.select([-0.0, 0.0, 0.0, -1.0], [0, 1, 2, 3], [], set(), -1, 0, 0, 4, strategy=STRATEGY_FIXED_TOP, fixed_k=2)
    assert sel.candidates == [0, 1]


def test_select_closure_random():
    rng = random.Random(8)
    for _ in range(4000):
        B = rng.randint(1, 16)
        committed = set(j for j in range(B) if rng.random() < 0.2)
        P = [j for j in range(B) if j not in committed]
        if not P:
            continue
        M = [j for j in P if rng.random() < 0.7]
        if not M:
            continue
        U = [j for j in P if j not in M]
        R = rng.randint(-1, B - 1)
        d = [rng.choice([0.0, 0.25, -0.25, rng.uniform(-1, 1)]) for _ in range(B)]
        mode = rng.choice([PLACEHOLDER_UNPROCESSED_ONLY, PLACEHOLDER_ALL_MASKED])
        sel = F.select(d, M, U, committed, R, rng.randint(0, 30), rng.randint(0, 10), B,
                       rng.randint(2, 9), rng.randint(1, 2), placeholder_mode=mode)
        S = sel.S
        assert S and S <= set(P)                                              # non-empty, within P
        assert set(U) <= S                                                    # uncached decoded kept
        assert len(sel.candidates) == min(sel.K, len(M))
        for i in sel.candidates:                                              # predecessor closure
            assert i == 0 or (i - 1) in S or (i - 1) in committed
        mx = max(set(sel.candidates) | {i - 1 for i in sel.candidates if i > 0 and i - 1 not in committed} | {-1})
        for j in M:                                                           # placeholder closure
            if j < mx and (mode == PLACEHOLDER_ALL_MASKED or j > R):
                assert j in S
        others = [j for j in M if j not in sel.candidates]                    # top-K by (-d, j)
        for i in sel.candidates:
            for j in others:
                assert (-d[i], i) < (-d[j], j)


def test_compact_pin():
    p = G["compact"]
    rows, offs = F.compact([set(p["S"])])
    assert {str(j): n for n, (_, j) in enumerate(rows)} == p["map"]
    rows, offs = F.compact([{0, 2}, set(), {1, 3, 5}])
    assert rows == [(0, 0), (0, 2), (2, 1), (2, 3), (2, 5)] and offs == [0, 2, 2, 5]


# ----------------------------------------------------------------- decode / commit
def test_confidence_and_decide():
    tok, c = F.confidence(np.zeros(4))
    assert (tok, c) == (0, G["confidence_uniform"]["conf"])
    z = np.zeros(8); z[5] = 50.0
    tok, c = F.confidence(z)
    assert tok == 5 and abs(c - 1.0) < 1e-20
    z = np.array([1.0, 3.0, 3.0, -np.inf])
    tok, c = F.confidence(z)
    assert tok == 1 and abs(c - 1 / (2 + math.exp(-2))) < 1e-15
    assert F.decide({0: 0.2, 3: 0.5, 5: 0.5}, 0.9) == [3]            # fallback, ties lowest
    assert F.decide({1: 0.95, 2: 0.91, 4: 0.3}, 0.9) == [1, 2]       # both above
    assert F.decide({1: 0.9}, 0.9) == [1]                            # >= threshold
    assert F.decide({1: 0.999}, 1.0) == [1]                          # tau = 1 falls back


def _commit_times_closed_form(dstep, B):
    """Straight-line DC+ commit step of each position from the full event history:
    j < B-1: max(dstep[j] + 1, dstep[j+1]); j = B-1: max(dstep[j] + 1, max_j' dstep[j'])."""
    last = max(dstep)
    return [max(dstep[j] + 1, dstep[j + 1]) if j < B - 1 else max(dstep[j] + 1, last) for j in range(B)]


def _simulate(dsteps, B, mode):
    committed, timeline = set(), {}
    t_end = max(dsteps) + 1
    for t in range(1, t_end + 1):
        ds = [d if d <= t else None for d in dsteps]
        P = [j for j in range(B) if j not in committed]
        new = F.kv_commit(ds, committed, P, t, B, mode)
        committed |= new
        timeline[t] = new
    return timeline, committed


def test_dcplus_trace_and_random():
    p = G["dcplus_trace"]
    B = p["B"]
    ds = [p["decode_steps"][str(j)] for j in range(B)]
    tl, com = _simulate(ds, B, CACHE_DC_PLUS)
    assert {str(t): sorted(v) for t, v in tl.items()} == p["commits"] and com == set(range(B))
    rng = random.Random(9)
    for _ in range(10000):
        B = rng.randint(1, 8)
        ds = [rng.randint(1, B + 2) for _ in range(B)]
        tl, com = _simulate(ds, B, CACHE_DC_PLUS)
        assert com == set(range(B))
        when = {j: t for t, v in tl.items() for j in v}
        assert [when[j] for j in range(B)] == _commit_times_closed_form(ds, B)
        tl_dc, _ = _simulate(ds, B, CACHE_DC)
        cum_p, cum_d = set(), set()
        for t in sorted(tl):                                             # DC+ subset of DC
            cum_p |= tl[t]; cum_d |= tl_dc.get(t, set())
            assert cum_p <= cum_d
        tl_none, _ = _simulate(ds, B, CACHE_NONE)                        # NONE: all at max+1
        assert {j for t, v in tl_none.items() for j in v if t == max(ds) + 1} == set(range(B))


def test_integrated_scripted_trace():
    from oracle.engine import OracleEngine
    from synth import get_config
    p = G["integrated_trace"]
    run = get_config("C1")
    eng = OracleEngine(run)
    eng.set_context_kv(0, 4, 8, [np.zeros((4, 4, 16))] * 2, [np.zeros((4, 4, 16))] * 2)
    eng.script = {}
    for sp in p["steps"]:
        if not sp.get("flush"):
            eng.script[(0, sp["t"])] = {"dI": {int(k): v for k, v in sp["dI"].items()},
                                        "conf": {int(k): v for k, v in sp["conf"].items()},
                                        "tok": {int(k): 7 for k in sp["conf"]}}
    for sp in p["steps"]:
        rec = eng.step_one(0)
        com = eng.commit_one(0)
        assert rec.S == sp["S"], sp["t"]
        assert sorted(com.new_committed) == sp["commit"], sp["t"]
        if sp.get("flush"):
            assert rec.flush and com.block_done
            continue
        s = rec.sel
        assert abs(s.sigma - sp["sigma"]) < 1e-7
        assert (s.n_sigma, s.k_hist, s.K, s.candidates, rec.R_new, com.decoded) == \
            (sp["n_sigma"], sp["k_hist"], sp["K"], sp["C"], sp["R_new"], sp["D"])
    st = eng.req[0]
    assert [st.token_sum, st.total_steps] == p["final_stats"]
    assert st.R == -1 and st.committed == set() and st.s == 8 and st.output == [7, 7, 7, 7]
    # next block's first K_hist uses the persisted statistics: ceil(3/2 * 4/3) = 2
    assert F.k_hist(3, 2, st.token_sum, st.total_steps) == 2


def test_logit_scale_is_an_exact_power_of_two_scaling():
    """focus_config::logit_scale (SURVEY 8(b), A-M3 "logit_scale * W_lm"): a power-of-two scale of the
    recipe's LM-head weights, so z(s) = s * z(1) exactly and conf(s) = softmax max-prob at
    temperature 1/s; non-powers of two are rejected."""
    import dataclasses
    from oracle.model import Backbone, OracleWeights
    from synth.configs import ModelConfig
    from synth.gen import logit_scale_log2
    m1 = ModelConfig(n_layers=2, d_model=32, n_q_heads=2, n_kv_heads=1, head_dim=16, d_ff=64, vocab=41, rope_theta=1e4)
    m8 = dataclasses.replace(m1, logit_scale=8.0)
    w1, w8 = OracleWeights(m1).lm_head(), OracleWeights(m8).lm_head()
    assert np.array_equal(w8, 8.0 * w1)
    x = np.random.default_rng(0).standard_normal((3, 32))
    z1 = Backbone(m1, OracleWeights(m1), "gpu").logits(x)
    z8 = Backbone(m8, OracleWeights(m8), "gpu").logits(x)
    fin = np.isfinite(z1)
    assert np.array_equal(z8[fin], 8.0 * z1[fin])
    assert [logit_scale_log2(s) for s in (0, 1, 2, 0.5, 65536)] == [0, 0, 1, -1, 16]
    for bad in (3.0, 2.0 ** 20, -4.0):
        with pytest.raises(ValueError):
            logit_scale_log2(bad)
