"""Pins of the oracle's MoE FFN (LLaDA2.0-mini-shaped workload; readings A-M5, A-M6).

- Routing (A-M6) on hand-worked logits: top-k by logit, ties to the lower expert id, weights the
  softmax over the selected logits; top_k = E reduces to the full softmax (closed form).
- Identical routed experts make the MoE FFN a dense SwiGLU (the weights sum to 1): the MoE layer
  equals the oracle's dense layer built from the same matrices plus the shared expert.
- Brute force: every expert evaluated for every row and gated by its routing weight (0 if unselected).
- The LLaDA2.0-mini shape of reading A-M5 has 16.3B total / 1.43B active parameters, the paper's
  "16B total and 1.4B active".
"""
import dataclasses
import math

import numpy as np
import pytest

from oracle import moe as MOE
from oracle.model import Backbone, OracleWeights
from oracle.numerics import rms_norm
from synth import get_config
from synth.configs import ModelConfig

TINY_MOE = ModelConfig(n_layers=3, d_model=64, n_q_heads=4, n_kv_heads=2, head_dim=16, d_ff=128, vocab=37,
                       rope_theta=1e4, n_experts=8, top_k=2, d_expert=32, n_shared_experts=1, n_dense_layers=1)


def test_route_hand_worked():
    r = MOE.route([1.0, 3.0, 3.0, 0.0], 2)
    assert [e for e, _ in r] == [1, 2] and all(abs(w - 0.5) < 1e-15 for _, w in r)
    r = MOE.route([2.0, 1.0, 1.0, 0.0], 2)                  # tie for the second place: lower id
    assert [e for e, _ in r] == [0, 1]
    w0 = 1.0 / (1.0 + math.exp(-1.0))                        # softmax([2, 1])
    assert abs(r[0][1] - w0) < 1e-15 and abs(r[1][1] - (1 - w0)) < 1e-15
    z = [0.3, -1.2, 2.5, 0.0, 0.7]
    full = dict(MOE.route(z, len(z)))                        # top_k = E: the full softmax
    ez = np.exp(np.array(z) - max(z))
    assert all(abs(full[e] - ez[e] / ez.sum()) < 1e-15 for e in range(len(z)))
    assert abs(sum(w for _, w in MOE.route(z, 3)) - 1.0) < 1e-15


def _same_experts(w, e0=0):
    w = dict(w)
    w["experts"] = [w["experts"][e0]] * len(w["experts"])
    return w


def test_identical_experts_reduce_to_dense():
    x = np.random.default_rng(3).standard_normal((5, TINY_MOE.d_model))
    W = OracleWeights(TINY_MOE)
    l = 1
    w = _same_experts(W.layer(l))
    W._layers[l] = w
    got = Backbone(TINY_MOE, W, "ref").moe(l, x)
    # dense layer with the expert's matrices (the oracle's dense path), plus the shared expert
    dense_cfg = dataclasses.replace(TINY_MOE, n_experts=0, d_ff=TINY_MOE.d_expert)
    Wd = OracleWeights(dense_cfg)
    ex = w["experts"][0]
    Wd._layers[l] = {**{k: w[k] for k in ("q", "k", "v", "o")}, "gate": ex["gate"], "up": ex["up"], "down": ex["down"]}
    want = Backbone(dense_cfg, Wd, "ref").mlp(l, x)
    h = rms_norm(x, 1.0, TINY_MOE.rms_eps)
    g, u = h @ w["sgate"].T, h @ w["sup"].T
    want = want + (g / (1 + np.exp(-g)) * u) @ w["sdown"].T
    assert np.max(np.abs(got - want)) < 1e-12


def test_moe_brute_force_all_experts():
    x = np.random.default_rng(4).standard_normal((6, TINY_MOE.d_model))
    W = OracleWeights(TINY_MOE)
    l = 2
    w = W.layer(l)
    got = Backbone(TINY_MOE, W, "ref").moe(l, x)
    h = rms_norm(x, 1.0, TINY_MOE.rms_eps)
    z = h @ w["router"].T
    out = x.copy()
    g, u = h @ w["sgate"].T, h @ w["sup"].T
    out += (g / (1 + np.exp(-g)) * u) @ w["sdown"].T
    for n in range(x.shape[0]):
        # gate of every expert: its softmax weight among the top-k by (logit desc, id asc), else 0
        ranked = sorted(range(TINY_MOE.n_experts), key=lambda e: (-z[n, e], e))
        top = ranked[:TINY_MOE.top_k]
        ez = {e: math.exp(z[n, e] - z[n, top[0]]) for e in top}
        for e in range(TINY_MOE.n_experts):
            gate = ez[e] / sum(ez.values()) if e in top else 0.0
            ex = w["experts"][e]
            ge, ue = h[n] @ ex["gate"].T, h[n] @ ex["up"].T
            out[n] += gate * ((ge / (1 + np.exp(-ge)) * ue) @ ex["down"].T)
    assert np.max(np.abs(got - out)) < 1e-12


def test_llada2_mini_shape_matches_paper_parameter_counts():
    c = get_config("C6").model
    attn = c.n_layers * (c.d_model * c.qkv_dim + c.n_q_heads * c.head_dim * c.d_model)
    emb = 2 * c.vocab * c.d_model
    dense = c.n_dense_layers * 3 * c.d_model * c.d_ff
    per_expert = 3 * c.d_model * c.d_expert
    n_moe = c.n_layers - c.n_dense_layers
    total = attn + emb + dense + n_moe * ((c.n_experts + c.n_shared_experts) * per_expert + c.n_experts * c.d_model)
    active = attn + emb + dense + n_moe * ((c.top_k + c.n_shared_experts) * per_expert + c.n_experts * c.d_model)
    assert 15.5e9 < total < 16.5e9, total                    # "16B total"
    assert 1.35e9 < active < 1.45e9, active                  # "1.4B active"


@pytest.mark.parametrize("mode", ["ref", "gpu"], ids=["binary64", "storage_rounding"])
def test_moe_engine_runs_and_is_deterministic(mode):
    from oracle.engine import run_to_completion
    from synth.configs import MethodConfig
    run = get_config("C1").with_(model=TINY_MOE, method=MethodConfig(block_size=4), n_requests=2)
    a, _ = run_to_completion(run, mode)
    b, _ = run_to_completion(run, mode)
    assert a.req[0].output == b.req[0].output and len(a.req[1].output) == run.gen_len
