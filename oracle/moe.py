"""Mixture-of-Experts FFN of the LLaDA2.0-mini-shaped workload.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md names the model (LLaDA2.0-mini, "a Mixture-of-Experts (MoE) DLLM with 16B total and 1.4B
active parameters") but not its FFN; the FOCUS method is unchanged on it (selection, compaction
and commit act on the rows; the FFN only changes what a row's layer computes).  Readings
(DESIGN.md A-M5, A-M6):

  A-M5  layers >= n_dense_layers: y = shared(h) + sum_{k < top_k} w_k * expert_{e_k}(h), h = RMSNorm(x),
        every expert (and the shared one) a SwiGLU (silu(h Wg^T) * (h Wu^T)) Wd^T of width d_expert.
  A-M6  router logits z = h W_r^T; the top_k experts by z, ties to the lower expert id (softmax is
        monotonic, so this is the top_k by router probability); weights = softmax over the selected
        logits only (= the full softmax renormalised over the selected experts).
"""
from __future__ import annotations

import math

import numpy as np


def route(z, top_k: int):
    """A-M6 on one row of router logits z [E]: returns [(expert, weight)] in selection order
    (logit descending, expert id ascending on ties)."""
    z = [float(v) for v in z]
    order = sorted(range(len(z)), key=lambda e: (-z[e], e))[:top_k]
    m = z[order[0]]
    ex = [math.exp(z[e] - m) for e in order]
    tot = sum(ex)
    return [(e, x / tot) for e, x in zip(order, ex)]


def swiglu(h: np.ndarray, wg: np.ndarray, wu: np.ndarray, wd: np.ndarray, rnd_f32=None, rnd_bf16=None):
    """(silu(h Wg^T) * (h Wu^T)) Wd^T with optional storage roundings (gpu emulation)."""
    f = rnd_f32 or (lambda a: a)
    b = rnd_bf16 or (lambda a: a)
    g = f(h @ wg.T)
    u = f(h @ wu.T)
    a = b(g / (1.0 + np.exp(-g)) * u)
    return f(a @ wd.T)
