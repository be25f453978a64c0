"""Dense numeric primitives of the oracle (binary64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import math

import numpy as np


def bf16_round(x) -> np.ndarray:
    """Round to the nearest bf16 (ties to even), returned as float64.

    Emulates the GPU's storage points: the GPU
    holds an fp32 value and stores its bf16 rounding, so we round fp64 -> fp32
    (nearest) first, then fp32 -> bf16 by the IEEE round-half-even rule on the
    upper 16 bits.
    """
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    b = (b + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def f32(x) -> np.ndarray:
    """Round to fp32 (the GPU's residual-stream / accumulator storage type)."""
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def softmax(v: np.ndarray) -> np.ndarray:
    """Row softmax with max subtraction (Eq.2 "Softmax")."""
    v = np.asarray(v, dtype=np.float64)
    m = np.max(v, axis=-1, keepdims=True)
    e = np.exp(v - m)
    return e / np.sum(e, axis=-1, keepdims=True)


def maxpool1d_same(v, kernel: int) -> np.ndarray:
    """MaxPool1D, stride 1, 'same' length, out-of-range = -inf (Eq.2; k=3 P:941;
    edges per SPEC S:46-53, reading A-I5).  Written as the window loop."""
    if kernel < 1 or kernel % 2 == 0:
        raise ValueError("maxpool kernel must be odd and >= 1")
    v = np.asarray(v, dtype=np.float64)
    n = v.shape[-1]
    r = kernel // 2
    out = np.empty_like(v)
    for j in range(n):
        lo, hi = max(0, j - r), min(n, j + r + 1)
        out[..., j] = np.max(v[..., lo:hi], axis=-1)
    return out


def rms_norm(x: np.ndarray, gain: np.ndarray, eps: float) -> np.ndarray:
    """x / sqrt(mean(x^2) + eps) * gain per row (SURVEY c.1)."""
    x = np.asarray(x, dtype=np.float64)
    ms = np.mean(x * x, axis=-1, keepdims=True)
    return x / np.sqrt(ms + eps) * gain


def rope(x: np.ndarray, positions, theta: float) -> np.ndarray:
    """Rotary embedding, rotate-half pairing (k, k + d/2), angle pos * theta^(-2k/d)
    (SURVEY c.1; standard RoPE).  x: [n, H, d] or [n, d]; positions: [n]."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    if d % 2:
        raise ValueError("RoPE needs an even head dim")
    half = d // 2
    pos = np.asarray(positions, dtype=np.float64)
    inv = theta ** (-2.0 * np.arange(half, dtype=np.float64) / d)
    ang = pos[:, None] * inv[None, :]                       # [n, half]
    if x.ndim == 3:
        ang = ang[:, None, :]
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return x / (1.0 + np.exp(-x))


def attend(q: np.ndarray, K: np.ndarray, V: np.ndarray) -> np.ndarray:
    """Plain softmax attention of query rows q [n, d] over keys K [m, d], values V [m, d]:
    sum_j softmax_j(q.k_j / sqrt(d)) v_j (SURVEY c.1)."""
    d = q.shape[-1]
    s = (q @ K.T) / math.sqrt(d)
    return softmax(s) @ V
