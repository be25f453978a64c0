"""Counter-based generators for synthetic weights and prompts (inputs only).

Weight element (tensor t, flat index i of the logical [out][in] matrix):

    key = (t << 40) + i                       (i < 2**40)
    z   = key + (seed + 1) * 0x9E3779B97F4A7C15   (mod 2**64)
    u   = mix64(z)                            (splitmix64 finaliser)
    k   = u >> 56                             (0..255)
    w   = (2k - 255) * 2**e,  e = -ceil(log2(255 * sqrt(fan_in / 3)))

(2k-255) is odd with |.| <= 255, i.e. at most 8 significant bits, so every w is
exactly representable in bf16 and in fp32 (SURVEY
A-M3: uniform on about +-sqrt(3)*std with std ~ 1/sqrt(fan_in); no
transcendental per element, so CUDA and CPU agree bit for bit).  e is never at
a rounding boundary: 255^2 * fan_in / 3 = 3*5^2*17^2*fan_in is never a power
of 4, so log2(.) is never an integer.

Tensor ids: embedding E = 1, LM head W_lm = 2, prompt tokens = 3, prompt
lengths = 4; layer l: 16*(l+1) + {q:0, k:1, v:2, o:3, gate:4, up:5, down:6, router:7, shared
gate:8, shared up:9, shared down:10}; routed expert e of layer l: expert_tid(l, kind, e).
"""
from __future__ import annotations

import math

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

TID_EMBED = 1
TID_LMHEAD = 2
TID_PROMPT = 3
TID_PROMPT_LEN = 4
KIND = {"q": 0, "k": 1, "v": 2, "o": 3, "gate": 4, "up": 5, "down": 6, "router": 7, "sgate": 8, "sup": 9,
        "sdown": 10}
EXPERT_KIND = {"gate": 0, "up": 1, "down": 2}


def layer_tid(layer: int, kind: str) -> int:
    return 16 * (layer + 1) + KIND[kind]


def expert_tid(layer: int, kind: str, expert: int) -> int:
    """Tensor id of routed expert `expert` of MoE layer `layer` (kind gate / up / down): a separate id
    range 2^20 + (3 layer + kind) 2^12 + expert (tid < 2^24, so tid << 40 fits in 64 bits)."""
    return (1 << 20) + ((3 * layer + EXPERT_KIND[kind]) << 12) + expert


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def _stream(tid: int, start: int, count: int, seed: int) -> np.ndarray:
    idx = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = (np.uint64(tid) << np.uint64(40)) + np.uint64(seed + 1) * GOLDEN
        return mix64(idx + base)


def weight_scale_exp(fan_in: int) -> int:
    return -int(math.ceil(math.log2(255.0 * math.sqrt(fan_in / 3.0))))


_FAST = None


def _fast():
    """ctypes handle of synth/libsynthgen.so (same recipe in C + OpenMP), or None."""
    global _FAST
    if _FAST is None:
        import ctypes
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynthgen.so")
        try:
            if not os.path.exists(path):
                from .build_gen import build
                build()
            lib = ctypes.CDLL(path)
            lib.synth_weight_values.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                                ctypes.c_uint64, ctypes.c_int]
            _FAST = lib
        except Exception:
            _FAST = False
    return _FAST or None


def weight_values(tid: int, start: int, count: int, fan_in: int, seed: int = 0, fast: bool = True,
                  exp_offset: int = 0) -> np.ndarray:
    """Flat weight elements [start, start+count) of tensor `tid` as float32, times 2**exp_offset
    (a power-of-two scale keeps every value exact in bf16; used for the LM-head logit_scale)."""
    e = weight_scale_exp(fan_in) + exp_offset
    lib = _fast() if fast else None
    if lib is not None:
        out = np.empty(count, dtype=np.float32)
        lib.synth_weight_values(out.ctypes.data, tid, start, count, seed, e)
        return out
    u = _stream(tid, start, count, seed)
    k = (u >> np.uint64(56)).astype(np.int32)
    return np.ldexp((2 * k - 255).astype(np.float32), e).astype(np.float32)


def weight_matrix(tid: int, rows: int, cols: int, fan_in: int, seed: int = 0,
                  row_lo: int = 0, row_hi: int | None = None, chunk: int = 1 << 28,
                  exp_offset: int = 0) -> np.ndarray:
    """Rows [row_lo, row_hi) of the logical [rows][cols] matrix, float32."""
    row_hi = rows if row_hi is None else row_hi
    n = (row_hi - row_lo) * cols
    out = np.empty(n, dtype=np.float32)
    start = row_lo * cols
    for off in range(0, n, chunk):
        c = min(chunk, n - off)
        out[off:off + c] = weight_values(tid, start + off, c, fan_in, seed, exp_offset=exp_offset)
    return out.reshape(row_hi - row_lo, cols)


def logit_scale_log2(scale: float) -> int:
    """log2 of a power-of-two LM-head scale (focus_config::logit_scale; 0 means 1)."""
    if scale == 0:
        return 0
    m, e = math.frexp(scale)
    if m != 0.5 or not -15 <= e <= 17:
        raise ValueError(f"logit_scale must be a power of two in [2^-16, 2^16], got {scale}")
    return e - 1


def prompt_tokens(request_id: int, n: int, vocab: int) -> np.ndarray:
    """Prompt ids uniform over [0, vocab-1); the mask id is vocab-1 (A-M2)."""
    u = _stream(TID_PROMPT, 0, n, 1 + request_id)
    return (u % np.uint64(vocab - 1)).astype(np.int32)


def prompt_lengths(n_requests: int, lo: int, hi: int, seed: int = 7) -> np.ndarray:
    """Mixed prompt lengths uniform over [lo, hi] (C4)."""
    u = _stream(TID_PROMPT_LEN, 0, n_requests, seed)
    return (np.uint64(lo) + u % np.uint64(hi - lo + 1)).astype(np.int32)
