"""Shared helpers of the GPU parity tests (feed the oracle the GPU's inputs, compare outputs)."""
from __future__ import annotations

import numpy as np

from oracle.engine import OracleEngine, RequestState

INT32_MAX = 0x7FFFFFFF


def bits(m: int, B: int) -> list:
    return [j for j in range(B) if (m >> j) & 1]


def oracle_state_from_gpu(g, rid: int, B: int, prompt_len: int) -> RequestState:
    st = RequestState(rid=rid, prompt=np.zeros(prompt_len, np.int32), gen_len=g.gen_len, B=B)
    st.s, st.b, st.R, st.t = g.s, g.b, g.R, g.t
    st.token_sum, st.total_steps = int(g.token_sum), int(g.total_steps)
    st.tok = list(g.tok[:B])
    st.dstep = [None if d == INT32_MAX else int(d) for d in g.dstep[:B]]
    st.committed = set(bits(g.committed, B))
    st.finished = bool(g.finished)
    return st


def gpu_importance_sums(raw: np.ndarray, counters, P_masks, n_kv_heads: int, B: int) -> np.ndarray:
    """I_j = sum over the request's partials (chunks that hold rows, kv heads) in the GPU's fixed
    order, in fp32 (part of 'feed the GPU's I').  counters[4] = rows per chunk, counters[5] = chunks."""
    rpc, n_chunks = int(counters[4]), int(counters[5])
    n_req = len(P_masks)
    parts = raw[: n_req * n_chunks * n_kv_heads * B].reshape(n_req, n_chunks * n_kv_heads, B).astype(np.float32)
    out = np.zeros((n_req, B), dtype=np.float32)
    for i, P in enumerate(P_masks):
        n_parts = ((bin(int(P)).count("1") + rpc - 1) // rpc) * n_kv_heads
        for p in range(n_parts):
            out[i] = (out[i] + parts[i, p, :]).astype(np.float32)
    return out


def rel_l2(a, b) -> float:
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
