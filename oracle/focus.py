"""FOCUS method rules (§3-§4, Alg.1, App. E), written as plain Python.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Sets are Python sets / sorted lists of block positions j in [0, B).  Statistics
use Python floats (binary64, each operation rounded, no FMA), integer budget
arithmetic is exact.  The readings taken where the paper is silent are the
DESIGN.md ambiguity register (A-I*, A-S*, A-B*, A-E*, A-CF*, A-DC*).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from synth.configs import (CACHE_DC, CACHE_DC_PLUS, CACHE_NONE, PLACEHOLDER_ALL_MASKED,
                           PLACEHOLDER_UNPROCESSED_ONLY, STRATEGY_FIXED_BOTTOM,
                           STRATEGY_FIXED_RANDOM, STRATEGY_FIXED_TOP, STRATEGY_FOCUS,
                           STRATEGY_NONE)

from .numerics import maxpool1d_same


# ----------------------------------------------------------------------------- Eq.2
def importance_from_scores(scores: np.ndarray, P, kernel: int = 3, rows=None) -> np.ndarray:
    """Eq.2 (App.E Eq. appendix_importance, k=3 P:941):

        I_j = sum_{i in P} sum_h Softmax_j( MaxPool1D_j( S^{(h)}_{i,j} ) )

    scores: [H, B, B] pre-softmax scores S^{(h)}_{i,j} over the block (rows i, columns j).
    Readings: A-I2 softmax over intra-block keys only; A-I3 queries = keys = P, pooling on
    the block-position axis with columns outside P at -inf, softmax over P; A-I5 'same'
    pooling with -inf padding; A-I7 the query rows are all of P (`rows` overrides that only to
    reproduce SPEC's single-row example S:224).  Returns I [B] (0 outside P)."""
    scores = np.asarray(scores, dtype=np.float64)
    H, B, _ = scores.shape
    Pl = sorted(P)
    rows = Pl if rows is None else sorted(rows)
    I = np.zeros(B)
    for h in range(H):
        for i in rows:
            a = np.full(B, -np.inf)
            for j in Pl:
                a[j] = scores[h, i, j]
            p = maxpool1d_same(a, kernel)
            m = max(p[j] for j in Pl)
            e = {j: math.exp(p[j] - m) for j in Pl}
            z = sum(e[j] for j in Pl)
            for j in Pl:
                I[j] += e[j] / z
    return I


def block_scores(q: np.ndarray, k: np.ndarray, group: int) -> np.ndarray:
    """S^{(h)}_{i,j} = q_i^h . k_j^{floor(h/G)} / sqrt(d_h)  (reading A-I1: post-RoPE logits the
    attention softmax sees; A-I6: every query head, GQA kv head of its group).
    q: [B, Hq, dh], k: [B, Hkv, dh] -> [Hq, B, B]."""
    Hq, dh = q.shape[1], q.shape[2]
    out = np.empty((Hq, q.shape[0], k.shape[0]))
    for h in range(Hq):
        out[h] = (q[:, h, :] @ k[:, h // group, :].T) / math.sqrt(dh)
    return out


def importance(q: np.ndarray, k: np.ndarray, P, group: int, kernel: int = 3) -> np.ndarray:
    return importance_from_scores(block_scores(q, k, group), P, kernel)


# ----------------------------------------------------------------------------- Eq.3-5, Alg.1
@dataclass
class Selection:
    S: set
    K: int = 0
    n_sigma: int = 0
    k_hist: int = 0
    mu: float = 0.0
    sigma: float = 0.0
    candidates: list = field(default_factory=list)
    provenance: dict = field(default_factory=dict)


def delta(I0, I1) -> list:
    """Eq.3: dI_j = I^(L1)_j - I^(L0)_j, in the fp32 the importance is held in
    (DESIGN.md A-S4: dI_j = fl32(I1_j - I0_j))."""
    a = np.asarray(I1, dtype=np.float32)
    b = np.asarray(I0, dtype=np.float32)
    return [float(x) for x in (a - b).astype(np.float32)]


def stats_mean_std(values: list) -> tuple[float, float]:
    """Block-wise mean and population std of dI over masked positions (App.E P:779 "mu, sigma
    are the block-wise mean and standard deviation"; A-S2/A-S3/A-S4: masked only, /n, two-pass
    binary64 in ascending position order from +0.0)."""
    n = len(values)
    s = 0.0
    for v in values:
        s = s + v
    mu = s / n
    acc = 0.0
    for v in values:
        dv = v - mu
        acc = acc + dv * dv
    return mu, math.sqrt(acc / n)


def n_sigma(d: list, M) -> tuple[int, float, float]:
    """Eq.5 read as App.E's "dI > mu + sigma" with >= (reading A-S1):
    N_sigma = #{j in M : dI_j >= mu + sigma}."""
    Ml = sorted(M)
    if not Ml:
        return 0, 0.0, 0.0
    vals = [d[j] for j in Ml]
    mu, sg = stats_mean_std(vals)
    th = mu + sg
    return sum(1 for v in vals if v >= th), mu, sg


def k_hist(alpha_num: int, alpha_den: int, token_sum: int, total_steps: int) -> int:
    """ceil(alpha * N_bar) with N_bar = token_sum / total_steps (App.E, cumulative,
    reading A-B1), N_bar = 1 at the request's first step (Alg.1, A-B2).
    Exact rational arithmetic (A-B3)."""
    T, N = (token_sum, total_steps) if total_steps > 0 else (1, 1)
    num, den = alpha_num * T, alpha_den * N
    return -((-num) // den)


def budget(alpha_num, alpha_den, token_sum, total_steps, ns, B) -> tuple[int, int]:
    """Eq.4: K = min(B, max(ceil(alpha * N_bar), N_sigma))."""
    kh = k_hist(alpha_num, alpha_den, token_sum, total_steps)
    return min(B, max(kh, ns)), kh


def random_priority(request_id: int, step: int, j: int, seed: int) -> int:
    """Counter-based priority for the fixed-random strategy (tab:selection_strategy "Random").
    Same recipe as the CUDA side implements: mix64 of a packed counter."""
    from synth.gen import mix64, GOLDEN
    key = (np.uint64(request_id) << np.uint64(32)) | (np.uint64(step & 0xFFFFFF) << np.uint64(8)) | np.uint64(j)
    with np.errstate(over="ignore"):
        return int(mix64(np.array([key + np.uint64(seed + 1) * GOLDEN], dtype=np.uint64))[0])


def select(d: list, M, U, committed, R: int, token_sum: int, total_steps: int, B: int,
           alpha_num: int = 3, alpha_den: int = 2, placeholder_mode: int = PLACEHOLDER_UNPROCESSED_ONLY,
           strategy: int = STRATEGY_FOCUS, fixed_k: int = 0, request_id: int = 0, step: int = 0,
           seed: int = 0) -> Selection:
    """Alg.1 Phase 2-3, §4.2 constraints, App.E P:770-777.

    d: dI per block position (only masked entries are read); M masked, U decoded-uncommitted,
    committed: set of committed positions; R: rightmost processed (-1 at block open)."""
    Ml = sorted(M)
    n = len(Ml)
    sel = Selection(S=set())
    if n == 0:
        raise ValueError("select() needs at least one masked position (flush steps skip selection)")
    ns, mu, sg = n_sigma(d, Ml)
    sel.n_sigma, sel.mu, sel.sigma = ns, mu, sg
    if strategy == STRATEGY_FOCUS:
        K, kh = budget(alpha_num, alpha_den, token_sum, total_steps, ns, B)
        sel.k_hist = kh
    elif strategy == STRATEGY_NONE:
        K = B
    else:
        K = fixed_k
    sel.K = K
    Kp = min(K, n)
    # TopK_Indices (Alg.1): order by (dI descending, j ascending)  (A-E1)
    if strategy == STRATEGY_FIXED_BOTTOM:
        order = sorted(Ml, key=lambda j: (d[j], j))
    elif strategy == STRATEGY_FIXED_RANDOM:
        order = sorted(Ml, key=lambda j: (random_priority(request_id, step, j, seed), j))
    else:
        order = sorted(Ml, key=lambda j: (-d[j], j))
    C = order[:Kp]
    sel.candidates = list(C)
    S = set(C)
    prov = {j: "topk" for j in C}
    # AR-Context Preservation (Alg.1): predecessor of each candidate, unless
    # it is committed (its KV is final and referable; A-E2)
    for i in C:
        if i > 0 and (i - 1) not in committed:
            if (i - 1) not in S:
                prov[i - 1] = "predecessor"
            S.add(i - 1)
    # Placeholder Integrity (Alg.1; App.E) (A-E3)
    mx = max(S) if S else -1       # C can only be empty if K' = 0 (invalid alpha / stats)
    for j in Ml:
        if j < mx and (placeholder_mode == PLACEHOLDER_ALL_MASKED or j > R):
            if j not in S:
                prov[j] = "placeholder"
            S.add(j)
    # decoded-but-uncommitted positions are re-forwarded until committed (A-E4)
    for j in U:
        if j not in S:
            prov[j] = "uncached_decoded"
        S.add(j)
    # Minimum Retention Guarantee |S| >= 1; unreachable since n >= 1 (A-E6)
    if not S:
        S.add(order[0])
        prov[order[0]] = "min_retention"
    sel.S, sel.provenance = S, prov
    return sel


def compact(S_per_request: list) -> tuple[list, list]:
    """Order-preserving gather map ("Gather"; App.E P:781-782 prefix-sum):
    row(r, j) = sum_{r'<r} |S_r'| + #{j' in S_r : j' < j}.  Returns (rows, offsets) where rows is
    the list of (request index, j) in dense-row order."""
    rows, offs = [], [0]
    for r, S in enumerate(S_per_request):
        for j in sorted(S):
            rows.append((r, j))
        offs.append(len(rows))
    return rows, offs


# ----------------------------------------------------------------------------- decode / commit
def confidence(z: np.ndarray) -> tuple[int, float]:
    """Max softmax probability at temperature 1 and its argmax (Fast-dLLM style confidence
    decoding, reading A-CF1; argmax ties to the lowest id, A-CF4).  The mask id must
    already be -inf in z.  conf = 1 / sum_v exp(z_v - max)."""
    z = np.asarray(z, dtype=np.float64)
    m = float(np.max(z))
    tok = int(np.flatnonzero(z == m)[0])
    return tok, 1.0 / float(np.sum(np.exp(z - m)))


def decide(conf: dict, tau: float) -> list:
    """Decode_and_Verify (Alg.1): D = {i : conf_i >= tau}; if empty, the single best
    position, ties to the lowest position (A-CF2).  conf: {position: confidence}."""
    D = sorted(i for i, c in conf.items() if c >= tau)
    if not D and conf:
        best = max(conf.values())
        D = [min(i for i, c in conf.items() if c == best)]
    return D


def kv_commit(dstep: list, committed: set, P, t: int, B: int, cache_mode: int) -> set:
    """Intra-block KV cache commit at the end of step t (§4.3; App.E P:812-818,
    P:848-853).  dstep[j] = step at which j was decoded (None = still masked).

    DC+ (Neighbor-Aware Stability, reading A-DC1/A-DC3): commit j in P iff decoded at an
        earlier step (forwarded once after decoding) and (j < B-1 ? its right neighbour is
        decoded (by step t) : the whole block is decoded).
    DC: commit iff decoded at an earlier step.
    NONE (A-DC5): nothing until the whole block is decoded and forwarded once more."""
    dec = lambda j, by: dstep[j] is not None and dstep[j] <= by  # noqa: E731
    new = set()
    if cache_mode == CACHE_NONE:
        if all(dec(j, t - 1) for j in range(B)):
            new = set(P)
        return new
    for j in P:
        if j in committed or not dec(j, t - 1):
            continue
        if cache_mode == CACHE_DC:
            new.add(j)
        elif j < B - 1:
            if dec(j + 1, t):
                new.add(j)
        elif all(dec(jj, t) for jj in range(B)):
            new.add(j)
    return new
