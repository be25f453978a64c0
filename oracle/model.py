"""The oracle's backbone: a Qwen3-like GQA transformer (SURVEY c.1, reading A-M1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md does not give the backbone (it evaluates SDAR, continually pre-trained
from an AR LLM).  Reading A-M1: pre-RMSNorm blocks,
q = h Wq^T, k = h Wk^T, v = h Wv^T, rotate-half RoPE on q and k at absolute
positions, GQA (q-head h uses kv-head floor(h/G)), x += attn(...) Wo^T,
x += (silu(h Wg^T) * (h Wu^T)) Wd^T, untied LM head, mask id = V-1 excluded
from the logits.  Norm gains are 1.

Two precisions:
  mode="ref": binary64 throughout.
  mode="gpu": binary64 arithmetic, but values are rounded at the GPU's storage
              points: bf16 for GEMM inputs
              (normed h, attention output, silu*mul), q and K/V; fp32 for the
              residual stream and the logits.  Emulation by specification,
              not shared code.
"""
from __future__ import annotations

import numpy as np

from synth.configs import ModelConfig
from synth.gen import (TID_EMBED, TID_LMHEAD, expert_tid, layer_tid, logit_scale_log2, weight_matrix)

from . import moe as MOE
from .numerics import attend, bf16_round, f32, rms_norm, rope, silu


class OracleWeights:
    """Weights regenerated from the synth counter hash (exact bf16 values, held as float64).

    Per-layer tensors are generated on first use; `cache=False` regenerates on every use
    (bounded memory for 8B-shaped models)."""

    def __init__(self, cfg: ModelConfig, seed: int = 0, cache: bool = True):
        self.cfg, self.seed, self.cache = cfg, seed, cache
        self._layers: dict[int, dict[str, np.ndarray]] = {}
        self._lm: np.ndarray | None = None

    def embed_rows(self, tokens) -> np.ndarray:
        c = self.cfg
        return np.stack([weight_matrix(TID_EMBED, c.vocab, c.d_model, c.d_model, self.seed, t, t + 1)[0]
                         for t in np.asarray(tokens).tolist()]).astype(np.float64) \
            if len(tokens) else np.zeros((0, c.d_model))

    def layer(self, l: int) -> dict[str, np.ndarray]:
        if l in self._layers:
            return self._layers[l]
        c = self.cfg
        d, hq, hkv, dh, ff = c.d_model, c.n_q_heads, c.n_kv_heads, c.head_dim, c.d_ff
        w = {
            "q": weight_matrix(layer_tid(l, "q"), hq * dh, d, d, self.seed),
            "k": weight_matrix(layer_tid(l, "k"), hkv * dh, d, d, self.seed),
            "v": weight_matrix(layer_tid(l, "v"), hkv * dh, d, d, self.seed),
            "o": weight_matrix(layer_tid(l, "o"), d, hq * dh, hq * dh, self.seed),
        }
        if c.is_moe_layer(l):
            # MoE FFN (reading A-M5): router [E][d], routed experts e: gate/up [de][d], down [d][de];
            # shared experts: gate/up [ns*de][d], down [d][ns*de]
            de, E, ns = c.d_expert, c.n_experts, c.n_shared_experts
            w["router"] = weight_matrix(layer_tid(l, "router"), E, d, d, self.seed)
            w["experts"] = [{k: weight_matrix(expert_tid(l, k, e), *(shape + (fan,)), self.seed).astype(np.float64)
                             for k, shape, fan in (("gate", (de, d), d), ("up", (de, d), d), ("down", (d, de), de))}
                            for e in range(E)]
            if ns:
                w["sgate"] = weight_matrix(layer_tid(l, "sgate"), ns * de, d, d, self.seed)
                w["sup"] = weight_matrix(layer_tid(l, "sup"), ns * de, d, d, self.seed)
                w["sdown"] = weight_matrix(layer_tid(l, "sdown"), d, ns * de, ns * de, self.seed)
        else:
            w["gate"] = weight_matrix(layer_tid(l, "gate"), ff, d, d, self.seed)
            w["up"] = weight_matrix(layer_tid(l, "up"), ff, d, d, self.seed)
            w["down"] = weight_matrix(layer_tid(l, "down"), d, ff, ff, self.seed)
        w = {k: (v.astype(np.float64) if k != "experts" else v) for k, v in w.items()}
        if self.cache:
            self._layers[l] = w
        return w

    def lm_head(self) -> np.ndarray:
        if self._lm is not None:
            return self._lm
        c = self.cfg
        # W_lm = logit_scale * recipe weights (a power of two: exact; focus_config::logit_scale)
        lm = weight_matrix(TID_LMHEAD, c.vocab, c.d_model, c.d_model, self.seed,
                           exp_offset=logit_scale_log2(c.logit_scale)).astype(np.float64)
        if self.cache:
            self._lm = lm
        return lm


class Backbone:
    """Layer pieces of the forward pass on a set of rows of ONE request."""

    def __init__(self, cfg: ModelConfig, weights: OracleWeights, mode: str = "ref"):
        assert mode in ("ref", "gpu")
        self.cfg, self.w, self.mode = cfg, weights, mode

    # storage-point rounding (identity in ref mode)
    def _bf(self, x):
        return bf16_round(x) if self.mode == "gpu" else np.asarray(x, dtype=np.float64)

    def _f32(self, x):
        return f32(x) if self.mode == "gpu" else np.asarray(x, dtype=np.float64)

    def embed(self, tokens) -> np.ndarray:
        """x_j = E[tok_j] (Alg.1 input "Masked Block X")."""
        return self.w.embed_rows(tokens)

    def qkv(self, l: int, x: np.ndarray, positions) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """RMSNorm, projections, RoPE at absolute positions.  Returns q [n,Hq,dh], k, v [n,Hkv,dh]."""
        c, w = self.cfg, self.w.layer(l)
        h = self._bf(rms_norm(x, 1.0, c.rms_eps))
        n = h.shape[0]
        q = (h @ w["q"].T).reshape(n, c.n_q_heads, c.head_dim)
        k = (h @ w["k"].T).reshape(n, c.n_kv_heads, c.head_dim)
        v = (h @ w["v"].T).reshape(n, c.n_kv_heads, c.head_dim)
        q = self._bf(rope(self._f32(q), positions, c.rope_theta))
        k = self._bf(rope(self._f32(k), positions, c.rope_theta))
        v = self._bf(v)
        return q, k, v

    def attention(self, q: np.ndarray, K: np.ndarray, V: np.ndarray) -> np.ndarray:
        """Each query row attends to ALL given keys (the caller builds the key set:
        block-diffusion = context + block extent, bidirectional inside the block).
        q [n,Hq,dh]; K, V [m,Hkv,dh] -> [n, Hq*dh]."""
        c = self.cfg
        out = np.empty((q.shape[0], c.n_q_heads, c.head_dim))
        for h in range(c.n_q_heads):
            g = h // c.group
            out[:, h, :] = attend(q[:, h, :], K[:, g, :], V[:, g, :])
        return self._bf(out.reshape(q.shape[0], -1))

    def attention_causal(self, q: np.ndarray, K: np.ndarray, V: np.ndarray, first_pos: int) -> np.ndarray:
        """Prefill: query row i (absolute position first_pos+i) attends to keys [0, first_pos+i]
        (exact AR-style KV; reading A-K5)."""
        c = self.cfg
        out = np.empty((q.shape[0], c.n_q_heads, c.head_dim))
        for i in range(q.shape[0]):
            lim = first_pos + i + 1
            for h in range(c.n_q_heads):
                g = h // c.group
                out[i, h, :] = attend(q[i:i + 1, h, :], K[:lim, g, :], V[:lim, g, :])[0]
        return self._bf(out.reshape(q.shape[0], -1))

    def o_proj(self, l: int, x: np.ndarray, o: np.ndarray) -> np.ndarray:
        """x + o Wo^T (residual stream fp32 in gpu mode)."""
        w = self.w.layer(l)
        return self._f32(x + self._f32(o @ w["o"].T))

    def mlp(self, l: int, x: np.ndarray) -> np.ndarray:
        """x + (silu(h Wg^T) * h Wu^T) Wd^T with h = RMSNorm(x); MoE layers: oracle/moe.py."""
        c, w = self.cfg, self.w.layer(l)
        if c.is_moe_layer(l):
            return self.moe(l, x)
        h = self._bf(rms_norm(x, 1.0, c.rms_eps))
        g = self._f32(h @ w["gate"].T)
        u = self._f32(h @ w["up"].T)
        a = self._bf(silu(g) * u)
        return self._f32(x + self._f32(a @ w["down"].T))

    def moe_route(self, l: int, x: np.ndarray):
        """Router of an MoE layer (A-M6): z = RMSNorm(x) W_r^T (fp32 in gpu mode) and each row's
        [(expert, weight)] selection."""
        c, w = self.cfg, self.w.layer(l)
        h = self._bf(rms_norm(x, 1.0, c.rms_eps))
        z = self._f32(h @ w["router"].T)
        return h, z, [MOE.route(z[n], c.top_k) for n in range(z.shape[0])]

    def moe(self, l: int, x: np.ndarray) -> np.ndarray:
        """x + shared(h) + sum_k w_k expert_{e_k}(h) (A-M5).  gpu mode rounding points: router logits,
        expert projections and outputs fp32, silu*mul bf16; the shared expert's output is added to the
        residual first, then the routed experts' weighted sum (selection order, fp32)."""
        c, w = self.cfg, self.w.layer(l)
        f = self._f32 if self.mode == "gpu" else None
        b = self._bf if self.mode == "gpu" else None
        h, z, sel = self.moe_route(l, x)
        x = np.asarray(x, dtype=np.float64)
        if c.n_shared_experts:
            x = self._f32(x + MOE.swiglu(h, w["sgate"], w["sup"], w["sdown"], f, b))
        out = np.empty_like(x)
        for n in range(x.shape[0]):
            acc = np.zeros(x.shape[1])
            for e, wt in sel[n]:
                ex = w["experts"][e]
                y = MOE.swiglu(h[n:n + 1], ex["gate"], ex["up"], ex["down"], f, b)[0]
                acc = self._f32(acc + self._f32(self._f32(wt) * y))
            out[n] = x[n] + acc
        return self._f32(out)

    def logits(self, x: np.ndarray) -> np.ndarray:
        """z = RMSNorm(x) W_lm^T; z[mask id] = -inf (A-CF1)."""
        c = self.cfg
        h = self._bf(rms_norm(x, 1.0, c.rms_eps))
        z = self._f32(h @ self.w.lm_head().T)
        z[:, c.mask_token_id] = -np.inf
        return z
