"""Workload configurations C1..C5 (BASELINE.json `configs`) as plain data.

Shapes beyond BASELINE.json (head_dim, d_ff, theta, eps, vocab for 8B) are the
SURVEY A-M1 readings; method defaults are SURVEY 8(d) (alpha=3/2, tau=0.9,
MaxPool k=3, DC+, unprocessed-only placeholders).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Optional

# enums shared with include/focus.h (values only)
CACHE_NONE, CACHE_DC, CACHE_DC_PLUS = 0, 1, 2
PLACEHOLDER_UNPROCESSED_ONLY, PLACEHOLDER_ALL_MASKED = 0, 1
STRATEGY_FOCUS, STRATEGY_NONE, STRATEGY_FIXED_TOP, STRATEGY_FIXED_RANDOM, STRATEGY_FIXED_BOTTOM = 0, 1, 2, 3, 4


@dataclass(frozen=True)
class ModelConfig:
    n_layers: int
    d_model: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    rope_theta: float
    rms_eps: float = 1e-6
    logit_scale: float = 1.0             # W_lm scale, a power of two (focus_config::logit_scale)
    # Mixture-of-Experts FFN (LLaDA2.0-mini-shaped workload; reading A-M5): layers
    # >= n_dense_layers replace the dense SwiGLU by n_experts routed experts (top_k per token,
    # d_expert wide) plus n_shared_experts shared experts; n_experts = 0: dense model
    n_experts: int = 0
    top_k: int = 0
    d_expert: int = 0
    n_shared_experts: int = 0
    n_dense_layers: int = 1

    def is_moe_layer(self, layer: int) -> bool:
        return self.n_experts > 0 and layer >= self.n_dense_layers

    @property
    def mask_token_id(self) -> int:
        return self.vocab - 1            # A-M2

    @property
    def group(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    @property
    def qkv_dim(self) -> int:
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.head_dim


@dataclass(frozen=True)
class MethodConfig:
    block_size: int
    alpha_num: int = 3
    alpha_den: int = 2
    conf_threshold: float = 0.9
    maxpool_kernel: int = 3
    cache_mode: int = CACHE_DC_PLUS
    placeholder_mode: int = PLACEHOLDER_UNPROCESSED_ONLY
    strategy: int = STRATEGY_FOCUS
    fixed_k: int = 0


@dataclass(frozen=True)
class RunConfig:
    name: str
    model: ModelConfig
    method: MethodConfig
    n_requests: int
    prompt_len: int                      # fixed length, or lower bound when prompt_len_hi is set
    gen_len: int
    prompt_len_hi: Optional[int] = None  # mixed lengths uniform in [prompt_len, prompt_len_hi] (C4)
    weight_seed: int = 0
    page_size: int = 64
    description: str = ""

    def with_(self, **kw) -> "RunConfig":
        return replace(self, **kw)


TINY = ModelConfig(n_layers=2, d_model=64, n_q_heads=4, n_kv_heads=4, head_dim=16, d_ff=256,
                   vocab=32, rope_theta=1e4)
SDAR_1P7B = ModelConfig(n_layers=28, d_model=2048, n_q_heads=16, n_kv_heads=8, head_dim=128,
                        d_ff=6144, vocab=151936, rope_theta=1e6)
SDAR_8B = ModelConfig(n_layers=36, d_model=4096, n_q_heads=32, n_kv_heads=8, head_dim=128,
                      d_ff=12288, vocab=151936, rope_theta=1e6)
# LLaDA2.0-mini-shaped MoE (16B total, ~1.4B active; PAPER.md P:426 gives only the totals -- the
# layout is reading A-M5): 20 layers, d 2048, GQA 16/4 x 128, vocab 157184, layer 0 dense (d_ff 5120),
# layers 1.. with 256 routed experts of width 512 (top-8) + 1 shared expert of width 512
LLADA2_MINI = ModelConfig(n_layers=20, d_model=2048, n_q_heads=16, n_kv_heads=4, head_dim=128, d_ff=5120,
                          vocab=157184, rope_theta=6e5, n_experts=256, top_k=8, d_expert=512,
                          n_shared_experts=1, n_dense_layers=1)

CONFIGS = {
    "C1": RunConfig("C1", TINY, MethodConfig(block_size=4), n_requests=1, prompt_len=16, gen_len=16,
                    page_size=16, description="tiny synthetic block-diffusion model"),
    "C2": RunConfig("C2", SDAR_1P7B, MethodConfig(block_size=4), n_requests=16, prompt_len=512, gen_len=256,
                    description="SDAR-1.7B-shaped, block 4, batch 16"),
    "C3": RunConfig("C3", SDAR_8B, MethodConfig(block_size=16), n_requests=64, prompt_len=1024, gen_len=512,
                    description="SDAR-8B-shaped, block 16, batch 64"),
    "C4": RunConfig("C4", SDAR_8B, MethodConfig(block_size=16), n_requests=256, prompt_len=256, prompt_len_hi=4096,
                    gen_len=512, description="SDAR-8B-shaped, block 16, batch 256 request-sharded, mixed prompts"),
    "C5": RunConfig("C5", SDAR_8B, MethodConfig(block_size=32), n_requests=32, prompt_len=16384, gen_len=1024,
                    description="SDAR-8B-shaped, block 32, long context"),
    # the paper's second model family, LLaDA2.0-mini (MoE), at its default block 32
    "C6": RunConfig("C6", LLADA2_MINI, MethodConfig(block_size=32), n_requests=64, prompt_len=1024, gen_len=512,
                    description="LLaDA2.0-mini-shaped MoE, block 32, batch 64 (f4)"),
    # the paper's large-block regime (fig:throughput_blocks P:506-511, 3.52x at B = 64)
    "C3B64": RunConfig("C3B64", SDAR_8B, MethodConfig(block_size=64), n_requests=64, prompt_len=1024, gen_len=512,
                       description="SDAR-8B-shaped, block 64, batch 64 (f3)"),
}


def get_config(name: str, **overrides) -> RunConfig:
    cfg = CONFIGS[name]
    return cfg.with_(**overrides) if overrides else cfg
