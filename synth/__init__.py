"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds ONLY input definitions: model/method configurations
(C1..C5 of BASELINE.json), the counter-based weight generator and the
prompt generator.  It contains none of the method's arithmetic (no
importance, selection, attention, commit ...).  Both the CPU oracle
(`oracle/`) and the GPU path consume it; the GPU path re-implements the same
counter-based weight generator in CUDA (paper_2601_23278_b200/csrc/), so the
two sides regenerate bit-identical bf16 weights without sharing code.
"""
from .configs import ModelConfig, MethodConfig, RunConfig, CONFIGS, get_config  # noqa: F401
from .gen import mix64, weight_scale_exp, weight_values, weight_matrix, prompt_tokens, prompt_lengths  # noqa: F401
