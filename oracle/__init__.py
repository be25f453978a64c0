"""CPU oracle for the FOCUS block-diffusion decode step (arxiv 2601.23278).

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call, link
or execute anything under `oracle/`; only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s `cpu_baseline` / `--impl reference` legs do.  The CUDA path
(paper_2601_23278_b200/) shares no code with it: the only common module is
`synth/` (seeded input generators, no method arithmetic).

Plain, slow, obviously-correct code in binary64 (NumPy float64 for the model
math, pure-Python ints/floats for the rules), following PAPER.md step by step:
  numerics.py  softmax / MaxPool1D / RMSNorm / RoPE / SiLU / bf16 rounding
  model.py     the Qwen3-like backbone (SURVEY A-M1) and its weights
  focus.py     Eq.2 importance, Eq.3 delta, Eq.4/5 budget, Alg.1 selection,
               compaction, confidence decode, Neighbor-Aware DC+ commit
  engine.py    Alg.1 composed per request (prefill, step, commit)
Each function cites the passage it follows ("P:n" = PAPER.md line n,
"S:n" = SPEC.md line n) and the DESIGN.md reading it takes where the paper is
silent.  Pins live in tests/test_oracle_*.py (run with -m "not gpu").
"""
