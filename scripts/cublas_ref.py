"""cuBLAS reference timings (torch.matmul, bf16) at the C3 decode GEMM shapes, L2 flushed between reps.
Development reference only (the product path uses libfocus's tcgen05 GEMM)."""
import os
import sys

import torch

M = int(sys.argv[1]) if len(sys.argv) > 1 else 428
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, N, K in [("qkv", 6144, 4096), ("o", 4096, 4096), ("gu", 24576, 4096), ("down", 4096, 12288),
                   ("lm", 151936, 4096)]:
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    W = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    best = 1e9
    for r in range(7):
        if not os.environ.get("GEMM_NOFLUSH"):
            flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        C = A @ W.t()
        e1.record()
        torch.cuda.synchronize()
        if r:
            best = min(best, e0.elapsed_time(e1))
    print(f"cuBLAS M={M} {name:5s} N={N:6d} K={K:5d} {best * 1e3:8.1f} us {2 * M * N * K / (best * 1e-3) / 1e12:7.1f} TFLOP/s")
