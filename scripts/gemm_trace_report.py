"""Summarise the pair-GEMM clock64 trace written by scripts/gemm_bench.cu (GEMM_TRACE=1)."""
import sys

import numpy as np

for fn in sys.argv[1:]:
    t = np.fromfile(fn, dtype=np.int64).reshape(148, 3, 256)
    print(fn)
    rows = []
    for b in range(148):
        t0 = t[b, 0, 0]
        if t0 == 0:
            continue
        prod = t[b, 0, 1:][t[b, 0, 1:] > 0] - t0
        mma = t[b, 1, 1:][t[b, 1, 1:] > 0] - t0
        epi = t[b, 2, 1:][t[b, 2, 1:] > 0] - t0
        d = np.diff(mma) if len(mma) > 1 else np.array([0])
        rows.append((b, len(mma), mma[0] if len(mma) else -1, np.median(d), d.max(), mma[-1] if len(mma) else -1,
                     epi[-1] if len(epi) else -1, prod[0] if len(prod) else -1))
    print(f"{'cta':>4} {'stages':>6} {'first':>7} {'med':>6} {'max':>7} {'last':>7} {'end':>7} {'p0':>6}")
    for r in rows[:6] + rows[-4:]:
        print(f"{r[0]:4d} {r[1]:6d} {r[2]:7d} {r[3]:6.0f} {r[4]:7d} {r[5]:7d} {r[6]:7d} {r[7]:6d}")
    lead = [r for r in rows if r[1] > 0]
    if lead:
        print("leaders: median per-stage cycles %.0f, median first-stage %.0f, median end %.0f" %
              (np.median([r[3] for r in lead]), np.median([r[2] for r in lead]), np.median([r[6] for r in rows])))
