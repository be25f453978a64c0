"""Summarise gpurun_out/attn_trace.npz: per-role event timelines of a few CTAs (cycles since kernel
start) and per-role average gaps between event kinds."""
import sys

import numpy as np

d = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/attn_trace.npz")["trace"]
ROLES = ["Kprod", "Vprod", "MMA", "PV", "softmax", "epilogue"]
MASK = (1 << 56) - 1


def events(cta, role):
    v = d[cta, role]
    v = v[v != 0]
    return [(int(x) >> 56, int(x) & MASK) for x in v]


for cta in (0, 77):
    t0 = int(d[cta, 7, 0]) & MASK
    print(f"=== CTA {cta}")
    for r, name in enumerate(ROLES):
        ev = events(cta, r)
        s = " ".join(f"{k}:{(t - t0) / 1000:.1f}" for k, t in ev[:60])
        print(f"{name:9s} n={len(ev):3d} {s}")

# aggregate: average duration from event kind a to the next event of kind b, per role
print("=== averages over all CTAs (k cycles)")
for r, name in enumerate(ROLES):
    gaps = {}
    for cta in range(d.shape[0]):
        ev = events(cta, r)
        for (k1, t1), (k2, t2) in zip(ev, ev[1:]):
            gaps.setdefault((k1, k2), []).append(t2 - t1)
    s = "  ".join(f"{a}->{b}: {np.mean(v) / 1000:.2f}x{len(v)}" for (a, b), v in sorted(gaps.items()))
    print(f"{name:9s} {s}")
ends = []
for cta in range(d.shape[0]):
    t0 = int(d[cta, 7, 0]) & MASK
    last = max((t for r in range(6) for _, t in events(cta, r)), default=t0)
    ends.append(last - t0)
print("CTA span k cycles: min %.1f med %.1f max %.1f" % (min(ends) / 1e3, np.median(ends) / 1e3, max(ends) / 1e3))

# entry -> t0 (prologue + PDL wait + plan load) and kernel extent in global time (ns)
r7 = d[:, 7, :5].astype(np.int64)
if (r7[:, 2] > 0).all() and (r7[:, 4] > 0).all():
    pro = (r7[:, 0] & MASK) - (r7[:, 1] & MASK)
    tail = (r7[:, 3] & MASK) - (r7[:, 0] & MASK)
    print("prologue (entry->t0) k cycles: min %.1f med %.1f max %.1f" % (pro.min() / 1e3, np.median(pro) / 1e3, pro.max() / 1e3))
    print("t0->exit k cycles: min %.1f med %.1f max %.1f" % (tail.min() / 1e3, np.median(tail) / 1e3, tail.max() / 1e3))
    e0, e1 = r7[:, 2], r7[:, 4]
    print("global time: first entry -> last exit %.1f us; entries spread %.1f us; exits spread %.1f us" %
          ((e1.max() - e0.min()) / 1e3, (e0.max() - e0.min()) / 1e3, (e1.max() - e1.min()) / 1e3))
