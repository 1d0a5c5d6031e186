"""Summarise a KR_STEP_TRACE file (per timed Lanczos step: step index, step-kernel ms, step-to-step ms) by step
range: mean / min / max step-kernel time and the effective bandwidth 24 n / t. Usage: trace_summary.py FILE N_CELLS"""
import sys

import numpy as np

rows = [l.split() for l in open(sys.argv[1]) if l.strip() and not l.startswith("#")]
n = float(sys.argv[2])
st = np.array([int(r[0]) for r in rows])
ms = np.array([float(r[1]) for r in rows])
edges = [1, 51, 257, 601, 1001, 2001, 3001, 4001, 5001, 10 ** 9]
for a, b in zip(edges[:-1], edges[1:]):
    m = (st >= a) & (st < b)
    if not m.any():
        continue
    t = ms[m]
    print(f"steps {a:5d}-{min(b - 1, st.max()):5d}: mean {t.mean():.3f} ms  min {t.min():.3f}  max {t.max():.3f}  -> "
          f"{24 * n / (t.mean() * 1e-3) / 1e9:.0f} GB/s effective")
