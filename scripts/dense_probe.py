"""Dense-regime probe: Lanczos far enough that the vectors fill the grid (diagnostics for profiling).
python scripts/dense_probe.py {dir|bc} m k"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

kind, m, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
if kind == "bc":
    p = W.heat_paper(m, eps=0.0, k_max=k)
    p["eps"] = 0.0
else:
    p = W.heat(m, m // 10, k, n_steps=100)
p["n_steps"] = 100
with KrylovReach(p) as h:
    h.project(want=False)
    t = h.last_timing()
print(kind, m, k, t)
