import sys, json
sys.path.insert(0, '.')
import workloads as W
from paper_1804_01583_b200 import KrylovReach
for m in (16, 32, 48, 64, 100):
    p = W.heat_paper(m, eps=0.0, k_max=300)
    p["eps"] = 0.0
    with KrylovReach(p) as h:
        for _ in range(3):
            h.project()
        t = h.last_timing()
    print(m, "step_ms_mean %.4f" % t["step_ms_mean"], "iter_ms %.3f" % t["iter_ms"], flush=True)
