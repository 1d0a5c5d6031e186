"""Time the heater variant (NEXT-4) at m = 100: Arnoldi k steps (CGS2 path) + large-k exponentials."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for k in [int(x) for x in (sys.argv[2:] or ["100", "400"])]:
    p = W.heat_heater(m, k=k)
    with KrylovReach(p) as h:
        for _ in range(2):
            t0 = time.perf_counter()
            coeff, stats = h.project()
            wall = time.perf_counter() - t0
        t = h.last_timing()
    c = coeff[:, 0, 0]
    print(json.dumps({"m": m, "k": k, "k_eff": stats[0]["k_eff"], "wall_s": wall, "iter_ms": t["iter_ms"],
                      "large_ms": t["large_ms"], "center_T500": float(c[-1]), "center_max": float(c.max()),
                      "monotone": bool((c[1:] >= c[:-1] - 1e-12).all()), "total_heat_T500": float(coeff[-1, 1, 0])}),
          flush=True)
