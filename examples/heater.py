"""The paper's nonsymmetric heat variant: a permanent heater on the z = 0 patch
x <= 0.4, y <= 0.2, insulated faces, exchange 0.5 at x = 1, T = 500, delta = 0.5 — a lifted (affine) stencil
system simulated by Arnoldi. Prints the reachable center temperature for two Krylov dimensions.

    python examples/heater.py [m=100] [k1=400] [k2=800]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for k in [int(x) for x in sys.argv[2:]] or [400, 800]:
    p = W.heat_heater(m, k=k)
    t0 = time.perf_counter()
    with KrylovReach(p) as h:
        coeff, stats = h.project()
    c = coeff[:, 0, 0]
    print(f"m={m} k={k}: center temperature at T=500: {c[-1]:.6f} (max {c.max():.6f}); total heat "
          f"{coeff[-1, 1, 0]:.1f}; {time.perf_counter() - t0:.2f} s")
