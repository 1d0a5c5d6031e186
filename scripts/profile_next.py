"""Profiling targets for the NEXT-row kernels (one short run each):
  cgs:  heater variant m = 100, k = 300 (stored-basis Arnoldi on the CGS2 path)
  gemm: paper heat m = 300, fixed k = 2500 (large-k route: dense band-aware fp64 GEMMs + doubling)
  lp:   C2 in transpose mode + the 41-row polytope LP of tests/test_gpu_next3.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

mode = sys.argv[1]
if mode == "cgs":
    with KrylovReach(W.heat_heater(100, k=300)) as h:
        h.project(want=False)
elif mode == "gemm":
    p = W.heat_paper(300, eps=0.0, k_max=2500)
    p["eps"] = 0.0
    with KrylovReach(p) as h:
        h.project(want=False)
        print(h.last_timing())
elif mode == "lp":
    p = W.config2()
    with KrylovReach(p, sim="transpose") as h:
        coeff, _ = h.project()
        IA = np.vstack([np.eye(20), -np.eye(20), np.ones((1, 20))])
        Ib = np.r_[np.full(40, 0.01), 0.1]
        yf = coeff[:, :, 20]
        th0 = 0.5 * (yf[0, 0] + yf[-1, 0])
        lp = h.check_lp(IA, Ib, [[1.0, 0, 0]], [th0])
        print(lp["found"], lp["step"])
print("ok")
