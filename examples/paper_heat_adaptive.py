"""The paper's 3D heat benchmark (§5.3): m x m x m grid, insulated faces with heat exchange 0.5 at
x = 1, a heated corner region in [0.9, 1.1], adaptive Krylov dimension by Lemma 1 to 1e-6 (Alg. 4), T = 20,
delta = 0.02. Prints the accepted k (the paper: 544 at m = 100, 5932 at m = 1000), the bound, the reachable
center temperature and the verdict for an unsafe set "center >= theta".

    python examples/paper_heat_adaptive.py [m=100] [theta=0.0079]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100
theta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0079
p = W.heat_paper(m)
t0 = time.perf_counter()
with KrylovReach(p) as h:
    coeff, stats = h.project()
    verdict = h.check_box([(0, W.GE, theta)])  # row 0 = center temperature
    checks = h.adaptive_checks(0)
wall = time.perf_counter() - t0
hi = verdict["hi"][:, 0]
print(f"m={m} (n={m ** 3:.3g}): k={stats[0]['k_eff']} after {len(checks)} checkpoints, Lemma-1 bound "
      f"{checks[-1][1]:.3g} (unit start vector), {wall:.2f} s")
print(f"max reachable center temperature {hi.max():.6f} at t = {np.argmax(hi) * p['step']:.2f}")
if verdict["found"]:
    print(f"UNSAFE: center >= {theta} reachable at step {verdict['step']} (t = {verdict['time']:.2f}), "
          f"initial heated temperature z = {verdict['z'][0]:.4f}")
else:
    print(f"SAFE: center < {theta} for every t <= {p['n_steps'] * p['step']}")
