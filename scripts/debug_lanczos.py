"""Debug helper: GPU fused Lanczos H/P vs the oracle on a heat problem."""
import sys
import numpy as np
sys.path.insert(0, '.')
import oracle
import workloads as W
from paper_1804_01583_b200 import KrylovReach

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100
k = int(sys.argv[2]) if len(sys.argv) > 2 else 40
b = max(2, m // 10)
p = W.heat(m, b, k, n_steps=20)
v = oracle.directions(p)[0]
r = oracle.lanczos(p, v, k)
with KrylovReach(p) as h:
    coeff, stats = h.project()
    H, P = h.krylov_data(0)
print("k_eff gpu/oracle", stats[0]["k_eff"], r["k_eff"])
ka = min(stats[0]["k_eff"], r["k_eff"])
a_g = np.diag(H[:ka, :ka]); b_g = np.array([H[i + 1, i] for i in range(ka)])
print("alpha rel err", np.abs(a_g - r["alpha"][:ka]) / np.abs(r["alpha"][:ka]))
print("beta  rel err", np.abs(b_g - r["beta"][:ka]) / np.abs(r["beta"][:ka]))
print("P err", np.abs(P[:, :ka] - r["P"][:, :ka]).max(axis=0))
print("coeff finite", np.isfinite(coeff).all())
