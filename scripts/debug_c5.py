"""Debug helper: C5 fused Lanczos H on the GPU (eigenvalues must be negative; first step closed form)."""
import math
import sys
import numpy as np
sys.path.insert(0, '.')
import workloads as W
from paper_1804_01583_b200 import KrylovReach

p = W.config5(n_steps=int(sys.argv[1]) if len(sys.argv) > 1 else 1000)
with KrylovReach(p) as h:
    coeff, stats = h.project()
    H, P = h.krylov_data(0)
k = stats[0]["k_eff"]
Hk = H[:k, :k]
print("k_eff", k, "beta0", stats[0]["beta0"])
print("alpha", np.diag(Hk))
print("beta", [H[i + 1, i] for i in range(k)])
print("sym", np.abs(Hk - Hk.T).max(), "eig max", np.linalg.eigvalsh(0.5 * (Hk + Hk.T)).max())
m, b = 1000, 100
c = 0.01 * (m + 1) ** 2
s = sum(math.comb(3, q) * 2 ** q * (b - 2) ** (3 - q) * (6 / b - q) ** 2 for q in range(4))
print("closed form a1", -6 * c / b, "b1", math.sqrt(c * c * (s + 3 * b * b) / b ** 3))
print("P", P[:, :6])
print("coeff finite", np.isfinite(coeff).all())
