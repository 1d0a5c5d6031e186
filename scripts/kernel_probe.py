"""Step-kernel probe (diagnostics): per-step fused-kernel times in the sparse regime (first steps) and the
dense regime (late steps, Krylov vectors fill the grid), Dirichlet and general-boundary variants.
python scripts/kernel_probe.py [m=400] [k=1000]"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 400
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
os.environ["KR_MAX_EV"] = str(k)
for kind in ("dirichlet", "paper_bc"):
    if kind == "paper_bc":
        p = W.heat_paper(m, eps=0.0, k_max=k)
        p["eps"] = 0.0
    else:
        p = W.heat(m, m // 10, k, n_steps=20)
    p["n_steps"] = 20
    tr = tempfile.mktemp()
    os.environ["KR_STEP_TRACE"] = tr
    with KrylovReach(p) as h:
        h.project(want=False)
        h.project(want=False)
    t = np.loadtxt(tr)[:, 1]
    nbytes = 24.0 * m ** 3
    sp, de = t[:50].mean(), t[-300:].mean()
    print(f"{kind:10s} m={m} k={k}: sparse(1-50) {sp:.4f} ms = {nbytes / sp / 1e6:.0f} GB/s | "
          f"dense(last 300) {de:.4f} ms = {nbytes / de / 1e6:.0f} GB/s", flush=True)
