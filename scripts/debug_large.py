"""Diagnostics: large-k route, doubling vs sequential march, per k (fixed k, paper heat m=30)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 30
full = None
for k in [65, 100, 128, 150, 154, 170]:
    p = W.heat_paper(m, eps=0.0, k_max=k)
    p["eps"] = 0.0
    res = {}
    for kd in ("0", "100000"):
        os.environ["KR_KDOUBLE"] = kd
        with KrylovReach(p) as h:
            c, st = h.project()
        res[kd] = (c, st[0])
    r = oracle.lanczos(p, oracle.directions(p)[0], k)
    X = oracle.eig_e1_times(r["alpha"], r["beta"], p["step"], p["n_steps"])
    b_or = r["beta0"] * oracle.lemma1_bound(r["beta"][k - 1], X, p["step"], 0.0)
    c0, s0 = res["0"]
    c1, s1 = res["100000"]
    print(k, "lemma chain", s0["lemma1"], "dbl", s1["lemma1"], "oracle", b_or, "max|dc|", np.abs(c0 - c1).max(),
          flush=True)
