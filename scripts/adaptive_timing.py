"""Time the adaptive (Alg. 4) paper-heat runs on one GPU: total device time, Lanczos steps, checkpoints,
and the share of the large-k exponential route. Usage: python scripts/adaptive_timing.py 100 200 ..."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

for arg in sys.argv[1:]:
    m = int(arg)
    p = W.heat_paper(m, k_max=8000)
    with KrylovReach(p) as h:
        for rep in range(1 if m >= 400 else 2):
            t0 = time.perf_counter()
            coeff, stats = h.project()
            wall = time.perf_counter() - t0
        t = h.last_timing()
        ch = h.adaptive_checks(0)
    out = {"m": m, "n": m ** 3, "k": stats[0]["k_eff"], "bound": ch[-1][1] if ch else None, "checkpoints": len(ch),
           "wall_s": wall, "iter_ms": t["iter_ms"], "large_ms": t["large_ms"], "large_evals": t["large_evals"],
           "step_ms_mean": t["step_ms_mean"], "steps_run": t["step_launches"],
           "lanczos_ms_est": t["iter_ms"] - t["large_ms"],
           "step_gbs": t["step_bytes"] / (t["step_ms_mean"] * 1e-3) / 1e9 if t["step_ms_mean"] else None,
           "center_max": float(coeff[:, 0, 0].max()), "center_argmax_t": float(coeff[:, 0, 0].argmax() * p["step"])}
    print(json.dumps(out), flush=True)
