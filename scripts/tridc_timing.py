"""Checkpoint-route timing on one GPU: one large-route evaluation at fixed k on the paper's heat model
(m = 100), by the device eigen-solve (default) and the Taylor route (KR_LARGE_TAYLOR=1), plus adaptive P100
runs with and without the pipelined checkpoints. Usage: python scripts/tridc_timing.py [k ...]"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import workloads as W
    from paper_1804_01583_b200 import KrylovReach
    mode, m, k = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    if mode == "fixed":
        p = W.heat_paper(m, eps=0.0, k_max=k)
        p["eps"] = 0.0
    else:
        p = W.heat_paper(m, k_max=8000)
    with KrylovReach(p) as h:
        for rep in range(3):
            coeff, stats = h.project()
            t = h.last_timing()
    print(json.dumps({"mode": mode, "m": m, "k": stats[0]["k_eff"], "env": os.environ.get("TAG", ""),
                      "iter_ms": t["iter_ms"], "large_ms": t["large_ms"], "large_evals": t["large_evals"],
                      "per_eval_ms": t["large_ms"] / max(1, t["large_evals"])}), flush=True)
    sys.exit(0)

ks = [int(a) for a in sys.argv[1:]] or [128, 256, 544]
runs = []
for k in ks:
    runs += [("fixed", 100, k, {}), ("fixed", 100, k, {"KR_LARGE_TAYLOR": "1"})]
runs += [("adaptive", 100, 0, {}), ("adaptive", 100, 0, {"KR_NO_SPECULATE": "1"}),
         ("adaptive", 100, 0, {"KR_LARGE_TAYLOR": "1"})]
for mode, m, k, env in runs:
    e = dict(os.environ, **env, TAG=",".join(f"{a}={b}" for a, b in env.items()))
    subprocess.run([sys.executable, __file__, "child", mode, str(m), str(k)], env=e, timeout=600)
