"""Step-kernel probe at equal data density (diagnostics): dense start vector (all ones) for the Dirichlet and
the general-boundary variants, with nvidia-smi clocks / power sampled; per-step times of steps 1-50."""
import os
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 60
os.environ["KR_MAX_EV"] = str(k)
for kind in ("dirichlet", "paper_bc", "dirichlet", "paper_bc"):
    if kind == "paper_bc":
        p = W.heat_paper(m, eps=0.0, k_max=k)
        p["eps"] = 0.0
    else:
        p = W.heat(m, m // 10, k, n_steps=20)
    p["gens"] = [W.allv(1.0)]
    p["n_steps"] = 20
    tr = tempfile.mktemp()
    os.environ["KR_STEP_TRACE"] = tr
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.PIPE, text=True)
    with KrylovReach(p) as h:
        h.project(want=False)
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    clk = [float(l.split(",")[0]) for l in out if l.strip()]
    pw = [float(l.split(",")[1]) for l in out if l.strip()]
    t = np.loadtxt(tr)[:, 1]
    print(f"{kind:10s} m={m} dense start: steps 2-{k} mean {t[1:].mean():.4f} ms = {24 * m ** 3 / t[1:].mean() / 1e6:.0f} GB/s"
          f" | sm clk median {np.median(clk):.0f} MHz, power max {max(pw):.0f} W", flush=True)
