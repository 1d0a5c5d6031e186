"""Sustained per-step time of the fused step kernel on a dense workload (C5D or P1000D): `runs` fixed-k runs back to
back (the SM clock settles under the power cap), the mean over steps 3..k-1 of the last five runs, with nvidia-smi
clocks / power sampled meanwhile. Usage: python scripts/dense_ab.py CONFIG [runs]"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("KR_MAX_EV", "64")
import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

cfg = sys.argv[1]
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 30
p = W.CONFIGS[cfg]()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "250"],
                       stdout=subprocess.PIPE, text=True)
with KrylovReach(p) as h:
    per = []
    for _ in range(runs):
        h.project(want=False)
        st = np.array(h.step_times())
        per.append(np.nanmean(st[2:-1]))
smi.terminate()
rows = [r.split(",") for r in smi.communicate()[0].strip().splitlines() if "," in r]
mhz = np.median([float(r[0]) for r in rows]) if rows else float("nan")
pw = np.median([float(r[1]) for r in rows]) if rows else float("nan")
n = (p["mx"] * p["my"] * p["mz"])
last = float(np.mean(per[-5:]))
print(f"{cfg}: steps3..k-1 first run {per[0]:.4f} ms, last five {last:.4f} ms = {24 * n / last / 1e6:.0f} GB/s; "
      f"median {mhz:.0f} MHz {pw:.0f} W over {runs} runs")
