"""Per-step fused-kernel times of one C5 run (KR_MAX_EV=64: every step timed): step 1 reads only the compact u_1
(L2-resident, no HBM reads), so it separates the kernel's SM-side time from the HBM-bound steps 3..k-1.
Usage: python scripts/step_profile.py [CONFIG]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("KR_MAX_EV", "64")
import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
p = W.CONFIGS[cfg]()
with KrylovReach(p) as h:
    for _ in range(3):
        h.project(want=False)
    runs = []
    for _ in range(3):
        h.project(want=False)
        runs.append(h.step_times())
st = np.nanmean(np.array(runs), axis=0)
print(f"{cfg}: step1 {st[0]:.4f} ms step2 {st[1]:.4f} "
      f"steps3..k-1 {np.mean(st[2:-1]):.4f} last {st[-1]:.4f}")
