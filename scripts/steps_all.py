import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import workloads as W
from paper_1804_01583_b200 import KrylovReach
p = W.CONFIGS[sys.argv[1]]()
with KrylovReach(p) as h:
    for _ in range(3):
        h.project(want=False); h.check_box(want_bounds=False)
    runs = []
    for _ in range(6):
        h.project(want=False); h.check_box(want_bounds=False)
        runs.append(h.step_times())
a = np.array(runs)
np.set_printoptions(precision=3, linewidth=250)
print("sampled steps (1-based) with timing:", [i + 1 for i in range(a.shape[1]) if np.isfinite(a[0, i])])
for r in a:
    print(r[np.isfinite(r)])
