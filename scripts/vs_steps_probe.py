import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import workloads as W
from paper_1804_01583_b200 import KrylovReach
p = W.heat(1000, 100, 30, n_steps=1000)
with KrylovReach(p, virtual_slabs=int(sys.argv[1])) as h:
    h.project(want=False); h.project(want=False)
    t = h.last_timing(); st = h.step_times()
    print(os.environ.get("KR_MAX_EV"), round(t["iter_ms"], 2), round(t["step_ms_mean"], 4), " ".join(f"{x:.3f}" for x in st))
