"""Host wall-clock of create / project / destroy (KR_TRACE=1 adds the per-phase marks on stderr). Usage: KR_TRACE=1 python scripts/create_trace.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_1804_01583_b200 import KrylovReach
for cfg in ["C3", "C4", "C2"]:
    p = W.CONFIGS[cfg]()
    for i in range(3):
        t0 = time.perf_counter()
        h = KrylovReach(p)
        t1 = time.perf_counter()
        h.project(want=False)
        t2 = time.perf_counter()
        h.close()
        t3 = time.perf_counter()
        print(f"{cfg} run {i}: create {1e3*(t1-t0):.3f} project {1e3*(t2-t1):.3f} destroy {1e3*(t3-t2):.3f} ms", file=sys.stderr, flush=True)
