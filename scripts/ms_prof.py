"""KR_MS_PROF=1 phase times of the multi-step kernel (two runs of a config). Usage: KR_MS_PROF=1 KR_NO_GRAPH=1 python scripts/ms_prof.py C3"""
import os, sys
sys.path.insert(0, os.getcwd())
import workloads as W
from paper_1804_01583_b200 import KrylovReach
cfg = sys.argv[1]
p = W.CONFIGS[cfg]()
with KrylovReach(p) as h:
    h.project(want=False)
    print("---- second run", file=sys.stderr, flush=True)
    h.project(want=False)
