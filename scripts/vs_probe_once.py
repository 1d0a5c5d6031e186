"""One project of the C5 recipe on P virtual slabs (diagnostics for launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

p = W.heat(1000, 100, 6, n_steps=10)
with KrylovReach(p, virtual_slabs=int(sys.argv[1])) as h:
    h.project(want=False)
