"""C5 on P virtual z-slabs in one process (the slab code path of a P-GPU run: per-slab launches, halo planes stored by
the step kernel into the sibling slab's buffer), to estimate strong scaling: the slabs run one after
the other on the one GPU, so iter_ms / P is the per-GPU Lanczos time at P GPUs. Usage: python scripts/vslab_timing.py 1 2 4 8"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

p = W.config5()
for P in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    kw = dict(virtual_slabs=P, part="zslab") if P > 1 else {}
    with KrylovReach(p, **kw) as h:
        for _ in range(2):
            h.project(want=False)
        its = []
        for _ in range(3):
            h.project(want=False)
            its.append(h.last_timing()["iter_ms"])
    it = min(its)
    print(f"P={P}: Lanczos iteration {it:.2f} ms over all slabs, {it / P:.2f} ms per slab "
          f"({p['k'] / (it / P / 1000):.0f} Krylov steps/s per run if the slabs ran concurrently)", flush=True)
