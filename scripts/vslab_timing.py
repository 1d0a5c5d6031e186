"""Virtual z-slab timing (diagnostics): C5 recipe on 1 GPU split into P slabs, in-kernel halo writes vs
the copy transport (KR_HALO_COPY=1 in the environment)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
for vs in [int(x) for x in sys.argv[2:]] or [1, 8]:
    p = W.heat(m, m // 10, 30, n_steps=1000)
    with KrylovReach(p, virtual_slabs=vs) as h:
        h.project(want=False)
        h.project(want=False)
        t = h.last_timing()
    print(f"m={m} vs={vs} copy={os.environ.get('KR_HALO_COPY', '0')}: iter {t['iter_ms']:.2f} ms, "
          f"step kernel {t['step_ms_mean']:.4f} ms x {t['step_launches']} launches", flush=True)
