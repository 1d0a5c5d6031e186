"""Debug helper: repeat a project on one handle / fresh handles; report non-finite or non-identical runs."""
import sys
import numpy as np
sys.path.insert(0, '.')
import workloads as W
from paper_1804_01583_b200 import KrylovReach

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = W.CONFIGS[cfg]()
ref = None
for fresh in (False, True):
    h = KrylovReach(p)
    for it in range(reps):
        if fresh and it > 0:
            h.close()
            h = KrylovReach(p)
        coeff, stats = h.project()
        H, P = h.krylov_data(0)
        fin = np.isfinite(coeff).all()
        same = ref is None or np.array_equal(coeff, ref[0])
        sameH = ref is None or np.array_equal(H, ref[1])
        print(f"fresh={fresh} it={it} finite={fin} same={same} sameH={sameH} keff={stats[0]['k_eff']}", flush=True)
        if not fin:
            bad = np.where(~np.isfinite(coeff))
            print("  first non-finite step", bad[0].min(), "H finite", np.isfinite(H).all())
            k = stats[0]['k_eff']
            print("  eig max", np.linalg.eigvalsh(0.5 * (H[:k, :k] + H[:k, :k].T)).max())
        if ref is None:
            ref = (coeff, H)
    h.close()
