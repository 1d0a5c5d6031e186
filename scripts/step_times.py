"""Per-step device times (CUDA events around each step-kernel launch) for one config.
Usage: python scripts/step_times.py C5 [runs]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach, krylov_workspace_bytes  # noqa: E402

os.environ.setdefault("KR_MAX_EV", "1000000")  # time every step (diagnostics)
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if name.startswith("PAPER:"):  # PAPER:m:k -> the paper's heat model at fixed k (no adaptive checkpoints)
    _, m, k = name.split(":")
    p = W.heat_paper(int(m), eps=0.0, k_max=int(k))
else:
    p = W.CONFIGS[name]()
st = torch.cuda.current_stream().cuda_stream
wsb = krylov_workspace_bytes(p, device=0, stream=st)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
with KrylovReach(p, device=0, stream=st, workspace=ws.data_ptr(), workspace_bytes=wsb) as h:
    rows = []
    for r in range(runs + 1):
        h.project(want=False)
        t = h.last_timing()
        if r:
            rows.append(h.step_times())
    a = np.array(rows)  # NaN: step not timed (KR_MAX_EV=k times every step)
    print(name, os.environ.get("KR_NO_COMPACT", "compact"), "iter_ms", round(t["iter_ms"], 3))
    print(" per-step ms (mean over runs):", " ".join(f"{x:.3f}" for x in np.nanmean(a, 0)))
