"""Host wall-clock breakdown of the public API path (create / project / check_box / destroy) per config.
Usage (GPU box): python scripts/e2e_breakdown.py C2 C2T P100 C3 C5"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach, krylov_workspace_bytes  # noqa: E402


def sync():
    torch.cuda.synchronize()


def main():
    torch.cuda.set_device(0)
    for name in sys.argv[1:] or ["C2", "C2T", "P100", "C3"]:
        p = W.CONFIGS[name]()
        st = torch.cuda.current_stream().cuda_stream
        wsb = krylov_workspace_bytes(p, device=0, stream=st)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        for it in range(3):
            sync()
            t0 = time.perf_counter()
            h = KrylovReach(p, device=0, stream=st, workspace=ws.data_ptr(), workspace_bytes=wsb)
            sync()
            t1 = time.perf_counter()
            c, s = h.project()
            t2 = time.perf_counter()
            h.project(want=False)
            sync()
            t3 = time.perf_counter()
            h.check_box()
            t4 = time.perf_counter()
            h.close()
            sync()
            t5 = time.perf_counter()
            tm = h_last = None
            print(f"{name} it{it}: create {1e3*(t1-t0):8.2f} ms  project#1 {1e3*(t2-t1):8.2f}  project#2 {1e3*(t3-t2):8.2f}"
                  f"  check_box {1e3*(t4-t3):7.2f}  destroy {1e3*(t5-t4):7.2f}  total(1 proj) "
                  f"{1e3*(t5-t0-(t3-t2)):8.2f}", flush=True)
        del ws


if __name__ == "__main__":
    main()
