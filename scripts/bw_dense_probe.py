"""HBM ceiling on dense data (diagnostics): torch copy (1R1W) and add (2R1W) over 1e9 fp64 elements of random
data, back to back for a few seconds each (sustained, as a long Lanczos run is), with nvidia-smi clocks / power
sampled during each phase. The constant-data probe (bw_probe.py) toggles almost no bits; random data is the
access mix and bit activity of the dense Krylov vectors. Usage: python scripts/bw_dense_probe.py [seconds]"""
import subprocess
import sys
import time

import torch

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
n = 1_000_000_000
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
c = torch.empty(n, dtype=torch.float64, device="cuda")


def smi_start():
    return subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                             "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)


def smi_stop(p):
    p.terminate()
    out = p.communicate()[0]
    rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") == 2]
    mhz = sorted(float(r[0]) for r in rows)
    pw = sorted(float(r[1]) for r in rows)
    reasons = sorted({r[2].strip() for r in rows})
    med = lambda v: v[len(v) // 2] if v else float("nan")
    return f"SM MHz median {med(mhz):.0f} (min {mhz[0] if mhz else 0:.0f}), power median {med(pw):.0f} W, reasons {reasons}"


for name, fn, nbytes in [("copy 1R1W random", lambda: c.copy_(a), 16 * n),
                         ("add 2R1W random", lambda: torch.add(a, b, out=c), 24 * n)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    p = smi_start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    t_end = time.time() + secs
    while time.time() < t_end:
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 20)
    s = smi_stop(p)
    first, last = times[0], sum(times[-5:]) / len(times[-5:])
    print(f"{name}: first {nbytes / first / 1e6:.0f} GB/s, sustained (last 100 launches) {nbytes / last / 1e6:.0f} GB/s, "
          f"best {nbytes / min(times) / 1e6:.0f} GB/s; {s}", flush=True)
