"""HBM ceiling vs data content (diagnostics): torch add (2R+1W) and copy on 1e9 fp64 with zeros vs random data."""
import torch

n = 1_000_000_000
for kind in ("zeros", "random"):
    a = torch.zeros(n, dtype=torch.float64, device="cuda")
    b = torch.zeros(n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, dtype=torch.float64, device="cuda")
    if kind == "random":
        a.normal_()
        b.normal_()
    for name, fn, nbytes in [("copy", lambda: c.copy_(a), 16 * n), ("add", lambda: torch.add(a, b, out=c), 24 * n)]:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(10):
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{kind:7s} {name}: {best:.3f} ms  {nbytes / best / 1e6:.0f} GB/s", flush=True)
    del a, b, c
    torch.cuda.empty_cache()
