"""HBM ceiling probe (diagnostics): torch copy (1R+1W) and add (2R+1W) on 1e9 fp64 elements."""
import torch

n = 1_000_000_000
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
c = torch.empty(n, dtype=torch.float64, device="cuda")
a.fill_(1.0)
b.fill_(2.0)
for name, fn, nbytes in [("copy 1R1W", lambda: c.copy_(a), 16 * n), ("add 2R1W", lambda: torch.add(a, b, out=c), 24 * n),
                         ("read-only sum", lambda: a.sum(), 8 * n)]:
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
    print(f"{name}: {best:.3f} ms  {nbytes / best / 1e6:.0f} GB/s", flush=True)
