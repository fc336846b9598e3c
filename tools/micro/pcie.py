"""Pinned host <-> device copy times of config 3's per-step e2e bytes (269 MB in, 303 MB out),
each alone and both at once on two streams: the bound of bench.py's e2e number."""
import time, torch
n_in, n_out = 269475856, 302760000
hi = torch.empty(n_in, dtype=torch.uint8).pin_memory(); ho = torch.empty(n_out, dtype=torch.uint8).pin_memory()
di = torch.empty(n_in, dtype=torch.uint8, device="cuda"); do = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, n=10):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
h2d = t(lambda: di.copy_(hi, non_blocking=True)); d2h = t(lambda: ho.copy_(do, non_blocking=True))
def both():
    with torch.cuda.stream(s1): di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
bb = t(both)
print(f"h2d {h2d:.2f} ms {n_in/h2d/1e6:.1f} GB/s; d2h {d2h:.2f} ms {n_out/d2h/1e6:.1f} GB/s; concurrent {bb:.2f} ms")
