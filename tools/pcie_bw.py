"""Host<->device copy bandwidth on this box: H2D alone, D2H alone, both at once
(pinned buffers, the e2e bench's sizes: 176 MB in, 336 MB out)."""
import time
import torch

dev = torch.device("cuda", 0)
hi = torch.empty(176_000_000, dtype=torch.uint8).pin_memory()
ho = torch.empty(336_000_000, dtype=torch.uint8).pin_memory()
di = torch.empty(176_000_000, dtype=torch.uint8, device=dev)
do = torch.empty(336_000_000, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return min(ts) * 1e3, sorted(ts)[len(ts) // 2] * 1e3


def h2d():
    with torch.cuda.stream(s1):
        di.copy_(hi, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn, mb in (("H2D 176 MB", h2d, 176), ("D2H 336 MB", d2h, 336), ("both at once", both, 512)):
    mn, med = timed(fn)
    print(f"{name:14s} min {mn:7.3f} ms  median {med:7.3f} ms  ({mb / med:6.1f} GB/s aggregate)", flush=True)
