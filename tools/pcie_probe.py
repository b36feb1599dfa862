"""PCIe probe: pinned H2D / D2H bandwidth, one stream vs the copy split over two streams, and both
directions at once (bounds bench.py's e2e number)."""
import torch

n = 218 * 2**20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d1():
    d.copy_(h, non_blocking=True)


def h2d2():
    half = n // 2
    with torch.cuda.stream(s1):
        s1.wait_stream(torch.cuda.default_stream())
        d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        s2.wait_stream(torch.cuda.default_stream())
        d[half:].copy_(h[half:], non_blocking=True)


def d2h1():
    h2.copy_(d2, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        s1.wait_stream(torch.cuda.default_stream())
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        s2.wait_stream(torch.cuda.default_stream())
        h2.copy_(d2, non_blocking=True)


for name, fn in (("h2d 1 stream", h2d1), ("h2d 2 streams", h2d2), ("d2h 1 stream", d2h1), ("h2d+d2h", both)):
    ms = timed(fn)
    print(f"{name:14s} {ms:7.3f} ms  {n / ms / 1e6:6.1f} GB/s per direction")
