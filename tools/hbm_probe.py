"""HBM probe: write-only (fill), read-only (sum) and copy bandwidth on 1 GiB, CUDA events, best of 10 --
the ceilings the store-heavy kernels (down-proj Y, dX~) are held against."""
import torch

n = 1 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
a.fill_(1)


def best(fn, reps=10):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


av = a.view(torch.int64)
for name, fn, bytes_ in (("write (fill_)", lambda: b.fill_(3), n), ("write (zero_/memset)", lambda: b.zero_(), n),
                         ("write (bf16 fill)", lambda: b.view(torch.bfloat16).fill_(1.5), n),("read (sum)", lambda: av.sum(), n),
                         ("copy (read+write)", lambda: b.copy_(a), 2 * n)):
    ms = best(fn)
    print(f"{name:18s} {ms:7.3f} ms  {bytes_ / ms / 1e6:7.1f} GB/s")
