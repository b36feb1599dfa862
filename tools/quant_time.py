"""Time the e4m3 quantisation kernels at a config's sizes (X per row, W1 per column)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_14080_b200 import sonic  # noqa: E402
from paper_2512_14080_b200.inputs import CONFIGS, make_inputs  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "7b"]
inp = make_inputs(**c, seed=0, device="cuda")


def t(fn, n=50):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


xr = t(lambda: sonic.sonic_quantize_e4m3_rows(inp.X))
wc = t(lambda: sonic.sonic_quantize_e4m3_cols(inp.W1))
xb, wb = inp.X.numel() * 3, inp.W1.numel() * 5  # X read twice... rows: read 2x + write 1x; cols: read 2x + write
print(f"rows X {tuple(inp.X.shape)}: {xr:.1f} us ({inp.X.numel() * 5 / xr / 1e3:.0f} GB/s at 2 reads + 1 write)")
print(f"cols W1 {tuple(inp.W1.shape)}: {wc:.1f} us ({inp.W1.numel() * 5 / wc / 1e3:.0f} GB/s at 2 reads + 1 write)")
