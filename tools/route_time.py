"""Time sonic_route alone (CUDA events, back to back, L2 warm) for a config and route mode.
  python tools/route_time.py [config] [mode]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_14080_b200 import sonic  # noqa: E402
from paper_2512_14080_b200.inputs import CONFIGS, make_inputs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "7b"
mode = {"tc": sonic.SONIC_ROUTE_TC, "tr": sonic.SONIC_ROUTE_TR_NRF}[sys.argv[2] if len(sys.argv) > 2 else "tc"]
c = CONFIGS[cfg]
inp = make_inputs(**c, seed=0, device="cuda")
desc = sonic.make_desc(c["T"], c["d"], c["n"], c["E"], c["K"], mode=mode)
rt = sonic.alloc_routing(desc, inp.S.device)
ws = torch.empty(max(256, sonic.sonic_route_workspace_size(desc)), dtype=torch.uint8, device="cuda")
for _ in range(10):
    sonic.sonic_route(desc, inp.S, rt, ws)
torch.cuda.synchronize()
N = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N):
    sonic.sonic_route(desc, inp.S, rt, ws)
e1.record()
torch.cuda.synchronize()
print(f"route {cfg} {sys.argv[2] if len(sys.argv) > 2 else 'tc'}: {e0.elapsed_time(e1) / N * 1e3:.1f} us per call "
      f"({sonic.sonic_last_launch_count()} launches)")
