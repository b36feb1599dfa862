"""Router top-K against torch.topk (the paper's motivation for its top-K kernel): time
torch.topk(S, K) + torch's own histogram / sort-based metadata on the 7B router scores, beside the
whole sonic_route (top-K + counts + offsets + gather map + token CSR + gates), CUDA events."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_14080_b200 import sonic  # noqa: E402
from paper_2512_14080_b200.inputs import CONFIGS, make_inputs  # noqa: E402


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for name in ("7b", "kimi"):
    c = CONFIGS[name]
    T, E, K = c["T"], c["E"], c["K"]
    inp = make_inputs(**c, seed=0, device="cuda")
    S = inp.S
    desc = sonic.make_desc(T, c["d"], c["n"], E, K)
    rt = sonic.alloc_routing(desc, "cuda")
    ws = torch.empty(max(256, sonic.sonic_route_workspace_size(desc)), dtype=torch.uint8, device="cuda")

    def torch_router():
        v, i = torch.topk(S, K, dim=1)
        flat = i.flatten()
        counts = torch.bincount(flat, minlength=E)
        order = torch.sort(flat * T + torch.arange(T, device="cuda").repeat_interleave(K), stable=True)[1]
        return v, counts, order

    t_topk = timed(lambda: torch.topk(S, K, dim=1))
    t_torch = timed(torch_router)
    t_sonic = timed(lambda: sonic.sonic_route(desc, S, rt, ws))
    print(f"{name}: T={T} E={E} K={K}  torch.topk {t_topk:7.1f} us | torch topk+bincount+sort {t_torch:7.1f} us | "
          f"sonic_route (all metadata) {t_sonic:7.1f} us")
