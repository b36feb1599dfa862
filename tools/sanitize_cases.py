"""Small route + fwd + bwd cases that together launch every libsonic kernel variant, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck): tools/sanitize.sh runs this
under each tool.  No oracle, no timing: the cases only have to exercise the code paths.

  python tools/sanitize_cases.py [--ep]     (--ep adds the expert-parallel virtual-rank cases)
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_14080_b200 import sonic  # noqa: E402
from paper_2512_14080_b200.inputs import make_inputs  # noqa: E402

R = sonic
CASES = [
    # (label, T, d, n, E, K, route mode, flags)
    ("tiny_tc n32 (1-CTA kinds, dH BN=32)", 256, 64, 32, 8, 2, R.SONIC_ROUTE_TC, 0),
    ("tiny_tr n32", 256, 64, 32, 8, 2, R.SONIC_ROUTE_TR_NRF, 0),
    ("ragged_tc n64 (BN 128 2-CTA + 64 1-CTA)", 1000, 128, 64, 16, 4, R.SONIC_ROUTE_TC, 0),
    ("multi_tr n128 (fused up/down NU=1)", 2048, 256, 128, 16, 4, R.SONIC_ROUTE_TR_NRF, R.SONIC_F_FUSED_UPDOWN),
    ("n256 fused NU=2, dH ring, half pairs", 512, 256, 256, 64, 8, R.SONIC_ROUTE_TC, R.SONIC_F_FUSED_UPDOWN),
    ("n256 unfused up/down kernels", 512, 256, 256, 64, 8, R.SONIC_ROUTE_TC, 0),
    ("fused D jobs of 128 columns", 1000, 384, 128, 16, 4, R.SONIC_ROUTE_TC, R.SONIC_F_FUSED_UPDOWN),
    ("wide n384 (dH 3 N-tiles + dS reduce)", 1024, 256, 384, 8, 2, R.SONIC_ROUTE_TC, 0),
    ("bf16 dW", 1000, 192, 384, 8, 2, R.SONIC_ROUTE_TC, R.SONIC_F_DW_BF16),
    ("dW accumulate, empty experts", 64, 128, 64, 64, 2, R.SONIC_ROUTE_TC, R.SONIC_F_DW_ACCUMULATE),
    ("EC, E > 128", 4097, 128, 64, 256, 8, R.SONIC_ROUTE_EC, 0),
    ("E = 1 single pair tile", 300, 128, 64, 1, 1, R.SONIC_ROUTE_TC, 0),
    ("TR up", 1000, 128, 64, 16, 4, R.SONIC_ROUTE_TR_UP, 0),
    ("TR down", 1000, 128, 64, 16, 4, R.SONIC_ROUTE_TR_DOWN, 0),
    ("TR balance", 1000, 128, 64, 16, 4, R.SONIC_ROUTE_TR_BALANCE, 0),
    ("TR SR", 1000, 128, 64, 16, 4, R.SONIC_ROUTE_TR_SR, 0),
    ("TR NR-s", 1000, 128, 64, 16, 4, R.SONIC_ROUTE_TR_NRS, 0),
    ("many experts E=260 K=8", 1500, 64, 64, 260, 8, R.SONIC_ROUTE_TC, 0),
]


def run_case(label, T, d, n, E, K, mode, flags):
    inp = make_inputs(T, d, n, E, K, seed=7, device="cuda")
    desc = sonic.make_desc(T, d, n, E, K, mode=mode, flags=flags, seed=99)
    rt = sonic.sonic_route(desc, inp.S)
    O, H, _ = sonic.sonic_moe_fwd(desc, inp.X, inp.W1, inp.W2, rt)
    kw = {}
    if flags & sonic.SONIC_F_DW_ACCUMULATE:
        kw = dict(dW1=torch.zeros(E, d, 2 * n, device="cuda"), dW2=torch.zeros(E, n, d, device="cuda"))
    dX, dW1, dW2, dS, _ = sonic.sonic_moe_bwd(desc, inp.dO, inp.X, H, inp.W1, inp.W2, rt, **kw)
    if mode != sonic.SONIC_ROUTE_GIVEN:
        sonic.sonic_router_bwd(desc, inp.S, rt, dS)
    torch.cuda.synchronize()
    ok = bool(torch.isfinite(O.float()).all() and torch.isfinite(dX.float()).all())
    print(f"case {label}: ok={ok}", flush=True)


def run_ep(peer=False):
    from paper_2512_14080_b200 import ep
    T, d, n, E, K, G = 384, 128, 64, 16, 4, 2
    base = make_inputs(T, d, n, E, K, seed=40, device="cuda")
    L = E // G
    # the peer exchange's flag barriers spin until every virtual rank's kernel runs: under a sanitizer
    # (launches serialised) that never happens, so the peer path is only run on request (--ep-peer)
    for comm_kind in (("sim", "peer") if peer else ("sim",)):
        ins = [make_inputs(T, d, n, E, K, seed=41 + r, device="cuda") for r in range(G)]
        ranks = [ep.EPRank(T, d, n, E, K, G, r, base.W1[r * L:(r + 1) * L].contiguous(),
                           base.W2[r * L:(r + 1) * L].contiguous(), mode=sonic.SONIC_ROUTE_TR_NRF) for r in range(G)]
        comm = ep.SimComm(G) if comm_kind == "sim" else ep.PeerComm(G, T, d, L, range(G))
        ep.ep_forward(ranks, comm, [i.X for i in ins], [i.S for i in ins])
        ep.ep_backward(ranks, comm, [i.dO for i in ins])
        torch.cuda.synchronize()
        if comm_kind == "peer":
            comm.close()
        print(f"case ep G={G} {comm_kind}: ok", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ep", action="store_true")
    ap.add_argument("--ep-peer", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for c in CASES:
        if a.only and not any(o in c[0] for o in a.only.split(",")):
            continue
        run_case(*c)
    if a.ep or a.ep_peer:
        run_ep(peer=a.ep_peer)
