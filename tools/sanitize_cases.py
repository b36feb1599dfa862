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
    ("fp8 up-projection", 1000, 256, 128, 16, 4, R.SONIC_ROUTE_TC, R.SONIC_F_FP8_UP),
    ("fp8 up-projection TR, n256", 777, 384, 256, 8, 2, R.SONIC_ROUTE_TR_NRF, R.SONIC_F_FP8_UP),
]


def run_router_cases():
    """NEXT-4 router: fused softmax routing (warp top-K path and row-softmax path), router GEMMs
    and the whole router chain."""
    for (T, d, E, K, m) in ((1000, 128, 64, 4, R.SONIC_ROUTE_TC), (999, 128, 40, 3, R.SONIC_ROUTE_TC),
                            (1024, 128, 32, 2, R.SONIC_ROUTE_TR_NRF)):
        g = torch.Generator(device="cuda").manual_seed(3)
        X = torch.randn(T, d, device="cuda", generator=g).bfloat16()
        Wr = (torch.randn(d, E, device="cuda", generator=g) / d ** 0.5).bfloat16()
        desc = sonic.make_desc(T, d, 64, E, K, mode=m)
        logits = sonic.sonic_router_fwd(desc, X, Wr)
        S, rt = sonic.sonic_route_logits(desc, logits)
        dS = torch.randn(sonic.sonic_rows_max(desc), device="cuda", generator=g)
        dlog = sonic.sonic_router_bwd(desc, S, rt, dS)
        dX = torch.zeros(T, d, dtype=torch.bfloat16, device="cuda")
        sonic.sonic_router_grad(desc, X, Wr, dlog, dX=dX)
        torch.cuda.synchronize()
        print(f"case router T={T} E={E}: ok={bool(torch.isfinite(dX.float()).all())}", flush=True)
    xq, sx = sonic.sonic_quantize_e4m3_rows(torch.randn(333, 136, device="cuda").bfloat16())
    wq, sw = sonic.sonic_quantize_e4m3_cols(torch.randn(3, 100, 264, device="cuda").bfloat16())
    torch.cuda.synchronize()
    print("case e4m3 quantisers: ok", flush=True)


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
    if not a.only or "router" in a.only:
        run_router_cases()
    if a.ep or a.ep_peer:
        run_ep(peer=a.ep_peer)
