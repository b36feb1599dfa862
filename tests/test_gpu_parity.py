"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle."""
import pytest
import torch

from paper_2512_14080_b200 import sonic
from paper_2512_14080_b200.inputs import CONFIGS, make_inputs
from tests.parity import full_parity

pytestmark = pytest.mark.gpu

SMALL = [
    # (name, T, d, n, E, K, mode)
    ("tiny_tc", 256, 64, 32, 8, 2, "tc"),
    ("tiny_tr", 256, 64, 32, 8, 2, "tr"),
    ("ragged_tc", 1000, 128, 64, 16, 4, "tc"),        # ragged T, pad rows, several tiles
    ("multi_tc", 2048, 256, 128, 16, 4, "tc"),        # BN=256 paths, K-loop of 4
    ("multi_tr", 2048, 256, 128, 16, 4, "tr"),
    ("wide_n_tc", 1024, 256, 384, 8, 2, "tc"),       # dH with 3 N-tiles (dS partials)
    ("many_e_tc", 512, 128, 64, 64, 8, "tc"),         # empty / tiny experts
    # n = 256: the dH kernel's BN = 256 H-chunk ring (the 7B production path); 2048 rows per expert:
    # 32 k-blocks in the varlen-K dW kernels, past the 16-deep gather-index ring (ring refill)
    ("n256_tc", 8192, 256, 256, 8, 2, "tc"),
    ("n256_tr", 8192, 256, 256, 8, 2, "tr"),
    # the 7B layer's d and n (every 7B kernel configuration) with 8 experts of ~2048 rows
    ("7b_dims_tc", 8192, 1536, 256, 8, 2, "tc"),
    ("7b_dims_tr", 8191, 1536, 256, 8, 2, "tr"),
    # the fused up/down kernel: D jobs of 128 columns (d % 256 != 0); empty experts and half pairs
    # (experts with one 128-row tile) with n = 256
    ("fused_bnd128_tc", 1000, 384, 128, 16, 4, "tc"),
    ("fused_many_e_tc", 512, 256, 256, 64, 8, "tc"),
]


@pytest.mark.parametrize("case", SMALL, ids=[c[0] for c in SMALL])
def test_small_parity(case):
    name, T, d, n, E, K, mode = case
    inp = make_inputs(T, d, n, E, K, seed=1, device="cuda")
    m = sonic.SONIC_ROUTE_TC if mode == "tc" else sonic.SONIC_ROUTE_TR_NRF
    # the fused up/down kernel is opt-in (SONIC_F_FUSED_UPDOWN); the fused_* shapes exercise it
    desc = sonic.make_desc(T, d, n, E, K, mode=m, flags=sonic.SONIC_F_FUSED_UPDOWN if name.startswith("fused") else 0)
    stats = full_parity(desc, inp, mode=mode)
    print(name, {k: f"{v[0]:.2e}/{v[1]:.2e}" for k, v in stats.items()})


# NEXT-3: the other token-rounding subroutines and expert choice, against the oracle
VARIANTS = [
    ("up", sonic.SONIC_ROUTE_TR_UP), ("down", sonic.SONIC_ROUTE_TR_DOWN),
    ("balance", sonic.SONIC_ROUTE_TR_BALANCE), ("sr", sonic.SONIC_ROUTE_TR_SR), ("ec", sonic.SONIC_ROUTE_EC),
    ("nrs", sonic.SONIC_ROUTE_TR_NRS),
]


@pytest.mark.parametrize("shape", [(1000, 128, 64, 16, 4), (2048, 256, 128, 16, 4)], ids=["ragged", "multi"])
@pytest.mark.parametrize("name,m", VARIANTS, ids=[v[0] for v in VARIANTS])
def test_routing_variants_parity(name, m, shape):
    T, d, n, E, K = shape
    inp = make_inputs(T, d, n, E, K, seed=2, device="cuda")
    desc = sonic.make_desc(T, d, n, E, K, mode=m, seed=12345)
    mode, rounding = sonic.ROUTE_MODE_NAMES[m]
    stats = full_parity(desc, inp, mode=mode, rounding=rounding)
    print(name, {k: f"{v[0]:.2e}" for k, v in stats.items()})


def test_sr_seed_changes_decisions():
    """SR-f draws depend on the descriptor's seed (and match the oracle for each)."""
    from tests.parity import check_routing, routing_to_numpy
    from oracle import moe_oracle as om
    T, d, n, E, K = 4096, 64, 64, 64, 8
    inp = make_inputs(T, d, n, E, K, seed=4, device="cuda")
    frs = []
    for seed in (1, 2, 3):
        desc = sonic.make_desc(T, d, n, E, K, mode=sonic.SONIC_ROUTE_TR_SR, seed=seed)
        rt = sonic.sonic_route(desc, inp.S)
        torch.cuda.synchronize()
        g = routing_to_numpy(rt, desc)
        check_routing(g, om.route(inp.S.cpu().numpy(), K, mode="tr", rounding="sr", seed=seed))
        frs.append(tuple(g["f_rounded"].tolist()))
    assert len(set(frs)) > 1


@pytest.mark.parametrize("mode,m,flags", [("tc", sonic.SONIC_ROUTE_TC, 0), ("tr", sonic.SONIC_ROUTE_TR_NRF, 0),
                                          ("tc", sonic.SONIC_ROUTE_TC, sonic.SONIC_F_GATE_RAW),
                                          ("ec", sonic.SONIC_ROUTE_EC, 0)], ids=["tc", "tr", "tc_raw", "ec"])
def test_router_bwd_parity(mode, m, flags):
    """NEXT-4: sonic_router_bwd on the GPU's own dS equals the oracle's router_backward (fp64) on that
    same dS (fp32 arithmetic: 1e-5 relative)."""
    import numpy as np
    from oracle import moe_oracle as om
    from tests.parity import routing_to_numpy, check_routing
    T, d, n, E, K = 1000, 128, 64, 16, 4
    inp = make_inputs(T, d, n, E, K, seed=9, device="cuda")
    desc = sonic.make_desc(T, d, n, E, K, mode=m, flags=flags)
    rt = sonic.sonic_route(desc, inp.S)
    O, H, _ = sonic.sonic_moe_fwd(desc, inp.X, inp.W1, inp.W2, rt)
    _, _, _, dS, _ = sonic.sonic_moe_bwd(desc, inp.dO, inp.X, H, inp.W1, inp.W2, rt)
    dl = sonic.sonic_router_bwd(desc, inp.S, rt, dS)
    torch.cuda.synchronize()
    S = inp.S.cpu().numpy()
    rto = om.route(S, K, mode=mode, m_tile=128, gate_raw=bool(flags & sonic.SONIC_F_GATE_RAW))
    check_routing(routing_to_numpy(rt, desc), rto)
    dSg = dS.cpu().numpy().astype(np.float64)
    dense = np.zeros((T, E))
    rows = np.nonzero(rto.row_token >= 0)[0]
    dense[rto.row_token[rows], rto.row_expert[rows]] = dSg[rows]
    ref = om.router_backward(S, rto, dense, gate_raw=bool(flags & sonic.SONIC_F_GATE_RAW))
    got = dl.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-5, err


def test_dw_accumulate():
    """SONIC_F_DW_ACCUMULATE: dW += (the overwrite result), bit-exactly (one fp32 add per element);
    experts with no rows keep their initial values."""
    T, d, n, E, K = 64, 128, 64, 64, 2  # 64 experts, 128 rows: some experts have no rows
    inp = make_inputs(T, d, n, E, K, seed=13, device="cuda")
    desc = sonic.make_desc(T, d, n, E, K)
    rt = sonic.sonic_route(desc, inp.S)
    O, H, _ = sonic.sonic_moe_fwd(desc, inp.X, inp.W1, inp.W2, rt)
    _, dW1, dW2, _, _ = sonic.sonic_moe_bwd(desc, inp.dO, inp.X, H, inp.W1, inp.W2, rt)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    init1 = torch.randn(dW1.shape, generator=g, device="cuda")
    init2 = torch.randn(dW2.shape, generator=g, device="cuda")
    acc1, acc2 = init1.clone(), init2.clone()
    dacc = sonic.make_desc(T, d, n, E, K, flags=sonic.SONIC_F_DW_ACCUMULATE)
    rt2 = sonic.sonic_route(dacc, inp.S)
    sonic.sonic_moe_bwd(dacc, inp.dO, inp.X, H, inp.W1, inp.W2, rt2, dW1=acc1, dW2=acc2)
    torch.cuda.synchronize()
    assert torch.equal(acc1, init1 + dW1)
    assert torch.equal(acc2, init2 + dW2)
    empty = (rt.f[:E] == 0).nonzero().flatten()
    assert len(empty) > 0 and torch.equal(acc1[empty], init1[empty])


M256 = [
    # (T, d, n, E, K, mode, rounding): token rounding / expert choice to 256-row multiples (Q16)
    (4096, 128, 64, 16, 4, "tr", "nrf"),
    (3000, 128, 64, 16, 4, "tr", "nrf"),     # T not a multiple of 256: capped ups (Q15)
    (4096, 128, 64, 16, 4, "tr", "up"),
    (4096, 128, 64, 16, 4, "tr", "down"),
    (4096, 128, 64, 16, 4, "tr", "balance"),
    (4096, 128, 64, 16, 4, "ec", "nrf"),
]
_M256_MODE = {("tr", "nrf"): sonic.SONIC_ROUTE_TR_NRF, ("tr", "up"): 3, ("tr", "down"): 4, ("tr", "balance"): 5,
              ("ec", "nrf"): 7}


@pytest.mark.parametrize("case", M256, ids=[f"T{c[0]}_{c[5]}_{c[6]}" for c in M256])
def test_m_tile_256(case):
    """m_tile = 256 (a 2-CTA pair's M tile): routing bit-exact vs the oracle at M = 256, every
    kept count a multiple of 256 (or capped at T), values within tolerance."""
    T, d, n, E, K, mode, rounding = case
    inp = make_inputs(T, d, n, E, K, seed=23, device="cuda")
    desc = sonic.make_desc(T, d, n, E, K, mode=_M256_MODE[(mode, rounding)], m_tile=256)
    full_parity(desc, inp, mode=mode, rounding=rounding)
    rt = sonic.sonic_route(desc, inp.S)
    fr = rt.f_rounded[:E].cpu()
    assert bool(((fr % 256 == 0) | (fr == T)).all())


@pytest.mark.parametrize("shape", [(64, 128, 64, 64, 2), (2048, 256, 128, 16, 4), (1000, 192, 384, 8, 2)],
                         ids=["empty_experts", "multi", "wide_n"])
def test_dw_bf16(shape):
    """SONIC_F_DW_BF16: dW1 / dW2 stored as bf16 are the fp32 results rounded to nearest even, bit for bit
    (same fp32 accumulation; experts with no rows get zeros); with DW_ACCUMULATE the call is rejected."""
    T, d, n, E, K = shape
    inp = make_inputs(T, d, n, E, K, seed=17, device="cuda")
    desc = sonic.make_desc(T, d, n, E, K)
    rt = sonic.sonic_route(desc, inp.S)
    O, H, _ = sonic.sonic_moe_fwd(desc, inp.X, inp.W1, inp.W2, rt)
    _, dW1, dW2, _, _ = sonic.sonic_moe_bwd(desc, inp.dO, inp.X, H, inp.W1, inp.W2, rt)
    db = sonic.make_desc(T, d, n, E, K, flags=sonic.SONIC_F_DW_BF16)
    rtb = sonic.sonic_route(db, inp.S)
    _, b1, b2, _, _ = sonic.sonic_moe_bwd(db, inp.dO, inp.X, H, inp.W1, inp.W2, rtb)
    torch.cuda.synchronize()
    assert b1.dtype == torch.bfloat16 and b2.dtype == torch.bfloat16
    assert torch.equal(b1, dW1.to(torch.bfloat16)) and torch.equal(b2, dW2.to(torch.bfloat16))
    bad = sonic.make_desc(T, d, n, E, K, flags=sonic.SONIC_F_DW_BF16 | sonic.SONIC_F_DW_ACCUMULATE)
    with pytest.raises(sonic.SonicError):
        sonic.sonic_moe_bwd(bad, inp.dO, inp.X, H, inp.W1, inp.W2, rtb)


# Shape sweep over the edge cases of the routing and GEMM paths: E not a multiple of 4 or 32
# (scalar S staging, partial expert chunks), E > 128 (several S slabs), K = 1, tiny / ragged T,
# n = 32 and 64, d = 64.
FUZZ = [
    # (T, d, n, E, K, mode)
    (33, 64, 32, 5, 1, "tc"),
    (97, 64, 64, 33, 3, "tr"),
    (300, 128, 64, 200, 6, "tc"),
    (300, 128, 64, 200, 6, "tr"),
    (777, 64, 32, 7, 7, "tr"),
    (129, 192, 128, 130, 2, "ec"),
    (1500, 64, 64, 260, 8, "tc"),
    (1, 64, 32, 1, 1, "tc"),      # a single token, a single expert
    (1, 64, 32, 4, 2, "tr"),      # TR with T < m_tile: every chosen "up" is capped at T (Q15)
    (2, 64, 64, 3, 3, "tr"),      # K = E with two tokens
    (4097, 128, 64, 256, 8, "ec"),  # EC with E > 128 and T K not divisible by E (rows bound)
    (300, 128, 64, 1, 1, "tc"),   # E = 1 with 2-CTA dW tiles: a single varlen-K pair tile
    (64, 128, 128, 1, 1, "tr"),
]


@pytest.mark.parametrize("case", FUZZ, ids=[f"T{c[0]}_d{c[1]}_n{c[2]}_E{c[3]}_K{c[4]}_{c[5]}" for c in FUZZ])
def test_shape_sweep(case):
    T, d, n, E, K, mode = case
    inp = make_inputs(T, d, n, E, K, seed=T + E, device="cuda")
    m = {"tc": sonic.SONIC_ROUTE_TC, "tr": sonic.SONIC_ROUTE_TR_NRF, "ec": sonic.SONIC_ROUTE_EC}[mode]
    desc = sonic.make_desc(T, d, n, E, K, mode=m)
    full_parity(desc, inp, mode=mode)


def test_split_backward_matches_monolithic():
    """SONIC_F_BWD_NO_DW then SONIC_F_BWD_DW_ONLY (same workspace) give exactly the one-call result."""
    T, d, n, E, K = 1000, 128, 64, 16, 4
    inp = make_inputs(T, d, n, E, K, seed=17, device="cuda")
    desc = sonic.make_desc(T, d, n, E, K)
    rt = sonic.sonic_route(desc, inp.S)
    O, H, _ = sonic.sonic_moe_fwd(desc, inp.X, inp.W1, inp.W2, rt)
    dX, dW1, dW2, dS, _ = sonic.sonic_moe_bwd(desc, inp.dO, inp.X, H, inp.W1, inp.W2, rt)
    d1 = sonic.make_desc(T, d, n, E, K, flags=sonic.SONIC_F_BWD_NO_DW)
    d2 = sonic.make_desc(T, d, n, E, K, flags=sonic.SONIC_F_BWD_DW_ONLY)
    dXa, w1a, w2a, dSa, ws = sonic.sonic_moe_bwd(d1, inp.dO, inp.X, H, inp.W1, inp.W2, rt)
    assert w1a is None and w2a is None
    dXb, w1b, w2b, dSb, _ = sonic.sonic_moe_bwd(d2, inp.dO, inp.X, H, inp.W1, inp.W2, rt, ws=ws)
    assert dXb is None and dSb is None
    torch.cuda.synchronize()
    R = int(rt.offsets[E].item())
    assert torch.equal(dXa, dX) and torch.equal(w1b, dW1) and torch.equal(w2b, dW2)
    assert torch.equal(dSa[:R], dS[:R])


@pytest.mark.parametrize("shape,mode", [((2048, 256, 128, 16, 4), "tc"), ((8192, 1536, 256, 8, 2), "tr"),
                                        ((512, 256, 256, 64, 8), "tc")], ids=["n128", "7b_dims_tr", "half_pairs"])
def test_fused_updown_equals_two_kernels(shape, mode):
    """NEXT-1: the fused up/down kernel (A kept in shared memory) gives the same H and O as the
    separate up- and down-projection kernels (the default) bit for bit: the same MMA shapes and K
    order, the same bf16 A; and the fused path is parity-green against the oracle."""
    T, d, n, E, K = shape
    inp = make_inputs(T, d, n, E, K, seed=31, device="cuda")
    m = sonic.SONIC_ROUTE_TC if mode == "tc" else sonic.SONIC_ROUTE_TR_NRF
    d_f = sonic.make_desc(T, d, n, E, K, mode=m, flags=sonic.SONIC_F_FUSED_UPDOWN)
    d_u = sonic.make_desc(T, d, n, E, K, mode=m)
    assert sonic.sonic_fwd_workspace_size(d_f) < sonic.sonic_fwd_workspace_size(d_u)  # no A in the workspace
    rt = sonic.sonic_route(d_f, inp.S)
    Of, Hf, _ = sonic.sonic_moe_fwd(d_f, inp.X, inp.W1, inp.W2, rt)
    Ou, Hu, _ = sonic.sonic_moe_fwd(d_u, inp.X, inp.W1, inp.W2, rt)
    torch.cuda.synchronize()
    R_pad = int(rt.pad_offsets[E])
    assert torch.equal(Hf[:R_pad], Hu[:R_pad])
    assert torch.equal(Of, Ou)
    full_parity(d_f, inp, mode=mode)


POISON = [
    # every GEMM template instance (1-CTA and 2-CTA kinds, fused and unfused up/down, the dH ring and
    # dS partials), TC and TR, with pad rows, half pairs and empty experts
    ("tiny_tc", 256, 64, 32, 8, 2, "tc", 0),
    ("ragged_tc", 1000, 128, 64, 16, 4, "tc", 0),
    ("multi_tr", 2048, 256, 128, 16, 4, "tr", 0),
    ("n256_half_pairs", 512, 256, 256, 64, 8, "tc", 0),
    ("n256_fused", 512, 256, 256, 64, 8, "tc", sonic.SONIC_F_FUSED_UPDOWN),
    ("n128_fused_tr", 2048, 256, 128, 16, 4, "tr", sonic.SONIC_F_FUSED_UPDOWN),
    ("wide_n_tr", 1024, 256, 384, 8, 2, "tr", 0),
]


@pytest.mark.parametrize("case", POISON, ids=[c[0] for c in POISON])
def test_poisoned_buffers(case):
    """Outputs, routing and workspaces start as NaN / -1 bytes: parity (which rejects NaN) holds, so no
    kernel reads a location that its producer did not write -- including rows written by TMA bulk
    stores, which compute-sanitizer's initcheck does not track (sanitizers)."""
    name, T, d, n, E, K, mode, flags = case
    inp = make_inputs(T, d, n, E, K, seed=5, device="cuda")
    m = sonic.SONIC_ROUTE_TC if mode == "tc" else sonic.SONIC_ROUTE_TR_NRF
    full_parity(sonic.make_desc(T, d, n, E, K, mode=m, flags=flags), inp, mode=mode, poison=True)


# NEXT-4: router softmax fused into the routing, sonic_route_logits
LOGIT_CASES = [
    # (name, T, E, K, route mode): TC with E <= 128 fuses the softmax into the warp top-K; the others
    # run the row-softmax kernel first (TR / EC need S^T; E = 384 > 128; E = 40 is not a multiple of 32)
    ("tc_e128", 4096, 128, 8, sonic.SONIC_ROUTE_TC),
    ("tc_e64_ragged_T", 1000, 64, 4, sonic.SONIC_ROUTE_TC),
    ("tr_e128", 4096, 128, 8, sonic.SONIC_ROUTE_TR_NRF),
    ("ec_e64", 2048, 64, 4, sonic.SONIC_ROUTE_EC),
    ("tc_e384", 2048, 384, 8, sonic.SONIC_ROUTE_TC),
    ("tc_e40", 999, 40, 3, sonic.SONIC_ROUTE_TC),
    ("tc_e1000", 300, 1000, 16, sonic.SONIC_ROUTE_TC),
    ("tc_T1_K1", 1, 64, 1, sonic.SONIC_ROUTE_TC),
    ("tc_K_eq_E", 100, 16, 16, sonic.SONIC_ROUTE_TC),  # K <= 16 (TC)
    ("tr_nrs", 1024, 64, 4, sonic.SONIC_ROUTE_TR_NRS),
]


@pytest.mark.parametrize("case", LOGIT_CASES, ids=[c[0] for c in LOGIT_CASES])
def test_route_logits_fused_softmax(case):
    """S = softmax(logits) within the fp32 bound of the arithmetic stated in include/sonic.h
    ((E + 64) * 2^-24 relative per element: max-subtracted expf, an E-term fp32 sum, one division),
    the routing bit-exact against the oracle's route on that S, and identical to sonic_route(S)."""
    import numpy as np
    from oracle import moe_oracle as om
    from tests.parity import check_routing, routing_to_numpy
    name, T, E, K, m = case
    g = torch.Generator(device="cuda").manual_seed(77)
    logits = torch.randn(T, E, device="cuda", generator=g) * 2.0
    desc = sonic.make_desc(T, 64, 64, E, K, mode=m)
    S, rt = sonic.sonic_route_logits(desc, logits)
    rt2 = sonic.sonic_route(desc, S.clone())
    torch.cuda.synchronize()
    S_ref = om.softmax(logits.double().cpu().numpy())
    Sg = S.double().cpu().numpy()
    bound = (E + 64) * 2.0 ** -24 * S_ref + 1e-40
    assert np.all(np.abs(Sg - S_ref) <= bound), f"{name}: max rel err {np.max(np.abs(Sg - S_ref) / S_ref):.3e}"
    ga, gb = routing_to_numpy(rt, desc), routing_to_numpy(rt2, desc)  # the written extents
    for f in ga:
        assert np.array_equal(ga[f], gb[f]), f"{name}: {f} differs from sonic_route(S)"
    mode, rounding = sonic.ROUTE_MODE_NAMES[m]
    check_routing(ga, om.route(S.cpu().numpy(), K, mode=mode, rounding=rounding))


@pytest.mark.parametrize("shape", [(4096, 256, 128), (1000, 1536, 128), (777, 384, 40)], ids=["7bE", "7bd", "ragged"])
def test_router_gemms(shape):
    """NEXT-4 router GEMMs: logits = X W_r within the fp32-accumulation bound (bf16 products are
    exact in fp32, so |err| <= d 2^-24 sum_k |X_tk W_ke|); dX += dlogits W_r^T and dW_r = X^T dlogits
    (d logits rounded to bf16 for the tensor cores, by design) within the north-star criterion."""
    import numpy as np
    from oracle import moe_oracle as om
    from tests.parity import assert_close
    T, d, E = shape
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    Wr = (torch.randn(d, E, device="cuda", generator=g) / d ** 0.5).bfloat16()
    dl = torch.randn(T, E, device="cuda", generator=g) * 1e-2
    dX0 = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    desc = sonic.make_desc(T, d, 64, E, min(2, E))
    logits = sonic.sonic_router_fwd(desc, X, Wr)
    dX = dX0.clone()
    dX, dWr = sonic.sonic_router_grad(desc, X, Wr, dl, dX=dX)
    torch.cuda.synchronize()
    Xn, Wn = X.double().cpu().numpy(), Wr.double().cpu().numpy()
    ref = om.router_logits(Xn, Wn)
    bound = d * 2.0 ** -24 * (np.abs(Xn) @ np.abs(Wn)) + 1e-30
    assert np.all(np.abs(logits.double().cpu().numpy() - ref) <= bound)
    dX_r, dW_r = om.router_input_grads(Xn, Wn, dl.double().cpu().numpy())
    assert_close("dX", dX.double().cpu().numpy(), dX0.double().cpu().numpy() + dX_r)
    assert_close("dWr", dWr.double().cpu().numpy(), dW_r)


def test_router_full_chain():
    """The training step around the expert layer, all through the C ABI: router GEMM -> fused
    softmax + routing -> MoE fwd/bwd -> router backward (dS -> d logits) -> router GEMM grads;
    dX (expert path + router path) and dW_r against the oracle chain on the same inputs."""
    import numpy as np
    from oracle import moe_oracle as om
    from tests.parity import assert_close
    T, d, n, E, K = 2048, 256, 128, 32, 4
    inp = make_inputs(T, d, n, E, K, seed=8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(6)
    Wr = (torch.randn(d, E, device="cuda", generator=g) / d ** 0.5).bfloat16()
    desc = sonic.make_desc(T, d, n, E, K)
    logits = sonic.sonic_router_fwd(desc, inp.X, Wr)
    S, rt = sonic.sonic_route_logits(desc, logits)
    O, H, _ = sonic.sonic_moe_fwd(desc, inp.X, inp.W1, inp.W2, rt)
    dX, dW1, dW2, dS, _ = sonic.sonic_moe_bwd(desc, inp.dO, inp.X, H, inp.W1, inp.W2, rt)
    dlog = sonic.sonic_router_bwd(desc, S, rt, dS)
    dX, dWr = sonic.sonic_router_grad(desc, inp.X, Wr, dlog, dX=dX)
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()
    Xn, Wn = f(inp.X), f(Wr)
    Sn = S.cpu().numpy()  # the S the GPU routed on (its own parity: test_route_logits_fused_softmax)
    rto = om.route(Sn, K, mode="tc")
    bw = om.backward(f(inp.dO), Xn, f(inp.W1), f(inp.W2), rto)
    dlog_ref = om.router_backward(Sn, rto, om.dS_dense(rto, bw.dS))
    dXr, dWr_ref = om.router_input_grads(Xn, Wn, dlog_ref)
    assert_close("dlogits", f(dlog), dlog_ref)
    assert_close("dX (experts + router)", f(dX), bw.dX + dXr)
    assert_close("dWr", f(dWr), dWr_ref)


# NEXT-4: FP8 (e4m3) up-projection, SONIC_F_FP8_UP
def test_quantize_e4m3_bit_exact():
    """The library's e4m3 quantisation equals the oracle's bit for bit: the codes (through torch's
    float8_e4m3fn view) and the fp32 scales, per token row of X and per output column of W1_e
    (zero rows / columns get scale 1 and zero codes)."""
    import numpy as np
    from oracle import moe_oracle as om
    g = torch.Generator(device="cuda").manual_seed(3)
    X = (torch.randn(1000, 1536, device="cuda", generator=g) * torch.exp(torch.randn(1000, 1, device="cuda",
                                                                                      generator=g))).bfloat16()
    X[7] = 0
    W = (torch.randn(8, 256, 512, device="cuda", generator=g) * 0.05).bfloat16()
    W[2, :, 17] = 0
    xq, sx = sonic.sonic_quantize_e4m3_rows(X)
    wq, sw = sonic.sonic_quantize_e4m3_cols(W)
    torch.cuda.synchronize()
    to_f = lambda q: q.view(torch.float8_e4m3fn).float().cpu().numpy()
    oq, osx = om.quantize_e4m3(X.float().cpu().numpy(), axis=1)
    np.testing.assert_array_equal(to_f(xq), oq)
    np.testing.assert_array_equal(sx.cpu().numpy(), osx.astype(np.float32))
    oq, osw = om.quantize_e4m3(W.float().cpu().numpy(), axis=1)
    np.testing.assert_array_equal(to_f(wq), oq)
    np.testing.assert_array_equal(sw.cpu().numpy(), osw.astype(np.float32))


FP8_CASES = [
    ("fp8_tiny_T1", 1, 128, 128, 4, 2, "tc"),
    ("fp8_tc", 2048, 256, 128, 16, 4, "tc"),
    ("fp8_tr", 2048, 256, 128, 16, 4, "tr"),
    ("fp8_n256_ragged", 1000, 384, 256, 8, 2, "tc"),
    ("fp8_7b_dims", 4096, 1536, 256, 8, 2, "tc"),
]


@pytest.mark.parametrize("case", FP8_CASES, ids=[c[0] for c in FP8_CASES])
def test_fp8_up_parity(case):
    """SONIC_F_FP8_UP: every output of route + fwd + bwd against the oracle whose up-projection
    runs on the same e4m3 operands (forward(fp8_up=True); the backward through the cached H), within
    the north-star criterion; the bf16 layer is only a quantisation error away (checked loosely)."""
    name, T, d, n, E, K, mode = case
    inp = make_inputs(T, d, n, E, K, seed=11, device="cuda")
    m = sonic.SONIC_ROUTE_TC if mode == "tc" else sonic.SONIC_ROUTE_TR_NRF
    desc = sonic.make_desc(T, d, n, E, K, mode=m, flags=sonic.SONIC_F_FP8_UP)
    stats = full_parity(desc, inp, mode=mode)
    print(name, {k: f"{v[0]:.2e}/{v[1]:.2e}" for k, v in stats.items()})


FP8_DXT_CASES = [
    ("fp8dxt_tc", 2048, 256, 128, 16, 4, "tc", 0),
    ("fp8dxt_tr", 2048, 256, 128, 16, 4, "tr", 0),
    ("fp8dxt_n64_ragged", 1000, 512, 64, 8, 2, "tc", 0),
    ("fp8dxt_7b_dims", 4096, 1536, 256, 8, 2, "tc", 0),
    ("fp8dxt_with_fp8_up", 2048, 256, 128, 16, 4, "tc", 1),
    ("fp8dxt_qwen3_dims", 2048, 2048, 768, 8, 2, "tr", 0),
    ("fp8dxt_2n_640_generic", 1024, 256, 320, 4, 2, "tc", 0),
    ("fp8dxt_T1", 1, 256, 64, 4, 2, "tc", 0),
    ("fp8dxt_empty_experts", 40, 256, 128, 32, 2, "tr", 1),
]


@pytest.mark.parametrize("case", FP8_DXT_CASES, ids=[c[0] for c in FP8_DXT_CASES])
def test_fp8_dxt_parity(case):
    """SONIC_F_FP8_DXT: every output of route + fwd + bwd against the oracle whose dX~ runs on the
    e4m3 operands of reading Q25 (backward(fp8_dxt=True): the stored bf16 dH times the forward's
    per-column W1 scales, quantised per row, against the forward's e4m3 W1), within the north-star
    criterion; dH, dS, dW1, dW2 are the bf16 path's.  The GPU quantises its own bf16 dH, the oracle the
    bf16 rounding of its fp64 dH: where the two bf16 values differ by an ulp, an e4m3 code can flip
    (~1/32 of those elements), a perturbation far inside the criterion."""
    name, T, d, n, E, K, mode, up8 = case
    inp = make_inputs(T, d, n, E, K, seed=13, device="cuda")
    m = sonic.SONIC_ROUTE_TC if mode == "tc" else sonic.SONIC_ROUTE_TR_NRF
    fl = sonic.SONIC_F_FP8_DXT | (sonic.SONIC_F_FP8_UP if up8 else 0)
    desc = sonic.make_desc(T, d, n, E, K, mode=m, flags=fl)
    stats = full_parity(desc, inp, mode=mode)
    print(name, {k: f"{v[0]:.2e}/{v[1]:.2e}" for k, v in stats.items()})


def test_fp8_w1_cached_reuses_the_copy():
    """SONIC_F_FP8_W1_CACHED reuses the e4m3 W1 left in the workspace by the previous call: the same
    outputs as quantising again (same W1), and different from a call whose cached copy is stale."""
    T, d, n, E, K = 2048, 256, 128, 16, 4
    inp = make_inputs(T, d, n, E, K, seed=12, device="cuda")
    d8 = sonic.make_desc(T, d, n, E, K, flags=sonic.SONIC_F_FP8_UP)
    dc = sonic.make_desc(T, d, n, E, K, flags=sonic.SONIC_F_FP8_UP | sonic.SONIC_F_FP8_W1_CACHED)
    rt = sonic.sonic_route(d8, inp.S)
    O1, H1, ws = sonic.sonic_moe_fwd(d8, inp.X, inp.W1, inp.W2, rt)
    O2, H2, _ = sonic.sonic_moe_fwd(dc, inp.X, inp.W1, inp.W2, rt, ws=ws)
    O3, _, _ = sonic.sonic_moe_fwd(dc, inp.X, (inp.W1 * 2).contiguous(), inp.W2, rt, ws=ws)  # stale copy used
    torch.cuda.synchronize()
    R_pad = int(rt.pad_offsets[E])  # H rows past R_pad are never written
    assert torch.equal(O1, O2) and torch.equal(H1[:R_pad], H2[:R_pad])
    assert torch.equal(O1, O3)
