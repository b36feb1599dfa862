"""Expert-parallel layer on one GPU: G virtual ranks exchange through SimComm or through peer memory
(PeerComm: each virtual rank drives its own stream, the dispatch kernels store into the other
ranks' regions and the flag barriers order the phases; the same ep.py code runs one rank per process
over NCCL or CUDA IPC).  Every rank's outputs are compared with the fp64 oracle run
on that rank's own microbatch with the full expert set; dW shards with the oracle's dW summed over
all ranks' tokens."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as om
from paper_2512_14080_b200 import ep, sonic
from paper_2512_14080_b200.inputs import make_inputs
from tests.parity import assert_close, f64

pytestmark = pytest.mark.gpu


def _run_ep(G, mode, E, comm_kind, T=768, d=128, n=64, K=4, steps=1, cap_pairs=None, chunked=False):
    m = sonic.SONIC_ROUTE_TC if mode == "tc" else sonic.SONIC_ROUTE_TR_NRF
    base = make_inputs(T, d, n, E, K, seed=40, device="cuda")
    W1, W2 = base.W1, base.W2
    L = E // G
    ins = [make_inputs(T, d, n, E, K, seed=41 + r, device="cuda") for r in range(G)]
    ranks = [ep.EPRank(T, d, n, E, K, G, r, W1[r * L:(r + 1) * L].contiguous(), W2[r * L:(r + 1) * L].contiguous(),
                       mode=m) for r in range(G)]
    comm = (ep.SimComm(G) if comm_kind == "sim" else
            ep.PeerComm(G, T, d, L, range(G), sync_free=comm_kind == "peer_sf", cap_pairs=cap_pairs))
    for _ in range(steps):  # later steps reuse the regions (stale rows of the earlier step)
        Os = ep.ep_forward(ranks, comm, [i.X for i in ins], [i.S for i in ins], chunked=chunked)
        outs = ep.ep_backward(ranks, comm, [i.dO for i in ins])
    torch.cuda.synchronize()
    res = [(Os[r].clone(), outs[r][0].clone(), outs[r][1].clone(), ranks[r].dW1.clone(), ranks[r].dW2.clone())
           for r in range(G)]
    if comm_kind.startswith("peer"):
        comm.close()
    if comm_kind == "peer_sf":
        res.append([rk.overflowed() for rk in ranks])
    return res


@pytest.mark.parametrize("G,mode,E", [(2, "tc", 16), (4, "tr", 16), (2, "tc", 64)])
def test_ep_peer_equals_sim(G, mode, E):
    """The peer-memory exchange moves the same rows to the same places as the staged exchange: every
    output of every rank is bit-identical."""
    a = _run_ep(G, mode, E, "sim")
    b = _run_ep(G, mode, E, "peer")
    for r in range(G):
        for name, x, y in zip(("O", "dX", "dS", "dW1", "dW2"), a[r], b[r]):
            assert torch.equal(x, y), f"rank {r} {name} differs between SimComm and PeerComm"


@pytest.mark.parametrize("G,mode,E,comm_kind", [(1, "tc", 16, "sim"), (2, "tc", 16, "sim"), (4, "tc", 16, "sim"),
                                                (2, "tr", 16, "sim"), (4, "tr", 16, "sim"), (2, "tc", 64, "sim"),
                                                (2, "tc", 16, "peer"), (4, "tr", 16, "peer")])
def test_ep_matches_oracle(G, mode, E, comm_kind):
    """E = 64 over 2 ranks: 32 local experts, so the receive side's GIVEN routing has K = 32 > 16."""
    T, d, n, K = 768, 128, 64, 4
    m = sonic.SONIC_ROUTE_TC if mode == "tc" else sonic.SONIC_ROUTE_TR_NRF
    base = make_inputs(T, d, n, E, K, seed=40, device="cuda")
    W1, W2 = base.W1, base.W2
    L = E // G
    ins = [make_inputs(T, d, n, E, K, seed=41 + r, device="cuda") for r in range(G)]
    ranks = [ep.EPRank(T, d, n, E, K, G, r, W1[r * L:(r + 1) * L].contiguous(), W2[r * L:(r + 1) * L].contiguous(),
                       mode=m) for r in range(G)]
    comm = ep.SimComm(G) if comm_kind == "sim" else ep.PeerComm(G, T, d, L, range(G))
    Os = ep.ep_forward(ranks, comm, [i.X for i in ins], [i.S for i in ins])
    outs = ep.ep_backward(ranks, comm, [i.dO for i in ins])
    torch.cuda.synchronize()
    for rk in ranks:  # the receive side is sized by the routed pairs, not R_in * L
        ld, lrt = rk.ctx["ldesc"], rk.ctx["lrt"]
        assert ld.rows_cap > 0 and sonic.sonic_rows_max(ld) <= int(lrt.offsets[L]) + L * 127 + 127
    W1n, W2n = f64(W1), f64(W2)
    dW1_ref = np.zeros_like(W1n)
    dW2_ref = np.zeros_like(W2n)
    for r in range(G):
        X, dO, S = f64(ins[r].X), f64(ins[r].dO), ins[r].S.cpu().numpy()
        rto = om.route(S, K, mode=mode, m_tile=128)  # TR is per source-rank microbatch (Q19)
        fw = om.forward(X, W1n, W2n, rto)
        bw = om.backward(dO, X, W1n, W2n, rto)
        assert_close(f"O[{r}]", f64(Os[r]), fw.O)
        assert_close(f"dX[{r}]", f64(outs[r][0]), bw.dX)
        dW1_ref += bw.dW1
        dW2_ref += bw.dW2
        rows = np.nonzero(rto.row_token >= 0)[0]
        dSref = np.concatenate([bw.dS[e] for e in range(E) if len(bw.dS[e])])
        assert_close(f"dS[{r}]", f64(outs[r][1])[rows], dSref)
    dW1 = np.concatenate([f64(rk.dW1) for rk in ranks], 0)
    dW2 = np.concatenate([f64(rk.dW2) for rk in ranks], 0)
    assert_close("dW1", dW1, dW1_ref)
    assert_close("dW2", dW2, dW2_ref)
    if comm_kind == "peer":
        comm.close()


def test_ep_plan_dedup():
    """One send row per (token, destination rank); counts add up; rows ascend per rank."""
    T, d, n, E, K, G = 1000, 64, 64, 32, 8, 4
    inp = make_inputs(T, d, n, E, K, seed=7, device="cuda")
    desc = sonic.make_desc(T, d, n, E, K)
    rt = sonic.sonic_route(desc, inp.S)
    plan = sonic.sonic_ep_build_plan(desc, G, rt)
    torch.cuda.synchronize()
    ids = rt.topk_ids[: T * K].view(T, K).cpu().numpy()
    L = E // G
    want = np.zeros(G, int)
    for t in range(T):
        for g in set((ids[t] // L).tolist()):
            want[g] += 1
    cnt = plan.send_counts[:G].cpu().numpy()
    assert np.array_equal(cnt, want)
    off = plan.send_offsets[: G + 1].cpu().numpy()
    tok = plan.send_token[: off[G]].cpu().numpy()
    for g in range(G):
        seg = tok[off[g]: off[g + 1]]
        assert np.all(np.diff(seg) > 0)
        assert set(seg.tolist()) == {t for t in range(T) if g in set((ids[t] // L).tolist())}


@pytest.mark.parametrize("comm_kind", ["sim", "peer"])
def test_ep_zero_gate_pairs_keep_their_rows(comm_kind):
    """A routed (token, expert) pair whose gate is exactly 0 (K = E picks zero scores) contributes
    nothing to O but has dS = <dA', A> != 0.  The dispatch sends it as -0.0 so the receiving rank's
    GIVEN routing keeps the row: dS matches the single-GPU oracle on every kept pair."""
    G, T, d, n, E, K = 2, 256, 128, 64, 8, 8
    base = make_inputs(T, d, n, E, K, seed=50, device="cuda")
    L = E // G
    ins = [make_inputs(T, d, n, E, K, seed=51 + r, device="cuda") for r in range(G)]
    for r, i in enumerate(ins):  # zero scores on two experts (one per rank) for every other token
        S = i.S.clone()
        S[::2, 1] = 0.0
        S[1::2, 6] = 0.0
        i.S = (S / S.sum(1, keepdim=True)).contiguous()
        i.S[::2, 1] = 0.0
        i.S[1::2, 6] = 0.0
    ranks = [ep.EPRank(T, d, n, E, K, G, r, base.W1[r * L:(r + 1) * L].contiguous(),
                       base.W2[r * L:(r + 1) * L].contiguous(), mode=sonic.SONIC_ROUTE_TC) for r in range(G)]
    comm = ep.SimComm(G) if comm_kind == "sim" else ep.PeerComm(G, T, d, L, range(G))
    ep.ep_forward(ranks, comm, [i.X for i in ins], [i.S for i in ins])
    outs = ep.ep_backward(ranks, comm, [i.dO for i in ins])
    torch.cuda.synchronize()
    W1n, W2n = f64(base.W1), f64(base.W2)
    for r in range(G):
        S = ins[r].S.cpu().numpy()
        rto = om.route(S, K, mode="tc", m_tile=128)
        assert (rto.kept & (S == 0)).sum() == T  # the zero-score pairs are routed
        bw = om.backward(f64(ins[r].dO), f64(ins[r].X), W1n, W2n, rto)
        rows = np.nonzero(rto.row_token >= 0)[0]
        dSref = np.concatenate([bw.dS[e] for e in range(E) if len(bw.dS[e])])
        zero_rows = rows[rto.row_gate[rows] == 0]
        assert np.all(np.abs(dSref[np.isin(rows, zero_rows)]) > 0)
        assert_close(f"dS[{r}]", f64(outs[r][1])[rows], dSref)
    if comm_kind == "peer":
        comm.close()


@pytest.mark.parametrize("G,mode,E", [(2, "tc", 16), (4, "tr", 16), (2, "tc", 64)])
def test_ep_sync_free_equals_sim(G, mode, E):
    """NEXT-2: the host-sync-free peer exchange (offsets read on the device, capacity-sized receive
    side with the routed-pair guard) gives every rank bit-identical outputs to the staged exchange,
    also on a second step over regions holding the first step's rows; no rank overflows."""
    a = _run_ep(G, mode, E, "sim")
    b = _run_ep(G, mode, E, "peer_sf", steps=2)
    assert not any(b[G]), "unexpected capacity overflow"
    for r in range(G):
        for name, x, y in zip(("O", "dX", "dS", "dW1", "dW2"), a[r], b[r]):
            assert torch.equal(x, y), f"rank {r} {name} differs between SimComm and the sync-free PeerComm"


def test_ep_sync_free_overflow_is_flagged():
    """A capacity below the received routed pairs: the guarded GIVEN routing empties the rank's
    routing (nothing written out of bounds, its expert outputs are zero) and overflowed() says so."""
    res = _run_ep(2, "tc", 16, "peer_sf", cap_pairs=64)
    assert all(res[2])


@pytest.mark.parametrize("G,mode,E", [(1, "tc", 16), (2, "tc", 16), (4, "tr", 16), (4, "tc", 64), (8, "tr", 64)])
def test_ep_chunked_equals_unchunked(G, mode, E):
    """NEXT-2 chunked dispatch (the self block computed before the remote blocks arrive, each chunk
    its own GIVEN routing and GEMMs): every row's arithmetic is the unchunked one, so O, dX and dS are
    bit-identical; dW1 / dW2 sum the chunks' fp32 partials (SONIC_F_DW_ACCUMULATE), equal to the
    one-pass sums up to fp32 reassociation."""
    a = _run_ep(G, mode, E, "sim")
    b = _run_ep(G, mode, E, "sim", chunked=True, steps=2)
    for r in range(G):
        for name, x, y in zip(("O", "dX", "dS"), a[r][:3], b[r][:3]):
            assert torch.equal(x, y), f"rank {r} {name} differs between chunked and unchunked dispatch"
        for name, x, y in zip(("dW1", "dW2"), a[r][3:], b[r][3:]):
            err = (x - y).abs().max().item()
            assert err <= 1e-5 * max(1.0, x.abs().max().item()), f"rank {r} {name}: max |diff| {err}"
