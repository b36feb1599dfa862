"""Expert parallelism across PROCESSES: world_size 2, one rank per process, both on cuda:0 (the GPU
box has one GPU), exchanging through DistComm over gloo (host-staged all-to-all).  This is the code
path bench.py runs under torchrun over NCCL, minus the transport.  Each rank's O, dX, dS and dW
shard are compared with the fp64 oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

T, d, n, E, K = 640, 128, 64, 16, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q, comm_kind="dist"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_14080_b200 import ep, sonic
        from paper_2512_14080_b200.inputs import make_expert_weights, make_token_inputs
        torch.cuda.set_device(0)
        L = E // world
        # drawn on the host (the parent re-draws the same tensors for the oracle), then moved
        X, dO, S = (t.cuda() for t in make_token_inputs(T, d, E, seed=70 + rank))
        W1, W2 = (t.cuda() for t in make_expert_weights(rank * L, (rank + 1) * L, d, n, seed=5))
        m = sonic.SONIC_ROUTE_TC if mode == "tc" else sonic.SONIC_ROUTE_TR_NRF
        rk = ep.EPRank(T, d, n, E, K, world, rank, W1, W2, mode=m)
        # dist: host-staged all-to-all over gloo; peer: CUDA IPC regions (handles exchanged over gloo),
        # the dispatch/return kernels store into the other process's region, flag barriers order them
        comm = (ep.DistComm() if comm_kind.startswith("dist") else
                ep.PeerComm(world, T, d, L, [rank], sync_free=comm_kind == "peer_sf"))
        (O,) = ep.ep_forward([rk], comm, [X], [S], chunked=comm_kind == "dist_chunked")
        ((dX, dS),) = ep.ep_backward([rk], comm, [dO])
        torch.cuda.synchronize()
        if comm_kind.startswith("peer"):
            assert not rk.overflowed()
            O, dX, dS = O.clone(), dX.clone(), dS.clone()
            dist.barrier()  # no rank unmaps its region while a peer may still store into it
            comm.close()
        # numpy by value: torch CPU tensors would travel as shared-memory handles that die with this process
        q.put((rank,) + tuple(t.float().cpu().numpy() for t in (O, dX, dS, rk.dW1, rk.dW2)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,comm_kind", [("tc", "dist"), ("tr", "dist"), ("tc", "peer"), ("tr", "peer"),
                                            ("tc", "peer_sf"), ("tr", "peer_sf"),
                                            ("tc", "dist_chunked"), ("tr", "dist_chunked")])
def test_ep_two_processes(mode, comm_kind):
    from oracle import moe_oracle as om
    from paper_2512_14080_b200.inputs import make_expert_weights, make_token_inputs
    from tests.parity import assert_close, f64

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, mode, q, comm_kind)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, *outs = q.get(timeout=300)
        res[r] = outs
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0

    W1, W2 = make_expert_weights(0, E, d, n, seed=5)
    W1n, W2n = f64(W1), f64(W2)
    dW1_ref, dW2_ref = np.zeros_like(W1n), np.zeros_like(W2n)
    for r in range(world):
        X, dO, S = make_token_inputs(T, d, E, seed=70 + r)
        Xn, dOn = f64(X), f64(dO)
        rto = om.route(S.numpy(), K, mode=mode, m_tile=128)
        fw = om.forward(Xn, W1n, W2n, rto)
        bw = om.backward(dOn, Xn, W1n, W2n, rto)
        O, dX, dS, _, _ = res[r]
        assert_close(f"O[{r}]", O.astype(np.float64), fw.O)
        assert_close(f"dX[{r}]", dX.astype(np.float64), bw.dX)
        rows = np.nonzero(rto.row_token >= 0)[0]
        dSref = np.concatenate([bw.dS[e] for e in range(E) if len(bw.dS[e])])
        assert_close(f"dS[{r}]", dS.astype(np.float64)[rows], dSref)
        dW1_ref += bw.dW1
        dW2_ref += bw.dW2
    assert_close("dW1", np.concatenate([res[r][3] for r in range(world)], 0).astype(np.float64), dW1_ref)
    assert_close("dW2", np.concatenate([res[r][4] for r in range(world)], 0).astype(np.float64), dW2_ref)
