"""DistComm plumbing on CPU: world_size 2 over gloo (127.0.0.1).  Checks the count exchange and the
variable-size all-to-all that carry the expert-parallel dispatch/combine (ep.py), including empty
splits, against what each rank must receive."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_14080_b200.ep import DistComm
        comm = DistComm()
        # rank r sends (r+1)*(g+1) rows to rank g (rank 1 sends none to rank 0 -> empty split)
        sc = [(rank + 1) * (g + 1) if not (rank == 1 and g == 0) else 0 for g in range(world)]
        rc = comm.exchange_counts([sc])[0]
        # two count blocks in one exchange (send rows | routed pairs per destination)
        rc2 = comm.exchange_counts([sc + [10 * rank + g for g in range(world)]])[0]
        assert rc2 == rc + [10 * s + rank for s in range(world)], rc2
        rows = []
        for g in range(world):
            rows += [[rank * 1000 + g * 100 + i, -1.0] for i in range(sc[g])]
        send = torch.tensor(rows, dtype=torch.float32).view(-1, 2) if rows else torch.zeros(0, 2)
        (recv,) = comm.alltoallv([send], [sc], [rc])
        q.put((rank, rc, recv[:, 0].tolist()))
    finally:
        dist.destroy_process_group()


def test_distcomm_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, rc, vals = q.get(timeout=120)
        res[r] = (rc, vals)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    # expected: rank g receives from source s the rows s*1000 + g*100 + i, i < count(s->g), sources ascending
    for g in range(world):
        want_counts, want_vals = [], []
        for s in range(world):
            c = (s + 1) * (g + 1) if not (s == 1 and g == 0) else 0
            want_counts.append(c)
            want_vals += [float(s * 1000 + g * 100 + i) for i in range(c)]
        assert res[g][0] == want_counts
        assert res[g][1] == want_vals


def test_simcomm_count_blocks():
    from paper_2512_14080_b200.ep import SimComm
    G = 3
    send = [[100 * s + g for g in range(G)] + [1000 * s + g for g in range(G)] for s in range(G)]
    recv = SimComm(G).exchange_counts(send)
    for g in range(G):
        assert recv[g] == [100 * s + g for s in range(G)] + [1000 * s + g for s in range(G)]


def test_chunked_dispatch_geometry():
    """NEXT-2 chunked dispatch, host side: for every rank the self block (taken from the rank's own send
    buffer) and the remote rows before / after it partition the received rows exactly once, the self
    block is as long in the send buffer as in the receive buffer, and the routed-pair bounds of the
    chunks add up to the rank's total (ep._chunk_rows and the pair slices of _ep_forward_chunked)."""
    import random
    from paper_2512_14080_b200 import ep

    class R:  # the fields _chunk_rows reads
        def __init__(self, rank):
            self.rank = rank

    rnd = random.Random(7)
    for G in (1, 2, 3, 8):
        M = [[rnd.choice([0, 0, 1, 5, 17, 128]) for _ in range(G)] for _ in range(G)]  # M[s][g]: rows s -> g
        P = [[m * rnd.randint(1, 4) for m in row] for row in M]                        # routed pairs s -> g
        for r in range(G):
            sc = M[r]                          # this rank's send counts per destination
            rc = [M[s][r] for s in range(G)]   # rows received from each source
            so, ns, ro = ep._chunk_rows(R(r), sc, rc)
            R_in = sum(rc)
            assert ns == sc[r] == rc[r] and so == sum(sc[:r]) and ro == sum(rc[:r])
            spans = [(ro, ro + ns), (0, ro), (ro + ns, R_in)]
            covered = sorted(i for lo, hi in spans for i in range(lo, hi))
            assert covered == list(range(R_in))
            pr = [P[s][r] for s in range(G)]
            assert pr[r] + sum(pr[:r]) + sum(pr[r + 1:]) == sum(pr)
