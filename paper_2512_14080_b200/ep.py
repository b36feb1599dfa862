"""Expert parallelism: G ranks, rank g owns experts [g*L, (g+1)*L), L = E/G.

Per layer and direction there is one exchange each way, an all-to-all-v over NVLink:

  forward   route (own tokens, all E experts) -> plan -> pack X rows + gates -> a2a ->
            GIVEN-route the received rows to the L local experts -> sonic_moe_fwd (its aggregation
            pre-sums the local experts per received row) -> a2a back -> combine (ascending rank);
  backward  pack dO rows -> a2a -> sonic_moe_bwd part 1 (dH, dS, dX~) on the received rows ->
            a2a back of dX~ partial sums and of the dense per-row dS, overlapped with part 2 (the local
            dW2 / dW1, SONIC_F_BWD_DW_ONLY) -> combine dX, scatter dS.

One send row per (token, destination rank): a token whose K experts live on k ranks is sent k
times, not K times.  Every step of the data path runs in libsonic's CUDA kernels; this module only
moves tensors between ranks (torch.distributed all_to_all_single over NCCL -- plumbing) and sizes
buffers (one device->host copy of the G send counts per direction: NCCL takes host split sizes).

The algorithm is written for a LIST of local ranks so that the same code runs
  * one rank per process under torchrun (DistComm, list of length 1), and
  * G virtual ranks in one process on one GPU (SimComm) -- used by the single-GPU tests.
"""
from __future__ import annotations

import contextlib
from dataclasses import dataclass, field

import torch

from . import sonic


# ------------------------------------------------------------------------------- communicators
class SimComm:
    """G virtual ranks in one process: the all-to-all is a local shuffle of device buffers."""

    def __init__(self, G):
        self.G = G

    def exchange_counts(self, send_counts):
        """send_counts[s] (host ints, n blocks of G: block j, entry g = what s sends to g) ->
        recv[g] (n blocks of G: block j, entry s = what g gets from s)."""
        G = self.G
        nb = len(send_counts[0]) // G
        return [[send_counts[s][j * G + g] for j in range(nb) for s in range(G)] for g in range(G)]

    def exchange_counts_dev(self, send_dev):
        """Device count tensors [n*G] per local rank -> (send, recv) host lists, one host read."""
        host = torch.stack(list(send_dev)).cpu().tolist()
        return host, self.exchange_counts(host)

    def rank_stream(self, i):
        return contextlib.nullcontext()

    def alltoallv(self, sends, send_counts, recv_counts, tag=None):
        outs = []
        for g in range(self.G):
            parts = []
            for s in range(self.G):
                off = sum(send_counts[s][:g])
                parts.append(sends[s][off: off + send_counts[s][g]])
            outs.append(parts[0] if len(parts) == 1 else torch.cat(parts, 0))  # G = 1: a view, no copy
        return outs

    def alltoallv_start(self, sends, send_counts, recv_counts, tag=None):
        return self.alltoallv(sends, send_counts, recv_counts)

    def alltoallv_finish(self, pending):
        return pending


class DistComm:
    """One rank per process (torch.distributed; NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.G = dist.get_world_size(group)

    def exchange_counts(self, send_counts):
        """send_counts: [one host list of n blocks of G] -> [recv list, n blocks of G (entry s)]."""
        (sc,) = send_counts
        G = self.G
        nb = len(sc) // G
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor(sc, dtype=torch.int64, device=dev).view(nb, G).t().contiguous()  # row g -> rank g
        r = torch.empty_like(t)
        self.dist.all_to_all_single(r, t, group=self.group)
        return [r.t().reshape(-1).cpu().tolist()]  # row s of r came from s

    def exchange_counts_dev(self, send_dev):
        """The G send counts of this rank (device int32) -> (send, recv) host lists.  Under NCCL the
        count all-to-all runs on the device and one host read fetches both directions."""
        (c,) = send_dev
        G = self.G
        nb = c.numel() // G
        if self.dist.get_backend(self.group) != "nccl":
            sc = c.cpu().tolist()
            return [sc], self.exchange_counts([sc])
        t = c.to(torch.int64).view(nb, G).t().contiguous()
        r = torch.empty_like(t)
        self.dist.all_to_all_single(r, t, group=self.group)
        both = torch.stack([t.t().reshape(-1), r.t().reshape(-1)]).cpu().tolist()
        return [both[0]], [both[1]]

    def rank_stream(self, i):
        return contextlib.nullcontext()

    def alltoallv(self, sends, send_counts, recv_counts, tag=None):
        return self.alltoallv_finish(self.alltoallv_start(sends, send_counts, recv_counts))

    def alltoallv_start(self, sends, send_counts, recv_counts, tag=None):
        """Issue the exchange asynchronously (NCCL runs it on its own stream after the work already
        queued on the current stream); alltoallv_finish makes the current stream wait for it."""
        (s,), (sc,), (rc,) = sends, send_counts, recv_counts
        # gloo (CPU plumbing tests; several ranks sharing one GPU in the tests) exchanges host tensors
        stage = s.is_cuda and self.dist.get_backend(self.group) != "nccl"
        src = s[: sum(sc)].contiguous()
        if stage:
            src = src.cpu()
        out = torch.empty((sum(rc),) + tuple(s.shape[1:]), dtype=s.dtype, device=src.device)
        work = self.dist.all_to_all_single(out, src, output_split_sizes=rc, input_split_sizes=sc, group=self.group,
                                           async_op=True)
        return (out, work, s.device if stage else None, src)

    def alltoallv_finish(self, pending):
        out, work, dev, _src = pending
        work.wait()
        return [out.to(dev) if dev is not None else out]


class PeerComm:
    """The exchange through peer memory (libsonic sonic_peer_*; NEXT-2): no NCCL on the data path.

    Each local rank owns one symmetric region (CUDA IPC across processes -- NVLink peer memory on an
    NVSwitch box -- or raw pointers between virtual ranks of one process).  Region layout, rows of
    capacity NS = T*G (a destination receives at most T rows from each source, a source gets back at
    most its T*G send rows):

      counts [G, G] i32 | x [NS, d] bf16 | gate [NS, L] f32 | do [NS, d] bf16 | back [NS, d] bf16 |
      ds [NS, L] f32

    `back` serves the forward return (Y partial sums) and the backward return (dX~ partial sums):
    the pre-exchange barrier orders the backward's stores after the forward's combine on every rank.
    Each exchange is barrier -> stores into the peers -> barrier on the rank's stream; the dispatch
    stores come straight from the gather (sonic_ep_pack_peer), the returns are block puts.  The only
    host synchronisation is the read of the count matrix (received-row counts size the local GEMMs).

    ranks: the local ranks (one per process under torchrun, or G virtual ranks in one process, each
    on its own CUDA stream so their barriers can meet).

    Lifetime: one PeerComm serves ONE MoE layer with one training step in flight.  The received x
    and dO rows stay views into the region and the backward's dW1 / dW2 read them, so a second
    layer's dispatch through the same PeerComm would overwrite them before the first layer's
    backward (silently wrong weight gradients).  Stack layers with one PeerComm each.
    """

    NB = 2  # count blocks exchanged per rank: send rows per destination, routed pairs per destination

    def __init__(self, G, T, d, L, local_ranks, group=None, device=None, sync_free=False, cap_pairs=None):
        """sync_free (NEXT-2): no host read of the count matrix.  Every block offset is read on the
        device from the own count matrix (sonic_*_dev calls), the receive side works on the
        capacity NS = T*G rows (rows past this step's received ones are zeroed, so they route
        nowhere) and its routed pairs are sized by `cap_pairs` (default 2*T*K of the layer: twice the
        average load) with the capacity guard of sonic_route_given_capped -- a step whose received
        pairs exceed it is flagged (EPRank.overflowed()) and computes nothing on that rank.  The
        whole layer step is then free of host synchronisation (and graph-capturable)."""
        self.G, self.T, self.d, self.L = G, T, d, L
        self.sync_free = bool(sync_free)
        self.cap_pairs = cap_pairs
        self.local = list(local_ranks)
        ns = T * G
        off, lay = 0, {}
        for name, nbytes in (("counts", G * self.NB * G * 4), ("x", ns * d * 2), ("gate", ns * L * 4), ("do", ns * d * 2),
                             ("back", ns * d * 2), ("ds", ns * L * 4)):
            lay[name] = off
            off += (nbytes + 255) // 256 * 256
        self.lay, self.nbytes = lay, off
        self.regions = [sonic.PeerRegion(r, G, off) for r in self.local]
        blobs = [rg.handle() for rg in self.regions]
        if len(self.local) < G:  # one rank per process: exchange the handle blobs (setup only)
            import torch.distributed as dist
            allb = [None] * G
            dist.all_gather_object(allb, blobs[0], group=group)
            blobs = allb
        for rg in self.regions:
            rg.open(blobs)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.streams = [torch.cuda.Stream(device=dev) for _ in self.local] if len(self.local) > 1 else [None]
        self.M = None

    def close(self):
        torch.cuda.synchronize()
        for rg in self.regions:
            rg.close()
        self.regions = []

    # ---------------------------------------------------------------- streams
    @contextlib.contextmanager
    def rank_stream(self, i):
        st = self.streams[i]
        if st is None:
            yield
            return
        st.wait_stream(torch.cuda.default_stream(st.device))
        with torch.cuda.stream(st):
            yield

    def join(self):
        """Make the default stream wait for the virtual ranks' streams."""
        cur = torch.cuda.current_stream()
        for st in self.streams:
            if st is not None:
                cur.wait_stream(st)

    # ---------------------------------------------------------------- counts
    def exchange_counts_dev(self, send_dev):
        """Every rank stores its G send counts into row `rank` of every rank's count matrix; one host
        read of the own matrix gives M[s][g] = rows s sends to g (none in sync_free mode)."""
        G, nb = self.G, self.NB
        for i, (rg, c) in enumerate(zip(self.regions, send_dev)):
            assert c.numel() == nb * G
            with self.rank_stream(i):
                rg.barrier()
                rg.put_rows(c.to(torch.int32).contiguous(), nb * G * 4, [0] * G, [1] * G, [rg.rank] * G,
                            self.lay["counts"])
                rg.barrier()
        if self.sync_free:
            self.M = None
            return None, None
        Ms = []
        for i, rg in enumerate(self.regions):
            with self.rank_stream(i):
                Ms.append(rg.view(self.lay["counts"], (G, nb * G), torch.int32).cpu().tolist())
        full = Ms[0]
        assert all(m == full for m in Ms)
        self.M = [row[:G] for row in full]  # M[s][g]: send rows s -> g (block 0)
        send = [full[rg.rank] for rg in self.regions]
        recv = [[full[s][j * G + rg.rank] for j in range(nb) for s in range(G)] for rg in self.regions]
        return send, recv

    # ---------------------------------------------------------------- block offsets (from M)
    def _dispatch_rows(self, me):
        """dst_row0[g] = rows the lower sources put into g; my block i -> g is my send rows."""
        G, M = self.G, self.M
        return [sum(M[s][g] for s in range(me)) for g in range(G)]

    def _return_rows(self, me):
        """As a destination, the block received from source s (rows [recv_off[s], +M[s][me])) goes back
        to rows [send_off_s[me], ...) of s's return area (s's send-buffer order)."""
        G, M = self.G, self.M
        src0 = [sum(M[s2][me] for s2 in range(s)) for s in range(G)]
        cnt = [M[s][me] for s in range(G)]
        dst0 = [sum(M[s][g2] for g2 in range(me)) for s in range(G)]
        return src0, cnt, dst0

    # ---------------------------------------------------------------- exchanges
    def dispatch_packed(self, ranks, srcs, tag):
        """Fused pack + dispatch: each rank's kernel gathers src[send_token] straight into the
        destination ranks' `tag` area.  Returns the received rows of each local rank."""
        outs = []
        if self.sync_free:  # destination rows from the count matrix on the device; capacity views
            ns = self.T * self.G
            for i, (rk, rg, src) in enumerate(zip(ranks, self.regions, srcs)):
                with self.rank_stream(i):
                    rg.barrier()
                    rg.pack_dev(rk.desc(), self.G, rk.ctx["plan"], src, self.lay[tag], self.lay["counts"],
                                self.NB * self.G)
                    rg.barrier()
            return [rg.view(self.lay[tag], (ns, self.d), torch.bfloat16) for rg in self.regions]
        for i, (rk, rg, src) in enumerate(zip(ranks, self.regions, srcs)):
            with self.rank_stream(i):
                rg.barrier()
                rg.pack(rk.desc(), self.G, rk.ctx["plan"], src, self.lay[tag], self._dispatch_rows(rg.rank))
                rg.barrier()
        for i, rg in enumerate(self.regions):
            n_in = sum(self.M[s][rg.rank] for s in range(self.G))
            outs.append(rg.view(self.lay[tag], (n_in, self.d), torch.bfloat16))
        return outs

    _RETURN = {"y": "back", "dx": "back", "ds": "ds"}

    def alltoallv(self, sends, send_counts, recv_counts, tag=None):
        """Block exchange of per-destination-contiguous rows: dispatch direction for tag "gate",
        return direction (back to the sources, send-buffer order) for "y", "dx", "ds"."""
        outs = []
        ret = tag in self._RETURN
        area = self._RETURN.get(tag, tag)
        if self.sync_free:
            ns = self.T * self.G
            for i, (rg, snd) in enumerate(zip(self.regions, sends)):
                with self.rank_stream(i):
                    row_bytes = snd[0].numel() * snd.element_size() if snd.dim() > 1 else snd.element_size()
                    rg.barrier()
                    rg.put_rows_dev(snd.contiguous(), row_bytes, 1 if ret else 0, self.lay["counts"],
                                    self.NB * self.G, self.lay[area])
                    rg.barrier()
                    if not ret:  # received gate rows past this step's: zero, so they route nowhere
                        rg.zero_tail(row_bytes, self.lay["counts"], self.NB * self.G, self.lay[area], ns)
            return [rg.view(self.lay[area], (ns,) + tuple(snd.shape[1:]), snd.dtype)
                    for rg, snd in zip(self.regions, sends)]
        for i, (rg, snd) in enumerate(zip(self.regions, sends)):
            with self.rank_stream(i):
                row_bytes = snd[0].numel() * snd.element_size() if snd.dim() > 1 else snd.element_size()
                if ret:
                    src0, cnt, dst0 = self._return_rows(rg.rank)
                else:
                    me = rg.rank
                    cnt = list(self.M[me])
                    src0 = [sum(cnt[:g]) for g in range(self.G)]
                    dst0 = self._dispatch_rows(me)
                rg.barrier()
                if sum(cnt) and snd.numel():
                    rg.put_rows(snd.contiguous(), row_bytes, src0, cnt, dst0, self.lay[area])
                rg.barrier()
        for i, (rg, snd) in enumerate(zip(self.regions, sends)):
            me = rg.rank
            n = sum(self.M[me]) if ret else sum(self.M[s][me] for s in range(self.G))
            outs.append(rg.view(self.lay[area], (n,) + tuple(snd.shape[1:]), snd.dtype))
        return outs

    def alltoallv_start(self, sends, send_counts, recv_counts, tag=None):
        return self.alltoallv(sends, send_counts, recv_counts, tag=tag)

    def alltoallv_finish(self, pending):
        return pending


# ------------------------------------------------------------------------------- one rank
@dataclass
class EPRank:
    """One rank's share of an expert-parallel MoE layer."""
    T: int
    d: int
    n: int
    E: int
    K: int
    G: int
    rank: int
    W1: torch.Tensor          # [L, d, 2n] bf16, experts [rank*L, (rank+1)*L)
    W2: torch.Tensor          # [L, n, d]  bf16
    mode: int = sonic.SONIC_ROUTE_TC
    ctx: dict = field(default_factory=dict)

    @property
    def L(self):
        return self.E // self.G

    def desc(self):
        return sonic.make_desc(self.T, self.d, self.n, self.E, self.K, mode=self.mode)

    # -------------------------------------------------------------- forward
    def plan_fwd(self, S):
        """Route the own tokens over all E experts and build the dispatch plan -> (gates of the send
        rows [T*G, L], device send counts [G])."""
        desc = self.desc()
        rt = sonic.sonic_route(desc, S)
        plan = sonic.sonic_ep_build_plan(desc, self.G, rt)
        nmax = self.T * self.G
        self.ctx.update(rt=rt, plan=plan)
        gates = plan.send_gate[: nmax * self.L].view(nmax, self.L)
        # routed (token, expert) pairs per destination rank: sizes the receiver's GIVEN routing
        pairs = rt.f_rounded[: self.E].view(self.G, self.L).sum(1, dtype=torch.int32)
        # device counts [send rows per rank | routed pairs per rank]: read once, with the exchange
        return gates, torch.cat([plan.send_counts[: self.G], pairs])

    def pack(self, src):
        """Send rows (X forward, dO backward) into a staging buffer (the NCCL / SimComm path)."""
        send = torch.empty(self.T * self.G, self.d, dtype=torch.bfloat16, device=src.device)
        sonic.sonic_ep_pack(self.desc(), self.G, self.ctx["plan"], src, send)
        return send

    def compute_fwd(self, recv_x, recv_gate, pairs_in=0, cap_pairs=None):
        """pairs_in: routed (token, local expert) pairs in the received rows (0 = unknown: bound by
        R_in * L) -- sizes H and the workspaces instead of R_in * L rows.  cap_pairs (host-sync-free
        mode): recv_x / recv_gate are the capacity views and the routed pairs are bounded by
        cap_pairs with the overflow guard (overflowed())."""
        R_in = recv_x.shape[0]
        self.ctx.update(R_in=R_in, recv_x=recv_x)
        if R_in == 0:
            return recv_x.new_zeros(0, self.d)
        if cap_pairs is not None:
            ld = sonic.make_desc(R_in, self.d, self.n, self.L, self.L, mode=sonic.SONIC_ROUTE_GIVEN,
                                 rows_cap=int(cap_pairs))
            flag = self.ctx.get("overflow")
            if flag is None:
                flag = self.ctx["overflow"] = torch.zeros(1, dtype=torch.int32, device=recv_x.device)
            lrt = sonic.sonic_route_given_capped(ld, recv_gate, flag)
            O_part, H, _ = sonic.sonic_moe_fwd(ld, recv_x, self.W1, self.W2, lrt)
            self.ctx.update(ldesc=ld, lrt=lrt, H=H)
            return O_part
        ld = sonic.make_desc(R_in, self.d, self.n, self.L, self.L, mode=sonic.SONIC_ROUTE_GIVEN,
                             rows_cap=max(0, int(pairs_in)))
        lrt = sonic.sonic_route(ld, recv_gate.contiguous())
        O_part, H, _ = sonic.sonic_moe_fwd(ld, recv_x, self.W1, self.W2, lrt)
        self.ctx.update(ldesc=ld, lrt=lrt, H=H)
        return O_part

    def overflowed(self):
        """Host-sync-free mode: True when this rank's last step received more routed pairs than its
        capacity (that step computed nothing here and must be re-run with exact sizing).  Reads the
        device flag: call it after the step, not inside it."""
        flag = self.ctx.get("overflow")
        return bool(flag is not None and int(flag.item()) != 0)

    def combine_fwd(self, back):
        out = torch.empty(self.T, self.d, dtype=torch.bfloat16, device=back.device)
        buf = back if back.shape[0] else back.new_zeros(1, self.d)
        sonic.sonic_ep_combine(self.desc(), self.G, self.ctx["plan"], buf, out)
        return out

    # -------------------------------------------------------------- chunked dispatch (NEXT-2)
    # The received rows come in blocks by source rank; the block this rank sends itself is in its own
    # send buffer before the exchange starts.  Chunked mode computes that block first, while the
    # exchange of the remote blocks is in flight, then the remote rows before and after it: each
    # chunk is a contiguous row range with its own GIVEN routing, H cache and workspace, writing its
    # outputs straight into its rows of the return buffers.  The per-row arithmetic is the unchunked
    # one (O, dX~, dS rows bit-identical); dW1 / dW2 sum the chunks (fp32, SONIC_F_DW_ACCUMULATE).
    def chunk_begin(self, R_in):
        self.ctx.update(R_in=R_in, chunks=[])

    def compute_fwd_chunk(self, x, gate, out, pairs):
        """Forward of one chunk (rows x [Rc, d], gates [Rc, L]) into out [Rc, d]."""
        Rc = x.shape[0]
        if Rc == 0:
            return
        ld = sonic.make_desc(Rc, self.d, self.n, self.L, self.L, mode=sonic.SONIC_ROUTE_GIVEN,
                             rows_cap=max(0, int(pairs)))
        lrt = sonic.sonic_route(ld, gate.contiguous())
        _, H, _ = sonic.sonic_moe_fwd(ld, x, self.W1, self.W2, lrt, O=out)
        self.ctx["chunks"].append(dict(ldesc=ld, lrt=lrt, H=H, x=x, rows=Rc))

    def compute_bwd_chunk(self, k, do, dx_out, ds_out, split):
        """Backward of chunk k on its dO rows: dX~ partial sums into dx_out, dense dS into ds_out; the
        weight gradients now (split=False) or in compute_bwd_dw_chunk (split=True).  The first chunk
        with dW overwrites self.dW1 / dW2, later ones accumulate into them."""
        c = self.ctx["chunks"][k]
        ld = c["ldesc"]
        first = not self.ctx.get("dw_started")
        fl = (sonic.SONIC_F_BWD_NO_DW if split else (0 if first else sonic.SONIC_F_DW_ACCUMULATE))
        ldf = sonic.make_desc(ld.T, ld.d, ld.n, ld.E, ld.K, mode=ld.route_mode, flags=ld.flags | fl,
                              rows_cap=ld.rows_cap)
        if split:
            _, _, _, dS, ws = sonic.sonic_moe_bwd(ldf, do, c["x"], c["H"], self.W1, self.W2, c["lrt"], dX=dx_out)
            c.update(bws=ws, do=do)
        else:
            if first:
                self.dW1 = torch.empty(self.L, self.d, 2 * self.n, device=do.device)
                self.dW2 = torch.empty(self.L, self.n, self.d, device=do.device)
                self.ctx["dw_started"] = True
            _, _, _, dS, _ = sonic.sonic_moe_bwd(ldf, do, c["x"], c["H"], self.W1, self.W2, c["lrt"], dX=dx_out,
                                                 dW1=self.dW1, dW2=self.dW2)
        sonic.sonic_ep_ds_dense(ld, c["lrt"], dS, ds_out)

    def compute_bwd_dw_chunk(self, k):
        """Weight gradients of a split chunk from its part-1 dH / A' (same workspace)."""
        c = self.ctx["chunks"][k]
        ld = c["ldesc"]
        first = not self.ctx.get("dw_started")
        fl = sonic.SONIC_F_BWD_DW_ONLY | (0 if first else sonic.SONIC_F_DW_ACCUMULATE)
        ldf = sonic.make_desc(ld.T, ld.d, ld.n, ld.E, ld.K, mode=ld.route_mode, flags=ld.flags | fl,
                              rows_cap=ld.rows_cap)
        if first:
            self.dW1 = torch.empty(self.L, self.d, 2 * self.n, device=self.W1.device)
            self.dW2 = torch.empty(self.L, self.n, self.d, device=self.W1.device)
            self.ctx["dw_started"] = True
        sonic.sonic_moe_bwd(ldf, c["do"], c["x"], c["H"], self.W1, self.W2, c["lrt"], dW1=self.dW1, dW2=self.dW2,
                            ws=c["bws"])

    # -------------------------------------------------------------- backward
    def _ldesc(self, extra_flags):
        ld = self.ctx["ldesc"]
        return sonic.make_desc(ld.T, ld.d, ld.n, ld.E, ld.K, mode=ld.route_mode, flags=ld.flags | extra_flags,
                               rows_cap=ld.rows_cap)

    def compute_bwd(self, recv_do):
        """Backward part 1 on the received rows: dH, dS, dX~ partial sums (the dW come later, in
        compute_bwd_dw, so that they overlap the exchange of these results)."""
        R_in = self.ctx["R_in"]
        dev = recv_do.device
        if R_in == 0:
            self.ctx.update(bws=None, dw_done=False)
            return recv_do.new_zeros(0, self.d), torch.zeros(0, self.L, device=dev)
        lrt = self.ctx["lrt"]
        if self.G == 1:  # nothing to overlap: one call (the dX aggregation then overlaps dW2 inside)
            ld = self._ldesc(0)
            dX_part, self.dW1, self.dW2, dS, _ = sonic.sonic_moe_bwd(ld, recv_do, self.ctx["recv_x"], self.ctx["H"],
                                                                     self.W1, self.W2, lrt)
            self.ctx.update(bws=None, dw_done=True)
        else:
            ld = self._ldesc(sonic.SONIC_F_BWD_NO_DW)
            dX_part, _, _, dS, ws = sonic.sonic_moe_bwd(ld, recv_do, self.ctx["recv_x"], self.ctx["H"], self.W1,
                                                        self.W2, lrt)
            self.ctx.update(bws=ws, recv_do=recv_do, dw_done=False)
        dense = torch.empty(R_in, self.L, dtype=torch.float32, device=dev)
        sonic.sonic_ep_ds_dense(ld, lrt, dS, dense)
        return dX_part, dense

    def compute_bwd_dw(self):
        """Backward part 2: dW2, dW1 of the local experts from part 1's dH / A' (same workspace)."""
        dev = self.W1.device
        if self.ctx.get("dw_done"):
            return
        if self.ctx.get("bws") is None:
            self.dW1 = torch.zeros(self.L, self.d, 2 * self.n, device=dev)
            self.dW2 = torch.zeros(self.L, self.n, self.d, device=dev)
            return
        ld = self._ldesc(sonic.SONIC_F_BWD_DW_ONLY)
        _, dW1, dW2, _, _ = sonic.sonic_moe_bwd(ld, self.ctx["recv_do"], self.ctx["recv_x"], self.ctx["H"], self.W1,
                                                self.W2, self.ctx["lrt"], ws=self.ctx["bws"])
        self.dW1, self.dW2 = dW1, dW2

    def combine_bwd(self, back_dx, back_ds):
        desc, plan, rt = self.desc(), self.ctx["plan"], self.ctx["rt"]
        dX = torch.empty(self.T, self.d, dtype=torch.bfloat16, device=back_dx.device)
        sonic.sonic_ep_combine(desc, self.G, plan, back_dx if back_dx.shape[0] else back_dx.new_zeros(1, self.d), dX)
        dS = torch.zeros(sonic.sonic_rows_max(desc), dtype=torch.float32, device=back_dx.device)
        if back_ds.shape[0]:
            sonic.sonic_ep_ds_scatter(desc, self.G, rt, plan, back_ds.contiguous(), dS)
        return dX, dS


# ------------------------------------------------------------------------------- the layer step
def _dispatch(ranks, comm, srcs, send_counts, recv_counts, tag):
    """Rows src[send_token] of every local rank to their destination ranks."""
    if hasattr(comm, "dispatch_packed"):  # peer memory: the gather stores into the destinations
        return comm.dispatch_packed(ranks, srcs, tag)
    sends = []
    for i, (r, src) in enumerate(zip(ranks, srcs)):
        with comm.rank_stream(i):
            sends.append(r.pack(src))
    return comm.alltoallv(sends, send_counts, recv_counts, tag=tag)


def _chunk_rows(r, sc, rc):
    """(send offset, rows, recv offset) of rank r's self block."""
    return sum(sc[: r.rank]), sc[r.rank], sum(rc[: r.rank])


def _ep_forward_chunked(ranks, comm, Xs, disp, send_counts, recv_counts, recv_pairs):
    """NEXT-2 chunked dispatch (staged exchange): the self block's up/down-projection runs while the
    exchange of the remote blocks is in flight, then the remote rows before / after it."""
    n = len(ranks)
    sends = []
    for i, (r, X) in enumerate(zip(ranks, Xs)):
        with comm.rank_stream(i):
            sends.append(r.pack(X))
    gates = [g for g, _ in disp]
    p_x = comm.alltoallv_start(sends, send_counts, recv_counts, tag="x")
    p_g = comm.alltoallv_start(gates, send_counts, recv_counts, tag="gate")
    parts, geo = [], []
    for i, r in enumerate(ranks):
        so, ns, ro = _chunk_rows(r, send_counts[i], recv_counts[i])
        R_in = sum(recv_counts[i])
        geo.append((so, ns, ro, R_in))
        with comm.rank_stream(i):
            part = torch.empty(R_in, r.d, dtype=torch.bfloat16, device=sends[i].device)
            r.chunk_begin(R_in)
            r.compute_fwd_chunk(sends[i][so:so + ns], gates[i][so:so + ns], part[ro:ro + ns],
                                recv_pairs[i][r.rank])
            parts.append(part)
    recv_x = comm.alltoallv_finish(p_x)
    recv_g = comm.alltoallv_finish(p_g)
    for i, r in enumerate(ranks):
        so, ns, ro, R_in = geo[i]
        pr = recv_pairs[i]
        with comm.rank_stream(i):
            r.compute_fwd_chunk(recv_x[i][:ro], recv_g[i][:ro], parts[i][:ro], sum(pr[: r.rank]))
            r.compute_fwd_chunk(recv_x[i][ro + ns:], recv_g[i][ro + ns:], parts[i][ro + ns:], sum(pr[r.rank + 1:]))
    back = comm.alltoallv(parts, recv_counts, send_counts, tag="y")
    outs = []
    for i, (r, rc, b) in enumerate(zip(ranks, recv_counts, back)):
        r.ctx["recv_counts"] = rc
        with comm.rank_stream(i):
            outs.append(r.combine_fwd(b))
    return outs


def ep_forward(ranks, comm, Xs, Ss, chunked=False):
    """Forward of the EP layer over the local ranks -> [O_r].  chunked (staged exchange, NCCL or
    SimComm): the self block is computed while the remote blocks are exchanged (NEXT-2)."""
    disp = []
    for i, (r, S) in enumerate(zip(ranks, Ss)):
        with comm.rank_stream(i):
            disp.append(r.plan_fwd(S))
    # the send counts are host arguments of the exchange: the only host synchronisation of the step
    # (none with PeerComm(sync_free=True): the offsets are read on the device)
    send_both, recv_both = comm.exchange_counts_dev([c for _, c in disp])
    G = ranks[0].G
    sync_free = getattr(comm, "sync_free", False)
    if sync_free:
        send_counts = recv_counts = [None] * len(ranks)
        cap = comm.cap_pairs if comm.cap_pairs is not None else 2 * ranks[0].T * ranks[0].K
        pairs_in = [None] * len(ranks)
    else:
        send_counts = [sb[:G] for sb in send_both]
        recv_counts = [rb[:G] for rb in recv_both]
        pairs_in = [sum(rb[G:2 * G]) for rb in recv_both]
    for r, sc in zip(ranks, send_counts):
        r.ctx["counts"] = sc
        r.ctx["chunked"] = False
    if chunked and not sync_free and not hasattr(comm, "dispatch_packed"):
        for r in ranks:
            r.ctx["chunked"] = True
        return _ep_forward_chunked(ranks, comm, Xs, disp, send_counts, recv_counts,
                                   [rb[G:2 * G] for rb in recv_both])
    recv_x = _dispatch(ranks, comm, Xs, send_counts, recv_counts, "x")
    recv_g = comm.alltoallv([g for g, _ in disp], send_counts, recv_counts, tag="gate")
    parts = []
    for i, (r, x, g, pin) in enumerate(zip(ranks, recv_x, recv_g, pairs_in)):
        with comm.rank_stream(i):
            parts.append(r.compute_fwd(x, g, cap_pairs=cap) if sync_free else r.compute_fwd(x, g, pin))
    back = comm.alltoallv(parts, recv_counts, send_counts, tag="y")
    outs = []
    for i, (r, rc, b) in enumerate(zip(ranks, recv_counts, back)):
        r.ctx["recv_counts"] = rc
        with comm.rank_stream(i):
            outs.append(r.combine_fwd(b))
    if hasattr(comm, "join"):
        comm.join()
    return outs


def _ep_backward_chunked(ranks, comm, dOs, send_counts, recv_counts):
    """Backward of a chunked forward: the self block's dH / dX~ / dS / dW while the remote dO rows
    are exchanged, then the remote chunks' dX~ / dS, whose return exchange overlaps their dW."""
    sends = []
    for i, (r, dO) in enumerate(zip(ranks, dOs)):
        with comm.rank_stream(i):
            sends.append(r.pack(dO))
    p_do = comm.alltoallv_start(sends, send_counts, recv_counts, tag="do")
    dxs, dss, geo = [], [], []
    for i, r in enumerate(ranks):
        so, ns, ro = _chunk_rows(r, send_counts[i], recv_counts[i])
        R_in = sum(recv_counts[i])
        geo.append((so, ns, ro))
        r.ctx["dw_started"] = False
        with comm.rank_stream(i):
            dx = torch.empty(R_in, r.d, dtype=torch.bfloat16, device=sends[i].device)
            ds = torch.empty(R_in, r.L, dtype=torch.float32, device=sends[i].device)
            k = 0
            if ns:
                r.compute_bwd_chunk(0, sends[i][so:so + ns], dx[ro:ro + ns], ds[ro:ro + ns], split=False)
                k = 1
            r.ctx["k_remote"] = k
            dxs.append(dx)
            dss.append(ds)
    recv = comm.alltoallv_finish(p_do)
    for i, r in enumerate(ranks):
        so, ns, ro = geo[i]
        with comm.rank_stream(i):
            k = r.ctx["k_remote"]
            for lo, hi in ((0, ro), (ro + ns, recv[i].shape[0])):
                if hi > lo:
                    r.compute_bwd_chunk(k, recv[i][lo:hi], dxs[i][lo:hi], dss[i][lo:hi], split=True)
                    k += 1
    p_dx = comm.alltoallv_start(dxs, recv_counts, send_counts, tag="dx")
    p_ds = comm.alltoallv_start(dss, recv_counts, send_counts, tag="ds")
    for i, r in enumerate(ranks):
        with comm.rank_stream(i):
            for k in range(r.ctx["k_remote"], len(r.ctx["chunks"])):
                r.compute_bwd_dw_chunk(k)
            if not r.ctx["dw_started"]:  # no rows at all: the local experts' gradients are zero
                r.dW1 = torch.zeros(r.L, r.d, 2 * r.n, device=r.W1.device)
                r.dW2 = torch.zeros(r.L, r.n, r.d, device=r.W1.device)
    back_dx = comm.alltoallv_finish(p_dx)
    back_ds = comm.alltoallv_finish(p_ds)
    res = []
    for i, (r, bx, bs) in enumerate(zip(ranks, back_dx, back_ds)):
        with comm.rank_stream(i):
            res.append(r.combine_bwd(bx, bs))
    return res


def ep_backward(ranks, comm, dOs):
    """Backward over the local ranks -> [(dX_r, dS_r)]; each rank keeps its local dW1 / dW2."""
    send_counts = [r.ctx["counts"] for r in ranks]
    recv_counts = [r.ctx["recv_counts"] for r in ranks]
    if ranks[0].ctx.get("chunked"):
        return _ep_backward_chunked(ranks, comm, dOs, send_counts, recv_counts)
    recv = _dispatch(ranks, comm, dOs, send_counts, recv_counts, "do")
    outs = []
    for i, (r, x) in enumerate(zip(ranks, recv)):
        with comm.rank_stream(i):
            outs.append(r.compute_bwd(x))
    # the dX~ / dS exchange runs while the local weight gradients are computed (NCCL path)
    p_dx = comm.alltoallv_start([o[0] for o in outs], recv_counts, send_counts, tag="dx")
    p_ds = comm.alltoallv_start([o[1] for o in outs], recv_counts, send_counts, tag="ds")
    for i, r in enumerate(ranks):
        with comm.rank_stream(i):
            r.compute_bwd_dw()
    back_dx = comm.alltoallv_finish(p_dx)
    back_ds = comm.alltoallv_finish(p_ds)
    res = []
    for i, (r, bx, bs) in enumerate(zip(ranks, back_dx, back_ds)):
        with comm.rank_stream(i):
            res.append(r.combine_bwd(bx, bs))
    if hasattr(comm, "join"):
        comm.join()
    return res
