"""Thin ctypes binding of libsonic (include/sonic.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
libsonic.so.  PyTorch provides device memory and the current stream.  There is no
CPU fallback: if the library is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SONIC_LIB: experiment builds only (tools/ab.sh); the product path is the in-tree libsonic.so
LIB_PATH = os.environ.get("SONIC_LIB") or os.path.join(_HERE, "libsonic.so")

SONIC_ROUTE_TC = 0
SONIC_ROUTE_TR_NRF = 1
SONIC_ROUTE_TR_UP = 3
SONIC_ROUTE_TR_DOWN = 4
SONIC_ROUTE_TR_BALANCE = 5
SONIC_ROUTE_TR_SR = 6
SONIC_ROUTE_EC = 7
SONIC_ROUTE_TR_NRS = 8
# oracle route(mode, rounding) of each TR-family mode
ROUTE_MODE_NAMES = {0: ("tc", "nrf"), 1: ("tr", "nrf"), 3: ("tr", "up"), 4: ("tr", "down"), 5: ("tr", "balance"),
                    6: ("tr", "sr"), 7: ("ec", "nrf"), 8: ("tr", "nrs")}
SONIC_F_GATE_RAW = 1
SONIC_F_NO_ORPHAN_RESCUE = 2
SONIC_F_DW_ACCUMULATE = 4
SONIC_F_BWD_NO_DW = 8
SONIC_F_BWD_DW_ONLY = 16
SONIC_F_DW_BF16 = 32
SONIC_F_NO_FUSED_UPDOWN = 64
SONIC_F_FUSED_UPDOWN = 128
SONIC_F_FP8_UP = 256
SONIC_F_FP8_W1_CACHED = 512
SONIC_F_FP8_DXT = 1024
GEMM_M = 128

ROUTING_FIELDS = ["topk_ids", "topk_s", "f", "f_rounded", "offsets", "pad_offsets", "row_token", "row_gate",
                  "token_rowptr", "token_rows", "tile_expert", "num_tiles", "tile_pairs", "num_pairs"]
_FLOAT_FIELDS = {"topk_s", "row_gate"}


class sonic_moe_desc(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int64), ("d", ctypes.c_int32), ("n", ctypes.c_int32), ("E", ctypes.c_int32),
                ("K", ctypes.c_int32), ("m_tile", ctypes.c_int32), ("route_mode", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("seed", ctypes.c_uint32), ("rows_cap", ctypes.c_int64)]


class sonic_routing(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ROUTING_FIELDS]


EP_PLAN_FIELDS = ["dmask", "bm", "wprefix", "send_counts", "send_offsets", "tokcnt", "ep_rowptr", "ep_rows",
                  "send_token", "send_gate"]


class sonic_ep_plan(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in EP_PLAN_FIELDS]


class SonicError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libsonic.so (built in-tree by __graft_entry__.build()).  Fails loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SonicError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        vp, sz = ctypes.c_void_p, ctypes.c_size_t
        L.sonic_rows_max.argtypes = [P(sonic_moe_desc)]
        L.sonic_rows_max.restype = ctypes.c_int64
        L.sonic_routing_sizes.argtypes = [P(sonic_moe_desc), P(sz)]
        L.sonic_routing_sizes.restype = ctypes.c_int
        for f in ("sonic_route_workspace_size", "sonic_fwd_workspace_size", "sonic_bwd_workspace_size"):
            getattr(L, f).argtypes = [P(sonic_moe_desc)]
            getattr(L, f).restype = sz
        L.sonic_workspace_offsets.argtypes = [P(sonic_moe_desc), ctypes.c_int, P(sz)]
        L.sonic_workspace_offsets.restype = ctypes.c_int
        L.sonic_route.argtypes = [P(sonic_moe_desc), vp, P(sonic_routing), vp, sz, vp]
        L.sonic_route.restype = ctypes.c_int
        L.sonic_route_logits.argtypes = [P(sonic_moe_desc), vp, vp, P(sonic_routing), vp, sz, vp]
        L.sonic_route_logits.restype = ctypes.c_int
        L.sonic_quantize_e4m3_rows.argtypes = [vp, ctypes.c_int64, ctypes.c_int32, vp, vp, vp]
        L.sonic_quantize_e4m3_rows.restype = ctypes.c_int
        L.sonic_quantize_e4m3_cols.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp, vp, vp]
        L.sonic_quantize_e4m3_cols.restype = ctypes.c_int
        L.sonic_router_fwd.argtypes = [P(sonic_moe_desc), vp, vp, vp, vp]
        L.sonic_router_fwd.restype = ctypes.c_int
        L.sonic_router_grad_workspace_size.argtypes = [P(sonic_moe_desc)]
        L.sonic_router_grad_workspace_size.restype = sz
        L.sonic_router_grad.argtypes = [P(sonic_moe_desc), vp, vp, vp, vp, vp, vp, sz, vp]
        L.sonic_router_grad.restype = ctypes.c_int
        L.sonic_moe_fwd.argtypes = [P(sonic_moe_desc), vp, vp, vp, P(sonic_routing), vp, vp, vp, sz, vp]
        L.sonic_moe_fwd.restype = ctypes.c_int
        L.sonic_moe_bwd.argtypes = [P(sonic_moe_desc), vp, vp, vp, vp, vp, P(sonic_routing), vp, vp, vp, vp, vp,
                                    sz, vp]
        L.sonic_moe_bwd.restype = ctypes.c_int
        L.sonic_router_bwd.argtypes = [P(sonic_moe_desc), vp, P(sonic_routing), vp, vp, vp]
        L.sonic_router_bwd.restype = ctypes.c_int
        L.sonic_status_string.argtypes = [ctypes.c_int]
        L.sonic_status_string.restype = ctypes.c_char_p
        L.sonic_last_launch_count.argtypes = []
        L.sonic_last_launch_count.restype = ctypes.c_int
        L.sonic_ep_plan_sizes.argtypes = [P(sonic_moe_desc), ctypes.c_int, P(sz)]
        L.sonic_ep_plan_sizes.restype = ctypes.c_int
        L.sonic_ep_build_plan.argtypes = [P(sonic_moe_desc), ctypes.c_int, P(sonic_routing), P(sonic_ep_plan), vp]
        L.sonic_ep_build_plan.restype = ctypes.c_int
        for f in ("sonic_ep_pack", "sonic_ep_combine"):
            getattr(L, f).argtypes = [P(sonic_moe_desc), ctypes.c_int, P(sonic_ep_plan), vp, vp, vp]
            getattr(L, f).restype = ctypes.c_int
        L.sonic_ep_ds_dense.argtypes = [P(sonic_moe_desc), P(sonic_routing), vp, vp, vp]
        L.sonic_ep_ds_dense.restype = ctypes.c_int
        L.sonic_ep_ds_scatter.argtypes = [P(sonic_moe_desc), ctypes.c_int, P(sonic_routing), P(sonic_ep_plan), vp,
                                          vp, vp]
        L.sonic_ep_ds_scatter.restype = ctypes.c_int
        L.sonic_peer_create.argtypes = [ctypes.c_int, ctypes.c_int, sz, P(vp), vp]
        L.sonic_peer_create.restype = ctypes.c_int
        L.sonic_peer_open.argtypes = [vp, vp]
        L.sonic_peer_open.restype = ctypes.c_int
        L.sonic_peer_base.argtypes = [vp, ctypes.c_int]
        L.sonic_peer_base.restype = vp
        L.sonic_peer_destroy.argtypes = [vp]
        L.sonic_peer_destroy.restype = ctypes.c_int
        L.sonic_peer_barrier.argtypes = [vp, vp]
        L.sonic_peer_barrier.restype = ctypes.c_int
        L.sonic_ep_pack_peer.argtypes = [P(sonic_moe_desc), ctypes.c_int, P(sonic_ep_plan), vp, vp, sz,
                                         P(ctypes.c_int32), vp]
        L.sonic_ep_pack_peer.restype = ctypes.c_int
        L.sonic_ep_pack_peer_dev.argtypes = [P(sonic_moe_desc), ctypes.c_int, P(sonic_ep_plan), vp, vp, sz, sz,
                                             ctypes.c_int, vp]
        L.sonic_ep_pack_peer_dev.restype = ctypes.c_int
        L.sonic_peer_put_rows_dev.argtypes = [vp, ctypes.c_int, vp, sz, ctypes.c_int, sz, ctypes.c_int, sz, vp]
        L.sonic_peer_put_rows_dev.restype = ctypes.c_int
        L.sonic_peer_zero_tail.argtypes = [vp, ctypes.c_int, sz, sz, ctypes.c_int, sz, ctypes.c_longlong, vp]
        L.sonic_peer_zero_tail.restype = ctypes.c_int
        L.sonic_route_given_capped.argtypes = [P(sonic_moe_desc), vp, P(sonic_routing), vp, sz, vp, vp]
        L.sonic_route_given_capped.restype = ctypes.c_int
        L.sonic_peer_put_rows.argtypes = [vp, ctypes.c_int, vp, sz, P(ctypes.c_int32), P(ctypes.c_int32),
                                          P(ctypes.c_int32), sz, vp]
        L.sonic_peer_put_rows.restype = ctypes.c_int
        L.sonic_profile_enable.argtypes = [ctypes.c_int]
        L.sonic_profile_enable.restype = None
        L.sonic_profile_collect.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                                            ctypes.c_int]
        L.sonic_profile_collect.restype = ctypes.c_int
        _lib = L
    return _lib


# cumulative count of libsonic kernel launches made through this binding (bench.py's gpu_launches)
LAUNCHES = [0]


def _check(status, what):
    if status != 0:
        raise SonicError(f"{what}: {lib().sonic_status_string(status).decode()} ({status})")


def _done(status, what):
    """_check a compute call and add the kernels it launched to LAUNCHES."""
    _check(status, what)
    LAUNCHES[0] += int(lib().sonic_last_launch_count())


def make_desc(T, d, n, E, K, mode=SONIC_ROUTE_TC, m_tile=128, flags=0, seed=0, rows_cap=0):
    return sonic_moe_desc(T, d, n, E, K, m_tile, mode, flags, seed, rows_cap)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def sonic_rows_max(desc):
    return int(lib().sonic_rows_max(ctypes.byref(desc)))


def sonic_routing_sizes(desc):
    arr = (ctypes.c_size_t * len(ROUTING_FIELDS))()
    _check(lib().sonic_routing_sizes(ctypes.byref(desc), arr), "sonic_routing_sizes")
    return dict(zip(ROUTING_FIELDS, list(arr)))


def sonic_route_workspace_size(desc):
    return int(lib().sonic_route_workspace_size(ctypes.byref(desc)))


def sonic_fwd_workspace_size(desc):
    return int(lib().sonic_fwd_workspace_size(ctypes.byref(desc)))


def sonic_bwd_workspace_size(desc):
    return int(lib().sonic_bwd_workspace_size(ctypes.byref(desc)))


def sonic_workspace_offsets(desc, which):
    arr = (ctypes.c_size_t * 4)()
    _check(lib().sonic_workspace_offsets(ctypes.byref(desc), which, arr), "sonic_workspace_offsets")
    return list(arr)


def sonic_last_launch_count():
    return int(lib().sonic_last_launch_count())


def sonic_profile_enable(on=True):
    lib().sonic_profile_enable(1 if on else 0)


def sonic_profile_collect(max_records=1 << 16, name_len=32):
    """[(name, ms), ...] of the kernels launched since profiling was enabled / last collected."""
    names = ctypes.create_string_buffer(max_records * name_len)
    ms = (ctypes.c_float * max_records)()
    n = lib().sonic_profile_collect(names, name_len, ms, max_records)
    raw = names.raw
    return [(raw[i * name_len:(i + 1) * name_len].split(b"\0", 1)[0].decode(), float(ms[i])) for i in range(n)]


@dataclass
class Routing:
    """Device buffers of a sonic_routing (torch tensors, owned here) + the C struct."""
    tensors: dict
    c: sonic_routing

    def __getattr__(self, name):
        t = self.__dict__.get("tensors")
        if t is not None and name in t:
            return t[name]
        raise AttributeError(name)


def alloc_routing(desc, device="cuda"):
    sizes = sonic_routing_sizes(desc)
    tensors = {}
    for f in ROUTING_FIELDS:
        dt = torch.float32 if f in _FLOAT_FIELDS else torch.int32
        tensors[f] = torch.empty(max(1, sizes[f] // 4), dtype=dt, device=device)
    c = sonic_routing(*[t.data_ptr() for t in tensors.values()])
    return Routing(tensors, c)


def _ws(nbytes, device):
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)


def sonic_route(desc, S, rt=None, ws=None):
    """sonic_route: S [T,E] fp32 -> Routing (device metadata)."""
    if rt is None:
        rt = alloc_routing(desc, S.device)
    if ws is None:
        ws = _ws(sonic_route_workspace_size(desc), S.device)
    _done(lib().sonic_route(ctypes.byref(desc), _ptr(S), ctypes.byref(rt.c), _ptr(ws), ws.numel(), _stream()),
           "sonic_route")
    return rt


def sonic_route_given_capped(desc, S, overflow, rt=None, ws=None):
    """SONIC_ROUTE_GIVEN with the capacity guard: overflow (device int32 [1]) = 1 and an empty routing
    when the routed pairs exceed desc.rows_cap."""
    if rt is None:
        rt = alloc_routing(desc, S.device)
    if ws is None:
        ws = _ws(sonic_route_workspace_size(desc), S.device)
    _done(lib().sonic_route_given_capped(ctypes.byref(desc), _ptr(S), ctypes.byref(rt.c), _ptr(ws), ws.numel(),
                                         _ptr(overflow), _stream()), "sonic_route_given_capped")
    return rt


def sonic_route_logits(desc, logits, S=None, rt=None, ws=None):
    """sonic_route_logits: router logits [T,E] fp32 -> (S = softmax(logits) [T,E] fp32, Routing); the
    softmax is fused into the routing."""
    if S is None:
        S = torch.empty_like(logits)
    if rt is None:
        rt = alloc_routing(desc, logits.device)
    if ws is None:
        ws = _ws(sonic_route_workspace_size(desc), logits.device)
    _done(lib().sonic_route_logits(ctypes.byref(desc), _ptr(logits), _ptr(S), ctypes.byref(rt.c), _ptr(ws), ws.numel(),
                                   _stream()), "sonic_route_logits")
    return S, rt


def sonic_moe_fwd(desc, X, W1, W2, rt, O=None, H=None, ws=None):
    """sonic_moe_fwd -> (O [T,d] bf16, H_cache [rows_max,2n] bf16, ws)."""
    rows = sonic_rows_max(desc)
    if O is None:
        O = torch.empty(desc.T, desc.d, dtype=torch.bfloat16, device=X.device)
    if H is None:
        H = torch.empty(rows, 2 * desc.n, dtype=torch.bfloat16, device=X.device)
    if ws is None:
        ws = _ws(sonic_fwd_workspace_size(desc), X.device)
    _done(lib().sonic_moe_fwd(ctypes.byref(desc), _ptr(X), _ptr(W1), _ptr(W2), ctypes.byref(rt.c), _ptr(O),
                               _ptr(H), _ptr(ws), ws.numel(), _stream()), "sonic_moe_fwd")
    return O, H, ws


def sonic_moe_bwd(desc, dO, X, H, W1, W2, rt, dX=None, dW1=None, dW2=None, dS=None, ws=None):
    """sonic_moe_bwd -> (dX [T,d] bf16, dW1 [E,d,2n], dW2 [E,n,d] (f32, or bf16 with SONIC_F_DW_BF16),
    dS [rows_max] f32, ws)."""
    rows = sonic_rows_max(desc)
    dev = X.device
    want_dx = not (desc.flags & SONIC_F_BWD_DW_ONLY)
    want_dw = not (desc.flags & SONIC_F_BWD_NO_DW)
    if dX is None and want_dx:
        dX = torch.empty(desc.T, desc.d, dtype=torch.bfloat16, device=dev)
    wdt = torch.bfloat16 if desc.flags & SONIC_F_DW_BF16 else torch.float32
    if dW1 is None and want_dw:
        dW1 = torch.empty(desc.E, desc.d, 2 * desc.n, dtype=wdt, device=dev)
    if dW2 is None and want_dw:
        dW2 = torch.empty(desc.E, desc.n, desc.d, dtype=wdt, device=dev)
    if dS is None and want_dx:
        dS = torch.empty(rows, dtype=torch.float32, device=dev)
    if ws is None:
        ws = _ws(sonic_bwd_workspace_size(desc), dev)
    _done(lib().sonic_moe_bwd(ctypes.byref(desc), _ptr(dO), _ptr(X), _ptr(H), _ptr(W1), _ptr(W2),
                               ctypes.byref(rt.c), _ptr(dX), _ptr(dW1), _ptr(dW2), _ptr(dS), _ptr(ws), ws.numel(),
                               _stream()), "sonic_moe_bwd")
    return dX, dW1, dW2, dS, ws


def sonic_router_bwd(desc, S, rt, dS, dlogits=None):
    """sonic_router_bwd: dS [rows_max] fp32 -> d logits [T,E] fp32 (NEXT-4)."""
    if dlogits is None:
        dlogits = torch.empty(desc.T, desc.E, dtype=torch.float32, device=S.device)
    _done(lib().sonic_router_bwd(ctypes.byref(desc), _ptr(S), ctypes.byref(rt.c), _ptr(dS), _ptr(dlogits),
                                 _stream()), "sonic_router_bwd")
    return dlogits


def sonic_quantize_e4m3_rows(X):
    """X [rows, cols] bf16 -> (q [rows, cols] uint8 e4m3 codes, scale [rows] fp32)."""
    q = torch.empty(X.shape, dtype=torch.uint8, device=X.device)
    s = torch.empty(X.shape[0], dtype=torch.float32, device=X.device)
    _done(lib().sonic_quantize_e4m3_rows(_ptr(X), X.shape[0], X.shape[1], _ptr(q), _ptr(s), _stream()),
          "sonic_quantize_e4m3_rows")
    return q, s


def sonic_quantize_e4m3_cols(W):
    """W [batch, K, N] bf16 -> (q [batch, K, N] uint8 e4m3 codes, scale [batch, N] fp32)."""
    q = torch.empty(W.shape, dtype=torch.uint8, device=W.device)
    s = torch.empty(W.shape[0], W.shape[2], dtype=torch.float32, device=W.device)
    _done(lib().sonic_quantize_e4m3_cols(_ptr(W), W.shape[0], W.shape[1], W.shape[2], _ptr(q), _ptr(s), _stream()),
          "sonic_quantize_e4m3_cols")
    return q, s


def sonic_router_fwd(desc, X, Wr, logits=None):
    """sonic_router_fwd: logits [T,E] fp32 = X [T,d] bf16 . Wr [d,E] bf16 (NEXT-4)."""
    if logits is None:
        logits = torch.empty(desc.T, desc.E, dtype=torch.float32, device=X.device)
    _done(lib().sonic_router_fwd(ctypes.byref(desc), _ptr(X), _ptr(Wr), _ptr(logits), _stream()), "sonic_router_fwd")
    return logits


def sonic_router_grad(desc, X, Wr, dlogits, dX=None, dWr=None, want_dWr=True, ws=None):
    """sonic_router_grad: dX += dlogits Wr^T (in place, if dX is given), dWr = X^T dlogits -> (dX, dWr)."""
    if dWr is None and want_dWr:
        dWr = torch.empty(desc.d, desc.E, dtype=torch.float32, device=X.device)
    if ws is None:
        ws = _ws(int(lib().sonic_router_grad_workspace_size(ctypes.byref(desc))), X.device)
    _done(lib().sonic_router_grad(ctypes.byref(desc), _ptr(X), _ptr(Wr), _ptr(dlogits), _ptr(dX) if dX is not None
                                  else None, _ptr(dWr) if dWr is not None else None, _ptr(ws), ws.numel(), _stream()),
          "sonic_router_grad")
    return dX, dWr


def ws_view(ws, offset, shape, dtype):
    """A typed view into a workspace buffer (for inspecting transients in tests)."""
    n = 1
    for s in shape:
        n *= s
    nbytes = n * torch.empty(0, dtype=dtype).element_size()
    return ws[offset: offset + nbytes].view(dtype).view(*shape)


# ---------------------------------------------------------------------------- expert parallelism
SONIC_ROUTE_GIVEN = 2


@dataclass
class EPPlan:
    tensors: dict
    c: sonic_ep_plan

    def __getattr__(self, name):
        t = self.__dict__.get("tensors")
        if t is not None and name in t:
            return t[name]
        raise AttributeError(name)


def sonic_ep_plan_sizes(desc, G):
    arr = (ctypes.c_size_t * len(EP_PLAN_FIELDS))()
    _check(lib().sonic_ep_plan_sizes(ctypes.byref(desc), G, arr), "sonic_ep_plan_sizes")
    return dict(zip(EP_PLAN_FIELDS, list(arr)))


def alloc_ep_plan(desc, G, device="cuda"):
    sizes = sonic_ep_plan_sizes(desc, G)
    tensors = {f: torch.empty(max(1, sizes[f] // 4), dtype=torch.float32 if f == "send_gate" else torch.int32,
                              device=device) for f in EP_PLAN_FIELDS}
    return EPPlan(tensors, sonic_ep_plan(*[t.data_ptr() for t in tensors.values()]))


def sonic_ep_build_plan(desc, G, rt, plan=None):
    if plan is None:
        plan = alloc_ep_plan(desc, G, rt.tensors["row_token"].device)
    _done(lib().sonic_ep_build_plan(ctypes.byref(desc), G, ctypes.byref(rt.c), ctypes.byref(plan.c), _stream()),
           "sonic_ep_build_plan")
    return plan


def sonic_ep_pack(desc, G, plan, src, send):
    _done(lib().sonic_ep_pack(ctypes.byref(desc), G, ctypes.byref(plan.c), _ptr(src), _ptr(send), _stream()),
           "sonic_ep_pack")
    return send


def sonic_ep_combine(desc, G, plan, back, out):
    _done(lib().sonic_ep_combine(ctypes.byref(desc), G, ctypes.byref(plan.c), _ptr(back), _ptr(out), _stream()),
           "sonic_ep_combine")
    return out


def sonic_ep_ds_dense(local_desc, local_rt, dS, dense):
    _done(lib().sonic_ep_ds_dense(ctypes.byref(local_desc), ctypes.byref(local_rt.c), _ptr(dS), _ptr(dense),
                                   _stream()), "sonic_ep_ds_dense")
    return dense


def sonic_ep_ds_scatter(desc, G, rt, plan, back, dS):
    _done(lib().sonic_ep_ds_scatter(ctypes.byref(desc), G, ctypes.byref(rt.c), ctypes.byref(plan.c), _ptr(back),
                                     _ptr(dS), _stream()), "sonic_ep_ds_scatter")
    return dS


# ---------------------------------------------------------------- peer-memory exchange (NEXT-2)
SONIC_PEER_HANDLE_BYTES = 256


def _i32(vals):
    return (ctypes.c_int32 * len(vals))(*[int(v) for v in vals])


class PeerRegion:
    """One rank's symmetric region, mapped into every rank of the group (sonic_peer_*)."""

    def __init__(self, rank, world, nbytes):
        self.rank, self.world, self.nbytes = rank, world, int(nbytes)
        self.h = ctypes.c_void_p()
        self.blob = ctypes.create_string_buffer(SONIC_PEER_HANDLE_BYTES)
        _check(lib().sonic_peer_create(rank, world, self.nbytes, ctypes.byref(self.h), self.blob),
               "sonic_peer_create")

    def handle(self):
        """The exportable handle blob (bytes) of this rank."""
        return self.blob.raw

    def open(self, blobs):
        """blobs: the handle blobs of all ranks, rank-ordered."""
        assert len(blobs) == self.world and all(len(b) == SONIC_PEER_HANDLE_BYTES for b in blobs)
        buf = ctypes.create_string_buffer(b"".join(blobs), SONIC_PEER_HANDLE_BYTES * self.world)
        _check(lib().sonic_peer_open(self.h, buf), "sonic_peer_open")

    def view(self, offset, shape, dtype):
        """A torch tensor over the OWN region at byte offset `offset` (no copy)."""
        base = lib().sonic_peer_base(self.h, self.rank)
        numel = 1
        for v in shape:
            numel *= int(v)
        es = torch.empty(0, dtype=dtype).element_size()
        assert offset % 16 == 0 and offset + numel * es <= self.nbytes
        return _wrap_device_ptr(base + offset, numel * es).view(dtype)[:numel].view(*shape)

    def barrier(self):
        _done(lib().sonic_peer_barrier(self.h, _stream()), "sonic_peer_barrier")

    def pack(self, desc, G, plan, src, region_off, dst_row0):
        _done(lib().sonic_ep_pack_peer(ctypes.byref(desc), G, ctypes.byref(plan.c), _ptr(src), self.h,
                                       int(region_off), _i32(dst_row0), _stream()), "sonic_ep_pack_peer")

    def pack_dev(self, desc, G, plan, src, region_off, counts_off, count_cols):
        """Dispatch with the destination rows read on the device from the own count matrix."""
        _done(lib().sonic_ep_pack_peer_dev(ctypes.byref(desc), G, ctypes.byref(plan.c), _ptr(src), self.h,
                                           int(region_off), int(counts_off), int(count_cols), _stream()),
              "sonic_ep_pack_peer_dev")

    def put_rows_dev(self, src, row_bytes, direction, counts_off, count_cols, region_off):
        """Block put with the blocks read on the device from the own count matrix (0 dispatch, 1 return)."""
        _done(lib().sonic_peer_put_rows_dev(self.h, self.world, _ptr(src), int(row_bytes), int(direction),
                                            int(counts_off), int(count_cols), int(region_off), _stream()),
              "sonic_peer_put_rows_dev")

    def zero_tail(self, row_bytes, counts_off, count_cols, region_off, cap_rows):
        _done(lib().sonic_peer_zero_tail(self.h, self.world, int(row_bytes), int(counts_off), int(count_cols),
                                         int(region_off), int(cap_rows), _stream()), "sonic_peer_zero_tail")

    def put_rows(self, src, row_bytes, src_row0, cnt, dst_row0, region_off):
        _done(lib().sonic_peer_put_rows(self.h, self.world, _ptr(src), int(row_bytes), _i32(src_row0), _i32(cnt),
                                        _i32(dst_row0), int(region_off), _stream()), "sonic_peer_put_rows")

    def close(self):
        if self.h:
            _check(lib().sonic_peer_destroy(self.h), "sonic_peer_destroy")
            self.h = ctypes.c_void_p()


class _DevBuf:
    """__cuda_array_interface__ over a raw device pointer owned by libsonic (the peer region)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _wrap_device_ptr(ptr, nbytes):
    return torch.as_tensor(_DevBuf(ptr, nbytes), device="cuda")
