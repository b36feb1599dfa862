"""fp64 CPU oracle for the SonicMoE hot path (arXiv 2512.14080).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2512_14080_b200``) never imports it and
shares no code with it: no kernels, helpers, tables or constants.

Citations: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n (the paper
text and the CPU-desk spec written from it); ``Qk`` = reading k listed in
DESIGN.md §3 (the ambiguities of the paper and the reading adopted).

What is computed, and in which notation:

* routing (``route``): token-choice top-K (§2.3; stable, ties to the
  lower expert id, §4.3), then optionally token rounding
  (Alg. 4) with the NR-f subroutine, then the
  orphan rescue (Q14), gates renormalised over the kept set (Q13), and
  the canonical grouped-row metadata (offsets, gather map, token CSR).
* values (``forward`` / ``backward``): the plain definition of the MoE layer
  (Alg. 1) and its textbook gradients written the paper's way
  (Alg. 3, Alg. 5, App. C).  The method is
  exact up to rounding ("Both yield identical results"), so the oracle
  for values is the definition in fp64.
* ``backward_reference``: the Y/dY-materialising path of App. C.1
  (P:1773-1803), the cross-check of the memory-efficient rewrite.
* ``forward_dense``: every expert on every token, masked and gate-scaled.

Every array is float64 (bf16/fp32 inputs are converted exactly).  A library
primitive (numpy matmul, numpy stable sort) serves as a step; there is no
blocking, fusion or reordering beyond what the definitions state.

Parity pins live in ``tests/test_oracle.py``: dense brute force, finite
differences, the App. C identities, TR invariants, the SPEC worked examples
and hand-traced golden files under ``tests/golden/``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GEMM_M = 128  # grouped-row padding granularity of the GPU layout


# --------------------------------------------------------------------------
# SwiGLU (§2.2; layout [gate | up] per Q1 / S:293)
# --------------------------------------------------------------------------
def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def silu(x):
    """silu(x) = x * sigma(x)."""
    return x * sigmoid(x)


def dsilu(x):
    """silu'(x) = sigma(x) (1 + x (1 - sigma(x)))."""
    s = sigmoid(x)
    return s * (1.0 + x * (1.0 - s))


def swiglu(H):
    """A = SwiGLU(H) = silu(H[:, :n]) * H[:, n:]  (Q1)."""
    n = H.shape[-1] // 2
    return silu(H[..., :n]) * H[..., n:]


def dswiglu(dA, H):
    """(A, dH) = dAct_func(dA, H) (Alg. 3).

    d gate = dA * up * silu'(gate);  d up = dA * silu(gate).
    """
    n = H.shape[-1] // 2
    g, u = H[..., :n], H[..., n:]
    A = silu(g) * u
    dH = np.concatenate([dA * u * dsilu(g), dA * silu(g)], axis=-1)
    return A, dH


# --------------------------------------------------------------------------
# Routing
# --------------------------------------------------------------------------
def topk_tc(S, K):
    """Token-choice TopK over each row of S (§2.3, Alg. 4 step (1) P:1135).

    Order: value descending, ties to the lower expert id -- the stability the
    paper's packed-index bitonic sort guarantees (§4.3, Q9).
    numpy's stable argsort of -S is exactly that order.
    """
    S = np.asarray(S, dtype=np.float64)
    assert np.all(np.isfinite(S)), "NaN/inf scores are invalid input (Q24)"
    T, E = S.shape
    assert 1 <= K <= E
    order = np.argsort(-S, axis=1, kind="stable")[:, :K]
    return order.astype(np.int64), np.take_along_axis(S, order, axis=1)


def round_up(f, M):
    """ceil(f/M)*M  (Alg. 4 step (2))."""
    return -(-np.asarray(f) // M) * M


def round_down(f, M):
    """floor(f/M)*M  (Alg. 4 step (2))."""
    return (np.asarray(f) // M) * M


def round_nrf(f, M):
    """NR-f round_and_sparsify decision.

    "pad EC selected tokens if ceil(f)-f is smaller than f-floor(f)":
    strict '<', so an exact tie at M/2 rounds down (Q11).
    Returns the rounded counts.
    """
    f = np.asarray(f, dtype=np.int64)
    up, dn = round_up(f, M), round_down(f, M)
    return np.where((up - f) < (f - dn), up, dn)


def round_balance(f, M, T=None):
    """Balance-f (Alg. 6): one pass over the experts in index order with the
    accumulator z of the residuals chosen so far; expert e pads (rounds up) iff
    |r_up + z| < |r_down + z| (strict, as printed), else it drops (rounds down).  The up option is
    capped at T first (Q15), so r_up uses the capped count."""
    f = np.asarray(f, dtype=np.int64)
    out = np.empty_like(f)
    z = 0
    for e, fe in enumerate(f):
        up = int(round_up(fe, M))
        if T is not None:
            up = min(up, T)
        dn = int(round_down(fe, M))
        r_up, r_dn = up - int(fe), dn - int(fe)
        if abs(r_up + z) < abs(r_dn + z):
            out[e] = up
            z += r_up
        else:
            out[e] = dn
            z += r_dn
    return out


_MASK64 = (1 << 64) - 1


def sr_u64(seed, e):
    """The counter-based generator of SR-f (Q21): SplitMix64's output function applied to
    the state (seed << 32 | e) + 0x9E3779B97F4A7C15 (one step of SplitMix64 from that state)."""
    x = (((int(seed) & 0xFFFFFFFF) << 32) | (int(e) & 0xFFFFFFFF)) + 0x9E3779B97F4A7C15
    x &= _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


def round_sr(f, M, seed, T=None):
    """SR-f: expert e pads with probability (f_e - floor(f_e)) / M.  The draw is
    u_e = sr_u64(seed, e) >> 40, uniform on [0, 2^24); pad iff u_e / 2^24 < (f_e - floor) / M,
    i.e. u_e * M < (f_e - floor) * 2^24 (exact integer comparison)."""
    f = np.asarray(f, dtype=np.int64)
    out = np.empty_like(f)
    for e, fe in enumerate(f):
        up = int(round_up(fe, M))
        if T is not None:
            up = min(up, T)
        dn = int(round_down(fe, M))
        u = sr_u64(seed, e) >> 40
        out[e] = up if u * M < (int(fe) - dn) * (1 << 24) else dn
    return out


def round_nrs(S, tc, f, M, seed, T):
    """NR-s: pad expert e with probability
        p_e = (sum_t s_e,t - sum_t floor(s)_e,t) / (sum_t ceil(s)_e,t - sum_t floor(s)_e,t),
    s_e the scores of e's TC tokens, floor(s)_e those of pi_e[:floor(f_e)], ceil(s)_e those of
    pi_e[:ceil(f_e)] (pi_e = Alg. 4's ranking, _rank_expert_column).  The sums are fp64 sums of the
    fp32 scores; the draw is SR-f's (u_e = sr_u64(seed, e) >> 40, Q21): pad iff u_e < p_e 2^24."""
    f = np.asarray(f, dtype=np.int64)
    out = np.empty_like(f)
    for e, fe in enumerate(f):
        fe = int(fe)
        dn = int(round_down(fe, M))
        up = min(int(round_up(fe, M)), T)
        if dn == fe:
            out[e] = fe
            continue
        order = _rank_expert_column(S[:, e], tc[:, e])
        s_tc = float(np.sum(S[order[:fe], e]))
        s_dn = float(np.sum(S[order[:dn], e]))
        s_up = float(np.sum(S[order[:up], e]))
        with np.errstate(divide="ignore", invalid="ignore"):
            p = np.float64(s_tc - s_dn) / np.float64(s_up - s_dn)
        u = sr_u64(seed, e) >> 40
        out[e] = up if float(u) < float(p) * 16777216.0 else dn
    return out


def ec_capacity(T, K, E, M):
    """Expert-choice capacity (Q22): the average TC load ceil(T K / E), rounded up to a multiple of
    M_tile and capped at T."""
    return min(int(round_up(-(-T * K // E), M)), T)


def _rank_expert_column(S_col, tc_col):
    """Alg. 4 steps (3)-(4) for one expert: pi_e = sort(S'_e) descending.

    The paper builds S' = S - 1 with the top-K entries restored to S
     so that TC tokens rank above every non-TC token, then sorts
    the column.  Reading Q10: the intent is the lexicographic key
    (in-TC desc, S desc, token asc) -- S - 1 rounds tiny scores together in
    fp32.  Ties in S go to the lower token index (Q12).
    """
    T = S_col.shape[0]
    # np.lexsort: last key is primary.
    return np.lexsort((np.arange(T), -S_col, ~tc_col))


def _paper_S_prime(S, tc):
    """Alg. 4 step (3) literally: S' = S - 1, TC entries restored.

    Used only by the tests to pin _rank_expert_column to the paper's form.
    """
    Sp = np.asarray(S, np.float64) - 1.0
    Sp[tc] = np.asarray(S, np.float64)[tc]
    return Sp


@dataclass
class Routing:
    """Routing result plus the canonical grouped-row metadata.

    Fields mirror ``sonic_routing`` in include/sonic.h.
    """
    topk_ids: np.ndarray      # [T,K] int  TC choice, value-desc, ties -> lower id
    topk_s: np.ndarray        # [T,K] f64
    f: np.ndarray             # [E]   TC counts (Alg. 4 step (2))
    f_rounded: np.ndarray     # [E]   kept counts (== f under TC)
    kept: np.ndarray          # [T,E] bool, pi (kept set)
    gate: np.ndarray          # [T,E] f64, g_te = S_te / sum_{kept} S_te' (0 off the kept set)
    offsets: np.ndarray       # [E+1] exclusive prefix of f_rounded
    pad_offsets: np.ndarray   # [E+1] exclusive prefix of ceil(f_rounded/GEMM_M)*GEMM_M
    row_token: np.ndarray     # [R_pad] token of each grouped row, -1 on pad rows
    row_expert: np.ndarray    # [R_pad] expert of each grouped row
    row_gate: np.ndarray      # [R_pad] gate of each grouped row, 0 on pad rows
    token_rowptr: np.ndarray  # [T+1]  CSR over tokens
    token_rows: np.ndarray    # [R]    grouped rows of each token, expert-ascending
    tile_expert: np.ndarray   # [R_pad/GEMM_M] expert of each 128-row tile
    flipped: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))  # experts flipped by the rescue

    @property
    def R(self):
        return int(self.offsets[-1])

    @property
    def R_pad(self):
        return int(self.pad_offsets[-1])


TR_ROUNDINGS = ("nrf", "up", "down", "balance", "sr", "nrs")


def route(S, K, mode="tc", m_tile=128, rescue=True, gate_raw=False, rounding="nrf", seed=0):
    """Routing per Alg. 4, plain TC or expert choice.

    mode "tc": kept = TC top-K set.
    mode "tr": token rounding; ``rounding`` picks the subroutine of App.: "nrf"
      (default), "up", "down", "balance" (Alg. 6), "sr" (the
      draws from ``sr_u64(seed, e)``), "nrs" (score-weighted, same draws).  The orphan rescue (Q14) applies to every subroutine.
    mode "ec": expert choice (NEXT-3, Q22): every expert keeps the ``ec_capacity`` highest-scoring
      tokens (S desc, token asc); no rescue -- tokens no expert chose have no rows.
    """
    S = np.asarray(S, dtype=np.float64)
    T, E = S.shape
    ids, vals = topk_tc(S, K)                                  # step (1)
    tc = np.zeros((T, E), dtype=bool)
    tc[np.arange(T)[:, None], ids] = True
    f = tc.sum(axis=0).astype(np.int64)                        # step (2): f_e
    flipped = np.zeros(0, np.int64)
    if mode == "tc":
        f_r = f.copy()
        kept = tc.copy()
    elif mode == "ec":
        C = ec_capacity(T, K, E, m_tile)
        f_r = np.full(E, C, dtype=np.int64)
        kept = np.zeros((T, E), dtype=bool)
        for e in range(E):
            order = np.lexsort((np.arange(T), -S[:, e]))       # S desc, token asc
            kept[order[:C], e] = True
    elif mode == "tr":
        f_up = np.minimum(round_up(f, m_tile), T)              # Q15: cap at T
        if rounding == "nrf":
            f_r = np.minimum(round_nrf(f, m_tile), T)          # round_and_sparsify (NR-f)
        elif rounding == "up":
            f_r = f_up.copy()
        elif rounding == "down":
            f_r = round_down(f, m_tile).astype(np.int64)
        elif rounding == "balance":
            f_r = round_balance(f, m_tile, T)
        elif rounding == "sr":
            f_r = round_sr(f, m_tile, seed, T)
        elif rounding == "nrs":
            f_r = round_nrs(S, tc, f, m_tile, seed, T)
        else:
            raise ValueError(rounding)
        kept = np.zeros((T, E), dtype=bool)

        def select(e):                                         # step (4), one expert
            kept[:, e] = False
            order = _rank_expert_column(S[:, e], tc[:, e])     # steps (3)+(4): sort(S'_e)
            kept[order[: f_r[e]], e] = True

        for e in range(E):
            select(e)
        if rescue:                                             # Q14 orphan rescue
            orphan = ~kept.any(axis=1)
            flip = np.unique(ids[orphan, 0])
            for e in flip:
                f_r[e] = f_up[e]
                select(e)
            flipped = flip.astype(np.int64)
            assert kept.any(axis=1).all()
    else:
        raise ValueError(mode)

    if gate_raw:
        gate = np.where(kept, S, 0.0)
    else:                                                      # P:1488 renormalisation (Q13)
        denom = np.where(kept, S, 0.0).sum(axis=1, keepdims=True)
        gate = np.where(kept, S / np.where(denom == 0, 1.0, denom), 0.0)
    return build_metadata(ids, vals, f, f_r, kept, gate, flipped)


def build_metadata(ids, vals, f, f_r, kept, gate, flipped):
    """Canonical grouped layout (P:787 footnote "routing metadata").

    Segment e holds e's kept tokens in ascending token order (Q17) and starts
    at a GEMM_M-aligned row; rows past f_r[e] inside the last tile are pad rows.
    Token CSR lists each token's rows in ascending expert order.
    """
    T, E = kept.shape
    offsets = np.zeros(E + 1, np.int64)
    offsets[1:] = np.cumsum(f_r)
    padded = round_up(f_r, GEMM_M)
    pad_offsets = np.zeros(E + 1, np.int64)
    pad_offsets[1:] = np.cumsum(padded)
    R_pad = int(pad_offsets[-1])
    row_token = np.full(R_pad, -1, np.int64)
    row_expert = np.zeros(R_pad, np.int64)
    row_gate = np.zeros(R_pad, np.float64)
    row_of = np.full((T, E), -1, np.int64)
    for e in range(E):
        toks = np.nonzero(kept[:, e])[0]                       # ascending
        base = pad_offsets[e]
        row_token[base: base + len(toks)] = toks
        row_expert[base: pad_offsets[e + 1]] = e
        row_gate[base: base + len(toks)] = gate[toks, e]
        row_of[toks, e] = base + np.arange(len(toks))
    cnt = kept.sum(axis=1)
    token_rowptr = np.zeros(T + 1, np.int64)
    token_rowptr[1:] = np.cumsum(cnt)
    token_rows = np.zeros(int(token_rowptr[-1]), np.int64)
    for t in range(T):
        es = np.nonzero(kept[t])[0]                            # ascending expert
        token_rows[token_rowptr[t]: token_rowptr[t + 1]] = row_of[t, es]
    tile_expert = row_expert[::GEMM_M].copy() if R_pad else np.zeros(0, np.int64)
    return Routing(ids, vals, f, f_r, kept, gate, offsets, pad_offsets, row_token,
                   row_expert, row_gate, token_rowptr, token_rows, tile_expert, flipped)


# --------------------------------------------------------------------------
# Forward (Alg. 1 P:200-242 as the definition; Alg. 2 P:528-592 stages)
# --------------------------------------------------------------------------
@dataclass
class ForwardResult:
    O: np.ndarray            # [T,d]
    H: dict                  # e -> [f_e, 2n]  (cached, §3.2)
    A: dict                  # e -> [f_e, n]
    Y: dict                  # e -> [f_e, d]   gate-scaled (Q2)
    tokens: dict             # e -> kept tokens ascending


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def expert_forward(Xe, W1e, W2e, ge):
    """One expert's forward on its gathered rows (Alg. 2):
    H_e = X_e W1_e;  A_e = act(H_e) (SwiGLU);  Y_e = g_e * (A_e W2_e) (gate before
    aggregation, Q2 / P:1774 option (1)).  ``Xe`` = Gather(X, pi_:,e) [f_e, d], ``ge`` [f_e]."""
    He = Xe @ W1e                                              # H_e = X_e W1_e
    Ae = swiglu(He)                                            # A_e = act(H_e)
    Ye = np.asarray(ge)[:, None] * (Ae @ W2e)                  # Y_e scaled by g (Q2)
    return He, Ae, Ye


# --------------------------------------------------------------------------
# FP8 up-projection (NEXT-4; the paper's future work): e4m3 operands with one scale per
# token row of X and one per output column of W1_e, fp32 accumulation, the scales applied to the sum
# --------------------------------------------------------------------------
E4M3_MAX = 448.0


def e4m3_round(x):
    """Round to the nearest OCP FP8 E4M3 value, ties to even, finite values beyond the largest
    (448) saturated to +-448 (cvt.rn.satfinite).  E4M3: bias 7, 3 mantissa bits: normals
    m * 2^e with m in [1, 2) on a grid of 2^(e-3) for e >= -6, subnormals on the grid 2^-9."""
    x = np.asarray(x, dtype=np.float64)
    a = np.abs(x)
    _, ex = np.frexp(np.where(a > 0, a, 1.0))       # a = m 2^ex, m in [0.5, 1): floor(log2 a) = ex - 1
    e = np.maximum(ex - 1, -6)                      # below 2^-6 the spacing stays 2^-9 (subnormals)
    q = np.ldexp(1.0, e - 3)                        # spacing of the grid around a
    r = np.minimum(np.rint(a / q) * q, E4M3_MAX)    # a / q and the product are exact; rint: ties to even
    return np.copysign(r, x)


def quantize_e4m3(M, axis):
    """Per-slice e4m3 quantisation along `axis` (the reduction dimension K): scale = amax / 448 in
    fp32 (1 where amax = 0), q = e4m3_round(fl32(M / scale)).  Returns (q, scale) with
    M ~= q * scale; q and scale are exactly what the GPU's quantisation kernels produce."""
    M32 = np.asarray(M, dtype=np.float32)
    amax = np.max(np.abs(M32), axis=axis, keepdims=True).astype(np.float32)
    scale = np.where(amax > 0, amax / np.float32(E4M3_MAX), np.float32(1.0)).astype(np.float32)
    q = e4m3_round((M32 / scale).astype(np.float32))
    return q, np.squeeze(scale, axis=axis).astype(np.float64)


def bf16_round(x):
    """Round to the nearest bfloat16 value (ties to even) from float64 in one step: 8 significant
    bits, so the grid around |x| in [2^e, 2^(e+1)) is 2^(e-7) (normals from 2^-126)."""
    x = np.asarray(x, dtype=np.float64)
    a = np.abs(x)
    _, ex = np.frexp(np.where(a > 0, a, 1.0))
    e = np.maximum(ex - 1, -126)
    q = np.ldexp(1.0, e - 7)
    return np.copysign(np.rint(a / q) * q, x)


def fp8_dxt_rows(dH_e, sw_e):
    """The e4m3 operand of the FP8 dX~ GEMM (NEXT-4, Q25): the stored (bf16) dH rows times the forward's
    per-column W1 scales sw_e[j] in fp32 -- folding the weight scale, which varies along this GEMM's
    reduction dimension j, into dH -- then quantised per row: s = fl32(amax / 448) (1 where amax = 0),
    r = fl32(1 / s), q = e4m3_round(fl32(M r)) (one multiply per element by the row's reciprocal scale).
    Returns (q [f_e, 2n], s [f_e])."""
    dHb = bf16_round(dH_e).astype(np.float32)
    M = (dHb * np.asarray(sw_e, dtype=np.float32)[None, :]).astype(np.float32)
    amax = np.max(np.abs(M), axis=1, keepdims=True).astype(np.float32)
    scale = np.where(amax > 0, amax / np.float32(E4M3_MAX), np.float32(1.0)).astype(np.float32)
    rcp = (np.float32(1.0) / scale).astype(np.float32)
    q = e4m3_round((M * rcp).astype(np.float32))
    return q, np.squeeze(scale, axis=1).astype(np.float64)


def expert_dxt_fp8(dH_e, W1q_e, sw_e):
    """dX~_e on e4m3 operands: s_r * sum_j q_rj W1q_e[i, j] with (q, s) = fp8_dxt_rows(dH_e, sw_e):
    = sum_j (s_r q_rj / sw_j) (sw_j W1q_e[i, j]), the definition on the dequantised operands."""
    q, s = fp8_dxt_rows(dH_e, sw_e)
    return _f64(s)[:, None] * (_f64(q) @ _f64(W1q_e).T)


def fp8_up_operands(X, W1):
    """X [T,d] -> (Xq, sx [T]) per token row; W1 [E,d,2n] -> (W1q, sw [E,2n]) per output column."""
    Xq, sx = quantize_e4m3(X, axis=1)
    W1q, sw = quantize_e4m3(W1, axis=1)
    return Xq, sx, W1q, sw


def expert_forward_fp8(Xq_e, sx_e, W1q_e, sw_e, W2e, ge):
    """expert_forward with the up-projection on the quantised operands:
    H_e = (Xq_e W1q_e) * sx_e[:, None] * sw_e[None, :]; the rest as expert_forward."""
    He = (_f64(Xq_e) @ _f64(W1q_e)) * _f64(sx_e)[:, None] * _f64(sw_e)[None, :]
    Ae = swiglu(He)
    Ye = np.asarray(ge)[:, None] * (Ae @ _f64(W2e))
    return He, Ae, Ye


def forward(X, W1, W2, rt: Routing, experts=None, fp8_up=False):
    """O_t = sum_e pi_te g_te Y_{e,t},  Y_e = SwiGLU(X_e W1_e) W2_e.

    The gate multiplies Y before aggregation (Q2, P:1774 option (1)); the
    result is identical in exact arithmetic.
    """
    X, W1, W2 = _f64(X), _f64(W1), _f64(W2)
    T, d = X.shape
    E = W1.shape[0]
    O = np.zeros((T, d))
    H, A, Y, tokens = {}, {}, {}, {}
    if fp8_up:
        Xq, sx, W1q, sw = fp8_up_operands(X, W1)
    for e in (range(E) if experts is None else experts):
        toks = np.nonzero(rt.kept[:, e])[0]
        if fp8_up:
            He, Ae, Ye = expert_forward_fp8(Xq[toks], sx[toks], W1q[e], sw[e], W2[e], rt.gate[toks, e])
        else:
            He, Ae, Ye = expert_forward(X[toks], W1[e], W2[e], rt.gate[toks, e])  # X_e = Gather(X, pi_:,e)
        np.add.at(O, toks, Ye)                                 # O_t = sum_e ...
        H[e], A[e], Y[e], tokens[e] = He, Ae, Ye, toks
    return ForwardResult(O, H, A, Y, tokens)


def forward_dense(X, W1, W2, kept, gate):
    """Brute force: every expert on every token, masked by pi and scaled by g."""
    X, W1, W2 = _f64(X), _f64(W1), _f64(W2)
    O = np.zeros((X.shape[0], W2.shape[2]))
    for e in range(W1.shape[0]):
        Ye = swiglu(X @ W1[e]) @ W2[e]
        O += (kept[:, e] * gate[:, e])[:, None] * Ye
    return O


# --------------------------------------------------------------------------
# Backward, memory-efficient path (Alg. 3 P:595-706 + Alg. 5)
# --------------------------------------------------------------------------
@dataclass
class BackwardResult:
    dX: np.ndarray           # [T,d]
    dW1: np.ndarray          # [E,d,2n]
    dW2: np.ndarray          # [E,n,d]
    dS: dict                 # e -> [f_e]  dL/dg for each kept (t,e), ascending t
    dH: dict                 # e -> [f_e,2n]
    A_prime: dict            # e -> [f_e,n]
    dXt: dict                # e -> [f_e,d]  dX~ rows


@dataclass
class ExpertGrads:
    """One expert's backward outputs (Alg. 3 + Alg. 5), rows in ascending token order."""
    dAp: np.ndarray          # [f_e,n]   dA' = Gather(dO) W2_e^T
    A: np.ndarray            # [f_e,n]   A = SwiGLU(H)
    dH: np.ndarray           # [f_e,2n]
    A_prime: np.ndarray      # [f_e,n]   A' = s A
    dS: np.ndarray           # [f_e]     <dA', A>
    dW1: np.ndarray          # [d,2n]
    dW2: np.ndarray          # [n,d]
    dXt: np.ndarray          # [f_e,d]   dX~ rows


def expert_backward(dOe, Xe, W1e, W2e, ge, He=None):
    """One expert's backward on its gathered rows, Alg. 3 then Alg. 5:

    dA'_e = Gather(dO) W2_e^T;  dA_e = s_e dA'_e;  (A_e, dH_e) = dSwiGLU(dA_e, H_e);
    A'_e = s_e A_e;  dS_e,t = <dA'_e,t, A_e,t> (boxed eq. P:1752);
    dW2_e = A'_e^T dO_e (Q4);  dX~_e = dH_e W1_e^T;  dW1_e = X_e^T dH_e.
    H_e is recomputed from X_e unless given (only X and H are cached, sec. 3.2)."""
    s = np.asarray(ge)[:, None]                                # s_e = Gather(S, pi_:,e)
    if He is None:
        He = Xe @ W1e
    dAp = dOe @ W2e.T                                          # dA'_e
    dA = s * dAp                                               # dA_e
    Ae, dHe = dswiglu(dA, He)                                  # A_e, dH_e
    Ape = s * Ae                                               # A'_e
    return ExpertGrads(dAp=dAp, A=Ae, dH=dHe, A_prime=Ape,
                       dS=np.sum(dAp * Ae, axis=1),            # <dA'_e,t, A_e,t>
                       dW1=Xe.T @ dHe,                         # dW1_e = X_e^T dH_e
                       dW2=Ape.T @ dOe,                        # dW2_e = A'^T dO_e
                       dXt=dHe @ W1e.T)                        # dX~_e = dH_e W1_e^T


def backward(dO, X, W1, W2, rt: Routing, experts=None, H_cache=None, fp8_dxt=False):
    """Alg. 3 then Alg. 5 for every expert (``expert_backward``), then
    dX_t = sum_e pi_te dX~_e,t (Alg. 5's aggregation).
    ``experts`` restricts the work (dX then holds only those experts' terms).
    fp8_dxt: dX~_e on e4m3 operands (``expert_dxt_fp8``; W1 quantised per column as in the forward's
    fp8 up-projection) from the dH the method stores -- computed from the bf16-cached H and
    rounded to bf16 (Q25); every other output is the bf16 path's.
    """
    dO, X, W1, W2 = _f64(dO), _f64(X), _f64(W1), _f64(W2)
    T, d = X.shape
    E, _, n2 = W1.shape
    n = n2 // 2
    dX = np.zeros((T, d))
    dW1 = np.zeros((E, d, n2))
    dW2 = np.zeros((E, n, d))
    dS, dH, Ap, dXt = {}, {}, {}, {}
    if fp8_dxt:
        W1q, sw = quantize_e4m3(W1, axis=1)
    for e in (range(E) if experts is None else experts):
        toks = np.nonzero(rt.kept[:, e])[0]
        g = expert_backward(dO[toks], X[toks], W1[e], W2[e], rt.gate[toks, e],
                            None if H_cache is None else _f64(H_cache[e]))
        if fp8_dxt:
            Hb = bf16_round(X[toks] @ W1[e] if H_cache is None else _f64(H_cache[e]))
            gb = expert_backward(dO[toks], X[toks], W1[e], W2[e], rt.gate[toks, e], Hb)
            g.dXt = expert_dxt_fp8(gb.dH, W1q[e], sw[e])
        dW1[e], dW2[e] = g.dW1, g.dW2
        np.add.at(dX, toks, g.dXt)                             # dX_t = sum_e dX~_e,t
        dS[e], dH[e], Ap[e], dXt[e] = g.dS, g.dH, g.A_prime, g.dXt
    return BackwardResult(dX, dW1, dW2, dS, dH, Ap, dXt)


def backward_reference(dO, X, W1, W2, rt: Routing):
    """App. C.1 path: materialise Y (unscaled) and dY = s dO.

    dS_t,e = <dO_t, Y_e,t> with Y_e = A_e W2_e (P:1752 first form);
    dW2_e = A_e^T dY_e;  dA_e = dY_e W2_e^T.
    """
    dO, X, W1, W2 = _f64(dO), _f64(X), _f64(W1), _f64(W2)
    T, d = X.shape
    E, _, n2 = W1.shape
    n = n2 // 2
    dX = np.zeros((T, d))
    dW1 = np.zeros((E, d, n2))
    dW2 = np.zeros((E, n, d))
    dS, dH = {}, {}
    for e in range(E):
        toks = np.nonzero(rt.kept[:, e])[0]
        s = rt.gate[toks, e][:, None]
        He = X[toks] @ W1[e]
        Ae = swiglu(He)
        Ye = Ae @ W2[e]                                        # unscaled Y
        dYe = s * dO[toks]                                     # eq. dY
        dS[e] = np.sum(dO[toks] * Ye, axis=1)                  # <dO_t, Y_e,t>
        dW2[e] = Ae.T @ dYe                                    # A^T dY
        dA = dYe @ W2[e].T
        _, dHe = dswiglu(dA, He)
        dW1[e] = X[toks].T @ dHe
        np.add.at(dX, toks, dHe @ W1[e].T)
        dH[e] = dHe
    return BackwardResult(dX, dW1, dW2, dS, dH, {}, {})


# --------------------------------------------------------------------------
# Per-token evaluation for sampled parity at full size (same definitions, one token at a time)
# --------------------------------------------------------------------------
def forward_tokens(X, W1, W2, rt: Routing, tokens):
    """O_t = sum_{e in kept(t)} g_te SwiGLU(X_t W1_e) W2_e for the listed tokens."""
    out = np.zeros((len(tokens), W2.shape[2]))
    for i, t in enumerate(tokens):
        x = _f64(X[t])
        for e in np.nonzero(rt.kept[t])[0]:
            a = swiglu(x @ _f64(W1[e]))
            out[i] += rt.gate[t, e] * (a @ _f64(W2[e]))
    return out


def backward_experts(dO, X, W1, W2, rt: Routing, experts):
    """dW1_e, dW2_e and the dS of every kept row of each listed expert (``expert_backward``),
    converting only those experts' weights to fp64 (W1 / W2 may be lazy per-expert views).
    Returns {e: (dW1_e, dW2_e, dS_e)}.  Pinned against ``backward`` in tests/test_oracle.py."""
    out = {}
    for e in experts:
        toks = np.nonzero(rt.kept[:, e])[0]
        g = expert_backward(_f64(dO[toks]), _f64(X[toks]), _f64(W1[e]), _f64(W2[e]), rt.gate[toks, e])
        out[e] = (g.dW1, g.dW2, g.dS)
    return out


def backward_tokens(dO, X, W1, W2, rt: Routing, tokens):
    """dX_t and dS_(t,e) for the listed tokens, Alg. 3 + Alg. 5 row by row.

    Returns (dX [len(tokens), d], {(t, e): dS}).
    """
    dX = np.zeros((len(tokens), X.shape[1]))
    dS = {}
    for i, t in enumerate(tokens):
        x, g_o = _f64(X[t]), _f64(dO[t])
        for e in np.nonzero(rt.kept[t])[0]:
            s = rt.gate[t, e]
            h = x @ _f64(W1[e])
            dap = g_o @ _f64(W2[e]).T                          # dA' row
            a, dh = dswiglu(s * dap, h)                        # dA = s dA'
            dS[(t, e)] = float(np.dot(dap, a))                 # <dA', A>
            dX[i] += dh @ _f64(W1[e]).T                        # dX~ row, summed
    return dX, dS


# --------------------------------------------------------------------------
# Finite differences: L = sum G * O with routing held fixed
# --------------------------------------------------------------------------
def loss_fixed_routing(X, W1, W2, kept, gate, G):
    return float(np.sum(_f64(G) * forward_dense(X, W1, W2, kept, gate)))


def fd_grad(fun, x, h=1e-5, coords=None):
    """Central differences (f(x+h) - f(x-h)) / 2h at the given flat coords."""
    x = np.array(x, dtype=np.float64)
    flat = x.reshape(-1)
    idx = range(flat.size) if coords is None else coords
    out = {}
    for i in idx:
        old = flat[i]
        flat[i] = old + h
        fp = fun(x)
        flat[i] = old - h
        fm = fun(x)
        flat[i] = old
        out[i] = (fp - fm) / (2 * h)
    return out


# --------------------------------------------------------------------------
# Closed forms (§3.2; Eq. 4)
# --------------------------------------------------------------------------
def model_flops(T, d, n, K, fwd_only=False):
    """(6+12) T n K d; forward alone is 6 T n K d."""
    return (6 if fwd_only else 18) * T * n * K * d


def activation_bytes(T, d, n, K):
    """2Td + 4TKn bytes: X and H in bf16."""
    return 2 * T * d + 4 * T * K * n


def arithmetic_intensity(T, d, n, E, K):
    """Eq. 4: 3 / ((2+2G)/d + 3/(T rho)), G = d/n, rho = K/E."""
    G, rho = d / n, K / E
    return 3.0 / ((2 + 2 * G) / d + 3.0 / (T * rho))


# --------------------------------------------------------------------------
# Router softmax (NEXT-4; "optional softmax fusion on top-K values")
# --------------------------------------------------------------------------
def softmax(logits):
    """S_te = exp(l_te) / sum_e' exp(l_te'), per token (row), in fp64; the max-subtraction is the
    textbook overflow guard (it cancels exactly in the ratio).  The scores S that ``route`` takes
    (S = softmax of the router logits)."""
    lg = np.asarray(logits, dtype=np.float64)
    z = np.exp(lg - lg.max(axis=1, keepdims=True))
    return z / z.sum(axis=1, keepdims=True)


def router_logits(X, Wr):
    """The router GEMM (scores S = softmax(X W_r)): logits = X W_r, [T, d] x [d, E]."""
    return np.asarray(X, dtype=np.float64) @ np.asarray(Wr, dtype=np.float64)


def router_input_grads(X, Wr, dlogits):
    """Gradients of the router GEMM given d logits (chain rule of logits = X W_r):
    dX_router = dlogits W_r^T (added to the MoE layer's dX), dW_r = X^T dlogits."""
    X = np.asarray(X, dtype=np.float64)
    Wr = np.asarray(Wr, dtype=np.float64)
    dl = np.asarray(dlogits, dtype=np.float64)
    return dl @ Wr.T, X.T @ dl


# --------------------------------------------------------------------------
# Router backward (NEXT-4): dS -> d logits through the renormalisation and the softmax
# --------------------------------------------------------------------------
def router_backward(S, rt: Routing, dS_te, gate_raw=False):
    """d logits of the router for a fixed routing (the top-K / rounding choice is piecewise
    constant and has no gradient).

    Gates (Q13): g_te = S_te / Z_t with Z_t = sum_{e' kept for t} S_te' (or g = S with
    ``gate_raw``).  Chain rule, written per token:
      dS_full_te = (dS_te - sum_{e' kept} dS_te' g_te') / Z_t   for kept e, 0 otherwise
      (gate_raw: dS_full_te = dS_te for kept e);
      d logit_tj = S_tj (dS_full_tj - sum_i S_ti dS_full_ti)      (softmax Jacobian, S = softmax).
    ``dS_te`` is a dense [T, E] array holding dL/dg_te on kept (t, e) and zeros elsewhere.
    """
    S = np.asarray(S, dtype=np.float64)
    dS_te = np.asarray(dS_te, dtype=np.float64)
    kept = rt.kept
    T, E = S.shape
    dfull = np.zeros((T, E))
    for t in range(T):
        ks = np.nonzero(kept[t])[0]
        if len(ks) == 0:
            continue
        if gate_raw:
            dfull[t, ks] = dS_te[t, ks]
        else:
            Z = S[t, ks].sum()
            g = S[t, ks] / Z
            dfull[t, ks] = (dS_te[t, ks] - np.dot(dS_te[t, ks], g)) / Z
    dot = (S * dfull).sum(axis=1, keepdims=True)
    return S * (dfull - dot)


def dS_dense(rt: Routing, dS_by_expert):
    """The per-expert dS lists of ``backward`` as a dense [T, E] array (zeros off the kept set)."""
    T, E = rt.kept.shape
    out = np.zeros((T, E))
    for e in range(E):
        toks = np.nonzero(rt.kept[:, e])[0]
        if len(toks):
            out[toks, e] = dS_by_expert[e]
    return out
