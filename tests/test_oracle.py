"""Pins for the fp64 oracle (oracle/moe_oracle.py) -- things the paper and the
mathematics fix, chosen so that a dropped term, a wrong sign/index or a
transposed operand anywhere in the oracle fails at least one of them.

None of these tests touch the GPU path.
"""
import json
import os

import numpy as np
import pytest

from oracle import moe_oracle as om

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tr_examples.json")))


def rand_case(seed, T, d, n, E, K, mode="tc", m_tile=4, ties=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((T, d))
    W1 = rng.standard_normal((E, d, 2 * n)) / np.sqrt(d)
    W2 = rng.standard_normal((E, n, d)) / np.sqrt(n)
    L = rng.standard_normal((T, E))
    if ties:
        L = np.round(L * ties) / ties
    S = np.exp(L) / np.exp(L).sum(1, keepdims=True)
    dO = rng.standard_normal((T, d))
    rt = om.route(S, K, mode=mode, m_tile=m_tile)
    return X, W1, W2, S, dO, rt


# ------------------------------------------------------------------ SwiGLU
def test_swiglu_golden():
    g = GOLD["swiglu"]
    assert om.swiglu(np.array([1.0, 1.0])) == pytest.approx(g["sigma1"], abs=1e-16)
    assert om.dsilu(0.0) == g["dsilu0"]
    assert om.dsilu(1.0) == pytest.approx(g["dsilu1"], abs=1e-15)
    assert om.dsilu(-2.0) == pytest.approx(g["dsilu_m2"], abs=1e-15)
    A, dH = om.dswiglu(np.array([1.0]), np.array([0.0, 1.0]))
    assert A[0] == 0.0 and dH[0] == 0.5 and dH[1] == 0.0
    assert om.swiglu(np.array([0.0, 7.0]))[0] == 0.0


def test_dswiglu_matches_finite_differences():
    rng = np.random.default_rng(1)
    H = rng.standard_normal((5, 6))
    dA = rng.standard_normal((5, 3))
    _, dH = om.dswiglu(dA, H)
    h = 1e-6
    for i in range(5):
        for j in range(6):
            Hp, Hm = H.copy(), H.copy()
            Hp[i, j] += h
            Hm[i, j] -= h
            fd = (np.sum(dA * om.swiglu(Hp)) - np.sum(dA * om.swiglu(Hm))) / (2 * h)
            assert dH[i, j] == pytest.approx(fd, rel=1e-7, abs=1e-9)


# ------------------------------------------------------------------ top-K
def test_topk_spec_example():
    ex = GOLD["topk"][0]
    ids, vals = om.topk_tc(np.array([ex["row"]]), ex["K"])
    assert ids[0].tolist() == ex["ids"] and vals[0].tolist() == ex["vals"]


@pytest.mark.parametrize("E,K", [(8, 1), (8, 8), (64, 8), (512, 16), (4096, 16)])
def test_topk_brute_force_with_ties(E, K):
    rng = np.random.default_rng(E * 31 + K)
    rows = np.round(rng.standard_normal((40, E)) * 3) / 3       # many exact ties
    ids, vals = om.topk_tc(rows, K)
    for r in range(rows.shape[0]):
        ref = sorted(range(E), key=lambda i: (-rows[r, i], i))[:K]
        assert ids[r].tolist() == ref
        assert vals[r].tolist() == [rows[r, i] for i in ref]


def test_topk_monotone_transform_invariance():
    rng = np.random.default_rng(3)
    S = rng.standard_normal((50, 32))
    a, _ = om.topk_tc(S, 8)
    b, _ = om.topk_tc(np.exp(3 * S) + 1.0, 8)
    assert np.array_equal(a, b)


# ------------------------------------------------------------------ rounding
def test_nrf_and_updown_golden():
    ex = GOLD["nrf"][0]
    assert om.round_nrf(ex["f"], ex["M"]).tolist() == ex["f_r"]
    ex = GOLD["updown"][0]
    assert om.round_up(ex["f"], ex["M"]).tolist() == ex["up"]
    assert om.round_down(ex["f"], ex["M"]).tolist() == ex["down"]


@pytest.mark.parametrize("ex", GOLD["tr"], ids=lambda e: e["cite"][:40])
def test_token_rounding_hand_traced(ex):
    S = np.array(ex["S"])
    rt = om.route(S, ex["K"], mode="tr", m_tile=ex["M"], rescue=ex["rescue"])
    assert rt.f.tolist() == ex["f"]
    assert rt.f_rounded.tolist() == ex["f_r"]
    for e, toks in enumerate(ex["kept"]):
        assert np.nonzero(rt.kept[:, e])[0].tolist() == toks
    assert rt.flipped.tolist() == ex["flipped"]


def test_rank_matches_paper_S_prime_form():
    """Alg. 4 step (3) literally (S' = S - 1, TC restored, sorted descending,
    ties to the lower token) ranks exactly as the lexicographic key (Q10)
    whenever S - 1 is exact in fp64 (softmax scores of N(0,1) logits)."""
    for seed in range(10):
        rng = np.random.default_rng(seed)
        L = np.round(rng.standard_normal((300, 16)) * 4) / 4
        S = (np.exp(L) / np.exp(L).sum(1, keepdims=True)).astype(np.float32).astype(np.float64)
        ids, _ = om.topk_tc(S, 3)
        tc = np.zeros(S.shape, bool)
        tc[np.arange(300)[:, None], ids] = True
        Sp = om._paper_S_prime(S, tc)
        for e in range(16):
            paper = np.argsort(-Sp[:, e], kind="stable")
            assert np.array_equal(paper, om._rank_expert_column(S[:, e], tc[:, e]))


@pytest.mark.parametrize("M", [4, 16, 128, 256])  # 256: the 2-CTA pair's M tile (Q16)
def test_token_rounding_invariants(M):
    """North-star TR invariants + P:1236/P:1243 locality, over 100 seeds."""
    for seed in range(100 if M < 128 else 20):
        rng = np.random.default_rng(seed)
        T, E, K = (64, 8, 2) if M < 128 else (1024, 16, 4)
        L = rng.standard_normal((T, E)) + (rng.standard_normal((1, E)) if seed % 2 else 0)
        S = np.exp(L) / np.exp(L).sum(1, keepdims=True)
        for rescue in (False, True):
            rt = om.route(S, K, mode="tr", m_tile=M, rescue=rescue)
            ids, _ = om.topk_tc(S, K)
            tc = np.zeros((T, E), bool)
            tc[np.arange(T)[:, None], ids] = True
            f = tc.sum(0)
            assert np.all(rt.f == f)
            assert np.all(rt.f_rounded % M == 0)
            assert np.all(np.abs(rt.f_rounded - f) < M)
            assert np.all(rt.kept.sum(0) == rt.f_rounded)
            if not rescue:
                assert np.all(np.abs(rt.f_rounded - f) <= M // 2)
            else:
                assert rt.kept.any(1).all()                     # every token keeps >= 1 expert
            for e in range(E):
                col_tc, col_k = tc[:, e], rt.kept[:, e]
                if rt.f_rounded[e] >= f[e]:                     # padded: kept ⊇ TC, extra = best non-TC
                    assert np.all(col_k[col_tc])
                    extra = np.nonzero(col_k & ~col_tc)[0]
                    rest = np.nonzero(~col_k & ~col_tc)[0]
                else:                                           # dropped: kept ⊆ TC, dropped = worst TC
                    assert not np.any(col_k & ~col_tc)
                    extra = np.nonzero(col_k)[0]
                    rest = np.nonzero(col_tc & ~col_k)[0]
                if len(extra) and len(rest):
                    worst_in = min(extra, key=lambda t: (S[t, e], -t))
                    best_out = max(rest, key=lambda t: (S[t, e], -t))
                    assert (S[worst_in, e], -worst_in) > (S[best_out, e], -best_out)


def test_tr_down_on_tile_multiples_is_tc():
    """when every f is already a tile multiple, TR == TC."""
    T, E, K, M = 64, 4, 2, 8
    # expert e is chosen by tokens [16e, 16e+16) first and by the next block second
    S = np.full((T, E), 0.01)
    for t in range(T):
        S[t, t // 16] = 0.9
        S[t, (t // 16 + 1) % E] = 0.5
    S /= S.sum(1, keepdims=True)
    a, b = om.route(S, K, "tc"), om.route(S, K, "tr", m_tile=M)
    assert np.array_equal(a.kept, b.kept) and np.array_equal(a.f_rounded, b.f_rounded)


# ------------------------------------------------------------------ metadata
@pytest.mark.parametrize("mode", ["tc", "tr"])
def test_metadata_is_consistent(mode):
    X, W1, W2, S, dO, rt = rand_case(5, 700, 4, 2, 12, 3, mode=mode, m_tile=128)
    E = S.shape[1]
    assert rt.offsets[0] == 0 and np.all(np.diff(rt.offsets) == rt.f_rounded)
    assert np.all(rt.pad_offsets % om.GEMM_M == 0)
    assert rt.R == rt.kept.sum() == len(rt.token_rows)
    for e in range(E):
        seg = rt.row_token[rt.pad_offsets[e]: rt.pad_offsets[e] + rt.f_rounded[e]]
        assert np.all(np.diff(seg) > 0)                                     # ascending tokens
        assert np.all(rt.row_token[rt.pad_offsets[e] + rt.f_rounded[e]: rt.pad_offsets[e + 1]] == -1)
        assert np.all(rt.row_expert[rt.pad_offsets[e]: rt.pad_offsets[e + 1]] == e)
    for t in range(S.shape[0]):                                             # CSR is the inverse map
        rows = rt.token_rows[rt.token_rowptr[t]: rt.token_rowptr[t + 1]]
        assert np.all(rt.row_token[rows] == t)
        assert np.all(np.diff(rt.row_expert[rows]) > 0)
        assert set(rt.row_expert[rows]) == set(np.nonzero(rt.kept[t])[0])
        assert rt.gate[t].sum() == pytest.approx(1.0)
    assert np.all(rt.tile_expert == rt.row_expert[:: om.GEMM_M])


# ------------------------------------------------------------------ forward
@pytest.mark.parametrize("T,d,n,E,K,mode", [
    (8, 4, 2, 4, 2, "tc"), (32, 8, 4, 8, 4, "tc"), (24, 6, 3, 5, 5, "tc"),   # K = E
    (6, 4, 2, 8, 1, "tc"),                                                   # empty experts
    (64, 8, 4, 8, 2, "tr")])
def test_forward_equals_dense_brute_force(T, d, n, E, K, mode):
    X, W1, W2, S, dO, rt = rand_case(T + E, T, d, n, E, K, mode=mode, m_tile=4)
    O = om.forward(X, W1, W2, rt).O
    Od = om.forward_dense(X, W1, W2, rt.kept, rt.gate)
    assert np.max(np.abs(O - Od)) <= 1e-13 * max(1.0, np.max(np.abs(Od)))
    if E > T:
        assert (rt.f == 0).any()


def test_forward_special_cases():
    X, W1, W2, S, dO, rt = rand_case(0, 16, 4, 2, 4, 2)
    assert np.all(om.forward(np.zeros_like(X), W1, W2, rt).O == 0)
    # E = K = 1 with gate 1: a dense SwiGLU MLP, written out element-wise
    rng = np.random.default_rng(2)
    X1, W11, W21 = rng.standard_normal((5, 3)), rng.standard_normal((1, 3, 4)), rng.standard_normal((1, 2, 3))
    rt1 = om.route(np.ones((5, 1)), 1)
    O = om.forward(X1, W11, W21, rt1).O
    for t in range(5):
        h = [sum(X1[t, k] * W11[0, k, j] for k in range(3)) for j in range(4)]
        a = [h[j] / (1 + np.exp(-h[j])) * h[2 + j] for j in range(2)]
        for c in range(3):
            assert O[t, c] == pytest.approx(sum(a[j] * W21[0, j, c] for j in range(2)), rel=1e-12)


def test_forward_permutation_equivariance():
    X, W1, W2, S, dO, rt = rand_case(4, 40, 6, 3, 6, 2)
    P = np.random.default_rng(9).permutation(40)
    rtp = om.route(S[P], 2)
    assert np.allclose(om.forward(X[P], W1, W2, rtp).O, om.forward(X, W1, W2, rt).O[P], rtol=0, atol=1e-13)


# ------------------------------------------------------------------ backward
def test_backward_finite_differences():
    """>= 20 seeds, T<=32, d<=8, n<=4, E<=8, K<=4; h=1e-5; 1e-6 rel."""
    for seed in range(20):
        rng = np.random.default_rng(100 + seed)
        T, d, n, E = int(rng.integers(4, 33)), int(rng.integers(2, 9)), int(rng.integers(1, 5)), int(rng.integers(1, 9))
        K = int(rng.integers(1, min(4, E) + 1))
        X, W1, W2, S, _, rt = rand_case(seed, T, d, n, E, K)
        G = rng.standard_normal((T, d))                          # L = sum G * O  =>  dO = G
        bw = om.backward(G, X, W1, W2, rt)

        def check(an, fd):
            for i, v in fd.items():
                ref = an.reshape(-1)[i]
                if abs(v) > 1e-8:
                    assert ref == pytest.approx(v, rel=1e-6)
                else:
                    assert abs(ref - v) < 1e-10

        pick = lambda a: rng.choice(a.size, size=min(a.size, 12), replace=False)
        check(bw.dX, om.fd_grad(lambda x: om.loss_fixed_routing(x, W1, W2, rt.kept, rt.gate, G), X, coords=pick(X)))
        check(bw.dW1, om.fd_grad(lambda w: om.loss_fixed_routing(X, w, W2, rt.kept, rt.gate, G), W1, coords=pick(W1)))
        check(bw.dW2, om.fd_grad(lambda w: om.loss_fixed_routing(X, W1, w, rt.kept, rt.gate, G), W2, coords=pick(W2)))
        # dS = dL/dg for each kept (t, e)
        gfd = om.fd_grad(lambda g: om.loss_fixed_routing(X, W1, W2, rt.kept, g, G), rt.gate)
        for e, toks in enumerate(np.nonzero(rt.kept[:, e])[0] for e in range(E)):
            for i, t in enumerate(toks):
                v = gfd[t * E + e]
                assert bw.dS[e][i] == pytest.approx(v, rel=1e-6, abs=1e-10)


def test_backward_dual_path_identity():
    """App. C: memory-efficient == Y/dY path to 1e-12, 50 seeds."""
    for seed in range(50):
        X, W1, W2, S, dO, rt = rand_case(seed, 24, 8, 4, 6, 3, mode="tc" if seed % 2 else "tr")
        a, b = om.backward(dO, X, W1, W2, rt), om.backward_reference(dO, X, W1, W2, rt)
        for name in ("dX", "dW1", "dW2"):
            assert np.max(np.abs(getattr(a, name) - getattr(b, name))) < 1e-12
        for e in a.dS:
            assert np.max(np.abs(a.dS[e] - b.dS[e]), initial=0) < 1e-12
            assert np.max(np.abs(a.dH[e] - b.dH[e]), initial=0) < 1e-12


def test_backward_zero_dO():
    X, W1, W2, S, dO, rt = rand_case(1, 16, 4, 2, 4, 2)
    bw = om.backward(np.zeros_like(dO), X, W1, W2, rt)
    assert not bw.dX.any() and not bw.dW1.any() and not bw.dW2.any()
    assert all(not v.any() for v in bw.dS.values())


def test_backward_uses_cached_H():
    X, W1, W2, S, dO, rt = rand_case(3, 32, 8, 4, 4, 2)
    fw = om.forward(X, W1, W2, rt)
    a = om.backward(dO, X, W1, W2, rt)
    b = om.backward(dO, X, W1, W2, rt, H_cache=fw.H)
    assert np.allclose(a.dW1, b.dW1, atol=1e-13)


def _lazy(W):
    """Per-expert views the way the full-size GPU tests hand weights to the oracle."""
    class Lazy:
        shape = W.shape

        def __getitem__(self, e):
            return W[int(e)].copy()
    return Lazy()


@pytest.mark.parametrize("mode", ["tc", "tr"])
def test_backward_experts_matches_full_backward(mode):
    """backward_experts (the dW1 / dW2 / dS checker of the sampled and streamed full-size GPU tests)
    equals backward (FD- and dual-path-pinned above) on every expert, including empty ones, with the
    weights passed as lazy per-expert views."""
    for seed in range(4):
        X, W1, W2, S, dO, rt = rand_case(60 + seed, 48, 8, 4, 10, 3, mode=mode, m_tile=4)
        bw = om.backward(dO, X, W1, W2, rt)
        E = W1.shape[0]
        got = om.backward_experts(dO, X, _lazy(W1), _lazy(W2), rt, range(E))
        for e in range(E):
            dW1e, dW2e, dSe = got[e]
            assert np.array_equal(dW1e, bw.dW1[e]) and np.array_equal(dW2e, bw.dW2[e])
            assert np.array_equal(dSe, bw.dS[e])
        # an independent spot check of one expert's dW2 / dW1 written out as sums over its rows
        e = int(np.argmax(rt.f_rounded))
        toks = np.nonzero(rt.kept[:, e])[0]
        dW2_sum = np.zeros_like(W2[e])
        dW1_sum = np.zeros_like(W1[e])
        for t in toks:
            g = rt.gate[t, e]
            h = X[t] @ W1[e]
            dap = W2[e] @ dO[t]                                  # dA' row = dO_t W2_e^T
            a, dh = om.dswiglu(g * dap, h)
            dW2_sum += np.outer(g * a, dO[t])
            dW1_sum += np.outer(X[t], dh)
        assert np.allclose(got[e][1], dW2_sum, rtol=0, atol=1e-12)
        assert np.allclose(got[e][0], dW1_sum, rtol=0, atol=1e-12)


@pytest.mark.parametrize("mode", ["tc", "tr"])
def test_metadata_brute_force(mode):
    """build_metadata against an independent construction: the grouped rows are the kept (expert,
    token) pairs sorted lexicographically, each expert's segment padded to a GEMM_M multiple; the
    token CSR is the same pairs sorted by (token, expert)."""
    X, W1, W2, S, dO, rt = rand_case(8, 300, 4, 2, 9, 3, mode=mode, m_tile=16)
    T, E = rt.kept.shape
    pairs = sorted((e, t) for t in range(T) for e in range(E) if rt.kept[t, e])
    row_token, row_expert, row_gate, row_of = [], [], [], {}
    for e in range(E):
        mine = [t for (ee, t) in pairs if ee == e]
        for t in mine:
            row_of[(t, e)] = len(row_token)
            row_token.append(t)
            row_expert.append(e)
            row_gate.append(rt.gate[t, e])
        while len(row_token) % om.GEMM_M:
            row_token.append(-1)
            row_expert.append(e)
            row_gate.append(0.0)
    assert rt.row_token.tolist() == row_token
    assert rt.row_expert.tolist() == row_expert
    assert rt.row_gate.tolist() == row_gate
    by_token = sorted((t, e) for (e, t) in pairs)
    assert rt.token_rows.tolist() == [row_of[p] for p in by_token]
    counts = [sum(1 for (t, _) in by_token if t == tt) for tt in range(T)]
    assert rt.token_rowptr.tolist() == [0] + np.cumsum(counts).tolist()
    assert rt.offsets.tolist() == [0] + np.cumsum([sum(1 for (e, _) in pairs if e == ee) for ee in range(E)]).tolist()
    assert rt.tile_expert.tolist() == row_expert[:: om.GEMM_M]


# ------------------------------------------------------------------ closed forms
def test_cost_spot_values():
    c = GOLD["cost"]
    assert om.model_flops(c["T"], c["d"], c["n"], c["K"]) == c["flops"]
    assert om.activation_bytes(c["T"], c["d"], c["n"], c["K"]) == c["act_bytes"]
    assert om.arithmetic_intensity(c["T"], c["d"], c["n"], c["E"], c["K"]) == pytest.approx(c["ai"], abs=0.01)
    # iso-FLOP granularity invariance of the minimal activation set
    assert om.activation_bytes(24576, 1536, 512, 4) == om.activation_bytes(24576, 1536, 256, 8)


def test_per_token_entry_points_match_full_passes():
    X, W1, W2, S, dO, rt = rand_case(11, 40, 8, 4, 6, 2)
    toks = [0, 7, 39]
    fw = om.forward(X, W1, W2, rt)
    assert np.allclose(om.forward_tokens(X, W1, W2, rt, toks), fw.O[toks], atol=1e-13)
    bw = om.backward(dO, X, W1, W2, rt)
    dXs, dSs = om.backward_tokens(dO, X, W1, W2, rt, toks)
    assert np.allclose(dXs, bw.dX[toks], atol=1e-13)
    for (t, e), v in dSs.items():
        i = list(np.nonzero(rt.kept[:, e])[0]).index(t)
        assert v == pytest.approx(bw.dS[e][i], abs=1e-13)


# ---------------------------------------------------------------- NEXT-3 rounding subroutines, EC
def test_round_up_down_golden():
    """UP / DOWN: the M-multiples above / below f, by hand."""
    f = np.array([0, 1, 63, 64, 65, 127, 128, 200])
    assert om.round_up(f, 64).tolist() == [0, 64, 64, 64, 128, 128, 128, 256]
    assert om.round_down(f, 64).tolist() == [0, 0, 0, 64, 64, 64, 128, 192]


def test_balance_hand_traced():
    """Alg. 6 traced by hand.  M=4, f=(1,1,1,1): z: -1 (|3-0|<|-1-0| no), -2 (2<2 no),
    +1 (1<3 yes), 0 (4<0 no) -> (0,0,4,0).  f=(3,3,3): up z=1; |2|<|-2| no -> down z=-2; up z=-1."""
    assert om.round_balance([1, 1, 1, 1], 4).tolist() == [0, 0, 4, 0]
    assert om.round_balance([3, 3, 3], 4).tolist() == [4, 0, 4]
    assert om.round_balance([4, 8, 0], 4).tolist() == [4, 8, 0]  # multiples are kept


@pytest.mark.parametrize("M", [4, 16, 128])
def test_balance_invariants(M):
    """Alg. 6's guarantee |sum_e f_r - sum_e f| <= M/2, each f_r one of the two
    neighbouring multiples."""
    rng = np.random.default_rng(M)
    for _ in range(200):
        f = rng.integers(0, 5 * M, size=rng.integers(1, 40))
        fr = om.round_balance(f, M)
        assert abs(int(fr.sum()) - int(f.sum())) <= M // 2
        assert np.all((fr == om.round_up(f, M)) | (fr == om.round_down(f, M)))


def test_sr_generator_is_splitmix64():
    """sr_u64(0, 0) is one SplitMix64 step from state 0: the generator's published first output
    for seed 0, 0xE220A8397B1DCDAF."""
    assert om.sr_u64(0, 0) == 0xE220A8397B1DCDAF


def test_sr_rounding_probabilities():
    """SR-f: pad with probability (f - floor f)/M; multiples never move."""
    M = 128
    f = np.array([128 + 32, 256 + 96, 384, 7])  # p = 0.25, 0.75, 0 (multiple), 7/128
    ups = np.zeros(len(f))
    n = 3000
    for seed in range(n):
        fr = om.round_sr(f, M, seed)
        assert np.all((fr == om.round_up(f, M)) | (fr == om.round_down(f, M)))
        ups += fr > f
    rate = ups / n
    assert abs(rate[0] - 0.25) < 0.03 and abs(rate[1] - 0.75) < 0.03
    assert rate[2] == 0.0 and abs(rate[3] - 7 / 128) < 0.02


def test_ec_brute_force():
    """Expert choice: every expert keeps the C highest scores (ties to the lower token), C from
    ec_capacity; brute force with Python's sort on tiny inputs, including exact ties."""
    rng = np.random.default_rng(3)
    T, E, K, M = 40, 6, 2, 4
    S = np.round(rng.random((T, E)) * 8) / 8  # quantised: exact ties
    C = om.ec_capacity(T, K, E, M)
    assert C == 16  # ceil(80/6) = 14 -> 16
    rt = om.route(S, K, mode="ec", m_tile=M)
    for e in range(E):
        want = sorted(range(T), key=lambda t: (-S[t, e], t))[:C]
        assert set(np.nonzero(rt.kept[:, e])[0].tolist()) == set(want)
    assert np.all(rt.f_rounded == C)


@pytest.mark.parametrize("rounding", ["up", "down", "balance", "sr"])
def test_tr_subroutine_route_invariants(rounding):
    """Every subroutine: f_r is a multiple of M (or T), the kept set of an expert is its TC set
    plus / minus the best / worst-ranked tokens (up: TC subset of kept; down: kept subset of TC),
    kept counts equal f_r, and the rescue leaves no orphan."""
    rng = np.random.default_rng(11)
    T, E, K, M = 200, 8, 2, 16
    S = rng.random((T, E))
    rt = om.route(S, K, mode="tr", m_tile=M, rounding=rounding, seed=5)
    tc = np.zeros((T, E), bool)
    tc[np.arange(T)[:, None], rt.topk_ids] = True
    for e in range(E):
        fr, fe = int(rt.f_rounded[e]), int(rt.f[e])
        assert fr % M == 0 or fr == T
        assert rt.kept[:, e].sum() == fr
        if fr >= fe:
            assert np.all(rt.kept[tc[:, e], e])
        else:
            assert not np.any(rt.kept[~tc[:, e], e])
    assert rt.kept.any(axis=1).all()
    if rounding == "up":
        assert np.all(rt.f_rounded == np.minimum(om.round_up(rt.f, M), T))


# ---------------------------------------------------------------- NEXT-4 router softmax
def test_softmax_closed_forms():
    """Pins of om.softmax against the mathematics: two experts reduce to the logistic sigmoid of the
    logit difference; equal logits give 1/E; rows sum to 1; adding a constant per row changes nothing;
    a large negative offset of one logit sends its probability to ~0; order is preserved."""
    rng = np.random.default_rng(3)
    a = rng.normal(size=50) * 4
    b = rng.normal(size=50) * 4
    S2 = om.softmax(np.stack([a, b], axis=1))
    np.testing.assert_allclose(S2[:, 0], 1.0 / (1.0 + np.exp(b - a)), rtol=1e-15, atol=1e-300)
    np.testing.assert_allclose(om.softmax(np.full((3, 7), 2.5)), 1.0 / 7, rtol=1e-15)
    lg = rng.normal(size=(40, 96)) * 3
    S = om.softmax(lg)
    np.testing.assert_allclose(S.sum(1), 1.0, rtol=0, atol=1e-14)
    np.testing.assert_allclose(om.softmax(lg + rng.normal(size=(40, 1)) * 50), S, rtol=1e-12)
    assert np.all(np.argsort(-S, axis=1, kind="stable")[:, :5] == np.argsort(-lg, axis=1, kind="stable")[:, :5])
    lg2 = lg.copy()
    lg2[:, 0] -= 1000.0
    assert np.all(om.softmax(lg2)[:, 0] < 1e-300)
    # a worked value: softmax([0, ln 2, ln 3]) = [1, 2, 3] / 6
    np.testing.assert_allclose(om.softmax(np.log([[1.0, 2.0, 3.0]])), [[1 / 6, 2 / 6, 3 / 6]], rtol=1e-15)


def test_router_chain_finite_differences():
    """The whole router chain -- logits = X W_r, S = softmax, gates renormalised over the frozen kept
    sets -- differentiated by router_backward then router_input_grads equals central finite
    differences of L(X, W_r) = sum_{kept (t,e)} c_te g_te, for every coordinate of X and W_r."""
    rng = np.random.default_rng(9)
    T, d, E, K = 10, 5, 6, 2
    X = rng.normal(size=(T, d))
    Wr = rng.normal(size=(d, E))
    S = om.softmax(om.router_logits(X, Wr))
    rt = om.route(S, K, mode="tc")
    c = rng.normal(size=(T, E)) * rt.kept

    def loss(Xv, Wv):
        s = om.softmax(Xv @ Wv)
        z = np.where(rt.kept, s, 0.0).sum(1, keepdims=True)
        return float((np.where(rt.kept, s / z, 0.0) * c).sum())

    dX, dW = om.router_input_grads(X, Wr, om.router_backward(S, rt, c))
    h = 1e-6
    for arr, got, which in ((X, dX, 0), (Wr, dW, 1)):
        fd = np.zeros_like(arr)
        for idx in np.ndindex(*arr.shape):
            p_, m_ = arr.copy(), arr.copy()
            p_[idx] += h
            m_[idx] -= h
            fd[idx] = ((loss(p_, Wr) - loss(m_, Wr)) if which == 0 else (loss(X, p_) - loss(X, m_))) / (2 * h)
        np.testing.assert_allclose(got, fd, rtol=1e-6, atol=1e-9)


# ---------------------------------------------------------------- NEXT-4 router backward
@pytest.mark.parametrize("gate_raw", [False, True])
@pytest.mark.parametrize("mode", ["tc", "tr"])
def test_router_backward_finite_differences(mode, gate_raw):
    """d logits from router_backward equals central finite differences of
    L(logits) = sum_{kept (t,e)} g_te(softmax(logits)) c_te with the routing (kept sets) frozen."""
    rng = np.random.default_rng(21 if gate_raw else 22)
    T, E, K, M = 12, 6, 2, 4
    logits = rng.normal(size=(T, E))
    S = np.exp(logits - logits.max(1, keepdims=True))
    S /= S.sum(1, keepdims=True)
    rt = om.route(S, K, mode=mode, m_tile=M, gate_raw=gate_raw)
    c = rng.normal(size=(T, E)) * rt.kept

    def loss(lg):
        s = np.exp(lg - lg.max(1, keepdims=True))
        s /= s.sum(1, keepdims=True)
        if gate_raw:
            g = np.where(rt.kept, s, 0.0)
        else:
            z = np.where(rt.kept, s, 0.0).sum(1, keepdims=True)
            g = np.where(rt.kept, s / np.where(z == 0, 1.0, z), 0.0)
        return float((g * c).sum())

    got = om.router_backward(S, rt, c, gate_raw=gate_raw)
    h = 1e-6
    fd = np.zeros_like(logits)
    for t in range(T):
        for j in range(E):
            lp, lm = logits.copy(), logits.copy()
            lp[t, j] += h
            lm[t, j] -= h
            fd[t, j] = (loss(lp) - loss(lm)) / (2 * h)
    np.testing.assert_allclose(got, fd, rtol=1e-6, atol=1e-8)


def test_router_backward_rows_sum_to_zero():
    """softmax Jacobian: every row of d logits sums to 0 (shifting all logits changes nothing)."""
    rng = np.random.default_rng(5)
    S = rng.random((30, 8))
    S /= S.sum(1, keepdims=True)
    rt = om.route(S, 3, mode="tc")
    d = om.router_backward(S, rt, rng.normal(size=S.shape) * rt.kept)
    np.testing.assert_allclose(d.sum(1), 0.0, atol=1e-12)


def test_nrs_probability_by_brute_force():
    """NR-s: over many seeds the pad frequency of each expert matches the probability
    computed independently with Python's sort of (not-in-TC, -S, t) -- pi_e of Alg. 4 -- and
    plain Python sums; tile multiples never move."""
    rng = np.random.default_rng(31)
    T, E, K, M = 60, 5, 2, 8
    S = rng.random((T, E))
    ids, _ = om.topk_tc(S, K)
    tc = np.zeros((T, E), bool)
    tc[np.arange(T)[:, None], ids] = True
    f = tc.sum(0)
    p_ref = []
    for e in range(E):
        pi = sorted(range(T), key=lambda t: (not tc[t, e], -S[t, e], t))
        fe = int(f[e])
        dn, up = fe // M * M, min(-(-fe // M) * M, T)
        s_tc = sum(S[t, e] for t in pi[:fe])
        s_dn = sum(S[t, e] for t in pi[:dn])
        s_up = sum(S[t, e] for t in pi[:up])
        p_ref.append(None if dn == fe else (s_tc - s_dn) / (s_up - s_dn))
    n = 3000
    ups = np.zeros(E)
    for seed in range(n):
        fr = om.round_nrs(S, tc, f, M, seed, T)
        for e in range(E):
            if p_ref[e] is None:
                assert fr[e] == f[e]
        ups += fr > f
    for e in range(E):
        if p_ref[e] is not None:
            sd = (p_ref[e] * (1 - p_ref[e]) / n) ** 0.5
            assert abs(ups[e] / n - p_ref[e]) < 4 * sd + 1e-3, (e, ups[e] / n, p_ref[e])


def test_nrs_route_invariants():
    rng = np.random.default_rng(12)
    T, E, K, M = 200, 8, 2, 16
    S = rng.random((T, E)).astype(np.float32).astype(np.float64)
    rt = om.route(S, K, mode="tr", m_tile=M, rounding="nrs", seed=9)
    assert np.all((rt.f_rounded % M == 0) | (rt.f_rounded == T))
    assert rt.kept.any(axis=1).all()
    assert np.all(rt.kept.sum(0) == rt.f_rounded)


# ---------------------------------------------------------------- NEXT-4 FP8 up-projection
def test_e4m3_round_against_the_format():
    """om.e4m3_round against torch's float8_e4m3fn cast (an independent library rounding, ties to
    even) on every finite code, every midpoint between neighbouring codes and random values; and
    saturation of finite values beyond 448 (the satfinite cvt; torch's cast has no saturation)."""
    import torch
    codes = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).float().numpy().astype(np.float64)
    fin = np.unique(codes[np.isfinite(codes)])
    np.testing.assert_array_equal(om.e4m3_round(fin), fin)
    mids = (fin[1:] + fin[:-1]) / 2
    rng = np.random.default_rng(1)
    vals = np.concatenate([mids, rng.normal(size=20000) * 30, rng.normal(size=5000) * 1e-2,
                           rng.normal(size=2000) * 1e-3])
    vals = vals[np.abs(vals) <= 448].astype(np.float32)
    ref = torch.tensor(vals).to(torch.float8_e4m3fn).float().numpy()
    np.testing.assert_array_equal(om.e4m3_round(vals), ref)
    np.testing.assert_array_equal(om.e4m3_round(np.array([449.0, 464.0, 1e6, -500.0])), [448, 448, 448, -448])
    # the grid: spacing 2^-9 below 2^-6 (subnormals), 2^(e-3) above
    assert om.e4m3_round(np.array([2.0 ** -9 * 1.4]))[0] == 2.0 ** -9
    assert om.e4m3_round(np.array([1.0 + 2.0 ** -4]))[0] == 1.0  # tie -> even (1.0 vs 1.125)


def test_quantize_e4m3_properties():
    """Per-slice scales: amax / 448 in fp32; every slice's largest |q| is exactly 448; q * scale
    is within half an e4m3 step of the input (2^-4 relative, or 2^-10 * scale in the subnormal range)."""
    rng = np.random.default_rng(2)
    M = (rng.normal(size=(64, 96)) * np.exp(rng.normal(size=(64, 1)))).astype(np.float32)
    M[5] = 0.0
    q, s = om.quantize_e4m3(M, axis=1)
    assert s[5] == 1.0 and np.all(q[5] == 0)
    nz = np.arange(64) != 5
    np.testing.assert_array_equal(np.max(np.abs(q[nz]), axis=1), 448.0)
    np.testing.assert_array_equal(s.astype(np.float32), (np.max(np.abs(M), axis=1) / np.float32(448)).astype(np.float32)
                                  * nz + (~nz))
    err = np.abs(q * s[:, None] - M)
    assert np.all(err <= 2.0 ** -4 * np.abs(M) * (1 + 1e-6) + 2.0 ** -10 * s[:, None] * (1 + 1e-6))


def test_forward_fp8_up_is_the_quantised_definition():
    """forward(fp8_up=True) equals the dense definition on the dequantised operands
    (Xq sx) (W1q sw): the scales factor out of the K sum exactly; and it stays within the
    quantisation error of the bf16 forward."""
    rng = np.random.default_rng(4)
    T, d, n, E, K = 48, 32, 16, 4, 2
    X = rng.normal(size=(T, d))
    W1 = rng.normal(size=(E, d, 2 * n)) / np.sqrt(d)
    W2 = rng.normal(size=(E, n, d)) / np.sqrt(n)
    S = rng.random((T, E))
    S /= S.sum(1, keepdims=True)
    rt = om.route(S, K, mode="tc")
    Xq, sx, W1q, sw = om.fp8_up_operands(X, W1)
    Xdq = Xq * sx[:, None]
    W1dq = W1q * sw[:, None, :]
    f8 = om.forward(X, W1, W2, rt, fp8_up=True)
    ref = om.forward(Xdq, W1dq, W2, rt)
    np.testing.assert_allclose(f8.O, ref.O, rtol=1e-12, atol=1e-12)
    full = om.forward(X, W1, W2, rt)
    assert np.linalg.norm(f8.O - full.O) / np.linalg.norm(full.O) < 0.1


def test_bf16_round_against_torch():
    """om.bf16_round against torch's bfloat16 cast (an independent library rounding, ties to even) on
    fp32 values (where torch's single fp32 -> bf16 rounding is the exact one), incl. exact ties."""
    rng = np.random.default_rng(11)
    v = (rng.normal(size=4000) * np.exp2(rng.integers(-30, 30, size=4000))).astype(np.float32)
    import torch
    ties = (np.float32(1.0) + np.float32(2.0 ** -8) * np.arange(1, 64, 2, dtype=np.float32)).astype(np.float32)
    v = np.concatenate([v, ties, -ties, np.float32([0.0, 1.0, -2.5])])
    ref = torch.tensor(v).to(torch.bfloat16).float().numpy().astype(np.float64)
    np.testing.assert_array_equal(om.bf16_round(v.astype(np.float64)), ref)


def test_backward_fp8_dxt_is_the_quantised_definition():
    """backward(fp8_dxt=True): dX~ is the definition on the dequantised operands -- dH~ = s q / sw
    (the row-quantised dH' = bf16(dH) sw, the forward's W1 column scales divided back out) and
    W1~ = W1q sw -- so the scales factor out exactly; dX stays within the quantisation error of the
    bf16 backward; dW1 / dW2 / dS are untouched."""
    rng = np.random.default_rng(5)
    T, d, n, E, K = 40, 32, 16, 4, 2
    X = rng.normal(size=(T, d))
    W1 = rng.normal(size=(E, d, 2 * n)) / np.sqrt(d)
    W2 = rng.normal(size=(E, n, d)) / np.sqrt(n)
    dO = rng.normal(size=(T, d))
    S = rng.random((T, E))
    S /= S.sum(1, keepdims=True)
    rt = om.route(S, K, mode="tc")
    full = om.backward(dO, X, W1, W2, rt)
    f8 = om.backward(dO, X, W1, W2, rt, fp8_dxt=True)
    W1q, sw = om.quantize_e4m3(W1, axis=1)
    dX_ref = np.zeros_like(full.dX)
    for e in range(E):
        toks = np.nonzero(rt.kept[:, e])[0]
        Hb = om.bf16_round(X[toks] @ W1[e])  # the dH the method stores comes from the bf16-cached H
        dHe = om.expert_backward(dO[toks], X[toks], W1[e], W2[e], rt.gate[toks, e], Hb).dH
        q, s = om.fp8_dxt_rows(dHe, sw[e])
        assert np.all(np.abs(q) <= 448) and np.all(s > 0)
        dH_dq = s[:, None] * q / sw[e][None, :]
        W1_dq = W1q[e] * sw[e][None, :]
        np.add.at(dX_ref, toks, dH_dq @ W1_dq.T)
    np.testing.assert_allclose(f8.dX, dX_ref, rtol=1e-10, atol=1e-12)
    assert np.linalg.norm(f8.dX - full.dX) / np.linalg.norm(full.dX) < 0.1
    for a, b in ((f8.dW1, full.dW1), (f8.dW2, full.dW2)):
        np.testing.assert_array_equal(a, b)
    for e in range(E):
        np.testing.assert_array_equal(f8.dS[e], full.dS[e])
