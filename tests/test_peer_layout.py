"""Host logic of the peer-memory exchange (ep.PeerComm, no GPU): the block offsets computed from the
count matrix M[s][g] (rows source s sends to destination g) must
  * dispatch: tile each destination's receive area exactly, sources in ascending rank order (the
    layout an all-to-all-v produces), with no overlap;
  * return: put each received block back at the rows of the source's own send order, again tiling
    the source's return area exactly."""
import random

from paper_2512_14080_b200.ep import PeerComm


def _comm(M):
    c = PeerComm.__new__(PeerComm)  # the offset logic needs only G and M (no regions, no GPU)
    c.G, c.M = len(M), M
    return c


def _check(M):
    G = len(M)
    c = _comm(M)
    # dispatch: rank s's block for g lands at rows [dst0[g], dst0[g] + M[s][g]) of g's area
    for g in range(G):
        spans = sorted((c._dispatch_rows(s)[g], c._dispatch_rows(s)[g] + M[s][g], s) for s in range(G))
        pos = 0
        for a, b, s in spans:
            if a == b:
                continue
            assert a == pos, (M, g, spans)
            pos = b
        assert pos == sum(M[s][g] for s in range(G))
        # ascending source order
        starts = [c._dispatch_rows(s)[g] for s in range(G)]
        assert starts == sorted(starts)
    # return: destination g's block from source s (rows [src0[s], +cnt[s]) of g's received rows)
    # goes to rows [dst0[s], ...) of s's area = s's send-order block for g
    for g in range(G):
        src0, cnt, dst0 = c._return_rows(g)
        recv_start = 0
        for s in range(G):
            assert cnt[s] == M[s][g]
            assert src0[s] == recv_start  # received rows are source-major
            recv_start += M[s][g]
            assert dst0[s] == sum(M[s][:g])  # s's send offsets for destination g
    for s in range(G):
        spans = sorted((c._return_rows(g)[2][s], c._return_rows(g)[2][s] + M[s][g]) for g in range(G))
        pos = 0
        for a, b in spans:
            if a == b:
                continue
            assert a == pos
            pos = b
        assert pos == sum(M[s])


def test_peer_offsets_small():
    _check([[3, 1], [0, 2]])
    _check([[0, 0], [0, 0]])
    _check([[5]])


def test_peer_offsets_random():
    rnd = random.Random(3)
    for _ in range(200):
        G = rnd.choice([1, 2, 3, 4, 8])
        M = [[rnd.choice([0, rnd.randint(0, 50)]) for _ in range(G)] for _ in range(G)]
        _check(M)
