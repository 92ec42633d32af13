"""GPU parity of NEXT-f3, test-time k-NN under the learned metric.

Several answers are correct when two references are (nearly) equidistant, so the test
compares what is unique and checks that the rest is valid (reading R14):
  * each returned distance equals the oracle's exact d_S of the returned pair, and
  * the exact distances of the returned set match the oracle's sorted k smallest,
both within the fp32 gate 2e-5*sqrt(h) relative to ||z_q||^2 + ||z_r||^2 (the terms of
the expansion ||z_q||^2 + ||z_r||^2 - 2 z_q.z_r the tensor cores evaluate); and the
indices agree exactly except at such near-ties.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gi

pytestmark = pytest.mark.gpu
hh = pytest.importorskip("paper_1811_07624_b200")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def knn_case(n, h, Mr, Mq, seed):
    g = gi.rng(400, seed, n, h)
    U = gi.unit_reflectors(g, h, n, "f32")
    d = gi.metric_diag(g, n, "f32")
    Pr = gi.gaussian_columns(g, Mr, n, "f32")
    Pq = gi.gaussian_columns(g, Mq, n, "f32")
    Pq[:3] = Pr[[5, 77 % Mr, Mr - 1]]          # exact duplicates: distance 0 must rank first
    return U, d, Pr, Pq


def sq_norms(U, d, P):
    """||L x||^2 = d_S(x, 0) by the oracle (the literal per-pair form against 0)."""
    Z = np.vstack([P.astype(np.float64), np.zeros((1, P.shape[1]))])
    ia = np.arange(P.shape[0], dtype=np.int32)
    ib = np.full(P.shape[0], P.shape[0], dtype=np.int32)
    return oracle.mahalanobis(U, d, Z, ia, ib)


@pytest.mark.parametrize("n,h,Mr,Mq,k", [(40, 6, 2000, 300, 3), (100, 7, 1500, 200, 5),
                                         (200, 24, 1000, 130, 16), (64, 0, 700, 129, 1),
                                         (256, 9, 513, 257, 8),
                                         # rows not 16-byte strided: the transform runs on K1g
                                         (41, 6, 900, 150, 3), (30, 5, 600, 100, 4),
                                         (255, 8, 400, 70, 2), (3, 2, 300, 40, 5)])
def test_knn_parity(n, h, Mr, Mq, k):
    U, d, Pr, Pq = knn_case(n, h, Mr, Mq, seed=1)
    idx, dist = hh.hh_knn(dev(U) if h else torch.empty(0, n, device="cuda"), dev(d), dev(Pr),
                          dev(Pq), k)
    torch.cuda.synchronize()
    assert hh.last_launch_info()["variant"].startswith("knn_")
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy().astype(np.float64)
    ridx, rdist = oracle.knn(U, d, Pr, Pq, k)
    nq, nr = sq_norms(U, d, Pq), sq_norms(U, d, Pr)
    gate = 2e-5 * math.sqrt(max(h, 1))
    assert np.all((idx >= 0) & (idx < Mr))
    for q in range(Mq):
        assert len(set(idx[q].tolist())) == k
        # exact d_S of the returned pairs (oracle, literal per-pair form)
        true = oracle.mahalanobis(U, d, np.vstack([Pr, Pq[q:q + 1]]).astype(np.float64),
                                  idx[q].astype(np.int32), np.full(k, Mr, dtype=np.int32))
        scale = nq[q] + nr[idx[q]]
        assert np.all(np.abs(dist[q] - true) <= gate * scale), (q, dist[q], true)
        assert np.all(np.abs(np.sort(true) - rdist[q]) <= gate * (nq[q] + nr.max())), q
    assert np.mean(idx == ridx) > 0.99
    for q, r in enumerate([5, 77 % Mr, Mr - 1]):
        assert idx[q, 0] == r and abs(dist[q, 0]) <= gate * 2 * nq[q]


def test_knn_paper_shape_sampled():
    """A Table-I-shaped synthetic stand-in (MNIST after PCA: n = 40, h = ceil(log2 n) = 6,
    70/30 split of 70000 points) at full size; the oracle checks 200 sampled queries."""
    n, h, Mr, Mq, k = 40, 6, 49000, 21000, 3
    U, d, Pr, Pq = knn_case(n, h, Mr, Mq, seed=2)
    idx, dist = hh.hh_knn(dev(U), dev(d), dev(Pr), dev(Pq), k)
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy().astype(np.float64)
    sel = np.unique(np.concatenate([gi.rng(401).integers(0, Mq, 197), [0, 1, 2, Mq - 1]]))
    ridx, rdist = oracle.knn(U, d, Pr, Pq[sel], k)
    assert np.mean(idx[sel] == ridx) > 0.99
    gate = 2e-5 * math.sqrt(h)
    nq = sq_norms(U, d, Pq[sel])
    nr_max = sq_norms(U, d, Pr).max()
    assert np.all(np.abs(dist[sel] - rdist) <= gate * (nq[:, None] + nr_max))


def test_knn_errors():
    L = hh.hh.lib()
    P = torch.randn(40, 300, device="cuda")
    ok = torch.ones(300, device="cuda")
    i = torch.empty(10, 3, dtype=torch.int32, device="cuda")
    o = torch.empty(10, 3, device="cuda")
    ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    args = lambda n, k, M=40: (n, 0, None, hh.hh._ptr(ok), hh.hh._ptr(P), M, hh.hh._ptr(P), 10, k,  # noqa: E731
                               hh.hh._ptr(i), hh.hh._ptr(o), 0, hh.hh._ptr(ws), ws.numel(), None)
    assert L.hh_knn(*args(300, 3)) == hh.hh.HH_ERR_UNSUPPORTED     # n > 256
    assert L.hh_knn(*args(64, 17)) == hh.hh.HH_ERR_UNSUPPORTED     # k > 16
    assert L.hh_knn(*args(64, 3, M=2)) == hh.hh.HH_ERR_INVALID_VALUE   # M_ref < k


@pytest.mark.parametrize("k", [2, 3, 5])
def test_knn_exact_ties(k):
    """Reading R14 / hh.h "ties by the smaller reference index": duplicated references give
    bit-identical transformed points and distances on the GPU too (same bytes, same
    arithmetic), so the returned indices are unique and must equal the oracle's exactly.
    The duplicates sit in different 256-reference tiles and in different reference splits
    (the CTA range cut and the merge kernel), at the k-th place and inside the list."""
    n, h, Mr, Mq = 40, 6, 6000, 64
    U, d, Pr, _ = knn_case(n, h, Mr, 4, seed=3)
    groups = [(10, 700, 2999, 5990), (5, 300), (4000, 4001, 255, 256)]
    for grp in groups:
        for r in grp[1:]:
            Pr[r] = Pr[grp[0]]
    g = gi.rng(402, k)
    Pq = np.empty((Mq, n), dtype=np.float32)
    for q in range(Mq):
        base = groups[q % len(groups)][0]
        Pq[q] = Pr[base] + (0.0 if q < 3 else 1e-3) * g.standard_normal(n).astype(np.float32)
    idx, dist = hh.hh_knn(dev(U), dev(d), dev(Pr), dev(Pq), k)
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
    ridx, _ = oracle.knn(U, d, Pr, Pq, k)
    assert np.array_equal(idx, ridx), np.nonzero((idx != ridx).any(1))[0][:5]
    for q in range(Mq):
        grp = sorted(groups[q % len(groups)])
        m = min(k, len(grp))
        assert list(idx[q, :m]) == grp[:m]              # the tie group, ascending index
        assert np.all(dist[q, :m] == dist[q, 0])        # bit-identical distances
