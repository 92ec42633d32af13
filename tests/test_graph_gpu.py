"""CUDA-graph capture of the library calls (the launch-bound small cases of a serving loop
are replayed from a graph): every call enqueues only stream-ordered work -- kernels,
cudaMemsetAsync -- with no host synchronisation or allocation, so it can be captured once
and replayed on new inputs.  Each replay must equal the eager call on the same inputs
bit for bit (same kernels, same order)."""
import numpy as np
import pytest
import torch

from gen import inputs as gi

pytestmark = pytest.mark.gpu
hh = pytest.importorskip("paper_1811_07624_b200")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def capture(fn):
    """Warm up (first-call attribute setup happens outside the capture), then capture."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = fn()
    torch.cuda.synchronize()
    return g, out


@pytest.mark.parametrize("algo,n,h,N", [("fused", 256, 8, 3000), ("wy", 512, 64, 2000),
                                        ("wy", 384, 300, 1500)])
@pytest.mark.parametrize("op", [0, 1])
def test_graph_apply(algo, n, h, N, op):
    g0 = gi.rng(900, n, h, op)
    U = dev(gi.unit_reflectors(g0, h, n, "f32"))
    X = dev(gi.gaussian_columns(g0, N, n, "f32"))
    Y = torch.empty_like(X)
    a = hh.HH_ALGO_FUSED if algo == "fused" else hh.HH_ALGO_WY
    wsb = hh.hh_workspace_bytes(hh.HH_CALL_APPLY, n, h, N, 0, torch.float32) if algo == "wy" else 0
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    with hh.algo(a):
        graph, _ = capture(lambda: hh.hh_apply(op, U, X, Y, workspace=ws if wsb else None))
        for rep in range(3):
            X.copy_(dev(gi.gaussian_columns(gi.rng(901, rep), N, n, "f32")))
            graph.replay()
            torch.cuda.synchronize()
            got = Y.clone()
            ref = hh.hh_apply(op, U, X, workspace=ws if wsb else None)
            torch.cuda.synchronize()
            assert torch.equal(got, ref), (algo, rep)


@pytest.mark.parametrize("n,h,N", [(1023, 10, 900), (101, 7, 3000), (1021, 40, 700), (9001, 5, 64)])
def test_graph_unaligned_strides(n, h, N):
    """Unaligned column strides under capture: K1r (TMEM and shared-memory forms), K1g, and the
    padded detour (copies + the aligned call + the copy back are all stream-ordered kernels)."""
    g0 = gi.rng(905, n, h)
    U = dev(gi.unit_reflectors(g0, h, n, "f32"))
    X = dev(gi.gaussian_columns(g0, N, n, "f32"))
    Y = torch.empty_like(X)
    wsb = hh.hh_workspace_bytes(hh.HH_CALL_APPLY, n, h, N, 0, torch.float32)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    graph, _ = capture(lambda: hh.hh_apply(0, U, X, Y, workspace=ws if wsb else None))
    for rep in range(2):
        X.copy_(dev(gi.gaussian_columns(gi.rng(906, rep), N, n, "f32")))
        graph.replay()
        torch.cuda.synchronize()
        got = Y.clone()
        ref = hh.hh_apply(0, U, X, workspace=ws if wsb else None)
        torch.cuda.synchronize()
        assert torch.equal(got, ref), (n, h, rep)


def test_graph_sym_and_mahalanobis_and_knn():
    n, h, N = 256, 32, 2000
    g0 = gi.rng(902)
    U = dev(gi.unit_reflectors(g0, h, n, "f32"))
    lam = dev(np.exp(-np.arange(n) / 50.0).astype(np.float32))
    X = dev(gi.gaussian_columns(g0, N, n, "f32"))
    Y = torch.empty_like(X)
    d = dev(gi.metric_diag(g0, n, "f32"))
    ia = dev(g0.integers(0, N, 5000).astype(np.int32))
    ib = dev(g0.integers(0, N, 5000).astype(np.int32))
    dist = torch.empty(5000, dtype=torch.float32, device="cuda")
    wss = torch.empty(max(hh.hh_workspace_bytes(hh.HH_CALL_SYM, n, h, N, 0, torch.float32), 1),
                      dtype=torch.uint8, device="cuda")
    wsm = torch.empty(hh.hh_workspace_bytes(hh.HH_CALL_MAHALANOBIS, n, h, N, 5000, torch.float32),
                      dtype=torch.uint8, device="cuda")
    Pq = dev(gi.gaussian_columns(g0, 300, n, "f32"))
    wsk = torch.empty(hh.hh_workspace_bytes(hh.HH_CALL_KNN, n, h, N, 300, torch.float32),
                      dtype=torch.uint8, device="cuda")

    def step():
        hh.hh_sym_apply(U, lam, X, Y, workspace=wss)
        hh.hh_mahalanobis(U, d, X, ia, ib, dist, workspace=wsm)
        return hh.hh_knn(U, d, X, Pq, 5, workspace=wsk)

    graph, (idx_g, dist_g) = capture(step)
    for rep in range(2):
        X.copy_(dev(gi.gaussian_columns(gi.rng(903, rep), N, n, "f32")))
        graph.replay()
        torch.cuda.synchronize()
        got = (Y.clone(), dist.clone(), idx_g.clone(), dist_g.clone())
        Y2 = hh.hh_sym_apply(U, lam, X, workspace=wss)
        dist2 = hh.hh_mahalanobis(U, d, X, ia, ib, workspace=wsm)
        idx2, dk2 = hh.hh_knn(U, d, X, Pq, 5, workspace=wsk)
        torch.cuda.synchronize()
        assert torch.equal(got[0], Y2) and torch.equal(got[1], dist2)
        assert torch.equal(got[2], idx2) and torch.equal(got[3], dk2)
