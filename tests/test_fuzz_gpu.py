"""Randomised GPU parity sweep (seeded): random shapes across every kernel path, both
dtypes where supported, against the oracle -- plus concurrent launches of the
tensor-core paths on two streams (TMEM allocation under contention)."""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gi
from tests._util import assert_parity

pytestmark = pytest.mark.gpu
hh = pytest.importorskip("paper_1811_07624_b200")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def shapes(seed, count):
    g = gi.rng(800, seed)
    out = []
    for _ in range(count):
        n = int(g.integers(1, 96)) * 4 * int(g.choice([1, 1, 2, 4, 8]))
        h = int(g.integers(0, min(n, 300)))
        N = int(g.integers(1, 700))
        out.append((n, h, N))
    return out


@pytest.mark.parametrize("n,h,N", shapes(1, 24))
@pytest.mark.parametrize("algo", ["auto", "fused"])
def test_fuzz_apply(n, h, N, algo):
    a = hh.HH_ALGO_AUTO if algo == "auto" else hh.HH_ALGO_FUSED
    for dt in ("f32", "f64"):
        if dt == "f64" and n % 2:
            continue
        c = gi.make_case("apply", n, h, N, dt, seed=n + h)
        op = (n + h + N) % 2
        with hh.algo(a):
            got = hh.hh_apply(op, dev(c.U) if h else torch.empty(0, n, device="cuda",
                                                                 dtype=torch.float32 if dt == "f32"
                                                                 else torch.float64),
                              dev(c.X)).cpu().numpy()
        assert_parity(got, oracle.apply(op, c.U, c.X), dt, h, f"fuzz apply n{n} h{h} N{N} {dt}")


def any_shapes(seed, count):
    """Arbitrary n (mostly not a multiple of 4: K1g), a few past the vector kernels' n."""
    g = gi.rng(810, seed)
    out = []
    for _ in range(count):
        n = int(g.integers(1, 3000)) if g.random() < 0.8 else int(g.integers(8193, 30000))
        h = int(g.integers(0, 24))
        N = int(g.integers(1, 200 if n < 3000 else 20))
        out.append((n, h, N))
    return out


@pytest.mark.parametrize("n,h,N", any_shapes(1, 20))
def test_fuzz_any_n(n, h, N):
    """Every n: the apply (both ops), the symmetric form and the per-pair distance, fp32 and
    fp64, whichever kernel the library picks (K1g unless the shape happens to fit K1)."""
    for dt, tdt in (("f32", torch.float32), ("f64", torch.float64)):
        if dt == "f64" and n > 25000:
            continue
        c = gi.make_case("sym", n, h, N, dt, seed=n + 3 * h)
        U = dev(c.U) if h else torch.empty(0, n, device="cuda", dtype=tdt)
        for op in (0, 1):
            got = hh.hh_apply(op, U, dev(c.X)).cpu().numpy()
            assert_parity(got, oracle.apply(op, c.U, c.X), dt, h, f"any-n apply n{n} h{h} op{op} {dt}")
        got = hh.hh_sym_apply(U, dev(c.lam), dev(c.X)).cpu().numpy()
        assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), dt, h, f"any-n sym n{n} h{h} {dt}")
        m = gi.make_case("mahalanobis", n, h, max(N, 2), dt, seed=n, npairs=3 * N + 5)
        got = hh.hh_mahalanobis(dev(m.U) if h else torch.empty(0, n, device="cuda", dtype=tdt),
                                dev(m.d), dev(m.X), dev(m.ia), dev(m.ib)).cpu().numpy()
        assert_parity(got, oracle.mahalanobis(m.U, m.d, m.X, m.ia, m.ib), dt, h,
                      f"any-n pairs n{n} h{h} {dt}")


def test_fuzz_unaligned_offsets():
    """A seeded subset of tools/stress_unaligned.py: random n / h / N / dtype / op, operands at
    random element offsets from a 16-byte boundary, in place or not, apply / sym / D, with each
    of K1r's forms, K1g and the padded detour forced in turn -- all against the oracle."""
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools",
                        "stress_unaligned.py")
    spec = importlib.util.spec_from_file_location("stress_unaligned", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    g = gi.rng(990, 77)
    fails = []
    for i in range(120):
        ok, msg = mod.one_case(g, i)
        if not ok:
            fails.append(msg)
    assert not fails, fails


@pytest.mark.parametrize("n,h,N", shapes(2, 12))
def test_fuzz_sym_and_signed(n, h, N):
    h = max(h, 1)
    c = gi.make_case("sym", n, h, N, "f32", seed=h)
    d = gi.sign_diag(gi.rng(801, n), n, "f32")
    got = hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X)).cpu().numpy()
    assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), "f32", h, f"fuzz sym n{n} h{h}")
    got = hh.hh_apply_signed(1, hh.HH_SIDE_LEFT, dev(c.U), dev(d), dev(c.X)).cpu().numpy()
    assert_parity(got, oracle.apply_signed(1, 0, c.U, d, c.X), "f32", h, f"fuzz signed n{n} h{h}")


@pytest.mark.parametrize("n,h,M", [(s[0], s[1] % 40, s[2]) for s in shapes(3, 10)])
def test_fuzz_mahalanobis(n, h, M):
    c = gi.make_case("mahalanobis", n, h, max(M, 2), "f32", seed=M, npairs=int(3 * M + 17))
    for fused in (False, True):
        got = hh.hh_mahalanobis(dev(c.U) if h else torch.empty(0, n, device="cuda"), dev(c.d),
                                dev(c.X), dev(c.ia), dev(c.ib), fused=fused).cpu().numpy()
        assert_parity(got, oracle.mahalanobis(c.U, c.d, c.X, c.ia, c.ib), "f32", h,
                      f"fuzz maha n{n} h{h} fused={fused}")


def test_concurrent_streams_tensor_paths():
    """Two streams running the compact-WY apply and the k-NN kernel concurrently (both
    allocate TMEM): results equal the serial ones."""
    c = gi.make_case("apply", 1024, 200, 3000, "f32", seed=5)
    U, X = dev(c.U), dev(c.X)
    ref_apply = hh.hh_apply(0, U, X).clone()
    Pr, Pq = torch.randn(3000, 64, device="cuda"), torch.randn(500, 64, device="cuda")
    Uk, dk = torch.nn.functional.normalize(torch.randn(6, 64, device="cuda"), dim=1), \
        torch.rand(64, device="cuda") + 0.1
    ref_idx, ref_d = hh.hh_knn(Uk, dk, Pr, Pq, 4)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            y = hh.hh_apply(0, U, X)
        with torch.cuda.stream(s2):
            r = hh.hh_knn(Uk, dk, Pr, Pq, 4)
        outs.append((y, r))
    torch.cuda.synchronize()
    for y, (i, d) in outs:
        assert torch.equal(y, ref_apply)
        assert torch.equal(i, ref_idx) and torch.equal(d, ref_d)


def k1w_shapes(seed, count):
    g = gi.rng(810, seed)
    out = []
    for _ in range(count):
        n = int(g.integers(257, 1025)) * 4        # (1024, 4096]: multi-warp column groups
        h = int(g.integers(1, 17))                 # the reflectors fit the TMEM columns
        N = int(g.integers(1, 900))
        out.append((n, h, N))
    return out


@pytest.mark.parametrize("n,h,N", k1w_shapes(1, 10))
def test_fuzz_k1_tmem_blocked(n, h, N):
    """K1t in blocks of four reflectors (K1w, forced) on random multi-warp shapes: both ops and
    the symmetric form, ragged h (blocks shorter than four) and N."""
    L = hh.hh.lib()
    prev = (L.hh_debug_k1_stream(0), L.hh_debug_k1_tmem(1), L.hh_debug_k1_blocked(1))
    try:
        c = gi.make_case("sym", n, h, N, "f32", seed=n + h)
        for op in (0, 1):
            with hh.algo(hh.HH_ALGO_FUSED):
                got = hh.hh_apply(op, dev(c.U), dev(c.X)).cpu().numpy()
                assert hh.last_launch_info()["variant"].endswith("_kb4")
            assert_parity(got, oracle.apply(op, c.U, c.X), "f32", h, f"fuzz K1w n{n} h{h} N{N} op{op}")
        with hh.algo(hh.HH_ALGO_FUSED):
            got = hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X)).cpu().numpy()
        assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), "f32", 2 * h, f"fuzz K1w sym n{n} h{h}")
    finally:
        L.hh_debug_k1_blocked(prev[2])
        L.hh_debug_k1_tmem(prev[1])
        L.hh_debug_k1_stream(prev[0])


@pytest.mark.parametrize("seed", range(6))
def test_fuzz_shf_cost(seed):
    """The SHF objective and its gradient (K8) on random shapes and both dtypes against the
    oracle, per candidate (reading R21)."""
    g = gi.rng(820, seed)
    n, K = int(g.integers(1, 700)), int(g.integers(1, 150))
    for dt, tol in ((np.float32, 1e-6), (np.float64, 1e-13)):
        A = g.standard_normal((n, n))
        B = g.standard_normal((n, n))
        A, B = ((A + A.T) / 2).astype(dt), ((B + B.T) / 2).astype(dt)
        U = g.standard_normal((K, n)).astype(dt)
        cost, grad = hh.hh_shf_cost(dev(A), dev(B), dev(U))
        c_ref, g_ref = oracle.shf_cost(A, B, U)
        A64, B64, U64 = (x.astype(np.float64) for x in (A, B, U))
        a, b = U64 @ A64, U64 @ B64
        al, be = np.sum(U64 * a, 1), np.sum(U64 * b, 1)
        na, nb = np.linalg.norm(a, axis=1), np.linalg.norm(b, axis=1)
        t = tol * np.sqrt(n)
        assert np.all(np.abs(cost.cpu().numpy() - c_ref) <= t * (2 * na * nb + 2 * np.abs(al * be)))
        sg = 2 * (np.linalg.norm(A64) * nb + np.linalg.norm(B64) * na) + 4 * (np.abs(al) * nb + np.abs(be) * na)
        assert np.all(np.linalg.norm(grad.cpu().numpy() - g_ref, axis=1) <= t * sg)
