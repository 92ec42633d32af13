"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by element.
(The BASELINE configs at full size, every output element: tests/test_fullsize_gpu.py.)

Gates (BASELINE.json north_star): whole-output relative Frobenius error <= 1e-12
(fp64) and <= 2e-5*sqrt(h) (fp32); no non-finite output.  Inputs come from
gen/inputs.py (seeded); the oracle never sees anything produced by the GPU.
"""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gi
from tests._util import assert_parity, gate, rel_fro

pytestmark = pytest.mark.gpu

hh = pytest.importorskip("paper_1811_07624_b200")
TDT = {"f32": torch.float32, "f64": torch.float64}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_apply(op, U, X, Y=None):
    out = hh.hh_apply(op, dev(U), dev(X), Y)
    torch.cuda.synchronize()
    return out.cpu().numpy()


# ------------------------------------------------------------------ BASELINE configs
@pytest.mark.parametrize("op", [0, 1])
def test_C1_fp64_full(op):
    """configs[0]: fp64 n=64 h=6 N=4096, whole output vs oracle (and oracle vs dense)."""
    c = gi.make_config(1)
    got = run_apply(op, c.U, c.X)
    ref = oracle.apply(op, c.U, c.X)
    assert_parity(got, ref, "f64", c.h, f"C1 op{op}")


@pytest.mark.parametrize("op", [0, 1])
def test_C2_small(op):
    """configs[1] shapes at oracle size: n=1024 h=10, 3000 columns (ragged last tile)."""
    c = gi.make_config(2, N=3001)
    got = run_apply(op, c.U, c.X)
    assert_parity(got, oracle.apply(op, c.U, c.X), "f32", c.h, f"C2 op{op}")


def test_C3_sym_small():
    """configs[2] shapes: fp32 sym n=2048 h=32, 1500 columns (U 256 KiB -> chunked)."""
    c = gi.make_config(3, N=1500)
    with hh.algo(hh.HH_ALGO_FUSED):            # the SIMT K2 kernel with U streamed in chunks
        got = hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X)).cpu().numpy()
        info = hh.last_launch_info()
    assert info["nchunks"] > 1, info
    assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), "f32", c.h, "C3")


@pytest.mark.parametrize("fused", [False, True])
def test_C4_mahalanobis_small(fused):
    """configs[3] shapes: n=512 h=9, 4096 points, 50000 pairs (+ forced a == b pairs)."""
    c = gi.make_config(4, N=4096, npairs=50000)
    c.ia[:64] = c.ib[:64]
    got = hh.hh_mahalanobis(dev(c.U), dev(c.d), dev(c.X), dev(c.ia), dev(c.ib),
                            fused=fused).cpu().numpy()
    ref = oracle.mahalanobis(c.U, c.d, c.X, c.ia, c.ib)
    assert_parity(got, ref, "f32", c.h, f"C4 fused={fused}")
    assert np.all(got[:64] == 0.0)


@pytest.mark.parametrize("h", gi.C5_H)
@pytest.mark.parametrize("path", ["auto", "fused"])
def test_C5_sweep(h, path):
    """configs[4]: n=4096, h in {12, 64, 256, 1024}; oracle-sized column counts.  `auto`
    takes the crossover (compact-WY tensor-core path for large h), `fused` forces K1."""
    N = {12: 777, 64: 515, 256: 260, 1024: 130}[h]
    c = gi.make_config(5, h=h, N=N)
    with hh.algo(hh.HH_ALGO_AUTO if path == "auto" else hh.HH_ALGO_FUSED):
        got = run_apply(0, c.U, c.X)
    assert_parity(got, oracle.apply(0, c.U, c.X), "f32", h, f"C5 h={h} {path}")


# ------------------------------------------------------------------ shapes / edges
SHAPES = [  # (n, h, N, dtype) spanning every variant, full and ragged chunk counts
    (4, 3, 37, "f32"), (8, 1, 5, "f32"), (64, 6, 1000, "f32"), (100, 7, 2339, "f32"),
    (40, 6, 1031, "f32"), (200, 24, 777, "f32"), (256, 9, 513, "f32"), (384, 17, 300, "f32"),
    (512, 9, 1000, "f32"), (1000, 12, 250, "f32"), (2048, 20, 130, "f32"),
    (3000, 5, 64, "f32"), (4096, 12, 70, "f32"), (8192, 4, 20, "f32"), (6000, 40, 9, "f32"),
    (2, 1, 17, "f64"), (64, 6, 333, "f64"), (100, 10, 100, "f64"), (256, 16, 99, "f64"),
    (510, 8, 50, "f64"), (1024, 11, 40, "f64"), (2048, 6, 20, "f64"), (4096, 3, 9, "f64"),
    # 512-thread variants (n in (512, 8192] fp32, (512, 4096] fp64) over several batches per
    # unit, ragged n, and the chunked-U ring (n = 8192, h = 9: U does not fit next to X)
    (1536, 13, 1001, "f32"), (5000, 9, 301, "f32"), (8192, 9, 150, "f32"), (1024, 21, 2000, "f32"),
    (3000, 7, 517, "f64"), (4096, 5, 200, "f64"),
]


@pytest.mark.parametrize("n,h,N,dt", SHAPES)
def test_apply_shapes(n, h, N, dt):
    c = gi.make_case("apply", n, h, N, dt, seed=1)
    for op in (0, 1):
        got = run_apply(op, c.U, c.X)
        assert_parity(got, oracle.apply(op, c.U, c.X), dt, h, f"{c.name} op{op}")


@pytest.mark.parametrize("n,h,N,dt", SHAPES[::2])
def test_sym_shapes(n, h, N, dt):
    c = gi.make_case("sym", n, h, N, dt, seed=2)
    got = hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X)).cpu().numpy()
    assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), dt, h, c.name)


@pytest.mark.parametrize("n,h,M,dt", [(64, 6, 100, "f32"), (512, 9, 300, "f32"),
                                      (100, 7, 50, "f32"), (2048, 11, 40, "f32"),
                                      (4096, 4, 17, "f32"), (64, 5, 90, "f64"),
                                      (1024, 3, 33, "f64")])
@pytest.mark.parametrize("fused", [False, True])
def test_mahalanobis_shapes(n, h, M, dt, fused):
    c = gi.make_case("mahalanobis", n, h, M, dt, seed=3, npairs=1001)
    got = hh.hh_mahalanobis(dev(c.U), dev(c.d), dev(c.X), dev(c.ia), dev(c.ib),
                            fused=fused).cpu().numpy()
    assert_parity(got, oracle.mahalanobis(c.U, c.d, c.X, c.ia, c.ib), dt, h, c.name)


def test_h_zero_and_zero_slots():
    """h = 0: apply -> X exactly, sym -> lambda * X, Mahalanobis -> sum d diff^2;
    u = 0 slots are identities."""
    c = gi.make_case("sym", 256, 0, 100, "f32", seed=4)
    X = dev(c.X)
    assert torch.equal(hh.hh_apply(0, torch.empty(0, 256, device="cuda"), X), X)
    lam = dev(c.lam)
    assert torch.equal(hh.hh_sym_apply(torch.empty(0, 256, device="cuda"), lam, X), X * lam)
    z = gi.make_case("apply", 256, 9, 100, "f32", seed=5, zero_slots=(0, 4, 8))
    got = run_apply(0, z.U, z.X)
    assert_parity(got, oracle.apply(0, z.U, z.X), "f32", 9, "zero slots")
    keep = [1, 2, 3, 5, 6, 7]
    assert rel_fro(got, run_apply(0, z.U[keep], z.X)) < 1e-6


def test_N_zero_one_and_alias():
    c = gi.make_case("apply", 1024, 10, 1, "f32", seed=6)
    U = dev(c.U)
    Y = hh.hh_apply(0, U, torch.empty(0, 1024, device="cuda"))
    assert Y.shape == (0, 1024)
    got = run_apply(1, c.U, c.X)
    assert_parity(got, oracle.apply(1, c.U, c.X), "f32", 10, "N=1")
    c = gi.make_case("apply", 1024, 10, 999, "f32", seed=7)
    U, X = dev(c.U), dev(c.X)
    out = hh.hh_apply(0, U, X, Y=X)        # exact alias Y == X
    torch.cuda.synchronize()
    assert out.data_ptr() == X.data_ptr()
    assert_parity(X.cpu().numpy(), oracle.apply(0, c.U, c.X), "f32", 10, "alias")


def test_round_trip_and_norm():
    """Q^T (Q X) = X and ||Q x|| = ||x|| on the GPU (fp64, fp64-normalised u)."""
    c = gi.make_case("apply", 512, 30, 400, "f64", seed=8)
    U, X = dev(c.U), dev(c.X)
    Y = hh.hh_apply(0, U, X)
    Z = hh.hh_apply(1, U, Y)
    assert rel_fro(Z.cpu().numpy(), c.X) < 1e-13
    nr = (Y.norm(dim=1) / X.norm(dim=1) - 1).abs().max().item()
    assert nr < 1e-13


def test_forced_chunking_matches_resident():
    """A large h forces the chunked-U schedule; results must still match the oracle."""
    c = gi.make_case("apply", 1024, 200, 600, "f32", seed=9)   # U = 800 KiB
    for op in (0, 1):
        with hh.algo(hh.HH_ALGO_FUSED):
            got = run_apply(op, c.U, c.X)
            assert hh.last_launch_info()["nchunks"] > 1
        assert_parity(got, oracle.apply(op, c.U, c.X), "f32", 200, f"chunked op{op}")


def test_errors_write_nothing():
    X = torch.randn(10, 1024, device="cuda")
    Y = torch.full_like(X, 7.0)
    U = torch.randn(3, 1024, device="cuda")
    st = hh.hh.lib().hh_apply(0, 1024, 3, hh.hh._ptr(U), X.data_ptr() + 2, Y.data_ptr(), 2, 0,
                              None, 0, None)       # X not aligned to its element
    assert st == hh.hh.HH_ERR_UNSUPPORTED
    torch.cuda.synchronize()
    assert torch.all(Y == 7.0)
    with pytest.raises(ValueError):
        hh.hh_apply(0, U.cpu(), X.cpu())           # CPU tensors: no fallback
    Xo = torch.randn(10, 1023, device="cuda", dtype=torch.float64)
    with pytest.raises(hh.HHError), hh.algo(hh.HH_ALGO_WY):
        hh.hh_apply(0, torch.randn(40, 1023, device="cuda", dtype=torch.float64), Xo)  # forced WY, fp64
    P = torch.randn(10, 64, device="cuda")
    ia = torch.zeros(5, dtype=torch.int32, device="cuda")
    # the binding re-allocates a too-small workspace, so call the ABI directly
    st =hh.hh.lib().hh_mahalanobis(64, 2, hh.hh._ptr(torch.randn(2, 64, device="cuda")),
                                    hh.hh._ptr(torch.ones(64, device="cuda")), hh.hh._ptr(P), 10,
                                    hh.hh._ptr(ia), hh.hh._ptr(ia), 5,
                                    hh.hh._ptr(torch.empty(5, device="cuda")), 0,
                                    hh.hh._ptr(torch.empty(16, dtype=torch.uint8, device="cuda")),
                                    16, None)
    assert st == hh.hh.HH_ERR_WORKSPACE


def test_apply_host_e2e():
    """hh_apply_host: host buffers in, host buffers out, chunked H2D/compute/D2H ring."""
    c = gi.make_config(2, N=40000)
    X = torch.from_numpy(c.X).pin_memory()
    U = torch.from_numpy(c.U)
    for op in (0, 1):
        Y = hh.hh_apply_host(op, U, X)
        assert_parity(Y.numpy(), oracle.apply(op, c.U, c.X[:]), "f32", c.h, f"host op{op}")


def test_streams_are_respected():
    """Work is queued on the given stream: a side stream result equals the default one."""
    c = gi.make_case("apply", 1024, 10, 5000, "f32", seed=10)
    U, X = dev(c.U), dev(c.X)
    ref = hh.hh_apply(0, U, X)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        out = hh.hh_apply(0, U, X)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    assert gate("f32", 10) > 0


def test_binding_validates_operands():
    """hh.py checks every operand against X before calling libhh.so: shapes,
    dtypes, devices and contiguity; a wrong Y or vector never reaches the kernels."""
    X = torch.randn(10, 64, device="cuda")
    U = torch.randn(3, 64, device="cuda")
    lam = torch.ones(64, device="cuda")
    bad = [
        lambda: hh.hh_apply(0, U, X, Y=torch.empty(9, 64, device="cuda")),      # Y rows
        lambda: hh.hh_apply(0, U, X, Y=torch.empty(10, 64, device="cuda", dtype=torch.float64)),
        lambda: hh.hh_apply(0, U.double(), X),                                  # U dtype
        lambda: hh.hh_apply(0, torch.randn(3, 32, device="cuda"), X),           # U width
        lambda: hh.hh_apply(0, U, X.t()),                                       # not contiguous
        lambda: hh.hh_apply(0, U.cpu(), X),                                     # U on the host
        lambda: hh.hh_sym_apply(U, torch.ones(63, device="cuda"), X),           # lambda length
        lambda: hh.hh_sym_apply(U, lam.double(), X),                            # lambda dtype
        lambda: hh.hh_apply_signed(0, 0, U, lam.cpu(), X),                      # d on the host
        lambda: hh.hh_mahalanobis(U, lam, X, torch.zeros(4, dtype=torch.int32, device="cuda"),
                                  torch.zeros(5, dtype=torch.int32, device="cuda")),
        lambda: hh.hh_mahalanobis(U, lam, X, torch.zeros(4, dtype=torch.int64, device="cuda"),
                                  torch.zeros(4, dtype=torch.int64, device="cuda")),
        lambda: hh.hh_mahalanobis(U, lam, X, torch.zeros(4, dtype=torch.int32, device="cuda"),
                                  torch.zeros(4, dtype=torch.int32, device="cuda"),
                                  dist=torch.empty(3, device="cuda")),
        lambda: hh.hh_congruence(0, U, torch.randn(2, 64, 64, device="cuda"),
                                 out=torch.empty(2, 64, 63, device="cuda")),
        lambda: hh.hh_knn(U, lam, X, torch.randn(5, 60, device="cuda"), 2),
        lambda: hh.hh_apply_host(0, U.cpu(), X.cpu(), Y=torch.empty(10, 32)),
    ]
    for i, f in enumerate(bad):
        with pytest.raises(ValueError):
            f()
            pytest.fail(f"case {i} accepted")
    # the valid calls still work, and nothing above launched anything
    assert_parity(hh.hh_apply(0, U, X).cpu().numpy(), oracle.apply(0, U.cpu().numpy(),
                                                                     X.cpu().numpy()),
                  "f32", 3, "valid call")


@pytest.fixture(params=[0, 1], ids=["K1", "K1s"])
def k1_kind(request):
    """Force the persistent staged K1 (0) or the non-persistent streaming K1s (1) for fp32
    n <= 1024 (hh_stream.cu); the default picks by the measured policy."""
    L = hh.hh.lib()
    prev = L.hh_debug_k1_stream(request.param)
    yield request.param
    L.hh_debug_k1_stream(prev)


K1S_SHAPES = [(4, 3, 37), (16, 5, 1001), (32, 4, 999), (64, 6, 1000), (100, 7, 2339), (128, 9, 513),
              (200, 24, 777), (256, 9, 513), (384, 17, 300), (512, 9, 1000), (1000, 12, 250),
              (1024, 10, 3001), (1024, 40, 257)]


@pytest.mark.parametrize("n,h,N", K1S_SHAPES)
def test_k1_and_k1s(k1_kind, n, h, N):
    """Both fused kernels on every fp32 shape class they serve: both ops, the symmetric form,
    the D factor on both sides, the transform-once of Mahalanobis, exact alias."""
    c = gi.make_case("sym", n, h, N, "f32", seed=41)
    d = gi.sign_diag(gi.rng(41, n), n, "f32")
    for op in (0, 1):
        with hh.algo(hh.HH_ALGO_FUSED):
            got = run_apply(op, c.U, c.X)
            want = "f32s_" if k1_kind else "f32_"
            assert hh.last_launch_info()["variant"].startswith(want), hh.last_launch_info()
        assert_parity(got, oracle.apply(op, c.U, c.X), "f32", h, f"{c.name} op{op}")
    with hh.algo(hh.HH_ALGO_FUSED):
        got = hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X)).cpu().numpy()
    assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), "f32", h, f"{c.name} sym")
    for side in (0, 1):
        with hh.algo(hh.HH_ALGO_FUSED):
            got = hh.hh_apply_signed(1, side, dev(c.U), dev(d), dev(c.X)).cpu().numpy()
        assert_parity(got, oracle.apply_signed(1, side, c.U, d, c.X), "f32", h, f"signed {side}")
    m = gi.make_case("mahalanobis", n, h, max(N // 4, 2), "f32", seed=42, npairs=3000)
    got = hh.hh_mahalanobis(dev(m.U), dev(m.d), dev(m.X), dev(m.ia), dev(m.ib)).cpu().numpy()
    assert_parity(got, oracle.mahalanobis(m.U, m.d, m.X, m.ia, m.ib), "f32", h, "mahalanobis")
    X = dev(c.X)
    with hh.algo(hh.HH_ALGO_FUSED):
        hh.hh_apply(0, dev(c.U), X, Y=X)
    torch.cuda.synchronize()
    assert_parity(X.cpu().numpy(), oracle.apply(0, c.U, c.X), "f32", h, "alias")


def test_apply_host_takes_the_wy_path():
    """hh_apply_host past the crossover runs the compact-WY program on each device chunk
    (it had always run K1) and matches the oracle."""
    c = gi.make_case("apply", 1024, 64, 40000, "f32", seed=43)
    X = torch.from_numpy(c.X).pin_memory()
    U = torch.from_numpy(c.U)
    for op in (0, 1):
        Y = hh.hh_apply_host(op, U, X)
        assert hh.last_launch_info()["variant"].startswith("wy_"), hh.last_launch_info()
        assert_parity(Y.numpy(), oracle.apply(op, c.U, c.X), "f32", 64, f"host WY op{op}")


@pytest.fixture(params=[0, 1, 2], ids=["u-smem", "u-tmem", "u-tmem-blocked"])
def k1_tmem(request):
    """Force K1 with the reflectors in shared memory (0), in TMEM (1, K1t) or in TMEM applied in
    blocks (2, K1w) -- the default picks by the measured policy (hh_fused.cu: k1t_preferred,
    k1w_preferred); K1s off so K1 runs."""
    L = hh.hh.lib()
    prev_s = L.hh_debug_k1_stream(0)
    prev_t = L.hh_debug_k1_tmem(1 if request.param else 0)
    prev_b = L.hh_debug_k1_blocked(1 if request.param == 2 else 0)
    yield request.param
    L.hh_debug_k1_blocked(prev_b)
    L.hh_debug_k1_tmem(prev_t)
    L.hh_debug_k1_stream(prev_s)


# every K1 variant built with a TMEM form (TPC = 32 at 256 / 512 threads, 64, 128), full and
# ragged n, up to the largest h whose reflectors fit the CTA's TMEM columns
K1T_SHAPES = [(300, 7, 333), (512, 16, 400), (780, 11, 259), (1024, 16, 1000), (1500, 13, 300),
              (2048, 16, 700), (3000, 9, 150), (4096, 12, 300), (4096, 16, 160), (1024, 3, 77),
              (2048, 5, 90), (4000, 1, 50)]


@pytest.mark.parametrize("n,h,N", K1T_SHAPES)
def test_k1_tmem_reflectors(k1_tmem, n, h, N):
    """K1t (reflectors in TMEM) against the oracle: both ops, the symmetric form, D on both
    sides, the Mahalanobis transform-once, exact alias."""
    c = gi.make_case("sym", n, h, N, "f32", seed=45)
    d = gi.sign_diag(gi.rng(45, n), n, "f32")
    for op in (0, 1):
        with hh.algo(hh.HH_ALGO_FUSED):
            got = run_apply(op, c.U, c.X)
            v = hh.last_launch_info()["variant"]
        assert ("_tmem" in v) == bool(k1_tmem), v
        if n > 512:   # (the 256-thread n <= 512 variant has no blocked form)
            assert ("_kb" in v) == (k1_tmem == 2), v
        assert_parity(got, oracle.apply(op, c.U, c.X), "f32", h, f"{c.name} op{op}")
    with hh.algo(hh.HH_ALGO_FUSED):
        got = hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X)).cpu().numpy()
    assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), "f32", 2 * h, f"{c.name} sym")
    for side in (0, 1):
        with hh.algo(hh.HH_ALGO_FUSED):
            got = hh.hh_apply_signed(0, side, dev(c.U), dev(d), dev(c.X)).cpu().numpy()
        assert_parity(got, oracle.apply_signed(0, side, c.U, d, c.X), "f32", h, f"signed {side}")
    m = gi.make_case("mahalanobis", n, h, max(N // 4, 2), "f32", seed=46, npairs=2000)
    got = hh.hh_mahalanobis(dev(m.U), dev(m.d), dev(m.X), dev(m.ia), dev(m.ib)).cpu().numpy()
    assert_parity(got, oracle.mahalanobis(m.U, m.d, m.X, m.ia, m.ib), "f32", h, "mahalanobis")
    X = dev(c.X)
    with hh.algo(hh.HH_ALGO_FUSED):
        hh.hh_apply(1, dev(c.U), X, Y=X)
    torch.cuda.synchronize()
    assert_parity(X.cpu().numpy(), oracle.apply(1, c.U, c.X), "f32", h, "alias")


def test_k1t_policy():
    """The default picks K1t where the A/B measured it faster (hh_fused.cu: k1t_preferred), in
    blocks of four reflectors (K1w) for multi-warp groups from h = 12 (k1w_preferred)."""
    g = torch.Generator().manual_seed(3)
    for n, h, want, blk in ((4096, 12, True, True), (2048, 9, True, False), (2048, 16, True, True),
                            (1024, 16, True, False), (1024, 10, False, False),
                            (1024, 40, False, False)):
        U = torch.randn(h, n, generator=g, dtype=torch.float64)
        U = (U / U.norm(dim=1, keepdim=True)).float().cuda()
        X = torch.randn(64, n, generator=g).cuda()
        L = hh.hh.lib()
        prev = L.hh_debug_k1_stream(0)
        try:
            with hh.algo(hh.HH_ALGO_FUSED):
                hh.hh_apply(0, U, X)
            v = hh.last_launch_info()["variant"]
        finally:
            L.hh_debug_k1_stream(prev)
        assert ("_tmem" in v) == want, (n, h, v)
        assert v.endswith("_kb4") == blk, (n, h, v)


def test_mahalanobis_sort_beside_transform_matches_serial():
    """hh_mahalanobis runs the pair sort on a second stream beside the transform (fork / join);
    with the overlap off (hh_debug_mahal_fork 0) the result is bit-identical, and both match
    the oracle.  Called twice per mode: the cached side stream is reused."""
    m = gi.make_case("mahalanobis", 256, 7, 3000, "f32", seed=91, npairs=20000)
    args = [dev(a) for a in (m.U, m.d, m.X, m.ia, m.ib)]
    L = hh.hh.lib()
    outs = {}
    for f in (1, 0):
        prev = L.hh_debug_mahal_fork(f)
        try:
            outs[f] = [hh.hh_mahalanobis(*args) for _ in range(2)]
        finally:
            L.hh_debug_mahal_fork(prev)
    torch.cuda.synchronize()
    for a in outs[1] + outs[0][1:]:
        assert torch.equal(a, outs[0][0])
    assert_parity(outs[1][0].cpu().numpy(), oracle.mahalanobis(m.U, m.d, m.X, m.ia, m.ib), "f32", 7,
                  "mahalanobis fork")


def test_fused_path_policy_defaults():
    """HH_ALGO_FUSED's default kernel per shape (all from same-box A/Bs): K1s for n <= 512 and
    for n <= 1024 outside h = 9..16, the staged K1 at n = 1024, h = 10 (C2), K1t at n = 1024,
    h = 12..16 (profiles/r2/k1t_vs_k1s_r2.txt), K1w for multi-warp groups from h = 12."""
    g = torch.Generator().manual_seed(4)
    for n, h, want in ((512, 12, "f32s_"), (1024, 8, "f32s_"), (1024, 10, "f32_tpc32_ch8_c2"),
                       (1024, 12, "f32_tpc32_ch8_c2_tmem"), (1024, 16, "f32_tpc32_ch8_c2_tmem"),
                       (1024, 20, "f32s_"), (4096, 12, "f32_tpc128_ch8_c2_tmem_kb4")):
        U = torch.randn(h, n, generator=g, dtype=torch.float64)
        U = (U / U.norm(dim=1, keepdim=True)).float().cuda()
        X = torch.randn(300, n, generator=g).cuda()
        with hh.algo(hh.HH_ALGO_FUSED):
            hh.hh_apply(0, U, X)
        v = hh.last_launch_info()["variant"]
        assert v == want or (want == "f32s_" and v.startswith(want)), (n, h, v)


# ------------------------------------------------------------------ K1g: every other shape
# n*size not a multiple of 16 bytes, n beyond the vector kernels' tables, n = 1; several
# column groups per CTA and a ragged last group; fp32 and fp64
GENERAL_SHAPES = [
    # one shape per K1r table row (ragged n inside each), several batches per unit
    (63, 5, 3000, "f32"), (127, 6, 2500, "f32"), (250, 9, 2100, "f32"), (511, 12, 1900, "f32"),
    (2047, 11, 1300, "f32"), (4095, 7, 700, "f32"), (8191, 3, 300, "f32"), (1021, 40, 900, "f32"),
    (63, 5, 1500, "f64"), (127, 4, 1100, "f64"), (255, 8, 900, "f64"), (509, 10, 800, "f64"),
    (1023, 9, 700, "f64"), (4095, 3, 200, "f64"),
    (1, 3, 17, "f32"), (3, 2, 50, "f64"), (30, 5, 333, "f32"), (50, 7, 1001, "f32"),
    (101, 9, 257, "f64"), (1023, 10, 700, "f32"), (1022, 4, 90, "f32"), (2049, 6, 130, "f64"),
    (9000, 5, 41, "f32"), (20000, 3, 10, "f32"), (5001, 4, 23, "f64"), (40000, 2, 5, "f32"),
]


def is_general(dt):
    """K1r (scalar-element persistent kernel, `f32r_...`) or K1g (`f32_general...`) ran."""
    v = hh.last_launch_info()["variant"]
    return v.startswith(f"{dt}r_") or v.startswith(f"{dt}_general")


class padded:
    """Test hook: 1 = take the padded detour whenever the stride is unaligned, 0 = never."""

    def __init__(self, on):
        self.on = on

    def __enter__(self):
        self.prev = hh.hh.lib().hh_debug_general_pad(self.on)
        hh.hh.clear_workspace_cache()       # the knob sizes the workspace

    def __exit__(self, *exc):
        hh.hh.lib().hh_debug_general_pad(self.prev)
        hh.hh.clear_workspace_cache()


class k1r_smem:
    """Test hook: K1r with U in shared memory (0: its TMEM form off), or TMEM wherever the
    variant has the form (2: also the multi-warp groups the policy leaves on shared memory)."""

    def __init__(self, mode=0):
        self.mode = mode

    def __enter__(self):
        self.prev = hh.hh.lib().hh_debug_k1r_tmem(self.mode)

    def __exit__(self, *exc):
        hh.hh.lib().hh_debug_k1r_tmem(self.prev)


class k1r_nostage:
    """Test hook: K1r loading columns straight into registers (its staged tiles off)."""

    def __enter__(self):
        self.prev = hh.hh.lib().hh_debug_k1r_stage(0)

    def __exit__(self, *exc):
        hh.hh.lib().hh_debug_k1r_stage(self.prev)


class k1g_only:
    """Test hook: keep K1r off so that K1g also serves the shapes K1r would take."""

    def __enter__(self):
        self.prev = hh.hh.lib().hh_debug_general_scalar(0)

    def __exit__(self, *exc):
        hh.hh.lib().hh_debug_general_scalar(self.prev)


@pytest.mark.parametrize("n,h,N,dt", GENERAL_SHAPES)
@pytest.mark.parametrize("k1r", [True, "smem", "nostage", False])
def test_general_apply(n, h, N, dt, k1r):
    """Shapes the vector kernels refuse run on K1r / K1g: both ops, and in place (Y == X);
    once as the library picks (K1r while n is inside its tables, its TMEM form for fp32
    n in (512, 4096], h <= 16), once with K1r's shared-memory form, once on K1g alone."""
    import contextlib
    c = gi.make_case("apply", n, h, N, dt, seed=31)
    ctx = contextlib.nullcontext() if k1r is True else k1r_smem(0) if k1r == "smem" else \
        k1r_nostage() if k1r == "nostage" else k1g_only()
    with ctx, padded(0):
        for op in (0, 1):
            got = run_apply(op, c.U, c.X)
            assert is_general(dt), hh.last_launch_info()
            v = hh.last_launch_info()["variant"]
            if not k1r or n > (4096 if dt == "f32" else 2048):
                assert v.startswith(f"{dt}_general")
            else:
                assert v.startswith(f"{dt}r_")
                tm = dt == "f32" and 0 < h <= 16 and 512 < n and k1r != "smem"
                assert v.endswith("_tmem") == tm, v
            assert_parity(got, oracle.apply(op, c.U, c.X), dt, h, f"K1r/K1g n={n} op{op}")
        X = dev(c.X)
        out = hh.hh_apply(0, dev(c.U), X, X)
        assert out.data_ptr() == X.data_ptr()
        assert_parity(out.cpu().numpy(), oracle.apply(0, c.U, c.X), dt, h, f"K1r/K1g n={n} alias")


@pytest.mark.parametrize("n,h,N,dt", [(30, 5, 333, "f32"), (101, 9, 257, "f64"),
                                      (1023, 10, 300, "f32"), (9000, 5, 41, "f32")])
@pytest.mark.parametrize("k1r", [True, False])
def test_general_sym_signed_mahalanobis(n, h, N, dt, k1r):
    import contextlib
    with (contextlib.nullcontext() if k1r else k1g_only()), padded(0):
        _general_sym_signed_mahalanobis(n, h, N, dt)


def _general_sym_signed_mahalanobis(n, h, N, dt):
    c = gi.make_case("sym", n, h, N, dt, seed=32)
    got = hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X)).cpu().numpy()
    assert is_general(dt)
    assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), dt, h, f"K1g sym n={n}")
    g = gi.rng(33, n)
    d = np.where(g.random(n) < 0.5, -1.0, 1.0).astype(c.X.dtype)
    for op in (0, 1):
        for side in (0, 1):
            got = hh.hh_apply_signed(op, side, dev(c.U), dev(d), dev(c.X)).cpu().numpy()
            assert_parity(got, oracle.apply_signed(op, side, c.U, d, c.X), dt, h,
                          f"K1g signed n={n} op{op} side{side}")
    got = hh.hh_sym_apply_signed(dev(c.U), dev(d), dev(c.lam), dev(c.X)).cpu().numpy()
    assert_parity(got, oracle.sym_apply_signed(c.U, d, c.lam, c.X), dt, h, f"K1g sym signed n={n}")
    m = gi.make_case("mahalanobis", n, h, 64, dt, seed=34, npairs=999)
    m.ia[:8] = m.ib[:8]
    dist = hh.hh_mahalanobis(dev(m.U), dev(m.d), dev(m.X), dev(m.ia), dev(m.ib)).cpu().numpy()
    assert is_general(dt)
    assert_parity(dist, oracle.mahalanobis(m.U, m.d, m.X, m.ia, m.ib), dt, h, f"K1g pairs n={n}")
    assert np.all(dist[:8] == 0.0)


def test_general_misaligned_pointers_and_edges():
    """16-byte misaligned (but element-aligned) operands take K1g; h = 0 copies; N < group."""
    c = gi.make_case("apply", 64, 6, 40, "f32", seed=35)
    buf = torch.zeros(40 * 64 + 1, device="cuda")
    Xo = buf[1:].view(40, 64)                      # data_ptr % 16 == 4
    Xo.copy_(dev(c.X))
    assert Xo.data_ptr() % 16 == 4
    got = hh.hh_apply(0, dev(c.U), Xo).cpu().numpy()
    assert is_general("f32")
    assert_parity(got, oracle.apply(0, c.U, c.X), "f32", 6, "K1g misaligned X")
    e = gi.make_case("apply", 30, 0, 3, "f32", seed=36)
    U0 = torch.empty(0, 30, device="cuda")
    assert np.array_equal(hh.hh_apply(1, U0, dev(e.X)).cpu().numpy(), e.X)
    z = gi.make_case("apply", 50, 4, 2, "f64", seed=37, zero_slots=(1,))
    assert_parity(run_apply(0, z.U, z.X), oracle.apply(0, z.U, z.X), "f64", 4, "K1g u = 0 slot")


def test_general_host_path():
    c = gi.make_case("apply", 1022, 8, 500, "f32", seed=38)
    out = hh.hh_apply_host(0, torch.from_numpy(c.U), torch.from_numpy(c.X)).numpy()
    assert_parity(out, oracle.apply(0, c.U, c.X), "f32", 8, "K1g host")


# ------------------------------------------------------------------ the padded detour
@pytest.mark.parametrize("n,h,N,dt", [(30, 5, 333, "f32"), (101, 9, 257, "f64"), (1023, 10, 700, "f32"),
                                      (1021, 40, 900, "f32"), (2047, 70, 300, "f32"),
                                      (4095, 300, 140, "f32"), (9001, 20, 64, "f32"),
                                      (509, 33, 500, "f64"), (8190, 12, 70, "f32")])
def test_padded_detour(n, h, N, dt):
    """Unaligned column strides through the padded copy (forced by the hook so that small h
    takes it too): apply (both ops, alias), D on both sides, the symmetric forms -- and the
    policy's own choice at these shapes."""
    c = gi.make_case("sym", n, h, N, dt, seed=41)
    d = np.where(gi.rng(42, n).random(n) < 0.5, -1.0, 1.0).astype(c.X.dtype)
    for mode in (1, -1):
        with padded(mode):
            for op in (0, 1):
                got = run_apply(op, c.U, c.X)
                if mode == 1:
                    assert not is_general(dt), hh.last_launch_info()
                assert_parity(got, oracle.apply(op, c.U, c.X), dt, h, f"padded n={n} op{op}")
            got = hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X)).cpu().numpy()
            assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), dt, h, f"padded sym n={n}")
    with padded(1):
        X = dev(c.X)
        out = hh.hh_apply(1, dev(c.U), X, X)
        assert_parity(out.cpu().numpy(), oracle.apply(1, c.U, c.X), dt, h, f"padded alias n={n}")
        for side in (0, 1):
            got = hh.hh_apply_signed(0, side, dev(c.U), dev(d), dev(c.X)).cpu().numpy()
            assert_parity(got, oracle.apply_signed(0, side, c.U, d, c.X), dt, h, f"padded D n={n}")
        got = hh.hh_sym_apply_signed(dev(c.U), dev(d), dev(c.lam), dev(c.X)).cpu().numpy()
        assert_parity(got, oracle.sym_apply_signed(c.U, d, c.lam, c.X), dt, h, f"padded sym D n={n}")
        if dt == "f32" and n >= 32:
            with hh.algo(hh.HH_ALGO_WY):                 # a forced block program runs on the copy
                got = run_apply(0, c.U, c.X)
                assert hh.last_launch_info()["variant"].startswith("wy_"), hh.last_launch_info()
            assert_parity(got, oracle.apply(0, c.U, c.X), dt, h, f"padded WY n={n}")


@pytest.mark.parametrize("n,h,M,npairs,dt", [(30, 5, 64, 999, "f32"), (101, 9, 300, 5000, "f64"),
                                             (511, 9, 2000, 30000, "f32"), (1023, 0, 100, 777, "f32")])
def test_padded_mahalanobis(n, h, M, npairs, dt):
    """Unaligned point stride with a workspace: transform-once + bucketed gather on the padded
    copy (a = b stays exactly 0); without the detour the per-pair form on K1r / K1g."""
    m = gi.make_case("mahalanobis", n, h, M, dt, seed=43, npairs=npairs)
    m.ia[:8] = m.ib[:8]
    ref = oracle.mahalanobis(m.U, m.d, m.X, m.ia, m.ib)
    U = dev(m.U) if h else torch.empty(0, n, device="cuda", dtype=TDT[dt])
    for mode in (-1, 0):
        with padded(mode):
            dist = hh.hh_mahalanobis(U, dev(m.d), dev(m.X), dev(m.ia), dev(m.ib)).cpu().numpy()
            assert is_general(dt) == (mode == 0), hh.last_launch_info()
            assert_parity(dist, ref, dt, h, f"padded pairs n={n} mode={mode}")
            assert np.all(dist[:8] == 0.0)
