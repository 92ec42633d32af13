"""GPU parity of the compact-WY tensor-core path (K4 + K5, hh_wy.cu) against the oracle.

K5 evaluates the same product Q = H_1 ... H_h in the blocked form I - W T W^T
 on tcgen05 with a bf16x3 split; the gate is the north_star's
fp32 gate 2e-5*sqrt(h).  The debug hook checks the intermediate G = W^T X and
V = W T of the first applied block against plain fp64 numpy written from Eq. 2.
"""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gi
from tests._util import assert_parity, rel_fro

pytestmark = pytest.mark.gpu
hh = pytest.importorskip("paper_1811_07624_b200")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def wy(op, U, X, Y=None):
    with hh.algo(hh.HH_ALGO_WY):
        out = hh.hh_apply(op, dev(U), dev(X), Y)
        assert hh.last_launch_info()["variant"].startswith("wy_"), hh.last_launch_info()
    torch.cuda.synchronize()
    return out.cpu().numpy()


def bf16_pair_to_f64(ws, off, count, lo_off):
    raw = ws[off:off + 2 * count].view(torch.int16).to(torch.int32).cpu().numpy()
    hi = (raw.astype(np.int64) & 0xFFFF) << 16
    raw_lo = ws[off + 2 * lo_off:off + 2 * lo_off + 2 * count].view(torch.int16).to(
        torch.int32).cpu().numpy()
    lo = (raw_lo.astype(np.int64) & 0xFFFF) << 16
    f = lambda a: a.astype(np.uint32).view(np.float32).astype(np.float64)  # noqa: E731
    return f(hi) + f(lo)


@pytest.mark.parametrize("n,h,N,op", [(256, 40, 300, 0), (512, 70, 257, 1), (4096, 256, 130, 0),
                                      (1024, 300, 129, 1)])
def test_wy_intermediates(n, h, N, op):
    """G = W^T X and V = W T of the first applied block match fp64 numpy.  Blocks are cut in
    product order -- Q^T X runs the REVERSED reflector list as a Q X program --
    and the last block is applied first; T by the forward recurrence
    T[:i, i] = -2 T[:i,:i] W[:, :i]^T w_i."""
    c = gi.make_case("apply", n, h, N, "f32", seed=21)
    U, X = dev(c.U), dev(c.X)
    with hh.algo(hh.HH_ALGO_WY):
        wsb = hh.hh_workspace_bytes(hh.HH_CALL_APPLY, n, h, N, 0, torch.float32)
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
    off = hh.debug_wy_project(op, U, X, ws)
    torch.cuda.synchronize()
    b, nblk, n_pad = off["b"], off["nblk"], off["n_pad"]
    order = np.arange(h) if op == 0 else np.arange(h)[::-1]
    Wfull = np.zeros((nblk * b, n))
    Wfull[:h] = c.U.astype(np.float64)[order]
    k = nblk - 1
    W = Wfull[k * b:(k + 1) * b]                       # (b, n): rows w_i
    G_ref = c.X.astype(np.float64) @ W.T               # (N, b)
    G = bf16_pair_to_f64(ws, off["G"], N * b, N * b).reshape(N, b)
    # bf16x3: each operand carries ~2^-17 relative split error, hi*hi + hi*lo + lo*hi
    # drops lo*lo (~2^-18), and G itself is stored as a hi+lo pair (2^-17): a few
    # times 2^-17 = 7.6e-6 relative
    assert rel_fro(G, G_ref) < 4e-5, rel_fro(G, G_ref)
    T = np.zeros((b, b))
    for i in range(b):
        T[i, i] = 2.0
        if i:
            T[:i, i] = -2.0 * T[:i, :i] @ (W[:i] @ W[i])
    V_ref = W.T @ T                                    # (n, b)
    V = bf16_pair_to_f64(ws, off["V"] + 2 * k * n_pad * b, n_pad * b,
                         nblk * n_pad * b).reshape(n_pad, b)[:n]
    assert rel_fro(V, V_ref) < 4e-5, rel_fro(V, V_ref)
    # the block formula reproduces the sequential product (fp64, pins the recurrence)
    Qb = np.eye(n) - W.T @ T @ W
    Qs = np.eye(n)
    for i in range(b):
        Qs = Qs @ (np.eye(n) - 2.0 * np.outer(W[i], W[i]))
    assert np.abs(Qb - Qs).max() < 1e-10


WY_SHAPES = [  # (n, h, N): several tiles + ragged tails, b in {32, 64, 160, 256}, nblk up to 4
    (256, 40, 300), (512, 33, 777), (1024, 64, 1000), (2048, 32, 1500), (100, 50, 129),
    (4096, 64, 515), (4096, 300, 130), (1000, 257, 200), (4096, 1024, 130), (32, 20, 64),
]


@pytest.mark.parametrize("n,h,N", WY_SHAPES)
@pytest.mark.parametrize("op", [0, 1])
def test_wy_parity(n, h, N, op):
    c = gi.make_case("apply", n, h, N, "f32", seed=22)
    got = wy(op, c.U, c.X)
    assert_parity(got, oracle.apply(op, c.U, c.X), "f32", h, f"WY n{n} h{h} N{N} op{op}")


@pytest.mark.parametrize("n,h,N", [(8196, 40, 300), (12288, 24, 260), (16384, 64, 300),
                                   (32768, 300, 140), (65536, 33, 130)])
def test_wy_large_n(n, h, N):
    """n beyond the fused kernels' tables (8192): the block program takes aligned shapes up to
    n = 65536 -- apply (both ops, AUTO picks it past the crossover) and the symmetric form."""
    c = gi.make_case("sym", n, h, N, "f32", seed=29)
    for op in (0, 1):
        got = wy(op, c.U, c.X)
        assert hh.last_launch_info()["variant"].startswith("wy_"), hh.last_launch_info()
        assert_parity(got, oracle.apply(op, c.U, c.X), "f32", h, f"WY n{n} h{h} op{op}")
    got = hh.hh_apply(0, dev(c.U), dev(c.X)).cpu().numpy()      # AUTO
    assert_parity(got, oracle.apply(0, c.U, c.X), "f32", h, f"auto n{n} h{h}")
    with hh.algo(hh.HH_ALGO_WY):
        got = hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X)).cpu().numpy()
    assert hh.last_launch_info()["variant"].startswith("wy_sym"), hh.last_launch_info()
    assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), "f32", h, f"WY sym n{n} h{h}")


def test_wy_alias_zero_slots_and_round_trip():
    c = gi.make_case("apply", 1024, 96, 400, "f32", seed=23, zero_slots=(0, 5, 95))
    U, X = dev(c.U), dev(c.X)
    ref = oracle.apply(0, c.U, c.X)
    with hh.algo(hh.HH_ALGO_WY):
        out = hh.hh_apply(0, U, X, Y=X)                 # exact alias
        torch.cuda.synchronize()
        assert out.data_ptr() == X.data_ptr()
        assert_parity(X.cpu().numpy(), ref, "f32", 96, "WY alias")
        back = hh.hh_apply(1, U, X)                     # Q^T (Q X) = X (orthonormal up to fp32 u)
    torch.cuda.synchronize()
    assert rel_fro(back.cpu().numpy(), c.X) < 2e-5 * np.sqrt(96)


def test_wy_errors():
    X = torch.randn(10, 1024, device="cuda")
    U = torch.randn(40, 1024, device="cuda")
    with hh.algo(hh.HH_ALGO_WY):
        st = hh.hh.lib().hh_apply(0, 1024, 40, hh.hh._ptr(U), hh.hh._ptr(X),
                                  hh.hh._ptr(torch.empty_like(X)), 10, 0, None, 0, None)
        assert st == hh.hh.HH_ERR_WORKSPACE
    assert hh.hh_get_algo() == hh.HH_ALGO_AUTO
    with pytest.raises(hh.HHError):
        hh.hh_set_algo(7)


SYM_SHAPES = [  # (n, h, N): one block (b = 32..128) and several (m = 2, 3), ragged tails
    (2048, 32, 700), (256, 20, 300), (512, 100, 257), (1024, 129, 200), (4096, 300, 130),
    (100, 40, 129),
]


def wy_sym(U, lam, X):
    with hh.algo(hh.HH_ALGO_WY):
        out = hh.hh_sym_apply(dev(U), dev(lam), dev(X))
        assert hh.last_launch_info()["variant"].startswith("wy_sym"), hh.last_launch_info()
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("n,h,N", SYM_SHAPES)
def test_wy_sym_parity(n, h, N):
    """Q diag(lambda) Q^T X by the tensor-core block program vs the oracle (C3 spectrum
    recipe: exp(-k/200) with 10% sign flips)."""
    c = gi.make_case("sym", n, h, N, "f32", seed=24)
    got = wy_sym(c.U, c.lam, c.X)
    assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), "f32", h, f"WY sym n{n} h{h}")


def test_wy_sym_special_cases():
    """lambda == 1 -> X (Q Q^T = I up to fp32 u); lambda == -1 -> -X; alias Y == X."""
    c = gi.make_case("sym", 1024, 48, 300, "f32", seed=25)
    ones = np.ones(1024, dtype=np.float32)
    assert rel_fro(wy_sym(c.U, ones, c.X), c.X) < 2e-5 * np.sqrt(48)
    assert rel_fro(wy_sym(c.U, -ones, c.X), -c.X) < 2e-5 * np.sqrt(48)
    X = dev(c.X)
    with hh.algo(hh.HH_ALGO_WY):
        hh.hh_sym_apply(dev(c.U), dev(c.lam), X, Y=X)
    torch.cuda.synchronize()
    assert_parity(X.cpu().numpy(), oracle.sym_apply(c.U, c.lam, c.X), "f32", 48, "sym alias")


@pytest.fixture
def ts_everywhere():
    """Run the update in TS mode (G in TMEM, wy_update_ts_kernel) at every block width."""
    L = hh.hh.lib()
    prev = L.hh_debug_wy_ts_min(32)
    yield
    L.hh_debug_wy_ts_min(prev)


@pytest.mark.parametrize("n,h,N", [(256, 40, 300), (2048, 32, 1500), (100, 50, 129),
                                   (4096, 300, 130), (1000, 257, 200)])
@pytest.mark.parametrize("op", [0, 1])
def test_wy_ts_parity_all_widths(ts_everywhere, n, h, N, op):
    """The TS-mode update (used by default only for 256-wide blocks) at b = 32 ... 160 and
    ragged shapes, against the oracle."""
    c = gi.make_case("apply", n, h, N, "f32", seed=22)
    got = wy(op, c.U, c.X)
    assert_parity(got, oracle.apply(op, c.U, c.X), "f32", h, f"WY-TS n{n} h{h} N{N} op{op}")


def test_wy_ts_sym_and_qr(ts_everywhere):
    c = gi.make_case("sym", 512, 40, 333, "f32", seed=26)
    got = wy_sym(c.U, c.lam, c.X)
    assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), "f32", 40, "WY-TS sym")
    n, h, N = 512, 300, 200
    U = gi.qr_reflectors(gi.rng(27, n, h), h, n, "f32")
    X = gi.gaussian_columns(gi.rng(28, n, h), N, n, "f32")
    with hh.algo(hh.HH_ALGO_WY):
        out = hh.hh_apply_qr(0, dev(U), dev(X))
    torch.cuda.synchronize()
    assert_parity(out.cpu().numpy(), oracle.apply(0, U, X), "f32", h, "WY-TS QR")


# More tiles than SMs: the K5a balanced schedule cuts tiles between two CTAs (the split-tile
# hand-off) and K5b splits (tile, row chunk) ranges -- full output against the oracle.
MANY_TILES = [(512, 64, 40000), (256, 300, 20000), (1024, 33, 30001)]


@pytest.mark.parametrize("n,h,N", MANY_TILES)
@pytest.mark.parametrize("op", [0, 1])
def test_wy_many_tiles(n, h, N, op):
    c = gi.make_case("apply", n, h, N, "f32", seed=29)
    got = wy(op, c.U, c.X)
    assert_parity(got, oracle.apply(op, c.U, c.X), "f32", h, f"WY many tiles n{n} h{h} op{op}")
    col = np.linalg.norm(got - oracle.apply(op, c.U, c.X), axis=1) / np.linalg.norm(c.X, axis=1)
    assert col.max() <= 2e-5 * np.sqrt(h), col.max()


@pytest.mark.parametrize("n,h,N", [(512, 64, 40000), (256, 200, 20000)])
def test_wy_sym_many_tiles(n, h, N):
    c = gi.make_case("sym", n, h, N, "f32", seed=30)
    got = wy_sym(c.U, c.lam, c.X)
    assert_parity(got, oracle.sym_apply(c.U, c.lam, c.X), "f32", h, f"WY sym many tiles n{n} h{h}")


@pytest.mark.parametrize("op", [0, 1])
def test_wy_ts_many_tiles(ts_everywhere, op):
    c = gi.make_case("apply", 512, 64, 40000, "f32", seed=31)
    got = wy(op, c.U, c.X)
    assert_parity(got, oracle.apply(op, c.U, c.X), "f32", 64, f"WY-TS many tiles op{op}")


@pytest.fixture
def flow_on():
    """The single-launch dataflow form of the block program (K5f, opt-in: measured slower
    than the two-kernel program) for this test."""
    L = hh.hh.lib()
    prev = L.hh_debug_wy_flow(1, 0)
    yield
    L.hh_debug_wy_flow(prev, 0)


@pytest.mark.parametrize("call,n,h,N,op", [("apply", 512, 64, 40000, 0), ("apply", 512, 64, 40000, 1),
                                           ("apply", 4096, 64, 2000, 0), ("apply", 1024, 300, 3000, 1),
                                           ("apply", 4096, 1024, 700, 0), ("sym", 2048, 32, 5000, 0),
                                           ("sym", 512, 100, 3000, 0), ("apply", 100, 50, 129, 1)])
def test_wy_flow_parity(flow_on, call, n, h, N, op):
    c = gi.make_case(call, n, h, N, "f32", seed=5)
    if call == "sym":
        got = wy_sym(c.U, c.lam, c.X)
        ref = oracle.sym_apply(c.U, c.lam, c.X)
    else:
        got = wy(op, c.U, c.X)
        ref = oracle.apply(op, c.U, c.X)
    assert "flow" in hh.last_launch_info()["variant"], hh.last_launch_info()
    assert_parity(got, ref, "f32", h, f"K5f {call} n{n} h{h} N{N} op{op}")


@pytest.mark.parametrize("tsa", [0, 1])
@pytest.mark.parametrize("n,h,N", [(1024, 64, 40000), (1000, 40, 3001), (2048, 33, 20000), (512, 128, 9000)])
def test_wy_project_tmem_a_bit_identical(tsa, n, h, N):
    """K5a with X converted into TMEM (the default for blocks of <= 128) and the shared-memory
    form (hh_debug_wy_tsa 0) give bit-identical results: same bf16 splits, same MMA order --
    both ops, the symmetric program and a right D factor; and both match the oracle."""
    c = gi.make_case("sym", n, h, N, "f32", seed=3)
    d = gi.sign_diag(gi.rng(3, n), n, "f32")
    L = hh.hh.lib()
    outs = {}
    for on in (1 - tsa, tsa):
        prev = L.hh_debug_wy_tsa(on)
        try:
            with hh.algo(hh.HH_ALGO_WY):
                outs[on] = [hh.hh_apply(op, dev(c.U), dev(c.X)) for op in (0, 1)] + [
                    hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X)),
                    hh.hh_apply_signed(0, 1, dev(c.U), dev(d), dev(c.X))]
        finally:
            L.hh_debug_wy_tsa(prev)
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
    assert_parity(outs[tsa][2].cpu().numpy(), oracle.sym_apply(c.U, c.lam, c.X), "f32", 2 * h, "sym")
