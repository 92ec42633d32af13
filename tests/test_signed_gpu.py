"""GPU parity of the NEXT-f1 operator forms with the diagonal D of Eq. 1:
D op(Q) X, op(Q) D X and D Q diag(lambda) Q^T D X, on both the fused kernel (K1/K2) and
the compact-WY tensor-core path (K5), against the oracle's literal scale-apply-scale."""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gi
from tests._util import assert_parity

pytestmark = pytest.mark.gpu
hh = pytest.importorskip("paper_1811_07624_b200")
ALGOS = {"fused": 1, "wy": 2}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("path", ["fused", "wy"])
@pytest.mark.parametrize("n,h,N", [(1024, 10, 1000), (512, 70, 300), (4096, 12, 200),
                                   (256, 300, 129)])
def test_apply_signed(path, n, h, N):
    c = gi.make_case("apply", n, h, N, "f32", seed=31)
    d = gi.sign_diag(gi.rng(31, n), n, "f32")
    with hh.algo(ALGOS[path]):
        for op in (0, 1):
            for side in (hh.HH_SIDE_LEFT, hh.HH_SIDE_RIGHT):
                got = hh.hh_apply_signed(op, side, dev(c.U), dev(d), dev(c.X)).cpu().numpy()
                if path == "wy":
                    assert hh.last_launch_info()["variant"].startswith("wy_")
                ref = oracle.apply_signed(op, side, c.U, d, c.X)
                assert_parity(got, ref, "f32", h, f"{path} op{op} side{side}")


def test_apply_signed_fp64():
    c = gi.make_case("apply", 64, 6, 500, "f64", seed=32)
    d = gi.sign_diag(gi.rng(32), 64)
    for op in (0, 1):
        for side in (0, 1):
            got = hh.hh_apply_signed(op, side, dev(c.U), dev(d), dev(c.X)).cpu().numpy()
            assert_parity(got, oracle.apply_signed(op, side, c.U, d, c.X), "f64", 6, "f64")


@pytest.mark.parametrize("path", ["fused", "wy"])
@pytest.mark.parametrize("n,h,N", [(2048, 32, 700), (512, 150, 257), (256, 20, 300)])
def test_sym_apply_signed(path, n, h, N):
    c = gi.make_case("sym", n, h, N, "f32", seed=33)
    d = gi.sign_diag(gi.rng(33, n), n, "f32")
    with hh.algo(ALGOS[path]):
        got = hh.hh_sym_apply_signed(dev(c.U), dev(d), dev(c.lam), dev(c.X)).cpu().numpy()
    ref = oracle.sym_apply_signed(c.U, d, c.lam, c.X)
    assert_parity(got, ref, "f32", h, f"sym signed {path}")


def test_signed_errors():
    X = torch.randn(4, 64, device="cuda")
    U = torch.randn(2, 64, device="cuda")
    L = hh.hh.lib()
    st = L.hh_apply_signed(0, 5, 64, 2, hh.hh._ptr(U), hh.hh._ptr(torch.ones(64, device="cuda")),
                           hh.hh._ptr(X), hh.hh._ptr(torch.empty_like(X)), 4, 0, None, 0, None)
    assert st == hh.hh.HH_ERR_INVALID_VALUE
    st = L.hh_apply_signed(0, 0, 64, 2, hh.hh._ptr(U), None, hh.hh._ptr(X),
                           hh.hh._ptr(torch.empty_like(X)), 4, 0, None, 0, None)
    assert st == hh.hh.HH_ERR_INVALID_VALUE
