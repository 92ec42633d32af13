"""GPU parity of NEXT-f2, QR-structured ("trapezoidal") reflectors: hh_apply_qr skips the
zero prefix u_i[r] = 0 for r < i (Result 3's partial QR) and must equal the
oracle's full apply on the same U; the h = n-1 QR reflectors of a random orthonormal
matrix reproduce it up to +-1 on the GPU too."""
import numpy as np
import pytest
import torch

import oracle
from gen import inputs as gi
from tests._util import assert_parity
from tests.test_oracle_pins import householder_qr_reflectors

pytestmark = pytest.mark.gpu
hh = pytest.importorskip("paper_1811_07624_b200")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n,h,N,dt,path", [(1024, 10, 700, "f32", "auto"), (512, 511, 300, "f32", "wy"),
                                           (4096, 1024, 130, "f32", "wy"), (256, 255, 200, "f64", "auto"),
                                           (300, 299, 129, "f32", "wy"), (512, 300, 257, "f32", "fused")])
def test_apply_qr(n, h, N, dt, path):
    g = gi.rng(700, n, h, N)
    U = gi.qr_reflectors(g, h, n, dt)
    X = gi.gaussian_columns(g, N, n, dt)
    a = {"auto": hh.HH_ALGO_AUTO, "wy": hh.HH_ALGO_WY, "fused": hh.HH_ALGO_FUSED}[path]
    for op in (0, 1):
        ref = oracle.apply(op, U, X)
        with hh.algo(a):
            got = hh.hh_apply_qr(op, dev(U), dev(X)).cpu().numpy()
            assert_parity(got, ref, dt, h, f"qr n{n} h{h} op{op} {path}")
            Xd = dev(X)
            hh.hh_apply_qr(op, dev(U), Xd, Y=Xd)            # in place
            torch.cuda.synchronize()
            assert_parity(Xd.cpu().numpy(), ref, dt, h, f"qr in place op{op} {path}")


@pytest.mark.parametrize("n,dt", [(64, "f64"), (512, "f32")])
def test_qr_reproduces_orthonormal(n, dt):
    G = gi.rng(701, n).standard_normal((n, n))
    U0, _ = np.linalg.qr(G)
    J, R = householder_qr_reflectors(U0)
    D = np.diag(np.diag(R))
    Jd = J.astype(np.float32 if dt == "f32" else np.float64)
    QD = hh.hh_apply_qr(0, dev(Jd), dev(D.astype(Jd.dtype))).cpu().numpy().T
    tol = 1e-12 if dt == "f64" else 2e-5 * np.sqrt(n - 1)
    assert np.linalg.norm(QD - U0) / np.linalg.norm(U0) < tol
