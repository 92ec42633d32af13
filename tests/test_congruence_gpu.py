"""GPU parity of NEXT-f4: op(Q) M op(Q)^T (the SHF congruences eq:ak / eq:bk)
against the oracle's literal apply-transpose-apply-transpose, on the fused and the
compact-WY apply paths."""
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


@pytest.mark.parametrize("n,h,count,dt,path", [(64, 6, 5, "f64", "auto"), (1024, 10, 3, "f32", "auto"),
                                               (512, 40, 2, "f32", "wy"), (512, 40, 2, "f32", "fused"),
                                               (100, 7, 4, "f32", "auto"), (2048, 33, 1, "f32", "auto"),
                                               # n * size not a multiple of 16 bytes: K1g applies
                                               (101, 7, 3, "f32", "auto"), (33, 5, 4, "f64", "auto"),
                                               (9, 4, 6, "f32", "auto"), (1025, 6, 1, "f32", "auto")])
def test_congruence(n, h, count, dt, path):
    g = gi.rng(600, n, h, count)
    U = gi.unit_reflectors(g, h, n, dt)
    M = g.standard_normal((count, n, n)).astype(np.float32 if dt == "f32" else np.float64)
    a = {"auto": hh.HH_ALGO_AUTO, "wy": hh.HH_ALGO_WY, "fused": hh.HH_ALGO_FUSED}[path]
    for op in (0, 1):
        with hh.algo(a):
            got = hh.hh_congruence(op, dev(U), dev(M)).cpu().numpy()
        ref = oracle.congruence(op, U, M)
        assert_parity(got, ref, dt, h, f"congruence n{n} h{h} op{op} {path}")


def test_congruence_alias_and_shf_blocks():
    """M_out may alias M; A_k (op T, prefix reflectors) and B_k (op N, suffix) as the SHF
    loop forms them."""
    n, h, k = 256, 12, 5
    g = gi.rng(601)
    U = gi.unit_reflectors(g, h, n, "f32")
    A = g.standard_normal((n, n))
    S = (A + A.T).astype(np.float32)[None]
    Mt = dev(S.copy())
    hh.hh_congruence(1, dev(U[:k - 1]), Mt, out=Mt)
    torch.cuda.synchronize()
    assert_parity(Mt.cpu().numpy(), oracle.congruence(1, U[:k - 1], S), "f32", k - 1, "A_k alias")
    s = np.diag(g.standard_normal(n)).astype(np.float32)[None]
    got = hh.hh_congruence(0, dev(U[k:]), dev(s)).cpu().numpy()
    assert_parity(got, oracle.congruence(0, U[k:], s), "f32", h - k, "B_k")


@pytest.mark.parametrize("n,h,count", [(300, 9, 5), (1000, 5, 2), (96, 12, 3), (4, 3, 7),
                                       (1024, 18, 2), (256, 64, 3)])
def test_congruence_row_kernel(n, h, count):
    """fp32 n <= 1024: the column apply followed by the row kernel K7 (every row of
    op(Q) M through op(Q)) -- ragged row slabs, both ops, and M_out aliasing M."""
    g = gi.rng(602, n, h, count)
    U = gi.unit_reflectors(g, h, n, "f32")
    M = g.standard_normal((count, n, n)).astype(np.float32)
    for op in (0, 1):
        ref = oracle.congruence(op, U, M)
        got = hh.hh_congruence(op, dev(U), dev(M)).cpu().numpy()
        assert_parity(got, ref, "f32", h, f"K7 n{n} h{h} op{op}")
        Mt = dev(M)
        hh.hh_congruence(op, dev(U), Mt, out=Mt)
        torch.cuda.synchronize()
        assert_parity(Mt.cpu().numpy(), ref, "f32", h, f"K7 alias n{n} op{op}")
