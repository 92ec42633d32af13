"""NEXT-f4: the SHF objective C(u) of one reflector and its gradient for a batch of candidate
vectors (hh_shf_cost; eq:theRk P:316-320, the trace identity P:371, eq:gradient P:373-377)
against the fp64 oracle (oracle.shf_cost, pinned in test_oracle_pins.py).

Gate (reading R21): C = 2 a.b - 2 (u.a)(u.b) cancels, so each candidate's error is
measured against the size of its terms, s_k = 2 |a||b| + 2 |u.a||u.b| (a = A u, b = B u), and
the gradient's against 2 (|A||b| + |B||a|) + 4 (|u.a||b| + |u.b||a|) (Frobenius norms): fp32
1e-6 sqrt(n), fp64 1e-13 sqrt(n) -- a length-n fp32 dot carries ~ sqrt(n) 2^-24 relative error."""
import numpy as np
import pytest
import torch

import oracle
import paper_1811_07624_b200 as hh

pytestmark = pytest.mark.gpu


def _case(n, K, dt, seed):
    g = np.random.default_rng(seed)
    A = g.standard_normal((n, n))
    B = g.standard_normal((n, n))
    A, B = (A + A.T) / 2, (B + B.T) / 2
    U = g.standard_normal((K, n))
    U /= np.linalg.norm(U, axis=1, keepdims=True)
    if K > 2:
        U[1] *= 3.0   # not unit: C and grad C are those of the unconstrained function
    npdt = np.float32 if dt == torch.float32 else np.float64
    return A.astype(npdt), B.astype(npdt), U.astype(npdt)


def _check(A, B, U, cost, grad, dt):
    A64, B64, U64 = (x.astype(np.float64) for x in (A, B, U))
    c_ref, g_ref = oracle.shf_cost(A64, B64, U64)
    a, b = U64 @ A64, U64 @ B64          # rows: (A u_k)^T (A symmetric)
    al, be = np.sum(U64 * a, 1), np.sum(U64 * b, 1)
    na, nb = np.linalg.norm(a, axis=1), np.linalg.norm(b, axis=1)
    n = A.shape[0]
    tol = (1e-6 if dt == torch.float32 else 1e-13) * np.sqrt(n)
    s_c = 2 * na * nb + 2 * np.abs(al * be)
    err_c = np.abs(cost.astype(np.float64) - c_ref)
    assert np.all(err_c <= tol * s_c), (n, float(np.max(err_c / s_c)), tol)
    if grad is not None:
        s_g = 2 * (np.linalg.norm(A64) * nb + np.linalg.norm(B64) * na) + 4 * (np.abs(al) * nb + np.abs(be) * na)
        err_g = np.linalg.norm(grad.astype(np.float64) - g_ref, axis=1)
        assert np.all(err_g <= tol * s_g), (n, float(np.max(err_g / s_g)), tol)


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
@pytest.mark.parametrize("n,K", [(1, 3), (37, 5), (64, 64), (129, 65), (500, 300), (1024, 17)])
def test_shf_cost_parity(dt, n, K):
    A, B, U = _case(n, K, dt, 80 + n)
    t = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
    cost, grad = hh.hh_shf_cost(t(A), t(B), t(U))
    assert hh.last_launch_info()["launches"] == 4
    _check(A, B, U, cost.cpu().numpy(), grad.cpu().numpy(), dt)
    cost2, none = hh.hh_shf_cost(t(A), t(B), t(U), grad=False)   # cost only: two launches
    assert none is None and hh.last_launch_info()["launches"] == 2
    assert torch.equal(cost, cost2)


def test_shf_cost_edge_cases():
    A, B, U = _case(16, 4, torch.float32, 9)
    t = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
    cost, grad = hh.hh_shf_cost(t(A), t(B), t(U[:0]))          # K = 0: nothing to do
    assert cost.numel() == 0 and grad.numel() == 0
    with pytest.raises(ValueError):
        hh.hh_shf_cost(t(A), t(B[:8, :8].copy()), t(U))         # shape mismatch
    with pytest.raises(ValueError):
        hh.hh_shf_cost(t(A), t(B), t(U).double())               # dtype mismatch
    # the shared-eigenvector closed form through the GPU path: C(v) = 0, grad = -4ab v
    g = np.random.default_rng(5)
    Qm, _ = np.linalg.qr(g.standard_normal((32, 32)))
    ea, eb = g.standard_normal(32), g.standard_normal(32)
    As, Bs = Qm @ np.diag(ea) @ Qm.T, Qm @ np.diag(eb) @ Qm.T
    As, Bs = (As + As.T) / 2, (Bs + Bs.T) / 2
    c, gr = hh.hh_shf_cost(t(As), t(Bs), t(np.ascontiguousarray(Qm.T)))
    assert np.allclose(c.cpu().numpy(), 0, atol=1e-12)
    assert np.allclose(gr.cpu().numpy(), -4 * (ea * eb)[:, None] * Qm.T, atol=1e-11)
