"""Pins of the fp64 oracle (oracle/hh_ref.c) to things other than itself.

Every test here runs on CPU (no GPU marker).  Each pin is chosen so that a
plausible oracle mistake fails at least one of them:
  * wrong product order / op N vs op T swapped   -> rotation worked example,
    dense brute force, QR reproduction, round trip
  * dropped factor 2, wrong sign of the update    -> H^2 = I, det, norm, closed form
  * transposed operand (u taken from rows of the wrong layout) -> brute force,
    Hadamard / FWHT, QR reproduction
  * lambda / d applied on the wrong side, missing square -> eigvalsh spectrum,
    dense quadratic form, d == 1 Euclidean reduction
Citations: P:L = /root/reference/PAPER.md line L, S:L = SPEC.md line L.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from gen import inputs as gi

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def dense_reflector(u):
    """I - 2 u u^T as an explicit n x n matrix (Eq. 2)."""
    u = np.asarray(u, dtype=np.float64)
    return np.eye(u.size) - 2.0 * np.outer(u, u)


def dense_Q(U):
    """Q = H_1 H_2 ... H_h formed explicitly by dense matrix products."""
    n = U.shape[1]
    Q = np.eye(n)
    for u in U:
        Q = Q @ dense_reflector(u)
    return Q


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def unit_rows(g, h, n):
    U = g.standard_normal((h, n))
    return U / np.linalg.norm(U, axis=1, keepdims=True)


# --------------------------------------------------------------------------- apply
@pytest.mark.parametrize("n,h,N", [(64, 6, 256), (5, 3, 7), (16, 15, 9), (33, 1, 4), (8, 0, 3)])
def test_apply_dense_bruteforce(n, h, N):
    """Brute force: Q formed densely from n x n reflector matrices."""
    g = gi.rng(900, n, h)
    U = unit_rows(g, h, n)
    X = g.standard_normal((N, n))
    Q = dense_Q(U)
    # X is (N, n) == columns; Q X  ->  (Q @ X.T).T
    assert rel(oracle.apply(oracle.OP_N, U, X), (Q @ X.T).T) < 1e-13
    assert rel(oracle.apply(oracle.OP_T, U, X), (Q.T @ X.T).T) < 1e-13


def test_apply_C1_config_bruteforce():
    """BASELINE.json configs[0]: n=64, h=6 fp64 with the dense 64x64 product."""
    c = gi.make_config(1)
    Q = dense_Q(c.U)
    assert rel(oracle.apply(oracle.OP_N, c.U, c.X), (Q @ c.X.T).T) < 1e-13
    assert rel(oracle.apply(oracle.OP_T, c.U, c.X), (Q.T @ c.X.T).T) < 1e-13


def test_rotation_worked_example_pins_order():
    """P:130 (||U - U_2 U_1||), P:158, P:172-175 Case 2 formulas: R(2pi/3) = U_2 U_1."""
    gold = json.load(open(os.path.join(GOLD, "rotation_2pi3.json")))
    th = gold["theta"]
    R = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
    assert np.allclose(R, np.array(gold["R"]), atol=1e-15)
    # eigenvector of R for lambda = alpha + i beta, recomputed by the paper's formulas
    alpha = math.cos(th)
    t = np.array([1.0, -1.0j]) / math.sqrt(2.0)
    assert np.allclose(R @ t, (math.cos(th) + 1j * math.sin(th)) * t)
    u1 = math.sqrt(2.0) * t.real
    gam, dlt = -math.sqrt(1 + alpha) / 2, -math.sqrt(1 - alpha) / 2
    u2 = 2.0 * (gam * t.real - dlt * t.imag)
    assert np.allclose(u1, gold["u1"], atol=1e-15)
    assert np.allclose(u2, gold["u2"], atol=1e-15)
    X = gi.rng(901).standard_normal((5, 2))
    want = (R @ X.T).T
    # paper order U_2 U_1 == our Q^T with columns [u1, u2] == our Q with columns [u2, u1]
    assert np.abs(oracle.apply(oracle.OP_T, np.array([u1, u2]), X) - want).max() < 1e-15
    assert np.abs(oracle.apply(oracle.OP_N, np.array([u2, u1]), X) - want).max() < 1e-15
    # the reversed order must NOT reproduce R (the pin discriminates the order)
    assert np.abs(oracle.apply(oracle.OP_N, np.array([u1, u2]), X) - want).max() > 0.5


def test_reflector_involution_and_symmetry():
    """H^2 = I (P:52 orthonormal + symmetric, P:235 J^T = J) with fp64-normalised u."""
    g = gi.rng(902)
    n = 37
    u = unit_rows(g, 1, n)
    X = g.standard_normal((11, n))
    UU = np.vstack([u, u])
    assert np.abs(oracle.apply(oracle.OP_N, UU, X) - X).max() < 1e-14
    # symmetry: op N and op T of a single reflector coincide exactly
    assert np.array_equal(oracle.apply(oracle.OP_N, u, X), oracle.apply(oracle.OP_T, u, X))
    # H applied to e_j columns is the symmetric dense H
    Hcols = oracle.apply(oracle.OP_N, u, np.eye(n))
    assert np.abs(Hcols - Hcols.T).max() < 1e-15
    assert np.abs(Hcols - dense_reflector(u[0])).max() < 1e-15


@pytest.mark.parametrize("n,h", [(50, 7), (128, 20)])
def test_norm_and_round_trip(n, h):
    """||Qx|| = ||x|| and Q^T(QX) = X (P:52 orthonormality)."""
    g = gi.rng(903, n, h)
    U = unit_rows(g, h, n)
    X = g.standard_normal((40, n))
    Y = oracle.apply(oracle.OP_N, U, X)
    assert np.abs(np.linalg.norm(Y, axis=1) / np.linalg.norm(X, axis=1) - 1).max() < 1e-14
    assert rel(oracle.apply(oracle.OP_T, U, Y), X) < 1e-14
    assert rel(oracle.apply(oracle.OP_N, U, oracle.apply(oracle.OP_T, U, X)), X) < 1e-14


@pytest.mark.parametrize("h", [0, 1, 2, 3, 5, 8])
def test_determinant(h):
    """det(prod U_k) = (-1)^h."""
    n = 8
    U = unit_rows(gi.rng(904, h), h, n)
    Q = oracle.apply(oracle.OP_N, U, np.eye(n)).T  # columns Q e_j
    assert abs(np.linalg.det(Q) - (-1) ** h) < 1e-12


def householder_qr_reflectors(A):
    """Textbook Householder QR (Golub & Van Loan 5.2.1, cited at P:218-222): returns the
    n-1 unit reflector vectors j_k (k-1 leading zeros) and R with
    J_{n-1} ... J_1 A = R.  Written here in the test, independent of the oracle."""
    A = np.array(A, dtype=np.float64)
    n = A.shape[0]
    J = np.zeros((n - 1, n))
    for k in range(n - 1):
        x = A[k:, k]
        v = x.copy()
        s = 1.0 if x[0] >= 0 else -1.0
        v[0] += s * np.linalg.norm(x)
        nv = np.linalg.norm(v)
        if nv == 0.0:
            continue                       # u = 0 identity slot
        v /= nv
        J[k, k:] = v
        A[k:, :] -= 2.0 * np.outer(v, v @ A[k:, :])
    return J, A


@pytest.mark.parametrize("n", [16, 64])
def test_qr_reflectors_reproduce_orthonormal(n):
    """n-1 reflectors + a +-1 diagonal reproduce any orthonormal U:
    U = J_1 ... J_{n-1} D with D = diag(R)."""
    G = gi.rng(905, n).standard_normal((n, n))
    U0, _ = np.linalg.qr(G)             # random orthonormal via QR of a Gaussian
    J, R = householder_qr_reflectors(U0)
    D = np.diag(np.diag(R))
    assert np.abs(np.abs(np.diag(R)) - 1).max() < 1e-13
    assert np.abs(R - D).max() < 1e-13
    # columns of Q D: apply op N to the columns of D (D is symmetric -> rows == columns)
    QD = oracle.apply(oracle.OP_N, J, D).T
    assert np.abs(QD - U0).max() < 1e-13
    # and Q^T U0 == D
    assert np.abs(oracle.apply(oracle.OP_T, J, U0.T).T - D).max() < 1e-13


def sylvester(n):
    H = np.array([[1.0]])
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H


def fwht(X):
    """Textbook fast Walsh-Hadamard transform along the last axis (unnormalised)."""
    X = np.array(X, dtype=np.float64)
    n = X.shape[-1]
    hlen = 1
    while hlen < n:
        Y = X.reshape(*X.shape[:-1], n // (2 * hlen), 2, hlen)
        a, b = Y[..., 0, :].copy(), Y[..., 1, :].copy()
        Y[..., 0, :], Y[..., 1, :] = a + b, a - b
        X = Y.reshape(*X.shape[:-1], n)
        hlen *= 2
    return X


def test_hadamard_exact_with_half_reflectors():
    """P:546 (golden): H/sqrt(n) + its transpose has n/2 eigenvalues -2 and n/2 at +2, so the
    n/2 orthonormal vectors of the -1 eigenspace give H/sqrt(n) = I - 2 W W^T exactly
    (Result 1).  Compared against an independent O(n log n) FWHT."""
    gold = json.load(open(os.path.join(GOLD, "hadamard_p546.json")))
    for case in gold["cases"]:
        n = case["n"]
        Hn = sylvester(n) / math.sqrt(n)
        z = np.linalg.eigvalsh(Hn + Hn.T)
        assert int(np.sum(np.abs(z + 2) < 1e-9)) == case["count_minus2"]
        assert int(np.sum(np.abs(z - 2) < 1e-9)) == case["count_plus2"]
        w, V = np.linalg.eigh(Hn)
        W = V[:, w < 0].T                    # (n/2, n) orthonormal rows
        assert W.shape[0] == case["count_minus2"]
        X = gi.rng(906, n).standard_normal((9, n))
        want = fwht(X) / math.sqrt(n)
        for op in (oracle.OP_N, oracle.OP_T):
            assert rel(oracle.apply(op, W, X), want) < 1e-13


def test_orthonormal_closed_form_and_order_independence():
    """Orthonormal u's: prod (I - 2 u_k u_k^T) = I - 2 W W^T."""
    n, h = 96, 12
    W, _ = np.linalg.qr(gi.rng(907).standard_normal((n, h)))
    W = W.T
    X = gi.rng(908).standard_normal((17, n))
    want = X - 2.0 * (X @ W.T) @ W
    assert rel(oracle.apply(oracle.OP_N, W, X), want) < 1e-14
    assert rel(oracle.apply(oracle.OP_T, W, X), want) < 1e-14
    perm = gi.rng(909).permutation(h)
    assert rel(oracle.apply(oracle.OP_N, W[perm], X), want) < 1e-14


def test_trivial_cases():
    """h = 0 -> X; u = e_1 flips coordinate 1; u = 0 -> identity slot."""
    g = gi.rng(910)
    n = 12
    X = g.standard_normal((6, n))
    assert np.array_equal(oracle.apply(oracle.OP_N, np.zeros((0, n)), X), X)
    e1 = np.zeros((1, n)); e1[0, 0] = 1.0
    Y = oracle.apply(oracle.OP_N, e1, X)
    assert np.array_equal(Y[:, 0], -X[:, 0]) and np.array_equal(Y[:, 1:], X[:, 1:])
    assert np.array_equal(oracle.apply(oracle.OP_T, np.zeros((3, n)), X), X)
    # a zero slot between real reflectors changes nothing
    U = unit_rows(g, 2, n)
    U3 = np.vstack([U[0], np.zeros(n), U[1]])
    assert np.array_equal(oracle.apply(oracle.OP_N, U3, X), oracle.apply(oracle.OP_N, U, X))


def test_linearity():
    """apply(a x + b y) = a apply(x) + b apply(y)."""
    g = gi.rng(911)
    n, h = 40, 9
    U = unit_rows(g, h, n)
    x, y = g.standard_normal((2, 5, n))
    a, b = 1.7, -0.3
    lhs = oracle.apply(oracle.OP_N, U, a * x + b * y)
    rhs = a * oracle.apply(oracle.OP_N, U, x) + b * oracle.apply(oracle.OP_N, U, y)
    assert rel(lhs, rhs) < 1e-14


def test_fp32_inputs_are_used_literally():
    """Reading R5: fp32 bytes are widened exactly, never renormalised: with a deliberately
    non-unit u the oracle still computes x - 2(u^T x)u, which is not orthogonal."""
    n = 8
    u = np.full((1, n), 0.5, dtype=np.float32)   # ||u||^2 = 2
    x = np.ones((1, n), dtype=np.float32)
    y = oracle.apply(oracle.OP_N, u, x)
    assert np.allclose(y, 1.0 - 2.0 * 4.0 * 0.5)


# --------------------------------------------------------------------------- symmetric
@pytest.mark.parametrize("n,h", [(16, 4), (64, 10), (7, 0)])
def test_sym_dense_bruteforce(n, h):
    """S = Q diag(lambda) Q^T formed densely (eq:thesbar)."""
    g = gi.rng(920, n, h)
    U = unit_rows(g, h, n)
    lam = g.standard_normal(n)
    X = g.standard_normal((13, n))
    Q = dense_Q(U)
    S = Q @ np.diag(lam) @ Q.T
    assert rel(oracle.sym_apply(U, lam, X), (S @ X.T).T) < 1e-13


def test_sym_spectrum_is_lambda():
    """Orthonormal congruence preserves the spectrum: eigvalsh(S) = sort(lambda)."""
    n, h = 48, 11
    g = gi.rng(921)
    U = unit_rows(g, h, n)
    lam = gi.c3_spectrum(g, n)
    S = oracle.sym_apply(U, lam, np.eye(n)).T
    assert np.abs(S - S.T).max() < 1e-15
    ev = np.linalg.eigvalsh(0.5 * (S + S.T))
    assert np.abs(ev - np.sort(lam)).max() < 1e-12 * np.abs(lam).max()


def test_sym_trivial():
    """lambda == 1 -> X; h = 0 -> lambda * X."""
    g = gi.rng(922)
    n = 20
    U = unit_rows(g, 5, n)
    X = g.standard_normal((4, n))
    assert rel(oracle.sym_apply(U, np.ones(n), X), X) < 1e-14
    lam = g.standard_normal(n)
    assert np.array_equal(oracle.sym_apply(np.zeros((0, n)), lam, X), X * lam)


# --------------------------------------------------------------------------- Mahalanobis
def _pairs(g, M, P):
    return g.integers(0, M, P).astype(np.int32), g.integers(0, M, P).astype(np.int32)


def test_mahalanobis_dense_quadratic_form():
    """d_S(x_a, x_b) = (x_a - x_b)^T S (x_a - x_b), S = Q diag(d) Q^T (R4)."""
    g = gi.rng(930)
    n, h, M, P = 32, 5, 50, 200
    U = unit_rows(g, h, n)
    d = g.uniform(0.1, 10.0, n)
    pts = g.standard_normal((M, n))
    ia, ib = _pairs(g, M, P)
    Q = dense_Q(U)
    S = Q @ np.diag(d) @ Q.T
    diff = pts[ia] - pts[ib]
    want = np.einsum("pi,ij,pj->p", diff, S, diff)
    got = oracle.mahalanobis(U, d, pts, ia, ib)
    assert rel(got, want) < 1e-13
    # L = sqrt(Lambda) U with U == Q^T: ||L (x_a - x_b)||^2
    L = np.diag(np.sqrt(d)) @ Q.T
    assert rel(got, np.sum((diff @ L.T) ** 2, axis=1)) < 1e-13


def test_mahalanobis_invariants():
    """a = b -> 0 exactly; symmetry; d == 1 -> Euclidean (orthogonal invariance);
    h = 0 -> sum d_r diff_r^2."""
    g = gi.rng(931)
    n, h, M = 24, 6, 30
    U = unit_rows(g, h, n)
    d = g.uniform(0.1, 10.0, n)
    pts = g.standard_normal((M, n))
    ia, ib = _pairs(g, M, 100)
    ia[:5] = ib[:5]
    got = oracle.mahalanobis(U, d, pts, ia, ib)
    assert np.all(got[:5] == 0.0)
    assert np.array_equal(got, oracle.mahalanobis(U, d, pts, ib, ia))
    diff = pts[ia] - pts[ib]
    e = oracle.mahalanobis(U, np.ones(n), pts, ia, ib)
    assert np.abs(e - np.sum(diff ** 2, axis=1)).max() < 1e-13 * np.sum(diff ** 2, axis=1).max()
    z = oracle.mahalanobis(np.zeros((0, n)), d, pts, ia, ib)
    assert rel(z, np.sum(d * diff ** 2, axis=1)) < 1e-15


def test_mahalanobis_rejects_bad_index():
    g = gi.rng(932)
    with pytest.raises(ValueError):
        oracle.mahalanobis(unit_rows(g, 1, 4), np.ones(4), g.standard_normal((3, 4)),
                           np.array([0], np.int32), np.array([3], np.int32))


def test_threads_control():
    t = oracle.num_threads()
    assert t >= 1
    oracle.set_threads(1)
    assert oracle.num_threads() == 1
    oracle.set_threads(t)



# --------------------------------------------------------------------------- NEXT-f1: D
@pytest.mark.parametrize("n,h", [(6, 3), (16, 9), (64, 6)])
def test_signed_dense_bruteforce(n, h):
    """Ubar = D U_h...U_1 (Eq. 1) and Ubar_2 D (Result 3) against the
    explicit dense products, both ops; S-bar = D Q Lambda Q^T D (eq:thesbar)."""
    g = gi.rng(905, n, h)
    U = unit_rows(g, h, n)
    X = g.standard_normal((7, n))
    d = gi.sign_diag(g, n)
    D = np.diag(d)
    Q = dense_Q(U)
    for op, Qop in ((0, Q), (1, Q.T)):
        assert rel(oracle.apply_signed(op, 0, U, d, X), (D @ Qop @ X.T).T) < 1e-13
        assert rel(oracle.apply_signed(op, 1, U, d, X), (Qop @ D @ X.T).T) < 1e-13
    lam = g.standard_normal(n)
    S = D @ Q @ np.diag(lam) @ Q.T @ D
    assert rel(oracle.sym_apply_signed(U, d, lam, X), (S @ X.T).T) < 1e-13


def test_signed_determinant_and_identity():
    """det(D U_h...U_1) = det(D) (-1)^h ("we use the diagonal D to ensure that the
    choice of h does not fix the determinant"); D = I reduces to the unsigned apply; the
    symmetric form keeps the spectrum (D orthonormal)."""
    n, h = 8, 3
    g = gi.rng(906)
    U = unit_rows(g, h, n)
    d = np.array([1, -1, 1, 1, -1, 1, 1, -1], dtype=np.float64)
    M = oracle.apply_signed(1, 0, U, d, np.eye(n)).T        # columns = images of e_i
    assert abs(np.linalg.det(M) - np.prod(d) * (-1) ** h) < 1e-12
    X = g.standard_normal((5, n))
    ones = np.ones(n)
    for op in (0, 1):
        for side in (0, 1):
            assert np.array_equal(oracle.apply_signed(op, side, U, ones, X), oracle.apply(op, U, X))
    lam = g.standard_normal(n)
    S = oracle.sym_apply_signed(U, d, lam, np.eye(n)).T
    assert np.allclose(np.linalg.eigvalsh((S + S.T) / 2), np.sort(lam), atol=1e-13)



# --------------------------------------------------------------------------- NEXT-f3: kNN
def test_knn_bruteforce_and_invariants():
    """k-NN under d_S: against the dense quadratic form (x_q - x_r)^T
    Q diag(d) Q^T (x_q - x_r) with numpy argsort (stable: ties by index); a query equal to
    a reference finds it at distance 0; d == 1 with orthonormal Q reduces to Euclidean
    k-NN (orthogonal invariance)."""
    g = gi.rng(907)
    n, h, Mr, Mq, k = 12, 4, 40, 9, 5
    U = unit_rows(g, h, n)
    d = g.uniform(0.1, 10.0, n)
    Pr = g.standard_normal((Mr, n))
    Pq = g.standard_normal((Mq, n))
    Pq[3] = Pr[17]
    Q = dense_Q(U)
    S = Q @ np.diag(d) @ Q.T
    idx, dist = oracle.knn(U, d, Pr, Pq, k)
    for q in range(Mq):
        diff = Pq[q] - Pr
        dd = np.einsum("ij,jk,ik->i", diff, S, diff)
        order = np.argsort(dd, kind="stable")[:k]
        assert np.array_equal(idx[q], order)
        assert np.allclose(dist[q], dd[order], rtol=1e-12, atol=1e-12)
    assert idx[3, 0] == 17 and dist[3, 0] == 0.0
    ie, de = oracle.knn(U, np.ones(n), Pr, Pq, k)
    for q in range(Mq):
        e = ((Pq[q] - Pr) ** 2).sum(1)
        assert np.array_equal(ie[q], np.argsort(e, kind="stable")[:k])


def test_knn_exact_ties_smaller_index_first():
    """Reading R14 (hh.h: "ascending, ties by the smaller reference index"): duplicated
    references give bit-identical distances, so the order among them is fixed by index
    alone -- inside the returned list and at the k-th place.  References 4, 17 and 31 are
    one point and 9, 25 another; a query next to point 4 must return [4, 17] for k = 2 (31
    ties with 17 at the cut: the earlier index is kept) and [4, 17, 31] for k = 3, and a
    query next to point 9 must return 9 before 25.  Expected orders come from the dense
    quadratic form with numpy's stable sort, not from the oracle."""
    g = gi.rng(909)
    n, h, Mr = 16, 5, 40
    U = unit_rows(g, h, n)
    d = g.uniform(0.1, 10.0, n)
    Pr = g.standard_normal((Mr, n))
    Pr[17] = Pr[4]
    Pr[31] = Pr[4]
    Pr[25] = Pr[9]
    Pq = np.vstack([Pr[4] + 1e-3 * g.standard_normal(n), Pr[9] + 1e-3 * g.standard_normal(n),
                    Pr[4].copy()])
    Q = dense_Q(U)
    S = Q @ np.diag(d) @ Q.T
    for k in (2, 3, 4):
        idx, dist = oracle.knn(U, d, Pr, Pq, k)
        for q in range(Pq.shape[0]):
            diff = Pq[q] - Pr
            dd = np.einsum("ij,jk,ik->i", diff, S, diff)
            dd[[17, 31]] = dd[4]                 # identical inputs: identical distances
            dd[25] = dd[9]
            assert np.array_equal(idx[q], np.argsort(dd, kind="stable")[:k]), (k, q, idx[q])
        assert list(idx[0, :2]) == [4, 17] and list(idx[1, :2]) == [9, 25]
        assert dist[0, 0] == dist[0, 1]
        if k >= 3:
            assert idx[0, 2] == 31 and list(idx[2, :3]) == [4, 17, 31]
            assert dist[2, 0] == dist[2, 1] == dist[2, 2] == 0.0



# --------------------------------------------------------------------------- NEXT-f4
def test_congruence_dense_and_shf_identity():
    """op(Q) M op(Q)^T against the dense product; and the SHF identity
    eq:symmetricWithHouseholder with D = I:
        ||S - Q diag(s) Q^T||_F = ||A_k - U_k B_k U_k||_F,
    A_k = (U_{k-1}..U_1) S (U_1..U_{k-1}) = congruence(op T, u_1..u_{k-1}, S),
    B_k = (U_{k+1}..U_h) diag(s) (U_h..U_{k+1}) = congruence(op N, u_{k+1}..u_h, diag(s))."""
    g = gi.rng(908)
    n, h = 10, 6
    U = unit_rows(g, h, n)
    M = g.standard_normal((3, n, n))            # storage: column-major (math matrix = M[b].T)
    Q = dense_Q(U)
    for op, Qop in ((0, Q), (1, Q.T)):
        out = oracle.congruence(op, U, M)
        for b in range(3):
            assert rel(out[b].T, Qop @ M[b].T @ Qop.T) < 1e-13
    A = g.standard_normal((n, n))
    S = A + A.T
    s = g.standard_normal(n)
    Sbar = Q @ np.diag(s) @ Q.T
    for k in range(1, h + 1):                   # 1-based k as in the paper
        Ak = oracle.congruence(1, U[:k - 1], S[None])[0].T
        Bk = oracle.congruence(0, U[k:], np.diag(s)[None])[0].T
        Hk = dense_reflector(U[k - 1])
        lhs = np.linalg.norm(S - Sbar)
        rhs = np.linalg.norm(Ak - Hk @ Bk @ Hk)
        assert abs(lhs - rhs) < 1e-12 * max(1.0, lhs)


# ---------------------------------------------------------------- NEXT-f4: C(u), grad C(u)
def _sym_pair(g, n):
    A = g.standard_normal((n, n))
    B = g.standard_normal((n, n))
    return A + A.T, B + B.T


def test_shf_cost_objective_identity():
    """eq:objectivefunctionS3: for unit u and H = I - 2 u u^T,
    ||A - H B H||_F^2 = ||A||_F^2 + ||B||_F^2 - 2 tr(A B) + 4 C(u) -- the paper's own expansion,
    computed densely here; a wrong sign, factor or dropped term of C fails it."""
    g = np.random.default_rng(71)
    for n in (3, 8, 33):
        A, B = _sym_pair(g, n)
        U = g.standard_normal((6, n))
        U /= np.linalg.norm(U, axis=1, keepdims=True)
        cost, _ = oracle.shf_cost(A, B, U, grad=False)
        for k, u in enumerate(U):
            H = dense_reflector(u)
            lhs = np.linalg.norm(A - H @ B @ H) ** 2
            rhs = np.linalg.norm(A) ** 2 + np.linalg.norm(B) ** 2 - 2 * np.trace(A @ B) + 4 * cost[k]
            assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs)), (n, k, lhs, rhs)


def test_shf_gradient_finite_differences():
    """eq:gradient against central differences of the oracle's own C (fp64),
    for arbitrary (not unit) u: the gradient formula is that of the unconstrained C."""
    g = np.random.default_rng(72)
    n = 11
    A, B = _sym_pair(g, n)
    U = g.standard_normal((4, n))
    _, G = oracle.shf_cost(A, B, U)
    eps = 1e-6
    for k in range(U.shape[0]):
        fd = np.empty(n)
        for i in range(n):
            up, um = U[k].copy(), U[k].copy()
            up[i] += eps
            um[i] -= eps
            fd[i] = (oracle.shf_cost(A, B, up[None], grad=False)[0][0] -
                     oracle.shf_cost(A, B, um[None], grad=False)[0][0]) / (2 * eps)
        assert np.allclose(G[k], fd, rtol=1e-6, atol=1e-6 * np.abs(G[k]).max()), (k, G[k], fd)


def test_shf_cost_shared_eigenvector():
    """Closed form: if A v = a v and B v = b v (unit v) then C(v) = 2ab - 2ab = 0 and
    grad C(v) = 4ab v - 8ab v = -4ab v (eq:theRk, eq:gradient)."""
    g = np.random.default_rng(73)
    n = 9
    Qm, _ = np.linalg.qr(g.standard_normal((n, n)))
    ea, eb = g.standard_normal(n), g.standard_normal(n)
    A = Qm @ np.diag(ea) @ Qm.T
    B = Qm @ np.diag(eb) @ Qm.T
    A, B = (A + A.T) / 2, (B + B.T) / 2
    cost, G = oracle.shf_cost(A, B, Qm.T)
    for k in range(n):
        assert abs(cost[k]) < 1e-12 * (1 + abs(ea[k] * eb[k])), (k, cost[k])
        assert np.allclose(G[k], -4 * ea[k] * eb[k] * Qm[:, k], atol=1e-11), k


def test_shf_cost_swap_and_scale():
    """C is symmetric in (A, B); C(u; sA, B) = s C(u; A, B) (both terms are linear in A)."""
    g = np.random.default_rng(74)
    n = 7
    A, B = _sym_pair(g, n)
    U = g.standard_normal((5, n))
    c1, g1 = oracle.shf_cost(A, B, U)
    c2, g2 = oracle.shf_cost(B, A, U)
    c3, g3 = oracle.shf_cost(2.5 * A, B, U)
    assert np.allclose(c1, c2, rtol=1e-12, atol=1e-12) and np.allclose(g1, g2, rtol=1e-12, atol=1e-11)
    assert np.allclose(c3, 2.5 * c1, rtol=1e-12, atol=1e-11) and np.allclose(g3, 2.5 * g1, rtol=1e-12, atol=1e-10)
