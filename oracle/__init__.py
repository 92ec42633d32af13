"""fp64 CPU oracle for the Householder-product apply path (ctypes over hh_ref.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  The product
package `paper_1811_07624_b200` never imports it.

Inputs may be fp32 or fp64; fp32 values are converted exactly to fp64 (reading
R5: the same bytes the GPU receives, never renormalised) and all arithmetic is
strict fp64 in hh_ref.c.  Outputs are fp64 numpy arrays.

Layout: U is (h, n) row-major == n x h column-major; X is (N, n) row-major ==
n x N column-major.  See hh_ref.c for the paper citations of each function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hh_ref.c")
_LIB = os.path.join(_HERE, "libhh_ref.so")
CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-std=c11", "-Wall", "-Wextra",
          "-fPIC", "-shared"]

OP_N, OP_T = 0, 1


def build(force: bool = False) -> str:
    """Compile hh_ref.c -> libhh_ref.so (gcc, strict fp64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64, p, i32 = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        L.hh_ref_apply.argtypes = [i32, i64, i64, p, p, p, i64]
        L.hh_ref_sym_apply.argtypes = [i64, i64, p, p, p, p, i64]
        L.hh_ref_mahalanobis.argtypes = [i64, i64, p, p, p, i64, p, p, i64, p]
        for f in (L.hh_ref_apply, L.hh_ref_sym_apply, L.hh_ref_mahalanobis):
            f.restype = i32
        L.hh_ref_apply_signed.argtypes = [i32, i32, i64, i64, p, p, p, p, i64]
        L.hh_ref_sym_apply_signed.argtypes = [i64, i64, p, p, p, p, p, i64]
        L.hh_ref_apply_signed.restype = i32
        L.hh_ref_knn.argtypes = [i64, i64, p, p, p, i64, p, i64, i32, p, p]
        L.hh_ref_knn.restype = i32
        L.hh_ref_congruence.argtypes = [i32, i64, i64, p, p, p, i64]
        L.hh_ref_congruence.restype = i32
        L.hh_ref_shf_cost.argtypes = [i64, p, p, p, i64, p, p]
        L.hh_ref_shf_cost.restype = i32
        L.hh_ref_sym_apply_signed.restype = i32
        L.hh_ref_num_threads.restype = i32
        L.hh_ref_set_threads.argtypes = [i32]
        _lib = L
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(t: int) -> None:
    lib().hh_ref_set_threads(int(t))


def num_threads() -> int:
    return int(lib().hh_ref_num_threads())


def apply(op: int, U, X) -> np.ndarray:
    """Y = Q X (op 0) or Q^T X (op 1), Q = H_1 ... H_h (hh_ref.c: hh_ref_apply)."""
    U = _f64(U).reshape(-1, np.shape(X)[-1]) if np.size(U) else np.zeros((0, np.shape(X)[-1]))
    X = _f64(X)
    h, n = U.shape
    N = X.shape[0]
    Y = np.empty_like(X)
    rc = lib().hh_ref_apply(int(op), n, h, _ptr(U), _ptr(X), _ptr(Y), N)
    if rc:
        raise ValueError(f"hh_ref_apply rc={rc}")
    return Y


def sym_apply(U, lam, X) -> np.ndarray:
    """Y = Q diag(lam) Q^T X (hh_ref.c: hh_ref_sym_apply)."""
    X = _f64(X)
    n = X.shape[-1]
    U = _f64(U).reshape(-1, n)
    lam = _f64(lam)
    Y = np.empty_like(X)
    rc = lib().hh_ref_sym_apply(n, U.shape[0], _ptr(U), _ptr(lam), _ptr(X), _ptr(Y), X.shape[0])
    if rc:
        raise ValueError(f"hh_ref_sym_apply rc={rc}")
    return Y


def mahalanobis(U, d, P, ia, ib) -> np.ndarray:
    """dist[j] = ||D^1/2 Q^T (P[ia[j]] - P[ib[j]])||^2 (hh_ref.c: hh_ref_mahalanobis)."""
    P = _f64(P)
    n = P.shape[-1]
    U = _f64(U).reshape(-1, n)
    d = _f64(d)
    ia = np.ascontiguousarray(ia, dtype=np.int32)
    ib = np.ascontiguousarray(ib, dtype=np.int32)
    dist = np.empty(ia.shape[0], dtype=np.float64)
    rc = lib().hh_ref_mahalanobis(n, U.shape[0], _ptr(U), _ptr(d), _ptr(P), P.shape[0],
                                  _ptr(ia), _ptr(ib), ia.shape[0], _ptr(dist))
    if rc:
        raise ValueError(f"hh_ref_mahalanobis rc={rc}")
    return dist


def apply_signed(op: int, side: int, U, d, X) -> np.ndarray:
    """side 0: Y = D op(Q) X (Eq. 1); side 1: Y = op(Q) D X (Result 3)
    (hh_ref.c: hh_ref_apply_signed, NEXT-f1)."""
    X = _f64(X)
    n = X.shape[-1]
    U = _f64(U).reshape(-1, n) if np.size(U) else np.zeros((0, n))
    d = _f64(d)
    Y = np.empty_like(X)
    rc = lib().hh_ref_apply_signed(int(op), int(side), n, U.shape[0], _ptr(U), _ptr(d), _ptr(X),
                                   _ptr(Y), X.shape[0])
    if rc:
        raise ValueError(f"hh_ref_apply_signed rc={rc}")
    return Y


def sym_apply_signed(U, d, lam, X) -> np.ndarray:
    """Y = D Q diag(lam) Q^T D X (hh_ref.c: hh_ref_sym_apply_signed, NEXT-f1)."""
    X = _f64(X)
    n = X.shape[-1]
    U = _f64(U).reshape(-1, n)
    d, lam = _f64(d), _f64(lam)
    Y = np.empty_like(X)
    rc = lib().hh_ref_sym_apply_signed(n, U.shape[0], _ptr(U), _ptr(d), _ptr(lam), _ptr(X),
                                       _ptr(Y), X.shape[0])
    if rc:
        raise ValueError(f"hh_ref_sym_apply_signed rc={rc}")
    return Y


def knn(U, d, P_ref, P_query, k: int):
    """(idx int32 (Mq, k), dist fp64 (Mq, k)): the k smallest d_S(q, r), ascending by
    (distance, reference index) (hh_ref.c: hh_ref_knn, NEXT-f3)."""
    Pr, Pq = _f64(P_ref), _f64(P_query)
    n = Pr.shape[-1]
    U = _f64(U).reshape(-1, n) if np.size(U) else np.zeros((0, n))
    d = _f64(d)
    Mq = Pq.shape[0]
    idx = np.empty((Mq, k), dtype=np.int32)
    dist = np.empty((Mq, k), dtype=np.float64)
    rc = lib().hh_ref_knn(n, U.shape[0], _ptr(U), _ptr(d), _ptr(Pr), Pr.shape[0], _ptr(Pq), Mq,
                          int(k), _ptr(idx), _ptr(dist))
    if rc:
        raise ValueError(f"hh_ref_knn rc={rc}")
    return idx, dist


def congruence(op: int, U, M) -> np.ndarray:
    """op(Q) M_b op(Q)^T for M of shape (count, n, n) holding column-major matrices, i.e.
    M[b] is the TRANSPOSE of the math matrix (hh_ref.c: hh_ref_congruence, NEXT-f4)."""
    M = _f64(M)
    count, n, _ = M.shape
    U = _f64(U).reshape(-1, n) if np.size(U) else np.zeros((0, n))
    out = np.empty_like(M)
    rc = lib().hh_ref_congruence(int(op), n, U.shape[0], _ptr(U), _ptr(M), _ptr(out), count)
    if rc:
        raise ValueError(f"hh_ref_congruence rc={rc}")
    return out


def shf_cost(A, B, Uc, grad: bool = True):
    """(cost (K,), grad (K, n) or None): the SHF objective C(u_k) of one reflector and its
    gradient for candidates Uc of shape (K, n) (hh_ref.c: hh_ref_shf_cost, eq:theRk,
    eq:gradient, NEXT-f4).  A, B: symmetric (n, n)."""
    A, B, Uc = _f64(A), _f64(B), _f64(Uc)
    n = A.shape[0]
    Uc = Uc.reshape(-1, n) if np.size(Uc) else np.zeros((0, n))
    K = Uc.shape[0]
    cost = np.empty(K, dtype=np.float64)
    g = np.empty((K, n), dtype=np.float64) if grad else None
    rc = lib().hh_ref_shf_cost(n, _ptr(A), _ptr(B), _ptr(Uc), K, _ptr(cost),
                               _ptr(g) if grad else None)
    if rc:
        raise ValueError(f"hh_ref_shf_cost rc={rc}")
    return cost, g
