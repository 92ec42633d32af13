"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module draws numbers only.  It holds none of the method's arithmetic (no
reflector application, no dot products, no distances): both `oracle/` and the
CUDA path receive the bytes it produces, so parity compares two independent
computations on provably identical inputs.

Recipes follow BASELINE.json `configs` and SURVEY.md §8(d):
  * reflector vectors u_i ~ iid N(0,1), each normalised to unit l2 norm in fp64
    and then cast (Eq. 2 "||u_k||_2 = 1");
  * X ~ iid N(0,1), column-major n x N  ==  a C-contiguous (N, n) array;
  * C3 spectrum lambda_k = exp(-k/200), with exactly round(0.1 n) signs flipped;
  * C4 metric diagonal d ~ U[0.1, 10], index pairs uniform with replacement.
Draws are always made in float64 and cast, because NumPy's float32 sampler is a
different stream.  The seed key is SeedSequence([181107624, cfg, ..., stream]).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

SEED_ROOT = 181107624

# stream ids
S_U, S_X, S_FLIP, S_D, S_IA, S_IB = 0, 1, 2, 3, 4, 5


def rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_ROOT, *key])))


def np_dtype(dtype: str):
    return {"f32": np.float32, "f64": np.float64}[dtype]


def unit_reflectors(g: np.random.Generator, h: int, n: int, dtype: str = "f64",
                    zero_slots=()) -> np.ndarray:
    """(h, n) array whose row i is u_{i+1} (== n x h column-major U).

    Rows listed in `zero_slots` are set to 0: the identity slot u_k = 0 of
    PAPER.md l.90 ("we set u_k = 0 ... U_k = I").
    """
    u = g.standard_normal((h, n))
    if h:
        u /= np.sqrt((u * u).sum(axis=1, keepdims=True))
    for k in zero_slots:
        u[k] = 0.0
    return np.ascontiguousarray(u.astype(np_dtype(dtype)))


def gaussian_columns(g: np.random.Generator, N: int, n: int, dtype: str = "f64") -> np.ndarray:
    """(N, n) C-contiguous array == column-major n x N matrix of iid N(0,1)."""
    if dtype == "f64":
        return g.standard_normal((N, n))
    out = np.empty((N, n), dtype=np_dtype(dtype))
    # chunked so the transient float64 buffer stays small at 1 GiB sizes
    step = max(1, (1 << 24) // max(n, 1))
    for j in range(0, N, step):
        out[j:j + step] = g.standard_normal((min(step, N - j), n))
    return out


def c3_spectrum(g: np.random.Generator, n: int, dtype: str = "f64", frac: float = 0.1) -> np.ndarray:
    """lambda_k = exp(-k/200), k=0..n-1, with exactly round(frac*n) random sign flips
    (BASELINE.json configs[2]; reading R7)."""
    lam = np.exp(-np.arange(n, dtype=np.float64) / 200.0)
    idx = g.choice(n, int(round(frac * n)), replace=False)
    lam[idx] = -lam[idx]
    return lam.astype(np_dtype(dtype))


def sign_diag(g: np.random.Generator, n: int, dtype: str = "f64") -> np.ndarray:
    """d in {+-1}^n, each sign fair (the diagonal D of Eq. 1)."""
    return np.where(g.random(n) < 0.5, -1.0, 1.0).astype(np_dtype(dtype))


def metric_diag(g: np.random.Generator, n: int, dtype: str = "f64") -> np.ndarray:
    return g.uniform(0.1, 10.0, n).astype(np_dtype(dtype))


def index_pairs(ga: np.random.Generator, gb: np.random.Generator, M: int, P: int):
    ia = ga.integers(0, M, P, dtype=np.int32)
    ib = gb.integers(0, M, P, dtype=np.int32)
    return ia, ib


# ----------------------------------------------------------------------------------
# BASELINE.json configurations
# ----------------------------------------------------------------------------------

@dataclasses.dataclass
class Case:
    name: str
    call: str                 # "apply" | "sym" | "mahalanobis"
    n: int
    h: int
    N: int                    # columns (apply/sym) or points M (mahalanobis)
    dtype: str
    U: np.ndarray
    X: np.ndarray
    lam: Optional[np.ndarray] = None
    d: Optional[np.ndarray] = None
    ia: Optional[np.ndarray] = None
    ib: Optional[np.ndarray] = None

    @property
    def npairs(self) -> int:
        return 0 if self.ia is None else int(self.ia.shape[0])


FULL = {
    # cfg: (call, n, h, N, dtype, extra)
    1: ("apply", 64, 6, 4096, "f64"),
    2: ("apply", 1024, 10, 262144, "f32"),
    3: ("sym", 2048, 32, 131072, "f32"),
    4: ("mahalanobis", 512, 9, 65536, "f32"),   # + P = 2**21 pairs
    5: ("apply", 4096, None, 65536, "f32"),      # h in C5_H
}
C4_PAIRS = 1 << 21
C5_H = (12, 64, 256, 1024)


def make_config(cfg: int, h: Optional[int] = None, N: Optional[int] = None,
                npairs: Optional[int] = None) -> Case:
    """Inputs for BASELINE.json config `cfg` (1-based).  `N` (and `npairs`) may be
    reduced for oracle-sized parity runs; the first columns/pairs are the same
    values the full-size draw would start with only where noted (X is drawn in
    row chunks, so a prefix of columns is identical to the full draw's prefix)."""
    call, n, h0, N0, dtype = FULL[cfg]
    if cfg == 5:
        if h is None:
            raise ValueError("config 5 needs h")
        gU, gX = rng(5, h, S_U), rng(5, 0, S_X)
    else:
        h = h0 if h is None else h
        gU, gX = rng(cfg, S_U), rng(cfg, S_X)
    N = N0 if N is None else N
    U = unit_reflectors(gU, h, n, dtype)
    X = gaussian_columns(gX, N, n, dtype)
    c = Case(f"C{cfg}", call, n, h, N, dtype, U, X)
    if call == "sym":
        c.lam = c3_spectrum(rng(cfg, S_FLIP), n, dtype)
    if call == "mahalanobis":
        c.d = metric_diag(rng(cfg, S_D), n, dtype)
        P = C4_PAIRS if npairs is None else npairs
        c.ia, c.ib = index_pairs(rng(cfg, S_IA), rng(cfg, S_IB), N, P)
    return c


def make_case(call: str, n: int, h: int, N: int, dtype: str, seed: int = 0,
              npairs: int = 0, zero_slots=()) -> Case:
    """Generic seeded case for parity/edge tests (key [root, 100, seed, n, h, N, stream])."""
    key = (100, seed, n, h, N)
    U = unit_reflectors(rng(*key, S_U), h, n, dtype, zero_slots)
    X = gaussian_columns(rng(*key, S_X), N, n, dtype)
    c = Case(f"{call}-n{n}-h{h}-N{N}-{dtype}", call, n, h, N, dtype, U, X)
    if call == "sym":
        c.lam = c3_spectrum(rng(*key, S_FLIP), n, dtype)
    if call == "mahalanobis":
        c.d = metric_diag(rng(*key, S_D), n, dtype)
        c.ia, c.ib = index_pairs(rng(*key, S_IA), rng(*key, S_IB), max(N, 1), npairs)
    return c


def paper_context_shapes():
    """Synthetic stand-ins for PAPER.md Table I test-time transforms (l.670, l.679):
    (n, N_test) with h in {ceil(log2 n), ceil(2 log2 n), ceil(3 log2 n)}.
    The datasets are not in the container; iid N(0,1) columns stand in for them."""
    out = []
    for n, Nt in ((100, 2339), (200, 5648), (40, 21000)):
        for mult in (1, 2, 3):
            out.append((n, int(math.ceil(mult * math.log2(n))), Nt))
    return out


def make_knn_case(n: int = 40, h: int = 6, M_ref: int = 49000, M_query: int = 21000,
                  k: int = 3, seed: int = 0) -> Case:
    """NEXT-f3 workload: synthetic stand-in for PAPER.md Table I's test-time k-NN (l.670:
    MNIST after PCA to n = 40, 70/30 split of 70000 points, h = ceil(log2 n) = 6).  The
    dataset is not in the container: iid N(0,1) points, unit Gaussian reflectors, metric
    diagonal U[0.1, 10].  X holds the references; `ia` is unused; the queries are in
    `lam` (reused field) -- see bench.py."""
    key = (500, seed, n, h, M_ref, M_query)
    U = unit_reflectors(rng(*key, S_U), h, n, "f32")
    Pr = gaussian_columns(rng(*key, S_X), M_ref, n, "f32")
    Pq = gaussian_columns(rng(*key, S_FLIP), M_query, n, "f32")
    d = metric_diag(rng(*key, S_D), n, "f32")
    c = Case(f"KNN-n{n}-h{h}", "knn", n, h, M_ref, "f32", U, Pr, lam=Pq, d=d)
    c.k = k
    return c


def qr_reflectors(g: np.random.Generator, h: int, n: int, dtype: str = "f64") -> np.ndarray:
    """(h, n) unit reflectors with the partial-QR structure of Result 3 (PAPER.md l.218-261:
    J_k has k-1 leading zeros): row i is zero before column i, Gaussian after, normalised."""
    u = g.standard_normal((h, n))
    for i in range(h):
        u[i, :i] = 0.0
    if h:
        u /= np.sqrt((u * u).sum(axis=1, keepdims=True))
    return np.ascontiguousarray(u.astype(np_dtype(dtype)))
