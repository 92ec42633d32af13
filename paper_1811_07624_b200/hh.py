"""Thin ctypes binding over libhh.so (include/hh.h).  Argument marshalling only.

Every computation runs in libhh.so's CUDA kernels.  PyTorch is used only to hold
device memory and to name the current CUDA stream.  If libhh.so is missing or a
tensor is not on a CUDA device the call raises -- there is no CPU fallback.

Names mirror the C ABI: hh_apply, hh_sym_apply, hh_mahalanobis, hh_apply_host,
hh_workspace_bytes.  Layout (hh.h): U is a (h, n) tensor (row i = u_{i+1},
== n x h column-major), X / Y / P are (N, n) tensors (== n x N column-major).
"""
from __future__ import annotations

import contextlib
import ctypes
import os
import re
from typing import Optional

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HH_LIB_PATH") or os.path.join(_PKG, "libhh.so")  # override: A/B runs only
HEADER = os.path.join(os.path.dirname(_PKG), "include", "hh.h")

HH_OK, HH_ERR_INVALID_VALUE, HH_ERR_UNSUPPORTED, HH_ERR_WORKSPACE, HH_ERR_CUDA = range(5)
HH_F32, HH_F64 = 0, 1
HH_OP_N, HH_OP_T = 0, 1
HH_CALL_APPLY, HH_CALL_SYM, HH_CALL_MAHALANOBIS, HH_CALL_APPLY_HOST, HH_CALL_KNN, \
    HH_CALL_CONGRUENCE, HH_CALL_SHF = range(7)
HH_ALGO_AUTO, HH_ALGO_FUSED, HH_ALGO_WY = range(3)
HH_SIDE_LEFT, HH_SIDE_RIGHT = range(2)

_DT = {torch.float32: HH_F32, torch.float64: HH_F64}


class HHError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} ({status})")


_lib = None


def lib() -> ctypes.CDLL:
    """Load libhh.so (built by paper_1811_07624_b200.build / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not found: run `python -m paper_1811_07624_b200.build` "
                               "(the CUDA extension is required; there is no fallback)")
        L = ctypes.CDLL(LIB_PATH)
        i64, p, i32, sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        L.hh_apply.argtypes = [i32, i64, i64, p, p, p, i64, i32, p, sz, p]
        L.hh_sym_apply.argtypes = [i64, i64, p, p, p, p, i64, i32, p, sz, p]
        L.hh_mahalanobis.argtypes = [i64, i64, p, p, p, i64, p, p, i64, p, i32, p, sz, p]
        L.hh_apply_host.argtypes = [i32, i64, i64, p, p, p, i64, i32, p, sz, p]
        L.hh_workspace_bytes.argtypes = [i32, i64, i64, i64, i64, i32, ctypes.POINTER(sz)]
        L.hh_apply_signed.argtypes = [i32, i32, i64, i64, p, p, p, p, i64, i32, p, sz, p]
        L.hh_sym_apply_signed.argtypes = [i64, i64, p, p, p, p, p, i64, i32, p, sz, p]
        L.hh_apply_signed.restype = i32
        L.hh_sym_apply_signed.restype = i32
        L.hh_apply_qr.argtypes = [i32, i64, i64, p, p, p, i64, i32, p, sz, p]
        L.hh_apply_qr.restype = i32
        L.hh_congruence.argtypes = [i32, i64, i64, p, p, p, i64, i32, p, sz, p]
        L.hh_congruence.restype = i32
        L.hh_shf_cost.argtypes = [i64, p, p, p, i64, p, p, i32, p, sz, p]
        L.hh_shf_cost.restype = i32
        L.hh_knn.argtypes = [i64, i64, p, p, p, i64, p, i64, i32, p, p, i32, p, sz, p]
        L.hh_knn.restype = i32
        L.hh_last_launch_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
        L.hh_last_launch_count.restype = i32
        L.hh_set_algo.argtypes = [i32]
        L.hh_set_algo.restype = i32
        L.hh_get_algo.restype = i32
        L.hh_debug_wy_project.argtypes = [i32, i64, i64, p, p, i64, p, sz,
                                          ctypes.POINTER(i64), p]
        L.hh_debug_wy_project.restype = i32
        if hasattr(L, "hh_debug_wy_ts_min"):   # test hook (absent from older builds)
            L.hh_debug_wy_ts_min.argtypes = [i32]
            L.hh_debug_wy_ts_min.restype = i32
        if hasattr(L, "hh_debug_wy_flow"):     # A/B hook: single-launch block program on/off
            L.hh_debug_wy_flow.argtypes = [i32, i32]
            L.hh_debug_wy_flow.restype = i32
            L.hh_debug_wy_flow_knobs.argtypes = [ctypes.POINTER(ctypes.c_int), i32]
            L.hh_debug_wy_flow_knobs.restype = None
        if hasattr(L, "hh_debug_k1"):
            L.hh_debug_k1.argtypes = [i32, i32]
            L.hh_debug_k1.restype = None
            L.hh_debug_k1_stream.argtypes = [i32]
            L.hh_debug_k1_stream.restype = i32
            L.hh_debug_k1_prefetch.argtypes = [i32]
            L.hh_debug_k1_prefetch.restype = i32
            L.hh_debug_k1_tmem.argtypes = [i32]
            L.hh_debug_k1_tmem.restype = i32
            if hasattr(L, "hh_debug_k1_blocked"):
                L.hh_debug_k1_blocked.argtypes = [i32]
                L.hh_debug_k1_blocked.restype = i32
            if hasattr(L, "hh_debug_k7_rows"):
                L.hh_debug_k7_rows.argtypes = [i32]
                L.hh_debug_k7_rows.restype = i32
            if hasattr(L, "hh_debug_mahal_fork"):
                L.hh_debug_mahal_fork.argtypes = [i32]
                L.hh_debug_mahal_fork.restype = i32
            L.hh_debug_wy_pdl.argtypes = [i32]
            L.hh_debug_wy_pdl.restype = i32
            if hasattr(L, "hh_debug_wy_symfuse"):
                L.hh_debug_wy_symfuse.argtypes = [i32]
                L.hh_debug_wy_symfuse.restype = i32
            if hasattr(L, "hh_debug_wy_tsa"):
                L.hh_debug_wy_tsa.argtypes = [i32]
                L.hh_debug_wy_tsa.restype = i32
        if hasattr(L, "hh_debug_wy_timeline"):
            L.hh_debug_wy_timeline.argtypes = [p]
            L.hh_debug_wy_timeline.restype = i32
        L.hh_status_string.argtypes = [i32]
        L.hh_status_string.restype = ctypes.c_char_p
        L.hh_version.restype = ctypes.c_char_p
        L.hh_last_launch_info.argtypes = [ctypes.POINTER(ctypes.c_char_p)] + \
            [ctypes.POINTER(ctypes.c_int)] * 4
        for f in ("hh_apply", "hh_sym_apply", "hh_mahalanobis", "hh_apply_host",
                  "hh_workspace_bytes", "hh_last_launch_info"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def declared_symbols() -> list:
    """Function names declared in include/hh.h."""
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_]\w*\s*\*?\s*(hh_\w+)\s*\(", src, re.M)))


def status_string(s: int) -> str:
    return lib().hh_status_string(int(s)).decode()


def version() -> str:
    return lib().hh_version().decode()


def last_launch_info() -> dict:
    v = ctypes.c_char_p()
    g, b, s, c = (ctypes.c_int() for _ in range(4))
    st = lib().hh_last_launch_info(ctypes.byref(v), ctypes.byref(g), ctypes.byref(b),
                                   ctypes.byref(s), ctypes.byref(c))
    if st != HH_OK:
        return {}
    kc = ctypes.c_int()
    lib().hh_last_launch_count(ctypes.byref(kc))
    return {"variant": v.value.decode(), "grid": g.value, "block": b.value, "smem": s.value,
            "nchunks": c.value, "launches": kc.value}


def _check(st: int, what: str):
    if st != HH_OK:
        raise HHError(st, what)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream, device=None) -> ctypes.c_void_p:
    """The given stream, else the current stream of the operands' device."""
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _dev(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _dtype(t: torch.Tensor) -> int:
    if t.dtype not in _DT:
        raise ValueError(f"unsupported dtype {t.dtype}")
    return _DT[t.dtype]


def _validate(X: torch.Tensor, xname: str = "X", U: Optional[torch.Tensor] = None,
              same: dict = None, vecs: dict = None, host: bool = False) -> tuple:
    """Check every operand against X before anything reaches libhh.so: X is a contiguous
    2-D (N, n) float tensor; U is (h, n) (or empty) of X's dtype; every tensor in `same`
    has X's shape and dtype; every tensor in `vecs` is n values of X's dtype; all of them
    contiguous and on X's device (CUDA, or the host for hh_apply_host).  Returns (N, n, h)."""
    if X.dim() != 2:
        raise ValueError(f"{xname} must be 2-D (N, n), got shape {tuple(X.shape)}")
    _dtype(X)
    N, n = X.shape

    def where(t, name):
        if host:
            if t.is_cuda:
                raise ValueError(f"{name} must be a host tensor for hh_apply_host")
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
        else:
            _dev(t, name)
            if t.device != X.device:
                raise ValueError(f"{name} is on {t.device}, {xname} on {X.device}")

    where(X, xname)
    h = 0
    if U is not None and U.numel():
        if U.dim() != 2 or U.shape[1] != n:
            raise ValueError(f"U must be (h, {n}), got {tuple(U.shape)}")
        if U.dtype != X.dtype:
            raise ValueError(f"U dtype {U.dtype} != {xname} dtype {X.dtype}")
        where(U, "U")
        h = U.shape[0]
    for name, t in (same or {}).items():
        if tuple(t.shape) != (N, n) or t.dtype != X.dtype:
            raise ValueError(f"{name} must be {(N, n)} {X.dtype}, got {tuple(t.shape)} {t.dtype}")
        where(t, name)
    for name, t in (vecs or {}).items():
        if t.numel() != n or t.dtype != X.dtype:
            raise ValueError(f"{name} must hold {n} values of {X.dtype}, got {t.numel()} {t.dtype}")
        where(t, name)
    return N, n, h


_NULLCTX = contextlib.nullcontext()


def _on(device: torch.device):
    """Run the call on `device` (its current stream): a device guard only when it is not
    already the current device (the guard costs microseconds per call)."""
    if device.type == "cuda" and device.index is not None and device.index != torch.cuda.current_device():
        return torch.cuda.device(device)
    return _NULLCTX


_WS_CACHE = {}


def clear_workspace_cache() -> None:
    """Forget the memoised workspace sizes (after changing a debug knob that sizes them)."""
    _WS_CACHE.clear()


def _workspace(call: int, n: int, h: int, N_or_M: int, npairs: int, like: torch.Tensor,
               workspace: Optional[torch.Tensor]):
    """(workspace tensor or None, bytes to pass): the query's size, allocated on `like`'s
    device when not given or too small; a given workspace must be on that device.  The
    library's size query is memoised per (call, shape, dtype, this thread's algo selection)."""
    key = (call, n, h, N_or_M, npairs, like.dtype, int(lib().hh_get_algo()))
    wsb = _WS_CACHE.get(key)
    if wsb is None:
        wsb = hh_workspace_bytes(call, n, h, N_or_M, npairs, like.dtype)
        if len(_WS_CACHE) > 4096:
            _WS_CACHE.clear()
        _WS_CACHE[key] = wsb
    if not wsb:
        return None, 0
    if workspace is not None:
        _dev(workspace, "workspace")
        if workspace.device != like.device:
            raise ValueError(f"workspace is on {workspace.device}, operands on {like.device}")
    if workspace is None or workspace.numel() * workspace.element_size() < wsb:
        workspace = torch.empty(wsb, dtype=torch.uint8, device=like.device)
    return workspace, workspace.numel() * workspace.element_size()


def hh_set_algo(algo: int) -> None:
    """Select the hh_apply path for this thread (hh.h: hh_set_algo)."""
    _check(lib().hh_set_algo(int(algo)), "hh_set_algo")


def hh_get_algo() -> int:
    return int(lib().hh_get_algo())


class algo:
    """Context manager: `with algo(HH_ALGO_WY): ...` (thread-local selection)."""

    def __init__(self, a: int):
        self.a = a

    def __enter__(self):
        self.prev = hh_get_algo()
        hh_set_algo(self.a)
        return self

    def __exit__(self, *exc):
        hh_set_algo(self.prev)


def debug_wy_project(op: int, U: torch.Tensor, X: torch.Tensor, workspace: torch.Tensor):
    """Test hook: compact-WY preparation + the first projection only.  Returns the
    offsets dict (G, V, b, nblk, n_pad, T) into `workspace`."""
    N, n = X.shape
    h = U.shape[0]
    off = (ctypes.c_int64 * 6)()
    st = lib().hh_debug_wy_project(int(op), n, h, _ptr(U), _ptr(X), N, _ptr(workspace),
                                   workspace.numel(), off, _stream(None))
    _check(st, "hh_debug_wy_project")
    return {"G": off[0], "V": off[1], "b": off[2], "nblk": off[3], "n_pad": off[4], "T": off[5]}


def hh_workspace_bytes(call: int, n: int, h: int, N_or_M: int, npairs: int, dtype) -> int:
    dt = _DT[dtype] if isinstance(dtype, torch.dtype) else int(dtype)
    out = ctypes.c_size_t()
    _check(lib().hh_workspace_bytes(int(call), n, h, N_or_M, npairs, dt, ctypes.byref(out)),
           "hh_workspace_bytes")
    return int(out.value)


def hh_apply(op: int, U: torch.Tensor, X: torch.Tensor, Y: Optional[torch.Tensor] = None,
             workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Y = Q X (op = HH_OP_N) or Q^T X (HH_OP_T), Q = H_1 ... H_h (hh.h: hh_apply).

    The workspace the selected path needs (hh_workspace_bytes) is allocated on the
    tensors' device when not given."""
    if Y is None:
        Y = torch.empty_like(X)
    N, n, h = _validate(X, U=U, same={"Y": Y})
    with _on(X.device):
        ws, wsb = _workspace(HH_CALL_APPLY, n, h, N, 0, X, workspace) if N else (None, 0)
        st = lib().hh_apply(int(op), n, h, _ptr(U) if h else None, _ptr(X), _ptr(Y), N,
                            _dtype(X), _ptr(ws), wsb, _stream(stream, X.device))
    _check(st, "hh_apply")
    return Y


def hh_sym_apply(U: torch.Tensor, lam: torch.Tensor, X: torch.Tensor,
                 Y: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
    """Y = Q diag(lam) Q^T X (hh.h: hh_sym_apply); allocates the workspace the selected
    path needs when not given."""
    if Y is None:
        Y = torch.empty_like(X)
    N, n, h = _validate(X, U=U, same={"Y": Y}, vecs={"lambda": lam})
    with _on(X.device):
        ws, wsb = _workspace(HH_CALL_SYM, n, h, N, 0, X, workspace) if N else (None, 0)
        st = lib().hh_sym_apply(n, h, _ptr(U) if h else None, _ptr(lam), _ptr(X), _ptr(Y), N,
                                _dtype(X), _ptr(ws), wsb, _stream(stream, X.device))
    _check(st, "hh_sym_apply")
    return Y


def hh_apply_signed(op: int, side: int, U: torch.Tensor, d: torch.Tensor, X: torch.Tensor,
                    Y: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                    stream=None) -> torch.Tensor:
    """Y = D op(Q) X (side HH_SIDE_LEFT, Eq. 1) or op(Q) D X (HH_SIDE_RIGHT, Result 3)
    (hh.h: hh_apply_signed)."""
    if Y is None:
        Y = torch.empty_like(X)
    N, n, h = _validate(X, U=U, same={"Y": Y}, vecs={"d": d})
    with _on(X.device):
        ws, wsb = _workspace(HH_CALL_APPLY, n, h, N, 0, X, workspace) if N else (None, 0)
        st = lib().hh_apply_signed(int(op), int(side), n, h, _ptr(U) if h else None, _ptr(d),
                                   _ptr(X), _ptr(Y), N, _dtype(X), _ptr(ws), wsb,
                                   _stream(stream, X.device))
    _check(st, "hh_apply_signed")
    return Y


def hh_sym_apply_signed(U: torch.Tensor, d: torch.Tensor, lam: torch.Tensor, X: torch.Tensor,
                        Y: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                        stream=None) -> torch.Tensor:
    """Y = D Q diag(lam) Q^T D X (hh.h: hh_sym_apply_signed, eq:thesbar)."""
    if Y is None:
        Y = torch.empty_like(X)
    N, n, h = _validate(X, U=U, same={"Y": Y}, vecs={"d": d, "lambda": lam})
    with _on(X.device):
        ws, wsb = _workspace(HH_CALL_SYM, n, h, N, 0, X, workspace) if N else (None, 0)
        st = lib().hh_sym_apply_signed(n, h, _ptr(U) if h else None, _ptr(d), _ptr(lam),
                                       _ptr(X), _ptr(Y), N, _dtype(X), _ptr(ws), wsb,
                                       _stream(stream, X.device))
    _check(st, "hh_sym_apply_signed")
    return Y


def hh_mahalanobis(U: torch.Tensor, d: torch.Tensor, P: torch.Tensor, ia: torch.Tensor,
                   ib: torch.Tensor, dist: Optional[torch.Tensor] = None,
                   workspace: Optional[torch.Tensor] = None, fused: bool = False,
                   stream=None) -> torch.Tensor:
    """dist[j] = ||D^1/2 Q^T (P[ia[j]] - P[ib[j]])||^2 (hh.h: hh_mahalanobis).

    By default a workspace is allocated for the transform-once path (K3a + K3b);
    `fused=True` passes NULL and runs the per-pair fused kernel (K3c)."""
    M, n, h = _validate(P, "P", U=U, vecs={"d": d})
    for t, nm in ((ia, "ia"), (ib, "ib")):
        _dev(t, nm)
        if t.dtype != torch.int32 or t.dim() != 1 or t.device != P.device:
            raise ValueError(f"{nm} must be a 1-D int32 tensor on {P.device}")
    if ia.numel() != ib.numel():
        raise ValueError(f"ia ({ia.numel()}) and ib ({ib.numel()}) differ in length")
    npairs = ia.numel()
    if dist is None:
        dist = torch.empty(npairs, dtype=P.dtype, device=P.device)
    _dev(dist, "dist")
    if dist.numel() != npairs or dist.dtype != P.dtype or dist.device != P.device:
        raise ValueError(f"dist must hold {npairs} values of {P.dtype} on {P.device}")
    with _on(P.device):
        ws, wsb = (None, 0) if fused else _workspace(HH_CALL_MAHALANOBIS, n, h, M, npairs, P,
                                                      workspace)
        st = lib().hh_mahalanobis(n, h, _ptr(U) if h else None, _ptr(d), _ptr(P), M, _ptr(ia),
                                  _ptr(ib), npairs, _ptr(dist), _dtype(P), _ptr(ws), wsb,
                                  _stream(stream, P.device))
    _check(st, "hh_mahalanobis")
    return dist


def hh_apply_qr(op: int, U: torch.Tensor, X: torch.Tensor, Y: Optional[torch.Tensor] = None,
                workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """hh_apply for QR-structured reflectors (u_i[r] = 0 for r < i), skipping the zero
    prefix (hh.h: hh_apply_qr, NEXT-f2)."""
    if Y is None:
        Y = torch.empty_like(X)
    N, n, h = _validate(X, U=U, same={"Y": Y})
    with _on(X.device):
        ws, wsb = _workspace(HH_CALL_APPLY, n, h, N, 0, X, workspace) if N else (None, 0)
        st = lib().hh_apply_qr(int(op), n, h, _ptr(U) if h else None, _ptr(X), _ptr(Y), N,
                               _dtype(X), _ptr(ws), wsb, _stream(stream, X.device))
    _check(st, "hh_apply_qr")
    return Y


def hh_congruence(op: int, U: torch.Tensor, M: torch.Tensor, out: Optional[torch.Tensor] = None,
                  workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """op(Q) M_b op(Q)^T for M of shape (count, n, n), each M[b] a column-major n x n
    matrix (i.e. the math matrix is M[b].T) (hh.h: hh_congruence, NEXT-f4)."""
    if M.dim() != 3 or M.shape[1] != M.shape[2]:
        raise ValueError(f"M must be (count, n, n), got {tuple(M.shape)}")
    count, n, _ = M.shape
    if out is None:
        out = torch.empty_like(M)
    if out.shape != M.shape or out.dtype != M.dtype:
        raise ValueError(f"out must be {tuple(M.shape)} {M.dtype}")
    _validate(M.view(count * n, n), "M", U=U, same={"out": out.view(count * n, n)})
    h = U.shape[0] if U.numel() else 0
    with _on(M.device):
        ws, wsb = _workspace(HH_CALL_CONGRUENCE, n, h, count, 0, M, workspace)
        st = lib().hh_congruence(int(op), n, h, _ptr(U) if h else None, _ptr(M), _ptr(out),
                                 count, _dtype(M), _ptr(ws), wsb, _stream(stream, M.device))
    _check(st, "hh_congruence")
    return out


def hh_shf_cost(A: torch.Tensor, B: torch.Tensor, Uc: torch.Tensor, grad: bool = True,
                cost: Optional[torch.Tensor] = None, grad_out: Optional[torch.Tensor] = None,
                workspace: Optional[torch.Tensor] = None, stream=None):
    """(cost (K,), grad (K, n) or None): the SHF objective C(u_k) of one reflector and its
    gradient for the candidates Uc of shape (K, n), A and B symmetric (n, n)
    (hh.h: hh_shf_cost, eq:theRk / eq:gradient, NEXT-f4)."""
    for t, nm in ((A, "A"), (B, "B"), (Uc, "Uc")):
        _dev(t, nm)
    if A.dim() != 2 or A.shape[0] != A.shape[1] or A.dtype not in _DT:
        raise ValueError(f"A must be a square fp32/fp64 matrix, got {tuple(A.shape)} {A.dtype}")
    n = A.shape[0]
    if B.shape != A.shape or B.dtype != A.dtype or B.device != A.device:
        raise ValueError(f"B must match A ({tuple(A.shape)} {A.dtype} on {A.device})")
    if Uc.dim() != 2 or Uc.shape[1] != n or Uc.dtype != A.dtype or Uc.device != A.device:
        raise ValueError(f"Uc must be (K, {n}) {A.dtype} on {A.device}")
    K = Uc.shape[0]
    if cost is None:
        cost = torch.empty(K, dtype=A.dtype, device=A.device)
    if grad and grad_out is None:
        grad_out = torch.empty_like(Uc)
    for t, nm, shp in ((cost, "cost", (K,)), (grad_out if grad else None, "grad_out", tuple(Uc.shape))):
        if t is None:
            continue
        _dev(t, nm)
        if tuple(t.shape) != shp or t.dtype != A.dtype or t.device != A.device:
            raise ValueError(f"{nm} must be {shp} {A.dtype} on {A.device}")
    with _on(A.device):
        ws, wsb = _workspace(HH_CALL_SHF, n, 0, K, 0, A, workspace) if K else (None, 0)
        st = lib().hh_shf_cost(n, _ptr(A), _ptr(B), _ptr(Uc), K, _ptr(cost),
                               _ptr(grad_out) if grad else None, _DT[A.dtype], _ptr(ws), wsb,
                               _stream(stream, A.device))
    _check(st, "hh_shf_cost")
    return cost, (grad_out if grad else None)


def hh_knn(U: torch.Tensor, d: torch.Tensor, P_ref: torch.Tensor, P_query: torch.Tensor, k: int,
           workspace: Optional[torch.Tensor] = None, stream=None):
    """k nearest references of every query under d_S = ||diag(sqrt d) Q^T (x_q - x_r)||^2
    (hh.h: hh_knn).  Returns (idx int32 (M_query, k), dist (M_query, k)), ascending."""
    Mr, n, h = _validate(P_ref, "P_ref", U=U, vecs={"d": d})
    if P_query.dim() != 2 or P_query.shape[1] != n or P_query.dtype != P_ref.dtype:
        raise ValueError(f"P_query must be (M_query, {n}) {P_ref.dtype}")
    _dev(P_query, "P_query")
    if P_query.device != P_ref.device:
        raise ValueError(f"P_query is on {P_query.device}, P_ref on {P_ref.device}")
    Mq = P_query.shape[0]
    idx = torch.empty(Mq, k, dtype=torch.int32, device=P_ref.device)
    dist = torch.empty(Mq, k, dtype=P_ref.dtype, device=P_ref.device)
    with _on(P_ref.device):
        ws, wsb = _workspace(HH_CALL_KNN, n, h, Mr, Mq, P_ref, workspace)
        st = lib().hh_knn(n, h, _ptr(U) if h else None, _ptr(d), _ptr(P_ref), Mr, _ptr(P_query),
                          Mq, int(k), _ptr(idx), _ptr(dist), _dtype(P_ref), _ptr(ws), wsb,
                          _stream(stream, P_ref.device))
    _check(st, "hh_knn")
    return idx, dist


def hh_apply_host(op: int, U: torch.Tensor, X: torch.Tensor, Y: Optional[torch.Tensor] = None,
                  workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """hh_apply on HOST (CPU, ideally pinned) tensors; device workspace (hh.h: hh_apply_host).
    The current CUDA device runs it unless `workspace` names another one."""
    if Y is None:
        Y = torch.empty_like(X, pin_memory=X.is_pinned())
    N, n, h = _validate(X, U=U, same={"Y": Y}, host=True)
    device = workspace.device if workspace is not None else torch.device(
        "cuda", torch.cuda.current_device())
    with _on(device):
        ws, wsb = _workspace(HH_CALL_APPLY_HOST, n, h, N, 0,
                             torch.empty(0, dtype=X.dtype, device=device), workspace)
        st = lib().hh_apply_host(int(op), n, h, _ptr(U) if h else None, _ptr(X), _ptr(Y), N,
                                 _dtype(X), _ptr(ws), wsb, _stream(stream, device))
    _check(st, "hh_apply_host")
    return Y
