"""CPU-side checks of the C ABI boundary: the library loads, exports every symbol
include/hh.h declares, and validates arguments before any launch (no GPU needed:
every call here returns before touching the CUDA runtime)."""
import ctypes
import os

import pytest

import paper_1811_07624_b200 as hhpkg
from paper_1811_07624_b200 import hh

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_declared_symbols():
    L = hh.lib()
    syms = hh.declared_symbols()
    for s in ("hh_apply", "hh_sym_apply", "hh_mahalanobis", "hh_apply_host",
              "hh_workspace_bytes", "hh_status_string", "hh_version", "hh_last_launch_info"):
        assert s in syms
    for s in syms:
        assert hasattr(L, s), f"libhh.so does not export {s}"
    assert hh.version().count(".") == 2


def test_library_is_sm100a():
    """libhh.so carries sm_100a SASS (cuobjdump), no PTX-only JIT path."""
    import shutil
    import subprocess
    cu = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cu):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cu, "--list-elf", hh.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    for s, name in enumerate(["HH_OK", "HH_ERR_INVALID_VALUE", "HH_ERR_UNSUPPORTED",
                              "HH_ERR_WORKSPACE", "HH_ERR_CUDA"]):
        assert hh.status_string(s) == name
    assert hh.status_string(99) == "HH_ERR_UNKNOWN"


def test_workspace_query():
    # small h: the fused kernel, no scratch; large h / the symmetric C3 shape (fp32): the
    # compact-WY block program's scratch, well below the 1 GiB operands; fp64: always 0
    assert hhpkg.hh_workspace_bytes(hh.HH_CALL_APPLY, 1024, 10, 262144, 0, 0) == 0
    big = hhpkg.hh_workspace_bytes(hh.HH_CALL_APPLY, 4096, 1024, 65536, 0, 0)
    assert 0 < big < 256 << 20
    sym = hhpkg.hh_workspace_bytes(hh.HH_CALL_SYM, 2048, 32, 131072, 0, 0)
    assert 0 < sym < 64 << 20
    assert hhpkg.hh_workspace_bytes(hh.HH_CALL_SYM, 2048, 32, 131072, 0, 1) == 0
    with hhpkg.algo(hhpkg.HH_ALGO_FUSED):
        assert hhpkg.hh_workspace_bytes(hh.HH_CALL_APPLY, 4096, 1024, 65536, 0, 0) == 0
        assert hhpkg.hh_workspace_bytes(hh.HH_CALL_SYM, 2048, 32, 131072, 0, 0) == 0
    r256 = lambda b: (b + 255) // 256 * 256  # noqa: E731
    assert hhpkg.hh_workspace_bytes(hh.HH_CALL_MAHALANOBIS, 512, 9, 65536, 1 << 21, 0) == \
        512 * 65536 * 4 + 2 * r256(65536 * 4) + r256(65537 * 4) + r256((1 << 21) * 4) + r256(16 * 4)
    b = hhpkg.hh_workspace_bytes(hh.HH_CALL_APPLY_HOST, 1024, 10, 262144, 0, 0)
    assert b >= 3 * (64 << 20) + 10 * 1024 * 4
    with pytest.raises(hh.HHError):
        hhpkg.hh_workspace_bytes(7, 16, 1, 1, 0, 0)


@pytest.mark.parametrize("n,h,N,wy", [
    (1024, 10, 262144, False),                      # C2
    (4096, 12, 65536, False), (4096, 16, 65536, False), (4096, 17, 65536, True),   # K1w to h = 16
    (2048, 18, 16384, False), (2048, 19, 16384, True),   # n = 2048, E = 2^25 band (r2 re-sweep)
    (2048, 16, 65536, False), (2048, 17, 65536, True),   # E = 2^27: large band
    (2048, 28, 131072, True),                       # the old n>=512, h>=32 rule kept K1 here
    (1024, 19, 32768, False), (1024, 20, 32768, True),   # E = 2^25: middle band (r2 re-sweep)
    (1024, 16, 262144, False), (1024, 17, 262144, True),  # K1t to h = 16, then K5 (r2)
    (1024, 31, 4096, False), (1024, 32, 4096, True),     # small problems: h >= 32
    (128, 23, 1 << 21, False), (128, 24, 1 << 21, True),   # n <= 512: against K1s (r2)
    (256, 19, 1 << 20, False), (256, 20, 1 << 20, True),
    (512, 17, 1 << 19, False), (512, 18, 1 << 19, True),
    (512, 22, 1 << 16, False), (512, 23, 1 << 16, True),
    (64, 512, 1 << 22, False),                      # n < 128: always K1
    (8192, 6, 32768, False), (8192, 7, 32768, True),
    (8192, 15, 4096, False), (8192, 16, 4096, True),
    (16384, 1, 16384, False), (16384, 2, 16384, True),   # n > 8192: against K1g
    (16384, 11, 128, False), (16384, 12, 128, True),
])
def test_auto_crossover(n, h, N, wy):
    """HH_ALGO_AUTO's K1/K5 choice (hh_api.cu wy_min_h; thresholds from the same-box sweep in
    profiles/r1/crossover_r1.txt): the apply workspace is non-zero exactly when K5 is chosen."""
    ws = hhpkg.hh_workspace_bytes(hh.HH_CALL_APPLY, n, h, N, 0, 0)
    assert (ws > 0) == wy, (n, h, N, ws)
    with pytest.raises(hh.HHError):
        hhpkg.hh_workspace_bytes(hh.HH_CALL_APPLY, 0, 1, 1, 0, 0)


def test_unaligned_stride_workspace_policy():
    """Column strides that are not a multiple of 16 bytes: no scratch while K1r / K1g serve the
    call, the padded copy (U, X, two n-vectors at the padded pitch) plus the aligned call's own
    scratch from the measured crossover (hh_api.cu use_padded)."""
    q = lambda call, n, h, N, dt=0: hhpkg.hh_workspace_bytes(call, n, h, N, 0, dt)
    assert q(hh.HH_CALL_APPLY, 1023, 49, 262144) == 0
    pad = q(hh.HH_CALL_APPLY, 1023, 50, 262144)
    assert pad >= (262144 + 50 + 2) * 1024 * 4            # copies at pitch 1024
    assert pad >= (262144 + 50 + 2) * 1024 * 4 + q(hh.HH_CALL_APPLY, 1024, 50, 262144)
    assert q(hh.HH_CALL_APPLY, 101, 43, 1 << 20) == 0 and q(hh.HH_CALL_APPLY, 101, 44, 1 << 20) > 0
    assert q(hh.HH_CALL_SYM, 1023, 21, 4096) == 0 and q(hh.HH_CALL_SYM, 1023, 22, 4096) > 0
    assert q(hh.HH_CALL_SYM, 2047, 16, 4096) == 0 and q(hh.HH_CALL_SYM, 2047, 17, 4096) > 0
    assert q(hh.HH_CALL_SYM, 101, 18, 4096) == 0 and q(hh.HH_CALL_SYM, 101, 19, 4096) > 0
    assert q(hh.HH_CALL_APPLY, 9001, 3, 4096) == 0 and q(hh.HH_CALL_APPLY, 9001, 4, 4096) > 0
    assert q(hh.HH_CALL_APPLY, 4097, 3, 4096) == 0 and q(hh.HH_CALL_APPLY, 4097, 4, 4096) > 0   # past K1r's tables
    assert q(hh.HH_CALL_APPLY, 4095, 16, 4096) == 0 and q(hh.HH_CALL_APPLY, 4095, 17, 4096) > 0  # U past K1r (TMEM holds 16)
    assert q(hh.HH_CALL_APPLY, 1023, 60, 4096, 1) > 0     # fp64: pitch of 2 (U past K1r's shared memory)
    assert q(hh.HH_CALL_APPLY, 1024, 10, 262144) == 0     # aligned shapes unchanged
    # Mahalanobis: transform-once on the padded copy of the points
    m_al = hhpkg.hh_workspace_bytes(hh.HH_CALL_MAHALANOBIS, 512, 9, 65536, 1 << 21, 0)
    m_un = hhpkg.hh_workspace_bytes(hh.HH_CALL_MAHALANOBIS, 511, 9, 65536, 1 << 21, 0)
    assert m_un >= m_al + 65536 * 512 * 4


def _apply(op, n, h, U, X, Y, N, dt):
    return hh.lib().hh_apply(op, n, h, U, X, Y, N, dt, None, 0, None)


def test_validation_before_launch():
    L = hh.lib()
    A = 1 << 20      # a fake but 16-B aligned address: never dereferenced on these paths
    # invalid values
    assert _apply(2, 16, 1, A, A, A, 4, 0) == hh.HH_ERR_INVALID_VALUE           # bad op
    assert _apply(0, 0, 1, A, A, A, 4, 0) == hh.HH_ERR_INVALID_VALUE            # n < 1
    assert _apply(0, 16, -1, A, A, A, 4, 0) == hh.HH_ERR_INVALID_VALUE          # h < 0
    assert _apply(0, 16, 1, A, A, A, -1, 0) == hh.HH_ERR_INVALID_VALUE          # N < 0
    assert _apply(0, 16, 1, None, A, A, 4, 0) == hh.HH_ERR_INVALID_VALUE        # U NULL
    assert _apply(0, 16, 1, A, A, A, 4, 5) == hh.HH_ERR_INVALID_VALUE           # bad dtype
    # unsupported: pointers not aligned to the element, n beyond K1g's shared memory
    # (any n*size and 16-B misalignment run on K1g: tests/test_parity_gpu.py::test_general_*)
    assert _apply(0, 16, 1, A + 2, A, A, 4, 0) == hh.HH_ERR_UNSUPPORTED         # U misaligned
    assert _apply(0, 16, 1, A, A + 2, A, 4, 0) == hh.HH_ERR_UNSUPPORTED         # X misaligned
    assert _apply(0, 16, 1, A, A, A + 4, 4, 1) == hh.HH_ERR_UNSUPPORTED         # Y misaligned (f64)
    assert _apply(0, 60000, 1, A, A, A, 4, 0) == hh.HH_ERR_UNSUPPORTED          # n > K1g capacity
    assert _apply(0, 30000, 1, A, A, A, 4, 1) == hh.HH_ERR_UNSUPPORTED          # ... fp64
    with hhpkg.algo(hh.HH_ALGO_WY):                                             # forced WY, K1g shape
        assert _apply(0, 18, 1, A, A, A, 4, 0) == hh.HH_ERR_UNSUPPORTED
        assert _apply(0, 70000, 1, A, A, A, 4, 0) == hh.HH_ERR_UNSUPPORTED      # beyond the block program
        assert _apply(0, 8196, 1, A, A, A, 4, 0) == hh.HH_ERR_WORKSPACE         # n > 8192: WY, needs scratch
    # empty batches are successful no-ops (no launch), h = 0 needs no U
    assert _apply(0, 16, 1, A, None, None, 0, 0) == hh.HH_OK
    assert _apply(1, 16, 0, None, None, None, 0, 0) == hh.HH_OK
    # sym / Mahalanobis
    assert L.hh_sym_apply(16, 1, A, None, A, A, 4, 0, None, 0, None) == hh.HH_ERR_INVALID_VALUE
    assert L.hh_sym_apply(16, 1, A, A + 2, A, A, 4, 0, None, 0, None) == hh.HH_ERR_UNSUPPORTED
    assert L.hh_sym_apply(16, 1, A, A, A, A, 0, 0, None, 0, None) == hh.HH_OK
    assert L.hh_mahalanobis(16, 1, A, A, A, 0, A, A, 3, A, 0, None, 0, None) == \
        hh.HH_ERR_INVALID_VALUE                                                  # M = 0, pairs
    assert L.hh_mahalanobis(16, 1, A, A, A, 5, A, A, 3, A, 0, A, 16, None) == \
        hh.HH_ERR_WORKSPACE                                                      # ws too small
    assert L.hh_mahalanobis(16, 1, A, A, A, 5, A, A, 0, A, 0, None, 0, None) == hh.HH_OK
    assert L.hh_apply_host(0, 16, 1, A, A, A, 4, 0, A, 16, None) == hh.HH_ERR_WORKSPACE
    assert L.hh_apply_host(0, 16, 1, A + 3, A, A, 0, 0, None, 0, None) == hh.HH_OK


def test_binding_refuses_cpu_tensors():
    import torch
    with pytest.raises(ValueError):
        hhpkg.hh_apply(0, torch.zeros(1, 16), torch.zeros(2, 16))


def test_product_does_not_touch_oracle():
    """The product package never imports, links or executes the oracle (or anything CPU)."""
    pkg = os.path.join(ROOT, "paper_1811_07624_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "oracle" not in src.replace("oracle/", ""), f
                assert "hh_ref" not in src, f
    L = hh.lib()
    assert not hasattr(L, "hh_ref_apply")
    ctypes.CDLL  # keep import used


@pytest.mark.parametrize("n,h,N,wy", [
    (2048, 32, 131072, True),                       # C3
    (2048, 11, 131072, False), (2048, 12, 131072, True),  # r2 re-sweep after K1w
    (4096, 9, 65536, False), (4096, 10, 65536, True),
    (4096, 11, 16384, False), (4096, 12, 16384, True),
    (1024, 10, 262144, False), (1024, 11, 262144, True),  # E = 2^28
    (1024, 14, 32768, False), (1024, 15, 32768, True),    # E = 2^25 (r2 re-sweep)
    (2048, 31, 2048, False), (2048, 32, 2048, True),      # small problems
    (128, 15, 1 << 21, False), (128, 16, 1 << 21, True),  # n <= 512: against K1s (r2)
    (256, 12, 1 << 20, False), (256, 13, 1 << 20, True),
    (64, 64, 1 << 22, False),                       # n < 128: always K2
])
def test_auto_crossover_sym(n, h, N, wy):
    """The same for the symmetric apply (hh_api.cu wy_min_h_sym)."""
    ws = hhpkg.hh_workspace_bytes(hh.HH_CALL_SYM, n, h, N, 0, 0)
    assert (ws > 0) == wy, (n, h, N, ws)


def test_wy_pass_cap_rejected_before_launch():
    """The block program has at most 128 passes (hh_wy.cu kMaxPasses): h > 32768 (apply,
    256-wide blocks) and h > 8192 (symmetric, 2m - 1 passes of 128-wide blocks) are refused
    with HH_ERR_UNSUPPORTED when the tensor-core path is forced -- before any launch, so
    nothing is written -- and AUTO keeps such shapes on the fused kernel (no scratch)."""
    L = hh.lib()
    A = 1 << 20
    big = 1 << 40
    with hhpkg.algo(hhpkg.HH_ALGO_WY):
        assert L.hh_apply(0, 1024, 32769, A, A, A, 4, 0, A, big, None) == hh.HH_ERR_UNSUPPORTED
        assert L.hh_apply(1, 1024, 40000, A, A, A, 4, 0, A, big, None) == hh.HH_ERR_UNSUPPORTED
        assert L.hh_sym_apply(256, 8193, A, A, A, A, 4, 0, A, big, None) == hh.HH_ERR_UNSUPPORTED
        assert L.hh_apply(0, 1024, 10, A, A, A, 4, 1, A, big, None) == hh.HH_ERR_UNSUPPORTED  # f64
        assert L.hh_apply(0, 16, 10, A, A, A, 4, 0, A, big, None) == hh.HH_ERR_UNSUPPORTED    # n < 32
        # the largest supported programs still get a (finite) scratch size
        assert hhpkg.hh_workspace_bytes(hh.HH_CALL_APPLY, 1024, 32768, 4096, 0, 0) > 0
        assert hhpkg.hh_workspace_bytes(hh.HH_CALL_SYM, 256, 8192, 4096, 0, 0) > 0
    assert hhpkg.hh_workspace_bytes(hh.HH_CALL_APPLY, 1024, 32769, 262144, 0, 0) == 0
    assert hhpkg.hh_workspace_bytes(hh.HH_CALL_SYM, 256, 8193, 262144, 0, 0) == 0


def test_mahalanobis_pair_count_limit():
    """The bucketed gather indexes pairs and points with int32: npairs >= 2^31 - 1 (or M) is
    HH_ERR_UNSUPPORTED in the workspace query and the call, before any launch."""
    L = hh.lib()
    A = 1 << 20
    with pytest.raises(hh.HHError) as ei:
        hhpkg.hh_workspace_bytes(hh.HH_CALL_MAHALANOBIS, 16, 1, 5, 1 << 31, 0)
    assert ei.value.status == hh.HH_ERR_UNSUPPORTED
    assert L.hh_mahalanobis(16, 1, A, A, A, 5, A, A, 1 << 31, A, 0, A, 1 << 40, None) == \
        hh.HH_ERR_UNSUPPORTED
    assert L.hh_mahalanobis(16, 1, A, A, A, 5, A, A, (1 << 31) - 1, A, 0, None, 0, None) == \
        hh.HH_ERR_UNSUPPORTED


def test_debug_hooks_are_thread_local():
    """The TS-mode test hook changes only the calling thread's setting (no process-global
    mutable state in the library)."""
    import threading
    L = hh.lib()
    prev = L.hh_debug_wy_ts_min(64)
    seen = []
    t = threading.Thread(target=lambda: seen.append(L.hh_debug_wy_ts_min(256)))
    t.start()
    t.join()
    assert seen == [256]                      # the other thread still had the default
    assert L.hh_debug_wy_ts_min(prev) == 64   # this thread's value was kept
