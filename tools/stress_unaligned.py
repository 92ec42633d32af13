"""Randomised stress of the any-shape paths (K1r staged / unstaged / TMEM / shared-memory U, K1g,
the padded detour) against the oracle: random n, h, N, dtype, op, base-pointer offsets of the
operands, in place or not, apply / sym / D.  GPU box; not part of the test suite (a seeded
subset is: tests/test_fuzz_gpu.py::test_fuzz_unaligned_offsets).
usage: python tools/stress_unaligned.py [cases] [seed]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402


def offset_copy(a, off_elems):
    """A device copy of `a` whose data pointer sits `off_elems` elements past a 256-B boundary."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    buf = torch.empty(t.numel() + off_elems + 64, dtype=t.dtype, device="cuda")
    base = (-buf.data_ptr() // t.element_size()) % (256 // t.element_size())
    v = buf[base + off_elems: base + off_elems + t.numel()].view(t.shape)
    v.copy_(t)
    return v


def one_case(g, idx):
    dt = "f32" if g.random() < 0.7 else "f64"
    q = 4 if dt == "f32" else 2
    r = g.random()
    n = int(g.integers(1, 300)) if r < 0.3 else int(g.integers(300, 4200)) if r < 0.9 else int(g.integers(4200, 12000))
    if g.random() < 0.25:
        n = max(q, n // q * q)                      # aligned stride, only the pointers offset
    h = int(g.integers(0, 22))
    N = int(g.integers(1, 40)) if g.random() < 0.3 else int(g.integers(40, 700))
    if n > 4200:
        N = min(N, 60)
    offs = [int(g.integers(0, q)) for _ in range(4)]      # U, X, Y, vec
    call = ["apply", "apply", "sym", "signed"][int(g.integers(0, 4))]
    op = int(g.integers(0, 2))
    alias = g.random() < 0.3
    mode = int(g.integers(0, 5))                    # 0 policy, 1 K1r smem, 2 K1r unstaged, 3 K1g, 4 padded
    c = gi.make_case("sym", n, h, N, dt, seed=1000 + idx)
    d = np.where(g.random(n) < 0.5, -1.0, 1.0).astype(c.X.dtype)
    L = hh.hh.lib()
    L.hh_debug_k1r_tmem(0 if mode == 1 else 1)
    L.hh_debug_k1r_stage(0 if mode == 2 else 1)
    L.hh_debug_general_scalar(0 if mode == 3 else 1)
    L.hh_debug_general_pad(1 if mode == 4 else (-1 if mode == 0 else 0))
    hh.hh.clear_workspace_cache()
    tdt = torch.float32 if dt == "f32" else torch.float64
    U = offset_copy(c.U, offs[0]) if h else torch.empty(0, n, device="cuda", dtype=tdt)
    X = offset_copy(c.X, offs[1])
    Y = X if alias else offset_copy(np.zeros_like(c.X), offs[2])
    try:
        if call == "apply":
            out = hh.hh_apply(op, U, X, Y)
            ref = oracle.apply(op, c.U, c.X)
        elif call == "sym":
            out = hh.hh_sym_apply(U, offset_copy(c.lam, offs[3]), X, Y)
            ref = oracle.sym_apply(c.U, c.lam, c.X)
        else:
            side = int(g.integers(0, 2))
            out = hh.hh_apply_signed(op, side, U, offset_copy(d, offs[3]), X, Y)
            ref = oracle.apply_signed(op, side, c.U, d, c.X)
        torch.cuda.synchronize()
    finally:
        L.hh_debug_k1r_tmem(1)
        L.hh_debug_k1r_stage(1)
        L.hh_debug_general_scalar(1)
        L.hh_debug_general_pad(-1)
        hh.hh.clear_workspace_cache()
    got = out.cpu().numpy().astype(np.float64)
    err = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))
    gate = 1e-12 if dt == "f64" else 2e-5 * max(h, 1) ** 0.5
    info = hh.last_launch_info().get("variant", "?")
    ok = np.all(np.isfinite(got)) and err <= gate
    return ok, f"{call} n={n} h={h} N={N} {dt} op={op} offs={offs} alias={alias} mode={mode} {info} err={err:.2e}"


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    g = gi.rng(990, seed)
    bad = 0
    kernels = {}
    for i in range(cases):
        ok, msg = one_case(g, i)
        k = msg.split()[-2]
        kernels[k] = kernels.get(k, 0) + 1
        if not ok:
            bad += 1
            print("FAIL", msg, flush=True)
    print(f"{cases} cases, {bad} failures; kernels: {dict(sorted(kernels.items()))}")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
