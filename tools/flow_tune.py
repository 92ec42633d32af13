"""K5f tuning aid: per-role timelines (hh_debug_wy_timeline) and knob sweeps of the single-
launch block program on the BASELINE workloads.  usage (GPU box):
  python tools/flow_tune.py timeline C3 C5h64 ...
  python tools/flow_tune.py sweep C3 "P=60,74,88" "nkc=2,4,8" ...
Knobs: on, P, nkc, rseg, D, G, pol (0 = default)."""
import ctypes
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()
KN = ["on", "P", "nkc", "rseg", "D", "G", "pol"]
NAMES = ["role", "total", "p_dep", "p_ring", "mma_in", "mma_acc", "epi_acc", "epi_red", "epi_x",
         "units", "cv_in", "cv_out", "epi_busy", "u_dep", "13", "14"]


def knobs(**kw):
    v = [kw.get(k, 0) for k in KN]
    if "on" not in kw:
        v[0] = 1
    if "pol" not in kw:
        v[6] = 3
    arr = (ctypes.c_int * 7)(*v)
    L.hh_debug_wy_flow_knobs(arr, 7)
    hh.hh.clear_workspace_cache()


def setup(name):
    if name == "C3":
        c = gi.make_config(3)
    elif name == "C2":
        c = gi.make_config(2)
    else:
        c = gi.make_config(5, h=int(name[3:]))
    U, X = torch.from_numpy(c.U).cuda(), torch.from_numpy(c.X).cuda()
    Y = torch.empty_like(X)
    lam = torch.from_numpy(c.lam).cuda() if c.call == "sym" else None

    def fn():
        with hh.algo(hh.HH_ALGO_WY):
            if lam is not None:
                hh.hh_sym_apply(U, lam, X, Y)
            else:
                hh.hh_apply(0, U, X, Y)
    return c, fn


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def timeline(name, **kw):
    c, fn = setup(name)
    knobs(**kw)
    ms = timeit(fn)
    buf = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
    L.hh_debug_wy_timeline(ctypes.c_void_p(buf.data_ptr()))
    fn()
    torch.cuda.synchronize()
    L.hh_debug_wy_timeline(None)
    t = buf.view(148, 16).cpu().numpy().astype(np.float64)
    print(f"== {name} {kw} {ms:.3f} ms  {2 * c.N * c.n * 4 / ms / 1e6:.0f} GB/s")
    for role in (0, 1):
        sel = t[:, 0] == role
        if not sel.any():
            continue
        tot = t[sel, 1].mean()
        cols = [f"{NAMES[k]}={t[sel, k].mean() / tot:.2f}" for k in range(2, 16)
                if k not in (9,) and t[sel, k].any()]
        print(f"  {'project' if role == 0 else 'update '} x{int(sel.sum())} total {tot / 1e3:.0f}k cyc"
              f" units {t[sel, 9].mean():.1f} | " + " ".join(cols), flush=True)


def sweep(name, specs):
    c, fn = setup(name)
    grid = []
    for sp in specs:
        k, vals = sp.split("=")
        grid.append([(k, int(v)) for v in vals.split(",")])
    for combo in itertools.product(*grid):
        kw = dict(combo)
        knobs(**kw)
        ms = timeit(fn)
        print(f"{name} {kw} {ms:.3f} ms {2 * c.N * c.n * 4 / ms / 1e6:.0f} GB/s", flush=True)
    knobs(on=0)
    ms = timeit(fn)
    print(f"{name} classic {ms:.3f} ms {2 * c.N * c.n * 4 / ms / 1e6:.0f} GB/s", flush=True)
    knobs()


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "timeline":
        for w in sys.argv[2:]:
            if ":" in w:
                w, extra = w.split(":")
                kw = {k: int(v) for k, v in (e.split("=") for e in extra.split(";"))}
            else:
                kw = {}
            timeline(w, **kw)
    else:
        sweep(sys.argv[2], sys.argv[3:])
