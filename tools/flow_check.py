"""K5f (single dataflow launch) vs the two-kernel program: parity against the oracle on a
few shapes, then same-box timings of the BASELINE workloads with the flow on and off.
usage (GPU box): python tools/flow_check.py [quick]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def flow(on, P=0):
    L.hh_debug_wy_flow(int(on), int(P))


shapes = [("apply", 512, 64, 40000, 0), ("apply", 512, 64, 40000, 1), ("apply", 4096, 64, 2000, 0),
          ("apply", 1024, 300, 3000, 1), ("apply", 4096, 1024, 700, 0), ("sym", 2048, 32, 5000, 0),
          ("sym", 512, 100, 3000, 0), ("apply", 256, 40, 301, 0), ("apply", 100, 50, 129, 1)]
for call, n, h, N, op in shapes:
    c = gi.make_case(call, n, h, N, "f32", seed=5)
    flow(1)
    with hh.algo(hh.HH_ALGO_WY):
        t0 = time.time()
        if call == "sym":
            Y = hh.hh_sym_apply(dev(c.U), dev(c.lam), dev(c.X))
        else:
            Y = hh.hh_apply(op, dev(c.U), dev(c.X))
        torch.cuda.synchronize()
        dt = time.time() - t0
        info = hh.last_launch_info()
    ref = oracle.sym_apply(c.U, c.lam, c.X) if call == "sym" else oracle.apply(op, c.U, c.X)
    e = rel(Y.cpu().numpy().astype(np.float64), ref)
    print(f"{call} n={n} h={h} N={N} op={op}: {info['variant']} rel {e:.2e} gate {2e-5*np.sqrt(h):.2e}"
          f" {'OK' if e < 2e-5*np.sqrt(h) else 'FAIL'} ({dt:.2f}s)", flush=True)

if len(sys.argv) > 1 and sys.argv[1] == "quick":
    sys.exit(0)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name in ["C3", "C5h12", "C5h64", "C5h256", "C5h1024", "C2"]:
    if name == "C3":
        c = gi.make_config(3)
    elif name == "C2":
        c = gi.make_config(2)
    else:
        c = gi.make_config(5, h=int(name[3:]))
    U, X = dev(c.U), dev(c.X)
    Y = torch.empty_like(X)
    if c.call == "sym":
        lam = dev(c.lam)
        with hh.algo(hh.HH_ALGO_WY):
            wsb = hh.hh_workspace_bytes(hh.HH_CALL_SYM, c.n, c.h, c.N, 0, X.dtype)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        fn = lambda: hh.hh_sym_apply(U, lam, X, Y, workspace=ws)  # noqa: E731
    else:
        with hh.algo(hh.HH_ALGO_WY):
            wsb = hh.hh_workspace_bytes(hh.HH_CALL_APPLY, c.n, c.h, c.N, 0, X.dtype)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        fn = lambda: hh.hh_apply(0, U, X, Y, workspace=ws)  # noqa: E731
    byts = 2 * c.N * c.n * 4
    res = []
    with hh.algo(hh.HH_ALGO_WY):
        for tag, on, P in [("classic", 0, 0), ("flow", 1, 0), ("flowP60", 1, 60), ("flowP88", 1, 88),
                           ("flow", 1, 0)]:
            flow(on, P)
            ms = timeit(fn)
            res.append(f"{tag} {ms:.3f}ms {byts / ms / 1e6:.0f}GB/s")
    flow(1)
    print(name, " | ".join(res), flush=True)
