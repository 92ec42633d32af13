"""Same-box A/B of the K5b epilogue: X boxes through shared memory (default) vs straight from
global memory (hh_debug_wy_pdl bit 2), with a parity check of the direct form against the
oracle on a small case first.  usage (GPU box): python tools/direct_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1811_07624_b200 as hh  # noqa: E402
from flow_tune import setup, timeit  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()
L.hh_debug_wy_pdl(3 | 4)
for n, h, N, op in ((512, 64, 40000, 0), (1000, 257, 300, 1), (2048, 32, 3000, 0)):
    c = gi.make_case("apply", n, h, N, "f32", seed=9)
    with hh.algo(hh.HH_ALGO_WY):
        Y = hh.hh_apply(op, torch.from_numpy(c.U).cuda(), torch.from_numpy(c.X).cuda()).cpu().numpy()
    ref = oracle.apply(op, c.U, c.X)
    print(f"direct parity n={n} h={h} N={N}: {np.linalg.norm(Y - ref) / np.linalg.norm(ref):.2e}", flush=True)
c = gi.make_case("sym", 2048, 32, 3000, "f32", seed=9)
with hh.algo(hh.HH_ALGO_WY):
    Y = hh.hh_sym_apply(torch.from_numpy(c.U).cuda(), torch.from_numpy(c.lam).cuda(),
                        torch.from_numpy(c.X).cuda()).cpu().numpy()
ref = oracle.sym_apply(c.U, c.lam, c.X)
print(f"direct parity sym: {np.linalg.norm(Y - ref) / np.linalg.norm(ref):.2e}", flush=True)
for name in ["C3", "C5h64", "C5h12"]:
    c, fn = setup(name)
    res = {3: [], 7: []}
    for rep in range(3):
        for mode in (3, 7):
            L.hh_debug_wy_pdl(mode)
            res[mode].append(timeit(fn, reps=20))
    print(f"{name:8s} smem-boxes {min(res[3]):.4f} ms   direct {min(res[7]):.4f} ms", flush=True)
L.hh_debug_wy_pdl(3)
