"""Same-box A/B of PDL launches in the compact-WY program (hh_debug_wy_pdl) on the WY
workloads, interleaved, 3 rounds.  usage (GPU box): python tools/pdl_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()
sys.path.insert(0, os.path.join(ROOT, "tools"))
from flow_tune import setup, timeit  # noqa: E402

for name in ["C3", "C5h64", "C5h256", "C5h1024"]:
    c, fn = setup(name)
    res = {0: [], 1: []}
    for rep in range(3):
        for on in (1, 0):
            L.hh_debug_wy_pdl(on)
            res[on].append(timeit(fn, reps=20 if name != "C5h1024" else 8))
    L.hh_debug_wy_pdl(1)
    print(f"{name:8s} PDL on {min(res[1]):.4f} ms (all {['%.4f' % x for x in res[1]]})  "
          f"off {min(res[0]):.4f} ms (all {['%.4f' % x for x in res[0]]})", flush=True)
