"""Same-box A/B of the compact-WY launch order (hh_debug_wy_pdl bits): 3 = PDL + preparation
beside the first projection (default), 1 = PDL only, 0 = neither; 3 interleaved rounds."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_1811_07624_b200 as hh  # noqa: E402
from flow_tune import setup, timeit  # noqa: E402

L = hh.hh.lib()
for name in ["C3", "C5h64", "C5h256", "C5h1024", "C5h12"]:
    c, fn = setup(name)
    res = {3: [], 1: [], 0: []}
    for rep in range(3):
        for mode in (3, 1, 0):
            L.hh_debug_wy_pdl(mode)
            res[mode].append(timeit(fn, reps=20 if name != "C5h1024" else 8))
    L.hh_debug_wy_pdl(3)
    print(f"{name:8s} " + "  ".join(f"mode{m} {min(v):.4f} ms" for m, v in res.items()), flush=True)
