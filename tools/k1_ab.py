"""Same-box A/B of K1 shapes for one workload: the default variant, forced alternatives
(hh_debug_k1 alt index) and persistent-grid multipliers; CUDA-event timing, parity of each
alternative against the default output.  usage (GPU box): python tools/k1_ab.py C2 [alts]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()
name = sys.argv[1]
alts = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3]
c = gi.make_config(2) if name == "C2" else gi.make_config(5, h=int(name[3:]))
U, X = torch.from_numpy(c.U).cuda(), torch.from_numpy(c.X).cuda()
Y = torch.empty_like(X)
byts = 2 * c.N * c.n * 4


def run(reps=30):
    with hh.algo(hh.HH_ALGO_FUSED):
        for _ in range(3):
            hh.hh_apply(0, U, X, Y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            hh.hh_apply(0, U, X, Y)
        e1.record()
        torch.cuda.synchronize()
        info = hh.last_launch_info()
    return e0.elapsed_time(e1) / reps, info


L.hh_debug_k1(-1, 1)
run()
ref = Y.clone()
configs = [(-1, 1)] + [(a, 1) for a in alts] + [(-1, g) for g in (2, 3, 4)]
for rep in range(2):
    for a, g in configs:
        L.hh_debug_k1(a, g)
        ms, info = run()
        err = ((Y - ref).norm() / ref.norm()).item()
        print(f"{name} alt={a:2d} gridx={g} {info['variant']:24s} grid {info['grid']:5d} "
              f"{ms * 1e3:7.1f} us {byts / ms / 1e6:6.0f} GB/s  rel-vs-default {err:.1e}", flush=True)
L.hh_debug_k1(-1, 1)
