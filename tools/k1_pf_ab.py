"""Same-box A/B of the unstaged K1's L2 prefetch distance (hh_debug_k1_prefetch: 0 = off).
usage (GPU box): python tools/k1_pf_ab.py [n:h,...]   (default: C5 h=12 and nearby shapes)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402

L = hh.hh.lib()
shapes = ([tuple(int(v) for v in s.split(":")) for s in sys.argv[1].split(",")] if len(sys.argv) > 1
          else [(4096, 12), (4096, 8), (4096, 10), (2048, 20), (2048, 24), (1024, 40)])
g = torch.Generator(device="cuda").manual_seed(1)
for n, h in shapes:
    N = (1 << 28) // n
    U = torch.randn(h, n, device="cuda", generator=g, dtype=torch.float64)
    U = (U / U.norm(dim=1, keepdim=True)).float()
    X = torch.randn(N, n, device="cuda", generator=g)
    Y = torch.empty_like(X)
    byts = 2 * N * n * 4

    def run(reps=20):
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
            return e0.elapsed_time(e1) / reps, hh.last_launch_info()

    L.hh_debug_k1_prefetch(0)
    run(3)
    ref = Y.clone()
    for rep in range(2):
        for d in (0, 1, 2, 3):
            L.hh_debug_k1_prefetch(d)
            ms, info = run()
            err = ((Y - ref).norm() / ref.norm()).item()
            print(f"n={n:5d} h={h:3d} pf={d} {info['variant']:22s} {ms * 1e3:7.1f} us "
                  f"{byts / ms / 1e6:6.0f} GB/s  diff-vs-off {err:.1e}", flush=True)
    L.hh_debug_k1_prefetch(1)
    del U, X, Y
    torch.cuda.empty_cache()
