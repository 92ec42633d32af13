"""Same-box A/B of K1t (TMEM reflectors) against its blocked form K1w at block sizes 2 / 4 / 8
(hh_debug_k1_blocked, the kb2 / kb8 forms through hh_debug_k1's alternative table) and the
staged-path L2 prefetch two tiles ahead (hh_debug_k1_prefetch).
usage (GPU box): python tools/k1w_ab.py [n:h[:op],...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402

L = hh.hh.lib()
DEFAULT = "4096:12,4096:8,4096:10,4096:16,2048:12,2048:10,2048:16"
ALT = {(4096, 2): 4, (4096, 8): 5, (2048, 2): 6, (2048, 8): 7}   # kF32Alt indices
spec = sys.argv[1] if len(sys.argv) > 1 else DEFAULT
g = torch.Generator(device="cuda").manual_seed(1)
for item in spec.split(","):
    f = [int(v) for v in item.split(":")]
    n, h, op = f[0], f[1], (f[2] if len(f) > 2 else 0)
    N = (1 << 28) // n
    U = torch.randn(h, n, device="cuda", generator=g, dtype=torch.float64)
    U = (U / U.norm(dim=1, keepdim=True)).float()
    X = torch.randn(N, n, device="cuda", generator=g)
    Y = torch.empty_like(X)
    byts = 2 * N * n * 4

    def run(reps=20):
        with hh.algo(hh.HH_ALGO_FUSED):
            for _ in range(3):
                hh.hh_apply(op, U, X, Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                hh.hh_apply(op, U, X, Y)
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps, hh.last_launch_info()

    L.hh_debug_k1_stream(0)
    L.hh_debug_k1_tmem(1)
    L.hh_debug_k1_blocked(0)
    run(2)
    ref = Y.clone()
    cfgs = [("K1t", 0, -1, 0), ("K1w kb4", 1, -1, 0), ("K1w kb2", 1, ALT.get((n, 2), -1), 0),
            ("K1w kb8", 1, ALT.get((n, 8), -1), 0), ("K1t pf2", 0, -1, 2), ("K1w kb4 pf2", 1, -1, 2)]
    for rep in range(2):
        for name, bk, alt, pf in cfgs:
            L.hh_debug_k1_blocked(bk)
            L.hh_debug_k1(alt, 1)
            L.hh_debug_k1_prefetch(pf)
            ms, info = run()
            d = ((Y - ref).norm() / ref.norm()).item()
            print(f"n={n:5d} h={h:3d} op={op} {name:12s} {info.get('variant', '?'):30s} {ms * 1e3:7.1f} us "
                  f"{byts / ms / 1e6:6.0f} GB/s  reldiff {d:.1e}", flush=True)
    L.hh_debug_k1(-1, 1)
    L.hh_debug_k1_prefetch(0)
    L.hh_debug_k1_stream(-1)
    L.hh_debug_k1_tmem(-1)
    L.hh_debug_k1_blocked(-1)
    del U, X, Y
    torch.cuda.empty_cache()
