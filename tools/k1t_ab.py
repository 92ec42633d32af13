"""Same-box A/B of K1 with the reflectors in shared memory vs in TMEM (K1t,
hh_debug_k1_tmem), plus K1s where it applies; outputs must be bit-identical.
usage (GPU box): python tools/k1t_ab.py [n:h[:op],...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402

L = hh.hh.lib()
DEFAULT = "1024:10,1024:10:1,4096:12,4096:8,4096:16,2048:12,2048:16,1024:16,1000:10,512:10,256:8,4096:12:2"
spec = sys.argv[1] if len(sys.argv) > 1 else DEFAULT
g = torch.Generator(device="cuda").manual_seed(1)
for item in spec.split(","):
    f = [int(v) for v in item.split(":")]
    n, h, op = f[0], f[1], (f[2] if len(f) > 2 else 0)
    N = (1 << 28) // n
    U = torch.randn(h, n, device="cuda", generator=g, dtype=torch.float64)
    U = (U / U.norm(dim=1, keepdim=True)).float()
    X = torch.randn(N, n, device="cuda", generator=g)
    lam = torch.rand(n, device="cuda", generator=g)
    Y = torch.empty_like(X)
    byts = 2 * N * n * 4

    def call():
        if op == 2:
            hh.hh_sym_apply(U, lam, X, Y)
        else:
            hh.hh_apply(op, U, X, Y)

    def run(reps=20):
        with hh.algo(hh.HH_ALGO_FUSED):
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                call()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps, hh.last_launch_info()

    L.hh_debug_k1_stream(0)
    L.hh_debug_k1_tmem(0)
    run(2)
    ref = Y.clone()
    for rep in range(2):
        for name, st, tm in (("K1 smem-u", 0, 0), ("K1t tmem-u", 0, 1), ("K1s", 1, 0)):
            if st == 1 and n > 1024:
                continue
            L.hh_debug_k1_stream(st)
            L.hh_debug_k1_tmem(tm)
            try:
                ms, info = run()
            except Exception as e:  # noqa: BLE001
                print(f"n={n} h={h} op={op} {name}: {e}", flush=True)
                continue
            d = (Y - ref).abs().max().item()
            print(f"n={n:5d} h={h:3d} op={op} {name:11s} {info.get('variant', '?'):26s} {ms * 1e3:7.1f} us "
                  f"{byts / ms / 1e6:6.0f} GB/s  maxdiff {d:.1e}", flush=True)
    L.hh_debug_k1_stream(-1)
    L.hh_debug_k1_tmem(-1)
    del U, X, Y
    torch.cuda.empty_cache()
