"""Same-box A/B of the symmetric program's fused preparation (hh_debug_wy_symfuse: bit 0 the
folded block's operands in one launch, bit 1 S and P in one Gram + one reduction launch) on C3
and a two-block symmetric shape; parity of every setting against the unfused one.
usage (GPU box): python tools/symfuse_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()
cases = [("C3", gi.make_config(3)), ("sym n=4096 h=64", gi.make_case("sym", 4096, 64, 65536, "f32", seed=5)),
         ("sym n=1024 h=48", gi.make_case("sym", 1024, 48, 262144, "f32", seed=6))]
for name, c in cases:
    U, X, lam = (torch.from_numpy(v).cuda() for v in (c.U, c.X, c.lam))
    Y = torch.empty_like(X)

    def run(reps=20):
        with hh.algo(hh.HH_ALGO_WY):
            for _ in range(3):
                hh.hh_sym_apply(U, lam, X, Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                hh.hh_sym_apply(U, lam, X, Y)
            e1.record()
            torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, hh.last_launch_info()["launches"]

    res, ref = {}, None
    for rep in range(6):   # alternating order: clock drift within a round biases neither side
        for f in ((0, 1, 3) if rep % 2 == 0 else (3, 1, 0)):
            L.hh_debug_wy_symfuse(f)
            ms, nl = run()
            res.setdefault(f, []).append(ms)
            if ref is None and f == 0:
                ref = Y.clone()
            elif rep == 0:
                d = ((Y - ref).norm() / ref.norm()).item()
                print(f"{name} symfuse={f}: launches {nl}, rel diff vs unfused {d:.2e}", flush=True)
    L.hh_debug_wy_symfuse(3)
    print(name, "  ".join(f"symfuse={f}: min {min(v):.4f} median {sorted(v)[len(v) // 2]:.4f} ms "
                          f"({'/'.join('%.4f' % x for x in v)})" for f, v in sorted(res.items())), flush=True)
    del U, X, lam, Y
    torch.cuda.empty_cache()
