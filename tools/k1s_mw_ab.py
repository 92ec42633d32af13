"""K1 vs the multi-warp K1s (hh_stream.cu, n in (1024, 4096]) at 1 GiB, same box, interleaved,
with a parity check of K1s against K1.  usage (GPU box): python tools/k1s_mw_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()
sys.path.insert(0, os.path.join(ROOT, "tools"))
from flow_tune import timeit  # noqa: E402

for n in (2048, 4096):
    N = (1 << 28) // n
    X = torch.randn(N, n, device="cuda")
    Y = torch.empty_like(X)
    for h in (4, 8, 12, 16):
        c = gi.make_case("apply", n, h, 1, "f32", seed=4)
        U = torch.from_numpy(c.U).cuda()
        f = lambda: hh.hh_apply(0, U, X, Y)  # noqa: E731
        t, outs = {}, {}
        with hh.algo(hh.HH_ALGO_FUSED):
            for rep in range(2):
                for on in (0, 1):
                    L.hh_debug_k1_stream(on)
                    t[on] = min(t.get(on, 9e9), timeit(f, reps=15))
                    if rep == 0:
                        outs[on] = (Y.clone(), hh.last_launch_info()["variant"])
        L.hh_debug_k1_stream(-1)
        d = ((outs[1][0] - outs[0][0]).norm() / outs[0][0].norm()).item()
        print(f"n={n} h={h:3d} K1 {t[0] * 1e3:7.1f} us [{outs[0][1]}]  K1s {t[1] * 1e3:7.1f} us "
              f"[{outs[1][1]}] ratio {t[1] / t[0]:.3f}  rel-diff {d:.1e}", flush=True)
