"""K1 vs K1s (hh_stream.cu) over n x h at 1 GiB (E = 2^28 fp32), same box, interleaved; the
data behind hh_fused.cu's K1s policy.  usage (GPU box): python tools/k1s_grid.py"""
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

for n in (64, 128, 256, 512, 1024):
    N = (1 << 28) // n
    X = torch.randn(N, n, device="cuda")
    Y = torch.empty_like(X)
    for h in (2, 4, 6, 8, 10, 12, 16, 24, 32):
        c = gi.make_case("apply", n, h, 1, "f32", seed=4)
        U = torch.from_numpy(c.U).cuda()
        f = lambda: hh.hh_apply(0, U, X, Y)  # noqa: E731
        t = {}
        with hh.algo(hh.HH_ALGO_FUSED):
            for rep in range(2):
                for on in (0, 1):
                    L.hh_debug_k1_stream(on)
                    v = timeit(f, reps=15)
                    t[on] = min(t.get(on, 9e9), v)
        L.hh_debug_k1_stream(0)
        print(f"n={n:5d} h={h:3d}  K1 {t[0] * 1e3:7.1f} us  K1s {t[1] * 1e3:7.1f} us  "
              f"ratio {t[1] / t[0]:.3f}", flush=True)
