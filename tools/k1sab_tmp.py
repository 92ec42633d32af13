import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
import paper_1811_07624_b200 as hh
from gen import inputs as gi
from flow_tune import timeit
tag = os.environ.get("HH_LIB_PATH", "")
for n, h in ((128, 8), (256, 8), (512, 9), (512, 16), (1024, 4)):
    N = (1 << 28) // n
    X = torch.randn(N, n, device="cuda"); Y = torch.empty_like(X)
    c = gi.make_case("apply", n, h, 1, "f32", seed=4); U = torch.from_numpy(c.U).cuda()
    with hh.algo(hh.HH_ALGO_FUSED):
        t = min(timeit(lambda: hh.hh_apply(0, U, X, Y), reps=20) for _ in range(2))
    print(os.path.basename(tag), f"n={n} h={h} {t*1e3:.1f} us", flush=True)
