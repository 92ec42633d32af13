"""Debug: run the compact-WY path on growing N and report the first failing size."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_07624_b200 as hh  # noqa: E402

n, h = int(sys.argv[1]), int(sys.argv[2])
Ns = [int(x) for x in sys.argv[3].split(",")]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
g = torch.Generator(device="cuda").manual_seed(0)
for N in Ns:
    U = torch.randn(h, n, device="cuda", generator=g)
    U /= U.norm(dim=1, keepdim=True)
    X = torch.randn(N, n, device="cuda", generator=g)
    with hh.algo(hh.HH_ALGO_WY):
        for r in range(reps):
            Y = hh.hh_apply(0, U, X)
            torch.cuda.synchronize()
    print("ok", N, float(Y.norm() / X.norm()), flush=True)
