"""Ragged aligned shapes on the TMEM forms (K1t / K1w): timing (GPU box)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_07624_b200 as hh


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n, h in ((3000, 12), (2560, 12), (1536, 12), (3000, 16), (1000, 14), (4000, 8), (4096, 12), (900, 16)):
    N = (1 << 28) // n
    U = torch.nn.functional.normalize(torch.randn(h, n, device="cuda"), dim=1)
    X = torch.randn(N, n, device="cuda")
    Y = torch.empty_like(X)
    with hh.algo(hh.HH_ALGO_FUSED):
        ms = t(lambda: hh.hh_apply(0, U, X, Y))
    print(json.dumps({"n": n, "h": h, "N": N, "ms": round(ms, 4), "GBps": round(2 * X.numel() * 4 / ms / 1e6, 1),
                      "kernel": hh.last_launch_info()["variant"]}), flush=True)
