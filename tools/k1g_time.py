"""Timing of K1g (the any-shape kernel) next to K1 on neighbouring shapes (GPU box)."""
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


for n, h, N in ((1024, 10, 262144), (1023, 10, 262144), (100, 7, 1 << 20), (101, 7, 1 << 20),
                (4096, 12, 65536), (4095, 12, 65536), (4097, 12, 65536), (2047, 12, 131072), (1023, 16, 262144),
                (16384, 8, 16384), (201, 16, 1 << 19)):
    U = torch.nn.functional.normalize(torch.randn(h, n, device="cuda"), dim=1)
    X = torch.randn(N, n, device="cuda")
    Y = torch.empty_like(X)
    ms = t(lambda: hh.hh_apply(0, U, X, Y))
    row = {"n": n, "h": h, "N": N, "ms": round(ms, 4), "GBps": round(2 * X.numel() * 4 / ms / 1e6, 1),
           "kernel": hh.last_launch_info()["variant"]}
    if "r_" in row["kernel"]:   # K1r: columns straight into registers instead of staged tiles
        hh.hh.lib().hh_debug_k1r_stage(0)
        row["nostage_ms"] = round(t(lambda: hh.hh_apply(0, U, X, Y)), 4)
        hh.hh.lib().hh_debug_k1r_stage(1)
    if "r_" in row["kernel"] and h <= 16 and 512 < n <= 4096:   # K1r: both forms
        hh.hh.lib().hh_debug_k1r_tmem(0)
        row["smem_ms"] = round(t(lambda: hh.hh_apply(0, U, X, Y)), 4)
        hh.hh.lib().hh_debug_k1r_tmem(1)
    print(json.dumps(row))
