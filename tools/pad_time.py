"""Unaligned strides: K1r / K1g against the padded detour over h (GPU box)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_07624_b200 as hh


def t(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


L = hh.hh.lib()
for n, N in ((1023, 262144), (101, 1 << 20), (4095, 65536), (9001, 29824)):
    for h in (4, 8, 12, 16, 20, 24, 32, 40, 56):
        U = torch.nn.functional.normalize(torch.randn(h, n, device="cuda"), dim=1)
        X = torch.randn(N, n, device="cuda")
        Y = torch.empty_like(X)
        lam = torch.rand(n, device="cuda")
        row = {"n": n, "N": N, "h": h}
        for mode, name in ((0, "direct"), (1, "padded")):
            L.hh_debug_general_pad(mode)
            hh.hh.clear_workspace_cache()
            row[name + "_ms"] = round(t(lambda: hh.hh_apply(0, U, X, Y)), 3)
            row[name + "_kernel"] = hh.last_launch_info()["variant"]
            if h <= 16:
                row[name + "_sym_ms"] = round(t(lambda: hh.hh_sym_apply(U, lam, X, Y)), 3)
        L.hh_debug_general_pad(-1)
        hh.hh.clear_workspace_cache()
        print(json.dumps(row), flush=True)
