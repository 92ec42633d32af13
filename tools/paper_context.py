"""Paper-shaped context rows (not graded): synthetic stand-ins for the
Table I test-time transforms of PAPER.md -- n = 100 / 200 / 40 with the test
split sizes and h in {ceil(log2 n), ceil(2 log2 n), ceil(3 log2 n)}; iid N(0,1) columns stand
in for the datasets, which are not in the container.  Each shape is applied as Q^T X (the
transform x <- Q^T x of P:668) through hh_apply, timed per call with CUDA events (median of
200) and as a CUDA-graph replay of 20 calls (launch cost amortised), parity-checked against
the oracle.  usage: python tools/paper_context.py
"""
import math
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402


def main():
    s = torch.cuda.Stream()
    print(f"{'n':>4} {'h':>3} {'N':>6}  {'call us':>8} {'vec/s (call)':>13}  {'graph us':>9} "
          f"{'vec/s (graph)':>14}  {'rel err':>9} {'gate':>9}")
    for n, h, N in gi.paper_context_shapes():
        c = gi.make_case("apply", n, h, N, "f32", seed=7)
        U, X = torch.from_numpy(c.U).cuda(), torch.from_numpy(c.X).cuda()
        Y = torch.empty_like(X)
        with torch.cuda.stream(s):
            for _ in range(20):
                hh.hh_apply(1, U, X, Y)
            torch.cuda.synchronize()
            times = []
            for _ in range(200):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                hh.hh_apply(1, U, X, Y)
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1) * 1e3)
        t_call = statistics.median(times)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                hh.hh_apply(1, U, X, Y)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        e1.synchronize()
        t_graph = e0.elapsed_time(e1) * 1e3 / 200
        ref = oracle.apply(1, c.U, c.X)
        err = float(np.linalg.norm(Y.cpu().numpy() - ref) / np.linalg.norm(ref))
        gate = 2e-5 * math.sqrt(h)
        print(f"{n:4d} {h:3d} {N:6d}  {t_call:8.1f} {N / t_call * 1e6:13.3g}  {t_graph:9.2f} "
              f"{N / t_graph * 1e6:14.3g}  {err:9.2e} {gate:9.2e}", flush=True)
        assert err <= gate


if __name__ == "__main__":
    main()
