"""K1 (fused SIMT) vs K5 (compact WY) sweep behind `wy_min_h` (hh_api.cu).

Times `Y = Q^T X` through hh_apply with the path forced, for each h of a list, at a fixed problem
size E = n*N = 2^s fp32 elements: median of 30 calls, each bracketed by CUDA events on the current
stream (eager launches, so K5's host-side chain cost is included as a caller sees it).
usage: python tools/crossover_sweep.py n fused|wy|fused-sym|wy-sym h1,h2,... [s=28]
(the -sym paths time Y = Q diag(lam) Q^T X through hh_sym_apply)
Output lines: n=.. N=.. path h=.. <us> us <GB/s of one read + one write of X>.
Evidence of the current thresholds: profiles/r1/crossover_r1.txt.
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1811_07624_b200 as hh  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    path = sys.argv[2] if len(sys.argv) > 2 else "fused"
    hs = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [4, 8, 12, 16, 20, 24, 32]
    N = (1 << int(sys.argv[4] if len(sys.argv) > 4 else 28)) // n
    algo = hh.HH_ALGO_WY if path.startswith("wy") else hh.HH_ALGO_FUSED
    sym = path.endswith("-sym")
    g = torch.Generator(device="cuda").manual_seed(1)
    X = torch.randn(N, n, device="cuda", generator=g)
    Y = torch.empty_like(X)
    lam = torch.exp(-torch.arange(n, device="cuda") / 200.0)

    def call(U):
        if sym:
            hh.hh_sym_apply(U, lam, X, Y)
        else:
            hh.hh_apply(1, U, X, Y)
    for h in hs:
        U = torch.randn(max(h, 1), n, device="cuda", generator=g)
        U = torch.nn.functional.normalize(U, dim=1)[:h].contiguous()
        with hh.algo(algo):
            for _ in range(5):
                call(U)
            torch.cuda.synchronize()
            ts = []
            for _ in range(30):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                call(U)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
        ts.sort()
        t = ts[len(ts) // 2]
        print(f"n={n} N={N} {path} h={h:3d} {t * 1e3:8.1f} us  {2 * N * n * 4 / t / 1e6:7.0f} GB/s",
              flush=True)


if __name__ == "__main__":
    main()
