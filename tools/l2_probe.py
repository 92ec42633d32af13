"""Does L2 keep a column range between the two K5 launches?  Per-column time of the
two-kernel compact-WY program at n = 1024, h = 64 as N grows from L2-resident (74 MB) to
1 GB; every size keeps >= 148 tiles so K5a runs on the full grid."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
h = int(sys.argv[2]) if len(sys.argv) > 2 else 64
for N in (18944, 28416, 37888, 75776, 151552, 262144):
    c = gi.make_case("apply", n, h, 1, "f32", seed=1)
    U = torch.from_numpy(c.U).cuda()
    X = torch.randn(N, n, device="cuda")
    Y = torch.empty_like(X)
    with hh.algo(hh.HH_ALGO_WY):
        wsb = hh.hh_workspace_bytes(hh.HH_CALL_APPLY, n, h, N, 0, X.dtype)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        f = lambda: hh.hh_apply(0, U, X, Y, workspace=ws)  # noqa: E731
        for _ in range(3):
            f()
        # a 256 MB scribble between calls: every call starts from a cold L2
        junk = torch.empty(64 << 20, device="cuda")
        ts = []
        for _ in range(10):
            junk.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    mb = N * n * 4 / 1e6
    print(f"n={n} h={h} N={N:7d} X={mb:6.0f} MB  {ms * 1e3:8.1f} us  {ms * 1e6 / N:6.3f} ns/col "
          f"{2 * mb / ms / 1e3:6.0f} GB/s (2-pass equivalent)", flush=True)
