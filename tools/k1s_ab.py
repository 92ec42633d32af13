"""Same-box A/B: K1 (persistent, staged) vs K1s (non-persistent streaming, hh_stream.cu) on
C2 (both ops), C4 (the transform-once K3a inside hh_mahalanobis) and small-n shapes; parity of
K1s against K1 on the same inputs.  usage (GPU box): python tools/k1s_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()


def timeit(fn, reps=30):
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


cases = []
c2 = gi.make_config(2)
U2, X2 = torch.from_numpy(c2.U).cuda(), torch.from_numpy(c2.X).cuda()
Y2 = torch.empty_like(X2)
for op in (0, 1):
    cases.append((f"C2 op{op}", 2 * X2.numel() * 4, lambda op=op: hh.hh_apply(op, U2, X2, Y2), Y2))
c4 = gi.make_config(4)
A4 = [torch.from_numpy(a).cuda() for a in (c4.U, c4.d, c4.X, c4.ia, c4.ib)]
D4 = torch.empty(c4.npairs, device="cuda")
wsb = hh.hh_workspace_bytes(hh.HH_CALL_MAHALANOBIS, c4.n, c4.h, c4.N, c4.npairs, torch.float32)
W4 = torch.empty(wsb, dtype=torch.uint8, device="cuda")
cases.append(("C4", c4.N * c4.n * 4, lambda: hh.hh_mahalanobis(*A4, dist=D4, workspace=W4), D4))
for n, h, N in ((512, 9, 1 << 19), (256, 8, 1 << 20), (128, 7, 1 << 21), (64, 6, 1 << 22), (1024, 4, 1 << 18)):
    c = gi.make_case("apply", n, h, 1, "f32", seed=3)
    U = torch.from_numpy(c.U).cuda()
    X = torch.randn(N, n, device="cuda")
    Y = torch.empty_like(X)
    cases.append((f"n{n} h{h} N{N}", 2 * X.numel() * 4, lambda U=U, X=X, Y=Y: hh.hh_apply(0, U, X, Y), Y))

for name, byts, fn, out in cases:
    res = []
    ref = None
    for rep in range(2):
        for on in (0, 1):
            L.hh_debug_k1_stream(on)
            ms = timeit(fn)
            info = hh.last_launch_info()
            if ref is None and on == 0:
                ref = out.clone()
            err = ((out.float() - ref.float()).norm() / ref.float().norm()).item()
            res.append(f"{'K1s' if on else 'K1 '} {ms * 1e3:7.1f}us {byts / ms / 1e6:5.0f}GB/s "
                       f"[{info['variant']}] d={err:.0e}")
    L.hh_debug_k1_stream(0)
    print(f"{name:22s} " + " | ".join(res), flush=True)
