"""Same-box A/B of hh_mahalanobis with the pair sort on a second stream beside the transform
(hh_debug_mahal_fork 1, default) or on the caller's stream (0), C4 shape, interleaved rounds;
outputs must be bit-identical.  usage (GPU box): python tools/mahal_fork_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()
c = gi.make_config(4)
U, d, P = (torch.from_numpy(v).cuda() for v in (c.U, c.d, c.X))
ia, ib = torch.from_numpy(c.ia).cuda(), torch.from_numpy(c.ib).cuda()
ws = torch.empty(hh.hh_workspace_bytes(hh.HH_CALL_MAHALANOBIS, c.n, c.h, P.shape[0], ia.numel(), P.dtype),
                 dtype=torch.uint8, device="cuda")
dist = torch.empty(ia.numel(), device="cuda", dtype=torch.float32)


def run(reps=50):
    for _ in range(3):
        hh.hh_mahalanobis(U, d, P, ia, ib, dist, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        hh.hh_mahalanobis(U, d, P, ia, ib, dist, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


outs = {}
res = {0: [], 1: []}
for rep in range(4):
    for f in (1, 0):
        L.hh_debug_mahal_fork(f)
        res[f].append(run())
        outs[f] = dist.clone()
L.hh_debug_mahal_fork(1)
print("fork on : " + " ".join("%.4f" % x for x in res[1]) + " ms")
print("fork off: " + " ".join("%.4f" % x for x in res[0]) + " ms")
print("max |diff| on vs off:", (outs[1] - outs[0]).abs().max().item())
