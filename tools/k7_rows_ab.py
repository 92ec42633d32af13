"""Same-box A/B of the congruence row kernel K7 with 2 or 4 rows per warp pass
(hh_debug_k7_rows) on CONG-shaped batches (and ragged n): bit-identity, then timing in
alternating order.  usage (GPU box): python tools/k7_rows_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402

L = hh.hh.lib()
g = torch.Generator(device="cuda").manual_seed(7)
for n, h, cnt in ((512, 18, 64), (500, 9, 40), (256, 16, 256), (128, 7, 512), (1024, 20, 16)):
    U = torch.randn(h, n, device="cuda", generator=g, dtype=torch.float64)
    U = (U / U.norm(dim=1, keepdim=True)).float()
    M = torch.randn(cnt, n, n, device="cuda", generator=g)
    outs, res = {}, {2: [], 4: []}
    for op in (0, 1):
        for rw in (2, 4):
            L.hh_debug_k7_rows(rw)
            outs[(op, rw)] = hh.hh_congruence(op, U, M).clone()
        same = torch.equal(outs[(op, 2)], outs[(op, 4)])
        print(f"n={n} h={h} count={cnt} op={op}: {'bit-identical' if same else 'DIFFERS'}", flush=True)
    ws = torch.empty(hh.hh_workspace_bytes(hh.HH_CALL_CONGRUENCE, n, h, cnt, 0, M.dtype), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(M)
    for rep in range(6):
        for rw in ((2, 4) if rep % 2 == 0 else (4, 2)):
            L.hh_debug_k7_rows(rw)
            for _ in range(3):
                hh.hh_congruence(0, U, M, out, workspace=ws)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                hh.hh_congruence(0, U, M, out, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            res[rw].append(e0.elapsed_time(e1) / 20)
    print(f"n={n} h={h} count={cnt}: " + "  ".join(f"rows={rw}: min {min(v) * 1e3:.1f} median {sorted(v)[3] * 1e3:.1f} us"
                                                   for rw, v in res.items()), flush=True)
    L.hh_debug_k7_rows(-1)
