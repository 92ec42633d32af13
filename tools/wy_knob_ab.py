"""Same-box A/B of one compact-WY debug knob (hh_debug_wy_<name>, one int argument) on the WY
workloads, alternating order; outputs must be bit-identical across the values.
usage (GPU box): python tools/wy_knob_ab.py rev 0,1 [C3,C5h64,C5h256,C5h1024]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()
knob = getattr(L, "hh_debug_wy_" + sys.argv[1])
vals = [int(v) for v in sys.argv[2].split(",")]
names = sys.argv[3].split(",") if len(sys.argv) > 3 else ["C3", "C5h64", "C5h256", "C5h1024"]
for name in names:
    c = gi.make_config(3) if name == "C3" else gi.make_config(5, h=int(name[3:]))
    U, X = torch.from_numpy(c.U).cuda(), torch.from_numpy(c.X).cuda()
    Y = torch.empty_like(X)
    lam = torch.from_numpy(c.lam).cuda() if c.call == "sym" else None

    def fn():
        with hh.algo(hh.HH_ALGO_WY):
            if lam is not None:
                hh.hh_sym_apply(U, lam, X, Y)
            else:
                hh.hh_apply(0, U, X, Y)
    outs, res = {}, {v: [] for v in vals}
    for v in vals:
        knob(v)
        fn()
        torch.cuda.synchronize()
        outs[v] = Y.clone()
    same = all(torch.equal(outs[vals[0]], outs[v]) for v in vals)
    reps = 20 if name != "C5h1024" else 6
    for rep in range(6):
        for v in (vals if rep % 2 == 0 else vals[::-1]):
            knob(v)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res[v].append(e0.elapsed_time(e1) / reps)
    knob(vals[0])
    print(name, "bit-identical" if same else "DIFFERS", "  ".join(
        f"{sys.argv[1]}={v}: min {min(r):.4f} median {sorted(r)[3]:.4f}" for v, r in res.items()), flush=True)
