"""K5a with X converted into TMEM (hh_debug_wy_tsa 1) against the shared-memory form (0):
bit-identity of the outputs on WY shapes (ragged n / N, both ops, symmetric, QR, D), then a
same-box timing of C3 / C5 h=64 / C5 h=256 in alternating order.
usage (GPU box): python tools/wy_tsa_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

L = hh.hh.lib()
t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
bad = 0
MODES = [int(v) for v in os.environ.get("TSA_MODES", "0,1").split(",")]
for (n, h, N) in [(1024, 64, 40000), (1000, 40, 3001), (4096, 96, 700), (2048, 33, 20000), (512, 128, 9000),
                  (1024, 256, 30000), (3000, 700, 2000)]:
    c = gi.make_case("sym", n, h, N, "f32", seed=3)
    d = gi.sign_diag(gi.rng(3, n), n, "f32")
    outs = {}
    for on in (MODES[0], MODES[-1]):
        L.hh_debug_wy_tsa(on)
        with hh.algo(hh.HH_ALGO_WY):
            r = [hh.hh_apply(op, t(c.U), t(c.X)) for op in (0, 1)]
            r.append(hh.hh_sym_apply(t(c.U), t(c.lam), t(c.X)))
            r.append(hh.hh_apply_signed(0, 1, t(c.U), t(d), t(c.X)))
        outs[on] = r
    for i, (a, b) in enumerate(zip(outs[MODES[0]], outs[MODES[-1]])):
        same = torch.equal(a, b)
        bad += not same
        print(f"n={n} h={h} N={N} call {i}: {'bit-identical' if same else 'DIFFERS max %.3e' % (a - b).abs().max().item()}",
              flush=True)
L.hh_debug_wy_tsa(1)
print("mismatches:", bad, flush=True)


def setup(name):
    c = gi.make_config(3) if name == "C3" else gi.make_config(5, h=int(name[3:]))
    U, X = t(c.U), t(c.X)
    Y = torch.empty_like(X)
    lam = t(c.lam) if c.call == "sym" else None

    def fn():
        with hh.algo(hh.HH_ALGO_WY):
            if lam is not None:
                hh.hh_sym_apply(U, lam, X, Y)
            else:
                hh.hh_apply(0, U, X, Y)
    return fn


def timeit(fn, reps=20):
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


for name in os.environ.get("TSA_WL", "C3,C5h64,C5h256,C5h1024").split(","):
    fn = setup(name)
    res = {m: [] for m in MODES}
    for rep in range(6):
        for on in (MODES if rep % 2 == 0 else MODES[::-1]):
            L.hh_debug_wy_tsa(on)
            res[on].append(timeit(fn, 20 if name != "C5h1024" else 6))
    L.hh_debug_wy_tsa(1)
    print(name, "  ".join(f"tsa={on}: min {min(v):.4f} median {sorted(v)[3]:.4f} ms" for on, v in res.items()),
          flush=True)
