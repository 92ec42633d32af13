"""Debug: per-role barrier wait cycles of K5b (CTA 0, last update launch of one step)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_1811_07624_b200 as hh  # noqa: E402
from gen import inputs as gi  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 256
c = gi.make_config(5, h=h)
U, X = torch.from_numpy(c.U).cuda(), torch.from_numpy(c.X).cuda()
Y = torch.empty_like(X)
buf = torch.zeros(16, dtype=torch.int64, device="cuda")
L = hh.hh.lib()
L.hh_debug_wy_timeline.argtypes = [ctypes.c_void_p]
for _ in range(3):
    hh.hh_apply(0, U, X, Y)
L.hh_debug_wy_timeline(ctypes.c_void_p(buf.data_ptr()))
hh.hh_apply(0, U, X, Y)
torch.cuda.synchronize()
L.hh_debug_wy_timeline(None)
t = buf.cpu().tolist()
names = ["kernel", "Vprod empty-wait", "-", "MMA full-wait (V data)", "MMA acc_empty-wait",
         "Xprod xempty-wait", "-", "epi acc_full-wait", "epi xfull-wait", "MMA gfull-wait (TS)",
         "epi gempty-wait (TS)"]
for i, nm in enumerate(names):
    if nm != "-":
        print(f"{nm:24s} {t[i]:12d} cycles  {100.0 * t[i] / max(t[0], 1):6.1f} %")
