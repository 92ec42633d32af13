timeout 500 python tools/k1s_mw_ab.py > gpurun_out/ab3_mw.txt 2>&1
cat > /tmp/c2pf.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
import paper_1811_07624_b200 as hh
from gen import inputs as gi
from flow_tune import timeit
L = hh.hh.lib()
c = gi.make_config(2)
U, X = torch.from_numpy(c.U).cuda(), torch.from_numpy(c.X).cuda()
Y = torch.empty_like(X)
t = {}
for rep in range(3):
    for k in (0, 1, 2):
        L.hh_debug_k1_stream(k)
        for op in (0, 1):
            v = timeit(lambda: hh.hh_apply(op, U, X, Y), reps=30)
            t[(k, op)] = min(t.get((k, op), 9e9), v)
L.hh_debug_k1_stream(-1)
for k, nm in ((0, "K1"), (1, "K1s"), (2, "K1s-pf")):
    print(f"C2 {nm:7s} op N {t[(k,0)]*1e3:7.1f} us  op T {t[(k,1)]*1e3:7.1f} us", flush=True)
PY
timeout 300 python /tmp/c2pf.py > gpurun_out/ab3_c2pf.txt 2>&1
