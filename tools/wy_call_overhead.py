"""Host and device cost of one K5 (compact-WY) apply call at a given shape: host microseconds per
eager call (GPU kept busy), eager event time, CUDA-graph replay time, launches per call.
usage: python tools/wy_call_overhead.py n h N   (evidence: profiles/r1/crossover_r1.txt)"""
import sys, time, torch
sys.path.insert(0, ".")
import paper_1811_07624_b200 as hh
n, h, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = torch.Generator(device="cuda").manual_seed(1)
X = torch.randn(N, n, device="cuda", generator=g); Y = torch.empty_like(X)
U = torch.nn.functional.normalize(torch.randn(h, n, device="cuda", generator=g), dim=1).contiguous()
ws = torch.empty(hh.hh_workspace_bytes(hh.HH_CALL_APPLY, n, h, N, 0, torch.float32), dtype=torch.uint8, device="cuda")
with hh.algo(hh.HH_ALGO_WY):
    for _ in range(5): hh.hh_apply(1, U, X, Y, workspace=ws)
    torch.cuda.synchronize()
    # host cost of one call (GPU kept busy so the launch queue never drains)
    hs = []
    for _ in range(20):
        t0 = time.perf_counter(); hh.hh_apply(1, U, X, Y, workspace=ws); hs.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    hs.sort(); print(f"host us per call (median): {hs[len(hs)//2]*1e6:.1f}")
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); hh.hh_apply(1, U, X, Y, workspace=ws); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    ts.sort(); print(f"eager event us: {ts[len(ts)//2]:.1f}")
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): hh.hh_apply(1, U, X, Y, workspace=ws)
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr): hh.hh_apply(1, U, X, Y, workspace=ws)
    gr.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): gr.replay()
    b.record(); b.synchronize(); print(f"graph replay us: {a.elapsed_time(b)*1e3/50:.1f}")
    print("launch info:", hh.last_launch_info())
