mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_shf_gpu.py tests/test_abi.py -m gpu -q -x -p no:cacheprovider > gpurun_out/shf_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/shf_pytest.log
timeout 300 python - > gpurun_out/shf_time.txt 2>&1 <<'PY'
import torch, paper_1811_07624_b200 as hh
for n, K in ((512, 256), (1024, 256), (2048, 128)):
    for dt in (torch.float32, torch.float64):
        A = torch.randn(n, n, device="cuda", dtype=dt); A = (A + A.T) / 2
        B = torch.randn(n, n, device="cuda", dtype=dt); B = (B + B.T) / 2
        U = torch.randn(K, n, device="cuda", dtype=dt)
        ws = torch.empty(hh.hh_workspace_bytes(hh.HH_CALL_SHF, n, 0, K, 0, dt), dtype=torch.uint8, device="cuda")
        c = torch.empty(K, device="cuda", dtype=dt); g = torch.empty_like(U)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3): hh.hh_shf_cost(A, B, U, cost=c, grad_out=g, workspace=ws)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(20): hh.hh_shf_cost(A, B, U, cost=c, grad_out=g, workspace=ws)
        gr.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): gr.replay()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 100
        print(f"n={n} K={K} {dt}: {ms*1e3:.1f} us  {8*n*n*K/ms/1e9:.1f} TFLOP/s (8 n^2 K)", flush=True)
PY
python - > gpurun_out/shf_launch.txt 2>&1 <<'PY'
import torch, paper_1811_07624_b200 as hh
n, K = 1024, 256
A = torch.randn(n, n, device="cuda"); A = (A + A.T) / 2
B = torch.randn(n, n, device="cuda"); B = (B + B.T) / 2
U = torch.randn(K, n, device="cuda")
for _ in range(5): hh.hh_shf_cost(A, B, U)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/shf_launches.csv python - <<'PY' > /dev/null 2>&1
import torch, paper_1811_07624_b200 as hh
n, K = 1024, 256
A = torch.randn(n, n, device="cuda"); A = (A + A.T) / 2
B = torch.randn(n, n, device="cuda"); B = (B + B.T) / 2
U = torch.randn(K, n, device="cuda")
for _ in range(3): hh.hh_shf_cost(A, B, U)
torch.cuda.synchronize()
PY
