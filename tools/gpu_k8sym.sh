mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_shf_gpu.py tests/test_wy_gpu.py tests/test_fullsize_gpu.py -k "shf or sym or C3" -m gpu -q -x -p no:cacheprovider > gpurun_out/k8s_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/k8s_pytest.log
timeout 300 python tools/symfuse_ab.py > gpurun_out/k8s_symfuse.txt 2>&1
for i in 1 2; do timeout 300 python bench.py --workload SHF --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/k8s_shf.jsonl 2>/dev/null; timeout 300 python bench.py --workload C3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/k8s_c3.jsonl 2>/dev/null; done
