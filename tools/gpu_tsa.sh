mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_wy_gpu.py tests/test_fullsize_gpu.py tests/test_qr_gpu.py tests/test_signed_gpu.py tests/test_fuzz_gpu.py tests/test_graph_gpu.py tests/test_congruence_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/tsa_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tsa_pytest.log
for w in C3 C5h64; do timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --cpu-seconds 2 >> gpurun_out/tsa_sweep.jsonl 2>/dev/null; done
