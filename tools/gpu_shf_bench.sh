mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_bench_gpu.py -m gpu -q -x -k "SHF" -p no:cacheprovider > gpurun_out/shfb_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/shfb_pytest.log
timeout 600 python bench.py --workload SHF --steps 50 --warmup 5 --no-e2e --cpu-seconds 3 > gpurun_out/shf_bench.json 2> gpurun_out/shf_bench.err
timeout 600 python bench.py --impl reference --workload SHF --steps 3 --warmup 3 > gpurun_out/shf_ref.json 2>> gpurun_out/shf_bench.err
