timeout 600 python -m pytest tests/test_congruence_gpu.py tests/test_oracle_pins.py -q -p no:cacheprovider > gpurun_out/cong_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/cong_pytest.log
for op in N T; do timeout 300 python bench.py --workload CONG --op $op --steps 30 --warmup 5 --no-e2e --cpu-seconds 2 > gpurun_out/cong_bench_$op.json 2>> gpurun_out/cong_bench.err; done
