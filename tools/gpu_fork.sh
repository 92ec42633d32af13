mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "mahalanobis or C4 or graph" -p no:cacheprovider > gpurun_out/fork_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fork_pytest.log
timeout 600 python tools/mahal_fork_ab.py > gpurun_out/fork_ab.txt 2>&1
timeout 600 python bench.py --workload C4 --steps 50 --warmup 5 --no-e2e --cpu-seconds 2 > gpurun_out/fork_bench.json 2> gpurun_out/fork_bench.err
