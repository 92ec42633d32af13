timeout 300 python -m pytest tests/test_congruence_gpu.py -q -p no:cacheprovider > gpurun_out/k7_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k7_pytest.log
out=gpurun_out/k7ab.txt; : > $out
for rep in 1 2 3; do
  for lib in abtest/libhh_k7a.so abtest/libhh_k7b.so; do
    HH_LIB_PATH=$lib timeout 200 python bench.py --workload CONG --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/k7ab.err | python -c "import sys,json; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$lib', round(d['ms_per_step'],4))" >> $out
  done
done
