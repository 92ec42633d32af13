out=gpurun_out/ab6.txt; : > $out
for rep in 1 2 3; do
  for lib in abtest/libhh_base.so abtest/libhh_fadd2.so; do
    for op in N T; do
      HH_LIB_PATH=$lib timeout 200 python bench.py --workload C2 --op $op --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/ab6.err | python -c "import sys,json; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$lib', '$op', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
    done
  done
done
