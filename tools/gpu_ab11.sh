out=gpurun_out/ab12.txt; : > $out
for rep in 1 2 3; do
  for lib in abtest/libhh_k12b.so abtest/libhh_k12c.so; do
    for w in C5h12; do
      HH_LIB_PATH=$lib timeout 200 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/ab11.err | python -c "import sys,json; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$lib', '$w', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
    done
  done
done
