out=gpurun_out/ab9.txt; : > $out
for rep in 1 2; do
  for lib in abtest/libhh_k1sf.so abtest/libhh_k1sfu.so; do
    HH_LIB_PATH=$lib timeout 200 python tools/k1s_grid.py >> $out 2>>gpurun_out/ab9.err
    HH_LIB_PATH=$lib timeout 200 python bench.py --workload C4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/ab9.err | python -c "import sys,json; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$lib C4', round(d['ms_per_step'],4))" >> $out
  done
done
