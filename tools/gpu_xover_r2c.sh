mkdir -p gpurun_out; out=gpurun_out/xover_r2c.txt; : > $out
for s in 28 26; do
  for p in fused wy; do timeout 300 python tools/crossover_sweep.py 1024 $p 12,14,16,17,18,19,20 $s >> $out 2>&1; done
  for p in fused-sym wy-sym; do timeout 300 python tools/crossover_sweep.py 1024 $p 8,10,11,12,13,14,16 $s >> $out 2>&1; done
done
