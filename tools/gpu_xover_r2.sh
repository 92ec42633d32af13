# crossover re-sweep after K1t / K1w and the TMEM-A K5a (n in (1024, 4096]), E = 2^28 and 2^26
mkdir -p gpurun_out; out=gpurun_out/xover_r2b.txt; : > $out
for s in 28 26; do
for n in 2048 4096; do
  for p in fused wy; do timeout 300 python tools/crossover_sweep.py $n $p 10,12,13,14,15,16,17,18,20 $s >> $out 2>&1; done
  for p in fused-sym wy-sym; do timeout 300 python tools/crossover_sweep.py $n $p 5,6,7,8,9,10,11,12 $s >> $out 2>&1; done
done
done
