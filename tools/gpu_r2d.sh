timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2d_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2d_pytest.log
for n in 128 256 512; do
  for s in 28 25; do
    timeout 200 python tools/crossover_sweep.py $n fused 12,16,20,24,28,32,40 $s >> gpurun_out/r2d_cross.txt 2>&1
    timeout 200 python tools/crossover_sweep.py $n wy 16,32 $s >> gpurun_out/r2d_cross.txt 2>&1
  done
  timeout 200 python tools/crossover_sweep.py $n fused-sym 6,8,10,12,14,16,20 28 >> gpurun_out/r2d_cross.txt 2>&1
  timeout 200 python tools/crossover_sweep.py $n wy-sym 8,16 28 >> gpurun_out/r2d_cross.txt 2>&1
done
