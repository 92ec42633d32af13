mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_wy_gpu.py tests/test_fullsize_gpu.py -k "wy or C3 or C5" -m gpu -q -x -p no:cacheprovider > gpurun_out/tsa2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tsa2_pytest.log
timeout 900 python tools/wy_tsa_ab.py > gpurun_out/tsa2_ab.txt 2>&1
python bench.py --workload C5h64 --steps 2 --warmup 3 --ncu > gpurun_out/tsa2_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wy_project_kernel -s 1 -c 1 \
  -o gpurun_out/tsa2_C5h64a -f python bench.py --workload C5h64 --steps 2 --warmup 3 --ncu > gpurun_out/tsa2_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/tsa2_ncu.log
