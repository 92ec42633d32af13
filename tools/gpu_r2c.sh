timeout 900 python -m pytest tests/test_wy_gpu.py tests/test_graph_gpu.py tests/test_qr_gpu.py tests/test_signed_gpu.py tests/test_congruence_gpu.py -q -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
bash tools/gpu_sweep.sh r2c
