mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "k1_tmem or k1t" -p no:cacheprovider > gpurun_out/k1w_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/k1w_pytest.log
timeout 900 python tools/k1t_ab.py "1024:10,1024:10:1,4096:12,4096:8,4096:16,2048:12,2048:16,1024:16,1024:12,2048:8,4096:12:2" > gpurun_out/k1w_ab.txt 2>&1
