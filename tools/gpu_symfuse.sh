mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_wy_gpu.py tests/test_fullsize_gpu.py tests/test_signed_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/symfuse_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/symfuse_pytest.log
timeout 900 python tools/symfuse_ab.py > gpurun_out/symfuse_ab.txt 2>&1
