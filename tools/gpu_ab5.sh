timeout 900 python -m pytest tests/test_wy_gpu.py tests/test_graph_gpu.py tests/test_qr_gpu.py tests/test_signed_gpu.py tests/test_congruence_gpu.py tests/test_fullsize_gpu.py -q -p no:cacheprovider -x > gpurun_out/ab5_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab5_pytest.log
timeout 600 python tools/prep_ab.py > gpurun_out/ab5_prep.txt 2>&1
