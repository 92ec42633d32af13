bash tools/gpu_ab8.sh
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2g_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2g_pytest.log
bash tools/gpu_sweep.sh r2g
