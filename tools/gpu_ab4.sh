timeout 500 python tools/k1s_mw_ab.py > gpurun_out/ab4_mw.txt 2>&1
bash tools/ab_libs.sh ab4 "C3 C5h64 C5h256 C5h1024" abtest/libhh_nolag.so abtest/libhh_lag.so
