timeout 200 python tools/flow_check.py quick > gpurun_out/flow2_check.txt 2>&1
timeout 300 python tools/flow_tune.py timeline C3 C5h64 C5h12 C5h256 "C5h64:P=100" "C5h64:nkc=2" "C5h64:pol=0" > gpurun_out/flow2_tl.txt 2>&1
timeout 300 python tools/flow_tune.py sweep C5h64 "P=74,100" "nkc=2,4,8" "rseg=2,8" >> gpurun_out/flow2_sweep.txt 2>&1
timeout 300 python tools/flow_tune.py sweep C5h1024 "G=2,4,8" >> gpurun_out/flow2_sweep.txt 2>&1
