timeout 400 python tools/flow_tune.py sweep C5h64 "P=74,84" "nkc=4,8" "rseg=1,2" "D=20,40,80,512" > gpurun_out/flow3_sweep.txt 2>&1
timeout 200 python tools/flow_tune.py timeline "C5h64:D=80;rseg=2;nkc=4" "C5h64:D=512;rseg=2;nkc=4" >> gpurun_out/flow3_sweep.txt 2>&1
