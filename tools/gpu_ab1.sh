timeout 300 python tools/k1_ab.py C2 > gpurun_out/ab1_k1.txt 2>&1
timeout 300 python tools/k1_ab.py C5h12 3 >> gpurun_out/ab1_k1.txt 2>&1
timeout 400 python tools/flow_tune.py sweep C5h64 "nkc=1,2,4" "D=40,80" > gpurun_out/ab1_flow.txt 2>&1
timeout 400 python tools/flow_tune.py sweep C3 "nkc=1,2,4" "D=40,80" >> gpurun_out/ab1_flow.txt 2>&1
timeout 400 python tools/flow_tune.py sweep C5h12 "nkc=1,2,4" "D=40,80" >> gpurun_out/ab1_flow.txt 2>&1
