timeout 300 python tools/k1s_ab.py > gpurun_out/ab2_k1s.txt 2>&1
timeout 400 python tools/pdl_ab.py > gpurun_out/ab2_pdl.txt 2>&1
