#!/bin/bash
# Refresh of the round-2 evidence after the K1 / K1s changes: traffic of the workloads they touch
# and a full capture of the C2 kernel that ships now.
mkdir -p gpurun_out
timeout 900 python tools/traffic.py run C2 C4 KNN CONG C5h12 > gpurun_out/tr_run2.log 2>&1
python bench.py --workload C2 --steps 2 --warmup 3 --ncu > gpurun_out/p3_C2_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hh_fused_kernel -s 3 -c 1 \
  -o gpurun_out/p3_C2 -f python bench.py --workload C2 --steps 2 --warmup 3 --ncu > gpurun_out/p3_C2_ncu.log 2>&1
echo "C2 rc=$?" >> gpurun_out/p3_rc.txt
python bench.py --workload C4 --steps 2 --warmup 3 --ncu > gpurun_out/p3_C4_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hh_stream_kernel -s 3 -c 1 \
  -o gpurun_out/p3_C4t -f python bench.py --workload C4 --steps 2 --warmup 3 --ncu > gpurun_out/p3_C4t_ncu.log 2>&1
echo "C4t rc=$?" >> gpurun_out/p3_rc.txt
