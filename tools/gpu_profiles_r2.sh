#!/bin/bash
# Round-2 evidence in one gpurun call: per-workload ncu DRAM traffic (tools/traffic.py) and one
# `ncu --set full` capture of each shipping hot kernel.  usage (GPU box): bash tools/gpu_profiles_r2.sh
mkdir -p gpurun_out
timeout 1500 python tools/traffic.py run C1 C2 C3 C4 C5h12 C5h64 C5h256 C5h1024 KNN > gpurun_out/tr_run.log 2>&1
cap() {   # tag workload kernel-regex skip
  python bench.py --workload $2 --steps 2 --warmup 3 --ncu > gpurun_out/p2_$1_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 \
    -o gpurun_out/p2_$1 -f python bench.py --workload $2 --steps 2 --warmup 3 --ncu > gpurun_out/p2_$1_ncu.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/p2_rc.txt
}
cap C2 C2 hh_fused_kernel 3
cap C5h12 C5h12 hh_fused_kernel 3
cap C5h64a C5h64 wy_project_kernel 3
cap C5h64b C5h64 wy_update_kernel 3
cap C3b C3 wy_update_kernel 3
cap C5h256ts C5h256 wy_update_ts_kernel 3
cap C4g C4 hh_gather_bucket_kernel 3
cap C4t C4 hh_fused_kernel 3
