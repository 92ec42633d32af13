#!/bin/bash
# ncu evidence for the shipping K1t kernel (C5 h=12): per-workload DRAM traffic and one
# --set full capture.  usage (GPU box, repo root): bash tools/gpu_prof_k1t.sh tag
tag=${1:-k1t}
mkdir -p gpurun_out
timeout 600 python tools/traffic.py run C5h12 > gpurun_out/${tag}_tr.log 2>&1
python bench.py --workload C5h12 --steps 2 --warmup 3 --ncu > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hh_fused_kernel -s 3 -c 1 \
  -o gpurun_out/${tag}_C5h12 -f python bench.py --workload C5h12 --steps 2 --warmup 3 --ncu > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}_ncu.log
