#!/bin/bash
# One `ncu --set full` capture of each kernel of the unaligned-stride paths (K1r, K1g), each
# after its own command exited 0 without ncu.
# usage (GPU box, repo root): bash tools/gpu_cap_unaligned.sh tag
tag=${1:-r2w}
mkdir -p gpurun_out
cap() {   # name workload kernel-regex skip
  python bench.py --workload $2 --steps 2 --warmup 3 --ncu > gpurun_out/${tag}_$1_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 \
    -o gpurun_out/${tag}_$1 -f python bench.py --workload $2 --steps 2 --warmup 3 --ncu > gpurun_out/${tag}_$1_ncu.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/${tag}_cap_rc.txt
  ncu -i gpurun_out/${tag}_$1.ncu-rep --page details > gpurun_out/${tag}_$1_details.txt 2>&1
}
cap K1r U1023H10 hh_fused_kernel 3
cap K1g U9001H3 hh_general_kernel 3
