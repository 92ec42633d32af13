#!/bin/bash
# One ncu --set full capture of the dominant kernel(s) of each workload class, each only
# after the same command line exited 0 without ncu.  usage: bash tools/gpu_profiles.sh tag
tag=${1:-prof}
mkdir -p gpurun_out
cap() {  # name workload kernel-regex skip count
  python bench.py --workload $2 --steps 1 --warmup 3 --ncu > gpurun_out/${tag}_$1.plain 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c $5 -o gpurun_out/${tag}_$1 -f \
      python bench.py --workload $2 --steps 1 --warmup 3 --ncu > gpurun_out/${tag}_$1.ncu.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/${tag}_profiles.txt
}
: > gpurun_out/${tag}_profiles.txt
cap C5h12 C5h12 hh_fused 3 1
cap C3 C3 "wy_(project|update)" 2 2
cap C4 C4 "hh_gather_bucket|hh_fused" 2 2
cap C5h1024 C5h1024 "wy_(project|update)" 8 2
cap KNN KNN knn_topk 3 1
