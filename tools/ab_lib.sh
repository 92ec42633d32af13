#!/bin/bash
# Same-box A/B of two builds of libhh.so on a list of workloads (full JSON lines).
# usage (GPU box): bash tools/ab_lib.sh tag old.so "C2 C5h12" [env assignments for the new lib]
tag=$1; old=$2; wls=$3; shift 3
mkdir -p gpurun_out; out=gpurun_out/${tag}_ablib.jsonl; : > $out
for rep in 1 2; do
for w in $wls; do
  HH_LIB_PATH=$old timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/${tag}_ablib.err | sed "s/^/old $w /" >> $out
  env "$@" timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/${tag}_ablib.err | sed "s/^/new $w /" >> $out
done
done
