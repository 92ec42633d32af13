#!/bin/bash
# Same-box A/B of several libhh.so builds.  usage: bash tools/ab_libs.sh tag "C3 C5h64" a.so b.so ...
tag=$1; wls=$2; shift 2
mkdir -p gpurun_out; out=gpurun_out/${tag}_ablibs.jsonl; : > $out
for rep in 1 2; do
  for w in $wls; do
    for lib in "$@"; do
      HH_LIB_PATH=$lib timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/${tag}_ablibs.err | sed "s|^|$(basename $lib) $w |" >> $out
    done
  done
done
