#!/bin/bash
# Bench every BASELINE.json workload once (device-timed, no e2e), one JSON line each.
# usage (GPU box, repo root): bash tools/gpu_sweep.sh tag [extra bench args]
tag=${1:-sweep}; shift
mkdir -p gpurun_out
out=gpurun_out/${tag}_sweep.jsonl; : > $out
for w in C1 C2 C3 C4 C5h12 C5h64 C5h256 C5h1024 KNN QR4095 CONG SHF; do
  steps=50; [ $w = C5h1024 ] && steps=20; [ $w = QR4095 ] && steps=5
  timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-e2e --cpu-seconds 3 "$@" >> $out 2>> gpurun_out/${tag}_sweep.err
  echo "$w rc=$?" >> gpurun_out/${tag}_sweep.err
done
# context: unaligned column strides (K1r; the padded detour onto K5 / K1w)
for w in U1023H10 U1023H40 U4095H16; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --cpu-seconds 3 "$@" >> $out 2>> gpurun_out/${tag}_sweep.err
  echo "$w rc=$?" >> gpurun_out/${tag}_sweep.err
done
timeout 300 python bench.py --workload C2 --op T --steps 50 --warmup 3 --no-e2e --no-cpu-baseline "$@" >> $out 2>> gpurun_out/${tag}_sweep.err
