#!/bin/bash
# One gpurun call: build check, GPU parity tests, bench, ncu launch list + one full capture.
# usage (from the repo root, on the GPU box): bash tools/gpu_check.sh [tag]
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 5 --warmup 3 \
  --no-cpu-baseline --no-e2e --no-parity > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "ncu-launch rc=$?" >> gpurun_out/${tag}_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hh_fused \
  --launch-skip 3 -c 1 -o gpurun_out/${tag}_full -f python bench.py --steps 5 --warmup 3 \
  --no-cpu-baseline --no-e2e --no-parity > gpurun_out/${tag}_ncu_full.log 2>&1
echo "ncu-full rc=$?" >> gpurun_out/${tag}_ncu_full.log
