#!/bin/bash
# End-of-round evidence on the final code in one gpurun call: smoke, the GPU suite, the default
# bench line + the reference arm, the per-workload sweep, and the ncu launch list of the
# default bench command.
# usage (GPU box, repo root): bash tools/gpu_final_r2w.sh tag
tag=${1:-r2w}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${tag}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2>> gpurun_out/${tag}_bench.err
bash tools/gpu_sweep.sh ${tag}
python bench.py --steps 5 --warmup 3 --ncu > gpurun_out/${tag}_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_C2_launches.csv python bench.py --steps 5 --warmup 3 --ncu > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "launches rc=$?" >> gpurun_out/${tag}_rc.txt
