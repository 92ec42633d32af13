#!/bin/bash
# Round-end style GPU evidence in one gpurun call: smoke, the full GPU test suite, the
# default bench line, the per-workload sweep, the ncu launch list of the default bench
# command and one full ncu capture of its dominant kernel.
# usage (GPU box, repo root): bash tools/gpu_round.sh tag
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${tag}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2>> gpurun_out/${tag}_bench.err
bash tools/gpu_sweep.sh ${tag}
python bench.py --steps 5 --warmup 3 --ncu > gpurun_out/${tag}_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 5 --warmup 3 --ncu > gpurun_out/${tag}_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hh_fused -s 3 -c 1 \
  -o gpurun_out/${tag}_full -f python bench.py --steps 5 --warmup 3 --ncu > gpurun_out/${tag}_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}_ncu_full.log
