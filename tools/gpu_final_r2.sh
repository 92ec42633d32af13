#!/bin/bash
# End-of-round-2 evidence in one gpurun call: smoke, the GPU test suite, the default bench
# line, the per-workload sweep, ncu DRAM traffic of the workloads whose kernels changed late in
# the round, and one `ncu --set full` capture of each new shipping kernel.
# usage (GPU box, repo root): bash tools/gpu_final_r2.sh tag
tag=${1:-r2z}
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
timeout 1200 python tools/traffic.py run C2 C3 C4 C5h12 SHF > gpurun_out/${tag}_tr_run.log 2>&1
cap() {   # tag workload kernel-regex skip
  python bench.py --workload $2 --steps 2 --warmup 3 --ncu > gpurun_out/${tag}_$1_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 \
    -o gpurun_out/${tag}_$1 -f python bench.py --workload $2 --steps 2 --warmup 3 --ncu > gpurun_out/${tag}_$1_ncu.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/${tag}_rc.txt
}
cap C5h12 C5h12 hh_fused_kernel 3
cap SHFg SHF shf_gemm_f32_kernel 6
cap C3s C3 wy_sym_rows_kernel 3
python bench.py --steps 5 --warmup 3 --ncu > gpurun_out/${tag}_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_C2_launches.csv python bench.py --steps 5 --warmup 3 --ncu > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "launches rc=$?" >> gpurun_out/${tag}_rc.txt
