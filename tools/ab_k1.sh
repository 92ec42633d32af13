#!/bin/bash
# A/B of the fused kernel's sequential vs blocked (compact-WY blocks) mode and of the
# n=4096 variants.  usage (GPU box): bash tools/ab_k1.sh tag
tag=${1:-ab}
mkdir -p gpurun_out
out=gpurun_out/${tag}_ab.txt; : > $out
HH_K1_BLOCKED=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_signed_gpu.py -q -x -p no:cacheprovider > gpurun_out/${tag}_pytest_blk.log 2>&1
echo "pytest blocked rc=$?" >> $out
run() {  # label env... -- bench args
  local label=$1; shift
  local envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  r=$(env "${envs[@]}" timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-parity "$@" 2>>gpurun_out/${tag}_ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline'].get('kernel'))")
  echo "$label $* : $r" >> $out
}
for w in C2 C4 C5h12; do
  run seq HH_K1_BLOCKED=0 -- --workload $w
  run blk HH_K1_BLOCKED=1 -- --workload $w
done
run seq HH_K1_BLOCKED=0 -- --workload C2 --op T
run blk HH_K1_BLOCKED=1 -- --workload C2 --op T
for v in f32_tpc128_ch8_c2_nt512 f32_tpc256_ch4_c4; do
  run seq HH_K1_BLOCKED=0 HH_K1_VARIANT=$v -- --workload C5h12
  run blk HH_K1_BLOCKED=1 HH_K1_VARIANT=$v -- --workload C5h12
done
