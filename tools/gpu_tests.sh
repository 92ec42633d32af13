#!/bin/bash
# One gpurun call: smoke, the GPU test suite, the default bench line.
# usage (GPU box, repo root): bash tools/gpu_tests.sh tag [pytest selection args]
tag=${1:-r2}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 "$@" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
