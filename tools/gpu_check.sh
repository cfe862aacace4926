#!/bin/bash
# GPU-box check used during development: smoke, GPU parity tests, short bench.
# usage: bash tools/gpu_check.sh [tag]
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
echo "nproc=$(nproc)"
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout 600 python bench.py --steps 100 --warmup 5 --no-sweep --cpu-budget 10 \
    > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -5 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
