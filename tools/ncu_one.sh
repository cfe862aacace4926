#!/bin/bash
# One ncu --set full capture of one kernel of a 4K step. usage: ncu_one.sh TAG REGEX [ENV=VAL ...]
TAG=$1; K=$2; shift 2
mkdir -p gpurun_out
env "$@" timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
    -k regex:$K -s 2 -c 1 -o gpurun_out/${TAG} -f python tools/profile_step.py --steps 4 \
    > gpurun_out/ncu_${TAG}.log 2>&1
echo "$TAG rc=$?"
