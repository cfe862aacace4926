#!/bin/bash
# usage: bash tools/ncu_bil.sh TAG VARIANT
TAG=$1; VAR=$2
P3S_BIL_VARIANT=$VAR timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
   -k regex:k_bilateral -s 1 -c 1 -o gpurun_out/prof_$TAG -f python tools/profile_step.py --steps 2 > gpurun_out/ncu_$TAG.log 2>&1
echo rc=$?
