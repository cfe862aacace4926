#!/bin/bash
# ncu launch list + full captures of each kernel of one 4K step.
# usage: bash tools/gpu_profile.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py --steps 4 > /dev/null 2>&1
echo "launch list rc=$?"
for K in ${KERNELS:-k_bilateral_sep k_bilateral_fixup k_dibr_quad k_depth_fused k_upsample_rows k_inpaint}; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o gpurun_out/${K}_$TAG -f python tools/profile_step.py --steps 4 > gpurun_out/ncu_${K}_$TAG.log 2>&1
  echo "$K rc=$?"
done
ls -la gpurun_out
