#!/bin/bash
# ncu launch durations (ns) of the depth-stage kernels of a 4K step (cold, serialised)
P3S_NO_GRAPHS=1 timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv \
    python tools/profile_step.py --steps 2 2>/dev/null | grep -E "depth_front|block_values|upsample" | head -3 | \
    python3 -c 'import sys,csv; [print(r[4].split("(")[0], r[-1]) for r in csv.reader(sys.stdin)]'
