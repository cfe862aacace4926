#!/bin/bash
# ncu launch durations (ns) of the DIBR kernel of a 4K step (cold, serialised)
P3S_NO_GRAPHS=1 timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_dibr -c 3 --csv \
    python tools/profile_step.py --steps 2 2>/dev/null | grep k_dibr | \
    python3 -c 'import sys,csv; [print(r[4].split("(")[0], r[-1]) for r in csv.reader(sys.stdin)]'
