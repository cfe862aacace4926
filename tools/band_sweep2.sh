#!/bin/bash
# e2e (p3s_convert, pinned 4K) per band layout (P3S_BAND_ENDS: tile-row ends, 128 rows each).
for E in ${ENDS:-"" "1,4,8,11,13,15,16" "1,4,7,10,12,14,15,16" "1,4,8,11,13,14,15,16" "1,3,6,9,11,13,15,16" "1,4,7,10,13,15,16" "1,4,8,11,13,15,16"}; do
  if [ -z "$E" ]; then unset P3S_BAND_ENDS; else export P3S_BAND_ENDS=$E; fi
  echo "ends=${E:-default} $(timeout 120 python tools/e2e_probe.py 60 2>&1 | tail -1)"
done
