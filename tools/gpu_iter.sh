#!/bin/bash
# Development iteration on the GPU box: parity subset, launch-time list, optional ncu capture.
# usage: bash tools/gpu_iter.sh TAG "pytest -k expr" [kernel-regex-for-full-capture]
TAG=$1; KEXPR=$2; KREGEX=$3
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -x -q -k "$KEXPR" 2>&1 | tail -15
timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py --steps 3 > /dev/null 2>&1
python - "$TAG" <<'PY'
import csv, sys
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/launches_{tag}.csv")))
hdr = None
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            print(d["ID"], d["Kernel Name"].split("(")[0][-40:], d["Metric Value"], d["Metric Unit"])
PY
if [ -n "$KREGEX" ]; then
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$KREGEX -s 1 -c 1 \
      -o gpurun_out/prof_$TAG -f python tools/profile_step.py --steps 3 > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu rc=$?"
fi
