#!/bin/bash
# Dev loop on the GPU box: targeted tests, full -m gpu, stage launch list, short bench.
# usage: bash tools/gpu_quick2.sh TAG "pytest -k expr"
TAG=${1:-q}; K=${2:-fused}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py --steps 3 > /dev/null 2>&1
python3 - "$TAG" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"gpurun_out/launches_{sys.argv[1]}.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = len(hdr) - 1
t = collections.defaultdict(list)
for r in rows[1:]:
    try: t[r[ki].split("(")[0].split("<")[0]].append(float(r[vi]))
    except ValueError: pass
for k, v in t.items(): print(f"{k:32s} n={len(v):3d} median={sorted(v)[len(v)//2]:10.1f}")
PY
timeout 600 python bench.py --steps 50 --warmup 5 --no-sweep --no-extra --no-cpu-baseline \
    > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python3 -c "
import json; d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])
print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'stages', {k: round(v,4) for k,v in d['stages_ms'].items()})
print([ (r['kernel'], round(r['frac'],3)) for r in d.get('roofline_hbm',[])], d['parity'])
"
