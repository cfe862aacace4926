#!/bin/bash
# Full GPU parity + one bench line (no CPU baseline, no sweep). usage: gpu_quick.sh TAG
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 100 --warmup 5 --no-sweep --no-cpu-baseline --no-extra > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
python - gpurun_out/bench_$TAG.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("fps %.1f" % d["value"], {k: round(v, 4) for k, v in d["stages_ms"].items()})
print("e2e %.1f stream %.1f" % (d["e2e"]["value"], d["e2e_stream"]["value"]), "roof %.3f" % d["roofline"]["frac"],
      [("%s %.3f" % (r["kernel"].split(" ")[0], r["frac"])) for r in d["roofline_hbm"]])
PY
