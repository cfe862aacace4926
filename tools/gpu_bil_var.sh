#!/bin/bash
# A/B of bilateral variants on the GPU box: parity tests, then 4K stage times per variant.
# usage: [EV=P3S_BIL_FOLD] bash tools/gpu_bil_var.sh TAG "0 1"  (env-selected kernel variants, default P3S_BIL_VAR)
TAG=${1:-ab}; VARS=${2:-"1 3"}
mkdir -p gpurun_out
for V in $VARS; do
  echo "var $V parity: $(env "${EV:-P3S_BIL_VAR}=$V" timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k 'golden or random or sweep or 4k' 2>&1 | tail -1)"
  env "${EV:-P3S_BIL_VAR}=$V" timeout 300 python bench.py --steps 60 --warmup 5 --no-sweep --no-cpu-baseline --no-extra \
      > gpurun_out/bench_${TAG}_v$V.json 2> gpurun_out/bench_${TAG}_v$V.err
  python - "$V" "gpurun_out/bench_${TAG}_v$V.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print("var", sys.argv[1], "fps %.1f" % d["value"], {k: round(v, 4) for k, v in d["stages_ms"].items()},
          "roof %.3f" % d["roofline"]["frac"], "kernel_ms %.4f" % d["roofline"]["kernel_ms"])
except Exception as e:
    print("var", sys.argv[1], "failed", e)
PY
done
