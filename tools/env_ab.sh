#!/bin/bash
# Device-resident bench value under different environment / argument settings.
# usage: bash tools/env_ab.sh "ENV=a|--arg x" ...   (the part after | is passed to bench.py)
for E in "$@"; do
  ENVS=${E%%|*}; ARGS=""; [[ "$E" == *"|"* ]] && ARGS=${E#*|}
  env $ENVS timeout 300 python bench.py --steps 200 --warmup 5 --no-sweep --no-cpu-baseline --no-extra $ARGS > /tmp/ab.json 2>/dev/null
  python3 -c "import json,sys; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); print(sys.argv[1], 'value %.1f single %.1f e2e %.1f stream %.1f' % (d['value'], d['single_stream']['frames_per_s'], d['e2e']['value'], d['e2e_stream']['value']))" "$E"
done
