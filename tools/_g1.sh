cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo rc=$?; tail -3 gpurun_out/bench_r2b.err
python - gpurun_out/bench_r2b.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("fps %.1f" % d["value"], "launches", d["gpu_launches"], {k: round(v, 4) for k, v in d["stages_ms"].items()})
print("e2e %.1f stream %.1f" % (d["e2e"]["value"], d["e2e_stream"]["value"]), d["e2e_stream"]["runs"], "roof %.3f" % d["roofline"]["frac"])
print({b: round(v["frames_per_s"],1) for b, v in d["sweep_base"].items()})
print(json.dumps(d["parity"]))
for k, v in d["configs_extra"].items(): print(k, round(v.get("frames_per_s", 0), 1))
print(json.dumps(d.get("cpu_baseline"))[:1500])
PY
