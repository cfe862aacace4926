"""Aggregate an ncu --set full capture's warp-stall samples by CUDA source line (cuda,sass
view). usage: python tools/ncu_lines.py REP.ncu-rep [top]"""
import csv, io, os, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
agg = defaultdict(lambda: defaultdict(float))
src = {}
cur_line = None
cur_file = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur_line = f"{cur_file}:{r[0]}"
        src[cur_line] = r[1].strip()
    d = dict(zip(hdr[2:], r[2:]))
    for k in ("Warp Stall Sampling (All Samples)", "Instructions Executed", "stall_long_sb",
              "stall_barrier", "stall_short_sb", "stall_lg", "stall_membar", "stall_branch_resolving",
              "stall_wait", "stall_mio", "stall_no_inst", "stall_math", "stall_dispatch", "stall_lg_throttle", "stall_drain"):
        try:
            agg[cur_line][k] += float(d.get(k, "0") or 0)
        except ValueError:
            pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
print(f"total samples {tot:.0f}")
items = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])
for ln, v in items[:top]:
    s = v["Warp Stall Sampling (All Samples)"]
    if not s:
        break
    det = " ".join(f"{k.replace('stall_', '')}={v[k]:.0f}" for k in
                   ("stall_long_sb", "stall_barrier", "stall_short_sb", "stall_lg", "stall_membar",
                    "stall_branch_resolving", "stall_wait", "stall_mio", "stall_no_inst", "stall_math",
                    "stall_dispatch", "stall_lg_throttle", "stall_drain") if v[k] > 0.05 * s)
    print(f"{100 * s / tot:5.1f}% {ln} inst={v['Instructions Executed']:.0f} [{det}] {src.get(ln, '')[:90]}")
