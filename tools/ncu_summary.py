"""Summarise the per-kernel ncu --set full captures of tools/gpu_profile.sh TAG into a
markdown table (stdout) and profiles/traffic.json (DRAM bytes per launch).
usage: python tools/ncu_summary.py TAG"""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = "/usr/local/cuda/bin/ncu"
KERNELS = ["k_depth_fused", "k_upsample_rows", "k_bilateral_sep", "k_bilateral_fixup", "k_dibr_quad",
           "k_inpaint"]
WANT = {"Duration": "us", "DRAM Throughput": "%", "Compute (SM) Throughput": "%",
        "Issue Slots Busy": "%", "L1/TEX Cache Throughput": "%", "Achieved Occupancy": "%",
        "Registers Per Thread": ""}


def raw_metrics(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {}
    for k, u, v in zip(hdr, units, vals):
        try:
            out[k] = float(v.replace(",", "")) * scale.get(u, 1)
        except ValueError:
            out[k] = v
    return out


def details(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    d, name = {}, ""
    for r in csv.reader(io.StringIO(out)):
        if len(r) < 15 or r[0] == "ID":
            continue
        name = r[4]
        key, val = r[12], r[14]
        if key in WANT and key not in d:
            d[key] = val + (" " + r[13] if key == "Duration" else "")
    return name, d


def main():
    tag = sys.argv[1]
    traffic = {"_doc": "ncu --set full, 4K default config, one launch each: dram__bytes_read.sum + "
                       "dram__bytes_write.sum, bytes per launch (capture tag %s). Writes still resident "
                       "in the 126 MB L2 when the kernel ends are not counted by dram__bytes_write; the "
                       "algorithmic bytes are in DESIGN.md." % tag}
    print("| Kernel | " + " | ".join(WANT) + " | DRAM R+W |")
    print("|---" * (len(WANT) + 2) + "|")
    for k in KERNELS:
        rep = os.path.join(ROOT, "gpurun_out", f"{k}_{tag}.ncu-rep")
        if not os.path.exists(rep):
            continue
        name, d = details(rep)
        m = raw_metrics(rep)
        try:
            rw = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        except (KeyError, TypeError):
            rw = float("nan")
        short = name.split("(")[0].replace("void ", "").replace("unnamed>::", "") or k
        key = "k_dibr" if k == "k_dibr_quad" else ("k_inpaint_tiles" if k == "k_inpaint" else
                                                   ("k_bilateral_fixup2" if k == "k_bilateral_fixup" else k))
        traffic[key] = rw
        print(f"| {short} | " + " | ".join(d.get(x, "") for x in WANT) + f" | {rw / 1e6:.2f} MB |")
    stage = ["k_depth_fused", "k_upsample_rows"]
    if all(k in traffic for k in stage):  # the depth stage as bench.py's roofline_hbm names it
        traffic["+".join(stage)] = sum(traffic[k] for k in stage)
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main()
