"""Minimal driver for ncu: runs the device-resident pipeline for a few steps on
synthetic frames (no e2e / sweep / CPU legs), so a profiler sees only the kernels."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09501_b200 as p3s  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--w", type=int, default=3840)
ap.add_argument("--h", type=int, default=2160)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--base", type=int, default=-1)
ap.add_argument("--formats", type=int, default=1)
ap.add_argument("--frames", type=int, default=2)
a = ap.parse_args()
p3s.set_device(0)
cfg = p3s.Config(base=a.base, formats=a.formats)
pipe = p3s.Pipeline(a.w, a.h, cfg)
bufs = []
for i in range(a.frames):
    d = p3s.DeviceBuffer(pipe.frame_bytes)
    pipe.upload(p3s.synthetic_frame(a.w, a.h, 1 + i), d.addr)
    bufs.append(d)
for i in range(a.steps):
    pipe.run(bufs[i % len(bufs)].addr)
p3s.stream_sync(pipe.stream)
print("done", a.steps, "steps")
if os.environ.get("P3S_REPORT_FIXUP"):
    import ctypes as C
    # count of uncertified pixels of the last bilateral (read through the stage API)
    img = p3s.synthetic_frame(a.w, a.h, 1)
    import numpy as np
    luma = p3s.luma(img)
    depth = p3s.generate_depth(img, cfg)
    raw = p3s.cross_bilateral_raw(depth, luma, cfg)
    f = raw + 0.5
    dist = np.minimum(f - np.floor(f), np.floor(f) + 1 - f)
    bound = raw * 44.0 / 2**24 + 1e-9
    print("uncertified pixels (predicted from raw):", int((dist <= bound).sum()), "of", raw.size)
