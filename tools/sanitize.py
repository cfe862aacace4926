"""Small-frame end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck):
every route (anaglyph-fused forward, backward, all formats, HSBS, FSBS-direct), odd sizes,
large parallax (multi-round inpaint), the stage API and the video paths. Compared against
the CPU oracle so a sanitizer-clean run is also a correct one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2009_09501_b200 as p3s

p3s.set_device(0)
chk = oracle.load("port")
cases = [(67, 33, dict()), (130, 72, dict(base=40, formats=7)), (96, 64, dict(mode=1, formats=1)),
         (161, 90, dict(base=60, formats=4)), (128, 48, dict(formats=2)), (1, 9, dict(base=4, formats=5)),
         (40, 30, dict(sigma_spatial=3.0, formats=3)),
         # tall enough for the banded synchronous path (engine.cpp plan_bands): fused
         # anaglyph, direct FSBS, materialised eyes, backward
         (200, 300, dict()), (170, 420, dict(formats=4, base=24)), (150, 400, dict(formats=7, base=40)),
         (130, 300, dict(mode=1, formats=1)),
         # fused depth stage (w % 16 == 0) through the banded path; a row wider than shared
         # memory (global z-buffer key slots), forward and backward
         (256, 300, dict(base=30)), (18784, 3, dict(base=40)), (18784, 3, dict(mode=1, formats=5))]
for w, h, over in cases:
    img = chk.synthetic_frame(w, h, w + h)
    ref = chk.convert(img, oracle.Cfg(**over))
    out = p3s.convert(img, p3s.Config(**over))
    for k in ("anaglyph", "hsbs", "fsbs", "depth", "filtered"):
        if k in ref:
            assert np.array_equal(out[k], ref[k]), (w, h, over, k)
# device pipeline with graphs + video (planar, interleaved, sharded)
w, h = 96, 64
cfg = p3s.Config(base=20)
frames = [chk.synthetic_frame(w, h, s) for s in range(1, 4)]
pipe = p3s.Pipeline(w, h, cfg)
buf = p3s.DeviceBuffer(pipe.frame_bytes)
for f in frames:
    pipe.upload(f, buf.addr)
    pipe.run(buf.addr)
    pipe.run(buf.addr, timed=True)
vid = p3s.Video(w, h, cfg, streams=2, devices=[0, 0])
src = [p3s.PinnedBuffer(3 * w * h) for _ in frames]
dst = [p3s.PinnedBuffer(3 * w * h) for _ in frames]
for b, f in zip(src, frames):
    b.array[:] = f.transpose(1, 2, 0).reshape(-1)
vid.convert_ptrs([b.ptr for b in src], [b.ptr for b in dst], interleaved=True)
print("sanitize workload ok")
