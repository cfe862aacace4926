"""Per-round inpaint timeline at 4K (P3S_DEBUG_INPAINT=1): one event-timed frame per B.
usage: P3S_DEBUG_INPAINT=1 python tools/inpaint_probe.py [B ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09501_b200 as p3s  # noqa: E402

W, H = 3840, 2160
bases = [int(a) for a in sys.argv[1:]] or [30, 510]
p3s.set_device(0)
for b in bases:
    pb = p3s.Pipeline(W, H, p3s.Config(base=b))
    d = p3s.DeviceBuffer(pb.frame_bytes)
    pb.upload(p3s.synthetic_frame(W, H, 1), d.addr)
    for i in range(2):
        print(f"--- B={b} run {i}", file=sys.stderr, flush=True)
        pb.run(d.addr, timed=True)
        p3s.stream_sync(pb.stream)
    print(f"B={b}", pb.timings(), flush=True)
