"""4K parallax sweep probe: per B, inpaint / DIBR / whole-frame time from event-timed runs on
one plan (same as bench.py's sweep_base leg). usage: python tools/sweep_probe.py [B ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09501_b200 as p3s  # noqa: E402

W, H = 3840, 2160
bases = [int(a) for a in sys.argv[1:]] or [0, 2, 16, 30, 60, 120, 254, 510]
p3s.set_device(0)
pipe0 = p3s.Pipeline(W, H, p3s.Config())
ring = []
for i in range(4):
    d = p3s.DeviceBuffer(pipe0.frame_bytes)
    pipe0.upload(p3s.synthetic_frame(W, H, 1 + i), d.addr)
    ring.append(d)
p3s.device_sync()
for b in bases:
    pb = p3s.Pipeline(W, H, p3s.Config(base=b))
    for i in range(3):
        pb.run(ring[i % 4].addr, timed=True)
    p3s.stream_sync(pb.stream)
    pb.timing_sum(reset=True)
    for i in range(20):
        pb.run(ring[i % 4].addr, timed=True)
    p3s.stream_sync(pb.stream)
    st, n = pb.timing_sum(reset=True)
    tot = sum(v for k, v in st.items() if k != "pure_ns") / n / 1e6
    ps = pb.inpaint_stats()
    print(f"B={b:4d} inpaint {st['inpaint_left_ns'] / n / 1e6 + st['inpaint_right_ns'] / n / 1e6:.4f} ms "
          f"dibr {st['dibr_ns'] / n / 1e6:.4f} filter {st['filter_ns'] / n / 1e6:.4f} "
          f"depth {st['depth_gen_ns'] / n / 1e6:.4f} total {tot:.4f} ms passes {int(ps[0])},{int(ps[3])}",
          flush=True)
    del pb
