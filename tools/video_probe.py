"""Streamed-video throughput vs stream count (4K anaglyph, pinned host frames)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, paper_2009_09501_b200 as p3s
p3s.set_device(0)
W, H = 3840, 2160
o = oracle.load("port")
frames = [o.synthetic_frame(W, H, 1 + i) for i in range(8)]
src = [p3s.PinnedBuffer(3 * W * H) for _ in frames]
dst = [p3s.PinnedBuffer(3 * W * H) for _ in frames]
for b, f in zip(src, frames):
    b.array[:] = f.reshape(-1)
cfg = p3s.Config()
for streams in (1, 2, 4, 6, 8):
    v = p3s.Video(W, H, cfg, streams=streams)
    v.convert_ptrs([b.ptr for b in src[:4]], [b.ptr for b in dst[:4]])
    n = 96
    t0 = time.perf_counter()
    v.convert_ptrs([src[i % 8].ptr for i in range(n)], [dst[i % 8].ptr for i in range(n)])
    dt = time.perf_counter() - t0
    print(f"streams {streams}: {n / dt:.1f} frames/s")
    del v
