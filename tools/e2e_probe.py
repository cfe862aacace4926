"""p3s_convert e2e probe: frames/s of synchronous calls on pinned 4K frames (the bench's e2e
leg), optionally for an experiment library (P3S_LIB_PATH); P3S_PROBE_SIZE=WxH picks another size.
usage: python tools/e2e_probe.py [n]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09501_b200 as p3s  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
W, H = (int(v) for v in os.environ.get("P3S_PROBE_SIZE", "3840x2160").split("x"))
L = p3s.lib()
cfg = p3s.Config()
imgs = [p3s.Image(p3s.synthetic_frame(W, H, s)) for s in range(1, 9)]
res, ana = C.c_void_p(), C.c_void_p()
for rep in range(3):
    for i in range(4):
        p3s._check(L.p3s_convert(imgs[i].h, cfg.h, C.byref(res)))
        L.p3s_result_free(res)
    t0 = time.perf_counter()
    for i in range(n):
        p3s._check(L.p3s_convert(imgs[i % 8].h, cfg.h, C.byref(res)))
        p3s._check(L.p3s_result_output(res, 1, C.byref(ana)))
        L.p3s_result_free(res)
    dt = time.perf_counter() - t0
    print(f"{os.path.basename(p3s.LIB_PATH)}: {n / dt:.1f} frames/s ({1e3 * dt / n:.3f} ms/call)", flush=True)
