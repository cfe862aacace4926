"""Concurrent p3s_convert callers (pinned 4K frames): frames/s for N long-lived host threads
(plans are cached per thread, so each thread warms its own plan first).
usage: python tools/conc_probe.py [threads] [calls_per_thread]"""
import ctypes as C
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09501_b200 as p3s  # noqa: E402

nthr = int(sys.argv[1]) if len(sys.argv) > 1 else 4
per = int(sys.argv[2]) if len(sys.argv) > 2 else 20
W, H = 3840, 2160
L = p3s.lib()
cfg = p3s.Config()
imgs = [p3s.Image(p3s.synthetic_frame(W, H, s)) for s in range(1, 9)]
bar = threading.Barrier(nthr + 1)


def worker(k):
    r, a = C.c_void_p(), C.c_void_p()
    for phase in (4, per):
        bar.wait()
        for j in range(phase):
            p3s._check(L.p3s_convert(imgs[(k + nthr * j) % 8].h, cfg.h, C.byref(r)))
            p3s._check(L.p3s_result_output(r, 1, C.byref(a)))
            L.p3s_result_free(r)
        bar.wait()


ths = [threading.Thread(target=worker, args=(k,)) for k in range(nthr)]
for th in ths:
    th.start()
bar.wait()
bar.wait()  # warm-up done
bar.wait()
t0 = time.perf_counter()
bar.wait()
dt = time.perf_counter() - t0
for th in ths:
    th.join()
print(f"threads={nthr}: {nthr * per / dt:.1f} frames/s", flush=True)
