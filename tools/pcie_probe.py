import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np, oracle, paper_2009_09501_b200 as p3s
p3s.set_device(0)
W, H = 3840, 2160
pipe = p3s.Pipeline(W, H, p3s.Config())
img = oracle.load("port").synthetic_frame(W, H, 1)
pb = p3s.PinnedBuffer(3 * W * H); pb.array[:] = img.reshape(-1)
d = p3s.DeviceBuffer(pipe.frame_bytes)
import ctypes as C
L = p3s.lib()
for rep in range(3):
    t0 = time.perf_counter()
    for i in range(20):
        L.p3s_pipeline_upload(pipe.handle, C.c_void_p(pb.ptr), C.c_void_p(pb.ptr + W*H), C.c_void_p(pb.ptr + 2*W*H), C.c_void_p(d.addr), None)
    p3s.stream_sync(pipe.stream)
    dt = (time.perf_counter() - t0) / 20
    print("H2D 24.9MB: %.3f ms  %.1f GB/s" % (dt * 1e3, 3*W*H/dt/1e9))
pipe.run(d.addr); p3s.stream_sync(pipe.stream)
o = p3s.PinnedBuffer(3 * W * H)
for rep in range(3):
    t0 = time.perf_counter()
    for i in range(20):
        outs = (C.c_void_p * 3)(o.ptr, o.ptr + W*H, o.ptr + 2*W*H)
        u8 = C.POINTER(C.c_uint8); L.p3s_pipeline_download(pipe.handle, None, None, 1, C.cast(o.ptr, u8), C.cast(o.ptr + W*H, u8), C.cast(o.ptr + 2*W*H, u8))
    dt = (time.perf_counter() - t0) / 20
    print("D2H 24.9MB (sync each): %.3f ms  %.1f GB/s" % (dt * 1e3, 3*W*H/dt/1e9))
res = C.c_void_p()
imgh = p3s.Image(img)
cfg = p3s.Config()
for rep in range(3):
    t0 = time.perf_counter()
    for i in range(20):
        p3s._check(L.p3s_convert(imgh.h, cfg.h, C.byref(res))); L.p3s_result_free(res)
    dt = (time.perf_counter() - t0) / 20
    print("p3s_convert: %.3f ms" % (dt * 1e3))
