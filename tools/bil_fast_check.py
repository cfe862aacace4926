"""Times exact vs certified-FP32 bilateral at 4K and checks both against the oracle, and
reports how many pixels needed the exact fallback."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2009_09501_b200 as p3s  # noqa: E402

p3s.set_device(0)
chk = oracle.load("best")
for (W, H, seed, base) in [(3840, 2160, 1, -1), (1920, 1080, 2, -1), (7680, 4320, 3, -1)]:
    img = chk.synthetic_frame(W, H, seed)
    ref = chk.convert(img, oracle.Cfg(), threads=os.cpu_count())["filtered"] if W < 7680 else None
    cfg = p3s.Config(base=base)
    pipe = p3s.Pipeline(W, H, cfg)
    d = p3s.DeviceBuffer(pipe.frame_bytes)
    pipe.upload(img, d.addr)
    for mode in sys.argv[1:] or ["0", "1", "2"]:
        os.environ["P3S_BIL_FAST"] = mode
        for _ in range(3):
            pipe.run(d.addr, timed=True)
        p3s.stream_sync(pipe.stream)
        pipe.timing_sum(reset=True)
        for _ in range(10):
            pipe.run(d.addr, timed=True)
        st, n = pipe.timing_sum(reset=True)
        _, filt, _ = pipe.download()
        ok = "n/a" if ref is None else bool(np.array_equal(filt, ref))
        print(f"{W}x{H} fast={mode}: bilateral {st['filter_ns'] / n / 1e6:.3f} ms exact={ok}",
              flush=True)
        if W >= 7680 and mode == "0":
            ref8 = filt.copy()
        if W >= 7680 and mode != "0":
            print("   8K fast == exact:", bool(np.array_equal(filt, ref8)))
