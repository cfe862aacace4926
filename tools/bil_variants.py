"""Times the bilateral kernel variants (P3S_BIL_VARIANT) on a 4K frame and checks each
variant's filtered depth against the CPU oracle (tuning experiment driver)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2009_09501_b200 as p3s  # noqa: E402

W, H = 3840, 2160
p3s.set_device(0)
chk = oracle.load("best")
img = chk.synthetic_frame(W, H, 1)
ref = chk.convert(img, oracle.Cfg(), threads=os.cpu_count())["filtered"]
cfg = p3s.Config()
pipe = p3s.Pipeline(W, H, cfg)
d = p3s.DeviceBuffer(pipe.frame_bytes)
pipe.upload(img, d.addr)
for var in sys.argv[1:] or ["0", "1", "2", "3", "4", "5", "6"]:
    os.environ["P3S_BIL_VARIANT"] = var
    for _ in range(3):
        pipe.run(d.addr, timed=True)
    p3s.stream_sync(pipe.stream)
    pipe.timing_sum(reset=True)
    for _ in range(10):
        pipe.run(d.addr, timed=True)
    st, n = pipe.timing_sum(reset=True)
    _, filt, _ = pipe.download()
    ok = np.array_equal(filt, ref)
    print(f"variant {var}: bilateral {st['filter_ns'] / n / 1e6:.3f} ms  exact={ok}", flush=True)
