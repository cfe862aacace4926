"""Randomised parity soak on the GPU box: p3s_convert (banded on pinned images, and the
plain path) and the certified bilateral stage against the CPU oracle over many random sizes
and configs, including every certified radius (sigma_s in (3, 12]). Not a unit test (it runs
for minutes); prints one line per failure and a summary.
usage: python tools/soak.py [seconds] [seed] [size scale, default 1]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2009_09501_b200 as p3s  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
chk = oracle.load("best")
ncpu = os.cpu_count() or 1
p3s.set_device(0)
t_end = time.time() + budget
runs = fails = 0
while time.time() < t_end:
    kind = rng.integers(0, 3)
    if kind == 0:  # whole conversion, sizes that take the banded path when tall enough
        w, h = int(rng.integers(16, int(1400 * scale))), int(rng.integers(8, int(900 * scale)))
        over = dict(base=int(rng.choice([-1, 0, 2, 16, 30, 60, 120])),
                    sigma_spatial=float(rng.uniform(0.5, 12.0)),
                    sigma_range=float(rng.choice([4.0, 16.0, 40.0])),
                    depth_block=int(rng.choice([4, 8, 16, 16, 16, 23, 64])),
                    mode=int(rng.integers(0, 2)), formats=int(rng.choice([1, 1, 3, 5, 7])))
        if over["formats"] & 2 and w % 2:
            over["formats"] &= ~2
        img = chk.synthetic_frame(w, h, int(rng.integers(1, 1 << 30)))
        ref = chk.convert(img, oracle.Cfg(**over), threads=ncpu)
        pimg = p3s.Image(img) if rng.integers(0, 2) else img  # pinned (banded) or plain
        out = p3s.convert(pimg, p3s.Config(**over))
        bad = [k for k in ("depth", "filtered", "anaglyph", "hsbs", "fsbs") if k in ref and not np.array_equal(out[k], ref[k])]
    else:  # the bilateral stage on random depth/guide maps with near-tie structure
        w, h = int(rng.integers(8, 700)), int(rng.integers(8, 500))
        s = float(rng.uniform(3.05, 12.0))
        cfg_kw = dict(sigma_spatial=s, sigma_range=float(rng.uniform(2.0, 60.0)))
        levels = rng.integers(0, 256, size=int(rng.integers(2, 5)))
        depth = levels[rng.integers(0, len(levels), size=(h, w))].astype(np.uint8)
        guide = (rng.integers(0, 3, size=(h, w)) * int(rng.integers(1, 60)) + 40).astype(np.uint8)
        ref = chk.cross_bilateral(depth, guide, oracle.Cfg(**cfg_kw), threads=ncpu)
        got = p3s.cross_bilateral(depth, guide, p3s.Config(**cfg_kw))
        bad = [] if np.array_equal(got, ref) else ["filtered"]
        over = dict(size=(w, h), **cfg_kw)
    runs += 1
    if bad:
        fails += 1
        print(f"FAIL {bad} {over}", flush=True)
print(f"soak: {runs} cases, {fails} failures", flush=True)
