import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, oracle, paper_2009_09501_b200 as p3s
chk = oracle.load("best")
rng = np.random.default_rng(7)
for i in range(24):
    w, h = int(rng.integers(1, 300)), int(rng.integers(1, 200))
    over = dict(base=int(rng.choice([-1, 0, 2, 8, 16, 30, 64])), pop_threshold=int(rng.integers(0, 256)),
                sigma_spatial=float(rng.choice([0.4, 1.0, 2.5, 3.3, 8.0, 12.0])), sigma_range=float(rng.choice([2.0, 16.0, 50.0])),
                depth_block=int(rng.integers(4, 40)), alpha=float(rng.choice([0.0, 0.7])), beta=0.3, mode=int(rng.integers(0, 2)), formats=int(rng.choice([1, 3, 4, 5, 7])))
    if over["formats"] & 2 and w % 2: over["formats"] &= ~2
    if over["mode"] != 1 or over["formats"] != 1: continue
    img = chk.synthetic_frame(w, h, i + 1)
    ref = chk.convert(img, oracle.Cfg(**over))
    out = p3s.convert(img, p3s.Config(**over))
    d = np.argwhere(out["anaglyph"] != ref["anaglyph"])
    print(i, w, h, len(d), "chan", np.unique(d[:,0]) if len(d) else None, "rows", np.unique(d[:,1])[:10] if len(d) else None)
    if len(d):
        y = d[0,1]
        print(" got", out["anaglyph"][1, y, :20]); print(" ref", ref["anaglyph"][1, y, :20]); print(" src", img[1, y, :20])
        print(" filt", ref["filtered"][y, :20])
