"""Determinism stress for the banded synchronous p3s_convert: many back-to-back calls over
alternating frames and sizes (plan switches, graph replays, early downloads + patch) must
return exactly the bytes of the first call for that frame. Optional oracle check of the
first outputs (--oracle)."""
import argparse, hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2009_09501_b200 as p3s

ap = argparse.ArgumentParser()
ap.add_argument("--calls", type=int, default=300)
ap.add_argument("--oracle", action="store_true")
args = ap.parse_args()
p3s.set_device(0)
chk = oracle.load("port")
cases = [((3840, 2160), 1, {}), ((3840, 2160), 2, {}), ((1920, 1080), 3, dict(base=40)),
         ((960, 540), 4, dict(formats=4)), ((1280, 720), 5, dict(formats=7, mode=1))]
frames = {i: chk.synthetic_frame(w, h, seed) for i, ((w, h), seed, _) in enumerate(cases)}
cfgs = {i: p3s.Config(**over) for i, (_, _, over) in enumerate(cases)}
first = {}
rng = np.random.default_rng(5)
for n in range(args.calls):
    i = int(rng.integers(0, len(cases))) if n >= len(cases) else n
    out = p3s.convert(frames[i], cfgs[i])
    digest = {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
              for k, v in out.items() if isinstance(v, np.ndarray)}
    if i not in first:
        first[i] = digest
        if args.oracle:
            ref = chk.convert(frames[i], oracle.Cfg(**cases[i][2]), threads=os.cpu_count() or 1)
            for k in ("depth", "filtered", "anaglyph", "hsbs", "fsbs"):
                if k in ref:
                    assert np.array_equal(out[k], ref[k]), (i, k)
    elif digest != first[i]:
        bad = [k for k in digest if digest[k] != first[i].get(k)]
        raise SystemExit(f"call {n}: case {i} differs from its first call in {bad}")
print(f"stress ok: {args.calls} calls over {len(cases)} frames/configs, all outputs stable")
