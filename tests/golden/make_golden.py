"""Generates tests/golden/ from the REFERENCE itself (oracle/_ref/libp3s_ref.so, compiled
from /root/reference/proj/src by oracle/Makefile). Run in the build container:

    python tests/golden/make_golden.py

Each case stores the synthetic input parameters, the config and every intermediate the
reference's stage API produces (depth, block values, filtered depth + raw means, DIBR
eyes and masks, inpainted eyes + stats, all output formats). Large frames are stored as
SHA-256 digests only. The fixtures pin both the plain-C oracle port and the CUDA path.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # name, w, h, seed, cfg overrides
    ("default_48x32", 48, 32, 1, {}),
    ("params_67x33", 67, 33, 3, dict(base=12, depth_block=5, sigma_spatial=2.5, formats=5,
                                     pop_threshold=100, alpha=0.5, beta=0.4)),
    ("backward_64x40", 64, 40, 5, dict(mode=1, formats=7, base=20)),
    ("wide_base_40x30", 40, 30, 7, dict(base=40, pop_threshold=0, formats=7)),
    ("sigma_big_50x44", 50, 44, 11, dict(sigma_spatial=6.3, sigma_range=5.0, base=16,
                                         depth_block=7, formats=3)),
    ("tiny_1x1", 1, 1, 1, dict(formats=5)),
    ("tiny_1x7", 1, 7, 2, dict(base=4, formats=5)),
    ("tiny_9x1", 9, 1, 5, dict(base=6, formats=5)),
    ("thin_2x31", 2, 31, 9, dict(base=10, formats=7)),
]

DIGEST_CASES = [
    ("default_1920x1080", 1920, 1080, 1, {}),
    # the bench workload (BASELINE configs[1]) and a large-parallax 4K frame, all formats
    ("default_3840x2160", 3840, 2160, 1, {}),
    ("b120_all_3840x2160", 3840, 2160, 2, dict(base=120, formats=7)),
    # the rest of configs[1]'s parallax sweep on the bench frame (B = 30 is the default
    # case above): B = 510 is a 249-pass, 16-round inpaint that no smaller frame reproduces
    *[(f"b{b}_3840x2160", 3840, 2160, 1, dict(base=b)) for b in (0, 2, 16, 60, 254, 510)],
    # configs[4]: 8K anamorph (HSBS) output
    ("hsbs_7680x4320", 7680, 4320, 1, dict(formats=2)),
    # configs[2]/[3] video frames (frame i: seed 1 + i; seed 1 is default_3840x2160): the
    # multi-device sharding test checks every frame against these
    *[(f"video4k_seed{s}", 3840, 2160, s, {}) for s in range(2, 9)],
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_case(R, w, h, seed, over):
    cfg = oracle.Cfg(**over)
    img = R.synthetic_frame(w, h, seed)
    out = {"input": img}
    guide = R.luma(img)
    out["luma"] = guide
    edges = R.sobel(guide)
    out["edges"] = edges
    out["block_values"] = R.block_depth(edges, cfg)
    depth = R.generate_depth(img, cfg)
    out["depth"] = depth
    out["filtered"] = R.cross_bilateral(depth, guide, cfg)
    out["filtered_raw"] = R.cross_bilateral_raw(depth, guide, cfg)
    left, right, lm, rm = R.reconstruct(img, out["filtered"], cfg)
    out.update(left=left, right=right, left_mask=lm, right_mask=rm)
    li, ls = R.inpaint(left, lm, cfg)
    ri, rs = R.inpaint(right, rm, cfg)
    out.update(left_inpainted=li, right_inpainted=ri, left_stats=np.array(ls),
               right_stats=np.array(rs))
    out["anaglyph_stage"] = R.anaglyph(li, ri)
    out["fsbs_stage"] = R.side_by_side(li, ri, False)
    if w % 2 == 0:
        out["hsbs_stage"] = R.side_by_side(li, ri, True)
    conv = R.convert(img, cfg)
    for k in ("anaglyph", "hsbs", "fsbs"):
        if k in conv:
            out["convert_" + k] = conv[k]
    assert (conv["depth"] == depth).all() and (conv["filtered"] == out["filtered"]).all()
    return cfg, out


def main():
    R = oracle.load("reference")
    assert R.kind == "reference", "golden vectors must come from the compiled reference"
    path = os.path.join(OUT, "manifest.json")
    # --digests-only: keep the .npz cases and add the digest cases missing from the manifest
    only = "--digests-only" in sys.argv
    if only:
        with open(path) as f:
            manifest = json.load(f)
    else:
        manifest = {"source": "oracle/_ref/libp3s_ref.so (reference proj/src compiled with "
                              "-O2 -ffp-contract=off)", "cases": {}, "digests": {}}
    for name, w, h, seed, over in ([] if only else CASES):
        cfg, out = run_case(R, w, h, seed, over)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
        manifest["cases"][name] = {"w": w, "h": h, "seed": seed, "cfg": cfg.__dict__}
    for name, w, h, seed, over in DIGEST_CASES:
        if only and name in manifest["digests"]:
            continue
        print("digest", name, flush=True)
        cfg = oracle.Cfg(**over)
        img = R.synthetic_frame(w, h, seed)
        conv = R.convert(img, cfg, threads=os.cpu_count() or 1)
        manifest["digests"][name] = {
            "w": w, "h": h, "seed": seed, "cfg": cfg.__dict__,
            "input": sha(img), "depth": sha(conv["depth"]), "filtered": sha(conv["filtered"]),
            **{k: sha(conv[k]) for k in ("anaglyph", "hsbs", "fsbs") if k in conv},
        }
    # SPEC known-answer tests, as evaluated by the reference code
    kat = {}
    kat["luma"] = [[r, g, b, int(R.luma(np.array([[[r]], [[g]], [[b]]], np.uint8))[0, 0])]
                   for r, g, b in [(255, 0, 0), (0, 255, 0), (0, 0, 255), (255, 255, 255),
                                   (10, 20, 30), (1, 2, 3), (128, 128, 128)]]
    kat["shift_pair"] = [[x, d, b, t, *R.shift_pair(x, d, b, t)]
                         for x, d, b, t in [(100, 255, 30, 150), (100, 150, 30, 150),
                                            (100, 0, 30, 150), (0, 200, 8, 150),
                                            (10, 17, 30, 150), (5, 51, 30, 0), (7, 0, 0, 150)]]
    manifest["kat"] = kat
    with open(path, "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print("wrote", len(CASES), "cases +", len(DIGEST_CASES), "digests")


if __name__ == "__main__":
    main()
