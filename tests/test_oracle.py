"""CPU: the plain-C oracle port (oracle/p3s_oracle.c) against the reference's golden
vectors (tests/golden, produced by the compiled reference) and, where oracle/_ref exists
in this container, differentially against the reference on randomised configs."""
import hashlib

import numpy as np
import pytest

import oracle
from conftest import load_case


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg_of(entry):
    return oracle.Cfg(**entry["cfg"])


@pytest.mark.parametrize("name", ["default_48x32", "params_67x33", "backward_64x40",
                                  "wide_base_40x30", "sigma_big_50x44", "tiny_1x1", "tiny_1x7",
                                  "tiny_9x1", "thin_2x31"])
def test_port_matches_golden(port, manifest, name):
    entry = manifest["cases"][name]
    cfg = cfg_of(entry)
    g = load_case(name)
    img = port.synthetic_frame(entry["w"], entry["h"], entry["seed"])
    assert np.array_equal(img, g["input"])
    guide = port.luma(img)
    assert np.array_equal(guide, g["luma"])
    edges = port.sobel(guide)
    assert np.array_equal(edges, g["edges"])
    vals = port.block_depth(edges, cfg)
    assert np.array_equal(vals.view(np.uint64), g["block_values"].view(np.uint64))
    depth = port.generate_depth(img, cfg)
    assert np.array_equal(depth, g["depth"])
    assert np.array_equal(port.cross_bilateral(depth, guide, cfg), g["filtered"])
    raw = port.cross_bilateral_raw(depth, guide, cfg)
    assert np.array_equal(raw.view(np.uint64), g["filtered_raw"].view(np.uint64))
    left, right, lm, rm = port.reconstruct(img, g["filtered"], cfg)
    for k, v in dict(left=left, right=right, left_mask=lm, right_mask=rm).items():
        assert np.array_equal(v, g[k]), k
    li, ls = port.inpaint(left, lm, cfg)
    ri, rs = port.inpaint(right, rm, cfg)
    assert np.array_equal(li, g["left_inpainted"]) and ls == tuple(g["left_stats"])
    assert np.array_equal(ri, g["right_inpainted"]) and rs == tuple(g["right_stats"])
    conv = port.convert(img, cfg)
    for k in ("anaglyph", "hsbs", "fsbs"):
        if "convert_" + k in g:
            assert np.array_equal(conv[k], g["convert_" + k]), k


def test_port_matches_reference_digest_1080p(port, manifest):
    d = manifest["digests"]["default_1920x1080"]
    img = port.synthetic_frame(d["w"], d["h"], d["seed"])
    assert sha(img) == d["input"]
    import os
    conv = port.convert(img, cfg_of(d), threads=os.cpu_count() or 1)
    assert sha(conv["depth"]) == d["depth"]
    assert sha(conv["filtered"]) == d["filtered"]
    assert sha(conv["anaglyph"]) == d["anaglyph"]


@pytest.mark.parametrize("name", ["default_3840x2160", "b120_all_3840x2160"])
def test_port_matches_reference_digest_4k(port, manifest, name):
    d = manifest["digests"][name]
    img = port.synthetic_frame(d["w"], d["h"], d["seed"])
    assert sha(img) == d["input"]
    import os
    conv = port.convert(img, cfg_of(d), threads=os.cpu_count() or 1)
    for k in ("depth", "filtered", "anaglyph", "hsbs", "fsbs"):
        if k in d:
            assert sha(conv[k]) == d[k], k


def test_spec_kats(port, manifest):
    # SPEC.md:88 says luma(255,0,0)=76; the reference computes 77
    for r, g, b, y in manifest["kat"]["luma"]:
        got = port.luma(np.array([[[r]], [[g]], [[b]]], np.uint8))[0, 0]
        assert got == y
    assert manifest["kat"]["luma"][0][3] == 77
    for x, d, b, t, left, right in manifest["kat"]["shift_pair"]:
        assert port.shift_pair(x, d, b, t) == (left, right)
    assert port.shift_pair(100, 255, 30, 150) == (85.0, 115.0)
    # 16x16 single block -> constant depth
    img = port.synthetic_frame(16, 16, 4)
    depth = port.generate_depth(img, oracle.Cfg())
    assert len(np.unique(depth)) == 1
    # B = 0 -> anaglyph == source (AC-7)
    img = port.synthetic_frame(33, 21, 2)
    assert np.array_equal(port.convert(img, oracle.Cfg(base=0))["anaglyph"], img)


def test_config_validation_messages(port):
    assert port.validate(oracle.Cfg(base=3)) == "base must be even"
    assert port.validate(oracle.Cfg(base=-2)) == "base must be >= 0"
    assert port.validate(oracle.Cfg(formats=8)) == "unknown output format bit"
    assert port.validate(oracle.Cfg(alpha=0.8, beta=0.3)) == "alpha + beta must be <= 1"
    assert port.validate(oracle.Cfg(depth_block=3)) == "depth_block must be >= 4"
    assert port.validate(oracle.Cfg()) is None
    assert port.effective_base(oracle.Cfg(), 3840) == 30
    assert port.effective_base(oracle.Cfg(), 1920) == 16


def random_cfg(rng):
    return oracle.Cfg(base=int(rng.choice([0, 2, 6, 10, 16, 24, 40])),
                      pop_threshold=int(rng.integers(0, 256)),
                      sigma_spatial=float(rng.choice([0.7, 1.0, 2.5, 3.3, 5.0])),
                      sigma_range=float(rng.choice([3.0, 16.0, 40.0])),
                      depth_block=int(rng.integers(4, 24)),
                      alpha=float(rng.choice([0.0, 0.3, 0.7])), beta=0.3,
                      mode=int(rng.integers(0, 2)), formats=int(rng.choice([1, 4, 5, 7])))


def test_port_differential_vs_reference(port, reference):
    rng = np.random.default_rng(1234)
    for _ in range(25):
        w = int(rng.integers(1, 70))
        h = int(rng.integers(1, 50))
        cfg = random_cfg(rng)
        if cfg.formats & 2 and w % 2:
            cfg.formats &= ~2
        img = reference.synthetic_frame(w, h, int(rng.integers(1, 1000)))
        a = port.convert(img, cfg)
        b = reference.convert(img, cfg)
        for k in ("depth", "filtered", "anaglyph", "hsbs", "fsbs"):
            if k in b:
                assert np.array_equal(a[k], b[k]), (k, w, h, cfg)


def test_inpaint_random_masks_vs_reference(port, reference):
    rng = np.random.default_rng(99)
    for _ in range(30):
        w, h = int(rng.integers(1, 40)), int(rng.integers(1, 30))
        img = rng.integers(0, 256, (3, h, w), dtype=np.uint8)
        mask = (rng.random((h, w)) < rng.choice([0.05, 0.3, 0.8, 0.995])).astype(np.uint8)
        a = port.inpaint(img, mask, oracle.Cfg())
        b = reference.inpaint(img, mask, oracle.Cfg())
        assert np.array_equal(a[0], b[0]) and a[1] == b[1]
