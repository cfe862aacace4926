"""The product's synthetic_frame (p3s_synthetic_frame, host code in the product library)
against the reference's own frames: SHA-256 input digests recorded by
tests/golden/make_golden.py from oracle/_ref, and the small golden cases' stored inputs.
No GPU needed."""
import hashlib

import numpy as np
import pytest

from conftest import load_case


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_synthetic_frame_matches_reference_digests(p3s, manifest):
    seen = set()
    for name, d in manifest["digests"].items():
        key = (d["w"], d["h"], d["seed"])
        if key in seen:
            continue
        seen.add(key)
        assert sha(p3s.synthetic_frame(*key)) == d["input"], name


def test_synthetic_frame_matches_golden_inputs(p3s, manifest):
    for name, entry in manifest["cases"].items():
        g = load_case(name)
        img = p3s.synthetic_frame(entry["w"], entry["h"], entry["seed"])
        assert np.array_equal(img, g["input"]), name


def test_synthetic_frame_rejects_bad_sizes(p3s):
    with pytest.raises(p3s.P3SError):
        p3s.synthetic_frame(0, 4, 1)
