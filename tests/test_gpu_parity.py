"""GPU parity: every stage and the full p3s_convert of the CUDA path, through the C ABI,
byte-exact (and bit-exact for FP64 raw means) against the reference's golden vectors and
the live CPU oracle (compiled reference when present, else the C port)."""
import hashlib
import os

import numpy as np
import pytest

from conftest import ROOT, load_case

pytestmark = pytest.mark.gpu

GOLDEN_CASES = ["default_48x32", "params_67x33", "backward_64x40", "wide_base_40x30",
                "sigma_big_50x44", "tiny_1x1", "tiny_1x7", "tiny_9x1", "thin_2x31"]
NCPU = os.cpu_count() or 1


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def pcfg(p3s, d):
    return p3s.Config(**d)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_stages_match_golden(p3s, manifest, name):
    entry = manifest["cases"][name]
    cfg = pcfg(p3s, entry["cfg"])
    g = load_case(name)
    img = g["input"]
    assert np.array_equal(p3s.luma(img), g["luma"])
    vals = p3s.block_depth(img, cfg)
    assert np.array_equal(vals.view(np.uint64), g["block_values"].view(np.uint64))
    assert np.array_equal(p3s.upsample(g["block_values"], entry["w"], entry["h"],
                                       entry["cfg"]["depth_block"]), g["depth"])
    assert np.array_equal(p3s.generate_depth(img, cfg), g["depth"])
    assert np.array_equal(p3s.cross_bilateral(g["depth"], g["luma"], cfg), g["filtered"])
    raw = p3s.cross_bilateral_raw(g["depth"], g["luma"], cfg)
    assert np.array_equal(raw.view(np.uint64), g["filtered_raw"].view(np.uint64))
    left, right, lm, rm = p3s.reconstruct(img, g["filtered"], cfg)
    for k, v in dict(left=left, right=right, left_mask=lm, right_mask=rm).items():
        assert np.array_equal(v, g[k]), k
    li, ls = p3s.inpaint(g["left"], g["left_mask"], cfg)
    ri, rs = p3s.inpaint(g["right"], g["right_mask"], cfg)
    assert np.array_equal(li, g["left_inpainted"]) and ls == tuple(g["left_stats"])
    assert np.array_equal(ri, g["right_inpainted"]) and rs == tuple(g["right_stats"])
    assert np.array_equal(p3s.anaglyph(li, ri), g["anaglyph_stage"])
    assert np.array_equal(p3s.side_by_side(li, ri, False), g["fsbs_stage"])
    if "hsbs_stage" in g:
        assert np.array_equal(p3s.side_by_side(li, ri, True), g["hsbs_stage"])
    out = p3s.convert(img, cfg)
    assert np.array_equal(out["depth"], g["depth"])
    assert np.array_equal(out["filtered"], g["filtered"])
    for k in ("anaglyph", "hsbs", "fsbs"):
        if "convert_" + k in g:
            assert np.array_equal(out[k], g["convert_" + k]), k


def test_1080p_matches_reference_digest(p3s, manifest):
    d = manifest["digests"]["default_1920x1080"]
    img = p3s.synthetic_frame(d["w"], d["h"], d["seed"])
    assert sha(img) == d["input"]
    out = p3s.convert(img, pcfg(p3s, d["cfg"]))
    assert sha(out["depth"]) == d["depth"]
    assert sha(out["filtered"]) == d["filtered"]
    assert sha(out["anaglyph"]) == d["anaglyph"]


DIGESTS_4K8K = ["default_3840x2160", "b120_all_3840x2160", "b0_3840x2160", "b2_3840x2160",
                "b16_3840x2160", "b60_3840x2160", "b254_3840x2160", "b510_3840x2160",
                "hsbs_7680x4320"]


@pytest.mark.parametrize("name", DIGESTS_4K8K)
def test_4k_8k_match_reference_digest(p3s, manifest, name):
    """The bench workload, configs[1]'s whole parallax sweep B in {0,2,16,30,60,120,254,510}
    at 4K (B = 510: a 249-pass, 16-round inpaint) and configs[4]'s 8K HSBS frame, against
    SHA-256 digests of the REFERENCE's own output (tests/golden/make_golden.py, oracle/_ref).
    Inputs come from the product's synthetic_frame, pinned by the manifest's input digest."""
    d = manifest["digests"][name]
    img = p3s.synthetic_frame(d["w"], d["h"], d["seed"])
    assert sha(img) == d["input"]
    out = p3s.convert(img, pcfg(p3s, d["cfg"]))
    for k in ("depth", "filtered", "anaglyph", "hsbs", "fsbs"):
        if k in d:
            assert sha(out[k]) == d[k], k
    # the device-resident pipeline (CUDA-graph replay, the bench's value loop) and the
    # streamed video API give the same bytes
    if d["cfg"].get("formats", 1) == 1:
        pipe = p3s.Pipeline(d["w"], d["h"], pcfg(p3s, d["cfg"]))
        buf = p3s.DeviceBuffer(pipe.frame_bytes)
        pipe.upload(img, buf.addr)
        for _ in range(3):  # direct launch, graph capture, graph replay
            pipe.run(buf.addr)
        depth, filt, ana = pipe.download()
        assert sha(ana) == d["anaglyph"] and sha(filt) == d["filtered"]


def compare_convert(p3s, checker, img, over):
    import oracle
    ref = checker.convert(img, oracle.Cfg(**over), threads=NCPU)
    out = p3s.convert(img, p3s.Config(**over))
    for k in ("depth", "filtered", "anaglyph", "hsbs", "fsbs"):
        if k in ref:
            if not np.array_equal(out[k], ref[k]):
                diff = np.argwhere(out[k] != ref[k])
                raise AssertionError(f"{k} differs at {len(diff)} px, first {diff[:3]} cfg={over}")
    return out


def test_random_sizes_and_configs(p3s, checker):
    rng = np.random.default_rng(7)
    for i in range(24):
        w, h = int(rng.integers(1, 300)), int(rng.integers(1, 200))
        over = dict(base=int(rng.choice([-1, 0, 2, 8, 16, 30, 64])),
                    pop_threshold=int(rng.integers(0, 256)),
                    sigma_spatial=float(rng.choice([0.4, 1.0, 2.5, 3.3, 8.0, 12.0])),
                    sigma_range=float(rng.choice([2.0, 16.0, 50.0])),
                    depth_block=int(rng.integers(4, 40)), alpha=float(rng.choice([0.0, 0.7])),
                    beta=0.3, mode=int(rng.integers(0, 2)), formats=int(rng.choice([1, 3, 4, 5, 7])))
        if over["formats"] & 2 and w % 2:
            over["formats"] &= ~2
        img = checker.synthetic_frame(w, h, i + 1)
        compare_convert(p3s, checker, img, over)


@pytest.mark.parametrize("w,h", [(16, 1), (16, 16), (32, 9), (48, 33), (1024, 17), (1040, 40),
                                 (2064, 50), (3072, 31)])
def test_fused_depth_front_shapes(p3s, checker, w, h):
    """The fused depth front (16-pixel blocks, w % 16 == 0: one thread per block, block
    values written directly) at its edges: one-block frames, partial last block rows,
    partial last CTAs (w not a multiple of 1024), one-row frames (clamped Sobel rows)."""
    img = checker.synthetic_frame(w, h, w + h)
    compare_convert(p3s, checker, img, dict(formats=1))
    compare_convert(p3s, checker, img, dict(formats=1, alpha=0.0, beta=1.0, base=8))


def test_random_fused_paths(p3s, checker):
    """Random shapes on the round-2 fast paths: the fused depth stage (w % 16 == 0, 16-pixel
    blocks), the quad DIBR splat fast path and its left-edge general region (large bases),
    and the interleaved video path (PPM-order payloads in and out), against the oracle."""
    import oracle
    rng = np.random.default_rng(11)
    for i in range(10):
        w = 16 * int(rng.integers(1, 90))
        h = int(rng.integers(1, 140))
        over = dict(base=int(rng.choice([-1, 0, 2, 30, 100, 254])),
                    pop_threshold=int(rng.integers(0, 256)),
                    sigma_spatial=float(rng.choice([2.5, 8.0])), alpha=float(rng.choice([0.0, 0.7])),
                    beta=float(rng.choice([0.0, 0.3])), formats=1)
        img = checker.synthetic_frame(w, h, 100 + i)
        compare_convert(p3s, checker, img, over)
        if i % 3 == 0:
            cfg = p3s.Config(**over)
            src, dst = p3s.PinnedBuffer(3 * w * h), p3s.PinnedBuffer(3 * w * h)
            src.array[:] = img.transpose(1, 2, 0).reshape(-1)
            vid = p3s.Video(w, h, cfg, streams=1)
            vid.convert_ptrs([src.ptr], [dst.ptr], interleaved=True)
            ref = checker.convert(img, oracle.Cfg(**over), threads=NCPU)["anaglyph"]
            assert np.array_equal(dst.array.reshape(h, w, 3), np.ascontiguousarray(ref.transpose(1, 2, 0))), over


@pytest.mark.parametrize("base", [0, 2, 16, 30, 60, 120, 254, 510])
def test_parallax_sweep_540p(p3s, checker, base):
    img = checker.synthetic_frame(960, 540, 3)
    compare_convert(p3s, checker, img, dict(base=base))


def test_large_radius_generic_kernel(p3s, checker):
    # sigma_s = 23 -> r = 46 > the tiled kernel's 43: exercises the generic path
    img = checker.synthetic_frame(130, 90, 5)
    compare_convert(p3s, checker, img, dict(sigma_spatial=23.0, formats=7, base=20))


def _identity(t):
    assert t["pure_ns"] == t["filter_ns"] + t["dibr_ns"] + t["inpaint_left_ns"] + \
        t["inpaint_right_ns"] + t["format_ns"]


def test_4k_default_full(p3s, checker):
    """The banded p3s_convert (pinned 4K frame): bytes = oracle, and its stage times are a
    partition of the frame's GPU timeline (engine.cpp banded_stage_ms): every stage present,
    the filter dominant, both eyes' inpaint reported, the reference's pure_ns identity."""
    img = p3s.synthetic_frame(3840, 2160, 1)
    out = compare_convert(p3s, checker, img, {})
    t = out["timings"]
    _identity(t)
    assert t["depth_gen_ns"] > 0 and t["dibr_ns"] > 0 and t["format_ns"] >= 0
    assert t["inpaint_left_ns"] > 0 and t["inpaint_right_ns"] > 0
    assert t["filter_ns"] > 5 * max(t["depth_gen_ns"], t["dibr_ns"])
    # non-banded reference point (P3S_BANDED-free path: a timed pipeline run of the same frame)
    pipe = p3s.Pipeline(3840, 2160, p3s.Config())
    buf = p3s.DeviceBuffer(pipe.frame_bytes)
    pipe.upload(img, buf.addr)
    pipe.run(buf.addr, timed=True)
    tp = pipe.timings()
    _identity(tp)
    assert 0.5 < t["filter_ns"] / tp["filter_ns"] < 1.5
    assert 0.25 < t["depth_gen_ns"] / tp["depth_gen_ns"] < 4


def test_b0_identity_and_backward_has_no_holes(p3s, checker):
    """B = 0 (forward) and backward mode leave no damage: the reference skips the inpaint
    (pipeline.cpp:56-65), so both eyes report 0 ns, on the banded and the plain path."""
    img = p3s.synthetic_frame(322, 177, 9)
    out = p3s.convert(img, p3s.Config(base=0))
    assert np.array_equal(out["anaglyph"], img)
    assert out["timings"]["inpaint_left_ns"] == 0 and out["timings"]["inpaint_right_ns"] == 0
    _identity(out["timings"])
    out = p3s.convert(img, p3s.Config(mode=1, formats=7))
    assert out["timings"]["inpaint_left_ns"] == 0 and out["timings"]["inpaint_right_ns"] == 0
    big = p3s.synthetic_frame(1920, 1080, 3)  # tall enough for the banded schedule
    out = p3s.convert(big, p3s.Config(base=0))
    assert out["timings"]["inpaint_left_ns"] == 0 and out["timings"]["inpaint_right_ns"] == 0
    _identity(out["timings"])
    pipe = p3s.Pipeline(1920, 1080, p3s.Config(base=0))
    buf = p3s.DeviceBuffer(pipe.frame_bytes)
    pipe.upload(big, buf.addr)
    pipe.run(buf.addr, timed=True)
    t = pipe.timings()
    assert t["inpaint_left_ns"] == 0 and t["inpaint_right_ns"] == 0


def test_result_maps_survive_later_work(p3s, checker):
    """p3s_result_depth / _filtered_depth of an earlier result stay valid (downloaded in the
    background) while later conversions reuse the plan."""
    import ctypes as C
    import oracle
    L = p3s.lib()
    cfg = p3s.Config()
    frames = [p3s.synthetic_frame(640, 360, s) for s in (1, 2, 3)]
    imgs = [p3s.Image(f) for f in frames]
    results = []
    for im in imgs:
        r = C.c_void_p()
        p3s._check(L.p3s_convert(im.h, cfg.h, C.byref(r)))
        results.append(r)
    try:
        for f, r in zip(frames, results):
            ref = checker.convert(f, oracle.Cfg(), threads=NCPU)
            d = L.p3s_result_depth(r)
            fd = L.p3s_result_filtered_depth(r)
            assert d and fd
            assert np.array_equal(p3s._gray_to_numpy(d), ref["depth"])
            assert np.array_equal(p3s._gray_to_numpy(fd), ref["filtered"])
    finally:
        for r in results:
            L.p3s_result_free(r)


def test_odd_width_hsbs_is_invalid(p3s):
    img = np.zeros((3, 4, 5), np.uint8)
    with pytest.raises(p3s.P3SError) as e:
        p3s.convert(img, p3s.Config(formats=2))
    assert e.value.status == 1
    assert e.value.message == "side_by_side: half mode requires an even width"


def test_device_pipeline_and_video_match_convert(p3s, checker):
    w, h = 640, 360
    cfg = p3s.Config(base=24)
    frames = [checker.synthetic_frame(w, h, s) for s in range(1, 7)]
    expect = [p3s.convert(f, cfg)["anaglyph"] for f in frames]
    pipe = p3s.Pipeline(w, h, cfg)
    dbuf = p3s.DeviceBuffer(pipe.frame_bytes)
    for f, e in zip(frames, expect):
        pipe.upload(f, dbuf.addr)
        pipe.run(dbuf.addr, timed=True)
        _, _, out = pipe.download()
        assert np.array_equal(out, e)
    vid = p3s.Video(w, h, cfg, streams=3)
    n = w * h * 3
    src = [p3s.PinnedBuffer(n) for _ in frames]
    dst = [p3s.PinnedBuffer(n) for _ in frames]
    for b, f in zip(src, frames):
        b.array[:] = f.reshape(-1)
    vid.convert_ptrs([b.ptr for b in src], [b.ptr for b in dst])
    for b, e in zip(dst, expect):
        assert np.array_equal(b.array.reshape(3, h, w), e)


def test_stream_and_plan_invariance(p3s, checker):
    # bytes do not depend on which plan/stream ran them (GPU analogue of AC-1)
    img = checker.synthetic_frame(500, 300, 4)
    a = p3s.convert(img, p3s.Config(formats=7, base=22))
    b = p3s.convert(img, p3s.Config(formats=1, base=22))
    c = p3s.convert(img, p3s.Config(formats=4, base=22))
    assert np.array_equal(a["anaglyph"], b["anaglyph"])
    assert np.array_equal(a["fsbs"], c["fsbs"])


def _stress_mask(rng, w, h):
    kind = int(rng.integers(0, 4))
    if kind == 0:  # uniform random density (dense -> mid-course stalls + gray fallback)
        return (rng.random((h, w)) < rng.choice([0.05, 0.3, 0.8, 0.97, 0.995])).astype(np.uint8)
    m = np.zeros((h, w), np.uint8)
    if kind == 1:  # wide vertical strips (many passes, multi-round temporal blocking)
        for _ in range(int(rng.integers(1, 6))):
            x = int(rng.integers(0, w))
            m[:, x:x + int(rng.integers(1, 90))] = 1
    elif kind == 2:  # DIBR-like staircase runs along a slanted edge
        for y in range(h):
            x = int((y * rng.uniform(0.2, 3.0)) % max(w, 1))
            m[y, x:x + int(rng.integers(1, 40))] = 1
    else:  # blobs + full-height border strip
        m[:, : int(rng.integers(1, 20))] = 1
        for _ in range(int(rng.integers(1, 8))):
            cx, cy, r = int(rng.integers(0, w)), int(rng.integers(0, h)), int(rng.integers(2, 50))
            yy, xx = np.ogrid[:h, :w]
            m[(yy - cy) ** 2 + (xx - cx) ** 2 < r * r] = 1
    return m


def test_inpaint_stress_vs_oracle(p3s, checker):
    """Jacobi inpaint on adversarial masks: wide strips needing many 16-pass rounds, dense
    random damage that stalls mid-course (gray fallback), thin frames, tile-edge sizes."""
    import oracle
    rng = np.random.default_rng(2024)
    sizes = [(1, 1), (1, 97), (97, 1), (2, 63), (31, 33), (64, 64), (65, 31), (200, 130),
             (333, 211), (700, 300)]
    for i in range(30):
        w, h = sizes[i % len(sizes)]
        img = rng.integers(0, 256, (3, h, w), dtype=np.uint8)
        mask = _stress_mask(rng, w, h)
        a, sa = p3s.inpaint(img, mask, p3s.Config())
        b, sb = checker.inpaint(img, mask, oracle.Cfg())
        assert np.array_equal(a, b), (i, w, h, int(mask.sum()))
        assert tuple(sa) == tuple(sb), (i, w, h, sa, sb)


def test_video_frame_sharding_matches_oracle(p3s, checker):
    """Multi-device frame sharding (p3s_video_create_devices): one host thread per device
    takes frames from a shared counter. On a one-GPU box the device is listed several times,
    which runs the same threading, queue and ordering logic; bytes must equal the CPU
    oracle's."""
    import oracle
    w, h = 320, 200
    over = dict(base=18, formats=p3s.FSBS)
    cfg = p3s.Config(**over)
    frames = [p3s.synthetic_frame(w, h, s) for s in range(1, 10)]
    expect = [checker.convert(f, oracle.Cfg(**over), threads=NCPU)["fsbs"] for f in frames]
    ndev = p3s.device_count()
    devices = [i % ndev for i in range(3)]
    vid = p3s.Video(w, h, cfg, streams=2, devices=devices)
    assert vid.shards == 3
    src = [p3s.PinnedBuffer(3 * w * h) for _ in frames]
    dst = [p3s.PinnedBuffer(3 * 2 * w * h) for _ in frames]
    for b, f in zip(src, frames):
        b.array[:] = f.reshape(-1)
    vid.convert_ptrs([b.ptr for b in src], [b.ptr for b in dst])
    for b, e in zip(dst, expect):
        assert np.array_equal(b.array.reshape(3, h, 2 * w), e)
    assert vid.requeued == 0 and vid.healthy_shards == 3


def test_video_4k_every_device_matches_reference_digests(p3s, manifest):
    """configs[2]/[3]: 4K video frames (frame i: seed 1 + i) sharded over every visible
    device (listed twice on a one-GPU box), pinned rings on each device's NUMA node, each
    anaglyph against the SHA-256 digest of the REFERENCE's own output."""
    names = ["default_3840x2160"] + [f"video4k_seed{s}" for s in range(2, 9)]
    digests = [manifest["digests"][n] for n in names]
    w, h = 3840, 2160
    ndev = p3s.device_count()
    devices = list(range(ndev)) if ndev > 1 else [0, 0]
    vid = p3s.Video(w, h, p3s.Config(), streams=2, devices=devices)
    src, dst = [], []
    for i, d in enumerate(digests):
        dev = devices[i % len(devices)]
        b = p3s.PinnedBuffer(3 * w * h, near_device=dev)
        b.array[:] = p3s.synthetic_frame(w, h, d["seed"]).reshape(-1)
        src.append(b)
        dst.append(p3s.PinnedBuffer(3 * w * h, near_device=dev))
    vid.convert_ptrs([b.ptr for b in src], [b.ptr for b in dst])
    for b, d in zip(dst, digests):
        assert sha(b.array) == d["anaglyph"], d["seed"]


def test_video_failed_device_frames_are_requeued(p3s, checker, monkeypatch):
    """A device failure (injected on shard 1 after 2 frames) retires that shard and re-runs
    every frame it took on the healthy shards; the call succeeds with the oracle's bytes."""
    import oracle
    monkeypatch.setenv("P3S_VIDEO_FAIL", "1:2")
    w, h = 160, 96
    over = dict(base=12)
    frames = [p3s.synthetic_frame(w, h, s) for s in range(1, 13)]
    expect = [checker.convert(f, oracle.Cfg(**over), threads=NCPU)["anaglyph"] for f in frames]
    vid = p3s.Video(w, h, p3s.Config(**over), streams=2, devices=[0, 0, 0])
    src = [p3s.PinnedBuffer(3 * w * h) for _ in frames]
    dst = [p3s.PinnedBuffer(3 * w * h) for _ in frames]
    for b, f in zip(src, frames):
        b.array[:] = f.reshape(-1)
    vid.convert_ptrs([b.ptr for b in src], [b.ptr for b in dst])
    assert vid.healthy_shards == 2 and vid.requeued >= 3
    for b, e in zip(dst, expect):
        assert np.array_equal(b.array.reshape(3, h, w), e)
    # the retired shard stays out of later calls
    for b in dst:
        b.array[:] = 0
    vid.convert_ptrs([b.ptr for b in src], [b.ptr for b in dst])
    for b, e in zip(dst, expect):
        assert np.array_equal(b.array.reshape(3, h, w), e)


def _ppm_bytes(img):
    _, h, w = img.shape
    return f"P6\n{w} {h}\n255\n".encode() + np.ascontiguousarray(img.transpose(1, 2, 0)).tobytes()


def test_convert_sequence_files_match_oracle(p3s, checker, tmp_path):
    """p3s_convert_sequence (reference sequence.cpp:52-145): PPM payloads go to the GPU
    as raw bytes (de-interleaved there) and come back interleaved; every output file must
    equal the oracle's frame encoded as P6. A corrupt frame stops the sequence with a decode
    error after the earlier frames' outputs were written."""
    import ctypes as C
    import oracle
    L = p3s.lib()
    src, out = tmp_path / "in", tmp_path / "out"
    src.mkdir()
    out.mkdir()
    sizes = [(96, 64), (96, 64), (50, 37), (96, 64)]  # a size change mid-sequence
    frames = [checker.synthetic_frame(w, h, 10 + i) for i, (w, h) in enumerate(sizes)]
    for i, f in enumerate(frames):
        (src / f"f_{i + 1:03d}.ppm").write_bytes(_ppm_bytes(f))  # starts at 1 (no frame 0)
    over = dict(base=10, formats=5)
    cfg = p3s.Config(**over)
    summ = p3s.SequenceSummary()
    csv = C.c_void_p()
    st = L.p3s_convert_sequence(str(src).encode(), b"f_%03d.ppm", str(out).encode(), cfg.h,
                                C.byref(summ), C.byref(csv))
    assert st == 0, L.p3s_last_error()
    assert summ.frames == 4
    text = C.string_at(L.p3s_buffer_data(csv), L.p3s_buffer_size(csv)).decode()
    L.p3s_buffer_free(csv)
    assert len(text.strip().splitlines()) == 5
    for i, f in enumerate(frames):
        ref = checker.convert(f, oracle.Cfg(**over))
        for name in ("anaglyph", "fsbs"):
            got = (out / f"f_{i + 1:03d}_{name}.ppm").read_bytes()
            assert got == _ppm_bytes(ref[name]), (i, name)
    # corrupt frame 3 -> DECODE error naming it; frames 1-2 written before
    (src / "f_003.ppm").write_bytes(b"P6\n50 37\n255\n\x00\x01")
    out2 = tmp_path / "out2"
    out2.mkdir()
    st = L.p3s_convert_sequence(str(src).encode(), b"f_%03d.ppm", str(out2).encode(), cfg.h,
                                None, None)
    assert st == 3
    assert b"frame 3" in L.p3s_last_error()
    assert sorted(p.name for p in out2.iterdir()) == sorted(
        f"f_{i:03d}_{n}.ppm" for i in (1, 2) for n in ("anaglyph", "fsbs"))
    # anaglyph only: the fused interleaved kernels for the 96-wide frames, planes for 50x37
    (src / "f_003.ppm").write_bytes(_ppm_bytes(frames[2]))
    over = dict(base=10, formats=1)
    out3 = tmp_path / "out3"
    out3.mkdir()
    cfg3 = p3s.Config(**over)
    st = L.p3s_convert_sequence(str(src).encode(), b"f_%03d.ppm", str(out3).encode(), cfg3.h,
                                None, None)
    assert st == 0, L.p3s_last_error()
    for i, f in enumerate(frames):
        ref = checker.convert(f, oracle.Cfg(**over))
        assert (out3 / f"f_{i + 1:03d}_anaglyph.ppm").read_bytes() == _ppm_bytes(ref["anaglyph"]), i


def test_video_interleaved_matches_oracle(p3s, checker):
    """p3s_video_convert_interleaved: PPM-order payloads in/out, (de)interleave on the GPU;
    both the 16-pixel vector path (w % 16 == 0) and the per-pixel path (odd width), against
    the CPU oracle's planar output interleaved on the host."""
    import oracle
    # anaglyph-only, forward, w % 16 == 0: the fused kernels read and write the payload
    # directly (no (de)interleave pass); the others split / join planes on the GPU
    for (w, h, fmt, extra) in ((128, 72, p3s.ANAGLYPH, {}), (1920, 1080, p3s.ANAGLYPH, dict(base=90)),
                               (128, 72, p3s.ANAGLYPH, dict(mode=1)), (97, 41, p3s.FSBS, {})):
        over = dict(base=12, formats=fmt)
        over.update(extra)
        cfg = p3s.Config(**over)
        frames = [p3s.synthetic_frame(w, h, s) for s in range(1, 5)]
        key = "anaglyph" if fmt == p3s.ANAGLYPH else "fsbs"
        expect = [checker.convert(f, oracle.Cfg(**over), threads=NCPU)[key] for f in frames]
        ow = 2 * w if fmt == p3s.FSBS else w
        src = [p3s.PinnedBuffer(3 * w * h) for _ in frames]
        dst = [p3s.PinnedBuffer(3 * ow * h) for _ in frames]
        for b, f in zip(src, frames):
            b.array[:] = f.transpose(1, 2, 0).reshape(-1)
        vid = p3s.Video(w, h, cfg, streams=2)
        vid.convert_ptrs([b.ptr for b in src], [b.ptr for b in dst], interleaved=True)
        for b, e in zip(dst, expect):
            assert np.array_equal(b.array.reshape(h, ow, 3), np.ascontiguousarray(e.transpose(1, 2, 0)))


@pytest.mark.parametrize("sigma_s", [3.1, 4.0, 4.3, 5.0, 5.5, 6.0, 6.5, 7.0, 7.4, 8.0, 8.3, 9.0,
                                     9.5, 10.0, 10.3, 11.0, 11.4, 12.0])
def test_certified_bilateral_radii(p3s, checker, sigma_s):
    """The certified FP32 bilateral covers radii 7..24 (ceil(2 sigma_s)); every radius must
    give the reference's filtered depth and anaglyph (odd size: clipped windows, edge tiles,
    a partial last tile row)."""
    img = checker.synthetic_frame(333, 277, int(sigma_s * 10))
    compare_convert(p3s, checker, img, dict(sigma_spatial=sigma_s, sigma_range=float(6 + sigma_s)))


def test_widest_shared_memory_rows(p3s, checker):
    """Up to 18768 px a DIBR row lives in one CTA's shared memory: the widest such frame
    converts bit-exactly in every route."""
    wmax = 18768
    img = checker.synthetic_frame(wmax, 6, 5)
    compare_convert(p3s, checker, img, dict(formats=7, base=60))
    compare_convert(p3s, checker, img, dict(formats=1))


@pytest.mark.parametrize("w,h", [(18784, 5), (20001, 4), (33000, 3)])
def test_rows_wider_than_shared_memory(p3s, checker, w, h):
    """Wider rows (the reference converts any width, dibr.cpp:65-104) keep the DIBR z-buffer
    in global per-CTA key slots: same bytes in every route, forward and backward, with the
    integer column tables (w < 32768) and the FP64 shift path (w >= 32768)."""
    img = checker.synthetic_frame(w, h, w % 97)
    compare_convert(p3s, checker, img, dict(formats=1))
    compare_convert(p3s, checker, img, dict(formats=5 if w % 2 else 7, base=90))
    compare_convert(p3s, checker, img, dict(formats=1, mode=1, base=40))


@pytest.mark.parametrize("w,h,block,sigma_s", [(500, 700, 4, 8.0), (1283, 389, 37, 3.1),
                                               (640, 1031, 16, 12.0), (900, 600, 64, 5.5),
                                               (777, 2100, 23, 8.0), (18768, 300, 16, 8.0)])
def test_banded_convert_boundaries(p3s, checker, w, h, block, sigma_s):
    """p3s_convert on pinned planes uploads the frame in two row parts and filters band A
    while band B is still crossing PCIe (engine.cpp plan_bands). The band edges depend on
    the depth block size, the radius and the height; every split must give the reference's
    bytes, and consecutive frames through the same captured graph must too."""
    over = dict(depth_block=block, sigma_spatial=sigma_s, alpha=0.7, beta=0.3,
                formats=7 if w % 2 == 0 else 5, base=20)
    for seed in (3, 4):
        compare_convert(p3s, checker, checker.synthetic_frame(w, h, seed), over)


@pytest.mark.parametrize("ctas", [1, 5, 37])
def test_inpaint_cta_cap_is_invisible(p3s, checker, ctas):
    """Pipeline.set_inpaint_ctas (the throughput option) changes only how many CTAs run the
    cooperative inpaint: multi-round damage (large parallax), graph replay after the change
    and the timed path all give the oracle's bytes and pass statistics."""
    w, h = 480, 270
    cfg = p3s.Config(base=90, formats=1)
    img = checker.synthetic_frame(w, h, 11)
    ref = checker.convert(img, __import__("oracle").Cfg(base=90, formats=1), threads=NCPU)
    pipe = p3s.Pipeline(w, h, cfg)
    dbuf = p3s.DeviceBuffer(pipe.frame_bytes)
    pipe.upload(img, dbuf.addr)
    pipe.run(dbuf.addr)  # graph captured with one CTA per SM
    pipe.set_inpaint_ctas(ctas)
    for timed in (False, True, False):
        pipe.run(dbuf.addr, timed=timed)
        _, _, out = pipe.download()
        assert np.array_equal(out, ref["anaglyph"])
    with pytest.raises(p3s.P3SError):
        pipe.set_inpaint_ctas(-1)


def test_banded_convert_random_configs(p3s, checker):
    """Random configurations through the row-banded p3s_convert (frames tall enough for
    several bands): every route, both DIBR modes, random parallax, depth blocks, radii and
    depth weights, against the oracle."""
    rng = np.random.default_rng(2024)
    for i in range(8):
        w = int(rng.integers(200, 641)) & ~1
        h = int(rng.integers(300, 721))
        over = dict(base=int(rng.choice([-1, 0, 8, 30, 64, 120])),
                    pop_threshold=int(rng.integers(0, 256)),
                    sigma_spatial=float(rng.choice([3.2, 5.0, 8.0, 11.5])),
                    sigma_range=float(rng.choice([6.0, 16.0, 40.0])),
                    depth_block=int(rng.integers(4, 48)), alpha=float(rng.choice([0.0, 0.5, 0.7])),
                    beta=0.3, mode=int(rng.integers(0, 2)), formats=int(rng.choice([1, 2, 4, 7])))
        img = checker.synthetic_frame(w, h, 100 + i)
        compare_convert(p3s, checker, img, over)


def test_convert_is_deterministic_across_calls():
    """tools/stress_convert.py: back-to-back p3s_convert calls over alternating frames, sizes
    and routes (plan switches, graph replays, the banded early downloads and host patch)
    return the same bytes every time."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress_convert.py"), "--calls", "80"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "stress ok" in r.stdout, r.stdout + r.stderr


def test_concurrent_convert_threads(p3s, checker):
    """p3s_convert from several host threads at once (reference capi.cpp: thread-safe on
    distinct handles): each thread gets its own plans and streams on the device, the banded
    schedules of different threads overlap on the GPU, and every result equals the
    single-threaded one."""
    import threading
    frames = [checker.synthetic_frame(640 + 32 * i, 480 + 16 * i, 40 + i) for i in range(4)]
    cfgs = [p3s.Config(), p3s.Config(formats=7, base=24), p3s.Config(mode=1), p3s.Config(formats=4)]
    expect = [p3s.convert(f, c) for f, c in zip(frames, cfgs)]
    errors = []

    def work(k):
        try:
            for rep in range(6):
                i = (k + rep) % 4
                out = p3s.convert(frames[i], cfgs[i])
                for key in ("anaglyph", "hsbs", "fsbs", "depth", "filtered"):
                    if key in expect[i] and not np.array_equal(out[key], expect[i][key]):
                        errors.append((k, rep, key))
        except Exception as e:  # noqa: BLE001 - surfaced by the assert below
            errors.append((k, repr(e)))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:5]


def _near_tie_cases(w, h):
    """Depth/guide pairs built to put the filtered value on or next to a .5 boundary: flat
    guides make the weights purely spatial, so two-level depth patterns average to k + 0.5
    up to the centre tap's and the window edges' asymmetry."""
    yy, xx = np.mgrid[0:h, 0:w]
    flat = np.full((h, w), 128, np.uint8)
    cases = {
        "checker": ((100 + ((xx + yy) & 1)).astype(np.uint8), flat),
        "row_stripes": ((40 + (yy & 1)).astype(np.uint8), flat),
        "col_stripes": ((200 + (xx & 1)).astype(np.uint8), flat),
        "wide_steps": ((10 * ((xx // 3) % 2) + 77).astype(np.uint8), flat),
        # a two-level guide: the range weights split the window into two classes
        "guide_edge": ((60 + ((xx + yy) & 1)).astype(np.uint8),
                       np.where(xx < w // 2, 90, 91).astype(np.uint8)),
        "saturated": (np.where((xx + yy) & 1, 255, 254).astype(np.uint8), flat),
    }
    return cases


@pytest.mark.parametrize("sigma_s", [8.0, 3.5, 11.7])
def test_bilateral_near_ties_vs_oracle(p3s, checker, sigma_s):
    """The certified FP32 filter (k_bilateral_sep, FP32 row folds) must defer every pixel it
    cannot prove to the exact FP64 fix-up: on inputs whose filtered values sit on or next to
    .5 boundaries the bytes still equal the reference's (bilateral.cpp:40-85)."""
    import oracle
    w, h = 213, 149
    cfg = p3s.Config(sigma_spatial=sigma_s, sigma_range=16.0)
    ocfg = oracle.Cfg(sigma_spatial=sigma_s, sigma_range=16.0)
    for name, (depth, guide) in _near_tie_cases(w, h).items():
        got = p3s.cross_bilateral(depth, guide, cfg)
        ref = checker.cross_bilateral(depth, guide, ocfg, threads=NCPU)
        assert np.array_equal(got, ref), (name, int((got != ref).sum()))
