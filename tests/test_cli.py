"""The p3s command-line front end (SPEC.md [MODULE] cli): a thin
mapping of convert / depth / video / bench onto the C ABI with exit codes 0 ok, 1 usage,
2 I/O, 3 decode (4 internal). CPU tests cover argument handling and the host-side error
paths; GPU tests compare every output with the oracle."""
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2009_09501_b200", "p3s")


def run(*args, cwd=None):
    if not os.path.exists(CLI):
        pytest.fail("p3s CLI not built (make -C paper_2009_09501_b200)")
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=False, cwd=cwd, timeout=600)


def write_ppm(path, img):
    c, h, w = img.shape
    with open(path, "wb") as f:
        f.write(b"P6\n%d %d\n255\n" % (w, h))
        f.write(np.ascontiguousarray(img.transpose(1, 2, 0)).tobytes())


def read_pnm(path):
    data = open(path, "rb").read()
    parts, pos = [], 0
    while len(parts) < 4:
        while data[pos:pos + 1].isspace():
            pos += 1
        end = pos
        while not data[end:end + 1].isspace():
            end += 1
        parts.append(data[pos:end])
        pos = end
    pos += 1
    w, h = int(parts[1]), int(parts[2])
    payload = np.frombuffer(data[pos:], np.uint8)
    if parts[0] == b"P6":
        return payload.reshape(h, w, 3).transpose(2, 0, 1)
    return payload.reshape(h, w)


def test_usage_errors_exit_1(tmp_path):
    assert run().returncode == 1
    assert run("--help").returncode == 0
    assert run("frobnicate").returncode == 1
    r = run("convert", "x.ppm", "--bogus")
    assert r.returncode == 1 and b"unknown flag --bogus" in r.stderr
    assert run("convert", "x.ppm").returncode == 1              # no --out
    assert run("convert", "--out", str(tmp_path)).returncode == 1  # no input
    assert run("convert", "x.ppm", "--out", str(tmp_path), "--format", "3d").returncode == 1
    assert run("convert", "x.ppm", "--out", str(tmp_path), "--base", "x").returncode == 1
    assert run("convert", "x.ppm", "--out", str(tmp_path), "--mode", "sideways").returncode == 1
    assert run("video", "--in", str(tmp_path)).returncode == 1
    assert run("bench", "--sizes", "64by64").returncode == 1


def test_invalid_config_exit_1(tmp_path):
    # the C ABI setters validate (config.cpp:8-31): odd base, negative sigma
    write_ppm(tmp_path / "a.ppm", np.zeros((3, 4, 4), np.uint8))
    r = run("convert", tmp_path / "a.ppm", "--out", tmp_path, "--base", "3")
    assert r.returncode == 1 and b"base must be even" in r.stderr
    assert run("convert", tmp_path / "a.ppm", "--out", tmp_path, "--sigma-range", "-1").returncode == 1


def test_io_and_decode_errors(tmp_path):
    r = run("convert", tmp_path / "missing.ppm", "--out", tmp_path)
    assert r.returncode == 2
    (tmp_path / "bad.ppm").write_bytes(b"P6\n2 2\n255\nabc")
    r = run("convert", tmp_path / "bad.ppm", "--out", tmp_path)
    assert r.returncode == 3 and b"truncated" in r.stderr
    (tmp_path / "bad2.ppm").write_bytes(b"P5\n2 2\n255\nabcd")
    assert run("depth", tmp_path / "bad2.ppm", "--out", tmp_path / "d.pgm").returncode == 3


@pytest.mark.gpu
def test_convert_b0_is_identity(tmp_path):
    # SPEC cli example: convert --format anaglyph --base 0 --mode forward -> output == input
    img = oracle.load("port").synthetic_frame(97, 61, 5)
    write_ppm(tmp_path / "img.ppm", img)
    r = run("convert", tmp_path / "img.ppm", "--format", "anaglyph", "--base", "0", "--mode", "forward",
            "--out", tmp_path)
    assert r.returncode == 0, r.stderr
    assert np.array_equal(read_pnm(tmp_path / "img_anaglyph.ppm"), img)


@pytest.mark.gpu
def test_convert_depth_video_match_oracle(tmp_path):
    chk = oracle.load("port")
    img = chk.synthetic_frame(160, 90, 7)
    write_ppm(tmp_path / "f.ppm", img)
    args = ["--base", "12", "--sigma-spatial", "3.5", "--depth-block", "9", "--pop-threshold", "120"]
    cfg = oracle.Cfg(base=12, sigma_spatial=3.5, depth_block=9, pop_threshold=120, formats=7)
    ref = chk.convert(img, cfg)
    r = run("convert", tmp_path / "f.ppm", "--out", tmp_path, "--format", "anaglyph", "--format", "hsbs",
            "--format", "fsbs", "--emit-depth", *args)
    assert r.returncode == 0, r.stderr
    for k in ("anaglyph", "hsbs", "fsbs"):
        assert np.array_equal(read_pnm(tmp_path / f"f_{k}.ppm"), ref[k]), k
    assert np.array_equal(read_pnm(tmp_path / "f_depth.pgm"), ref["depth"])
    r = run("depth", tmp_path / "f.ppm", "--out", tmp_path / "only.pgm", *args)
    assert r.returncode == 0, r.stderr
    assert np.array_equal(read_pnm(tmp_path / "only.pgm"), ref["depth"])
    # video on a directory of 3 frames -> 3 outputs + summary line + 3 CSV rows, exit 0
    vin, vout = tmp_path / "in", tmp_path / "out"
    vin.mkdir()
    vout.mkdir()
    frames = [chk.synthetic_frame(64, 48, 1 + i) for i in range(3)]
    for i, f in enumerate(frames):
        write_ppm(vin / f"frame_{i:06d}.ppm", f)
    r = run("video", "--in", vin, "--pattern", "frame_%06d.ppm", "--out", vout,
            "--timing-csv", tmp_path / "t.csv")
    assert r.returncode == 0, r.stderr
    assert b"frames=3" in r.stdout
    for i, f in enumerate(frames):
        assert np.array_equal(read_pnm(vout / f"frame_{i:06d}_anaglyph.ppm"), chk.convert(f, oracle.Cfg())["anaglyph"])
    assert len(open(tmp_path / "t.csv").read().strip().splitlines()) == 4


@pytest.mark.gpu
def test_bench_rows_and_odd_hsbs(tmp_path):
    # SPEC cli example: bench --threads 1 --reps 3 --sizes 64x64 --csv - -> 3 CSV rows + header
    r = run("bench", "--threads", "1", "--reps", "3", "--sizes", "64x64", "--csv", "-")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.decode().strip().splitlines()
    assert lines[0].startswith("width,height,threads,rep,") and len(lines) == 4
    # odd width with HSBS -> usage error
    write_ppm(tmp_path / "odd.ppm", oracle.load("port").synthetic_frame(33, 20, 2))
    r = run("convert", tmp_path / "odd.ppm", "--out", tmp_path, "--format", "hsbs")
    assert r.returncode == 1 and b"even width" in r.stderr
