"""CPU: host-side plan logic. The row-band plan of the synchronous p3s_convert schedule (engine.cpp band_plan,
DESIGN.md "Banded synchronous convert") respects the reference's dependency cones for every
band it cuts: the band's filter rows +-r are covered by the depth rows computed so far, those
depth rows only use block rows already valued (depth.cpp:76-121 locate()), those block rows
are fully summed by the depth-front tiles run so far, and the upload covers every Sobel row
they read. Host arithmetic only; no GPU."""
import numpy as np
import pytest

TYB, TD = 128, 16  # filter tile rows, depth-front tile rows


def ri1_of(h, blk):
    """i1 of upsample_block_grid's locate() per row (depth.cpp:82-102)."""
    by = (h + blk - 1) // blk
    c = [i * blk + (min(i * blk + blk, h) - 1 - i * blk) / 2.0 for i in range(by)]
    out = []
    for y in range(h):
        if y <= c[0]:
            i = 0
        elif y >= c[-1]:
            i = by - 1
        else:
            i = 0
            while y > c[i + 1]:
                i += 1
        out.append(min(i + 1, by - 1))
    return out


@pytest.fixture(scope="module")
def p3s():
    import paper_2009_09501_b200 as m
    return m


def check(p3s, w, h, blk, sigma_s):
    cfg = p3s.Config(depth_block=blk, sigma_spatial=sigma_s)
    bands = p3s.band_plan(w, h, cfg)
    r = int(np.ceil(2.0 * sigma_s))
    if not (7 <= r <= 24):
        assert bands == []
        return bands
    if not bands:
        return bands
    by = (h + blk - 1) // blk
    ri1 = ri1_of(h, blk)
    assert bands[-1] == (h, (h + TD - 1) // TD, by, h, (h + TYB - 1) // TYB)
    prev = (0, 0, 0, 0, 0)
    for k, (in_rows, dtile, brow, urow, btile) in enumerate(bands):
        assert all(a >= b for a, b in zip((in_rows, dtile, brow, urow, btile), prev)), bands
        assert btile > prev[4]
        if k + 1 < len(bands):
            need = btile * TYB + r
            assert need <= urow < h                              # filter window rows computed
            assert all(v < brow for v in ri1[:urow])              # those depth rows' block rows
            assert urow == h or ri1[urow] >= brow                 # (and no more than that)
            assert brow * blk <= dtile * TD < h                   # block rows fully summed
            assert in_rows == min(h, dtile * TD + 1)              # + the Sobel row below
            assert need <= dtile * TD                             # luma rows for the guide
        prev = (in_rows, dtile, brow, urow, btile)
    return bands


def test_4k_default_plan(p3s):
    bands = check(p3s, 3840, 2160, 16, 8.0)
    assert [b[4] for b in bands] == [1, 3, 6, 9, 11, 13, 15, 16, 17]  # 1, 2, 3, 3, 2, 2, 2, 1, 1 tile rows
    assert bands[0][0] == 161                                  # upload part 0: 161 rows


def test_random_plans(p3s):
    rng = np.random.default_rng(11)
    for _ in range(300):
        h = int(rng.integers(1, 5000))
        blk = int(rng.integers(4, 200))
        sigma = float(rng.choice([1.0, 3.2, 5.0, 8.0, 11.9, 12.5, 20.0]))
        check(p3s, 1920, h, blk, sigma)


def test_short_frames_are_one_piece(p3s):
    assert p3s.band_plan(640, 64, p3s.Config()) == []
    assert p3s.band_plan(640, 128 + 16, p3s.Config()) == []


def test_dibr_integer_column_tables_verify(p3s):
    """engine.cpp dibr_col_table: for every depth and direction, the reference's truncated
    destination column trunc(fl(x +- sigma_d)) (dibr.cpp:33-41) is x + off + (x >= X), except
    0 at one x; the host derives (off, X, z) from the exact double evaluation of every x and
    verifies it. A sample of widths, bases and thresholds must verify (a failure would only
    route the plan to the FP64 device path, but it would be a regression)."""
    rng = np.random.default_rng(3)
    cases = [(3840, -1, 150), (1920, -1, 150), (7680, -1, 150), (15360, 120, 150)]
    cases += [(int(rng.integers(1, 20000)), int(rng.choice([0, 2, 30, 60, 254, 510, 1000])),
               int(rng.integers(0, 256))) for _ in range(200)]
    for w, base, t in cases:
        cfg = p3s.Config(base=base, pop_threshold=t)
        assert p3s.dibr_integer_columns(w, cfg), (w, base, t)
