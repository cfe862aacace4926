"""TEST INFRASTRUCTURE ONLY — ctypes/numpy front end for the CPU oracles (oracle.h).

Imported only by tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs,
always as the checker (or the timed CPU baseline), never as the product path.

``load("port")``       -> oracle/_build/libp3s_oracle.so (plain-C restatement)
``load("reference")``  -> oracle/_ref/libp3s_ref.so     (the reference compiled from source)
``load("best")``       -> the reference when it was built, else the port
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libp3s_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libp3s_ref.so")
REF_ROOT = "/root/reference/proj"

u8p = C.POINTER(C.c_uint8)
f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)


class OracleCfg(C.Structure):
    _fields_ = [
        ("base", C.c_int),
        ("pop_threshold", C.c_int),
        ("sigma_spatial", C.c_double),
        ("sigma_range", C.c_double),
        ("depth_block", C.c_int),
        ("inpaint_block", C.c_int),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("mode", C.c_int),
        ("formats", C.c_uint),
    ]


def build(kind: str = "all") -> None:
    """Compile the oracle(s). The reference build needs /root/reference (not on GPU boxes)."""
    targets = ["port"]
    if kind in ("all", "ref", "reference") and os.path.isdir(REF_ROOT):
        targets.append("ref")
    subprocess.check_call(["make", "-s", "-C", HERE, "-j8", *targets])


def _ptr(a: np.ndarray, t=u8p):
    return a.ctypes.data_as(t)


@dataclass
class Cfg:
    """Python mirror of p3s::ConversionConfig (reference config.hpp:25-43)."""

    base: int = -1
    pop_threshold: int = 150
    sigma_spatial: float = 8.0
    sigma_range: float = 16.0
    depth_block: int = 16
    inpaint_block: int = 64
    alpha: float = 0.7
    beta: float = 0.3
    mode: int = 0
    formats: int = 1

    def c(self) -> OracleCfg:
        return OracleCfg(self.base, self.pop_threshold, self.sigma_spatial, self.sigma_range,
                         self.depth_block, self.inpaint_block, self.alpha, self.beta, self.mode,
                         self.formats)


class Oracle:
    def __init__(self, path: str):
        self.path = path
        self.lib = L = C.CDLL(path)
        L.oracle_kind.restype = C.c_char_p
        self.kind = L.oracle_kind().decode()
        L.oracle_validate.argtypes = [C.POINTER(OracleCfg), C.c_char_p, C.c_size_t]
        L.oracle_effective_base.argtypes = [C.POINTER(OracleCfg), C.c_int]
        L.oracle_synthetic_frame.argtypes = [C.c_int, C.c_int, C.c_uint64, u8p, u8p, u8p]
        L.oracle_luma.argtypes = [u8p, u8p, u8p, C.c_size_t, u8p]
        L.oracle_sobel.argtypes = [u8p, C.c_int, C.c_int, u8p]
        L.oracle_block_depth.argtypes = [u8p, C.c_int, C.c_int, C.POINTER(OracleCfg), f64p]
        L.oracle_upsample.argtypes = [f64p, C.c_int, C.c_int, C.c_int, u8p]
        L.oracle_generate_depth.argtypes = [u8p, u8p, u8p, C.c_int, C.c_int,
                                            C.POINTER(OracleCfg), u8p]
        L.oracle_cross_bilateral_raw.argtypes = [u8p, u8p, C.c_int, C.c_int,
                                                 C.POINTER(OracleCfg), C.c_int, f64p]
        L.oracle_cross_bilateral.argtypes = [u8p, u8p, C.c_int, C.c_int, C.POINTER(OracleCfg),
                                             C.c_int, u8p]
        L.oracle_shift_pair.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, f64p, f64p]
        L.oracle_reconstruct.argtypes = [u8p, u8p, u8p, u8p, C.c_int, C.c_int,
                                         C.POINTER(OracleCfg), C.c_int] + [u8p] * 8
        L.oracle_inpaint.argtypes = [u8p, u8p, u8p, u8p, C.c_int, C.c_int, C.POINTER(OracleCfg),
                                     C.c_int, u8p, u8p, u8p, i64p]
        L.oracle_anaglyph.argtypes = [u8p] * 6 + [C.c_int, C.c_int] + [u8p] * 3
        L.oracle_side_by_side.argtypes = [u8p] * 6 + [C.c_int, C.c_int, C.c_int] + [u8p] * 3
        L.oracle_convert.argtypes = ([u8p, u8p, u8p, C.c_int, C.c_int, C.POINTER(OracleCfg),
                                     C.c_int] + [u8p] * 11 + [i64p, C.c_char_p, C.c_size_t])

    # -- helpers -----------------------------------------------------------------------
    def validate(self, cfg: Cfg):
        buf = C.create_string_buffer(256)
        rc = self.lib.oracle_validate(C.byref(cfg.c()), buf, 256)
        return None if rc == 0 else buf.value.decode()

    def effective_base(self, cfg: Cfg, w: int) -> int:
        return self.lib.oracle_effective_base(C.byref(cfg.c()), w)

    def synthetic_frame(self, w: int, h: int, seed: int = 1) -> np.ndarray:
        img = np.zeros((3, h, w), np.uint8)
        self.lib.oracle_synthetic_frame(w, h, seed, _ptr(img[0]), _ptr(img[1]), _ptr(img[2]))
        return img

    def luma(self, img: np.ndarray) -> np.ndarray:
        img = np.ascontiguousarray(img)
        out = np.zeros(img.shape[1:], np.uint8)
        self.lib.oracle_luma(_ptr(img[0]), _ptr(img[1]), _ptr(img[2]), out.size, _ptr(out))
        return out

    def sobel(self, gray: np.ndarray) -> np.ndarray:
        gray = np.ascontiguousarray(gray)
        out = np.zeros_like(gray)
        self.lib.oracle_sobel(_ptr(gray), gray.shape[1], gray.shape[0], _ptr(out))
        return out

    def block_depth(self, edges: np.ndarray, cfg: Cfg) -> np.ndarray:
        h, w = edges.shape
        b = cfg.depth_block
        out = np.zeros(((h + b - 1) // b, (w + b - 1) // b), np.float64)
        self.lib.oracle_block_depth(_ptr(np.ascontiguousarray(edges)), w, h, C.byref(cfg.c()),
                                    _ptr(out, f64p))
        return out

    def upsample(self, values: np.ndarray, w: int, h: int, block: int) -> np.ndarray:
        out = np.zeros((h, w), np.uint8)
        self.lib.oracle_upsample(_ptr(np.ascontiguousarray(values, np.float64), f64p), w, h,
                                 block, _ptr(out))
        return out

    def generate_depth(self, img: np.ndarray, cfg: Cfg) -> np.ndarray:
        img = np.ascontiguousarray(img)
        out = np.zeros(img.shape[1:], np.uint8)
        self.lib.oracle_generate_depth(_ptr(img[0]), _ptr(img[1]), _ptr(img[2]), img.shape[2],
                                       img.shape[1], C.byref(cfg.c()), _ptr(out))
        return out

    def cross_bilateral(self, depth, guide, cfg: Cfg, threads: int = 1) -> np.ndarray:
        depth, guide = np.ascontiguousarray(depth), np.ascontiguousarray(guide)
        out = np.zeros_like(depth)
        self.lib.oracle_cross_bilateral(_ptr(depth), _ptr(guide), depth.shape[1],
                                        depth.shape[0], C.byref(cfg.c()), threads, _ptr(out))
        return out

    def cross_bilateral_raw(self, depth, guide, cfg: Cfg, threads: int = 1) -> np.ndarray:
        depth, guide = np.ascontiguousarray(depth), np.ascontiguousarray(guide)
        out = np.zeros(depth.shape, np.float64)
        self.lib.oracle_cross_bilateral_raw(_ptr(depth), _ptr(guide), depth.shape[1],
                                            depth.shape[0], C.byref(cfg.c()), threads,
                                            _ptr(out, f64p))
        return out

    def shift_pair(self, x: int, d: int, base: int, t: int):
        a, b = C.c_double(), C.c_double()
        self.lib.oracle_shift_pair(x, d, base, t, C.byref(a), C.byref(b))
        return a.value, b.value

    def reconstruct(self, img, depth, cfg: Cfg, threads: int = 1):
        img, depth = np.ascontiguousarray(img), np.ascontiguousarray(depth)
        _, h, w = img.shape
        left = np.zeros_like(img)
        right = np.zeros_like(img)
        lm = np.zeros((h, w), np.uint8)
        rm = np.zeros((h, w), np.uint8)
        self.lib.oracle_reconstruct(_ptr(img[0]), _ptr(img[1]), _ptr(img[2]), _ptr(depth), w, h,
                                    C.byref(cfg.c()), threads, _ptr(left[0]), _ptr(left[1]),
                                    _ptr(left[2]), _ptr(right[0]), _ptr(right[1]),
                                    _ptr(right[2]), _ptr(lm), _ptr(rm))
        return left, right, lm, rm

    def inpaint(self, img, mask, cfg: Cfg, threads: int = 1):
        img, mask = np.ascontiguousarray(img), np.ascontiguousarray(mask)
        _, h, w = img.shape
        out = np.zeros_like(img)
        st = np.zeros(3, np.int64)
        self.lib.oracle_inpaint(_ptr(img[0]), _ptr(img[1]), _ptr(img[2]), _ptr(mask), w, h,
                                C.byref(cfg.c()), threads, _ptr(out[0]), _ptr(out[1]),
                                _ptr(out[2]), _ptr(st, i64p))
        return out, tuple(int(v) for v in st)

    def anaglyph(self, left, right):
        left, right = np.ascontiguousarray(left), np.ascontiguousarray(right)
        _, h, w = left.shape
        out = np.zeros_like(left)
        self.lib.oracle_anaglyph(*[_ptr(p) for p in (*left, *right)], w, h,
                                 *[_ptr(p) for p in out])
        return out

    def side_by_side(self, left, right, half: bool):
        left, right = np.ascontiguousarray(left), np.ascontiguousarray(right)
        _, h, w = left.shape
        out = np.zeros((3, h, w if half else 2 * w), np.uint8)
        rc = self.lib.oracle_side_by_side(*[_ptr(p) for p in (*left, *right)], w, h, int(half),
                                          *[_ptr(p) for p in out])
        if rc:
            raise ValueError("side_by_side: half mode requires an even width")
        return out

    def convert(self, img, cfg: Cfg, threads: int = 1):
        """Full convert_image. Returns dict(depth, filtered, anaglyph?, hsbs?, fsbs?, timings)."""
        img = np.ascontiguousarray(img)
        _, h, w = img.shape
        depth = np.zeros((h, w), np.uint8)
        filt = np.zeros((h, w), np.uint8)
        ana = np.zeros((3, h, w), np.uint8)
        hsbs = np.zeros((3, h, w), np.uint8)
        fsbs = np.zeros((3, h, 2 * w), np.uint8)
        t = np.zeros(7, np.int64)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_convert(_ptr(img[0]), _ptr(img[1]), _ptr(img[2]), w, h,
                                     C.byref(cfg.c()), threads, _ptr(depth), _ptr(filt),
                                     *[_ptr(p) for p in ana], *[_ptr(p) for p in hsbs],
                                     *[_ptr(p) for p in fsbs], _ptr(t, i64p), msg, 256)
        if rc:
            raise ValueError(msg.value.decode())
        out = {"depth": depth, "filtered": filt, "timings": t}
        if cfg.formats & 1:
            out["anaglyph"] = ana
        if cfg.formats & 2:
            out["hsbs"] = hsbs
        if cfg.formats & 4:
            out["fsbs"] = fsbs
        return out


_cache: dict = {}


def available(kind: str) -> bool:
    return os.path.exists(REF_SO if kind == "reference" else PORT_SO)


def load(kind: str = "best") -> Oracle:
    if kind == "best":
        kind = "reference" if os.path.exists(REF_SO) else "port"
    path = REF_SO if kind == "reference" else PORT_SO
    if not os.path.exists(path):
        build("all" if kind == "reference" else "port")
    if path not in _cache:
        _cache[path] = Oracle(path)
    return _cache[path]
