"""paper_2009_09501_b200 — B200-native pseudo-stereo (2D -> 3D) synthesis.

The product is the in-tree C-ABI library ``libpseudo3d_b200.so`` (include/pseudo3d.h:
the reference's 49 functions; include/p3s_gpu.h: GPU extensions) over hand-written
sm_100a kernels. This module is a thin ctypes mirror of that C ABI with numpy arrays in
and out, shaped like the reference's own API (reference proj/include/pseudo3d.h) so tests
and harnesses read like the reference's usage. It contains no compute: every call goes
through the CUDA library, and importing it fails loudly when the library is not built.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# P3S_LIB_PATH: an in-tree experiment build (make VARIANT=...); default the product library
LIB_PATH = os.environ.get("P3S_LIB_PATH") or os.path.join(HERE, "libpseudo3d_b200.so")

P3S_OK, P3S_ERR_INVALID, P3S_ERR_IO, P3S_ERR_DECODE, P3S_ERR_INTERNAL = range(5)
MODE_FORWARD, MODE_BACKWARD = 0, 1
ANAGLYPH, HSBS, FSBS = 1, 2, 4

u8p = C.POINTER(C.c_uint8)
f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
vp = C.c_void_p


def build(jobs: int = 8) -> None:
    """Compile the CUDA/C++ library in-tree (nvcc cross-compiles sm_100a without a GPU)."""
    subprocess.check_call(["make", "-s", "-C", HERE, f"-j{jobs}"])


class P3SError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[{status}] {message}")
        self.status = status
        self.message = message


class Timings(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("depth_gen_ns", "filter_ns", "dibr_ns",
                                          "inpaint_left_ns", "inpaint_right_ns", "format_ns",
                                          "pure_ns")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class SequenceSummary(C.Structure):
    _fields_ = [("frames", C.c_int64), ("pure_sum_ns", C.c_int64), ("pure_min_ns", C.c_int64),
                ("pure_max_ns", C.c_int64), ("pure_mean_ns", C.c_double), ("wall_ns", C.c_int64)]


class Params(C.Structure):
    _fields_ = [("base", C.c_int), ("pop_threshold", C.c_int), ("sigma_spatial", C.c_double),
                ("sigma_range", C.c_double), ("depth_block", C.c_int),
                ("inpaint_block", C.c_int), ("alpha", C.c_double), ("beta", C.c_double),
                ("mode", C.c_int), ("formats", C.c_uint)]


_SIGS = {
    # pseudo3d.h
    "p3s_version": (C.c_char_p, []),
    "p3s_status_name": (C.c_char_p, [C.c_int]),
    "p3s_last_error": (C.c_char_p, []),
    "p3s_buffer_data": (vp, [vp]),
    "p3s_buffer_size": (C.c_size_t, [vp]),
    "p3s_buffer_free": (None, [vp]),
    "p3s_image_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(vp)]),
    "p3s_image_free": (None, [vp]),
    "p3s_image_width": (C.c_int, [vp]),
    "p3s_image_height": (C.c_int, [vp]),
    "p3s_image_plane": (vp, [vp, C.c_int]),
    "p3s_image_plane_mut": (vp, [vp, C.c_int]),
    "p3s_image_decode_ppm": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(vp)]),
    "p3s_image_encode_ppm": (C.c_int, [vp, C.POINTER(vp)]),
    "p3s_image_load_ppm": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "p3s_image_save_ppm": (C.c_int, [C.c_char_p, vp]),
    "p3s_graymap_free": (None, [vp]),
    "p3s_graymap_width": (C.c_int, [vp]),
    "p3s_graymap_height": (C.c_int, [vp]),
    "p3s_graymap_data": (vp, [vp]),
    "p3s_graymap_decode_pgm": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(vp)]),
    "p3s_graymap_encode_pgm": (C.c_int, [vp, C.POINTER(vp)]),
    "p3s_graymap_load_pgm": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "p3s_graymap_save_pgm": (C.c_int, [C.c_char_p, vp]),
    "p3s_config_create": (vp, []),
    "p3s_config_free": (None, [vp]),
    "p3s_config_set_base": (C.c_int, [vp, C.c_int]),
    "p3s_config_set_auto_base": (C.c_int, [vp]),
    "p3s_config_set_pop_threshold": (C.c_int, [vp, C.c_int]),
    "p3s_config_set_sigma_spatial": (C.c_int, [vp, C.c_double]),
    "p3s_config_set_sigma_range": (C.c_int, [vp, C.c_double]),
    "p3s_config_set_depth_block": (C.c_int, [vp, C.c_int]),
    "p3s_config_set_inpaint_block": (C.c_int, [vp, C.c_int]),
    "p3s_config_set_depth_weights": (C.c_int, [vp, C.c_double, C.c_double]),
    "p3s_config_set_mode": (C.c_int, [vp, C.c_int]),
    "p3s_config_set_formats": (C.c_int, [vp, C.c_uint]),
    "p3s_config_set_threads": (C.c_int, [vp, C.c_int]),
    "p3s_convert": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "p3s_result_output": (C.c_int, [vp, C.c_int, C.POINTER(vp)]),
    "p3s_result_depth": (vp, [vp]),
    "p3s_result_filtered_depth": (vp, [vp]),
    "p3s_result_timings": (C.c_int, [vp, C.POINTER(Timings)]),
    "p3s_result_free": (None, [vp]),
    "p3s_depth_map": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "p3s_convert_sequence": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, vp,
                                       C.POINTER(SequenceSummary), C.POINTER(vp)]),
    "p3s_bench": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_size_t,
                            C.POINTER(C.c_int), C.c_size_t, C.c_int, C.c_uint64, vp,
                            C.POINTER(vp)]),
    "p3s_bench_report_csv": (C.c_int, [vp, C.POINTER(vp)]),
    "p3s_bench_report_speedup": (C.c_double, [vp, C.c_int, C.c_int, C.c_int]),
    "p3s_bench_report_free": (None, [vp]),
    # p3s_gpu.h
    "p3s_config_get_params": (C.c_int, [vp, C.POINTER(Params)]),
    "p3s_config_set_params": (C.c_int, [vp, C.POINTER(Params)]),
    "p3s_gpu_device_count": (C.c_int, []),
    "p3s_gpu_set_device": (C.c_int, [C.c_int]),
    "p3s_gpu_device_name": (C.c_int, [C.c_char_p, C.c_size_t]),
    "p3s_gpu_sm_count": (C.c_int, [C.POINTER(C.c_int)]),
    "p3s_gpu_band_plan": (C.c_int, [C.c_int, C.c_int, vp, C.POINTER(C.c_int), C.c_int]),
    "p3s_gpu_dibr_integer_columns": (C.c_int, [C.c_int, vp]),
    "p3s_pipeline_set_inpaint_ctas": (C.c_int, [vp, C.c_int]),
    "p3s_gpu_luma": (C.c_int, [u8p, u8p, u8p, C.c_int, C.c_int, u8p]),
    "p3s_gpu_block_depth": (C.c_int, [u8p, u8p, u8p, C.c_int, C.c_int, vp, f64p]),
    "p3s_gpu_upsample": (C.c_int, [f64p, C.c_int, C.c_int, C.c_int, u8p]),
    "p3s_gpu_generate_depth": (C.c_int, [u8p, u8p, u8p, C.c_int, C.c_int, vp, u8p]),
    "p3s_gpu_cross_bilateral": (C.c_int, [u8p, u8p, C.c_int, C.c_int, vp, u8p]),
    "p3s_gpu_cross_bilateral_raw": (C.c_int, [u8p, u8p, C.c_int, C.c_int, vp, f64p]),
    "p3s_gpu_reconstruct": (C.c_int, [u8p, u8p, u8p, u8p, C.c_int, C.c_int, vp] + [u8p] * 8),
    "p3s_gpu_inpaint": (C.c_int, [u8p, u8p, u8p, u8p, C.c_int, C.c_int, vp, u8p, u8p, u8p,
                                  i64p]),
    "p3s_gpu_anaglyph": (C.c_int, [u8p] * 6 + [C.c_int, C.c_int] + [u8p] * 3),
    "p3s_gpu_side_by_side": (C.c_int, [u8p] * 6 + [C.c_int, C.c_int, C.c_int] + [u8p] * 3),
    "p3s_pipeline_create": (C.c_int, [C.c_int, C.c_int, vp, C.POINTER(vp)]),
    "p3s_pipeline_free": (None, [vp]),
    "p3s_pipeline_pitch": (C.c_int, [vp]),
    "p3s_pipeline_frame_bytes": (C.c_size_t, [vp]),
    "p3s_pipeline_stream": (vp, [vp]),
    "p3s_pipeline_run": (C.c_int, [vp, vp, C.c_int, vp]),
    "p3s_pipeline_timings": (C.c_int, [vp, C.POINTER(Timings)]),
    "p3s_pipeline_timing_sum": (C.c_int, [vp, C.POINTER(Timings), i64p, C.c_int]),
    "p3s_pipeline_download": (C.c_int, [vp, u8p, u8p, C.c_int, u8p, u8p, u8p]),
    "p3s_pipeline_inpaint_stats": (C.c_int, [vp, i64p]),
    "p3s_pipeline_upload": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "p3s_video_create": (C.c_int, [C.c_int, C.c_int, vp, C.c_int, C.POINTER(vp)]),
    "p3s_video_convert": (C.c_int, [vp, C.POINTER(vp), C.c_int, C.POINTER(vp)]),
    "p3s_video_create_devices": (C.c_int, [C.c_int, C.c_int, vp, C.POINTER(C.c_int), C.c_int,
                                           C.c_int, C.POINTER(vp)]),
    "p3s_video_shards": (C.c_int, [vp]),
    "p3s_video_convert_interleaved": (C.c_int, [vp, C.POINTER(vp), C.c_int, C.POINTER(vp)]),
    "p3s_video_free": (None, [vp]),
    "p3s_gpu_malloc": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
    "p3s_gpu_free": (None, [vp]),
    "p3s_gpu_memset": (C.c_int, [vp, C.c_int, C.c_size_t]),
    "p3s_gpu_stream_sync": (C.c_int, [vp]),
    "p3s_gpu_device_sync": (C.c_int, []),
    "p3s_gpu_event_create": (C.c_int, [C.POINTER(vp)]),
    "p3s_gpu_event_record": (C.c_int, [vp, vp]),
    "p3s_gpu_stream_wait_event": (C.c_int, [vp, vp]),
    "p3s_pipeline_bilateral_kernel_sum": (C.c_int, [vp, i64p, i64p, C.c_int]),
    "p3s_gpu_event_elapsed_ms": (C.c_int, [vp, vp, C.POINTER(C.c_float)]),
    "p3s_gpu_event_destroy": (None, [vp]),
    "p3s_host_alloc": (vp, [C.c_size_t]),
    "p3s_host_free": (None, [vp]),
    "p3s_gpu_fp64_peak": (C.c_int, [C.POINTER(C.c_double)]),
    "p3s_gpu_smem_peak": (C.c_int, [C.POINTER(C.c_double), C.c_int]),
    "p3s_gpu_bilateral_path": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "p3s_synthetic_frame": (C.c_int, [C.c_int, C.c_int, C.c_uint64, u8p, u8p, u8p]),
    "p3s_video_requeued": (C.c_longlong, [vp]),
    "p3s_video_healthy_shards": (C.c_int, [vp]),
    "p3s_gpu_numa_node": (C.c_int, [C.c_int]),
    "p3s_host_alloc_near": (vp, [C.c_int, C.c_size_t]),
    "p3s_gpu_launch_count": (C.c_ulonglong, []),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded product library. Raises if it was not built (no silent fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() or "
                              f"make -C {HERE}")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != P3S_OK:
        raise P3SError(status, lib().p3s_last_error().decode())


def _p(a: np.ndarray, t=u8p):
    return a.ctypes.data_as(t)


def last_error() -> str:
    return lib().p3s_last_error().decode()


def version() -> str:
    return lib().p3s_version().decode()


def device_count() -> int:
    return lib().p3s_gpu_device_count()


def set_device(ordinal: int) -> None:
    _check(lib().p3s_gpu_set_device(ordinal))


def band_plan(w: int, h: int, cfg: "Config"):
    """Row bands of the synchronous p3s_convert schedule: a list of (upload rows, depth
    tile rows, block rows, depth rows, filter tile rows) band ends; [] = one piece."""
    buf = (C.c_int * (5 * 64))()
    n = lib().p3s_gpu_band_plan(w, h, cfg.h, buf, 64)
    if n < 0:
        raise P3SError(1, lib().p3s_last_error().decode())
    return [tuple(buf[5 * i:5 * i + 5]) for i in range(n)]


def dibr_integer_columns(w: int, cfg: "Config") -> bool:
    """True when plans of width w use the host-verified integer DIBR column tables."""
    r = lib().p3s_gpu_dibr_integer_columns(w, cfg.h)
    if r < 0:
        raise P3SError(1, lib().p3s_last_error().decode())
    return bool(r)


def sm_count() -> int:
    n = C.c_int()
    _check(lib().p3s_gpu_sm_count(C.byref(n)))
    return n.value


def device_name() -> str:
    buf = C.create_string_buffer(256)
    _check(lib().p3s_gpu_device_name(buf, 256))
    return buf.value.decode()


class Config:
    """Owning wrapper of p3s_config (reference pseudo3d.h:109-124)."""

    def __init__(self, **kw):
        self.h = lib().p3s_config_create()
        if not self.h:
            raise MemoryError("p3s_config_create")
        if kw:
            self.set(**kw)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.p3s_config_free(self.h)
            self.h = None

    def params(self) -> Params:
        p = Params()
        _check(lib().p3s_config_get_params(self.h, C.byref(p)))
        return p

    def set(self, **kw) -> "Config":
        p = self.params()
        for k, v in kw.items():
            if k == "threads":
                _check(lib().p3s_config_set_threads(self.h, int(v)))
                continue
            if not hasattr(p, k):
                raise KeyError(k)
            setattr(p, k, v)
        _check(lib().p3s_config_set_params(self.h, C.byref(p)))
        return self


def _image_from_numpy(img: np.ndarray):
    img = np.ascontiguousarray(img, np.uint8)
    _, h, w = img.shape
    handle = vp()
    _check(lib().p3s_image_create(w, h, C.byref(handle)))
    n = w * h
    for c in range(3):
        dst = lib().p3s_image_plane_mut(handle, c)
        C.memmove(dst, img[c].ctypes.data, n)
    return handle


def _image_to_numpy(handle) -> np.ndarray:
    L = lib()
    w, h = L.p3s_image_width(handle), L.p3s_image_height(handle)
    out = np.empty((3, h, w), np.uint8)
    for c in range(3):
        C.memmove(out[c].ctypes.data, L.p3s_image_plane(handle, c), w * h)
    return out


def _gray_to_numpy(handle) -> np.ndarray:
    L = lib()
    w, h = L.p3s_graymap_width(handle), L.p3s_graymap_height(handle)
    out = np.empty((h, w), np.uint8)
    C.memmove(out.ctypes.data, L.p3s_graymap_data(handle), w * h)
    return out


class Image:
    """Owning p3s_image handle (planes are in the library's pinned host pool)."""

    def __init__(self, arr: np.ndarray | None = None, handle=None):
        self.h = handle if handle is not None else _image_from_numpy(arr)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.p3s_image_free(self.h)
            self.h = None

    def numpy(self) -> np.ndarray:
        return _image_to_numpy(self.h)


def convert(img, cfg: Config):
    """p3s_convert through the drop-in C ABI. Returns dict(depth, filtered, <formats>, timings)."""
    L = lib()
    im = img if isinstance(img, Image) else Image(img)
    res = vp()
    _check(L.p3s_convert(im.h, cfg.h, C.byref(res)))
    try:
        out = {"depth": _gray_to_numpy(L.p3s_result_depth(res)),
               "filtered": _gray_to_numpy(L.p3s_result_filtered_depth(res))}
        fm = cfg.params().formats
        for bit, name in ((ANAGLYPH, "anaglyph"), (HSBS, "hsbs"), (FSBS, "fsbs")):
            if fm & bit:
                o = vp()
                _check(L.p3s_result_output(res, bit, C.byref(o)))
                out[name] = _image_to_numpy(o)
        t = Timings()
        _check(L.p3s_result_timings(res, C.byref(t)))
        out["timings"] = t.as_dict()
        return out
    finally:
        L.p3s_result_free(res)


def depth_map(img, cfg: Config) -> np.ndarray:
    L = lib()
    im = img if isinstance(img, Image) else Image(img)
    g = vp()
    _check(L.p3s_depth_map(im.h, cfg.h, C.byref(g)))
    try:
        return _gray_to_numpy(g)
    finally:
        L.p3s_graymap_free(g)


# ---- stage entry points (p3s_gpu.h) ----------------------------------------------------
def _planes(img):
    img = np.ascontiguousarray(img, np.uint8)
    return img, [_p(img[c]) for c in range(3)]


def luma(img) -> np.ndarray:
    img, pl = _planes(img)
    out = np.zeros(img.shape[1:], np.uint8)
    _check(lib().p3s_gpu_luma(*pl, img.shape[2], img.shape[1], _p(out)))
    return out


def block_depth(img, cfg: Config) -> np.ndarray:
    img, pl = _planes(img)
    _, h, w = img.shape
    b = cfg.params().depth_block
    out = np.zeros(((h + b - 1) // b, (w + b - 1) // b), np.float64)
    _check(lib().p3s_gpu_block_depth(*pl, w, h, cfg.h, _p(out, f64p)))
    return out


def upsample(values: np.ndarray, w: int, h: int, block: int) -> np.ndarray:
    values = np.ascontiguousarray(values, np.float64)
    out = np.zeros((h, w), np.uint8)
    _check(lib().p3s_gpu_upsample(_p(values, f64p), w, h, block, _p(out)))
    return out


def generate_depth(img, cfg: Config) -> np.ndarray:
    img, pl = _planes(img)
    out = np.zeros(img.shape[1:], np.uint8)
    _check(lib().p3s_gpu_generate_depth(*pl, img.shape[2], img.shape[1], cfg.h, _p(out)))
    return out


def cross_bilateral(depth, guide, cfg: Config) -> np.ndarray:
    depth = np.ascontiguousarray(depth, np.uint8)
    guide = np.ascontiguousarray(guide, np.uint8)
    out = np.zeros_like(depth)
    _check(lib().p3s_gpu_cross_bilateral(_p(depth), _p(guide), depth.shape[1], depth.shape[0],
                                         cfg.h, _p(out)))
    return out


def cross_bilateral_raw(depth, guide, cfg: Config) -> np.ndarray:
    depth = np.ascontiguousarray(depth, np.uint8)
    guide = np.ascontiguousarray(guide, np.uint8)
    out = np.zeros(depth.shape, np.float64)
    _check(lib().p3s_gpu_cross_bilateral_raw(_p(depth), _p(guide), depth.shape[1],
                                             depth.shape[0], cfg.h, _p(out, f64p)))
    return out


def reconstruct(img, depth, cfg: Config):
    img, pl = _planes(img)
    depth = np.ascontiguousarray(depth, np.uint8)
    _, h, w = img.shape
    left, right = np.zeros_like(img), np.zeros_like(img)
    lm, rm = np.zeros((h, w), np.uint8), np.zeros((h, w), np.uint8)
    _check(lib().p3s_gpu_reconstruct(*pl, _p(depth), w, h, cfg.h, *[_p(left[c]) for c in range(3)],
                                     *[_p(right[c]) for c in range(3)], _p(lm), _p(rm)))
    return left, right, lm, rm


def inpaint(img, mask, cfg: Config):
    img, pl = _planes(img)
    mask = np.ascontiguousarray(mask, np.uint8)
    _, h, w = img.shape
    out = np.zeros_like(img)
    st = np.zeros(3, np.int64)
    _check(lib().p3s_gpu_inpaint(*pl, _p(mask), w, h, cfg.h, *[_p(out[c]) for c in range(3)],
                                 _p(st, i64p)))
    return out, tuple(int(v) for v in st)


def anaglyph(left, right) -> np.ndarray:
    left, lp = _planes(left)
    right, rp = _planes(right)
    _, h, w = left.shape
    out = np.zeros_like(left)
    _check(lib().p3s_gpu_anaglyph(*lp, *rp, w, h, *[_p(out[c]) for c in range(3)]))
    return out


def side_by_side(left, right, half: bool) -> np.ndarray:
    left, lp = _planes(left)
    right, rp = _planes(right)
    _, h, w = left.shape
    out = np.zeros((3, h, w if half else 2 * w), np.uint8)
    _check(lib().p3s_gpu_side_by_side(*lp, *rp, w, h, int(bool(half)),
                                      *[_p(out[c]) for c in range(3)]))
    return out


# ---- device-resident pipeline / video --------------------------------------------------
class Pipeline:
    """p3s_pipeline: one (size, config) plan with its own stream; frames in device memory."""

    def __init__(self, w: int, h: int, cfg: Config):
        self.w, self.h = w, h
        self.cfg = cfg
        self.handle = vp()
        _check(lib().p3s_pipeline_create(w, h, cfg.h, C.byref(self.handle)))
        self.pitch = lib().p3s_pipeline_pitch(self.handle)
        self.frame_bytes = lib().p3s_pipeline_frame_bytes(self.handle)
        self.stream = lib().p3s_pipeline_stream(self.handle)

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.p3s_pipeline_free(self.handle)
            self.handle = None

    def upload(self, img: np.ndarray, d_dst: int, stream=None) -> None:
        img = np.ascontiguousarray(img, np.uint8)
        _check(lib().p3s_pipeline_upload(self.handle, img[0].ctypes.data, img[1].ctypes.data,
                                         img[2].ctypes.data, d_dst, stream))

    def run(self, d_src: int, timed: bool = False, stream=None) -> None:
        _check(lib().p3s_pipeline_run(self.handle, d_src, int(timed), stream))

    def timings(self) -> dict:
        t = Timings()
        _check(lib().p3s_pipeline_timings(self.handle, C.byref(t)))
        return t.as_dict()

    def timing_sum(self, reset: bool = True):
        """(per-stage ns summed over every timed run since the last reset, run count)."""
        t = Timings()
        n = C.c_int64()
        _check(lib().p3s_pipeline_timing_sum(self.handle, C.byref(t), C.byref(n), int(reset)))
        return t.as_dict(), n.value

    def download(self, fmt: int = ANAGLYPH):
        ow = 2 * self.w if fmt == FSBS else self.w
        depth = np.zeros((self.h, self.w), np.uint8)
        filt = np.zeros((self.h, self.w), np.uint8)
        out = np.zeros((3, self.h, ow), np.uint8)
        _check(lib().p3s_pipeline_download(self.handle, _p(depth), _p(filt), fmt,
                                           *[_p(out[c]) for c in range(3)]))
        return depth, filt, out

    def set_inpaint_ctas(self, ctas: int) -> None:
        """CTAs of the cooperative inpaint (0 = one per SM). Fewer suit several concurrent
        pipelines (aggregate throughput); a single stream wants all SMs (latency)."""
        _check(lib().p3s_pipeline_set_inpaint_ctas(self.handle, int(ctas)))

    def bilateral_kernel_sum(self, reset: bool = True):
        """(sum of the main bilateral kernel's ns, runs) over the timed runs (no fix-up)."""
        v, n = C.c_int64(), C.c_int64()
        _check(lib().p3s_pipeline_bilateral_kernel_sum(self.handle, C.byref(v), C.byref(n),
                                                       int(reset)))
        return v.value, n.value

    def inpaint_stats(self):
        st = np.zeros(6, np.int64)
        _check(lib().p3s_pipeline_inpaint_stats(self.handle, _p(st, i64p)))
        return st


class Video:
    """p3s_video: frames pipelined over `streams` plans (H2D / kernels / D2H overlap)."""

    def __init__(self, w: int, h: int, cfg: Config, streams: int = 3, devices=None):
        """devices: list of CUDA ordinals to shard frames over (frame i -> devices[i % n],
        one host thread per device); None = the current device only."""
        self.w, self.h = w, h
        self.handle = vp()
        if devices is None:
            _check(lib().p3s_video_create(w, h, cfg.h, streams, C.byref(self.handle)))
        else:
            arr = (C.c_int * len(devices))(*devices)
            _check(lib().p3s_video_create_devices(w, h, cfg.h, arr, len(devices), streams,
                                                  C.byref(self.handle)))

    @property
    def shards(self) -> int:
        return lib().p3s_video_shards(self.handle)

    @property
    def requeued(self) -> int:
        """Frames re-run on healthy devices after a device failed."""
        return lib().p3s_video_requeued(self.handle)

    @property
    def healthy_shards(self) -> int:
        return lib().p3s_video_healthy_shards(self.handle)

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.p3s_video_free(self.handle)
            self.handle = None

    def convert_ptrs(self, frame_ptrs, out_ptrs, interleaved: bool = False) -> None:
        """Planar frames (3 planes of w*h) or, with interleaved=True, RGB-interleaved
        payloads (w*h*3 bytes) in; the first requested format out in the same layout."""
        n = len(frame_ptrs)
        fa = (vp * n)(*frame_ptrs)
        oa = (vp * n)(*out_ptrs)
        fn = lib().p3s_video_convert_interleaved if interleaved else lib().p3s_video_convert
        _check(fn(self.handle, fa, n, oa))


class PinnedBuffer:
    """A pinned host allocation from the library's pool, viewed as a numpy array
    (near_device: pages placed on that GPU's NUMA node)."""

    def __init__(self, nbytes: int, near_device: int | None = None):
        if near_device is None:
            self.ptr = lib().p3s_host_alloc(nbytes)
        else:
            self.ptr = lib().p3s_host_alloc_near(near_device, nbytes)
        if not self.ptr:
            raise MemoryError("p3s_host_alloc")
        self.nbytes = nbytes
        self.array = np.ctypeslib.as_array(C.cast(self.ptr, u8p), shape=(nbytes,))

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.p3s_host_free(self.ptr)
            self.ptr = None


class DeviceBuffer:
    def __init__(self, nbytes: int):
        self.ptr = vp()
        _check(lib().p3s_gpu_malloc(nbytes, C.byref(self.ptr)))
        self.nbytes = nbytes

    @property
    def addr(self) -> int:
        return self.ptr.value

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.p3s_gpu_free(self.ptr)
            self.ptr = None


class Event:
    def __init__(self):
        self.h = vp()
        _check(lib().p3s_gpu_event_create(C.byref(self.h)))

    def record(self, stream=None) -> None:
        _check(lib().p3s_gpu_event_record(self.h, stream))

    def wait(self, stream) -> None:
        """Make `stream` wait for this event."""
        _check(lib().p3s_gpu_stream_wait_event(stream, self.h))

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float()
        _check(lib().p3s_gpu_event_elapsed_ms(self.h, end.h, C.byref(ms)))
        return ms.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.p3s_gpu_event_destroy(self.h)
            self.h = None


def fp64_peak() -> float:
    """Measured non-FMA FP64 issue rate of the current device, ops/s."""
    v = C.c_double()
    _check(lib().p3s_gpu_fp64_peak(C.byref(v)))
    return v.value


def synthetic_frame(w: int, h: int, seed: int = 1) -> np.ndarray:
    """The reference's seeded synthetic frame (bench.cpp:23-46) as (3, h, w) u8 planes,
    generated by the product library (host code)."""
    out = np.empty((3, h, w), np.uint8)
    _check(lib().p3s_synthetic_frame(w, h, seed, _p(out[0]), _p(out[1]), _p(out[2])))
    return out


def launch_count() -> int:
    """Kernels the library launched in this process (graph replays count their kernel
    nodes)."""
    return int(lib().p3s_gpu_launch_count())


def numa_node(device: int) -> int:
    return int(lib().p3s_gpu_numa_node(device))


def bilateral_fast_path(cfg) -> bool:
    """True when p3s_convert runs the certified FP32 bilateral (+ exact fix-up) for cfg."""
    v = C.c_int()
    _check(lib().p3s_gpu_bilateral_path(cfg.h, C.byref(v)))
    return bool(v.value)


def smem_peak(gather: bool = False) -> float:
    """Measured conflict-free shared-memory load bandwidth of the current device, B/s
    (gather=True: data-dependent per-lane gathers, the bilateral's lookup pattern)."""
    v = C.c_double()
    _check(lib().p3s_gpu_smem_peak(C.byref(v), 1 if gather else 0))
    return v.value


def stream_sync(stream) -> None:
    _check(lib().p3s_gpu_stream_sync(stream))


def device_sync() -> None:
    _check(lib().p3s_gpu_device_sync())
