"""ctypes mirror of include/aaa.h and the loader of the in-tree libaaa.so."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libaaa.so"

AAA_FLAG_TIMING, AAA_FLAG_NO_TILE_CULL, AAA_FLAG_FORCE_FALLBACK, AAA_FLAG_NO_HIER_SORT, AAA_FLAG_NO_3D = 1, 2, 4, 8, 16
AAA_FLAG_SAVE_CONTRIBS = 32
AAA_FLAG_FORCE_DEEP = 64
AAA_FLAG_CULL_FP64 = 128
AAA_FLAG_FORCE_GIANT = 256
AAA_FLAG_NO_GSUB = 512
AAA_WARN_UNRESOLVED = 1  # aaa_get_stats / aaa_synchronize: pixels left inexact (spill queue full)
(AAA_DBG_GAUSS, AAA_DBG_KEYS, AAA_DBG_VALS, AAA_DBG_KEYS_UNSORTED, AAA_DBG_VALS_UNSORTED, AAA_DBG_RANGES,
 AAA_DBG_SPILL, AAA_DBG_RASTER, AAA_DBG_COLOR) = range(9)
AAA_DBG_GAUSS_FIELDS = 26

EXPORTED_SYMBOLS = ["aaa_version", "aaa_create", "aaa_destroy", "aaa_set_stream", "aaa_default_config",
                    "aaa_set_config", "aaa_load_gaussians", "aaa_set_camera", "aaa_render", "aaa_render_batch",
                    "aaa_render_tiles", "aaa_tile_row_costs", "aaa_get_stats", "aaa_synchronize",
                    "aaa_debug_copy", "aaa_last_error", "aaa_compute_vtrain", "aaa_render_backward",
                    "aaa_render_band"]


class AaaError(RuntimeError):
    def __init__(self, status, msg, first_bad=None):
        super().__init__(msg)
        self.status = status
        self.first_bad = first_bad


class Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("world_to_view", C.c_float * 16), ("near_z", C.c_float)]


class Config(C.Structure):
    _fields_ = [("k", C.c_float), ("tau_mode", C.c_int32), ("tau_fixed", C.c_float), ("alpha_max", C.c_float),
                ("T_eps", C.c_float), ("background", C.c_float * 3), ("window_k", C.c_int32),
                ("flags", C.c_uint32)]


class Gaussians(C.Structure):
    _fields_ = [("means", C.POINTER(C.c_float)), ("scales", C.POINTER(C.c_float)),
                ("quats", C.POINTER(C.c_float)), ("opacities", C.POINTER(C.c_float)),
                ("sh", C.POINTER(C.c_float)), ("v_train", C.POINTER(C.c_float)), ("n", C.c_int64),
                ("sh_degree", C.c_int32), ("device_ptrs", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("n", C.c_int64), ("visible", C.c_int64), ("candidates", C.c_int64), ("pairs", C.c_int64),
                ("spilled_pixels", C.c_int64), ("unresolved_pixels", C.c_int64), ("crossing", C.c_int64), ("evaluations", C.c_int64),
                ("launches", C.c_int64), ("timed_views", C.c_int64), ("ms", C.c_float * 10),
                ("deep_pixels", C.c_int64), ("giant_pixels", C.c_int64)]


_lib = None


def lib(path: Path | None = None):
    """Load libaaa.so (fails loudly if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        p = Path(path) if path else _LIB_PATH
        if not p.exists():
            raise RuntimeError(f"{p} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(str(p))
        V, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
        L.aaa_version.restype = I32
        L.aaa_create.argtypes = [I32, V, C.POINTER(V)]
        L.aaa_destroy.argtypes = [V]
        L.aaa_destroy.restype = None
        L.aaa_set_stream.argtypes = [V, V]
        L.aaa_default_config.argtypes = [C.POINTER(Config)]
        L.aaa_set_config.argtypes = [V, C.POINTER(Config)]
        L.aaa_load_gaussians.argtypes = [V, C.POINTER(Gaussians), C.POINTER(I64)]
        L.aaa_set_camera.argtypes = [V, C.POINTER(Camera)]
        L.aaa_render.argtypes = [V, V, V]
        L.aaa_render_batch.argtypes = [V, C.POINTER(Camera), I32, V, V]
        L.aaa_render_tiles.argtypes = [V, I32, I32, V, V]
        L.aaa_tile_row_costs.argtypes = [V, C.POINTER(I64), I32]
        L.aaa_render_band.argtypes = [V, I32, I32, V, V, C.POINTER(I32)]
        L.aaa_get_stats.argtypes = [V, C.POINTER(Stats)]
        L.aaa_synchronize.argtypes = [V]
        L.aaa_debug_copy.argtypes = [V, I32, V, C.c_size_t, C.POINTER(C.c_size_t)]
        L.aaa_compute_vtrain.argtypes = [V, C.POINTER(Camera), I32, V, I32]
        L.aaa_render_backward.argtypes = [V, V, V, V, V, V, V, V]
        L.aaa_last_error.argtypes = [V]
        L.aaa_last_error.restype = C.c_char_p
        for f in EXPORTED_SYMBOLS:
            if f not in ("aaa_version", "aaa_destroy", "aaa_last_error"):
                getattr(L, f).restype = I32
        _lib = L
    return _lib
