"""ctypes wrapper of the float64 CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: only tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this package.
It shares no code with the CUDA path (``paper_2504_12811_b200``) and never
imports it; the only module both sides consume is ``synth.scenes`` (inputs).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "liboracle.so"

G_FIELDS = ["vhat", "veff", "shat0", "shat1", "shat2", "A", "oA", "tau", "valid", "inside",
            "inside_rho2", "r", "g", "b", "muv0", "muv1", "muv2"]
C_FIELDS = ["z", "alpha", "rho2", "tau", "g", "r", "gg", "b", "included", "flags"]
F_CUTOFF, F_NEAR, F_TIE, F_GAUSS, F_TERMINATED = 1, 2, 4, 8, 16


def build(force: bool = False) -> Path:
    """Compile liboracle.so (portable x86-64, no -march=native so it runs on any host)."""
    src = _HERE / "oracle.cpp"
    if force or not _SO.exists() or _SO.stat().st_mtime < max(src.stat().st_mtime,
                                                             (_HERE / "oracle.h").stat().st_mtime):
        cmd = ["g++", "-O3", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", "-o", str(_SO), str(src)]
        subprocess.run(cmd, check=True)
    return _SO


class _Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("world_to_view", C.c_double * 16),
                ("near_z", C.c_double)]


class _Config(C.Structure):
    _fields_ = [("k", C.c_double), ("tau_mode", C.c_int32), ("tau_fixed", C.c_double),
                ("alpha_max", C.c_double), ("T_eps", C.c_double), ("bg", C.c_double * 3),
                ("band_rho", C.c_double), ("band_near", C.c_double), ("band_tie", C.c_double),
                ("band_gauss", C.c_double), ("order_mode", C.c_int32), ("order_scale", C.c_double),
                ("order_near", C.c_double), ("order_qmax", C.c_double), ("eval_mode", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            build()
        L = C.CDLL(str(_SO))
        P = C.c_void_p
        L.orc_create.restype = P
        L.orc_create.argtypes = [C.c_int64, C.c_int32] + [P] * 6
        L.orc_destroy.argtypes = [P]
        L.orc_num_threads.restype = C.c_int32
        L.orc_set_view.argtypes = [P, C.POINTER(_Camera), C.POINTER(_Config)]
        L.orc_gaussians.argtypes = [P, P]
        L.orc_render_pixels.argtypes = [P, C.c_int64, P, P, C.c_int32, P, P, P]
        L.orc_pixel_contribs.restype = C.c_int64
        L.orc_pixel_contribs.argtypes = [P, C.c_int32, C.c_int32, P, C.c_int64]
        L.orc_frustum_min_rho2.argtypes = [P, C.c_int64, P, P, P]
        L.orc_sh_basis.argtypes = [P, P]
        L.orc_qp_min_norm.restype = C.c_double
        L.orc_qp_min_norm.argtypes = [C.c_int32, P, P]
        L.orc_vtrain.argtypes = [P, C.c_int32, C.POINTER(_Camera), P, P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def default_config(**kw) -> dict:
    cfg = dict(k=0.3, tau_mode=0, tau_fixed=9.0, alpha_max=0.99, T_eps=1e-4, bg=(0.0, 0.0, 0.0),
               band_rho=4e-3, band_near=1e-5, band_tie=4e-6, band_gauss=1e-5,
               order_mode=0, order_scale=1.0, order_near=1.0, order_qmax=0.0, eval_mode=0)
    cfg.update(kw)
    return cfg


class Oracle:
    """Holds a float64 copy of a scene; ``set_view`` runs the per-Gaussian stage."""

    def __init__(self, scene):
        self.scene = scene
        self._arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in
                      (scene.means, scene.scales, scene.quats, scene.opacities, scene.sh, scene.v_train)]
        self.n = scene.n
        self._h = lib().orc_create(self.n, scene.sh_degree, *[_ptr(a) for a in self._arrs])
        self.cam = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_destroy(h)
            self._h = None

    def set_view(self, cam, **cfg):
        # the C-ABI camera is float32; the oracle takes the same float32 values, promoted exactly
        f32 = lambda v: float(np.float32(v))
        c = _Camera()
        c.width, c.height = int(cam.width), int(cam.height)
        c.fx, c.fy, c.cx, c.cy = f32(cam.fx), f32(cam.fy), f32(cam.cx), f32(cam.cy)
        c.world_to_view[:] = [f32(v) for v in np.asarray(cam.world_to_view, dtype=np.float64).reshape(16)]
        c.near_z = f32(cam.near)
        d = default_config(**cfg)
        k = _Config()
        for f, _ in _Config._fields_:
            if f == "bg":
                k.bg[:] = list(d["bg"])
            else:
                setattr(k, f, d[f])
        self._cam_struct, self._cfg_struct = c, k
        self.cam, self.cfg = cam, d
        rc = lib().orc_set_view(self._h, C.byref(c), C.byref(k))
        assert rc == 0
        return self

    def vtrain(self, cams):
        """v_hat_train over cameras (Eq. 6): (values float64, boundary-ambiguity flags)."""
        f32 = lambda v: float(np.float32(v))
        arr = (_Camera * max(len(cams), 1))()
        for i, cam in enumerate(cams):
            c = arr[i]
            c.width, c.height = int(cam.width), int(cam.height)
            c.fx, c.fy, c.cx, c.cy = f32(cam.fx), f32(cam.fy), f32(cam.cx), f32(cam.cy)
            c.world_to_view[:] = [f32(v) for v in np.asarray(cam.world_to_view, dtype=np.float64).reshape(16)]
            c.near_z = f32(cam.near)
        out = np.empty(self.n, dtype=np.float64)
        amb = np.empty(self.n, dtype=np.int32)
        assert lib().orc_vtrain(self._h, len(cams), arr, _ptr(out), _ptr(amb)) == 0
        return out, amb.astype(bool)

    def gaussians(self) -> np.ndarray:
        out = np.empty((self.n, len(G_FIELDS)), dtype=np.float64)
        assert lib().orc_gaussians(self._h, _ptr(out)) == 0
        return out

    def render_pixels(self, px, py, use_rejects: bool = True):
        px = np.ascontiguousarray(px, dtype=np.int32)
        py = np.ascontiguousarray(py, dtype=np.int32)
        n = px.shape[0]
        rgbT = np.empty((n, 4), dtype=np.float64)
        flags = np.empty(n, dtype=np.uint32)
        nb = np.empty(n, dtype=np.int32)
        rc = lib().orc_render_pixels(self._h, n, _ptr(px), _ptr(py), int(use_rejects), _ptr(rgbT),
                                     _ptr(flags), _ptr(nb))
        assert rc == 0
        return rgbT, flags, nb

    def render_image(self, use_rejects: bool = True):
        W, H = self.cam.width, self.cam.height
        yy, xx = np.mgrid[0:H, 0:W]
        rgbT, flags, nb = self.render_pixels(xx.ravel(), yy.ravel(), use_rejects)
        return rgbT.reshape(H, W, 4), flags.reshape(H, W), nb.reshape(H, W)

    def pixel_contribs(self, px: int, py: int) -> np.ndarray:
        cap = 4096
        while True:
            out = np.empty((cap, len(C_FIELDS)), dtype=np.float64)
            m = lib().orc_pixel_contribs(self._h, int(px), int(py), _ptr(out), cap)
            if m <= cap:
                return out[:m]
            cap = int(m)

    def frustum_min_rho2(self, g, rects) -> np.ndarray:
        g = np.ascontiguousarray(g, dtype=np.int64)
        rects = np.ascontiguousarray(rects, dtype=np.float64).reshape(-1, 4)
        out = np.empty(g.shape[0], dtype=np.float64)
        assert lib().orc_frustum_min_rho2(self._h, g.shape[0], _ptr(g), _ptr(rects), _ptr(out)) == 0
        return out


def sh_basis(d) -> np.ndarray:
    d = np.ascontiguousarray(d, dtype=np.float64)
    out = np.empty(16, dtype=np.float64)
    lib().orc_sh_basis(_ptr(d), _ptr(out))
    return out


def qp_min_norm(a, b) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return float(lib().orc_qp_min_norm(a.shape[0], _ptr(a), _ptr(b)))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def blend_variant(contribs: np.ndarray, included: np.ndarray, order: np.ndarray, cfg: dict):
    """Re-blend a (possibly flipped/swapped) contribution list — comparator helper
    (SURVEY 8c 'Comparator'); same rule as the oracle's blend (reading 3)."""
    C = np.zeros(3)
    T = 1.0
    for i in order:
        if not included[i]:
            continue
        a = contribs[i, 1]
        tT = T * (1.0 - a)
        if tT < cfg["T_eps"]:
            break
        C += a * contribs[i, 5:8] * T
        T = tT
    return np.concatenate([C + T * np.asarray(cfg["bg"]), [T]])
