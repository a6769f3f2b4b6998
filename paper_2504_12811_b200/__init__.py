"""B200-native forward renderer of AAA-Gaussians (arxiv 2504.12811).

Thin ctypes binding over the in-tree C-ABI library ``libaaa.so`` (include/aaa.h). The
binding only marshals arguments: every step of the render runs in the library's sm_100a
kernels. There is no CPU fallback — importing the binding on a box without the built
library, or calling it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from ._abi import (AAA_DBG_GAUSS, AAA_DBG_GAUSS_FIELDS, AAA_DBG_KEYS, AAA_DBG_KEYS_UNSORTED, AAA_DBG_SPILL,
                   AAA_DBG_RANGES, AAA_DBG_VALS, AAA_DBG_VALS_UNSORTED, AAA_FLAG_CULL_FP64, AAA_FLAG_FORCE_DEEP, AAA_FLAG_FORCE_GIANT, AAA_FLAG_FORCE_FALLBACK, AAA_FLAG_NO_GSUB,
                   AAA_FLAG_NO_3D, AAA_FLAG_NO_HIER_SORT, AAA_FLAG_NO_TILE_CULL, AAA_FLAG_SAVE_CONTRIBS, AAA_FLAG_TIMING, AAA_WARN_UNRESOLVED, AaaError, Camera, Config, Gaussians, Stats, lib,
                   EXPORTED_SYMBOLS)

__all__ = ["Renderer", "lib", "Camera", "Config", "Gaussians", "Stats", "AaaError", "camera_struct",
           "EXPORTED_SYMBOLS", "DBG_FIELDS"]

DBG_FIELDS = ["vhat", "veff", "shat0", "shat1", "shat2", "A", "oA", "tau", "valid", "inside", "inside_rho2",
              "r", "g", "b", "visible", "crossing", "tx0", "ty0", "tx1", "ty1", "zkey", "xlo", "xhi", "ylo",
              "yhi", "zlb"]


def camera_struct(cam) -> Camera:
    """synth.scenes.Camera (or any object with the same fields) -> aaa_camera."""
    c = Camera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    M = np.asarray(cam.world_to_view, dtype=np.float64).reshape(16)
    for i in range(16):
        c.world_to_view[i] = float(M[i])
    c.near_z = float(cam.near)
    return c


def _check(ctx, status, what):
    if status == AAA_WARN_UNRESOLVED:
        import warnings
        warnings.warn(f"{what}: " + (lib().aaa_last_error(ctx).decode() if ctx else "pixels unresolved"))
        return
    if status != 0:
        msg = lib().aaa_last_error(ctx).decode() if ctx else ""
        raise AaaError(status, f"{what}: status {status}: {msg}")


class Renderer:
    """One aaa_ctx on one CUDA device, driven from torch tensors or host numpy arrays."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2504_12811_b200 needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = device
        self._ctx = C.c_void_p()
        s = stream if stream is not None else torch.cuda.current_stream(device).cuda_stream
        _check(None, lib().aaa_create(device, C.c_void_p(s), C.byref(self._ctx)), "aaa_create")
        self.cfg = Config()
        lib().aaa_default_config(C.byref(self.cfg))
        self.width = self.height = None

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            lib().aaa_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- configuration
    def set_stream(self, stream_handle: int):
        _check(self._ctx, lib().aaa_set_stream(self._ctx, C.c_void_p(stream_handle)), "aaa_set_stream")

    def set_config(self, **kw):
        for k, v in kw.items():
            if k == "background":
                for i in range(3):
                    self.cfg.background[i] = float(v[i])
            else:
                setattr(self.cfg, k, v)
        _check(self._ctx, lib().aaa_set_config(self._ctx, C.byref(self.cfg)), "aaa_set_config")

    # ---- scene
    def load(self, scene=None, *, tensors=None) -> None:
        """Load a synth.scenes.Scene (host numpy) or a dict of CUDA tensors."""
        g = Gaussians()
        keep = []
        if tensors is not None:
            t = tensors
            for name in ("means", "scales", "quats", "opacities", "sh", "v_train"):
                a = t[name].contiguous().float()
                keep.append(a)
                setattr(g, name, C.cast(C.c_void_p(a.data_ptr()), C.POINTER(C.c_float)))
            g.n = int(t["means"].shape[0])
            g.sh_degree = int(t["sh_degree"])
            g.device_ptrs = 1
        else:
            for name in ("means", "scales", "quats", "opacities", "sh", "v_train"):
                a = np.ascontiguousarray(getattr(scene, name), dtype=np.float32)
                keep.append(a)
                setattr(g, name, a.ctypes.data_as(C.POINTER(C.c_float)))
            g.n = scene.n
            g.sh_degree = scene.sh_degree
            g.device_ptrs = 0
        bad = C.c_int64(-1)
        st = lib().aaa_load_gaussians(self._ctx, C.byref(g), C.byref(bad))
        if st != 0:
            raise AaaError(st, f"aaa_load_gaussians: first bad Gaussian {bad.value}: "
                               f"{lib().aaa_last_error(self._ctx).decode()}", first_bad=bad.value)
        self.n = g.n
        self.sh_degree = int(g.sh_degree)

    def set_camera(self, cam) -> None:
        c = camera_struct(cam)
        _check(self._ctx, lib().aaa_set_camera(self._ctx, C.byref(c)), "aaa_set_camera")
        self.width, self.height = c.width, c.height

    # ---- rendering
    def render(self, cam=None, out_rgb=None, out_T=None, with_T: bool = True):
        """Render into CUDA tensors (allocated if not given). Returns (rgb[3,H,W], T[H,W])."""
        torch = self.torch
        if cam is not None:
            self.set_camera(cam)
        H, W = self.height, self.width
        dev = torch.device("cuda", self.device)
        if out_rgb is None:
            out_rgb = torch.empty((3, H, W), dtype=torch.float32, device=dev)
        if out_T is None and with_T:
            out_T = torch.empty((H, W), dtype=torch.float32, device=dev)
        tp = C.c_void_p(out_T.data_ptr()) if out_T is not None else C.c_void_p()
        _check(self._ctx, lib().aaa_render(self._ctx, C.c_void_p(out_rgb.data_ptr()), tp), "aaa_render")
        return out_rgb, out_T

    def render_host(self, cam, rgb: np.ndarray, T: np.ndarray | None = None):
        """Render into host arrays (pinned or pageable); the library copies back."""
        self.set_camera(cam)
        tp = C.c_void_p(T.ctypes.data) if T is not None else C.c_void_p()
        _check(self._ctx, lib().aaa_render(self._ctx, C.c_void_p(rgb.ctypes.data), tp), "aaa_render")
        return rgb, T

    def render_batch(self, cams, out_rgb=None, out_T=None, with_T: bool = False, host_ptrs=None):
        """Render a list of cameras. With host_ptrs=(rgb_ptr, T_ptr) the outputs are host memory."""
        torch = self.torch
        n = len(cams)
        arr = (Camera * n)(*[camera_struct(c) for c in cams])
        H, W = arr[0].height, arr[0].width
        if host_ptrs is not None:
            r, t = host_ptrs
            _check(self._ctx, lib().aaa_render_batch(self._ctx, arr, n, C.c_void_p(r), C.c_void_p(t or 0)),
                   "aaa_render_batch")
            return None
        dev = torch.device("cuda", self.device)
        if out_rgb is None:
            out_rgb = torch.empty((n, 3, H, W), dtype=torch.float32, device=dev)
        if out_T is None and with_T:
            out_T = torch.empty((n, H, W), dtype=torch.float32, device=dev)
        tp = C.c_void_p(out_T.data_ptr()) if out_T is not None else C.c_void_p()
        _check(self._ctx, lib().aaa_render_batch(self._ctx, arr, n, C.c_void_p(out_rgb.data_ptr()), tp),
               "aaa_render_batch")
        self.width, self.height = W, H
        return out_rgb, out_T

    def compute_vtrain(self, cams, out=None, store: bool = False):
        """v_hat_train of every loaded Gaussian over the training cameras (Eq. 6, aaa_compute_vtrain).
        Returns a float32 CUDA tensor (or fills `out`); store=True also makes later renders use it."""
        torch = self.torch
        n = len(cams)
        arr = (Camera * max(n, 1))(*[camera_struct(c) for c in cams])
        if out is None:
            out = torch.empty((self.n,), dtype=torch.float32, device=torch.device("cuda", self.device))
        _check(self._ctx, lib().aaa_compute_vtrain(self._ctx, arr, n, C.c_void_p(out.data_ptr()), 1 if store else 0),
               "aaa_compute_vtrain")
        return out

    def backward(self, dL_drgb, dL_dT=None):
        """Gradients of a scalar loss through the last render made with AAA_FLAG_SAVE_CONTRIBS
        (aaa_render_backward). Returns dict of CUDA tensors: means, scales, quats, opacities, sh."""
        torch = self.torch
        dev = torch.device("cuda", self.device)
        dL_drgb = dL_drgb.contiguous().float()
        dT = dL_dT.contiguous().float() if dL_dT is not None else None
        K = (self.sh_degree + 1) ** 2
        out = dict(means=torch.empty((self.n, 3), device=dev), scales=torch.empty((self.n, 3), device=dev),
                   quats=torch.empty((self.n, 4), device=dev), opacities=torch.empty((self.n,), device=dev),
                   sh=torch.empty((self.n, K, 3), device=dev))
        p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p()
        _check(self._ctx, lib().aaa_render_backward(self._ctx, p(dL_drgb), p(dT), p(out["means"]), p(out["scales"]),
                                                    p(out["quats"]), p(out["opacities"]), p(out["sh"])),
               "aaa_render_backward")
        return out

    def render_tiles(self, row_begin: int, row_end: int, out_rgb=None, out_T=None):
        torch = self.torch
        H, W = self.height, self.width
        band_h = min(16 * row_end, H) - 16 * row_begin
        dev = torch.device("cuda", self.device)
        if out_rgb is None:
            out_rgb = torch.empty((3, band_h, W), dtype=torch.float32, device=dev)
        tp = C.c_void_p(out_T.data_ptr()) if out_T is not None else C.c_void_p()
        _check(self._ctx, lib().aaa_render_tiles(self._ctx, row_begin, row_end, C.c_void_p(out_rgb.data_ptr()), tp),
               "aaa_render_tiles")
        return out_rgb, out_T

    def render_band(self, rank: int, world: int, out_rgb=None, out_T=None):
        """This rank's tile-row band of the current camera's frame split over `world` ranks
        (aaa_render_band). Returns (rgb[3, band_h, W] view into out_rgb, T or None, cuts[world+1])."""
        torch = self.torch
        H, W = self.height, self.width
        dev = torch.device("cuda", self.device)
        if out_rgb is None:
            out_rgb = torch.empty((3 * H * W,), dtype=torch.float32, device=dev)
        cuts = np.zeros(world + 1, dtype=np.int32)
        tp = C.c_void_p(out_T.data_ptr()) if out_T is not None else C.c_void_p()
        _check(self._ctx, lib().aaa_render_band(self._ctx, int(rank), int(world), C.c_void_p(out_rgb.data_ptr()), tp,
                                                cuts.ctypes.data_as(C.POINTER(C.c_int32))), "aaa_render_band")
        a, b = int(cuts[rank]), int(cuts[rank + 1])
        bh = min(16 * b, H) - 16 * a
        rgb = out_rgb.reshape(-1)[: 3 * bh * W].view(3, bh, W)
        T = out_T.reshape(-1)[: bh * W].view(bh, W) if out_T is not None else None
        return rgb, T, cuts

    def tile_row_costs(self) -> np.ndarray:
        rows = (self.height + 15) // 16
        out = np.zeros(rows, dtype=np.int64)
        _check(self._ctx, lib().aaa_tile_row_costs(self._ctx, out.ctypes.data_as(C.POINTER(C.c_int64)), rows),
               "aaa_tile_row_costs")
        return out

    def synchronize(self):
        _check(self._ctx, lib().aaa_synchronize(self._ctx), "aaa_synchronize")

    def stats(self) -> dict:
        s = Stats()
        _check(self._ctx, lib().aaa_get_stats(self._ctx, C.byref(s)), "aaa_get_stats")
        d = {f: getattr(s, f) for f, _ in Stats._fields_ if f != "ms"}
        d["ms"] = list(s.ms)
        return d

    def debug_copy(self, what: int, dtype, cols: int = 1) -> np.ndarray:
        ln = C.c_size_t(0)
        cap = 1 << 20
        while True:
            buf = np.empty(cap, dtype=np.uint8)
            st = lib().aaa_debug_copy(self._ctx, what, C.c_void_p(buf.ctypes.data), cap, C.byref(ln))
            if st == 0:
                break
            if ln.value > cap:
                cap = ln.value
                continue
            _check(self._ctx, st, "aaa_debug_copy")
        a = buf[: ln.value].view(dtype)
        return a.reshape(-1, cols) if cols > 1 else a

    def gaussian_records(self) -> np.ndarray:
        return self.debug_copy(AAA_DBG_GAUSS, np.float64, AAA_DBG_GAUSS_FIELDS)

    def keys_vals(self, sorted_: bool = True):
        if sorted_:
            return self.debug_copy(AAA_DBG_KEYS, np.uint32), self.debug_copy(AAA_DBG_VALS, np.uint32)
        k = self.debug_copy(AAA_DBG_KEYS_UNSORTED, np.uint32)
        v = self.debug_copy(AAA_DBG_VALS_UNSORTED, np.uint32)
        return k, v

    def key_tile_shift(self) -> int:
        """Bits of the depth code in a sort key (key >> this = tile id)."""
        n_tiles = ((self.width + 15) // 16) * ((self.height + 15) // 16)
        return min(32 - n_tiles.bit_length(), 28)  # tile ids < 2^tile_bits - 1 (aaa_internal.cuh SKEY_NONE)

    def spilled_pixels(self) -> np.ndarray:
        """Linear indices (y * W + x) of the pixels of the last render continued by K6s (debug)."""
        return self.debug_copy(AAA_DBG_SPILL, np.uint32, 8)[:, 0].copy()

    def ranges(self) -> np.ndarray:
        return self.debug_copy(AAA_DBG_RANGES, np.uint32, 2)
