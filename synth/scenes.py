"""Seeded synthetic inputs for the five BASELINE.json configs (c1..c5).

This module is shared by the tests, ``bench.py`` and the oracle harness. It
holds NONE of the method's arithmetic (no filter, no bounding, no culling, no
evaluation, no blending): it only draws Gaussians and cameras with the shapes
and statistics SURVEY.md §8(d) specifies, so both the CUDA path and the oracle
(`oracle/`) consume identical bytes.

The one derived input is ``v_train`` (the stored max training sampling
frequency, PAPER.md P:247 / Eq. 6 at P:151). It is a per-Gaussian INPUT to the
renderer; the generator synthesises it as the max over the
config's nominal camera set of f / z for cameras whose image contains the mean
(SPEC S:154), exactly like a training run would have stored it.

Conventions: view space +z forward, y down, pixel centres at
+0.5; ``world_to_view`` is a 4x4 row-major rigid transform; quaternions are
(w, x, y, z).
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
import os
from pathlib import Path

import numpy as np

__all__ = [
    "Scene", "Camera", "make_config", "quat_to_rotmat", "rotmat_to_quat",
    "look_at", "c1_scene", "c2_scene", "c3_scene", "c2_cameras", "c3_cameras",
    "c4_cameras", "c5_camera", "random_box_scene", "CONFIGS",
]


@dataclasses.dataclass
class Camera:
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    world_to_view: np.ndarray  # (4,4) float64, row-major rigid transform
    near: float = 0.01

    def scaled(self, **kw) -> "Camera":
        d = dataclasses.asdict(self)
        d.update(kw)
        d["world_to_view"] = np.array(d["world_to_view"], dtype=np.float64)
        return Camera(**d)


@dataclasses.dataclass
class Scene:
    means: np.ndarray      # (N,3) f32 world units
    scales: np.ndarray     # (N,3) f32 standard deviations, > 0
    quats: np.ndarray      # (N,4) f32 (w,x,y,z), not necessarily normalised
    opacities: np.ndarray  # (N,)  f32 in (0,1)
    sh: np.ndarray         # (N,(deg+1)^2,3) f32, coefficient-major, channel-minor
    v_train: np.ndarray    # (N,)  f32, +inf allowed
    sh_degree: int

    @property
    def n(self) -> int:
        return int(self.means.shape[0])

    def subset(self, idx) -> "Scene":
        return Scene(self.means[idx], self.scales[idx], self.quats[idx],
                     self.opacities[idx], self.sh[idx], self.v_train[idx],
                     self.sh_degree)


# --------------------------------------------------------------------------
# small geometric helpers (input construction only)
# --------------------------------------------------------------------------
def quat_to_rotmat(q: np.ndarray) -> np.ndarray:
    """Hamilton (w,x,y,z) quaternion(s) -> rotation matrix."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - w * z)
    R[..., 0, 2] = 2 * (x * z + w * y)
    R[..., 1, 0] = 2 * (x * y + w * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - w * x)
    R[..., 2, 0] = 2 * (x * z - w * y)
    R[..., 2, 1] = 2 * (y * z + w * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def rotmat_to_quat(R: np.ndarray) -> np.ndarray:
    """Rotation matrices (...,3,3) -> (w,x,y,z) quaternions (Shepperd's method)."""
    R = np.asarray(R, dtype=np.float64)
    shp = R.shape[:-2]
    R = R.reshape(-1, 3, 3)
    q = np.empty((R.shape[0], 4))
    tr = R[:, 0, 0] + R[:, 1, 1] + R[:, 2, 2]
    cand = np.stack([tr, R[:, 0, 0], R[:, 1, 1], R[:, 2, 2]], axis=1)
    k = np.argmax(cand, axis=1)
    for case in range(4):
        m = k == case
        if not np.any(m):
            continue
        Rm = R[m]
        if case == 0:
            s = np.sqrt(1.0 + tr[m]) * 2
            q[m, 0] = 0.25 * s
            q[m, 1] = (Rm[:, 2, 1] - Rm[:, 1, 2]) / s
            q[m, 2] = (Rm[:, 0, 2] - Rm[:, 2, 0]) / s
            q[m, 3] = (Rm[:, 1, 0] - Rm[:, 0, 1]) / s
        elif case == 1:
            s = np.sqrt(1.0 + Rm[:, 0, 0] - Rm[:, 1, 1] - Rm[:, 2, 2]) * 2
            q[m, 0] = (Rm[:, 2, 1] - Rm[:, 1, 2]) / s
            q[m, 1] = 0.25 * s
            q[m, 2] = (Rm[:, 0, 1] + Rm[:, 1, 0]) / s
            q[m, 3] = (Rm[:, 0, 2] + Rm[:, 2, 0]) / s
        elif case == 2:
            s = np.sqrt(1.0 + Rm[:, 1, 1] - Rm[:, 0, 0] - Rm[:, 2, 2]) * 2
            q[m, 0] = (Rm[:, 0, 2] - Rm[:, 2, 0]) / s
            q[m, 1] = (Rm[:, 0, 1] + Rm[:, 1, 0]) / s
            q[m, 2] = 0.25 * s
            q[m, 3] = (Rm[:, 1, 2] + Rm[:, 2, 1]) / s
        else:
            s = np.sqrt(1.0 + Rm[:, 2, 2] - Rm[:, 0, 0] - Rm[:, 1, 1]) * 2
            q[m, 0] = (Rm[:, 1, 0] - Rm[:, 0, 1]) / s
            q[m, 1] = (Rm[:, 0, 2] + Rm[:, 2, 0]) / s
            q[m, 2] = (Rm[:, 1, 2] + Rm[:, 2, 1]) / s
            q[m, 3] = 0.25 * s
    return q.reshape(shp + (4,))


def look_at(eye, target, world_up=(0.0, 0.0, 1.0)) -> np.ndarray:
    """World->view 4x4 for an OpenCV-style camera (+z forward, y down)."""
    eye = np.asarray(eye, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - eye
    f /= np.linalg.norm(f)
    up = np.asarray(world_up, dtype=np.float64)
    r = np.cross(f, up)
    if np.linalg.norm(r) < 1e-9:          # looking straight up/down
        r = np.cross(f, np.array([0.0, 1.0, 0.0]))
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    M = np.eye(4)
    M[0, :3], M[1, :3], M[2, :3] = r, d, f
    M[:3, 3] = -M[:3, :3] @ eye
    return M


def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _tangent_frames(rng, normals):
    """Random tangent frame (t1, t2, n) per normal; returns rotation matrices
    whose third column is the normal, so local axis 3 (the thin one) lies along n."""
    n = _unit(normals)
    a = rng.standard_normal(n.shape)
    t1 = _unit(a - np.sum(a * n, axis=1, keepdims=True) * n)
    t2 = np.cross(n, t1)
    return np.stack([t1, t2, n], axis=2)


def _sh_coeffs(rng, n, deg):
    """dc ~ N(0, 0.6^2); band l>0 ~ N(0, 0.05^2) * 0.7^l."""
    K = (deg + 1) ** 2
    sh = np.empty((n, K, 3), dtype=np.float32)
    sh[:, 0, :] = rng.normal(0.0, 0.6, (n, 3))
    for l in range(1, deg + 1):
        sl = slice(l * l, (l + 1) * (l + 1))
        sh[:, sl, :] = rng.normal(0.0, 0.05 * 0.7 ** l, (n, 2 * l + 1, 3))
    return sh


def _bimodal_opacity(rng, n):
    """60% U[0.7,1.0) and 40% U[0.02,0.5)."""
    hi = rng.random(n) < 0.6
    o = np.where(hi, rng.uniform(0.7, 1.0, n), rng.uniform(0.02, 0.5, n))
    return np.clip(o, 0.02, 0.999).astype(np.float32)


def v_train_from_cameras(means: np.ndarray, cams) -> np.ndarray:
    """Synthesised stored training frequency: max over cameras whose image
    contains the mean of f/z, f = max(fx, fy); +inf if
    no camera sees it. Input synthesis, not a hot-path step."""
    mu = means.astype(np.float64)
    vt = np.full(mu.shape[0], -np.inf)
    for cam in cams:
        V = cam.world_to_view
        z = mu @ V[2, :3] + V[2, 3]
        x = mu @ V[0, :3] + V[0, 3]
        y = mu @ V[1, :3] + V[1, 3]
        ok = z > cam.near
        zs = np.where(ok, z, 1.0)
        px = cam.fx * x / zs + cam.cx
        py = cam.fy * y / zs + cam.cy
        ok &= (px >= 0) & (px <= cam.width) & (py >= 0) & (py <= cam.height)
        f = max(cam.fx, cam.fy)
        vt = np.where(ok, np.maximum(vt, f / zs), vt)
    vt[~np.isfinite(vt)] = np.inf
    return vt.astype(np.float32)


# --------------------------------------------------------------------------
# c1: 64 Gaussians, 64x64, SH0 (+ 4 adversarial Gaussians)
# --------------------------------------------------------------------------
def c1_camera() -> Camera:
    return Camera(64, 64, 56.0, 56.0, 32.0, 32.0, np.eye(4), 0.01)


def c1_scene(seed: int = 7) -> Scene:
    rng = np.random.Generator(np.random.PCG64(seed))
    n = 60
    means = np.column_stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n),
                             rng.uniform(1.5, 4.0, n)])
    scales = np.exp(rng.uniform(np.log(0.03), np.log(0.6), (n, 3)))
    quats = rng.standard_normal((n, 4))
    opac = rng.uniform(0.2, 0.95, n)
    # four adversarial Gaussians
    def q_axis(axis):  # rotation taking local x to `axis` (keeps y in x-z plane)
        a = _unit(np.asarray(axis, dtype=np.float64))
        b = _unit(np.cross(a, [0.0, 1.0, 0.0]) if abs(a[1]) < 0.9 else np.cross(a, [1.0, 0, 0]))
        c = np.cross(a, b)
        return rotmat_to_quat(np.stack([a, b, c], axis=1))
    adv_means = np.array([[0.30, 0.05, -0.30],    # (i) mean behind camera, crosses image plane
                          [0.00, 0.00, 0.20],     # (ii) camera inside -> discarded
                          [0.00, 0.20, 1.00],     # (iii) long thin, tangent > 90 deg from theta_mu
                          [-0.20, 0.10, 0.05]])   # (iv) straddles the near plane
    adv_scales = np.array([[0.05, 0.05, 0.60],
                           [0.30, 0.30, 0.30],
                           [1.00, 0.03, 0.03],
                           [0.10, 0.10, 0.015]])
    adv_quats = np.array([[1.0, 0, 0, 0], [1.0, 0, 0, 0], q_axis([2.0, 0.0, -1.0]),
                          [1.0, 0, 0, 0]])
    adv_opac = np.array([0.9, 0.8, 0.85, 0.9])
    means = np.vstack([means, adv_means])
    scales = np.vstack([scales, adv_scales])
    quats = np.vstack([quats, adv_quats])
    opac = np.concatenate([opac, adv_opac])
    N = means.shape[0]
    sh = np.zeros((N, 1, 3), dtype=np.float32)
    sh[:, 0, :] = rng.normal(0.0, 0.6, (N, 3))
    cam = c1_camera()
    vhat = np.where(means[:, 2] > 0, cam.fx / np.where(means[:, 2] > 0, means[:, 2], 1.0), np.inf)
    vt = np.where(np.arange(N) % 2 == 0, np.inf, 0.5 * vhat)
    return Scene(means.astype(np.float32), scales.astype(np.float32), quats.astype(np.float32),
                 opac.astype(np.float32), sh, vt.astype(np.float32), 0)


def random_box_scene(seed: int, n: int, deg: int = 0, box=((-1, 1), (-1, 1), (1.5, 4.0)),
                     scale_range=(0.01, 0.3)) -> Scene:
    """SPEC cmd_synth-style random scene: log-uniform scales,
    uniform rotations, opacity U[0.2,0.95]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    means = np.column_stack([rng.uniform(*box[i], n) for i in range(3)])
    scales = np.exp(rng.uniform(np.log(scale_range[0]), np.log(scale_range[1]), (n, 3)))
    quats = rng.standard_normal((n, 4))
    opac = rng.uniform(0.2, 0.95, n)
    sh = _sh_coeffs(rng, n, deg)
    vt = np.full(n, np.inf)
    return Scene(means.astype(np.float32), scales.astype(np.float32), quats.astype(np.float32),
                 opac.astype(np.float32), sh, vt.astype(np.float32), deg)


# --------------------------------------------------------------------------
# c2: Blender-like, 100k, SH3, 800x800, 100-view Fibonacci hemisphere
# --------------------------------------------------------------------------
def c2_cameras(n_views: int = 100) -> list:
    cams = []
    ga = math.pi * (3.0 - math.sqrt(5.0))
    for i in range(n_views):
        z = 0.05 + 0.9 * (i + 0.5) / n_views          # upper hemisphere
        r = math.sqrt(1 - z * z)
        th = ga * i
        eye = 4.0 * np.array([r * math.cos(th), r * math.sin(th), z])
        cams.append(Camera(800, 800, 1111.1, 1111.1, 400.0, 400.0, look_at(eye, (0, 0, 0)), 0.01))
    return cams


def _sample_sphere(rng, n, c, r):
    d = _unit(rng.standard_normal((n, 3)))
    return c + r * d, d


def _sample_torus(rng, n, c, R, r):
    # area-uniform via rejection on the minor angle
    u = rng.uniform(0, 2 * np.pi, 4 * n)
    v = rng.uniform(0, 2 * np.pi, 4 * n)
    keep = rng.uniform(0, 1, 4 * n) < (R + r * np.cos(v)) / (R + r)
    u, v = u[keep][:n], v[keep][:n]
    p = np.column_stack([(R + r * np.cos(v)) * np.cos(u), (R + r * np.cos(v)) * np.sin(u), r * np.sin(v)])
    nrm = np.column_stack([np.cos(v) * np.cos(u), np.cos(v) * np.sin(u), np.sin(v)])
    return c + p, nrm


def _sample_box(rng, n, c, ext):
    a, b, h = ext
    areas = np.array([b * h, b * h, a * h, a * h, a * b, a * b])
    face = rng.choice(6, n, p=areas / areas.sum())
    uv = rng.uniform(-0.5, 0.5, (n, 2))
    p = np.zeros((n, 3))
    nrm = np.zeros((n, 3))
    for f in range(6):
        m = face == f
        ax = f // 2
        sgn = 1.0 if f % 2 == 0 else -1.0
        other = [i for i in range(3) if i != ax]
        p[m, ax] = sgn * ext[ax] / 2
        p[m, other[0]] = uv[m, 0] * ext[other[0]]
        p[m, other[1]] = uv[m, 1] * ext[other[1]]
        nrm[m, ax] = sgn
    return c + p, nrm


def c2_scene(seed: int = 2, n: int = 100_000, n_views_vtrain: int = 100) -> Scene:
    rng = np.random.Generator(np.random.PCG64(seed))
    n_surf = int(0.8 * n)
    n_vol = n - n_surf
    shapes = [("s", (0.2, -0.3, 0.1), 0.5), ("s", (-0.6, 0.5, -0.2), 0.35),
              ("s", (0.7, 0.6, 0.4), 0.3), ("t", (-0.3, -0.5, -0.6), (0.6, 0.12)),
              ("b", (0.5, -0.6, 0.6), (0.5, 0.5, 0.4))]
    areas = np.array([4 * np.pi * 0.25, 4 * np.pi * 0.35 ** 2, 4 * np.pi * 0.09,
                      4 * np.pi ** 2 * 0.6 * 0.12, 2 * (0.25 + 0.2 + 0.2)])
    counts = np.floor(n_surf * areas / areas.sum()).astype(int)
    counts[0] += n_surf - counts.sum()
    P, Nn = [], []
    for (kind, c, prm), k in zip(shapes, counts):
        c = np.asarray(c)
        if kind == "s":
            p, nr = _sample_sphere(rng, k, c, prm)
        elif kind == "t":
            p, nr = _sample_torus(rng, k, c, *prm)
        else:
            p, nr = _sample_box(rng, k, c, prm)
        P.append(p)
        Nn.append(nr)
    P = np.vstack(P)
    Nn = np.vstack(Nn)
    spacing = math.sqrt(areas.sum() / n_surf)
    med = 0.7 * spacing
    s12 = med * np.exp(0.6 * rng.standard_normal((n_surf, 2)))
    s3 = 0.1 * np.sqrt(s12[:, 0] * s12[:, 1])
    R = _tangent_frames(rng, Nn)
    q_surf = rotmat_to_quat(R)
    s_surf = np.column_stack([s12, s3])
    # volume fill: isotropic-ish blobs, random rotations
    p_vol = rng.uniform(-1.3, 1.3, (n_vol, 3))
    s_vol = med * np.exp(0.6 * rng.standard_normal((n_vol, 3)))
    q_vol = rng.standard_normal((n_vol, 4))
    means = np.vstack([P, p_vol])
    scales = np.vstack([s_surf, s_vol])
    quats = np.vstack([q_surf, q_vol])
    perm = rng.permutation(n)
    means, scales, quats = means[perm], scales[perm], quats[perm]
    opac = _bimodal_opacity(rng, n)
    sh = _sh_coeffs(rng, n, 3)
    vt = v_train_from_cameras(means, c2_cameras(n_views_vtrain))
    return Scene(means.astype(np.float32), scales.astype(np.float32), quats.astype(np.float32),
                 opac, sh, vt, 3)


# --------------------------------------------------------------------------
# c3 / c4 / c5: M360-like surfel scene (calibrated in E11)
# --------------------------------------------------------------------------
C3_TARGET = np.array([0.0, 0.0, 0.5])


def c3_cameras(n_views: int = 200, width=1920, height=1080, f=1663.0, radius_scale=1.0) -> list:
    cams = []
    for i in range(n_views):
        a = 2 * np.pi * i / n_views
        eye = np.array([4.0 * radius_scale * math.cos(a), 3.2 * radius_scale * math.sin(a),
                        1.5 + 0.3 * math.sin(3 * a)])
        cams.append(Camera(width, height, f, f, width / 2.0, height / 2.0,
                           look_at(eye, C3_TARGET), 0.01))
    return cams


def c4_cameras(kind: str, n_views: int = 50) -> list:
    """c4 OOD sub-batches: 'wide' (120 deg FoV), 'zoomout' (orbit x8), 'inside'
    (dolly from the orbit into the object centre)."""
    if kind == "wide":
        base = c3_cameras(200)
        return [c.scaled(fx=554.3, fy=554.3) for c in base[::4][:n_views]]
    if kind == "zoomout":
        return c3_cameras(200, radius_scale=8.0)[::4][:n_views]
    if kind == "inside":
        # 40 views dolly from the orbit into the object region, then 10 views land on the ground
        # disc: heights log-spaced down to 4 mm, pitching down to 38 degrees, so the last views have
        # the camera inside ground surfels and every visible Gaussian crossing the near
        # plane (the exact 5-constraint culling path)
        cams = []
        start = np.array([4.0, 0.0, 1.5])
        end = np.array([0.0, 0.05, 0.5])      # object centre region
        n_dolly = n_views - 10 if n_views > 20 else n_views
        d0 = np.array([-1.0, 0.02, -0.15])
        for i in range(n_dolly):
            t = (i / max(1, n_views - 1)) ** 0.5
            eye = (1 - t) * start + t * end
            cams.append(Camera(1920, 1080, 1663.0, 1663.0, 960.0, 540.0, look_at(eye, eye + d0), 0.01))
        if n_dolly < n_views:
            e0 = (1 - ((n_dolly - 1) / (n_views - 1)) ** 0.5) * start + ((n_dolly - 1) / (n_views - 1)) ** 0.5 * end
            land = np.array([2.5, 0.0, 0.004])
            pitch = np.radians(38.0)
            d1 = np.array([-math.cos(pitch), 0.0, -math.sin(pitch)])
            m = n_views - n_dolly
            for k in range(1, m + 1):
                u = k / m
                h = math.exp((1 - u) * math.log(e0[2]) + u * math.log(land[2]))
                xy = (1 - u) * e0[:2] + u * land[:2]
                eye = np.array([xy[0], xy[1], h])
                d = (1 - u) * d0 / np.linalg.norm(d0) + u * d1
                cams.append(Camera(1920, 1080, 1663.0, 1663.0, 960.0, 540.0, look_at(eye, eye + d), 0.01))
        return cams
    raise ValueError(kind)


def c5_camera() -> Camera:
    c = c3_cameras(200)[0]
    return Camera(3840, 2160, 3326.0, 3326.0, 1920.0, 1080.0, c.world_to_view, 0.01)


def c3_scene(seed: int = 3, n: int = 3_000_000, vtrain_views: int = 200) -> Scene:
    rng = np.random.Generator(np.random.PCG64(seed))
    n_obj = int(0.55 * n)
    n_gnd = int(0.25 * n)
    n_bg = n - n_obj - n_gnd
    # 8 spheres
    radii = rng.uniform(0.2, 0.7, 8)
    centres = rng.uniform(-0.8, 0.8, (8, 3)) + C3_TARGET
    areas = 4 * np.pi * radii ** 2
    counts = np.floor(n_obj * areas / areas.sum()).astype(int)
    counts[0] += n_obj - counts.sum()
    sid = np.repeat(np.arange(8), counts)
    d = _unit(rng.standard_normal((n_obj, 3)))
    rj = radii[sid] * (1.0 + 0.002 * rng.standard_normal(n_obj))
    p_obj = centres[sid] + rj[:, None] * d
    sp_obj = math.sqrt(areas.sum() / n_obj)
    s_obj = 0.7 * sp_obj * np.ones(n_obj)
    # ground disc radius 6 at z = 0, normal +z
    rr = 6.0 * np.sqrt(rng.uniform(0, 1, n_gnd))
    ph = rng.uniform(0, 2 * np.pi, n_gnd)
    p_gnd = np.column_stack([rr * np.cos(ph), rr * np.sin(ph), np.zeros(n_gnd)])
    n_gnd_v = np.tile([0.0, 0.0, 1.0], (n_gnd, 1))
    s_gnd = 0.7 * math.sqrt(np.pi * 36.0 / n_gnd) * np.ones(n_gnd)
    # background hemisphere, r log-uniform in [15, 80]
    rb = np.exp(rng.uniform(np.log(15.0), np.log(80.0), n_bg))
    db = _unit(rng.standard_normal((n_bg, 3)))
    db[:, 2] = np.abs(db[:, 2])
    p_bg = rb[:, None] * db
    s_bg = 0.003 * rb
    means = np.vstack([p_obj, p_gnd, p_bg])
    normals = np.vstack([d, n_gnd_v, db])
    med = np.concatenate([s_obj, s_gnd, s_bg])
    s12 = med[:, None] * np.exp(0.6 * rng.standard_normal((n, 2)))
    s3 = 0.1 * np.sqrt(s12[:, 0] * s12[:, 1])
    scales = np.column_stack([s12, s3])
    quats = rotmat_to_quat(_tangent_frames(rng, normals))
    perm = rng.permutation(n)
    means, scales, quats = means[perm], scales[perm], quats[perm]
    opac = _bimodal_opacity(rng, n)
    sh = _sh_coeffs(rng, n, 3)
    vt = v_train_from_cameras(means, c3_cameras(vtrain_views))
    return Scene(means.astype(np.float32), scales.astype(np.float32), quats.astype(np.float32),
                 opac, sh, vt, 3)


# --------------------------------------------------------------------------
# caching + registry
# --------------------------------------------------------------------------
def _cache_dir() -> Path:
    d = os.environ.get("AAA_SCENE_CACHE")
    if d:
        return Path(d)
    # outside the repo, so the cached .npz bytes never travel with gpurun snapshots
    return Path.home() / ".cache" / "aaa_scenes"


def cached(name: str, fn, *args, **kw) -> Scene:
    """Generate (or load the cached bytes of) a seeded scene. The cache is an
    accelerator only: a missing cache just regenerates the same bytes."""
    key = hashlib.sha1(repr((name, args, sorted(kw.items()), 2)).encode()).hexdigest()[:16]
    path = _cache_dir() / f"{name}_{key}.npz"
    if path.exists():
        try:
            z = np.load(path)
            return Scene(z["means"], z["scales"], z["quats"], z["opacities"], z["sh"],
                         z["v_train"], int(z["sh_degree"]))
        except Exception:
            pass
    s = fn(*args, **kw)
    try:
        path.parent.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(".tmp.npz")
        np.savez(tmp, means=s.means, scales=s.scales, quats=s.quats, opacities=s.opacities,
                 sh=s.sh, v_train=s.v_train, sh_degree=s.sh_degree)
        os.replace(tmp, path)
    except OSError:
        pass
    return s


def make_config(name: str, n: int | None = None):
    """Return (scene, [cameras]) for a config id: c1, c2, c3, c4wide, c4zoomout,
    c4inside, c5. ``n`` overrides the Gaussian count (parity at reduced size)."""
    if name == "c1":
        return c1_scene(), [c1_camera()]
    if name == "c2":
        return cached("c2", c2_scene, n=n or 100_000), c2_cameras()
    if name == "c3":
        return cached("c3", c3_scene, n=n or 3_000_000), c3_cameras()
    if name.startswith("c4"):
        return cached("c3", c3_scene, n=n or 3_000_000), c4_cameras(name[2:])
    if name == "c5":
        return cached("c5", c3_scene, seed=5, n=n or 6_000_000), [c5_camera()]
    raise ValueError(name)


CONFIGS = ("c1", "c2", "c3", "c4wide", "c4zoomout", "c4inside", "c5")
