"""Test-side helpers: tiny hand-built scenes and INDEPENDENT re-derivations used to
pin the oracle (never the oracle's own formulas retyped)."""
from __future__ import annotations

import numpy as np

from synth import scenes as S


def one_gaussian(mu, s, q=(1.0, 0, 0, 0), o=0.9, rgb=(0.3, 0.6, 0.9), v_train=np.inf, deg=0):
    K = (deg + 1) ** 2
    sh = np.zeros((1, K, 3), dtype=np.float32)
    C0 = 0.28209479177387814
    sh[0, 0, :] = (np.asarray(rgb) - 0.5) / C0
    return S.Scene(np.asarray([mu], np.float32), np.asarray([s], np.float32),
                   np.asarray([q], np.float32), np.asarray([o], np.float32), sh,
                   np.asarray([v_train], np.float32), deg)


def concat(scenes):
    return S.Scene(*(np.concatenate([getattr(s, f) for s in scenes]) for f in
                     ("means", "scales", "quats", "opacities", "sh", "v_train")),
                   scenes[0].sh_degree)


def pinhole(W=64, H=64, f=56.0, V=None, near=0.01, cx=None, cy=None):
    return S.Camera(W, H, f, f, W / 2.0 if cx is None else cx, H / 2.0 if cy is None else cy,
                    np.eye(4) if V is None else np.asarray(V, np.float64), near)


def filtered_T_view(scene, g, cam, k=0.3):
    """T_view = V T with filtered scales: returns (M 3x3, mu_v 3) where a
    Gaussian-space point u maps to view space M u + mu_v. Filter per Eq. 6/13/12
    written from the paper's text (v_hat = f/d, v' = min, s_hat = s^2 + k/v'^2)."""
    V = np.asarray(cam.world_to_view, np.float64)
    mu = scene.means[g].astype(np.float64)
    muv = V[:3, :3] @ mu + V[:3, 3]
    f = max(cam.fx, cam.fy)
    vhat = f / muv[2] if muv[2] > 0 else np.inf
    veff = min(float(scene.v_train[g]), vhat)
    cf = 0.0 if np.isinf(veff) else k / veff ** 2
    shat = scene.scales[g].astype(np.float64) ** 2 + cf
    R = S.quat_to_rotmat(scene.quats[g].astype(np.float64))
    M = V[:3, :3] @ R @ np.diag(np.sqrt(shat))
    return M, muv, shat, R


def plane_form_rho2(M, muv, cam, px, py):
    """The paper's 3D evaluation (Eq. 4-5): pixel planes pi_x=(1,0,0,-x),
    pi_y=(0,1,0,-y) pulled back by T'^T with T' = M_vp P V T, then the distance of their
    intersection line to the Gaussian-space origin. Returns (rho^2, view z of that point)."""
    T = np.eye(4)
    T[:3, :3] = M
    T[:3, 3] = muv                           # V T (view <- Gaussian space)
    KP = np.array([[cam.fx, 0, cam.cx, 0], [0, cam.fy, cam.cy, 0], [0, 0, 0, 1.0], [0, 0, 1.0, 0]])
    Tp = KP @ T                              # T' = M_vp P V T (pixel-space projective map)
    pi_x = Tp.T @ np.array([1.0, 0, 0, -px])
    pi_y = Tp.T @ np.array([0, 1.0, 0, -py])
    A = np.stack([pi_x[:3], pi_y[:3]])
    b = -np.array([pi_x[3], pi_y[3]])
    u = A.T @ np.linalg.solve(A @ A.T, b)    # least-norm point on the line
    z = (T @ np.append(u, 1.0))[2]
    return float(u @ u), float(z)


def eq12_amplitude(s, shat, R, d):
    """Eq. 12 closed form with d' = R^T d (Eq. 11)."""
    dp = R.T @ d
    s2 = np.asarray(s, np.float64) ** 2
    num = dp[0] ** 2 * s2[1] * s2[2] + dp[1] ** 2 * s2[0] * s2[2] + dp[2] ** 2 * s2[0] * s2[1]
    den = dp[0] ** 2 * shat[1] * shat[2] + dp[1] ** 2 * shat[0] * shat[2] + dp[2] ** 2 * shat[0] * shat[1]
    return np.sqrt(num / den)
