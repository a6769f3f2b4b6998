"""Differentiable float64 reference of the forward render, for the backward-pass parity tests.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): imported by tests/ only, never by the
product path. Plain PyTorch CPU float64 written from the paper's definitions with the oracle's
algebra (not the CUDA path's): per Gaussian R(q) (Eq. 3), the adaptive filter (Eq. 6, 13,
P:153), the amplitude by the matrix form of Eq. 10, tau = 2 ln(255 o A) (reading 1), SH colour
(reading 15), the camera-inside discard; per pixel the maximum-response point by explicit
minimisation with Sigma_hat^-1, the exact (z*, g) order (reading 4) and the 3DGS blend
with termination (readings 2, 3). Dense over (pixel, Gaussian): for small scenes only.

The contribution set and the order are decided on detached values (the tau cutoff, near plane,
inside test and termination carry no derivative), exactly the convention the CUDA backward uses.
torch.autograd then differentiates the resulting piecewise-smooth function.
"""
from __future__ import annotations

import numpy as np
import torch

SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792, 0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154, -0.4570457994644658,
         1.445305721320277, -0.5900435899266435)


def _f32(x):
    return float(np.float32(x))


def sh_basis(d):
    """3DGS real SH basis (16) at unit directions d (..., 3) (reading 15)."""
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    xx, yy, zz, xy, yz, xz = x * x, y * y, z * z, x * y, y * z, x * z
    b = [torch.full_like(x, SH_C0), -SH_C1 * y, SH_C1 * z, -SH_C1 * x,
         SH_C2[0] * xy, SH_C2[1] * yz, SH_C2[2] * (2 * zz - xx - yy), SH_C2[3] * xz, SH_C2[4] * (xx - yy),
         SH_C3[0] * y * (3 * xx - yy), SH_C3[1] * xy * z, SH_C3[2] * y * (4 * zz - xx - yy),
         SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy), SH_C3[4] * x * (4 * zz - xx - yy), SH_C3[5] * z * (xx - yy),
         SH_C3[6] * x * (xx - 3 * yy)]
    return torch.stack(b, -1)


def render(params: dict, scene, cam, k=0.3, alpha_max=0.99, T_eps=1e-4, bg=(0.0, 0.0, 0.0)):
    """params: float64 tensors means (N,3), scales (N,3), quats (N,4), opacities (N,), sh (N,K,3).
    Returns (rgb (H,W,3), T (H,W)) as differentiable float64 tensors."""
    mu, s, q, o, sh = params["means"], params["scales"], params["quats"], params["opacities"], params["sh"]
    N = mu.shape[0]
    K = sh.shape[1]
    V = torch.tensor([[_f32(v) for v in row] for row in np.asarray(cam.world_to_view, np.float64)], dtype=torch.float64)
    Rv, tv = V[:3, :3], V[:3, 3]
    fx, fy, cx, cy, near = _f32(cam.fx), _f32(cam.fy), _f32(cam.cx), _f32(cam.cy), _f32(cam.near)
    Rvi = torch.linalg.inv(Rv)  # the given affine map's exact inverse (reading 37)
    cam_o = -Rvi @ tv
    vt = torch.tensor(np.asarray(scene.v_train, np.float64))
    # R(q), q normalised (Eq. 3)
    qn = q / q.norm(dim=1, keepdim=True)
    w, x, y, z = qn[:, 0], qn[:, 1], qn[:, 2], qn[:, 3]
    R = torch.stack([torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
                     torch.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
                     torch.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)], 1)
    muv = mu @ Rv.T + tv
    # Eq. 6 / 13: v_hat = f / d (inf behind the camera), v' = min(v_train, v_hat); k / v'^2
    f = max(fx, fy)
    vhat = torch.where(muv[:, 2] > 0, f / muv[:, 2].clamp(min=1e-300), torch.full_like(muv[:, 2], float("inf")))
    veff = torch.minimum(vt, vhat)
    cf = torch.where(torch.isinf(veff), torch.zeros_like(veff), k / (veff * veff).clamp(min=1e-300))
    Sig = R @ torch.diag_embed(s * s) @ R.transpose(1, 2)
    Shat = Sig + cf[:, None, None] * torch.eye(3, dtype=torch.float64)
    d = mu - cam_o
    d = d / d.norm(dim=1, keepdim=True)
    # Eq. 10: A = sqrt(|Sigma| d^T Sigma^-1 d / (|Sigma_hat| d^T Sigma_hat^-1 d))
    Sinv = torch.linalg.inv(Sig)
    Shinv = torch.linalg.inv(Shat)
    num = torch.linalg.det(Sig) * torch.einsum("ni,nij,nj->n", d, Sinv, d)
    den = torch.linalg.det(Shat) * torch.einsum("ni,nij,nj->n", d, Shinv, d)
    A = torch.where(cf > 0, torch.sqrt(num / den), torch.ones_like(cf))
    oA = o * A
    tau = (2 * torch.log(255 * oA)).detach()
    om = cam_o[None, :] - mu
    inside = (torch.einsum("ni,nij,nj->n", om, Shinv, om) < tau).detach()
    valid = (tau > 0) & ~inside
    col = torch.clamp(torch.einsum("nk,nkc->nc", sh_basis(d)[:, :K], sh) + 0.5, min=0.0)
    # per pixel
    H, W = cam.height, cam.width
    yy, xx = torch.meshgrid(torch.arange(H, dtype=torch.float64), torch.arange(W, dtype=torch.float64), indexing="ij")
    r = torch.stack([(xx + 0.5 - cx) / fx, (yy + 0.5 - cy) / fy, torch.ones_like(xx)], -1).reshape(-1, 3)
    v = r @ Rvi.T  # world direction with view-z 1 (rows: Rv^-1 r)
    mo = mu - cam_o
    Sv = torch.einsum("nij,pj->pni", Shinv, v)           # S^-1 v   (P,N,3)
    vSv = torch.einsum("pi,pni->pn", v, Sv)
    vSmo = torch.einsum("pni,ni->pn", Sv, mo)
    t = vSmo / vSv                                         # z* (view depth)
    e = cam_o[None, None, :] + t[..., None] * v[:, None, :] - mu[None, :, :]
    rho2 = torch.einsum("pni,nij,pnj->pn", e, Shinv, e)
    inc = ((rho2 < tau[None, :]) & (t >= near) & valid[None, :]).detach()
    alpha = torch.clamp(oA[None, :] * torch.exp(-0.5 * rho2), max=alpha_max)
    alpha = torch.where(inc, alpha, torch.zeros_like(alpha))
    # exact order (z*, g) on detached depths; excluded entries last
    key = torch.where(inc, t.detach(), torch.full_like(t, float("inf")))
    order = torch.argsort(key, dim=1, stable=True)
    a_s = torch.gather(alpha, 1, order)
    inc_s = torch.gather(inc, 1, order)
    one_m = 1 - a_s
    Tex = torch.cumprod(torch.cat([torch.ones_like(one_m[:, :1]), one_m[:, :-1]], 1), 1)  # T before each entry
    # termination (reading 3): the first included entry with T (1 - alpha) < T_eps and everything after
    stop = (inc_s & ((Tex * one_m).detach() < T_eps))
    after = torch.cumsum(stop.to(torch.int64), 1) > 0
    use = inc_s & ~after
    a_u = torch.where(use, a_s, torch.zeros_like(a_s))
    one_u = 1 - a_u
    Tu = torch.cumprod(torch.cat([torch.ones_like(one_u[:, :1]), one_u[:, :-1]], 1), 1)
    c_s = col[order]                                       # (P,N,3)
    C = torch.einsum("pn,pnc->pc", a_u * Tu, c_s)
    Tn = torch.prod(one_u, 1)
    C = C + Tn[:, None] * torch.tensor(bg, dtype=torch.float64)[None, :]
    return C.reshape(H, W, 3), Tn.reshape(H, W)


def params_of(scene, requires_grad=True) -> dict:
    K = (scene.sh_degree + 1) ** 2
    to = lambda a: torch.tensor(np.asarray(a, np.float32).astype(np.float64), requires_grad=requires_grad)
    return dict(means=to(scene.means), scales=to(scene.scales), quats=to(scene.quats), opacities=to(scene.opacities),
                sh=to(np.asarray(scene.sh, np.float32).reshape(scene.n, K, 3)))


def grads(scene, cam, w_rgb: np.ndarray, w_T: np.ndarray, **kw) -> dict:
    """Gradients of L = sum(w_rgb * rgb) + sum(w_T * T) (w_rgb: 3 x H x W, w_T: H x W)."""
    P = params_of(scene)
    rgb, T = render(P, scene, cam, **kw)
    L = (torch.tensor(w_rgb, dtype=torch.float64).permute(1, 2, 0) * rgb).sum() + \
        (torch.tensor(w_T, dtype=torch.float64) * T).sum()
    L.backward()
    return {k: v.grad.numpy() for k, v in P.items()}
