"""Pins of the float64 oracle against what the paper and mathematics fix
(closed forms, identities, independent re-derivations, brute force) — CPU only.

Each test names the passage it pins. None of these re-type the oracle's own
formula: the oracle uses Eq. 10 (matrix) for A, Sigma_hat^-1 ray minimisation for
rho^2, and active-set enumeration for culling; the tests use Eq. 12, Appendix A,
the plane pullback (Eq. 4-5), quadrature, scipy and brute force.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from synth import scenes as S
from tests.helpers import (concat, eq12_amplitude, filtered_T_view, one_gaussian, pinhole,
                           plane_form_rho2)

GOLDEN = Path(__file__).parent / "golden"
FI = {f: i for i, f in enumerate(O.G_FIELDS)}
CI = {f: i for i, f in enumerate(O.C_FIELDS)}


def _rand_scene(seed, n, deg=0, box=((-1, 1), (-1, 1), (1.5, 4.0)), vtrain_mode="half"):
    s = S.random_box_scene(seed, n, deg, box=box, scale_range=(0.005, 0.4))
    rng = np.random.default_rng(seed + 100)
    if vtrain_mode == "half":
        s.v_train[:] = np.where(rng.random(n) < 0.5, np.inf, rng.uniform(5.0, 80.0, n)).astype(np.float32)
    return s


# ---------------------------------------------------------------- filter
def test_golden_spec_filter_examples():
    """SPEC worked examples stored under tests/golden/."""
    gold = json.loads((GOLDEN / "spec_examples.json").read_text())
    for ex in gold["filter"]:
        cam = pinhole(W=2000, H=2000, f=ex["f"])
        sc = one_gaussian(mu=(0, 0, ex["d"]), s=ex["s"], v_train=ex.get("v_train", np.inf))
        G = O.Oracle(sc).set_view(cam, k=ex["k"]).gaussians()[0]
        assert G[FI["vhat"]] == pytest.approx(ex["v_hat"], rel=1e-12), ex["cite"]
        if "s_hat" in ex:
            np.testing.assert_allclose(G[FI["shat0"]:FI["shat2"] + 1], ex["s_hat"], rtol=1e-6, err_msg=ex["cite"])


def test_filter_k0_is_identity():
    """k = 0 -> s_hat = s^2 and A = 1."""
    sc = _rand_scene(1, 200)
    G = O.Oracle(sc).set_view(pinhole(), k=0.0).gaussians()
    np.testing.assert_array_equal(G[:, FI["A"]], 1.0)
    np.testing.assert_allclose(G[:, FI["shat0"]:FI["shat2"] + 1], sc.scales.astype(np.float64) ** 2, rtol=1e-15)


def test_filter_isotropic_closed_form():
    """Isotropic s = sigma: A = sigma^2 / (sigma^2 + k/v'^2) (Eq. 12 collapses)."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        sig = rng.uniform(0.001, 0.2)
        z = rng.uniform(0.5, 30)
        mu = (rng.uniform(-0.3, 0.3) * z, rng.uniform(-0.3, 0.3) * z, z)
        q = rng.standard_normal(4)
        sc = one_gaussian(mu, (sig, sig, sig), q=q)
        cam = pinhole(f=800.0)
        G = O.Oracle(sc).set_view(cam, k=0.3).gaussians()[0]
        cf = 0.3 / (800.0 / float(np.float32(z))) ** 2
        sig2 = np.float64(np.float32(sig)) ** 2
        assert G[FI["A"]] == pytest.approx(sig2 / (sig2 + cf), rel=1e-9)


def test_filter_axis_aligned():
    """d along local axis 1 -> A = sqrt(s2^2 s3^2 / (s_hat2 s_hat3))."""
    s = np.array([0.05, 0.01, 0.003], np.float32)
    sc = one_gaussian((0, 0, 3.0), s)          # identity rotation: local axis 1 = world x
    V = S.look_at([-2.0, 0, 3.0], [0, 0, 3.0])  # camera on the -x side looking along +x
    cam = pinhole(f=400.0, V=V)
    G = O.Oracle(sc).set_view(cam, k=0.3).gaussians()[0]
    shat = G[FI["shat0"]:FI["shat2"] + 1]
    s64 = s.astype(np.float64)
    assert G[FI["A"]] == pytest.approx(math.sqrt(s64[1] ** 2 * s64[2] ** 2 / (shat[1] * shat[2])), rel=1e-9)


def test_eq10_matches_eq12_and_appendix_a():
    """The oracle's Eq. 10 matrix form equals the Eq. 12 closed form and the
    Appendix A explicit-projection determinant ratio to 1e-9."""
    sc = _rand_scene(5, 2000)
    cam = pinhole(f=300.0)
    G = O.Oracle(sc).set_view(cam, k=0.3).gaussians()
    o = np.zeros(3)
    worst12 = worstA = 0.0
    for g in range(sc.n):
        M, muv, shat, R = filtered_T_view(sc, g, cam)
        s = sc.scales[g].astype(np.float64)
        d = sc.means[g].astype(np.float64) - o
        d /= np.linalg.norm(d)
        a12 = eq12_amplitude(s, shat, R, d)
        # Appendix A: orthonormal basis U with d first, Sigma' = U^T Sigma U, lower-right 2x2 block
        U, _ = np.linalg.qr(np.column_stack([d, np.random.default_rng(g).standard_normal((3, 2))]))
        Sig = R @ np.diag(s ** 2) @ R.T
        Shat = R @ np.diag(shat) @ R.T
        perp = np.linalg.det((U.T @ Sig @ U)[1:, 1:])
        perph = np.linalg.det((U.T @ Shat @ U)[1:, 1:])
        aA = math.sqrt(perp / perph)
        worst12 = max(worst12, abs(G[g, FI["A"]] / a12 - 1))
        worstA = max(worstA, abs(G[g, FI["A"]] / aA - 1))
    assert worst12 < 1e-9 and worstA < 1e-9, (worst12, worstA)


def test_amplitude_at_least_volume_factor_and_monotone():
    """A_perp >= sqrt(|Sigma|/|Sigma_hat|) (Eq. 8, P:224-227 motivation) and A is
    non-increasing in k."""
    sc = _rand_scene(6, 1000)
    cam = pinhole(f=200.0)
    orc = O.Oracle(sc)
    prev = None
    for k in (0.0, 0.1, 0.3, 1.0, 3.0):
        G = orc.set_view(cam, k=k).gaussians()
        shat = G[:, FI["shat0"]:FI["shat2"] + 1]
        vol = np.sqrt(np.prod(sc.scales.astype(np.float64) ** 2, axis=1) / np.prod(shat, axis=1))
        assert np.all(G[:, FI["A"]] >= vol * (1 - 1e-12))
        if prev is not None:
            assert np.all(G[:, FI["A"]] <= prev * (1 + 1e-12))
        prev = G[:, FI["A"]]


def test_closer_camera_invariance():
    """v_hat >= v_train -> v' = v_train: s_hat and A independent of a larger focal (Eq. 13)."""
    sc = _rand_scene(8, 300)
    sc.v_train[:] = 1.0
    orc = O.Oracle(sc)
    Ga = orc.set_view(pinhole(f=100.0), k=0.3).gaussians()
    Gb = orc.set_view(pinhole(f=1000.0), k=0.3).gaussians()
    front = sc.means[:, 2] > 0
    for f in ("veff", "shat0", "shat1", "shat2", "A", "tau"):
        np.testing.assert_array_equal(Ga[front, FI[f]], Gb[front, FI[f]])


# ---------------------------------------------------------------- SH colour (reading 15)
def test_sh_basis_against_scipy():
    """Oracle real-SH basis == scipy complex Y_lm (Condon-Shortley) in the 3DGS real form;
    Y00 = 1/(2 sqrt(pi)) (SURVEY 8c 'SH')."""
    from scipy.special import sph_harm_y
    rng = np.random.default_rng(0)
    for _ in range(200):
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        th = math.acos(d[2])
        ph = math.atan2(d[1], d[0])
        ref = []
        for l in range(4):
            for m in range(-l, l + 1):
                Y = sph_harm_y(l, abs(m), th, ph)
                ref.append(Y.real if m == 0 else math.sqrt(2) * (Y.imag if m < 0 else Y.real))
        np.testing.assert_allclose(O.sh_basis(d), ref, atol=1e-12)
    assert O.sh_basis(np.array([0, 0, 1.0]))[0] == pytest.approx(1 / (2 * math.sqrt(math.pi)), abs=1e-16)


def test_sh_orthonormal_by_quadrature():
    """Gauss-Legendre x uniform-phi quadrature (exact for degree <= 6 products)."""
    xs, ws = np.polynomial.legendre.leggauss(8)
    nphi = 16
    G = np.zeros((16, 16))
    for x, w in zip(xs, ws):
        for j in range(nphi):
            ph = 2 * math.pi * j / nphi
            st = math.sqrt(1 - x * x)
            Y = O.sh_basis(np.array([st * math.cos(ph), st * math.sin(ph), x]))
            G += np.outer(Y, Y) * w * (2 * math.pi / nphi)
    np.testing.assert_allclose(G, np.eye(16), atol=1e-12)


# ---------------------------------------------------------------- per-pixel evaluation
def _contrib_of(orc, px, py, g=0):
    c = orc.pixel_contribs(px, py)
    m = c[:, CI["g"]] == g
    return c[m][0] if np.any(m) else None


def test_rho2_matches_paper_plane_form():
    """Oracle rho^2/z* (Sigma_hat^-1 minimisation) == the paper's plane pullback
    T'^T pi_x, T'^T pi_y and distance of their intersection line (Eq. 4-5)."""
    rng = np.random.default_rng(11)
    cam = pinhole(W=64, H=64, f=56.0)
    checked = 0
    for t in range(60):
        mu = (rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), rng.uniform(1.0, 5.0))
        s = np.exp(rng.uniform(np.log(0.01), np.log(0.5), 3))
        sc = one_gaussian(mu, s, q=rng.standard_normal(4), v_train=rng.choice([np.inf, 20.0]))
        orc = O.Oracle(sc).set_view(cam, k=0.3)
        M, muv, _, _ = filtered_T_view(sc, 0, cam)
        for _ in range(10):
            px = int(np.clip(cam.fx * muv[0] / muv[2] + cam.cx + rng.uniform(-8, 8), 0, 63))
            py = int(np.clip(cam.fy * muv[1] / muv[2] + cam.cy + rng.uniform(-8, 8), 0, 63))
            c = _contrib_of(orc, px, py)
            if c is None:
                continue
            r2, z = plane_form_rho2(M, muv, cam, px + 0.5, py + 0.5)
            assert c[CI["rho2"]] == pytest.approx(r2, rel=1e-9, abs=1e-12)
            assert c[CI["z"]] == pytest.approx(z, rel=1e-9)
            checked += 1
    assert checked > 100


def test_rho2_max_response_by_line_search_and_ray_integral():
    """Max of the Gaussian-space density exp(-|u|^2/2) along the pixel ray by
    dense + golden-section search, and the closed-form ray integral
    int exp(-rho^2(t)/2) dt = exp(-rho_min^2/2) sqrt(2 pi / |w|^2) by quadrature."""
    rng = np.random.default_rng(12)
    cam = pinhole(W=64, H=64, f=56.0)
    for t in range(30):
        mu = (rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), rng.uniform(1.5, 4.0))
        s = np.exp(rng.uniform(np.log(0.02), np.log(0.4), 3))
        sc = one_gaussian(mu, s, q=rng.standard_normal(4))
        orc = O.Oracle(sc).set_view(cam, k=0.3)
        M, muv, _, _ = filtered_T_view(sc, 0, cam)
        Minv = np.linalg.inv(M)
        px, py = cam.fx * muv[0] / muv[2] + cam.cx + rng.uniform(-3, 3), cam.fy * muv[1] / muv[2] + cam.cy + rng.uniform(-3, 3)
        ix, iy = int(px), int(py)
        c = _contrib_of(orc, ix, iy)
        if c is None:
            continue
        r = np.array([(ix + 0.5 - cam.cx) / cam.fx, (iy + 0.5 - cam.cy) / cam.fy, 1.0])
        f = lambda z: float(np.sum((Minv @ (z * r - muv)) ** 2))   # |u(z)|^2, Gaussian space
        zs = np.linspace(0.01, 10.0, 20001)
        vals = np.array([f(z) for z in zs])
        k = int(np.argmin(vals))
        a, b = zs[max(k - 1, 0)], zs[min(k + 1, len(zs) - 1)]
        gr = (math.sqrt(5) - 1) / 2
        for _ in range(200):
            c1, c2 = b - gr * (b - a), a + gr * (b - a)
            if f(c1) < f(c2):
                b = c2
            else:
                a = c1
        zstar = 0.5 * (a + b)
        assert c[CI["z"]] == pytest.approx(zstar, rel=1e-6)
        assert c[CI["rho2"]] == pytest.approx(f(zstar), rel=1e-9, abs=1e-12)
        # ray integral over z of the unit-space density vs closed form with |w|^2 = |M^-1 r|^2
        zz = np.linspace(zstar - 5, zstar + 5, 200001)
        dens = np.exp(-0.5 * np.sum(((Minv @ (np.outer(r, zz) - muv[:, None])) ** 2), axis=0))
        integral = np.trapezoid(dens, zz)
        w2 = float(np.sum((Minv @ r) ** 2))
        assert integral == pytest.approx(math.exp(-0.5 * c[CI["rho2"]]) * math.sqrt(2 * math.pi / w2), rel=1e-6)


def test_isotropic_rho2_is_point_line_distance():
    """Isotropic sigma_hat: rho^2 = dist^2(mu, ray) / sigma_hat^2."""
    cam = pinhole()
    sc = one_gaussian((0.1, -0.05, 2.0), (0.1, 0.1, 0.1), q=(0.3, 0.2, -0.5, 0.7))
    orc = O.Oracle(sc).set_view(cam, k=0.3)
    shat = orc.gaussians()[0, FI["shat0"]]
    mu = sc.means[0].astype(np.float64)
    for px, py in [(34, 30), (36, 31), (40, 28), (33, 33)]:
        c = _contrib_of(orc, px, py)
        r = np.array([(px + 0.5 - 32) / 56.0, (py + 0.5 - 32) / 56.0, 1.0])
        d2 = mu @ mu - (mu @ r) ** 2 / (r @ r)
        assert c[CI["rho2"]] == pytest.approx(d2 / shat, rel=1e-10)


def test_single_gaussian_peak_alpha_and_colour():
    """Pixel at the projected mean of an on-axis Gaussian: rho^2 = 0, alpha = min(0.99, oA),
    colour = alpha c + (1-alpha) bg."""
    cam = pinhole(W=65, H=65, f=56.0)            # pixel 32's centre is the principal point 32.5
    for o in (0.5, 0.999):
        sc = one_gaussian((0, 0, 2.0), (0.05, 0.08, 0.02), o=o, rgb=(0.2, 0.4, 0.8))
        orc = O.Oracle(sc).set_view(cam, k=0.3, bg=(0.1, 0.2, 0.3))
        oA = orc.gaussians()[0, FI["oA"]]
        rgbT, flags, nb = orc.render_pixels([32], [32])
        a = min(0.99, oA)
        np.testing.assert_allclose(rgbT[0, :3], a * np.array([0.2, 0.4, 0.8]) + (1 - a) * np.array([0.1, 0.2, 0.3]), rtol=1e-6)
        assert rgbT[0, 3] == pytest.approx(1 - a, rel=1e-12)


def test_empty_scene_is_background():
    sc = S.Scene(np.zeros((0, 3), np.float32), np.zeros((0, 3), np.float32), np.zeros((0, 4), np.float32),
                 np.zeros(0, np.float32), np.zeros((0, 1, 3), np.float32), np.zeros(0, np.float32), 0)
    orc = O.Oracle(sc).set_view(pinhole(W=8, H=8), bg=(0.25, 0.5, 0.75))
    img, fl, nb = orc.render_image()
    np.testing.assert_array_equal(img[..., :3], np.broadcast_to([0.25, 0.5, 0.75], (8, 8, 3)))
    np.testing.assert_array_equal(img[..., 3], 1.0)


def test_permutation_invariance_and_T_range():
    """Input order does not change the image; T in [0,1]."""
    sc = _rand_scene(21, 300)
    perm = np.random.default_rng(0).permutation(sc.n)
    a = O.Oracle(sc).set_view(pinhole()).render_image()[0]
    b = O.Oracle(sc.subset(perm)).set_view(pinhole()).render_image()[0]
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)
    assert a[..., 3].min() >= 0 and a[..., 3].max() <= 1


def test_exact_rejects_are_bit_identical():
    """Tile sphere-vs-cone + ray sphere-vs-line rejects change nothing."""
    for sc, cam in [(S.c1_scene(), S.c1_camera()), (_rand_scene(31, 3000, deg=3, box=((-3, 3), (-3, 3), (-1, 6))), pinhole(W=80, H=48, f=40.0))]:
        orc = O.Oracle(sc).set_view(cam)
        a, fa, na = orc.render_image(use_rejects=True)
        b, fb, nb = orc.render_image(use_rejects=False)
        np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(fa, fb)
        assert na.max() > 0


def test_rotation_roll_90():
    """90 deg roll about the optical axis of a square, centred camera permutes pixels."""
    sc = _rand_scene(41, 200)
    cam = pinhole(W=48, H=48, f=40.0)
    Rz = np.eye(4)
    Rz[:2, :2] = [[0, -1], [1, 0]]               # view' = Rz view: (x,y) -> (-y, x)
    cam2 = pinhole(W=48, H=48, f=40.0, V=Rz)
    a = O.Oracle(sc).set_view(cam).render_image()[0]
    b = O.Oracle(sc).set_view(cam2).render_image()[0]
    # pixel (i, j) of cam2 sees the ray of cam pixel (j', i') with x' = -y: a[yy, xx] == b[xx, W-1-yy]
    H = W = 48
    for y in range(H):
        for x in range(W):
            np.testing.assert_allclose(b[x, W - 1 - y], a[y, x], atol=1e-9)


def test_fov_crop_equality():
    """The large-FOV protocol as a pixel-exact cut-out (reading 33): rendering
    (3W, 3H, f, c + (W,H)) and cropping the centre equals the base render."""
    sc = _rand_scene(51, 400, box=((-2, 2), (-2, 2), (-0.5, 4.0)))
    base = pinhole(W=32, H=24, f=30.0)
    wide = pinhole(W=96, H=72, f=30.0, cx=16.0 + 32, cy=12.0 + 24)
    a = O.Oracle(sc).set_view(base).render_image()[0]
    b = O.Oracle(sc).set_view(wide).render_image()[0]
    np.testing.assert_allclose(b[24:48, 32:64], a, atol=1e-12)


# ---------------------------------------------------------------- culling (Eq. 18)
def test_qp_against_brute_force():
    """Active-set QP == fine-grid + local polish minimum of |u|^2 over the polyhedron."""
    from scipy.optimize import minimize
    rng = np.random.default_rng(61)
    for t in range(40):
        nc = rng.integers(1, 6)
        a = rng.standard_normal((nc, 3))
        b = rng.standard_normal(nc) * 2
        val = O.qp_min_norm(a, b)
        cons = [{"type": "ineq", "fun": (lambda u, k=k: a[k] @ u + b[k])} for k in range(nc)]
        best = np.inf
        for s in range(8):
            r = minimize(lambda u: u @ u, rng.standard_normal(3) * 3, constraints=cons, method="SLSQP",
                         options={"ftol": 1e-14, "maxiter": 500})
            if r.success and np.all(a @ r.x + b >= -1e-9):
                best = min(best, r.fun)
        assert val == pytest.approx(best, rel=1e-6, abs=1e-9)


def _naive_4plane_4edge(M, muv, cam, rect):
    """The paper's naive search, written independently: mean-inside trivial case
    (P:317), closest point to the origin on each of the 4 side planes and 4 side edges
    (pulled back by T_view^T, Eq. 5), admissible if inside the other planes and in front."""
    x0, x1, y0, y1 = rect
    planes = [np.array([cam.fx, 0, cam.cx - x0, 0.0]), np.array([-cam.fx, 0, x1 - cam.cx, 0.0]),
              np.array([0, cam.fy, cam.cy - y0, 0.0]), np.array([0, -cam.fy, y1 - cam.cy, 0.0])]
    T = np.eye(4)
    T[:3, :3] = M
    T[:3, 3] = muv
    pl = [T.T @ p for p in planes]
    def ok(u):
        x = T @ np.append(u, 1)
        return x[2] > 0 and all(p @ np.append(u, 1) >= -1e-9 * (np.linalg.norm(p[:3]) * np.linalg.norm(u) + abs(p[3])) for p in pl)
    if ok(np.zeros(3)):
        return 0.0
    best = np.inf
    for p in pl:
        u = -p[3] * p[:3] / (p[:3] @ p[:3])
        if ok(u):
            best = min(best, u @ u)
    for i, j in [(0, 2), (0, 3), (1, 2), (1, 3)]:
        A = np.stack([pl[i][:3], pl[j][:3]])
        u = A.T @ np.linalg.solve(A @ A.T, -np.array([pl[i][3], pl[j][3]]))
        if ok(u):
            best = min(best, u @ u)
    return best


def test_frustum_qp_equals_paper_naive_search_in_front():
    """For Gaussians whose ellipsoid lies beyond near, the oracle's 5-constraint QP
    equals the paper's naive 4-plane/4-edge search."""
    rng = np.random.default_rng(71)
    cam = pinhole(W=256, H=256, f=200.0)
    sc = _rand_scene(72, 400, box=((-2, 2), (-2, 2), (1.0, 6.0)))
    orc = O.Oracle(sc).set_view(cam)
    G = orc.gaussians()
    gs, rects, naive = [], [], []
    for g in range(sc.n):
        M, muv, shat, _ = filtered_T_view(sc, g, cam)
        tau = G[g, FI["tau"]]
        if not tau > 0 or muv[2] - math.sqrt(tau * (M[2] @ M[2])) <= 2 * cam.near:
            continue
        mx = cam.fx * muv[0] / muv[2] + cam.cx
        my = cam.fy * muv[1] / muv[2] + cam.cy
        for _ in range(3):
            tx = int(np.clip(mx // 16 + rng.integers(-2, 3), 0, 15))
            ty = int(np.clip(my // 16 + rng.integers(-2, 3), 0, 15))
            rect = (16 * tx + 0.5, 16 * tx + 15.5, 16 * ty + 0.5, 16 * ty + 15.5)
            gs.append(g)
            rects.append(rect)
            naive.append(_naive_4plane_4edge(M, muv, cam, rect))
    qp = orc.frustum_min_rho2(gs, rects)
    naive = np.asarray(naive)
    tau = G[np.asarray(gs), FI["tau"]]
    # decisions agree everywhere; values agree wherever the minimum is within 4 tau (E3's band;
    # far above tau the true minimiser can sit on the near plane, which P:320 does not search)
    np.testing.assert_array_equal(qp < tau, naive < tau)
    m = qp < 4 * tau
    np.testing.assert_allclose(qp[m], naive[m], rtol=1e-9, atol=1e-12)
    assert len(gs) > 600 and m.sum() > 100 and (qp < tau).sum() > 20


def test_frustum_qp_sound_against_dense_rays():
    """Soundness: the min of rho^2 over sampled pixel rays of a tile (with the
    per-ray max-response point in front of near) is never below the QP minimum, and for
    kept tiles a sampled ray gets close to it."""
    rng = np.random.default_rng(81)
    cam = pinhole(W=128, H=128, f=100.0)
    sc = _rand_scene(82, 150, box=((-1.5, 1.5), (-1.5, 1.5), (-0.5, 3.0)))
    orc = O.Oracle(sc).set_view(cam)
    G = orc.gaussians()
    for g in range(sc.n):
        if not G[g, FI["valid"]]:
            continue
        M, muv, _, _ = filtered_T_view(sc, g, cam)
        Minv = np.linalg.inv(M)
        tx, ty = rng.integers(0, 8, 2)
        rect = (16 * tx + 0.5, 16 * tx + 15.5, 16 * ty + 0.5, 16 * ty + 15.5)
        qp = orc.frustum_min_rho2([g], [rect])[0]
        xs = np.linspace(rect[0], rect[1], 31)
        ys = np.linspace(rect[2], rect[3], 31)
        X, Y = np.meshgrid(xs, ys)
        r = np.stack([(X.ravel() - cam.cx) / cam.fx, (Y.ravel() - cam.cy) / cam.fy, np.ones(X.size)])
        w = Minv @ r
        c = -Minv @ muv
        t = -(c @ w) / np.sum(w * w, axis=0)
        t = np.maximum(t, cam.near)               # best point of each ray inside z >= near
        u = c[:, None] + t * w
        dense = np.min(np.sum(u * u, axis=0))
        assert dense >= qp * (1 - 1e-9) - 1e-12
        if qp < G[g, FI["tau"]] and qp > 0:
            assert dense <= qp * 1.2 + 0.05


def test_frustum_trivial_cases():
    """Mean inside the tile frustum -> 0; 20 sigma outside -> far above tau."""
    cam = pinhole(W=64, H=64, f=56.0)
    sc = one_gaussian((0.0, 0.0, 2.0), (0.01, 0.01, 0.01))
    orc = O.Oracle(sc).set_view(cam, k=0.0)
    assert orc.frustum_min_rho2([0], [(16.5, 47.5, 16.5, 47.5)])[0] == 0.0
    far = orc.frustum_min_rho2([0], [(48.5, 63.5, 48.5, 63.5)])[0]
    # closest tile ray x=48.5 at depth 2: lateral offset (48.5-32)/56*2 = 0.589 -> rho^2 ~ (0.589/0.01)^2 * cos^2
    assert far > 1000


def test_global_order_mode_equals_resorted_exact_contributions():
    """order_mode 1 (Table 5 "w/o hier. sort"): the blend order is the depth code of each
    Gaussian's view-space mean, then the index. Checked against the exact-mode contribution list
    re-sorted in numpy by codes computed here from the scene and the camera."""
    scene, cams = S.make_config("c1")
    cam = cams[0]
    kp = dict(order_mode=1, order_scale=2.0 ** 28 / 24.0, order_near=0.0099999, order_qmax=float(2 ** 28 - 1))
    orc1 = O.Oracle(scene).set_view(cam, **kp)
    orc0 = O.Oracle(scene).set_view(cam)
    W = np.asarray(cam.world_to_view, dtype=np.float64).reshape(4, 4)
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    muz = f32(W[2, :3]) @ scene.means.astype(np.float64).T + float(np.float32(W[2, 3]))
    u = kp["order_scale"] * np.log2(np.maximum(muz, kp["order_near"]) / kp["order_near"])
    code = np.floor(np.clip(u, 0, kp["order_qmax"]))
    CI = {f: i for i, f in enumerate(O.C_FIELDS)}
    rng = np.random.default_rng(5)
    n_diff = 0
    for px, py in zip(rng.integers(0, cam.width, 300), rng.integers(0, cam.height, 300)):
        c = orc0.pixel_contribs(int(px), int(py))
        inc = c[c[:, CI["included"]] > 0.5]
        g = inc[:, CI["g"]].astype(np.int64)
        order = np.lexsort((g, code[g]))
        T, C = 1.0, np.zeros(3)
        for k in order:
            a = inc[k, CI["alpha"]]
            if T * (1 - a) < 1e-4:
                break
            C += a * inc[k, CI["r"]:CI["b"] + 1] * T
            T *= 1 - a
        ref, _, _ = orc1.render_pixels(np.array([px]), np.array([py]))
        np.testing.assert_allclose(ref[0], [*C, T], rtol=0, atol=1e-12)
        n_diff += int(not np.array_equal(order, np.argsort(inc[:, CI["z"]], kind="stable")))
    assert n_diff > 0  # the two orders differ on some pixels of c1


def test_vtrain_spec_examples():
    """Eq. 6 and SPEC S:151-159 worked examples: one camera, f = 800, mean at depth 4
    on screen -> 200; cameras at depths 4 and 2 both seeing the mean -> 400; empty list -> +inf
    (S:192); a camera that does not see the mean (behind / off screen) does not count."""
    sc = one_gaussian((0.0, 0.0, 0.0), (0.1, 0.1, 0.1))
    orc = O.Oracle(sc)

    def cam_at(depth, W=800, H=600, f=800.0, shift=0.0):
        V = np.eye(4)
        V[2, 3] = depth           # world origin at view depth `depth`
        V[0, 3] = shift           # lateral offset in view space
        return pinhole(W, H, f, V)
    v, amb = orc.vtrain([cam_at(4.0)])
    assert v[0] == 200.0 and not amb[0]
    v, _ = orc.vtrain([cam_at(4.0), cam_at(2.0)])
    assert v[0] == 400.0
    v, _ = orc.vtrain([])
    assert np.isinf(v[0])
    v, _ = orc.vtrain([cam_at(-1.0), cam_at(4.0, shift=10.0)])   # behind; projects to x = 2400 > W
    assert np.isinf(v[0])
    v, _ = orc.vtrain([cam_at(4.0, f=600.0), cam_at(8.0, W=1600, f=1600.0)])
    assert v[0] == 200.0   # max(600/4, 1600/8)
    # anamorphic: f = max(fx, fy) (reading 10)
    c = cam_at(4.0)
    c = S.Camera(c.width, c.height, 800.0, 1200.0, c.cx, c.cy, c.world_to_view, c.near)
    v, _ = orc.vtrain([c])
    assert v[0] == 300.0


def test_vtrain_brute_force_on_c1():
    """orc_vtrain against a direct numpy evaluation of the same definition on c1 x 3 cameras."""
    scene, cams = S.make_config("c1")
    cl = [cams[0], cams[0].scaled(fx=40.0, fy=40.0), pinhole(64, 64, 56.0, np.diag([1.0, 1.0, 1.0, 1.0]) @ np.eye(4))]
    orc = O.Oracle(scene)
    v, amb = orc.vtrain(cl)
    mu = scene.means.astype(np.float64)
    best = np.full(len(mu), -np.inf)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    for c in cl:
        M = f32(np.asarray(c.world_to_view, np.float64))
        p = mu @ M[:3, :3].T + M[:3, 3]
        z = p[:, 2]
        with np.errstate(divide="ignore", invalid="ignore"):
            px = float(np.float32(c.fx)) * p[:, 0] / z + float(np.float32(c.cx))
            py = float(np.float32(c.fy)) * p[:, 1] / z + float(np.float32(c.cy))
        ok = (z >= float(np.float32(c.near))) & (px >= 0.5) & (px <= c.width - 0.5) & (py >= 0.5) & (py <= c.height - 0.5)
        best = np.where(ok, np.maximum(best, max(float(np.float32(c.fx)), float(np.float32(c.fy))) / np.where(ok, z, 1)), best)
    want = np.where(best > 0, best, np.inf)
    m = ~amb
    np.testing.assert_allclose(v[m], want[m], rtol=1e-14)
    assert np.isfinite(v).sum() > 10 and np.isinf(v).sum() > 0


def test_2d_splat_mode_closed_form_and_jacobian():
    """eval_mode 1 (Table 5 "w/o 3D"): rho^2 = d^T (J Sigma_v J^T)^-1 d with J the Jacobian
    of the pinhole projection at the mean. (a) On-axis isotropic Gaussian: rho^2 = z^2 |d|^2 /
    (f sigma)^2 in closed form. (b) An anisotropic off-axis Gaussian: J by central differences of
    the projection x -> (fx X/Z + cx, fy Y/Z + cy) in numpy."""
    cfg = dict(order_mode=1, order_scale=1.0, order_near=0.01, order_qmax=0.0, eval_mode=1, k=0.0)
    cam = pinhole(64, 64, 56.0)
    sig, z = 0.3, 3.0
    sc = one_gaussian((0.0, 0.0, z), (sig, sig, sig), o=0.8)
    orc = O.Oracle(sc).set_view(cam, **cfg)
    CI = {f: i for i, f in enumerate(O.C_FIELDS)}
    for px, py in ((32, 32), (36, 30), (40, 41)):
        c = orc.pixel_contribs(px, py)
        d = np.array([px + 0.5 - 32.0, py + 0.5 - 32.0])
        s32, z32 = float(np.float32(sig)), float(np.float32(z))
        want = z32 * z32 * (d @ d) / (56.0 * s32) ** 2
        assert c.shape[0] == 1
        np.testing.assert_allclose(c[0, CI["rho2"]], want, rtol=1e-12)
    # (b)
    q = np.array([0.9, 0.2, -0.3, 0.25]); q /= np.linalg.norm(q)
    mu, s = np.array([0.4, -0.3, 2.5]), np.array([0.25, 0.05, 0.12])
    sc = one_gaussian(tuple(mu), tuple(s), q=tuple(q), o=0.9)
    orc = O.Oracle(sc).set_view(cam, **cfg)
    mu32 = sc.means[0].astype(np.float64)
    qq = sc.quats[0].astype(np.float64); qq /= np.linalg.norm(qq)
    w, x, y, zq = qq
    R = np.array([[1 - 2 * (y * y + zq * zq), 2 * (x * y - w * zq), 2 * (x * zq + w * y)],
                  [2 * (x * y + w * zq), 1 - 2 * (x * x + zq * zq), 2 * (y * zq - w * x)],
                  [2 * (x * zq - w * y), 2 * (y * zq + w * x), 1 - 2 * (x * x + y * y)]])
    Sv = R @ np.diag(sc.scales[0].astype(np.float64) ** 2) @ R.T
    proj = lambda p: np.array([56.0 * p[0] / p[2] + 32.0, 56.0 * p[1] / p[2] + 32.0])
    h = 1e-6
    Jn = np.stack([(proj(mu32 + h * e) - proj(mu32 - h * e)) / (2 * h) for e in np.eye(3)], 1)
    C2 = np.linalg.inv(Jn @ Sv @ Jn.T)
    pm = proj(mu32)
    n_hit = 0
    for px in range(40, 56, 3):
        for py in range(10, 40, 3):
            c = orc.pixel_contribs(px, py)
            d = np.array([px + 0.5, py + 0.5]) - pm
            want = d @ C2 @ d
            if c.shape[0]:
                np.testing.assert_allclose(c[0, CI["rho2"]], want, rtol=1e-6)
                n_hit += 1
            else:
                assert want > orc.gaussians()[0, O.G_FIELDS.index("tau")] - 1e-3
    assert n_hit > 3


# ---------------------------------------------------------------- camera-inside and tau level set
def _alpha_level_rho2(oA):
    """The rho^2 at which alpha(rho^2) = oA exp(-rho^2/2) (Eq. 9 with amplitude A) falls to 1/255
    (reading 1: the tau-ellipsoid is the alpha >= 1/255 level set), found by bisection on the
    alpha curve itself — not the closed form."""
    lo, hi = 0.0, 200.0
    for _ in range(200):
        m = 0.5 * (lo + hi)
        if oA * math.exp(-0.5 * m) >= 1.0 / 255.0:
            lo = m
        else:
            hi = m
    return 0.5 * (lo + hi)


def test_camera_inside_discard_on_filtered_ellipsoid():
    """P:292 (reading 8): a Gaussian whose FILTERED tau-ellipsoid contains the camera is discarded.
    The camera is put at Mahalanobis distance (1 -/+ 2%) of the level set along a random ray: with
    v' = v_train (the camera is close, so v_hat > v_train) Sigma_hat and A do not change along the
    ray, and the camera's Gaussian-space point is lambda M^-1 dir (M from helpers.filtered_T_view,
    the paper's T_view with filtered scales). Just inside -> discarded (background image);
    just outside -> kept. Fails if the oracle tested Sigma instead of Sigma_hat, or dropped the 2 of
    tau (both checked once by mutation)."""
    rng = np.random.default_rng(77)
    cam = pinhole(W=32, H=32, f=56.0)
    n_in = n_out = 0
    for trial in range(40):
        s = np.exp(rng.uniform(np.log(0.03), np.log(0.3), 3))
        q = rng.standard_normal(4)
        d = rng.standard_normal(3)
        d[2] = abs(d[2]) + 0.5
        d /= np.linalg.norm(d)
        o = rng.uniform(0.3, 0.95)
        probe = one_gaussian(d, s, q=q, o=o, v_train=3.0)
        M, muv, shat, R = filtered_T_view(probe, 0, cam)
        assert 56.0 / muv[2] > 3.0 and np.isclose(shat[0], s[0] ** 2 + 0.3 / 9.0)  # v' = v_train
        A = eq12_amplitude(s, shat, R, d)
        lam_star = math.sqrt(_alpha_level_rho2(o * A)) / np.linalg.norm(np.linalg.solve(M, d))
        for fac, inside in ((0.98, True), (1.02, False)):
            mu = fac * lam_star * d
            sc = one_gaussian(mu, s, q=q, o=o, v_train=3.0)
            M2, muv2, shat2, _ = filtered_T_view(sc, 0, cam)
            if 56.0 / muv2[2] <= 3.0:
                continue  # filter would depend on the distance; keep the construction exact
            orc = O.Oracle(sc).set_view(cam)
            G = orc.gaussians()[0]
            assert bool(G[FI["inside"]]) == inside, (trial, fac, G[FI["inside_rho2"]], G[FI["tau"]])
            assert bool(G[FI["valid"]]) == (not inside)
            if inside:
                img = orc.render_image()[0]
                np.testing.assert_array_equal(img[..., 3], 1.0)
                n_in += 1
            else:
                n_out += 1
    assert n_in >= 20 and n_out >= 20


def test_tau_level_set_per_pixel():
    """P:276/P:312 with reading 1: a pixel receives a contribution iff alpha = o A exp(-rho^2/2)
    >= 1/255, rho^2 from the paper's plane pullback (Eq. 4-5, helpers.plane_form_rho2) and A from
    Eq. 12 (helpers.eq12_amplitude). Pixels straddle the boundary on both sides; a pixel counts as
    receiving a contribution iff its transmittance drops below 1. Fails if tau loses its factor 2
    or uses o instead of o A (checked once by mutation)."""
    rng = np.random.default_rng(5)
    cam = pinhole(W=96, H=96, f=120.0)
    n_straddle_in = n_straddle_out = 0
    for trial in range(6):
        s = np.exp(rng.uniform(np.log(0.05), np.log(0.25), 3))
        q = rng.standard_normal(4)
        mu = np.array([rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), rng.uniform(2.5, 4.0)])
        o = rng.uniform(0.4, 0.95)
        sc = one_gaussian(mu, s, q=q, o=o, v_train=8.0)
        M, muv, shat, R = filtered_T_view(sc, 0, cam)
        A = eq12_amplitude(s, shat, R, mu / np.linalg.norm(mu))
        assert A < 0.97  # the filter is active, so o and o A differ
        orc = O.Oracle(sc).set_view(cam)
        yy, xx = np.mgrid[0:cam.height, 0:cam.width]
        rgbT = orc.render_pixels(xx.ravel(), yy.ravel())[0]
        for idx in range(xx.size):
            px, py = xx.ravel()[idx], yy.ravel()[idx]
            rho2, z = plane_form_rho2(M, muv, cam, px + 0.5, py + 0.5)
            a = o * A * math.exp(-0.5 * rho2)
            margin = a * 255.0 - 1.0
            if abs(margin) < 1e-9:
                continue
            hit = rgbT[idx, 3] < 1.0
            assert hit == (margin > 0), (trial, px, py, rho2, a)
            if abs(margin) < 0.5:
                n_straddle_in += margin > 0
                n_straddle_out += margin < 0
    assert n_straddle_in >= 50 and n_straddle_out >= 50


def test_camera_is_the_given_affine_map():
    """Reading 37: the camera is the world->view map x_v = Rv x + t exactly as given. With a
    rotation block that is deliberately not orthonormal (a row scaled by 1 + 1e-4, far beyond the
    ~1e-7 of a float32-rounded matrix) the oracle's z* and rho^2 at a pixel still equal the paper's
    plane pullback through T' = M_vp P V T (helpers.plane_form_rho2, forward map only): the camera
    centre and the pixel rays use Rv^-1, not Rv^T."""
    rng = np.random.default_rng(37)
    V = np.eye(4)
    ang = 0.3
    V[:3, :3] = np.array([[np.cos(ang), 0, np.sin(ang)], [0, 1, 0], [-np.sin(ang), 0, np.cos(ang)]])
    V[0, :3] *= 1 + 1e-4
    V[:3, 3] = [0.4, -0.2, 2.5]
    V = V.astype(np.float32).astype(np.float64)
    cam = pinhole(W=48, H=48, f=60.0, V=V, near=0.01)
    for _ in range(5):
        mu = rng.uniform(-0.5, 0.5, 3) + np.array([-1.2, 0.2, 0.8])
        sc = one_gaussian(mu, rng.uniform(0.05, 0.2, 3), q=rng.standard_normal(4), o=0.9, v_train=20.0)
        M, muv, _, _ = filtered_T_view(sc, 0, cam)
        orc = O.Oracle(sc).set_view(cam)
        c = orc.pixel_contribs(24, 24)
        rows = c[c[:, CI["included"]] > 0.5]
        if not len(rows):
            continue
        rho2, z = plane_form_rho2(M, muv, cam, 24.5, 24.5)
        assert rows[0, CI["z"]] == pytest.approx(z, rel=1e-10)
        assert rows[0, CI["rho2"]] == pytest.approx(rho2, rel=1e-8, abs=1e-10)
