"""Pins of the differentiable float64 reference (oracle/autograd_ref.py) used by the backward
parity tests: its forward equals the C++ oracle's render, and its gradients equal central finite
differences of the C++ oracle's render."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402
from oracle import autograd_ref as AR  # noqa: E402
from synth import scenes as S  # noqa: E402


def _loss_weights(cam, seed=0):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((3, cam.height, cam.width)), rng.standard_normal((cam.height, cam.width))


def _copy(scene):
    return S.Scene(*(np.array(getattr(scene, f), copy=True) for f in
                     ("means", "scales", "quats", "opacities", "sh", "v_train")), scene.sh_degree)


def test_forward_equals_oracle_c1():
    scene, cams = S.make_config("c1")
    cam = cams[0]
    rgb, T = AR.render(AR.params_of(scene, requires_grad=False), scene, cam)
    orc = O.Oracle(scene).set_view(cam)
    yy, xx = np.mgrid[0:cam.height, 0:cam.width]
    ref, flags, _ = orc.render_pixels(xx.ravel(), yy.ravel())
    got = np.concatenate([rgb.detach().numpy().reshape(-1, 3), T.detach().numpy().reshape(-1, 1)], 1)
    np.testing.assert_allclose(got, ref, atol=1e-10)


@pytest.mark.parametrize("field,idx", [("means", (3, 0)), ("means", (10, 2)), ("scales", (5, 1)),
                                       ("quats", (7, 0)), ("quats", (20, 3)), ("opacities", (12,)),
                                       ("sh", (9, 0, 1)), ("means", (30, 1)), ("scales", (41, 2))])
def test_gradient_equals_finite_differences_of_oracle(field, idx):
    scene, cams = S.make_config("c1")
    cam = cams[0]
    wr, wt = _loss_weights(cam)
    g = AR.grads(scene, cam, wr, wt)
    yy, xx = np.mgrid[0:cam.height, 0:cam.width]

    def loss(sc):
        ref, _, _ = O.Oracle(sc).set_view(cam).render_pixels(xx.ravel(), yy.ravel())
        return float((wr.reshape(3, -1).T * ref[:, :3]).sum() + (wt.ravel() * ref[:, 3]).sum())

    x0 = float(getattr(scene, field)[idx])
    h = 2e-5 * max(abs(x0), 1e-2)  # small enough that no contribution crosses tau (no boundary term)
    vals = []
    for sgn in (1, -1):
        sc = _copy(scene)
        a = getattr(sc, field)
        a[idx] = np.float32(x0 + sgn * h)
        vals.append((loss(sc), float(a[idx]) - x0))
    fd = (vals[0][0] - vals[1][0]) / (vals[0][1] - vals[1][1])
    an = g[field][idx]
    assert abs(fd - an) <= 2e-3 * max(1.0, abs(an)), (field, idx, fd, an)
