"""OOD sampling-rate regression: rendering at a lower
resolution than the training one, the adaptive 3D filter (k = 0.3) is closer to the alias-free
target (the training-resolution render, box-downsampled) than no filter (k = 0)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2504_12811_b200 as pkg  # noqa: E402
from synth import scenes as S  # noqa: E402
from tools.ood_harness import run  # noqa: E402


def test_filter_reduces_aliasing_when_zooming_out():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    scene, cams = S.make_config("c2")
    R = pkg.Renderer(0)
    out = run(R, scene, cams, [0, 20, 40, 60, 80], factors=(2, 4, 8))
    # measured (tools/ood_harness.py, 5 views): f=2 +1.3 dB, f=4 -0.5 dB, f=8 +2.5 dB.
    # Why f=4 is a wash: at 1/f resolution v_hat' = v_train / f, so the filter adds a variance
    # k / v'^2 = 0.3 px^2 of the LOW-resolution image (sigma 0.55 px, Eq. 12-13) whatever f is, while
    # the alias-free target (a box of f x f training pixels = 1 low-res pixel) needs about
    # 1/12 px^2 (sigma 0.29 px). c2's surfels are ~2.2 training px wide, i.e. 2.2/f low-res px:
    # at f=2 both renders are close to the target (the filter's energy-preserving A wins a
    # little), at f=8 the unfiltered 0.27 px Gaussians alias badly and the filter wins clearly,
    # and at f=4 (0.55 px Gaussians) the filter's over-blur (0.78 vs 0.62 px total) and the
    # unfiltered aliasing cost about the same. The regression asserts all three.
    for f in (2, 8):
        assert out[f]["k0.3"] > out[f]["k0"] + 0.5, out
    assert abs(out[4]["k0.3"] - out[4]["k0"]) < 1.0, out
