"""v_hat_train kernel (Eq. 6, aaa_compute_vtrain) against the oracle, and a PLY
scene through load -> compute_vtrain(store) -> render against the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
import paper_2504_12811_b200 as pkg  # noqa: E402
from paper_2504_12811_b200 import ply  # noqa: E402
from synth import scenes as S  # noqa: E402
from tests.compare import compare  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_12811_b200 import _build
    _build.build()
    return pkg.Renderer(0)


def _img(R, cam):
    rgb, T = R.render(cam)
    torch.cuda.synchronize()
    return torch.cat([rgb, T[None]], 0).permute(1, 2, 0).cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_vtrain_matches_oracle(R, cfg):
    scene, cams = S.make_config(cfg)
    cl = list(cams) + [cams[0].scaled(fx=cams[0].fx * 0.5, fy=cams[0].fy * 0.5)]
    R.load(scene)
    got = R.compute_vtrain(cl).cpu().numpy()
    want, amb = O.Oracle(scene).vtrain(cl)
    want32 = want.astype(np.float32)
    m = ~amb
    assert np.array_equal(got[m], want32[m]), np.nonzero(got[m] != want32[m])[0][:5]
    assert np.isfinite(got).sum() > 0
    e = R.compute_vtrain([]).cpu().numpy()        # no cameras: unbounded
    assert np.all(np.isinf(e))


def test_vtrain_store_drives_the_render(R):
    scene, cams = S.make_config("c2")
    cl = cams[::4]
    R.load(scene)
    vt = R.compute_vtrain(cl, store=True).cpu().numpy()
    a = _img(R, cams[1])
    sc2 = S.Scene(scene.means, scene.scales, scene.quats, scene.opacities, scene.sh, vt, scene.sh_degree)
    R.load(sc2)
    b = _img(R, cams[1])
    assert np.array_equal(a, b)
    assert not np.array_equal(vt, scene.v_train)


def test_ply_scene_renders_like_the_oracle(R, tmp_path):
    scene, cams = S.make_config("c2")
    p = tmp_path / "c2.ply"
    ply.write_ply(p, scene, with_vtrain=False)
    sc = ply.read_ply(p)
    assert np.all(np.isinf(sc.v_train))
    R.load(sc)
    sc.v_train = R.compute_vtrain(cams, store=True).cpu().numpy()
    cam = cams[5]
    img = _img(R, cam)
    orc = O.Oracle(sc).set_view(cam)
    yy, xx = np.mgrid[0:cam.height, 0:cam.width]
    rep = compare(orc, img.reshape(-1, 4), xx.ravel(), yy.ravel())
    assert rep["ok"], rep
