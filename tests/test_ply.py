"""3DGS PLY IO: activations, layout, round trip, diagnostics."""
import numpy as np
import pytest

from paper_2504_12811_b200 import ply
from synth import scenes as S


def _one(tmp_path, **over):
    sc = ply.PlyScene(np.zeros((1, 3), np.float32), np.ones((1, 3), np.float32),
                      np.array([[1, 0, 0, 0]], np.float32), np.array([0.5], np.float32),
                      np.zeros((1, 1, 3), np.float32), np.array([np.inf], np.float32), 0)
    for k, v in over.items():
        setattr(sc, k, v)
    p = tmp_path / "one.ply"
    ply.write_ply(p, sc)
    return p


def test_activations_spec_examples(tmp_path):
    """stored scale 0 -> scale 1 (exp), stored opacity 0 -> 0.5 (sigmoid)."""
    p = _one(tmp_path)   # write_ply stores log(1) = 0 and logit(0.5) = 0
    raw = open(p, "rb").read()
    assert b"property float scale_0" in raw and b"property float opacity" in raw
    s = ply.read_ply(p)
    assert np.all(s.scales == 1.0) and s.opacities[0] == 0.5
    assert s.sh_degree == 0 and np.isinf(s.v_train[0])


def test_round_trip_c2_sh3(tmp_path):
    scene, _ = S.make_config("c2")
    p = tmp_path / "c2.ply"
    ply.write_ply(p, scene)
    s = ply.read_ply(p)
    assert s.sh_degree == 3 and s.n == scene.n
    np.testing.assert_array_equal(s.means, scene.means)
    np.testing.assert_allclose(s.scales, scene.scales, rtol=1e-6)
    np.testing.assert_allclose(s.opacities, scene.opacities, rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(s.quats, scene.quats / np.linalg.norm(scene.quats, axis=1, keepdims=True), atol=1e-7)
    np.testing.assert_array_equal(s.sh, scene.sh)
    np.testing.assert_array_equal(s.v_train, scene.v_train)


def test_f_rest_is_channel_major(tmp_path):
    """3DGS stores f_rest per channel (R coefficients 1..15, then G, then B)."""
    sh = np.arange(16 * 3, dtype=np.float32).reshape(1, 16, 3)
    p = _one(tmp_path, sh=sh, sh_degree=3)
    hdr = open(p, "rb").read().split(b"end_header")[0].decode()
    names = [ln.split()[-1] for ln in hdr.splitlines() if ln.startswith("property")]
    rest = np.frombuffer(open(p, "rb").read().split(b"end_header\n", 1)[1], dtype="<f4")
    vals = dict(zip(names, rest))
    assert vals["f_rest_0"] == sh[0, 1, 0] and vals["f_rest_15"] == sh[0, 1, 1] and vals["f_rest_44"] == sh[0, 15, 2]
    np.testing.assert_array_equal(ply.read_ply(p).sh, sh)


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b.replace(b"ply\n", b"plx\n", 1), "magic"),
    (lambda b: b.replace(b"binary_little_endian", b"ascii", 1), "unsupported format"),
    (lambda b: b.replace(b"property float rot_3\n", b"", 1), "missing vertex property 'rot_3'"),
    (lambda b: b[:-4], "truncated"),
    (lambda b: b.replace(b"end_header", b"end_headr", 1), "end_header"),
])
def test_malformed_headers_are_diagnosed(tmp_path, mutate, msg):
    p = _one(tmp_path)
    bad = tmp_path / "bad.ply"
    bad.write_bytes(mutate(p.read_bytes()))
    with pytest.raises(ply.PlyError, match=msg):
        ply.read_ply(bad)


def test_missing_property(tmp_path):
    p = _one(tmp_path)
    b = p.read_bytes()
    hdr, body = b.split(b"end_header\n", 1)
    hdr = hdr.replace(b"property float opacity\n", b"property float opacityX\n")
    (tmp_path / "m.ply").write_bytes(hdr + b"end_header\n" + body)
    with pytest.raises(ply.PlyError, match="missing vertex property 'opacity'"):
        ply.read_ply(tmp_path / "m.ply")
