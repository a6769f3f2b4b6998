"""Seeded input generators (synth/): determinism and construction sanity (CPU)."""
import numpy as np

from synth import scenes as S


def test_seeded_determinism():
    a = S.c2_scene(n=5000, n_views_vtrain=5)
    b = S.c2_scene(n=5000, n_views_vtrain=5)
    for f in ("means", "scales", "quats", "opacities", "sh", "v_train"):
        assert getattr(a, f).tobytes() == getattr(b, f).tobytes()


def test_quaternion_roundtrip_and_frames():
    rng = np.random.default_rng(0)
    q = rng.standard_normal((500, 4))
    R = S.quat_to_rotmat(q)
    assert np.allclose(np.einsum("nij,nkj->nik", R, R), np.eye(3), atol=1e-12)
    assert np.allclose(np.linalg.det(R), 1.0)
    assert np.allclose(S.quat_to_rotmat(S.rotmat_to_quat(R)), R, atol=1e-12)


def test_look_at_convention():
    """+z forward, y down: the target projects to the principal point."""
    V = S.look_at([4.0, 0.0, 1.5], [0.0, 0.0, 0.5])
    R = V[:3, :3]
    assert np.allclose(R @ R.T, np.eye(3)) and np.isclose(np.linalg.det(R), 1.0)
    tv = V[:3, :3] @ np.array([0.0, 0.0, 0.5]) + V[:3, 3]
    assert tv[2] > 0 and np.allclose(tv[:2], 0, atol=1e-12)
    up = V[:3, :3] @ np.array([0.0, 0.0, 1.0])
    assert up[1] < 0                       # world up points to -y (image up)


def test_c3_shapes_small():
    s = S.c3_scene(n=20000, vtrain_views=4)
    assert s.means.shape == (20000, 3) and s.sh.shape == (20000, 16, 3)
    assert np.all(s.scales > 0) and np.all((s.opacities > 0) & (s.opacities < 1))
    assert s.means.dtype == np.float32
