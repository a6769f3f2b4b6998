"""GPU parity at the full BASELINE sizes on the paths that break (VERDICT r01 'What's weak' 1):

* culling: every candidate (Gaussian, rect tile) pair of one view each of c3, c4wide, c4zoomout,
  c4inside (the landing views 48/49: camera inside ground surfels, every visible Gaussian crossing
  the near plane) decided by the oracle's exact frustum QP (readings 20-22) — exact
  outside the 1e-5 band; c5: every crossing Gaussian x all its rect tiles plus all candidates of a
  random 5% of the tiles. The 8x4 sub-tile masks are checked against the same QP on each
  sub-rectangle for a sample of kept pairs;
* sort: bit-exact against a stable sort of the emitted pairs on c4 x 3 and c5;
* images: targeted pixels — every pixel K6 spilled to K6s, all pixels of the 16 longest-list tiles,
  and pixels in the footprint of every crossing Gaussian — through the ambiguity-aware comparator.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
import paper_2504_12811_b200 as pkg  # noqa: E402
from synth import scenes as S  # noqa: E402
from tests.compare import compare  # noqa: E402

FI = {f: i for i, f in enumerate(O.G_FIELDS)}
DI = {f: i for i, f in enumerate(pkg.DBG_FIELDS)}
def _config(cfg):
    scene, cams = S.make_config(cfg)
    return scene, cams


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_12811_b200 import _build
    _build.build()
    return pkg.Renderer(0)


_loaded = {}


def _load(R, cfg):
    scene, cams = _config(cfg)
    key = "c3" if cfg.startswith("c4") else cfg
    if _loaded.get("key") != key:
        R.load(scene)
        _loaded["key"] = key
    return scene, cams


def _candidates(G, cam, tile_filter=None, gauss_filter=None):
    """All (g, tile) candidates of the visible Gaussians' tile rects (vectorised)."""
    tx = (cam.width + 15) // 16
    vis = np.nonzero(G[:, DI["visible"]] > 0)[0]
    if gauss_filter is not None:
        vis = vis[gauss_filter(vis)]
    x0, y0, x1, y1 = (G[vis, DI[f]].astype(np.int64) for f in ("tx0", "ty0", "tx1", "ty1"))
    w, h = x1 - x0 + 1, y1 - y0 + 1
    cnt = w * h
    g = np.repeat(vis, cnt)
    start = np.repeat(np.cumsum(cnt) - cnt, cnt)
    j = np.arange(cnt.sum()) - start
    wr = np.repeat(w, cnt)
    tile_x = np.repeat(x0, cnt) + j % wr
    tile_y = np.repeat(y0, cnt) + j // wr
    t = tile_y * tx + tile_x
    if tile_filter is not None:
        keep = tile_filter(t)
        g, t, tile_x, tile_y = g[keep], t[keep], tile_x[keep], tile_y[keep]
    return g, t, tile_x, tile_y


def _rects(tile_x, tile_y, cam):
    return np.column_stack([16 * tile_x + 0.5, np.minimum(16 * tile_x + 15.5, cam.width - 0.5),
                            16 * tile_y + 0.5, np.minimum(16 * tile_y + 15.5, cam.height - 0.5)])


def _check_cull(R, scene, cam, tile_frac=None, seed=0):
    R.set_camera(cam)
    G = R.gaussian_records()
    keys, vals = R.keys_vals(sorted_=False)
    orc = O.Oracle(scene).set_view(cam)
    tau = orc.gaussians()[:, FI["tau"]]
    n_tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    kdb = R.key_tile_shift()
    e_tile = (keys >> np.uint32(kdb)).astype(np.int64)
    e_g = (vals & np.uint32(0xFFFFFF)).astype(np.int64)
    e_mask = (vals >> np.uint32(24)).astype(np.int64)
    e_code = e_g * n_tiles + e_tile
    order = np.argsort(e_code)
    e_code, e_mask = e_code[order], e_mask[order]
    assert np.all(np.diff(e_code) > 0)  # no pair emitted twice
    crossing = G[:, DI["crossing"]] > 0
    if tile_frac is None:
        g, t, txx, tyy = _candidates(G, cam)
    else:
        rng = np.random.default_rng(seed)
        chosen = np.zeros(n_tiles, bool)
        chosen[rng.choice(n_tiles, max(1, int(tile_frac * n_tiles)), replace=False)] = True
        g1, t1, x1, y1 = _candidates(G, cam, tile_filter=lambda t: chosen[t])
        g2, t2, x2, y2 = _candidates(G, cam, gauss_filter=lambda v: crossing[v])
        cc = np.unique(np.concatenate([g1 * n_tiles + t1, g2 * n_tiles + t2]))
        g, t = cc // n_tiles, cc % n_tiles
        txx, tyy = t % ((cam.width + 15) // 16), t // ((cam.width + 15) // 16)
    code = g * n_tiles + t
    mn = orc.frustum_min_rho2(g, _rects(txx, tyy, cam))
    band = np.abs(mn - tau[g]) <= 1e-5 * np.maximum(1, tau[g])
    want = mn < tau[g]
    pos = np.searchsorted(e_code, code)
    got = (pos < len(e_code)) & (e_code[np.minimum(pos, len(e_code) - 1)] == code)
    mism = (got != want) & ~band
    assert not mism.any(), (int(mism.sum()), len(g), g[mism][:5], t[mism][:5], mn[mism][:5], tau[g][mism][:5])
    if tile_frac is None:
        assert got.sum() == len(e_code)  # nothing emitted outside the candidate rects
    # whole-view cull of the Gaussians K1 dropped although the oracle keeps them valid:
    # none may reach the screen frustum (sampled)
    Go = orc.gaussians()
    dropped = np.nonzero((Go[:, FI["valid"]] > 0) & (G[:, DI["visible"]] == 0))[0]
    rng0 = np.random.default_rng(seed + 7)
    if len(dropped) > 200000:
        dropped = rng0.choice(dropped, 200000, replace=False)
    if len(dropped):
        full = np.tile([0.5, cam.width - 0.5, 0.5, cam.height - 0.5], (len(dropped), 1))
        dm = orc.frustum_min_rho2(dropped, full)
        dband = np.abs(dm - tau[dropped]) <= 1e-5 * np.maximum(1, tau[dropped])
        assert not ((dm < tau[dropped]) & ~dband).any()
    # 8x4 sub-tile masks (K3): exact per sub-rectangle for tau-ellipsoids beyond near; all bits for
    # crossing Gaussians (the raster kernels evaluate them everywhere)
    kept = np.nonzero(got)[0]
    rng = np.random.default_rng(seed + 1)
    samp = kept[rng.choice(len(kept), min(len(kept), 20000), replace=False)]
    m = e_mask[pos[samp]]
    cr = crossing[g[samp]]
    assert np.all(m[cr] == 0xFF)
    nc = samp[~cr]
    mk = m[~cr]
    tx_ = (cam.width + 15) // 16
    sg, srect, sbit, sidx = [], [], [], []
    for s in range(8):
        spx = 16 * (t[nc] % tx_) + 8 * (s & 1)
        spy = 16 * (t[nc] // tx_) + 4 * (s >> 1)
        ok = (spx + 0.5 <= cam.width - 0.5) & (spy + 0.5 <= cam.height - 0.5)
        sg.append(g[nc][ok])
        srect.append(np.column_stack([spx[ok] + 0.5, np.minimum(spx[ok] + 7.5, cam.width - 0.5),
                                      spy[ok] + 0.5, np.minimum(spy[ok] + 3.5, cam.height - 0.5)]))
        sbit.append((mk[ok] >> s) & 1)
    sg = np.concatenate(sg)
    smn = orc.frustum_min_rho2(sg, np.concatenate(srect))
    sband = np.abs(smn - tau[sg]) <= 1e-5 * np.maximum(1, tau[sg])
    sbit = np.concatenate(sbit).astype(bool)
    smis = (sbit != (smn < tau[sg])) & ~sband
    assert not smis.any(), (int(smis.sum()), len(sg))
    return dict(candidates=len(g), kept=int(got.sum()), band=int(band.sum()), crossing=int(crossing.sum()),
                subtile_checked=len(sg))


@pytest.mark.parametrize("cfg,view", [("c3", 0), ("c4wide", 3), ("c4zoomout", 10), ("c4inside", 48),
                                      ("c4inside", 49)])
def test_cull_matches_oracle_qp_full_size(R, cfg, view):
    scene, cams = _load(R, cfg)
    info = _check_cull(R, scene, cams[view])
    assert info["kept"] > 0, info


def test_cull_matches_oracle_qp_c5(R):
    scene, cams = _load(R, "c5")
    info = _check_cull(R, scene, cams[0], tile_frac=0.05)
    assert info["kept"] > 100000, info


def test_c4inside_landing_exercises_inside_and_crossing(R):
    """the last views have the camera inside >= 1 ellipsoid and >= 1% of
    the visible Gaussians crossing the near plane (the FP64 5-constraint path)."""
    scene, cams = _load(R, "c4inside")
    for v in (48, 49):
        R.set_camera(cams[v])
        G = R.gaussian_records()
        R.render(cams[v], with_T=False)
        st = R.stats()
        assert (G[:, DI["inside"]] > 0).sum() >= 1, v
        assert st["crossing"] >= 0.01 * st["visible"] and st["crossing"] > 0, (v, st)


@pytest.mark.parametrize("cfg,view", [("c4wide", 3), ("c4zoomout", 10), ("c4inside", 49), ("c5", 0)])
def test_sort_bit_exact_full_size(R, cfg, view):
    scene, cams = _load(R, cfg)
    R.render(cams[view], with_T=False)
    ks, vs = R.keys_vals(sorted_=True)
    rng_ = R.ranges()
    ku, vu = R.keys_vals(sorted_=False)
    order = np.argsort(ku, kind="stable")
    assert np.array_equal(ks, ku[order]) and np.array_equal(vs, vu[order])
    tiles = (ks >> np.uint32(R.key_tile_shift())).astype(np.int64)
    starts = np.searchsorted(tiles, np.arange(rng_.shape[0]), "left")
    ends = np.searchsorted(tiles, np.arange(rng_.shape[0]), "right")
    ne = starts != ends
    assert np.array_equal(rng_[ne, 0], starts[ne]) and np.array_equal(rng_[ne, 1], ends[ne])
    assert np.all(rng_[~ne, 0] == rng_[~ne, 1])


def _targeted_pixels(R, G, cam, max_spill=40000, n_long=16, per_cross=64, seed=0):
    rng = np.random.default_rng(seed)
    W, H = cam.width, cam.height
    sp = R.spilled_pixels().astype(np.int64)
    if len(sp) > max_spill:
        sp = rng.choice(sp, max_spill, replace=False)
    rg = R.ranges()
    ln = rg[:, 1].astype(np.int64) - rg[:, 0]
    tx = (W + 15) // 16
    longest = np.argsort(-ln, kind="stable")[:n_long]
    lp = []
    for t in longest:
        yy, xx = np.mgrid[16 * (t // tx): min(16 * (t // tx) + 16, H), 16 * (t % tx): min(16 * (t % tx) + 16, W)]
        lp.append((yy * W + xx).ravel())
    cp = []
    for g in np.nonzero(G[:, DI["crossing"]] > 0)[0]:
        x0, x1 = int(G[g, DI["tx0"]]) * 16, min(int(G[g, DI["tx1"]]) * 16 + 16, W)
        y0, y1 = int(G[g, DI["ty0"]]) * 16, min(int(G[g, DI["ty1"]]) * 16 + 16, H)
        cp.append(rng.integers(y0, y1, per_cross) * W + rng.integers(x0, x1, per_cross))
    parts = dict(spilled=sp, longest_tiles=np.concatenate(lp) if lp else np.zeros(0, np.int64),
                 crossing=np.concatenate(cp) if cp else np.zeros(0, np.int64))
    return parts


@pytest.mark.parametrize("cfg,view", [("c3", 0), ("c4wide", 3), ("c4zoomout", 10), ("c4inside", 48),
                                      ("c4inside", 49), ("c5", 0)])
def test_image_targeted_pixels(R, cfg, view):
    scene, cams = _load(R, cfg)
    cam = cams[view]
    R.set_camera(cam)
    G = R.gaussian_records()
    rgb, T = R.render(cam)
    torch.cuda.synchronize()
    img = torch.cat([rgb, T[None]], 0).permute(1, 2, 0).reshape(-1, 4).cpu().numpy().astype(np.float64)
    st = R.stats()
    assert st["unresolved_pixels"] == 0, st
    parts = _targeted_pixels(R, G, cam, max_spill=20000 if cfg == "c5" else 40000, seed=view)
    orc = O.Oracle(scene).set_view(cam)
    for name, pix in parts.items():
        if len(pix) == 0:
            continue
        pix = np.unique(pix)
        rep = compare(orc, img[pix], pix % cam.width, pix // cam.width)
        assert rep["ok"], (name, rep, st)
    if cfg in ("c3", "c4wide"):
        assert len(parts["spilled"]) > 1000
    if cfg == "c4inside":
        assert len(parts["crossing"]) > 0
