"""Offline analysis of a tools/dump_view.py dump against the oracle: finds failing pixels and,
for each, replays the K6 per-pixel algorithm in float32 numpy from the dumped raster records,
listing where the GPU's contribution set or order departs from the oracle's. Diagnostic tool."""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import oracle as O  # noqa: E402
from synth import scenes as S  # noqa: E402

CI = {f: i for i, f in enumerate(O.C_FIELDS)}
f32 = np.float32


def eval_fp32(r, px, py, near):
    r = r.astype(np.float32)
    dx = f32(px + 0.5) - r[0]
    dy = f32(py + 0.5) - r[1]
    F0, E1, E2 = r[4:7], r[7:10], r[10:13]
    wref, a, b = r[13:16], r[16:19], r[19:22]
    cw0, ca, cb = r[22], r[23], r[24]
    v = F0 + dx * E1 + dy * E2
    w = wref + dx * a + dy * b
    cw = cw0 + dx * ca + dy * cb
    N = np.sum(v * v, dtype=np.float32)
    Q = np.sum(w * w, dtype=np.float32)
    rho2 = N / Q
    z = -cw / Q
    hit = rho2 < r[3] and z >= near
    alpha = min(f32(0.99), r[2] * np.exp(f32(-0.5) * rho2))
    return float(rho2), float(z), float(alpha), bool(hit)


def replay(d, px, py, tiles_x, near, K=32):
    tile = (py // 16) * tiles_x + px // 16
    s, e = d["ranges"][tile]
    sub = ((px % 16) // 8) + 2 * ((py % 16) // 4)
    out = []
    for j in range(s, e):
        v = int(d["vals"][j])
        g = v & 0xFFFFFF
        if not (v >> (24 + sub)) & 1:
            continue
        wm = 0.0  # watermarks are not needed by the offline replay of contributions
        rho2, z, a, hit = eval_fp32(d["raster"][g], px, py, near)
        out.append((j, g, float(wm), rho2, z, a, hit))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dump")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--scale3", action="store_true")
    ap.add_argument("--show", type=int, default=5)
    a = ap.parse_args()
    d = dict(np.load(a.dump))
    scene, cams = S.make_config(a.config)
    cam = cams[a.view]
    if a.scale3:
        cam = cam.scaled(width=3 * cam.width, height=3 * cam.height, cx=cam.cx + cam.width, cy=cam.cy + cam.height)
    orc = O.Oracle(scene).set_view(cam)
    img = d["img"]
    H, W = img.shape[1:]
    print("stats", d["stats"])
    yy, xx = np.mgrid[0:H, 0:W]
    ref, flags, nb = orc.render_pixels(xx.ravel(), yy.ravel())
    gpu = img.reshape(4, -1).T
    err = np.abs(gpu[:, :3] - ref[:, :3]).max(axis=1)
    bad = np.argsort(-err)
    print(f"max err {err.max():.3e}; > 5e-4: {(err > 5e-4).sum()} of {err.size}; flagged among them "
          f"{(flags[err > 5e-4] != 0).sum()}")
    badmap = (err > 5e-4).reshape(H, W)
    ys, xs = np.nonzero(badmap)
    print("bad pixel tiles (first 20):", sorted(set(zip((xs // 16).tolist(), (ys // 16).tolist())))[:20])
    tiles_x = (W + 15) // 16
    for k in bad[: a.show]:
        px, py = int(xx.ravel()[k]), int(yy.ravel()[k])
        print(f"\n=== pixel ({px},{py}) gpu {gpu[k]} oracle {ref[k]} flags {flags[k]}")
        c = orc.pixel_contribs(px, py)
        inc = c[c[:, CI["included"]] > 0.5]
        rp = {g: (rho2, z, al, hit, j, wm) for (j, g, wm, rho2, z, al, hit) in replay(d, px, py, tiles_x, cam.near)}
        G = d["gauss"]
        for row in inc[:40]:
            g = int(row[CI["g"]])
            gp = rp.get(g)
            vis = G[g, 14]
            print(f"  g={g:7d} z={row[0]:.6f} a={row[1]:.4f} rho2={row[2]:.4f} tau={row[3]:.3f} | gpu: "
                  + (f"rho2={gp[0]:.4f} z={gp[1]:.6f} a={gp[2]:.4f} hit={gp[3]} key={gp[5]:.6f}" if gp else
                     f"NOT IN LIST (visible={vis}, rect={G[g,16:20]})"))
        extra = [g for g, v in rp.items() if v[3] and g not in set(inc[:, CI["g"]].astype(int).tolist())]
        print("  gpu hits not in oracle:", extra[:10])


if __name__ == "__main__":
    main()
