"""Diagnose comparator failures around one pixel: render a view on the GPU, compare a window of
pixels with the oracle (ambiguity-aware), and for every failing pixel print the oracle's
contribution list (with ambiguity flags) next to the GPU's own contributions replayed in float32
from the K6 raster records in list order. Diagnostic tool:
    python tools/diag_pixels.py CFG VIEW X Y [RADIUS]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2504_12811_b200 as pkg  # noqa: E402
from paper_2504_12811_b200 import _abi  # noqa: E402
from synth import scenes as S  # noqa: E402
from tests.compare import _best_variant, compare  # noqa: E402
from tools.analyze_dump import eval_fp32  # noqa: E402

CI = {f: i for i, f in enumerate(O.C_FIELDS)}


def main():
    cfg, view, X, Y = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    rad = int(sys.argv[5]) if len(sys.argv) > 5 else 24
    scene, cams = S.make_config(cfg)
    cam = cams[view]
    R = pkg.Renderer(0)
    R.load(scene)
    rgb, T = R.render(cam)
    torch.cuda.synchronize()
    img = torch.cat([rgb, T[None]], 0).permute(1, 2, 0).cpu().numpy().astype(np.float64)
    ks, vs = R.keys_vals(True)
    rng = R.ranges()
    rast = R.debug_copy(_abi.AAA_DBG_RASTER, np.float32, 28)
    orc = O.Oracle(scene).set_view(cam)
    ys, xs = np.mgrid[max(0, Y - rad):min(cam.height, Y + rad + 1), max(0, X - rad):min(cam.width, X + rad + 1)]
    xs, ys = xs.ravel(), ys.ravel()
    rep = compare(orc, img[ys, xs], xs, ys)
    print("window report", rep)
    ref, flags, nb = orc.render_pixels(xs, ys)
    tiles_x = (cam.width + 15) // 16
    for k in range(len(xs)):
        x, y = int(xs[k]), int(ys[k])
        g_img = img[y, x]
        e0 = np.abs(g_img[:3] - ref[k, :3]).max()
        if e0 <= 5e-4:
            continue
        best = _best_variant(orc, x, y, g_img, e0, 5e-4)
        if best <= 5e-4:
            continue
        print(f"\n=== FAIL pixel ({x},{y}) gpu {g_img} oracle {ref[k]} flags {flags[k]} best variant err {best:.3e}")
        c = orc.pixel_contribs(x, y)
        tile = (y // 16) * tiles_x + x // 16
        s, e = rng[tile]
        sub = ((x % 16) // 8) + 2 * ((y % 16) // 4)
        gpu_hits = []
        for j in range(s, e):
            v = int(vs[j])
            if not (v >> (24 + sub)) & 1:
                continue
            g = v & 0xFFFFFF
            rho2, z, a, hit = eval_fp32(rast[g], x, y, cam.near)
            if hit:
                gpu_hits.append((z, j, g, a, rho2))
        gpu_hits.sort()
        Tg = 1.0
        print(" oracle contributions (z, g, alpha, rho2, tau, included, flags):")
        for r in c[:60]:
            print(f"   z={r[CI['z']]:.9f} g={int(r[CI['g']]):8d} a={r[CI['alpha']]:.5f} rho2={r[CI['rho2']]:.5f} "
                  f"tau={r[CI['tau']]:.5f} inc={int(r[CI['included']])} fl={int(r[CI['flags']])}")
        print(" gpu hits in (z, list position) order (z, g, alpha, rho2, T before):")
        for (z, j, g, a, rho2) in gpu_hits[:60]:
            print(f"   z={z:.9f} g={g:8d} a={a:.5f} rho2={rho2:.5f} T={Tg:.6f}")
            if Tg * (1 - a) < 1e-4:
                print("   (terminates)")
                break
            Tg *= 1 - a


if __name__ == "__main__":
    main()
