"""Dump every intermediate of one GPU render (image, K1 records, raster records, colours, sorted
pairs, ranges) to an .npz for offline analysis against the oracle. Diagnostic tool."""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--out", default="gpurun_out/dump.npz")
    ap.add_argument("--scale3", action="store_true", help="large-FOV 3x camera (crop protocol)")
    a = ap.parse_args()
    import torch
    import paper_2504_12811_b200 as pkg
    from paper_2504_12811_b200 import _abi
    from synth import scenes as S
    scene, cams = S.make_config(a.config)
    cam = cams[a.view]
    if a.scale3:
        cam = cam.scaled(width=3 * cam.width, height=3 * cam.height, cx=cam.cx + cam.width, cy=cam.cy + cam.height)
    R = pkg.Renderer(0)
    R.load(scene)
    rgb, T = R.render(cam)
    torch.cuda.synchronize()
    st = R.stats()
    img = torch.cat([rgb, T[None]], 0).cpu().numpy()
    ks, vs = R.keys_vals(True)
    rng = R.ranges()
    rast = R.debug_copy(_abi.AAA_DBG_RASTER, np.float32, 28)
    col = R.debug_copy(_abi.AAA_DBG_COLOR, np.float32, 4)
    G = R.gaussian_records()
    np.savez_compressed(a.out, img=img, keys=ks, vals=vs, ranges=rng, raster=rast, color=col, gauss=G,
                        stats=np.array([st[k] for k in ("visible", "candidates", "pairs", "spilled_pixels",
                                                         "unresolved_pixels")]))
    print("dumped", a.out, st)


if __name__ == "__main__":
    main()
