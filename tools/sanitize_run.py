"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): c1 and a reduced c2
view through every raster level (K6, forced K6s, forced K6d), the 16-entry window, the global-order
and 2D ablations, a band render and one backward pass.

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py small
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_12811_b200 as pkg  # noqa: E402
from synth import scenes as S  # noqa: E402


def main():
    small = len(sys.argv) > 1 and sys.argv[1] == "small"
    R = pkg.Renderer(0)
    c1, cams1 = S.make_config("c1")
    R.load(c1)
    R.render(cams1[0])
    sc, cams = S.make_config("c2", n=3000 if small else 100_000)
    cam = cams[7]
    if small:
        cam = cam.scaled(width=128, height=96, cx=64.0, cy=48.0, fx=170.0, fy=170.0)
    R.load(sc)
    for flags, wk in ((0, 32), (0, 16), (pkg.AAA_FLAG_FORCE_FALLBACK, 32),
                      (pkg.AAA_FLAG_FORCE_FALLBACK | pkg.AAA_FLAG_FORCE_DEEP, 32),
                      (pkg.AAA_FLAG_NO_HIER_SORT, 32), (pkg.AAA_FLAG_NO_3D, 32), (pkg.AAA_FLAG_NO_TILE_CULL, 32)):
        R.set_config(flags=flags, window_k=wk)
        R.render(cam)
        R.stats()
    R.set_config(flags=0, window_k=32)
    R.set_camera(cam)
    rows = (cam.height + 15) // 16
    R.render_tiles(1, max(2, rows - 1))
    R.render_batch([cams[1], cams[2]] if not small else [cam, cam])
    R.set_config(flags=pkg.AAA_FLAG_SAVE_CONTRIBS)
    R.render(cam)
    R.backward(torch.ones((3, cam.height, cam.width), device="cuda:0"))
    R.set_config(flags=0)
    R.compute_vtrain(cams[:4])
    torch.cuda.synchronize()
    print("sanitize workload done", R.stats())


if __name__ == "__main__":
    main()
