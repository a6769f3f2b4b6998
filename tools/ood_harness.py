"""OOD sampling-rate harness (the desk-scale analogue of the paper's
multi-resolution experiments): render c2 views at 1/f of the training
resolution (same field of view) with the adaptive 3D filter (k = 0.3) and without it (k = 0), and
compare each against the training-resolution render box-downsampled by f (the alias-free target).
Prints PSNR per factor. python tools/ood_harness.py [views]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_12811_b200 as pkg  # noqa: E402
from synth import scenes as S  # noqa: E402


def psnr(a, b):
    mse = float(((a - b) ** 2).mean())
    return 10.0 * np.log10(1.0 / max(mse, 1e-20))


def run(R, scene, cams, views, factors=(2, 4, 8)):
    R.load(scene)
    out = {}
    for f in factors:
        res = {"k0.3": [], "k0": []}
        for v in views:
            cam = cams[v]
            R.set_config(k=0.3)
            ref, _ = R.render(cam, with_T=False)
            ref = torch.nn.functional.avg_pool2d(ref[None], f)[0].cpu().numpy()
            lo = cam.scaled(width=cam.width // f, height=cam.height // f, fx=cam.fx / f, fy=cam.fy / f,
                            cx=cam.cx / f, cy=cam.cy / f)
            for k, name in ((0.3, "k0.3"), (0.0, "k0")):
                R.set_config(k=k)
                img, _ = R.render(lo, with_T=False)
                res[name].append(psnr(img.cpu().numpy(), ref))
        out[f] = {k: float(np.mean(v)) for k, v in res.items()}
    R.set_config(k=0.3)
    return out


def main():
    nv = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    scene, cams = S.make_config("c2")
    R = pkg.Renderer(0)
    out = run(R, scene, cams, list(range(0, 100, 100 // nv))[:nv])
    print(json.dumps({"config": "c2, 800x800 training resolution, PSNR vs box-downsampled training-res render",
                      "psnr_db": out}))


if __name__ == "__main__":
    main()
