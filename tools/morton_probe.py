"""Probe: does a spatially coherent Gaussian order (Morton order of the means) speed up the render?
Times c3 view batches with the scene in generator order and in Morton order (permuted on the host
before loading). Diagnostic only: `python tools/morton_probe.py`."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def morton_perm(means: np.ndarray) -> np.ndarray:
    lo, hi = means.min(0), means.max(0)
    q = np.clip(((means - lo) / np.maximum(hi - lo, 1e-12) * 1023).astype(np.int64), 0, 1023)

    def spread(v):
        v = (v | (v << 16)) & 0x030000FF
        v = (v | (v << 8)) & 0x0300F00F
        v = (v | (v << 4)) & 0x030C30C3
        v = (v | (v << 2)) & 0x09249249
        return v
    code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
    return np.argsort(code, kind="stable")


def main():
    import torch
    import paper_2504_12811_b200 as pkg
    from synth import scenes as S
    scene, cams = S.make_config("c3")
    views = [cams[i] for i in range(0, 200, 8)]
    R = pkg.Renderer(0)
    H, W = views[0].height, views[0].width
    out = torch.empty((len(views), 3, H, W), dtype=torch.float32, device="cuda:0")
    perm = morton_perm(scene.means)
    fields = ("means", "scales", "quats", "opacities", "sh", "v_train")
    sc_m = S.Scene(*[getattr(scene, f)[perm] for f in fields], scene.sh_degree)
    for name, sc in (("generator order", scene), ("morton order", sc_m), ("generator order", scene)):
        R.load(sc)
        R.set_config(flags=pkg.AAA_FLAG_TIMING)
        for _ in range(2):
            R.render_batch(views, out_rgb=out)
        torch.cuda.synchronize()
        R.stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            R.render_batch(views, out_rgb=out)
        e1.record()
        torch.cuda.synchronize()
        st = R.stats()
        fps = 3 * len(views) / (e0.elapsed_time(e1) / 1e3)
        print(name, f"FPS {fps:.1f}", [round(x, 3) for x in st["ms"][:7]], flush=True)


if __name__ == "__main__":
    main()
