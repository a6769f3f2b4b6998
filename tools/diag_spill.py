"""Diagnostic: compare K6 vs K6s (spill continuation) against the oracle on one view."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import oracle as O
    import paper_2504_12811_b200 as pkg
    from paper_2504_12811_b200 import _abi
    from synth import scenes as S
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    view = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    scene, cams = S.make_config(cfg)
    cam = cams[view]
    R = pkg.Renderer(0)
    R.load(scene)
    orc = O.Oracle(scene).set_view(cam)
    H, W = cam.height, cam.width
    yy, xx = np.mgrid[0:H, 0:W]
    ref, flags, nb = orc.render_pixels(xx.ravel(), yy.ravel())
    ref = ref.reshape(H, W, 4)
    for name, kw in [("K32", dict(window_k=32, flags=0)), ("K16", dict(window_k=16, flags=0)),
                     ("forced", dict(window_k=32, flags=pkg.AAA_FLAG_FORCE_FALLBACK))]:
        R.set_config(**kw)
        rgb, T = R.render(cam)
        torch.cuda.synchronize()
        img = torch.cat([rgb, T[None]], 0).permute(1, 2, 0).cpu().numpy()
        st = R.stats()
        hdr = R.debug_copy(_abi.AAA_DBG_SPILL, np.uint32, 8)
        spilled = np.zeros((H, W), bool)
        if len(hdr):
            pix = hdr[:, 0].astype(np.int64)
            spilled.ravel()[pix] = True
        err = np.abs(img[..., :3] - ref[..., :3]).max(axis=2)
        bad = err > 5e-4
        print(f"{name}: spilled={st['spilled_pixels']} unresolved={st['unresolved_pixels']} bad={bad.sum()} "
              f"bad&spilled={(bad & spilled).sum()} bad&~spilled={(bad & ~spilled).sum()} maxerr={err.max():.3e}")
        ys, xs = np.nonzero(bad & ~spilled)
        print("   non-spilled bad examples:", list(zip(xs[:8].tolist(), ys[:8].tolist())))
        if len(hdr):
            print("   spill hdr sample:", hdr[:3].tolist())
    R.set_config(window_k=32, flags=0)


if __name__ == "__main__":
    main()
