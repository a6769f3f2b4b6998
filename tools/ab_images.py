"""Bit-identity check between two builds (A/B of kernel variants that must not change any pixel):
    python tools/ab_images.py save /tmp/a.npz   (build A)
    python tools/ab_images.py cmp  /tmp/a.npz   (build B) -> one JSON line per config
Renders c2 (4 views), c3 (2), c4 wide / zoom-out / inside (1 each), RGB and T."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

CASES = [("c2", 4), ("c3", 2), ("c4wide", 1), ("c4zoomout", 1), ("c4inside", 1)]


def render_all():
    import numpy as np
    import torch
    import paper_2504_12811_b200 as pkg
    from synth import scenes as S
    out = {}
    for cfg, nv in CASES:
        scene, cams = S.make_config(cfg)
        R = pkg.Renderer(0)
        R.load(scene)
        for i in range(nv):
            cam = cams[(len(cams) * (2 * i + 1)) // (2 * nv)]
            rgb, T = R.render(cam)
            torch.cuda.synchronize()
            out[f"{cfg}_{i}"] = torch.cat([rgb, T[None]], 0).cpu().numpy()
        del R
    return out


def main():
    import numpy as np
    mode, path = sys.argv[1], sys.argv[2]
    imgs = render_all()
    if mode == "save":
        np.savez(path, **imgs)
        return
    ref = np.load(path)
    for k, v in imgs.items():
        a = ref[k]
        diff = a.view(np.uint32) != v.view(np.uint32)
        print(json.dumps({"case": k, "bit_identical": bool(not diff.any()), "differing_values": int(diff.sum()),
                          "max_abs": float(np.abs(a - v).max())}), flush=True)


if __name__ == "__main__":
    main()
