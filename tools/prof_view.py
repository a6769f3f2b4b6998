"""Render a few views of a config (for ncu capture): `python tools/prof_view.py c3 3`."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import paper_2504_12811_b200 as pkg
    from synth import scenes as S
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    nv = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    scene, cams = S.make_config(cfg)
    R = pkg.Renderer(0)
    R.load(scene)
    for i in range(nv):
        R.render(cams[(8 * i) % len(cams)], with_T=False)
    torch.cuda.synchronize()
    print(R.stats())


if __name__ == "__main__":
    main()
