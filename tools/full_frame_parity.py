"""Full-frame parity reports (SURVEY 8(d) 'checked subset'):
render whole views on the GPU through the C-ABI and compare EVERY pixel with the float64 oracle
through the ambiguity-aware comparator (tests/compare.py). Default set: c3 views 0 and 100, one
view per c4 sub-batch (wide 3, zoom-out 10, inside 48) and the full c5 4K frame.
Writes one JSON line per frame to profiles/<round>_full_frame_parity.jsonl.

    python tools/full_frame_parity.py r02 [cfg:view ...]
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2504_12811_b200 as pkg  # noqa: E402
from synth import scenes as S  # noqa: E402
from tests.compare import compare  # noqa: E402

DEFAULT = ["c3:0", "c3:100", "c4wide:3", "c4zoomout:10", "c4inside:48", "c5:0"]


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
    todo = sys.argv[2:] or DEFAULT
    out = ROOT / "profiles" / f"{rnd}_full_frame_parity.jsonl"
    out.parent.mkdir(exist_ok=True)
    R = pkg.Renderer(0)
    loaded = None
    for item in todo:
        cfg, view = item.split(":")
        view = int(view)
        scene, cams = S.make_config(cfg)
        key = "c3" if cfg.startswith("c4") else cfg
        if loaded != key:
            R.load(scene)
            loaded = key
        cam = cams[view]
        rgb, T = R.render(cam)
        torch.cuda.synchronize()
        st = R.stats()
        img = torch.cat([rgb, T[None]], 0).permute(1, 2, 0).reshape(-1, 4).cpu().numpy().astype(np.float64)
        t0 = time.perf_counter()
        orc = O.Oracle(scene).set_view(cam)
        yy, xx = np.mgrid[0:cam.height, 0:cam.width]
        rep = compare(orc, img, xx.ravel(), yy.ravel())
        dt = time.perf_counter() - t0
        rep.update(config=cfg, view=view, width=cam.width, height=cam.height, gaussians=scene.n,
                   oracle_seconds=round(dt, 1), oracle_cores=O.num_threads(),
                   host_cpus=len(os.sched_getaffinity(0)),
                   gpu_stats={k: st[k] for k in ("visible", "candidates", "pairs", "spilled_pixels",
                                                 "deep_pixels", "unresolved_pixels", "crossing")})
        line = json.dumps(rep)
        print(line, flush=True)
        for path in (out, ROOT / "gpurun_out" / out.name):  # gpurun_out/ comes back from a GPU box
            path.parent.mkdir(exist_ok=True)
            with open(path, "a") as f:
                f.write(line + "\n")


if __name__ == "__main__":
    main()
