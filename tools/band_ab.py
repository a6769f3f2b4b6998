"""Tile-band timing for A/B of the band path (one JSON line): c5, `world` bands rendered one after
another on one GPU (the per-rank compute of the multi-GPU frame), best of 3 per band after a
warm-up; the stacked bands are checked bit-identical to the single-GPU frame.
    python tools/band_ab.py [world]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch
    import paper_2504_12811_b200 as pkg
    from synth import scenes as S
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    scene, cams = S.make_config("c5")
    cam = cams[0]
    R = pkg.Renderer(0)
    R.load(scene)
    full, _ = R.render(cam, with_T=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best_full = None
    for _ in range(4):
        e0.record()
        R.render(cam, with_T=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best_full = ms if best_full is None else min(best_full, ms)
    buf = torch.empty((3 * cam.height * cam.width,), dtype=torch.float32, device="cuda:0")
    band_ms, parts, cuts = [], [], None
    for rank in range(world):
        best = None
        for it in range(4):
            e0.record()
            rgb, _, cuts = R.render_band(rank, world, out_rgb=buf)
            e1.record()
            torch.cuda.synchronize()
            if it:
                ms = e0.elapsed_time(e1)
                best = ms if best is None else min(best, ms)
        parts.append(rgb.clone())
        band_ms.append(best)
    stacked = torch.cat(parts, dim=1)
    print(json.dumps({"world": world, "frame_ms_1gpu": best_full, "band_ms": band_ms, "slowest_band_ms": max(band_ms),
                      "speedup": best_full / max(band_ms), "cuts": [int(c) for c in cuts],
                      "stacked_equals_full": bool(torch.equal(stacked, full))}), flush=True)


if __name__ == "__main__":
    main()
