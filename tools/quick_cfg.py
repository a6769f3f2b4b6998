"""Quick per-config timing for A/B runs of build or environment variants (one JSON line):
    [AAA_GIANT_LIST=...] python tools/quick_cfg.py CFG [n_views] [reps]
Best of `reps` batches after 2 warm-up batches, CUDA events; per-stage ms from the library."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

STAGES = ["preprocess", "scan", "cull_emit", "sort", "ranges", "raster", "raster_spill", "sync_gap", "copy", "total"]


def main():
    import os
    import torch
    import paper_2504_12811_b200 as pkg
    from synth import scenes as S
    cfg = sys.argv[1]
    nv = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    scene, cams = S.make_config(cfg)
    cams = cams[:: max(1, len(cams) // nv)][:nv]
    R = pkg.Renderer(0)
    R.load(scene)
    H, W = cams[0].height, cams[0].width
    out = torch.empty((len(cams), 3, H, W), dtype=torch.float32, device="cuda:0")
    R.set_config(flags=pkg.AAA_FLAG_TIMING)
    for _ in range(2):
        R.render_batch(cams, out_rgb=out)
    torch.cuda.synchronize()
    R.stats()
    best = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        e0.record()
        R.render_batch(cams, out_rgb=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    st = R.stats()
    R.set_config(flags=0)
    cnt = []
    maxlist = []
    for c in cams[:: max(1, len(cams) // 4)]:
        R.render(c, with_T=False)
        cnt.append(R.stats())
        rg = R.ranges()
        maxlist.append(int((rg[:, 1].astype("int64") - rg[:, 0]).max()))
    mean = {k: sum(s[k] for s in cnt) / len(cnt) for k in
            ("pairs", "evaluations", "spilled_pixels", "giant_pixels", "deep_pixels", "unresolved_pixels")}
    mean["max_list"] = maxlist
    env = {k: v for k, v in os.environ.items() if k.startswith("AAA_")}
    print(json.dumps({"config": cfg, "env": env, "views": len(cams), "fps": len(cams) / (best / 1e3),
                      "ms_per_view": best / len(cams),
                      "stages": {k: round(v, 4) for k, v in zip(STAGES, st["ms"])}, "counters": mean}), flush=True)


if __name__ == "__main__":
    main()
