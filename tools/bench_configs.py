"""Per-config measurements beyond the headline (c2 frames/s + per-kernel ms, c4 1-GPU
frames/s per OOD sub-batch, c5 single-frame ms on 1 GPU and per tile band).

    python tools/bench_configs.py [out.jsonl]

Timing: CUDA events on the caller's stream around whole batches after 3 warm-up batches; per
stage ms from the library's AAA_FLAG_TIMING events. c5 bands: the 135 tile rows are split into 8
cost-balanced bands (aaa_tile_row_costs -> partition.band_split, as the 8-GPU path does) and
each rank's band is rendered alone with aaa_render_band (K1 on all Gaussians + the row-cost model,
K2-K6 on the band) — the slowest band is the per-rank compute of the 8-GPU frame (the NCCL gather
is not included: one GPU here)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

STAGES = ["preprocess", "scan", "cull_emit", "sort", "ranges", "raster", "raster_spill", "sync_gap", "copy", "total"]


def timed(fn, reps=3, warm=3):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best


def main():
    import torch
    import paper_2504_12811_b200 as pkg
    from synth import scenes as S

    out_path = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "gpurun_out" / "configs.jsonl"
    R = pkg.Renderer(0)
    lines = []
    for cfg, nv in (("c2", 100), ("c4wide", 50), ("c4zoomout", 50), ("c4inside", 50)):
        scene, cams = S.make_config(cfg)
        R.load(scene)
        cams = cams[:nv]
        H, W = cams[0].height, cams[0].width
        out = torch.empty((len(cams), 3, H, W), dtype=torch.float32, device="cuda:0")
        R.set_config(flags=pkg.AAA_FLAG_TIMING)
        R.render_batch(cams, out_rgb=out)
        torch.cuda.synchronize()
        R.stats()
        ms = timed(lambda: R.render_batch(cams, out_rgb=out))
        st = R.stats()
        R.set_config(flags=0)
        cnt = []
        for c in cams[:: max(1, len(cams) // 5)]:
            R.render(c, with_T=False)
            cnt.append(R.stats())
        mean = {k: sum(s[k] for s in cnt) / len(cnt) for k in
                ("visible", "pairs", "evaluations", "spilled_pixels", "deep_pixels", "unresolved_pixels", "crossing")}
        rec = {"config": cfg, "gaussians": int(scene.means.shape[0]), "width": W, "height": H, "views": len(cams),
               "frames_per_s": len(cams) / (ms / 1e3), "mpix_per_s": len(cams) * W * H / (ms * 1e3),
               "ms_per_view": ms / len(cams), "stages_ms_per_view": dict(zip(STAGES, st["ms"])),
               "counters_per_view": mean}
        print(json.dumps(rec), flush=True)
        lines.append(rec)
        del out
    # c5: one 3840x2160 frame, 6M Gaussians
    scene, cams = S.make_config("c5")
    R.load(scene)
    cam = cams[0]
    R.set_camera(cam)
    H, W = cam.height, cam.width
    full = torch.empty((3, H, W), dtype=torch.float32, device="cuda:0")
    ms_full = timed(lambda: R.render(cam, out_rgb=full, with_T=False))
    buf = torch.empty((3 * H * W,), dtype=torch.float32, device="cuda:0")
    band_ms = []
    bands = None
    for rank in range(8):
        band_ms.append(timed(lambda: R.render_band(rank, 8, out_rgb=buf)))
        if bands is None:
            _, _, cuts = R.render_band(rank, 8, out_rgb=buf)
            bands = [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:])]
    rec = {"config": "c5", "gaussians": int(scene.means.shape[0]), "width": W, "height": H,
           "frame_ms_1gpu": ms_full, "bands_8": bands, "band_ms": band_ms, "slowest_band_ms": max(band_ms),
           "band_speedup_vs_1gpu": ms_full / max(band_ms),
           "note": "slowest band = per-rank compute of the 8-GPU tile-band frame (gather not included)"}
    print(json.dumps(rec), flush=True)
    lines.append(rec)
    out_path.parent.mkdir(exist_ok=True)
    out_path.write_text("".join(json.dumps(x) + "\n" for x in lines))


if __name__ == "__main__":
    main()
