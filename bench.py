#!/usr/bin/env python
"""Benchmark of the B200 AAA-Gaussians forward renderer (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2]): 3M synthetic M360-shaped Gaussians, SH
degree 3, 1920x1080 views on a 200-view orbit. One step = every rank renders its block of
`--views-per-rank` views (weak scaling: per-rank work fixed, views interleaved along the orbit,
view index k*8 + rank). Scene bytes (720 MB) exceed the 126 MB L2, so every view re-streams
its inputs from HBM (no flush needed). Prints ONE JSON line on rank 0.

--impl reference times the float64 CPU oracle (oracle/) on the host cores on a bounded pixel
sample of the same views (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # derived: SMs x FP32 lanes x 2 x max clock
METRIC = "frames/s (3M-Gaussian SH3 1920x1080 render, view batch)"
PAPER_CONTEXT = {"paper_fps_rtx4090_m360_indoor": 129.5, "source": "PAPER.md P:521 (Table 5), other GPU and scenes"}
STAGES = ["preprocess", "scan", "cull_emit", "sort", "ranges", "raster", "raster_spill", "sync_gap", "copy", "total"]
EVAL_FLOPS = 45  # FP32 operations of one pixel-Gaussian evaluation (K6 roofline)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d, "measured"
        except Exception:
            pass
    return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nme, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nme)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def scene_and_views(cfg: str, rank: int, world: int, per_rank: int):
    from synth import scenes as S
    scene, cams = S.make_config(cfg)
    stride = max(8, world)
    idx = [(k * stride + rank) % len(cams) for k in range(per_rank)]
    return scene, cams, idx


def stage_bytes(st, n, deg):
    """Algorithmic bytes per view for each HBM-bound stage."""
    V, C, P = st["visible"], st["candidates"], st["pairs"]
    sh_b = 12 * (deg + 1) ** 2
    passes = (24 + 13 + 7) // 8
    return {
        "preprocess": 48 * n + 4 * n + V * (sh_b + 80 + 112 + 16),
        "scan": 8 * n,
        "cull_emit": 80 * V + 4 * C + 12 * P,
        "sort": 8 * P + 24 * passes * P,
        "ranges": 8 * P,
        "raster": 12 * P + 112 * P,
    }


def cpu_baseline(scene, cams, idx, budget_s=20.0):
    """The float64 oracle, as it stands, on this host's cores: a bounded pixel sample."""
    import oracle as O
    O.build()
    orc = O.Oracle(scene)
    cores = O.num_threads()
    cam = cams[idx[0]]
    t0 = time.perf_counter()
    orc.set_view(cam)
    t_prep = time.perf_counter() - t0
    tx, ty = (cam.width + 15) // 16, (cam.height + 15) // 16
    rng = np.random.default_rng(0)
    n_tiles = max(1, cores)
    done_px, t_pix = 0, 0.0
    while t_pix < budget_s:
        tiles = rng.choice(tx * ty, n_tiles, replace=False)
        px = np.concatenate([(t % tx) * 16 + np.tile(np.arange(16), 16) for t in tiles])
        py = np.concatenate([(t // tx) * 16 + np.repeat(np.arange(16), 16) for t in tiles])
        ok = (px < cam.width) & (py < cam.height)
        t1 = time.perf_counter()
        orc.render_pixels(px[ok], py[ok])
        t_pix += time.perf_counter() - t1
        done_px += int(ok.sum())
        if t_pix + t_prep > budget_s:
            break
    frame_s = t_prep + t_pix * (cam.width * cam.height) / done_px
    return {"value": 1.0 / frame_s, "unit": "frames/s", "cores": cores, "kind": "oracle",
            "sample": f"view {idx[0]}: per-Gaussian stage on all {scene.n} Gaussians ({t_prep:.2f} s) + "
                      f"{done_px} pixels of {done_px // 256} random 16x16 tiles ({t_pix:.2f} s), extrapolated "
                      f"to {cam.width}x{cam.height}"}


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    import oracle as O
    scene, cams, idx = scene_and_views(args.config, 0, 1, args.views_per_rank)
    O.build()
    orc = O.Oracle(scene)
    cores = O.num_threads()
    cam = cams[idx[0]]
    tx, ty = (cam.width + 15) // 16, (cam.height + 15) // 16
    rng = np.random.default_rng(1)
    n_tiles = max(1, cores)

    def step(i):
        c = cams[idx[i % len(idx)]]
        t0 = time.perf_counter()
        orc.set_view(c)
        tiles = rng.choice(tx * ty, n_tiles, replace=False)
        px = np.concatenate([(t % tx) * 16 + np.tile(np.arange(16), 16) for t in tiles])
        py = np.concatenate([(t // tx) * 16 + np.repeat(np.arange(16), 16) for t in tiles])
        ok = (px < c.width) & (py < c.height)
        t1 = time.perf_counter()
        orc.render_pixels(px[ok], py[ok])
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1, int(ok.sum())

    for i in range(args.warmup):
        step(i)
    tp = tpx = 0.0
    npx = 0
    t_start = time.perf_counter()
    for i in range(args.steps):
        a, b, n = step(args.warmup + i)
        tp += a
        tpx += b
        npx += n
    wall = time.perf_counter() - t_start
    frame_s = tp / args.steps + tpx * (cam.width * cam.height) / npx
    v = 1.0 / frame_s
    sample = (f"per step: per-Gaussian stage on all {scene.n} Gaussians + {n_tiles} random 16x16 tiles "
              f"({n_tiles * 256} px) of one c3 view; frames/s extrapolated to {cam.width}x{cam.height}")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * wall / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": f"{args.config}: 3M Gaussians SH3 1920x1080, 200-view orbit",
                                           "sample": sample},
           "cpu_baseline": {"value": v, "unit": "frames/s", "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def run_ours(args, world, rank, local):
    import torch
    import paper_2504_12811_b200 as pkg
    from paper_2504_12811_b200 import _build

    _build.build()
    # one process per GPU; with fewer GPUs than ranks (a functional test of the N > 1 path on one
    # device), ranks share devices round-robin and AAA_DIST_BACKEND=gloo avoids NCCL's one-rank-
    # per-GPU rule
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("AAA_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2504_12811_b200 import partition as part

    # rank 0 builds the scene; NCCL broadcasts it (the only pre-render collective)
    scene_t, cams, sh_deg = part.load_scene_broadcast(args.config, rank, world, dev)
    idx = part.view_block(len(cams), rank, world, args.views_per_rank)
    views = [cams[i] for i in idx]
    R = pkg.Renderer(local)
    R.load(tensors=scene_t)
    n = int(scene_t["means"].shape[0])
    del scene_t
    torch.cuda.empty_cache()
    H, W = views[0].height, views[0].width
    out = torch.empty((len(views), 3, H, W), dtype=torch.float32, device=dev)
    abl = {"none": 0, "no_cull": pkg.AAA_FLAG_NO_TILE_CULL, "no_hier": pkg.AAA_FLAG_NO_HIER_SORT,
           "no_3d": pkg.AAA_FLAG_NO_3D}[args.ablation]
    R.set_config(flags=pkg.AAA_FLAG_TIMING | abl, window_k=int(os.environ.get("AAA_WINDOW_K", "32")))

    def step():
        R.render_batch(views, out_rgb=out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    R.stats()                      # reset the timing accumulation
    launches0 = R.stats()["launches"]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1)
    st_timed = R.stats()
    launches = st_timed["launches"] - launches0
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    total_views = args.steps * len(views) * world
    value = total_views / (ms_max / 1000.0)

    # per-view counters (V, C, P, E) on a sample of this rank's views, timing off
    R.set_config(flags=abl)
    samp = []
    for v in views[:: max(1, len(views) // 5)]:
        R.render(v, with_T=False)
        samp.append(R.stats())
    mean = {k: float(np.mean([s[k] for s in samp])) for k in
            ("visible", "candidates", "pairs", "evaluations", "spilled_pixels", "unresolved_pixels",
             "crossing")}
    peaks, peaks_src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    stage_ms = dict(zip(STAGES, st_timed["ms"]))
    sb = stage_bytes(mean, n, 3)
    stages = {}
    for k in STAGES[:7] + ["sync_gap"]:
        t = stage_ms[k]
        ent = {"ms_per_view": t, "share": t / stage_ms["total"] if stage_ms["total"] else None}
        if k == "raster":
            # K6 + K6s (spilled-pixel continuation) form one raster unit
            t_all = t + stage_ms["raster_spill"]
            fl = mean["evaluations"] * EVAL_FLOPS
            ent.update(bound="alu", ms_incl_fallback=t_all,
                       achieved_tflops=fl / (t_all * 1e-3) / 1e12 if t_all else None,
                       achieved_gbs=sb[k] / (t_all * 1e-3) / 1e9 if t_all else None)
        elif k in sb:
            ent.update(bound="hbm", algo_bytes=sb[k], achieved_gbs=sb[k] / (t * 1e-3) / 1e9 if t else None)
        stages[k] = ent
    unit_ms = {k: stage_ms[k] for k in STAGES[:5]}
    unit_ms["raster"] = stage_ms["raster"] + stage_ms["raster_spill"]
    dom = max(unit_ms, key=unit_ms.get)
    traffic = None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(dom)
        except Exception:
            traffic = None
    if stages[dom]["bound"] == "alu":
        ach = stages[dom]["achieved_tflops"]
        roof = {"kernel": dom, "bound": "alu", "achieved": ach, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / FP32_PEAK_TFLOPS, "traffic": traffic,
                "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 x 1.965 GHz (DESIGN.md)",
                "work": f"{EVAL_FLOPS} FP32 ops x {mean['evaluations']:.3g} pixel-Gaussian evaluations per view"}
    else:
        ach = stages[dom]["achieved_gbs"]
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": traffic, "peak_source": f"{peaks_src} hbm_gbs (MEASURED_PEAKS.json)",
                "work": f"{stages[dom]['algo_bytes']:.4g} algorithmic bytes per view"}

    # e2e: the public C-ABI with HOST output buffers; D2H of every rendered image inside the region
    e2e = None
    if not args.no_e2e:
        host = torch.empty((len(views), 3, H, W), dtype=torch.float32, pin_memory=True)
        ptr = host.data_ptr()
        R.render_batch(views, host_ptrs=(ptr, 0))
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        n_e2e = max(1, args.steps // 2)
        for _ in range(n_e2e):
            R.render_batch(views, host_ptrs=(ptr, 0))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        dt_t = torch.tensor([dt], device=dev)
        if world > 1:
            torch.distributed.all_reduce(dt_t, op=torch.distributed.ReduceOp.MAX)
        ev = n_e2e * len(views) * world / float(dt_t.item())
        e2e = {"value": ev, "unit": "frames/s", "h2d_bytes_per_step": len(views) * 88,
               "d2h_bytes_per_step": len(views) * 3 * H * W * 4,
               "how": "aaa_render_batch with pinned host rgb buffers (library copies each image back); "
                      "camera structs are the per-step input; wall clock, max over ranks"}
        del host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from synth import scenes as S2
        sc, cm = S2.make_config(args.config)
        cpu = cpu_baseline(sc, cm, idx, budget_s=args.cpu_budget)

    if rank == 0:
        res = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f32",
               "data": f"synthetic (seeded {args.config} generator; no datasets or trained weights exist offline)",
               "config": {"workload": f"{args.config}: {n / 1e6:g}M Gaussians SH{sh_deg}, {W}x{H}, "
                                      f"{len(cams)}-view set; {len(views)} views per rank per step",
                          "views_per_rank_per_step": len(views), "ablation": args.ablation, "gaussians": n, "width": W, "height": H,
                          "parallelism": f"view-sharded x{world}",
                          "l2": (f"inputs larger than L2 ({n * 240 / 1e6:.0f} MB scene re-streamed per view), no flush"
                                 if n * 240 > 126e6 else
                                 f"scene ({n * 240 / 1e6:.0f} MB) fits in L2 and stays resident across views, no flush")},
               "mpix_per_s": value * W * H / 1e6,
               "roofline": roof, "stages": stages, "counters_per_view": mean,
               "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
               "clocks": clk.summary(), "context": PAPER_CONTEXT}
        print(json.dumps(res), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--views-per-rank", type=int, default=25)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ablation", default="none", choices=["none", "no_cull", "no_hier", "no_3d"],
                    help="Table 5 switches (P:521-524): no 3D tile culling / no per-pixel re-sort / 2D splats")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
