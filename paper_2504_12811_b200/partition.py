"""Multi-GPU partitioner (L6): one process per GPU; work is split by camera (view batches) or,
for one huge frame, by screen-space tile-row bands. NCCL (torch.distributed) is used only to
broadcast the Gaussian set from rank 0 and to gather images — rendering itself exchanges
nothing. Pure host logic lives in plain functions so it can be tested on CPU with
the gloo backend.
"""
from __future__ import annotations

import numpy as np

SCENE_FIELDS = ("means", "scales", "quats", "opacities", "sh", "v_train")


def view_block(n_views: int, rank: int, world: int, per_rank: int) -> list[int]:
    """Views of `rank` for one step: per_rank views interleaved along the camera path
    (view k*stride + rank, stride = max(8, world)), so every rank sees the same mix of near and
    far views and the union over 8 ranks of 25 views is the whole 200-view orbit."""
    stride = max(8, world)
    return [(k * stride + rank) % n_views for k in range(per_rank)]


def view_shard(n_views: int, rank: int, world: int) -> list[int]:
    """Strong-scaling shard of a fixed batch: round-robin (balances cost along the path)."""
    return list(range(rank, n_views, world))


def band_split(row_costs, world: int) -> list[tuple[int, int]]:
    """Split tile rows [0, R) into `world` contiguous bands of near-equal cost (prefix-sum
    cut points); every band gets >= 1 row. Identical on every rank. world > R is rejected
    (an empty band cannot be rendered by aaa_render_tiles)."""
    c = np.asarray(row_costs, dtype=np.float64)
    R = c.shape[0]
    if world <= 1:
        return [(0, R)]
    if world > R:
        raise ValueError(f"band_split: {world} bands need at least {world} tile rows (have {R})")
    pref = np.concatenate([[0.0], np.cumsum(c + 1e-9)])   # +eps: empty rows still count a little
    total = pref[-1]
    cuts = [0]
    for k in range(1, world):
        target = total * k / world
        r = int(np.searchsorted(pref, target))
        lo = cuts[-1] + 1
        hi = R - (world - k)
        cuts.append(int(min(max(r, lo), hi)))
    cuts.append(R)
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def _host_staged(t):
    """gloo collectives run on host tensors (the N-ranks-on-fewer-GPUs functional mode and CPU
    tests); NCCL ones on the device tensors themselves."""
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend() == "gloo"


def _bcast(t, src):
    import torch.distributed as dist
    if _host_staged(t):
        h = t.cpu()
        dist.broadcast(h, src)
        t.copy_(h)
    else:
        dist.broadcast(t, src)


def scene_to_tensors(scene, device):
    import torch
    t = {f: torch.from_numpy(np.ascontiguousarray(getattr(scene, f), dtype=np.float32)).to(device)
         for f in SCENE_FIELDS}
    t["sh_degree"] = scene.sh_degree
    return t


def broadcast_scene(scene_or_none, rank: int, world: int, device, src: int = 0):
    """Broadcast the Gaussian SoA from `src` to every rank (NCCL on GPUs, gloo on CPU).
    Returns a dict of tensors on `device` (+ 'sh_degree')."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        return scene_to_tensors(scene_or_none, device)
    if rank == src:
        t = scene_to_tensors(scene_or_none, device)
        meta = torch.tensor([t["means"].shape[0], t["sh_degree"]], dtype=torch.int64, device=device)
    else:
        meta = torch.zeros(2, dtype=torch.int64, device=device)
    _bcast(meta, src)
    n, deg = int(meta[0]), int(meta[1])
    K = (deg + 1) ** 2
    shapes = {"means": (n, 3), "scales": (n, 3), "quats": (n, 4), "opacities": (n,), "sh": (n, K, 3),
              "v_train": (n,)}
    if rank != src:
        t = {f: torch.empty(shapes[f], dtype=torch.float32, device=device) for f in SCENE_FIELDS}
        t["sh_degree"] = deg
    for f in SCENE_FIELDS:
        _bcast(t[f], src)
    return t


def load_scene_broadcast(config: str, rank: int, world: int, device):
    """Rank 0 generates the seeded scene of `config`; NCCL broadcasts it. Cameras are cheap and
    deterministic, so every rank builds them locally."""
    from synth import scenes as S
    if rank == 0 or world <= 1:
        scene, cams = S.make_config(config)
    else:
        scene = None
        cams = _cameras_only(config)
    t = broadcast_scene(scene, rank, world, device)
    return t, cams, t["sh_degree"]


def _cameras_only(config: str):
    from synth import scenes as S
    if config == "c1":
        return [S.c1_camera()]
    if config == "c2":
        return S.c2_cameras()
    if config == "c3":
        return S.c3_cameras()
    if config.startswith("c4"):
        return S.c4_cameras(config[2:])
    if config == "c5":
        return [S.c5_camera()]
    raise ValueError(config)


def gather_views(images, rank: int, world: int, dst: int = 0):
    """Gather every rank's rendered views (v_r x 3 x H x W, equal v_r on every rank) to `dst`:
    one NCCL gather (rank `dst` receives world x v_r images). Returns the list on dst, else None."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        return [images]
    staged = _host_staged(images)
    src = images.cpu() if staged else images
    lst = [torch.empty_like(src) for _ in range(world)] if rank == dst else None
    dist.gather(src, lst, dst=dst)
    return lst


def gather_bands(band_rgb, bands, width: int, height: int, rank: int, world: int, dst: int = 0):
    """Assemble tile-row bands (3 x band_h x W each) into the full 3 x H x W frame on `dst`
    with one NCCL all-gather of equal-size padded bands."""
    import torch
    import torch.distributed as dist
    max_h = max(max(0, min(16 * b, height) - 16 * a) for a, b in bands)
    pad = torch.zeros((3, max_h, width), dtype=band_rgb.dtype, device=band_rgb.device)
    pad[:, : band_rgb.shape[1]] = band_rgb
    out = torch.empty((world * 3, max_h, width), dtype=band_rgb.dtype, device=band_rgb.device)
    if _host_staged(pad):
        h = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(h, pad.cpu())
        out.copy_(h)
    else:
        dist.all_gather_into_tensor(out, pad)
    out = out.view(world, 3, max_h, width)
    if rank != dst:
        return None
    parts = []
    for r, (a, b) in enumerate(bands):
        h = max(0, min(16 * b, height) - 16 * a)
        parts.append(out[r, :, :h])
    return torch.cat(parts, dim=1)
