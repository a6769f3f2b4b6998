"""Multi-GPU partitioner host logic (CPU): view blocks, cost-balanced tile bands, and the
broadcast / band-gather collectives exercised with world_size 2 over gloo."""
import os
import socket

import numpy as np
import pytest

from paper_2504_12811_b200 import partition as part


def test_view_blocks_cover_orbit_once_at_8_ranks():
    got = sorted(v for r in range(8) for v in part.view_block(200, r, 8, 25))
    assert got == list(range(200))
    # weak scaling: the per-rank block size is fixed, views are spread along the path
    b0 = part.view_block(200, 0, 1, 25)
    assert len(b0) == 25 and max(np.diff(b0)) == 8


def test_view_shard_round_robin():
    for w in (1, 2, 4, 8):
        got = sorted(v for r in range(w) for v in part.view_shard(200, r, w))
        assert got == list(range(200))


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_band_split_balanced_contiguous(world):
    rng = np.random.default_rng(world)
    costs = rng.gamma(0.5, 100.0, 135)
    costs[60:70] *= 20                          # a dense band of rows (2.6x)
    bands = part.band_split(costs, world)
    assert bands[0][0] == 0 and bands[-1][1] == 135
    assert all(a < b for a, b in bands)
    assert all(bands[i][1] == bands[i + 1][0] for i in range(world - 1))
    loads = [costs[a:b].sum() for a, b in bands]
    # each band is within one row of the ideal share
    assert max(loads) <= costs.sum() / world + costs.max() + 1e-6


def test_band_split_rejects_more_bands_than_rows():
    """An empty band cannot be rendered (aaa_render_tiles rejects it): world > R is an error."""
    with pytest.raises(ValueError):
        part.band_split(np.ones(3), 4)
    assert part.band_split(np.ones(4), 4) == [(0, 1), (1, 2), (2, 3), (3, 4)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from synth import scenes as S
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        scene = S.c2_scene(n=2000, n_views_vtrain=3) if rank == 0 else None
        t = part.broadcast_scene(scene, rank, world, torch.device("cpu"))
        ref = S.c2_scene(n=2000, n_views_vtrain=3)
        ok_bcast = all(np.array_equal(t[f].numpy(), getattr(ref, f)) for f in part.SCENE_FIELDS)
        ok_bcast = ok_bcast and t["sh_degree"] == 3
        # band gather: each rank contributes its rows of a known image
        H, W = 70, 20
        full = torch.arange(3 * H * W, dtype=torch.float32).reshape(3, H, W)
        bands = part.band_split(np.ones((H + 15) // 16), world)
        a, b = bands[rank]
        mine = full[:, 16 * a: min(16 * b, H)].clone()
        got = part.gather_bands(mine, bands, W, H, rank, world)
        ok_gather = bool(torch.equal(got, full)) if rank == 0 else got is None
        # view gather: each rank's block of images arrives at rank 0 in rank order
        imgs = torch.full((3, 3, 4, 5), float(rank))
        lst = part.gather_views(imgs, rank, world)
        if rank == 0:
            ok_gather = ok_gather and len(lst) == world and all(torch.equal(lst[r], torch.full((3, 3, 4, 5), float(r)))
                                                               for r in range(world))
        else:
            ok_gather = ok_gather and lst is None
        q.put((rank, ok_bcast, ok_gather))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_broadcast_and_band_gather():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _, _ in res) == [0, 1]
    assert all(b and g for _, b, g in res), res
