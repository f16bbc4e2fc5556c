"""Multi-GPU partition and gather logic (paper_2505_24796_b200/shard.py), on CPU.

The render itself needs the B200 (tests/test_gpu_parity.py covers band
rendering == full-frame rendering on one GPU); here the host-side pieces of
the N > 1 path run with world_size 2 over gloo: the view split, the
replicated band partition, the grouped send/recv gather of band rows and the
stats all-reduce.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_24796_b200 import shard
from paper_2505_24796_b200.raster import FragmentStats


def test_view_blocks_cover_every_view_once():
    for n in (0, 1, 7, 256):
        for g in (1, 2, 3, 8):
            b = shard.view_blocks(n, g)
            assert len(b) == g and b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(g - 1))
            sizes = [e - s for s, e in b]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_band_partition_contiguous_and_balanced(world):
    rng = np.random.default_rng(world)
    counts = rng.integers(0, 5000, size=135)  # 4K frame: 135 tile rows
    bands = shard.band_partition(counts, world)
    assert bands[0][0] == 0 and bands[-1][1] == 135
    assert all(bands[i][1] == bands[i + 1][0] for i in range(world - 1))
    assert all(e - s >= 1 for s, e in bands)
    w = counts + 1.0
    loads = [w[s:e].sum() for s, e in bands]
    # each boundary is within one row of its target: imbalance bounded by the heaviest row
    assert max(loads) - w.sum() / world <= w.max() + 1e-9
    assert bands == shard.band_partition(counts.copy(), world)  # deterministic (replicated on every rank)


def test_band_partition_skewed_rows_and_limits():
    counts = np.zeros(68)
    counts[30:34] = 1e6  # all the work in four rows
    b = shard.band_partition(counts, 4)
    assert [e - s for s, e in b if 30 <= s < 34 or 30 < e <= 34]  # boundaries land inside the hot rows
    assert sum(e - s for s, e in b) == 68
    with pytest.raises(ValueError):
        shard.band_partition(np.ones(3), 4)


def test_band_pixel_rows_clip_last_band():
    assert shard.band_pixel_rows((0, 2), 1080) == (0, 32)
    assert shard.band_pixel_rows((60, 68), 1080) == (960, 1080)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, H, W, rows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ref_rgb = torch.arange(H * W * 3, dtype=torch.float32).reshape(H, W, 3) / (H * W * 3)
        ref_T = torch.linspace(0, 1, H * W, dtype=torch.float32).reshape(H, W)
        ref_n = torch.arange(H * W, dtype=torch.int32).reshape(H, W) % 97
        bands = shard.band_partition(rows, world)
        r0, r1 = shard.band_pixel_rows(bands[rank], H)
        # this rank's local buffers: only its band rows hold real values (the rest is garbage)
        rgb = torch.full((H, W, 3), -1.0)
        T = torch.full((H, W), -1.0)
        n = torch.full((H, W), -1, dtype=torch.int32)
        rgb[r0:r1], T[r0:r1], n[r0:r1] = ref_rgb[r0:r1], ref_T[r0:r1], ref_n[r0:r1]
        full = [torch.zeros_like(rgb), torch.zeros_like(T), torch.zeros_like(n)] if rank == 0 else None
        shard.gather_bands([rgb, T, n], full, bands, H)
        st = FragmentStats(f_blend=10 + rank, f_cull=20, f_skip=30, exp_calls=5, n_splats=100 * (rank + 1),
                           dropped=7, pixels_terminated=rank, n_visible=11)
        tot = shard.reduce_stats(st, torch.device("cpu"))
        if rank == 0:
            ok = (torch.equal(full[0], ref_rgb) and torch.equal(full[1], ref_T) and torch.equal(full[2], ref_n))
            q.put(("gather", ok))
            q.put(("stats", (tot.f_blend, tot.f_cull, tot.n_splats, tot.dropped, tot.pixels_terminated, tot.n_visible)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("H,W", [(1080, 64), (40, 24)])
def test_gather_bands_world2_gloo(H, W):
    world = 2
    rows = np.random.default_rng(0).integers(0, 100, size=(H + 15) // 16)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, rows, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res["gather"], "assembled frame differs from the reference image"
    assert res["stats"] == (10 + 11, 40, 100 + 200, 7, 0 + 1, 11)


def _bench_worker(rank, world, port, q):
    """bench.py's multi-rank orchestration on CPU/gloo: view split (C4 orbit pool and yaw views of C2), the tile-band
    partition and gather of a C3-sized frame, the stats reduction and the max-over-ranks timing."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2505_24796_b200 import synthetic

        out = {}
        # views: C4's 256-camera orbit split into contiguous blocks, and C2's single camera expanded to yaw views
        _, orbit = synthetic.config_scene("c4", 0.0005)
        v4 = bench.rank_views(orbit, orbit[0], 25, rank, world, False)
        out["c4"] = [np.asarray(c.view).tobytes() for c in v4]
        base = synthetic.make_camera(64, 48)
        v2 = bench.rank_views([base], base, 7, rank, world, False)
        out["c2"] = [np.asarray(c.view).tobytes() for c in v2]
        vb = bench.rank_views([base], base, 7, rank, world, True)  # bands: the same frames on every rank
        out["bands"] = [np.asarray(c.view).tobytes() for c in vb]
        # timing: max over ranks
        out["max"] = bench.max_over_ranks([1.0 + rank, 5.0 - rank], "cpu", world)
        # bands: partition a 4K frame's row counts, each rank fills its rows, gather on rank 0
        H, W = 2160, 32
        rows = np.random.default_rng(7).integers(0, 5000, size=(H + 15) // 16)
        bands = shard.band_partition(rows, world)
        r0, r1 = shard.band_pixel_rows(bands[rank], H)
        ref = torch.arange(H * W * 3, dtype=torch.float32).reshape(H, W, 3)
        rgb = torch.full((H, W, 3), -1.0)
        rgb[r0:r1] = ref[r0:r1]
        T = torch.zeros((H, W))
        n = torch.zeros((H, W), dtype=torch.int32)
        full = [torch.zeros_like(rgb), torch.zeros_like(T), torch.zeros_like(n)] if rank == 0 else None
        shard.gather_bands([rgb, T, n], full, bands, H)
        out["gather"] = bool(torch.equal(full[0], ref)) if rank == 0 else None
        out["bands_cover"] = bands
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_bench_orchestration_world2_gloo():
    """bench.py --gpus 2 on CPU: every C4 orbit view rendered by exactly one rank, distinct C2 yaw views per rank,
    identical band frames, the band partition covering the 4K frame and gathering it on rank 0, max-over-ranks."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    a, b = res[0], res[1]
    assert not set(a["c4"]) & set(b["c4"]), "an orbit view rendered by both ranks"
    assert len(set(a["c4"]) | set(b["c4"])) == 50
    assert not set(a["c2"]) & set(b["c2"])
    assert a["bands"] == b["bands"]
    assert a["max"] == b["max"] == [2.0, 5.0]
    assert a["gather"]
    bands = a["bands_cover"]
    assert bands[0][0] == 0 and bands[-1][1] == (2160 + 15) // 16 and bands[0][1] == bands[1][0]
