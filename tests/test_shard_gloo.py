"""Multi-rank sharding on CPU (gloo, world_size 2): cost-balanced row bands
(computed from the index's table, as every rank does on its GPU) + the
retained-sample gather to rank 0 reassemble exactly the single-rank frame.
The per-rank compute here is the oracle (the device kernels need a GPU); the
sharding and collective logic is the same code
shard.search_and_sample_distributed / bench.py run over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2404_14044_b200 as hp
from paper_2404_14044_b200.shard import (balanced_row_bands, gather_samples, row_costs, row_costs_from_table,
                                         split_by_cost)


def _setup():
    cloud = hp.generate_scene(hp.SceneSpec("sphere_surface", n=20_000, seed=3, noise=0.005))
    cam = hp.scene_camera(48, 40, fov_deg=40)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.01), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
    return cloud, cam, cfg, dirs, pixels, slopes


def _frame(cloud, cam, cfg, dirs, pixels, slopes, lo, hi):
    from oracle import oracle as orc
    b = orc.build(cloud.positions, cam, cfg.pad)
    m = hi - lo
    q = orc.query(b["table_start"], b["table_count"], b["slot_x"], b["slot_y"], b["slot_z"],
                  b["reordered_ids"], cam.width + 2 * cfg.pad, cfg.pad, pixels[lo:hi, 0],
                  pixels[lo:hi, 1], dirs[lo:hi], cam.origin, np.ones(m), np.full(m, 10.0),
                  slopes[lo:hi])
    sc = hp.SamplerConfig()
    return orc.sample(*q[:4], slopes[lo:hi], sc.k_neighbors, sc.beta * sc.beta, sc.gamma, True,
                      sc.epsilon, sc.tau_min, cloud.colors)


def _worker(rank, world, port, result_q, mode="bands"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cloud, cam, cfg, dirs, pixels, slopes = _setup()
    if mode == "bands":  # bands from the index's table (as each GPU rank computes them)
        from oracle import oracle as orc
        tc = torch.from_numpy(orc.build(cloud.positions, cam, cfg.pad)["table_count"])
        bands = balanced_row_bands(None, cam, cfg.pad, world, table_count=tc)
        lo, hi = bands[rank][0] * cam.width, bands[rank][1] * cam.width
    else:  # "empty": rank 1 holds only sky rays (no samples), rank 0 the rest
        sky = 2 * cam.width  # the first two rows miss the sphere
        lo, hi = (sky, dirs.shape[0]) if rank == 0 else (0, sky)
    out = _frame(cloud, cam, cfg, dirs, pixels, slopes, lo, hi)
    tens = tuple(torch.from_numpy(np.ascontiguousarray(x)) for x in out)
    g = gather_samples(tens, dist)
    if rank == 0:
        result_q.put([x.numpy() for x in g])
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run_two(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


@pytest.mark.timeout(300)
def test_two_rank_gather_equals_single_rank():
    got = _run_two("bands")
    cloud, cam, cfg, dirs, pixels, slopes = _setup()
    ref = _frame(cloud, cam, cfg, dirs, pixels, slopes, 0, dirs.shape[0])
    assert len(ref[1]) > 0
    assert got[1].dtype == np.int64
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


@pytest.mark.timeout(300)
def test_gather_with_a_rank_without_samples_keeps_colours():
    """a rank whose band retained nothing (sky rows) packs the same
    tile width as the others, so colours survive the gather."""
    got = _run_two("empty")
    cloud, cam, cfg, dirs, pixels, slopes = _setup()
    sky = 2 * cam.width
    a = _frame(cloud, cam, cfg, dirs, pixels, slopes, sky, dirs.shape[0])
    b = _frame(cloud, cam, cfg, dirs, pixels, slopes, 0, sky)
    assert len(b[1]) == 0 and len(a[1]) > 0 and a[7].shape[0] == len(a[1])
    ref_off = np.concatenate([a[0], a[0][-1] + b[0][1:]])
    np.testing.assert_array_equal(got[0], ref_off)
    for k in range(1, 8):
        np.testing.assert_array_equal(got[k], a[k])
    np.testing.assert_array_equal(got[8], np.concatenate([a[8], b[8]]))


def test_row_costs_from_table_equal_host_projection():
    from oracle import oracle as orc
    cloud, cam, cfg, dirs, pixels, slopes = _setup()
    tc = torch.from_numpy(orc.build(cloud.positions, cam, cfg.pad)["table_count"])
    np.testing.assert_array_equal(row_costs_from_table(tc, cam, cfg.pad).numpy(),
                                  row_costs(cloud.positions, cam, cfg.pad))


def test_split_by_cost_is_contiguous_and_balanced():
    costs = np.array([1, 1, 1, 10, 10, 1, 1, 1, 1, 1], float)
    parts = split_by_cost(costs, 3)
    assert parts[0][0] == 0 and parts[-1][1] == 10
    assert all(parts[k][1] == parts[k + 1][0] for k in range(2))
    sums = [costs[a:b].sum() for a, b in parts]
    assert max(sums) <= costs.sum() / 3 + costs.max()


def test_row_costs_equal_oracle_scanned():
    from oracle import oracle as orc
    cloud, cam, cfg, dirs, pixels, slopes = _setup()
    b = orc.build(cloud.positions, cam, cfg.pad)
    m = dirs.shape[0]
    q = orc.query(b["table_start"], b["table_count"], b["slot_x"], b["slot_y"], b["slot_z"],
                  b["reordered_ids"], cam.width + 2 * cfg.pad, cfg.pad, pixels[:, 0], pixels[:, 1],
                  dirs, cam.origin, np.ones(m), np.full(m, 10.0), slopes)
    per_row = q[5].reshape(cam.height, cam.width).sum(axis=1) + cam.width
    np.testing.assert_array_equal(row_costs(cloud.positions, cam, cfg.pad), per_row)


def _views_worker(rank, world, port, result_q):
    from paper_2404_14044_b200.pipeline import _views_of
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    result_q.put((rank, _views_of(7, dist)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_views_are_split_across_ranks():
    """pipeline.search_and_sample_views: rank r runs views[r::world]; the
    ranks' views are disjoint and cover the batch (no data-path collective)."""
    from paper_2404_14044_b200.pipeline import _views_of
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_views_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: [0, 2, 4, 6], 1: [1, 3, 5]}
    assert _views_of(3, None) == [0, 1, 2]
