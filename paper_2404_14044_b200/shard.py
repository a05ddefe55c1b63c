"""Multi-GPU ray sharding (one process per GPU, torch.distributed).

Rays are independent given the read-only index (reference SPEC.md: "query is
read-only and safe to run concurrently", hash_index.py:263-293 splits rays
into contiguous chunks and concatenates results in input order).  Here:

* every rank builds the same index from the replicated cloud (O(n), small
  next to query + sample);
* the view's rays are split into contiguous bands of whole image rows with
  equal estimated cost: the slots each ray's window scans, a box sum over the
  index's per-pixel counts (a summed-area table of ``table_count`` on the
  device); every rank computes the same split from its own replicated index,
  no exchange;
* the only collective gathers the retained-sample tiles to rank 0 (the sizes
  with one all_gather, then padded ``gather`` calls of the int64 ids, the
  float64 values and the per-ray counts / t_end); concatenating in rank order
  reproduces the single-GPU output exactly, because bands are contiguous in
  ray order.

``search_and_sample_distributed`` is the library entry point (a whole view,
host arrays in, the reference's 9-tuple out on rank 0).
"""

from __future__ import annotations

import numpy as np

__all__ = ["row_costs", "row_costs_from_table", "balanced_row_bands", "split_by_cost", "gather_samples",
           "search_and_sample_distributed"]


def row_costs(positions: np.ndarray, camera, pad: int) -> np.ndarray:
    """Estimated scan cost of every image row of ray_grid rays (host: projects
    the cloud; see :func:`row_costs_from_table` for the device version)."""
    W, H = camera.width, camera.height
    wp, hp = W + 2 * pad, H + 2 * pad
    u, v, depth = camera.project(positions)
    fu, fv = np.floor(u) + pad, np.floor(v) + pad
    ok = (depth > 0) & (fu >= 0) & (fu < wp) & (fv >= 0) & (fv < hp)
    counts = np.zeros(hp * wp, np.int64)
    np.add.at(counts, fv[ok].astype(np.int64) * wp + fu[ok].astype(np.int64), 1)
    import torch
    return row_costs_from_table(torch.from_numpy(counts), camera, pad).numpy()


def row_costs_from_table(table_count, camera, pad: int):
    """Per image row, the slots the rays of that row scan (s x s window box
    sums of the index's ``table_count``, int64 [P] row-major over the padded
    grid) plus a fixed per-ray term.  torch ops on the tensor's device (the
    replicated index on a GPU, or CPU); returns int64 [H] on that device."""
    import torch
    W, H = int(camera.width), int(camera.height)
    wp, hp = W + 2 * pad, H + 2 * pad
    s = 2 * pad + 1
    grid = torch.zeros((hp + 1, wp + 1), dtype=torch.int64, device=table_count.device)
    grid[1:, 1:] = table_count.view(hp, wp)
    sat = grid.cumsum(0).cumsum(1)
    # ray (x, y) scans padded window [x, x+s) x [y, y+s)
    box = sat[s:s + H, s:s + W] - sat[0:H, s:s + W] - sat[s:s + H, 0:W] + sat[0:H, 0:W]
    return box.sum(dim=1) + W  # + W: fixed per-ray overhead


def split_by_cost(costs, parts: int):
    """Contiguous [lo, hi) ranges of ``costs`` with near-equal sums."""
    costs = np.asarray(costs)
    n = len(costs)
    parts = max(1, min(parts, n)) if n else 1
    cum = np.concatenate([[0], np.cumsum(costs, dtype=np.float64)])
    total = cum[-1]
    cuts = [0]
    for k in range(1, parts):
        cut = int(np.searchsorted(cum, total * k / parts, side="left"))
        cuts.append(min(max(cut, cuts[-1]), n))
    cuts.append(n)
    return [(cuts[k], cuts[k + 1]) for k in range(parts)]


def balanced_row_bands(positions, camera, pad, world, table_count=None):
    """Row bands [y0, y1) of the view, one per rank.  With ``table_count``
    (the index's, on any device) the costs come from it; else the cloud is
    projected on the host."""
    if world <= 1:
        return [(0, camera.height)]
    if table_count is not None:
        costs = row_costs_from_table(table_count, camera, pad).cpu().numpy()
    else:
        costs = row_costs(positions, camera, pad)
    return split_by_cost(costs, world)


def gather_samples(samples, dist, dst: int = 0):
    """Gather per-rank retained-sample tiles to rank ``dst``.

    ``samples`` is the 9-tuple of device.sample for this rank's rays (any
    rank may hold no rays or no samples).  Returns the concatenated 9-tuple on
    ``dst`` (offsets rebased; ids stay int64) and None elsewhere.  Colours are
    gathered when any rank has them (a rank with R = 0 cannot tell), so every
    rank packs the same tile width.  Works with any backend (NCCL on GPUs,
    gloo in the CPU tests).
    """
    import torch
    r_off, r_id, r_t, r_dist, r_udf, r_alpha, r_w, r_color, t_end = samples
    world = dist.get_world_size()
    rank = dist.get_rank()
    dev = r_id.device
    R, M = int(r_id.numel()), int(t_end.numel())
    mine = torch.tensor([R, M, 1 if r_color.numel() > 0 else 0], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(sizes, mine)
    sizes = [tuple(int(v) for v in s.tolist()) for s in sizes]
    maxR = max(max(s[0] for s in sizes), 1)
    maxM = max(max(s[1] for s in sizes), 1)
    has_color = any(s[2] for s in sizes)
    ncol = 8 if has_color else 5
    ids = torch.zeros(maxR, dtype=torch.int64, device=dev)
    ids[:R] = r_id
    vals = torch.zeros((maxR, ncol), dtype=torch.float64, device=dev)
    for k, x in enumerate((r_t, r_dist, r_udf, r_alpha, r_w)):
        vals[:R, k] = x
    if has_color and R:
        vals[:R, 5:8] = r_color
    per_ray = torch.zeros((maxM, 2), dtype=torch.float64, device=dev)
    per_ray[:M, 0] = t_end
    cnt = torch.zeros(maxM, dtype=torch.int64, device=dev)
    cnt[:M] = r_off[1:] - r_off[:-1]
    out = []
    for x in (ids, vals, per_ray, cnt):
        lst = [torch.empty_like(x) for _ in range(world)] if rank == dst else None
        dist.gather(x, lst, dst=dst)
        out.append(lst)
    if rank != dst:
        return None
    I = torch.cat([out[0][k][: sizes[k][0]] for k in range(world)])
    V = torch.cat([out[1][k][: sizes[k][0]] for k in range(world)])
    T = torch.cat([out[2][k][: sizes[k][1], 0] for k in range(world)])
    counts = torch.cat([out[3][k][: sizes[k][1]] for k in range(world)])
    off = torch.zeros(counts.numel() + 1, dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(counts, 0)
    color = V[:, 5:8].contiguous() if has_color else torch.zeros((0, 3), dtype=torch.float64, device=dev)
    return (off, I, V[:, 0].contiguous(), V[:, 1].contiguous(), V[:, 2].contiguous(), V[:, 3].contiguous(),
            V[:, 4].contiguous(), color, T.contiguous())


def search_and_sample_distributed(cloud, camera, search_cfg, t_near: float, t_far: float, dist,
                                  sampler_cfg=None, with_colors: bool = True, exact_t_end: bool = True,
                                  return_device: bool = False):
    """A whole view (every pixel's ray, row-major: ``ray_grid(camera)``) over
    all ranks of ``dist``: each rank uploads the cloud, builds the index, takes
    its cost-balanced band of rows (from the index's table), generates those
    rays on the device, queries and samples them; the tiles are gathered to
    rank 0.  Returns the reference's 9-tuple (``sample_batch_arrays``,
    sampler.py:196-217) as numpy on rank 0 (device tensors with
    ``return_device``), None on the other ranks."""
    import torch

    from . import device, pipeline
    from .sampler import SamplerConfig
    dev = torch.device("cuda", torch.cuda.current_device())
    world = dist.get_world_size()
    rank = dist.get_rank()
    xyz = torch.from_numpy(np.ascontiguousarray(cloud.positions)).to(dev, dtype=torch.float64, non_blocking=True)
    col = None
    if with_colors and cloud.colors is not None:
        col = torch.from_numpy(np.ascontiguousarray(cloud.colors)).to(dev, dtype=torch.float64,
                                                                      non_blocking=True)
    idx = device.build_layout(xyz, camera, search_cfg.pad)  # the query layout of the whole view
    counts = (idx.row_ptr[1:] - idx.row_ptr[:-1]).to(torch.int64)  # points per padded pixel (row-major)
    y0, y1 = balanced_row_bands(None, camera, search_cfg.pad, world, table_count=counts)[rank]
    W = int(camera.width)
    dirs, pixels, tn, tf = device.ray_grid(camera, dev, row0=y0, rows=y1 - y0, t_near=t_near, t_far=t_far)
    sl = device.radius_slopes(camera, search_cfg.kernel_radius, search_cfg.use_approx_radius, row0=y0,
                              m=(y1 - y0) * W, dev=dev)
    fr = pipeline._query_sample(idx, col, pixels, dirs, tn, tf, sl, sampler_cfg or SamplerConfig(), exact_t_end,
                                None)
    g = gather_samples(fr.samples, dist) if world > 1 else fr.samples
    if g is None or return_device:
        return g
    outs = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in g]
    for o, x in zip(outs, g):
        o.copy_(x, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return tuple(o.numpy() for o in outs)
