"""Multi-GPU ray sharding (one process per GPU, torch.distributed).

Rays are independent given the read-only index (reference SPEC.md: "query is
read-only and safe to run concurrently", hash_index.py:263-293 splits rays
into contiguous chunks and concatenates results in input order).  Here:

* every rank builds the same index from the replicated cloud (O(n), small
  next to query + sample);
* the frame's rays are split into contiguous bands of whole image rows with
  equal estimated cost (the number of slots each ray scans = a box sum over
  the per-pixel counts; every rank computes the same split, no exchange);
* the only collective gathers the retained-sample tiles to rank 0
  (all_gather of counts, then a padded all_gather of the tiles); concatenating
  in rank order reproduces the single-GPU output exactly, because bands are
  contiguous in ray order.
"""

from __future__ import annotations

import numpy as np

__all__ = ["row_costs", "balanced_row_bands", "split_by_cost", "gather_samples"]


def row_costs(positions: np.ndarray, camera, pad: int) -> np.ndarray:
    """Estimated scan cost of every image row of ray_grid rays."""
    W, H = camera.width, camera.height
    wp, hp = W + 2 * pad, H + 2 * pad
    u, v, depth = camera.project(positions)
    fu, fv = np.floor(u) + pad, np.floor(v) + pad
    ok = (depth > 0) & (fu >= 0) & (fu < wp) & (fv >= 0) & (fv < hp)
    grid = np.zeros((hp + 1, wp + 1), np.int64)
    np.add.at(grid, (fv[ok].astype(np.int64) + 1, fu[ok].astype(np.int64) + 1), 1)
    sat = grid.cumsum(0).cumsum(1)
    s = 2 * pad + 1
    # ray (x, y) scans padded window [x, x+s) x [y, y+s)
    box = sat[s:s + H, s:s + W] - sat[0:H, s:s + W] - sat[s:s + H, 0:W] + sat[0:H, 0:W]
    return box.sum(axis=1) + W  # + W: fixed per-ray overhead


def split_by_cost(costs: np.ndarray, parts: int):
    """Contiguous [lo, hi) ranges of ``costs`` with near-equal sums."""
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


def balanced_row_bands(positions, camera, pad, world):
    if world <= 1:
        return [(0, camera.height)]
    return split_by_cost(row_costs(positions, camera, pad), world)


def gather_samples(samples, dist, dst: int = 0):
    """Gather per-rank retained-sample tiles to rank ``dst``.

    ``samples`` is the 9-tuple of device.sample for this rank's rays.  Returns
    the concatenated 9-tuple on ``dst`` (offsets rebased) and None elsewhere.
    Works with any backend (NCCL on GPUs, gloo in the CPU tests).
    """
    import torch
    r_off, r_id, r_t, r_dist, r_udf, r_alpha, r_w, r_color, t_end = samples
    world = dist.get_world_size()
    dev = r_id.device
    R = torch.tensor([r_id.numel(), t_end.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(R) for _ in range(world)]
    dist.all_gather(sizes, R)
    sizes = [tuple(int(v) for v in s.tolist()) for s in sizes]
    maxR = max(s[0] for s in sizes)
    maxM = max(s[1] for s in sizes)
    has_color = r_color.numel() > 0
    f = torch.zeros((maxR, 8), dtype=torch.float64, device=dev)
    f[: r_id.numel(), 0] = r_id.to(torch.float64)  # ids < 2^53: exact in float64
    for k, x in enumerate((r_t, r_dist, r_udf, r_alpha, r_w), start=1):
        f[: x.numel(), k] = x
    if has_color:
        f[: r_id.numel(), 6] = 0.0
        f = torch.cat([f, torch.zeros((maxR, 3), dtype=torch.float64, device=dev)], dim=1)
        f[: r_id.numel(), 8:11] = r_color
    g = torch.zeros((maxM, 2), dtype=torch.float64, device=dev)
    g[: t_end.numel(), 0] = t_end
    g[: t_end.numel(), 1] = (r_off[1:] - r_off[:-1]).to(torch.float64)
    fs = [torch.empty_like(f) for _ in range(world)]
    gs = [torch.empty_like(g) for _ in range(world)]
    dist.all_gather(fs, f)
    dist.all_gather(gs, g)
    if dist.get_rank() != dst:
        return None
    F = torch.cat([fs[k][: sizes[k][0]] for k in range(world)])
    G = torch.cat([gs[k][: sizes[k][1]] for k in range(world)])
    counts = G[:, 1].to(torch.int64)
    off = torch.zeros(counts.numel() + 1, dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(counts, 0)
    color = F[:, 8:11].contiguous() if has_color else torch.zeros((0, 3), dtype=torch.float64,
                                                                    device=dev)
    return (off, F[:, 0].to(torch.int64), F[:, 1].contiguous(), F[:, 2].contiguous(),
            F[:, 3].contiguous(), F[:, 4].contiguous(), F[:, 5].contiguous(), color,
            G[:, 0].contiguous())
