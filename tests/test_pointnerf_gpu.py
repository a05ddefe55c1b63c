"""cfg5's aggregation MLP on the tensor cores (hp_pointnerf_aggregate /
hp_pointnerf_head: tcgen05.mma, TMEM accumulators) against its fp32 PyTorch
restatement (pointnerf.PointNeRFMLP.reference).  There is no reference
implementation of this stage; the tolerance is the bf16
operand rounding's: 2e-2 absolute / relative on the aggregated features and
on (sigma, rgb)."""

import numpy as np
import pytest
import torch

import golden_util as gu
import paper_2404_14044_b200 as hp
from paper_2404_14044_b200 import device as dv, pipeline
from paper_2404_14044_b200.pointnerf import PointNeRFMLP, render_step, sample_rays

pytestmark = pytest.mark.gpu

TOL = dict(rtol=2e-2, atol=2e-2)


def _frame(name, K):
    _, cloud, cam, cfg, tn, tf, stride, _ = gu.get_case(name)
    dev = torch.device("cuda")
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    xyz = up(cloud.positions)
    idx = dv.build(xyz, cam, cfg.pad)
    rays = (up(pixels), up(dirs), up(t_near), up(t_far), up(slopes))
    fr = pipeline._query_sample(idx, up(cloud.colors), *rays, hp.SamplerConfig(k_neighbors=K), True, None,
                                emit_knn=True)
    return cloud, cam, fr.samples, rays, xyz


@pytest.mark.parametrize("name", ["cfg1", "small_sphere_surface", "dup_planes"])
@pytest.mark.parametrize("K", [8, 4])
def test_aggregation_mlp_matches_fp32_reference(name, K):
    cloud, cam, s, rays, xyz = _frame(name, K)
    R = int(s[1].numel())
    assert R > 0
    mlp = PointNeRFMLP(cloud.count, seed=7)
    out, g = mlp(s, rays[1], cam.origin, xyz)
    torch.cuda.synchronize()
    ref_out, ref_g = mlp.reference(s[9], s[10], sample_rays(s[0]), s[2], rays[1], cam.origin, xyz)
    assert g.shape == (R, 128) and out.shape == (R, 4)
    torch.testing.assert_close(g.float(), ref_g, **TOL)
    torch.testing.assert_close(out, ref_out, **TOL)
    assert torch.isfinite(out).all()


def test_tiles_with_a_ragged_tail_and_missing_neighbours():
    """R not a multiple of the 16 samples of a tile; neighbours -1 (pools
    smaller than K) contribute nothing."""
    cloud, cam, s, rays, xyz = _frame("edge_points", 8)
    mlp = PointNeRFMLP(cloud.count, seed=1)
    out, g = mlp(s, rays[1], cam.origin, xyz)
    ref_out, ref_g = mlp.reference(s[9], s[10], sample_rays(s[0]), s[2], rays[1], cam.origin, xyz)
    torch.testing.assert_close(g.float(), ref_g, **TOL)
    torch.testing.assert_close(out, ref_out, **TOL)


def test_render_step_composites_the_mlp_output():
    cloud, cam, s, rays, xyz = _frame("cfg1", 8)
    mlp = PointNeRFMLP(cloud.count, seed=3)
    color, depth, out = render_step(mlp, s, rays[1], cam.origin, xyz, rays[0], rays[3], cam.width, cam.height)
    c = color.cpu().numpy()
    assert np.isfinite(c).all() and c.min() >= 0.0 and c.max() <= 1.0 + 1e-12
    assert np.isfinite(depth.cpu().numpy()).all() and (np.diff(s[0].cpu().numpy()) > 0).any()
