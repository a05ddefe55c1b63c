"""Device path (sm_100a kernels through the C ABI) vs the reference goldens and
the C oracle.  Bit-exact for ids/offsets/tables/t/dist/udf and the primary
surface point; alpha / w / colour / t_end within golden_util.VAL_RTOL (the
device exp() may differ from glibc's by an ulp; north_star's bar is 1e-5)."""

import numpy as np
import pytest
import torch

import golden_util as gu
from oracle import oracle as orc
from paper_2404_14044_b200 import device as dv

pytestmark = pytest.mark.gpu


def _dev_case(name):
    _, cloud, cam, cfg, tn, tf, stride, samplers = gu.get_case(name)
    dev = torch.device("cuda")
    idx = dv.build(torch.from_numpy(cloud.positions).to(dev), cam, cfg.pad)
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rays = (up(pixels), up(dirs), up(t_near), up(t_far), up(slopes))
    return cloud, cam, cfg, samplers, idx, rays


@pytest.mark.parametrize("name", gu.case_names())
def test_build_bit_exact(name):
    g = gu.load(name)
    cloud, cam, cfg, samplers, idx, rays = _dev_case(name)
    for k in gu.BUILD_FIELDS:
        assert gu.digest(getattr(idx, k).cpu().numpy()) == g[f"build_{k}_sha"], f"build {k}"
    assert idx.n_in == int(np.count_nonzero(orc.rasterize(cloud.positions, cam, cfg.pad) >= 0))


@pytest.mark.parametrize("name", gu.case_names())
def test_query_bit_exact(name):
    g = gu.load(name)
    cloud, cam, cfg, samplers, idx, rays = _dev_case(name)
    q = [x.cpu().numpy() for x in dv.query(idx, *rays)]
    for k, v in zip(gu.QUERY_FIELDS, q):
        assert gu.digest(v) == g[f"query_{k}_sha"], f"query {k}"


@pytest.mark.parametrize("name", gu.case_names())
@pytest.mark.parametrize("exact_t_end", [True, False])
def test_sample_matches_reference(name, exact_t_end):
    g = gu.load(name)
    cloud, cam, cfg, samplers, idx, rays = _dev_case(name)
    q = dv.query(idx, *rays)
    colors = torch.from_numpy(cloud.colors).cuda()
    for sname in samplers:
        sc = gu.sampler_config(sname)
        for colored in ((True, False) if sname == "default" else (True,)):
            out = dv.sample(q[0], q[1], q[2], q[3], rays[4], sc, colors if colored else None,
                            exact_t_end=exact_t_end)
            out = [x.cpu().numpy() for x in out]
            tag = f"sample_{sname}{'' if colored else '_nocolor'}_"
            gu.check_sample(g, tag, out, g["rows"], check_t_end=exact_t_end)
            pid, pt = dv.primary_surface(*[torch.from_numpy(a).cuda() for a in (out[0], out[1], out[2])])
            assert gu.digest(pid.cpu().numpy()) == g[tag + "primary_sha"]


def test_layout_from_reference_table_equals_build():
    name = "small_parallel_planes"
    g = gu.load(name)
    cloud, cam, cfg, samplers, idx, rays = _dev_case(name)
    t = lambda k: torch.from_numpy(g[f"build_{k}"]).cuda()  # noqa: E731
    idx2 = dv.build_from_table(t("table_start"), t("table_count"), t("slot_x"), t("slot_y"),
                               t("slot_z"), t("reordered_ids"), cam, cfg.pad)
    for k in ("row_ptr", "rel_x", "rel_y", "rel_z", "point_id"):
        assert torch.equal(getattr(idx2, k)[: idx.n_in + (1 if k == "row_ptr" else 0)],
                           getattr(idx, k)[: idx.n_in + (1 if k == "row_ptr" else 0)]), k
    q1 = dv.query(idx, *rays)
    q2 = dv.query(idx2, *rays)
    for a, b in zip(q1, q2):
        assert torch.equal(a, b)
