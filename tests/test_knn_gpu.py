"""emit_knn: each retained sample's K neighbour point ids and blend weights
(north_star stage 4 -- "candidate-point indices and blend weights emitted
per sample").  The neighbours are the reference sampler's K nearest
(_kernels.py:603-620: the pool rule, strict-< insertion, ties to the earlier
candidate) and the weights its colour blend's (:622-656): 1/d normalised, or
1/nz over coincident points; -1 / 0 past the pool size.  Checked bit for bit
against a restatement of those loops on the oracle's CSR, for the full-CSR
sampler and the head (prefix) path."""

import numpy as np
import pytest
import torch

import golden_util as gu
import paper_2404_14044_b200 as hp
from oracle import oracle as orc
from paper_2404_14044_b200 import device as dv, pipeline

pytestmark = pytest.mark.gpu


def _ref_knn(off, ids, ts, ds, slopes, K, r, j):
    lo = off[r]
    q = off[r + 1] - lo
    tj = ts[lo + j]
    rj = slopes[r] * tj
    n_el = int(np.sum(ds[lo:lo + q] <= rj))
    use_el = n_el >= K
    ksel = min(K, n_el if use_el else q)
    bd, bi = [np.inf] * ksel, [-1] * ksel
    for i in range(q):
        di = ds[lo + i]
        if use_el and di > rj:
            continue
        dt = ts[lo + i] - tj
        d2 = dt * dt + di * di
        if d2 < bd[ksel - 1]:
            b = ksel - 1
            while b > 0 and bd[b - 1] > d2:
                bd[b], bi[b] = bd[b - 1], bi[b - 1]
                b -= 1
            bd[b], bi[b] = d2, i
    nz = sum(1 for d in bd if d == 0.0)
    if nz:
        w = [1.0 / nz if d == 0.0 else 0.0 for d in bd]
    else:
        inv = [1.0 / np.sqrt(d) for d in bd]
        ws = 0.0
        for x in inv:
            ws += x
        w = [x / ws for x in inv]
    pid = [int(ids[lo + i]) for i in bi]
    return pid + [-1] * (K - ksel), w + [0.0] * (K - ksel)


def _check(out, q, slopes, K):
    r_off, r_id, r_t = (x.cpu().numpy() for x in out[:3])
    kid, kw = out[9].cpu().numpy(), out[10].cpu().numpy()
    assert kid.shape == (len(r_id), K) and kw.shape == (len(r_id), K)
    off, ids, ts, ds = q[0], q[1], q[2], q[3]
    for r in range(len(r_off) - 1):
        lo = off[r]
        for k in range(r_off[r], r_off[r + 1]):
            j = int(np.flatnonzero((ids[lo:off[r + 1]] == r_id[k]) & (ts[lo:off[r + 1]] == r_t[k]))[0])
            pid, w = _ref_knn(off, ids, ts, ds, slopes, K, r, j)
            np.testing.assert_array_equal(kid[k], pid)
            np.testing.assert_array_equal(kw[k], w)
            if pid[0] >= 0:
                assert abs(sum(w) - 1.0) < 1e-12


@pytest.mark.parametrize("name", ["small_sphere_surface", "dup_planes", "orbit_planes"])
@pytest.mark.parametrize("K", [1, 8, 20])
def test_knn_ids_and_weights_match_the_reference_loops(name, K):
    _, cloud, cam, cfg, tn, tf, stride, _ = gu.get_case(name)
    dev = torch.device("cuda")
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    b = orc.build(cloud.positions, cam, cfg.pad)
    q = orc.query(b["table_start"], b["table_count"], b["slot_x"], b["slot_y"], b["slot_z"], b["reordered_ids"],
                  cam.width + 2 * cfg.pad, cfg.pad, pixels[:, 0], pixels[:, 1], dirs, cam.origin, t_near, t_far,
                  slopes)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    sc = hp.SamplerConfig(k_neighbors=K)
    out = dv.sample(up(q[0]), up(q[1]), up(q[2]), up(q[3]), up(slopes), sc, up(cloud.colors), emit_knn=True)
    _check(out, q, slopes, K)
    # the head path emits the same rows (and the samples are unchanged by the flag)
    idx = dv.build(up(cloud.positions), cam, cfg.pad)
    rays = (up(pixels), up(dirs), up(t_near), up(t_far), up(slopes))
    fr = pipeline._query_sample(idx, up(cloud.colors), *rays, sc, True, None, prefix=True, emit_knn=True)
    for a, c in zip(fr.samples, out):
        assert torch.equal(a, c)
    plain = dv.sample(up(q[0]), up(q[1]), up(q[2]), up(q[3]), up(slopes), sc, up(cloud.colors))
    for a, c in zip(plain, out[:9]):
        assert torch.equal(a, c)
