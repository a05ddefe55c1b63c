"""The operator-level drop-in (paper_2404_14044_b200._kernels) driven with the
reference's own argument lists (hash_index.build's scatter call,
hash_index.query_batch_arrays, sampler.sample_batch_arrays; reference
hash_index.py:165-177, :224-235, sampler.py:206-217): outputs sha-equal to
the reference goldens; scatter_by_bucket mutates its arguments in place as
the reference loop does (_kernels.py:76-83)."""

import numpy as np
import pytest

import golden_util as gu
from oracle import oracle as orc
from paper_2404_14044_b200 import _kernels as K

pytestmark = pytest.mark.gpu


def _scatter_ref(buckets, orig_ids, cursor, out_ids):
    # the reference loop, restated (_kernels.py:79-83)
    for j in range(buckets.shape[0]):
        b = buckets[j]
        out_ids[cursor[b]] = orig_ids[j]
        cursor[b] += 1


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_scatter_by_bucket_matches_reference_loop(seed):
    rng = np.random.default_rng(seed)
    P, n = 257, 20_000
    buckets = rng.integers(0, P, n).astype(np.int64)
    buckets[:500] = 7  # one bucket far above the warp's insertion-sort size
    orig = rng.permutation(10 * n)[:n].astype(np.int64)
    counts = np.bincount(buckets, minlength=P)
    order = rng.permutation(P)  # destination ranges in a scrambled bucket order
    cursor = np.zeros(P, np.int64)
    cursor[order] = np.concatenate([[0], np.cumsum(counts[order])])[:-1]
    c_ref, o_ref = cursor.copy(), np.full(n + 5, -1, np.int64)
    _scatter_ref(buckets, orig, c_ref, o_ref)
    c_dev, o_dev = cursor.copy(), np.full(n + 5, -1, np.int64)
    K.scatter_by_bucket(buckets, orig, c_dev, o_dev)
    np.testing.assert_array_equal(c_dev, c_ref)
    np.testing.assert_array_equal(o_dev, o_ref)


def test_scatter_by_bucket_rejects_out_of_range():
    with pytest.raises(ValueError):
        K.scatter_by_bucket(np.array([0, 3]), np.array([0, 1]), np.zeros(2, np.int64), np.zeros(2, np.int64))


@pytest.mark.parametrize("name", gu.case_names())
def test_reference_call_sites_reproduce_goldens(name):
    g = gu.load(name)
    _, cloud, cam, cfg, tn, tf, stride, samplers = gu.get_case(name)
    pad, wp, hp = cfg.pad, cam.width + 2 * cfg.pad, cam.height + 2 * cfg.pad
    # hash_index.build's pass 3, with the reference's arguments
    lin_all = orc.rasterize(cloud.positions, cam, pad)
    valid = np.flatnonzero(lin_all >= 0).astype(np.int64)
    lin = lin_all[valid]
    counts = np.bincount(lin, minlength=wp * hp).astype(np.int64)
    b = orc.build(cloud.positions, cam, pad)
    starts = np.where(counts > 0, b["table_start"], 0)
    if valid.size:  # empty pixels' starts (zeroed in the table) are irrelevant to the scatter
        cursor = starts.copy()
        slot_ids = np.empty(valid.shape[0], np.int64)
        K.scatter_by_bucket(lin, valid, cursor, slot_ids)
        assert gu.digest(slot_ids) == g["build_reordered_ids_sha"]
        np.testing.assert_array_equal(cursor - starts, counts)
    # query_batch_arrays -> hash_query_batch
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    q = K.hash_query_batch(b["table_start"], b["table_count"], b["slot_x"], b["slot_y"], b["slot_z"],
                           b["reordered_ids"], wp, pad, np.ascontiguousarray(pixels[:, 0]),
                           np.ascontiguousarray(pixels[:, 1]), dirs, cam.origin, t_near, t_far, slopes)
    for k, v in zip(gu.QUERY_FIELDS, q):
        assert v.dtype == (np.int64 if k in ("offsets", "ids", "probes", "scanned") else np.float64)
        assert gu.digest(v) == g[f"query_{k}_sha"], f"query {k}"
    # sample_batch_arrays -> sample_batch
    for sname in samplers:
        sc = gu.sampler_config(sname)
        for colored in ((True, False) if sname == "default" else (True,)):
            col = np.ascontiguousarray(cloud.colors, dtype=np.float64) if colored else np.zeros((0, 3))
            out = K.sample_batch(q[0], q[1], q[2], q[3], slopes, sc.k_neighbors, sc.beta * sc.beta, sc.gamma,
                                 sc.retention_mode == "epsilon", sc.epsilon, sc.tau_min, col, colored)
            assert out[7].shape == ((len(out[1]), 3) if colored else (0, 3))
            gu.check_sample(g, f"sample_{sname}{'' if colored else '_nocolor'}_", out, g["rows"])
