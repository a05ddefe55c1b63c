"""Pin the C oracle (oracle/hp_oracle.c) against the REFERENCE's golden vectors.

tests/golden/*.npz were produced by oracle/make_golden.py running the
reference hashpoint package (numba) on the cases of golden_cases.py.  The
oracle must reproduce every array: build tables, query CSR (bit-exact), and
sampler outputs (bit-exact where the reference is deterministic IEEE; values
through exp() within VAL_RTOL, though on the same glibc they match exactly).
CPU only.
"""

import numpy as np
import pytest

import golden_util as gu
from oracle import oracle as orc


@pytest.fixture(scope="module", params=gu.case_names())
def case(request):
    name = request.param
    g = gu.load(name)
    c = gu.get_case(name)
    return name, g, c


def test_inputs_regenerate_identically(case):
    name, g, (_, cloud, cam, cfg, tn, tf, stride, _) = case
    assert gu.digest(cloud.positions) == g["positions_sha"], "scene generator drifted"
    assert int(g["kernel_size"]) == cfg.kernel_size


def test_build_matches_reference(case):
    name, g, (_, cloud, cam, cfg, *_r) = case
    out = orc.build(cloud.positions, cam, cfg.pad)
    for k in gu.BUILD_FIELDS:
        assert gu.digest(out[k]) == g[f"build_{k}_sha"], f"{name}: build {k} differs"
    lin = orc.rasterize(cloud.positions, cam, cfg.pad)
    mism = int(np.count_nonzero(gu.digest(lin) != g["build_bucket_sha"]))
    if "build_bucket" in g:
        mism = int(np.count_nonzero(lin != g["build_bucket"]))
    assert mism == 0, f"{name}: {mism} bucket assignments differ from the reference"


def _oracle_query(cloud, cam, cfg, tn, tf, stride, threads=2):
    b = orc.build(cloud.positions, cam, cfg.pad)
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    q = orc.query(b["table_start"], b["table_count"], b["slot_x"], b["slot_y"], b["slot_z"],
                  b["reordered_ids"], cam.width + 2 * cfg.pad, cfg.pad, pixels[:, 0], pixels[:, 1],
                  dirs, cam.origin, t_near, t_far, slopes, threads=threads)
    return q, slopes


def test_query_matches_reference(case):
    name, g, (_, cloud, cam, cfg, tn, tf, stride, _) = case
    q, _ = _oracle_query(cloud, cam, cfg, tn, tf, stride)
    for k, v in zip(gu.QUERY_FIELDS, q):
        assert gu.digest(v) == g[f"query_{k}_sha"], f"{name}: query {k} differs"
    rows = g["rows"]
    sub = gu.csr_rows(q[0], rows, q[1], q[2], q[3])
    for k, v in zip(gu.QUERY_FIELDS[:4], sub):
        np.testing.assert_array_equal(v, g[f"query_{k}"])


def test_query_thread_count_invariant(case):
    name, g, (_, cloud, cam, cfg, tn, tf, stride, _) = case
    q1, _ = _oracle_query(cloud, cam, cfg, tn, tf, stride, threads=1)
    q4, _ = _oracle_query(cloud, cam, cfg, tn, tf, stride, threads=4)
    for a, b in zip(q1, q4):
        np.testing.assert_array_equal(a, b)


def test_sample_matches_reference(case):
    name, g, (_, cloud, cam, cfg, tn, tf, stride, samplers) = case
    q, slopes = _oracle_query(cloud, cam, cfg, tn, tf, stride)
    for sname in samplers:
        sc = gu.sampler_config(sname)
        for colored in ((True, False) if sname == "default" else (True,)):
            out = orc.sample(q[0], q[1], q[2], q[3], slopes, sc.k_neighbors, sc.beta * sc.beta,
                             sc.gamma, sc.retention_mode == "epsilon", sc.epsilon, sc.tau_min,
                             cloud.colors if colored else None, threads=3)
            tag = f"sample_{sname}{'' if colored else '_nocolor'}_"
            gu.check_sample(g, tag, out, g["rows"])
