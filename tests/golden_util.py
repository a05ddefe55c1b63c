"""Helpers shared by the golden-vector tests (oracle and device)."""

from __future__ import annotations

import hashlib
import os

import numpy as np

import golden_cases
from paper_2404_14044_b200.geometry import radius_slopes
from paper_2404_14044_b200.sampler import SamplerConfig

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SAMPLE_FIELDS = ["r_off", "r_id", "r_t", "r_dist", "r_udf", "r_alpha", "r_w", "r_color", "t_end"]
QUERY_FIELDS = ["offsets", "ids", "t_proj", "dist_perp", "probes", "scanned"]
BUILD_FIELDS = ["table_start", "table_count", "reordered_ids", "slot_x", "slot_y", "slot_z"]

# Tolerance for fp64 values that pass through exp() (alpha, weights,
# transmittance): the device's exp and glibc's may differ by an ulp.  Far
# tighter than the north_star's 1e-5 relative bar.
VAL_RTOL = 1e-12


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def load(name):
    return dict(np.load(os.path.join(GOLDEN_DIR, f"{name}.npz")))


def all_cases():
    return list(golden_cases.cases())


def case_names():
    return [c[0] for c in golden_cases.cases()]


def get_case(name):
    for c in golden_cases.cases():
        if c[0] == name:
            return c
    raise KeyError(name)


def rays_and_slopes(cam, cfg, tn, tf, stride):
    pixels, dirs, t_near, t_far = golden_cases.rays_for(cam, tn, tf, stride)
    slopes = radius_slopes(cam, pixels, cfg.kernel_radius, cfg.use_approx_radius)
    return pixels, dirs, t_near, t_far, slopes


def sampler_config(name) -> SamplerConfig:
    return SamplerConfig(**golden_cases.SAMPLERS[name])


def csr_rows(off, rows, *arrays):
    counts = off[rows + 1] - off[rows]
    sub = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    if len(rows):
        idx = np.concatenate([np.arange(off[r], off[r + 1]) for r in rows]).astype(np.int64)
    else:
        idx = np.zeros(0, np.int64)
    return (sub,) + tuple(np.asarray(a)[idx] for a in arrays)


def primary_of(r_off, r_id):
    has = r_off[1:] > r_off[:-1]
    if len(r_id) == 0:
        return np.full(len(has), -1, np.int64)
    return np.where(has, r_id[np.minimum(r_off[:-1], len(r_id) - 1)], -1).astype(np.int64)


def check_sample(g, tag, out, rows, exact_values=False, check_t_end=True):
    """Compare a sample_batch 9-tuple against golden record ``tag``.

    Integer outputs (offsets, ids) and the t/dist columns (copied, not
    computed) must be bit-exact; udf is bit-exact by construction (sum of
    sqrt in ascending order); alpha/w/colour/t_end within VAL_RTOL unless
    ``exact_values``.
    """
    r_off = np.asarray(out[0])
    assert digest(r_off) == g[tag + "r_off_sha"], f"{tag}: retained offsets differ"
    assert digest(np.asarray(out[1])) == g[tag + "r_id_sha"], f"{tag}: retained ids differ"
    assert digest(primary_of(r_off, np.asarray(out[1]))) == g[tag + "primary_sha"]
    for k in ("r_t", "r_dist", "r_udf"):
        assert digest(np.asarray(out[SAMPLE_FIELDS.index(k)])) == g[tag + k + "_sha"], \
            f"{tag}: {k} not bit-exact"
    sub = csr_rows(r_off, rows, *out[1:7], out[7] if len(out[7]) else np.zeros((len(out[1]), 3)))
    for k, v in zip(SAMPLE_FIELDS[:8], sub):
        ref = g[tag + k]
        if k == "r_color" and g[tag + "r_color_sha"] == digest(np.zeros((0, 3))):
            continue
        if exact_values or k in ("r_off", "r_id", "r_t", "r_dist", "r_udf"):
            np.testing.assert_array_equal(v, ref, err_msg=f"{tag}{k}")
        else:
            np.testing.assert_allclose(v, ref, rtol=VAL_RTOL, atol=0, err_msg=f"{tag}{k}")
    if check_t_end:
        t_end = np.asarray(out[8])[rows]
        if exact_values:
            np.testing.assert_array_equal(t_end, g[tag + "t_end"])
        else:
            np.testing.assert_allclose(t_end, g[tag + "t_end"], rtol=VAL_RTOL, atol=1e-300)
