"""Generate tests/golden/*.npz by running the REFERENCE hashpoint package.

Runs only in the dev container (the reference is not on the GPU box).  The
reference is imported read-only from /root/reference/pkg/src with numba's cache
and Python bytecode redirected away from the source tree.

For every case of tests/golden_cases.py it records, from the reference:
  * build:  table_start, table_count, reordered_ids, slot_{x,y,z}
            (hash_index.build, hash_index.py:151-190) and the rasterized
            bucket of every point (rasterize_points, hash_index.py:95-112);
  * query:  offsets, ids, t_proj, dist_perp, probes, scanned
            (query_batch_arrays, hash_index.py:212-235);
  * sample: the 9-tuple of sample_batch_arrays (sampler.py:196-217) for each
            sampler configuration, with colours;
  * primary-surface point per ray (r_id[r_off[r]] or -1).
Small cases store full arrays; large ones (cfg1) store sha256 digests of every
full array plus explicit arrays for a strided ray subset.

Usage:  python oracle/make_golden.py
"""

from __future__ import annotations

import hashlib
import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "hp_numba_cache"))
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import hashpoint  # noqa: E402  (the reference)
from hashpoint import geometry as rgeo  # noqa: E402
from hashpoint import hash_index as ridx  # noqa: E402
from hashpoint import sampler as rsam  # noqa: E402
from hashpoint.cloud import PointCloud as RefCloud  # noqa: E402

import golden_cases  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
BIG_RAY_STRIDE = 97


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def ref_camera(cam):
    return rgeo.Camera(np.array(cam.origin), np.array(cam.orientation), cam.focal_length,
                       cam.width, cam.height, cam.pixel_width, cam.pixel_height)


def csr_subset(off, rows, *arrays):
    """Slice per-ray segments of CSR arrays for the given rays."""
    counts = off[rows + 1] - off[rows]
    sub_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    idx = np.concatenate([np.arange(off[r], off[r + 1]) for r in rows]) if len(rows) else \
        np.zeros(0, np.int64)
    idx = idx.astype(np.int64)
    return (sub_off,) + tuple(a[idx] for a in arrays)


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, cloud, cam, cfg, tn, tf, stride, samplers in golden_cases.cases():
        rcam = ref_camera(cam)
        rcfg = rgeo.SearchConfig(cfg.kernel_radius, cfg.pixel_disc_radius, cfg.use_approx_radius)
        assert rcfg.kernel_size == cfg.kernel_size
        rcloud = RefCloud(cloud.positions, cloud.colors)
        index = ridx.build(rcloud, rcam, rcfg)
        ok, pu, pv = ridx.rasterize_points(cloud.positions, rcam, rcfg.pad)
        wp = cam.width + 2 * rcfg.pad
        bucket = np.where(ok, pv * wp + pu, -1).astype(np.int64)
        pixels, dirs, t_near, t_far = golden_cases.rays_for(cam, tn, tf, stride)
        q = ridx.query_batch_arrays(index, pixels, dirs, t_near, t_far, rcfg)
        slopes = rgeo.radius_slopes(rcam, pixels, rcfg.kernel_radius, rcfg.use_approx_radius)
        big = cloud.count > 20_000
        rec = {"positions_sha": digest(cloud.positions), "kernel_size": cfg.kernel_size,
               "pad": cfg.pad}
        build_arrays = dict(table_start=index.table_start, table_count=index.table_count,
                            reordered_ids=index.reordered_ids, slot_x=index.slot_x,
                            slot_y=index.slot_y, slot_z=index.slot_z, bucket=bucket)
        qnames = ["offsets", "ids", "t_proj", "dist_perp", "probes", "scanned"]
        for k, v in build_arrays.items():
            rec["build_" + k + "_sha"] = digest(v)
            if not big:
                rec["build_" + k] = v
        for k, v in zip(qnames, q):
            rec["query_" + k + "_sha"] = digest(v)
        rows = np.arange(0, pixels.shape[0], BIG_RAY_STRIDE if big else 1)
        rec["rows"] = rows
        sub = csr_subset(q[0], rows, q[1], q[2], q[3])
        for k, v in zip(qnames[:4], sub):
            rec["query_" + k] = v
        rec["query_probes"] = q[4][rows]
        rec["query_scanned"] = q[5][rows]
        snames = ["r_off", "r_id", "r_t", "r_dist", "r_udf", "r_alpha", "r_w", "r_color", "t_end"]
        for sname in samplers:
            scfg = rsam.SamplerConfig(**golden_cases.SAMPLERS[sname])
            for colored in ((True, False) if sname == "default" else (True,)):
                cols = cloud.colors if colored else None
                s = rsam.sample_batch_arrays(q[0], q[1], q[2], q[3], slopes, scfg, cols)
                tag = f"sample_{sname}{'' if colored else '_nocolor'}_"
                for k, v in zip(snames, s):
                    rec[tag + k + "_sha"] = digest(v)
                r_off = s[0]
                primary = np.where(r_off[1:] > r_off[:-1],
                                   s[1][np.minimum(r_off[:-1], max(len(s[1]) - 1, 0))]
                                   if len(s[1]) else -1, -1).astype(np.int64)
                rec[tag + "primary_sha"] = digest(primary)
                rec[tag + "primary"] = primary[rows]
                ssub = csr_subset(r_off, rows, *s[1:7], s[7] if colored else np.zeros((len(s[1]), 3)))
                for k, v in zip(snames[:8], ssub):
                    rec[tag + k] = v
                rec[tag + "t_end"] = s[8][rows]
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **{k: np.asarray(v) for k, v in rec.items()})
        print(f"{name}: n={cloud.count} m={pixels.shape[0]} Q={len(q[1])} "
              f"s={cfg.kernel_size} -> {os.path.getsize(path) / 1e3:.0f} kB")
    print("reference version", hashpoint.__version__)


if __name__ == "__main__":
    main()
