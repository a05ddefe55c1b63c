#!/usr/bin/env python
"""HashPoint B200 benchmark: rays/s of hash build + per-ray query +
primary-surface sampling (BASELINE.json metric) on the cfg2 workload.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one frame: build the index of a 1M-point sphere-shell cloud for an
800x800 view (delta = 0.01 -> 41x41 kernel), query all 640,000 rays, sample
them (K = 8, eps retention, colours, exact transmittance).  Inputs are
synthetic (seeded generators of the reference) and resident in HBM when the
timed region starts; L2 is flushed (256 MB write) between timed steps.  With
N > 1 (torchrun) the rays are split into contiguous row bands (equal-cost by
the per-ray scan counts) and every rank runs its band of the same frame; the
retained samples are gathered to rank 0 with NCCL; the step time is the max
over ranks.

--impl reference runs the reference algorithm on the host CPU (the C oracle,
a step-for-step restatement of the reference's numba kernels, all host
threads) on a strided ray subset of the same frame and extrapolates.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (scene kwargs, (W, H, fov), delta)
    "cfg2": (dict(kind="sphere_surface", n=1_000_000, seed=0, noise=0.005), (800, 800, 40.0), 0.01),
    "cfg1": (dict(kind="sphere_surface", n=100_000, seed=0, noise=0.005), (200, 200, 40.0), 0.01),
    # dense large scene, smallest delta of the sweep: Q ~ 4.3e9 does not fit
    # one GPU's memory in one pass -> ray-chunk streaming (pipeline)
    "cfg4": (dict(kind="sphere_surface", n=10_000_000, seed=0, noise=0.005), (1920, 1080, 40.0), 0.005),
    # the rest of the cfg4 radius sweep (Q ~ 1.7e10 / 6.9e10: several ray chunks per frame)
    "cfg4_d01": (dict(kind="sphere_surface", n=10_000_000, seed=0, noise=0.005), (1920, 1080, 40.0), 0.01),
    "cfg4_d02": (dict(kind="sphere_surface", n=10_000_000, seed=0, noise=0.005), (1920, 1080, 40.0), 0.02),
    # full render step: cfg2's search + sampling (with the K neighbours emitted)
    # + the Point-NeRF aggregation MLP (bf16, tcgen05) + volume compositing
    "cfg5": (dict(kind="sphere_surface", n=1_000_000, seed=0, noise=0.005), (800, 800, 40.0), 0.01),
}
# ScanNet-shaped indoor batch: 64 views orbiting a multi-plane cloud, one
# index per view; views are sharded across ranks
CFG3 = dict(scene=dict(kind="parallel_planes", n=3_000_000, seed=0, plane_count=6, plane_gap=0.5,
                       extent=4.0, noise=0.005), size=(640, 480, 60.0), delta=0.01, views=64)
# rays checked against the oracle before timing / timed on the host CPU
# (the oracle runs the reference's O(q^2) sampler: sparser subsets for the larger radii)
PARITY_STRIDE = {"cfg1": 53, "cfg2": 53, "cfg5": 53, "cfg4": 4999, "cfg4_d01": 20011, "cfg4_d02": 200003}
CPU_STRIDE = {"cfg1": 97, "cfg2": 97, "cfg5": 97, "cfg4": 20011, "cfg4_d01": 200003, "cfg4_d02": 1000003}
T_NEAR, T_FAR = 1.0, 10.0


def make_workload(name):
    import paper_2404_14044_b200 as hp
    scene, (W, H, fov), delta = WORKLOADS[name]
    cloud = hp.generate_scene(hp.SceneSpec(**scene))
    cam = hp.scene_camera(W, H, fov_deg=fov)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, T_NEAR, delta),
                          hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    m = dirs.shape[0]
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius, cfg.use_approx_radius)
    return dict(name=name, cloud=cloud, cam=cam, cfg=cfg, dirs=dirs, pixels=pixels,
                t_near=np.full(m, T_NEAR), t_far=np.full(m, T_FAR), slopes=slopes, m=m,
                delta=delta)


def make_views(n_views=None):
    """cfg3: the cloud and the 64 orbiting views (camera, config, rays)."""
    import paper_2404_14044_b200 as hp
    cloud = hp.generate_scene(hp.SceneSpec(**CFG3["scene"]))
    W, H, fov = CFG3["size"]
    views = []
    for k in range(n_views or CFG3["views"]):
        th = 2.0 * np.pi * k / CFG3["views"]
        cam = hp.scene_camera(W, H, fov_deg=fov, origin=(0.4 * np.cos(th), 0.4 * np.sin(th), 0.0),
                              target=(0.0, 0.0, 4.0))
        cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, T_NEAR, CFG3["delta"]),
                              hp.pixel_disc_radius(cam))
        dirs, pixels = hp.ray_grid(cam)
        slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius, cfg.use_approx_radius)
        views.append(dict(cam=cam, cfg=cfg, dirs=dirs, pixels=pixels, slopes=slopes, m=dirs.shape[0]))
    return cloud, views


def run_views(args, rank, world, dist):
    """cfg3: every rank builds, queries and samples its share of the 64 views
    (views[rank::world]; no collective on the data path); the step time is
    the max over ranks; value = all views' rays / step time.  Parity gate
    (rank 0, after timing): every view's index (hence every point's bucket,
    the rotated-camera hazard of geometry.py:122-134) against the oracle's
    build, and every 8th view's timed samples on every 97th ray."""
    import torch

    import paper_2404_14044_b200 as hp
    from paper_2404_14044_b200 import _lib, device as dv, pipeline
    dev = torch.device("cuda", local_device())
    torch.cuda.set_device(dev)
    cloud, views = make_views(args.views)
    mine = list(range(len(views)))[rank::world]
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    xyz, col = up(cloud.positions), up(cloud.colors)
    rays = {i: [up(views[i]["pixels"]), up(views[i]["dirs"]), up(np.full(views[i]["m"], T_NEAR)),
                up(np.full(views[i]["m"], T_FAR)), up(views[i]["slopes"])] for i in mine}
    scfg = hp.SamplerConfig()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    gated = [i for i in mine if i % 8 == 0]
    kept = {}

    counts = {"head_resorted_rays": 0, "full_path_rays": 0}

    def step(keep=False):
        Q = R = 0
        counts["head_resorted_rays"] = counts["full_path_rays"] = 0
        for i in mine:
            v = views[i]
            fr = pipeline.frame_device(xyz, col, v["cam"], v["cfg"], *rays[i], scfg, True)
            Q += fr.Q
            R += fr.R
            counts["head_resorted_rays"] += fr.resorted
            counts["full_path_rays"] += fr.flagged
            if keep and i in gated:
                kept[i] = fr.samples
        return Q, R

    for _ in range(args.warmup):
        step()
    times, kern_tot = [], {}
    _lib.timing_enable(True)
    _lib.timing_collect()
    smi = ClockSampler(dev.index)
    with smi:
        for it in range(args.steps):
            flush.fill_(1.0)
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            Q, R = step(keep=it == args.steps - 1)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            for k, (v, c) in _lib.timing_collect().items():
                a0, b0 = kern_tot.get(k, (0.0, 0))
                kern_tot[k] = (a0 + v, b0 + c)
    _lib.timing_enable(False)
    ms = statistics.mean(times)
    qr = (Q, R)
    if dist is not None:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        x = torch.tensor([Q, R], device=dev, dtype=torch.int64)
        dist.all_reduce(x)
        qr = (int(x[0]), int(x[1]))
    e2e = None
    if not args.no_e2e:
        # end to end through the library's multi-view driver: numpy cloud in,
        # every view's numpy 9-tuple out (rays and slopes on the device,
        # view k's copies overlapping view k + 1); max over ranks
        cams, cfgs = [v["cam"] for v in views], [v["cfg"] for v in views]
        et, out = [], {}
        warm = max(args.warmup, 3)  # pinned host buffers reach the caching allocator's steady state
        for it in range(warm + args.steps):
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = pipeline.search_and_sample_views(cloud, cams, cfgs, T_NEAR, T_FAR, dist=dist)
            torch.cuda.synchronize()
            if it >= warm:
                et.append(time.perf_counter() - t0)
        t = torch.tensor([statistics.mean(et), cloud.positions.nbytes + cloud.colors.nbytes
                          + 8 * sum(views[i]["m"] for i in mine),
                          sum(int(x.nbytes) for o in out.values() for x in o)], device=dev, dtype=torch.float64)
        if dist is not None:
            mx = t.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(t)
            t[0] = mx[0]
        e2e = {"value": sum(v["m"] for v in views) / float(t[0]), "unit": "rays/s",
               "h2d_bytes_per_step": int(t[1]), "d2h_bytes_per_step": int(t[2]),
               "api": "paper_2404_14044_b200.pipeline.search_and_sample_views (numpy cloud in, every view's "
                      "numpy 9-tuple out; views[rank::world] per rank)"}
    if rank != 0:
        return
    parity = "skipped"
    if not args.no_parity:
        from oracle import oracle as orc
        bad_builds, checked = [], 0
        for i, v in enumerate(views):  # every view's build, bit for bit
            ob = orc.build(cloud.positions, v["cam"], v["cfg"].pad)
            idx = dv.build(xyz, v["cam"], v["cfg"].pad)
            same = all(np.array_equal(getattr(idx, k).cpu().numpy(), ob[k])
                       for k in ("table_start", "table_count", "reordered_ids", "slot_x", "slot_y", "slot_z"))
            if not same:
                bad_builds.append(i)
            if i in kept:  # this view's timed samples, every 97th ray
                sel = np.arange(0, v["m"], 97)
                ref, _ = oracle_samples(cloud, v["cam"], v["cfg"], v["pixels"][sel], v["dirs"][sel],
                                        np.full(len(sel), T_NEAR), np.full(len(sel), T_FAR), v["slopes"][sel],
                                        build=ob)
                if not same_samples(rays_of(kept[i], sel), ref):
                    raise SystemExit(f"parity gate failed: cfg3 view {i} differs from the oracle; number rejected")
                checked += 1
        if bad_builds:
            raise SystemExit(f"parity gate failed: cfg3 builds of views {bad_builds} differ from the oracle")
        parity = (f"pass ({len(views)} views' builds bit-exact vs the oracle: every point's bucket; timed "
                  f"samples of {checked} views (every 8th) on every 97th ray, ids/t/dist/udf/primary bit-exact, "
                  "alpha/w/colour/t_end rtol 1e-12)")
    m_total = sum(v["m"] for v in views)
    W, H, fov = CFG3["size"]
    line = {
        "metric": "rays/sec (search+primary-surface sampling)", "value": m_total / (ms / 1e3), "unit": "rays/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded reference scene generators)",
        "config": {"workload": f"cfg3: {cloud.count:,}-point 6-plane indoor cloud, {len(views)} orbiting "
                               f"{W}x{H} views (one index each), delta={CFG3['delta']}, t in [{T_NEAR},{T_FAR}], "
                               "SamplerConfig() eps retention K=8 with colours, exact transmittance",
                   "rays": m_total, "views": len(views), "Q": qr[0], "R": qr[1],
                   "l2": "flushed between timed steps (256 MB write)",
                   "parallelism": f"views x{world}" if world > 1 else "single GPU", "parity_gate": parity,
                   **counts},
        "kernels_ms": {k: round(v / args.steps, 3) for k, (v, _) in sorted(kern_tot.items(), key=lambda x: -x[1][0])},
        "clocks": smi.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    print(json.dumps(line), flush=True)


def describe(w):
    c = w["cam"]
    return (f"{w['name']}: {w['cloud'].count:,}-point sphere shell, {c.width}x{c.height} view, "
            f"delta={w['delta']} (s={w['cfg'].kernel_size}), t in [{T_NEAR},{T_FAR}], "
            "SamplerConfig() eps retention K=8 with colours, exact transmittance")


def frame_bytes(n, n_in, P, m, Q, R, colors=True):
    """Algorithmic bytes of one frame."""
    b_build = 24 * n + 16 * P + 32 * n_in
    b_query = 64 * m + 16 * P + 32 * n_in + 8 * (m + 1) + 24 * Q + 16 * m
    b_sample = 8 * (m + 1) + 24 * Q + 8 * m + 8 * (m + 1) + 48 * R + 8 * m + (24 * R if colors else 0)
    return b_build, b_query, b_sample


_CLOCK_CHILD = r"""
import select, sys, pynvml
pynvml.nvmlInit()
try:
    h = pynvml.nvmlDeviceGetHandleByPciBusId(sys.argv[1])
except Exception:
    h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[2]))
bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
        pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
print("ready", flush=True)
rows = []
while not select.select([sys.stdin], [], [], 0.005)[0]:
    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    rows.append("%d %d %s" % (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx,
                              "".join("1" if rs & b else "0" for b in bits)))
print("\n".join(rows), flush=True)
"""


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML
    every 5 ms in a child process (no GIL contention with the timed host
    loop), else nvidia-smi every 0.2 s from a thread."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, set of reason names)
        self.source = None
        self._stop = threading.Event()
        self._t = None
        self._child = None

    def _start_child(self):
        import torch
        p = torch.cuda.get_device_properties(self.index)
        bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        child = subprocess.Popen([sys.executable, "-c", _CLOCK_CHILD, bus, str(self.index)], stdin=subprocess.PIPE,
                                 stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        if child.stdout.readline().strip() != "ready":
            child.kill()
            raise RuntimeError("no NVML")
        return child

    def _run_smi(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                r = [x.strip() for x in out.split(",")]
                if len(r) >= 6 and r[0].replace(".", "").isdigit():
                    self.rows.append((float(r[0]), float(r[1]) if r[1].replace(".", "").isdigit() else None,
                                      {n for n, v in zip(self.NAMES, r[2:6]) if v.lower() == "active"}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        try:
            self._child = self._start_child()
            self.source = "nvml"
        except Exception:
            self._child = None
            self.source = "nvidia-smi"
            self._t = threading.Thread(target=self._run_smi, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._child is not None:
            try:
                out, _ = self._child.communicate(input="stop\n", timeout=30)
                for line in out.splitlines():
                    f = line.split()
                    if len(f) == 3:
                        self.rows.append((float(f[0]), float(f[1]),
                                          {n for n, c in zip(self.NAMES, f[2]) if c == "1"}))
            except Exception:
                self._child.kill()
            return
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows if r[1] is not None]
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(set().union(*[r[2] for r in self.rows])), "samples": len(self.rows),
                "source": self.source}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(span):
    """DRAM bytes (read + write) of one occurrence of a timing span, from the
    committed `ncu --set full` summary of the same bench command
    (profiles/*_ncu_full.json, scripts/ncu_summary.py); None if absent."""
    import glob
    # newest capture first: the names sort by round / version (mtimes do not survive a checkout)
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_full.json")), key=os.path.basename)
    for f in reversed(files):
        try:
            sp = json.load(open(f))["spans"].get(span)
        except Exception:
            continue
        if sp:
            return float(sp["dram_bytes"]), os.path.relpath(f, ROOT)
    return None, None


# --------------------------------------------------------------------------- CPU legs
def cpu_run(w, stride, threads):
    """Reference algorithm on the host (C oracle): full build, strided rays."""
    from oracle import oracle as orc
    cam, cfg, cloud = w["cam"], w["cfg"], w["cloud"]
    t0 = time.perf_counter()
    b = orc.build(cloud.positions, cam, cfg.pad)
    t_build = time.perf_counter() - t0
    sel = slice(0, None, stride)
    px = np.ascontiguousarray(w["pixels"][sel])
    t0 = time.perf_counter()
    q = orc.query(b["table_start"], b["table_count"], b["slot_x"], b["slot_y"], b["slot_z"],
                  b["reordered_ids"], cam.width + 2 * cfg.pad, cfg.pad, px[:, 0], px[:, 1],
                  w["dirs"][sel], cam.origin, w["t_near"][sel], w["t_far"][sel], w["slopes"][sel],
                  threads=threads)
    from paper_2404_14044_b200.sampler import SamplerConfig
    sc = SamplerConfig()
    orc.sample(*q[:4], w["slopes"][sel], sc.k_neighbors, sc.beta * sc.beta, sc.gamma, True,
               sc.epsilon, sc.tau_min, cloud.colors, threads=threads)
    t_sub = time.perf_counter() - t0
    m_sub = px.shape[0]
    secs = t_build + (w["m"] / m_sub) * t_sub
    return w["m"] / secs, dict(t_build_s=t_build, t_subset_s=t_sub, m_sub=m_sub)


def reference_numba_run(w, stride, threads):
    """The reference's OWN CPU path (hashpoint from baseline/_ref, numba,
    unmodified): hash_index.build, then query_batch_arrays +
    sample_batch_arrays on every stride-th ray of the frame, split into
    interleaved ray chunks over a thread pool (the kernels are nogil,
    _kernels.py:19; chunks are independent, hash_index.py:263-293), as the
    reference's bench convention times them (bench.py:175-199).  Returns
    (rays/s extrapolated to the frame, info) or None when the reference or
    numba is not importable."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "hashpoint")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/hp_numba_cache")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import hashpoint as R
        from hashpoint import geometry as RG, hash_index as RH, sampler as RS
    except Exception:
        return None
    from concurrent.futures import ThreadPoolExecutor
    scene, (W, H, fov), delta = WORKLOADS[w["name"]]
    cloud = R.generate_scene(R.SceneSpec(**scene))
    cam = R.scene_camera(W, H, fov_deg=fov)
    cfg = R.SearchConfig(R.kernel_radius_for_min_radius(cam, T_NEAR, delta), R.pixel_disc_radius(cam))
    dirs, pixels = RG.ray_grid(cam)
    sc = R.SamplerConfig()

    def run(idx, sel):
        px = np.ascontiguousarray(pixels[sel])
        m = len(px)
        tn, tf = np.full(m, T_NEAR), np.full(m, T_FAR)
        q = RH.query_batch_arrays(idx, px, dirs[sel], tn, tf, cfg)
        sl = RG.radius_slopes(cam, px, cfg.kernel_radius, cfg.use_approx_radius)
        RS.sample_batch_arrays(q[0], q[1], q[2], q[3], sl, sc, cloud.colors)

    small = R.generate_scene(R.SceneSpec("sphere_surface", n=2000, seed=1))  # numba JIT compile, untimed
    run(RH.build(small, cam, cfg), np.arange(0, len(dirs), max(len(dirs) // 64, 1)))
    t0 = time.perf_counter()
    idx = RH.build(cloud, cam, cfg)
    t_build = time.perf_counter() - t0
    sel = np.arange(0, len(dirs), stride)
    chunks = [sel[c::threads] for c in range(threads)]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda c: run(idx, c), chunks))
    t_sub = time.perf_counter() - t0
    secs = t_build + (len(dirs) / len(sel)) * t_sub
    return len(dirs) / secs, dict(t_build_s=t_build, t_subset_s=t_sub, m_sub=len(sel))


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, w, rank, world):
    """--impl reference: the reference's own CPU path (numba, from
    baseline/_ref) on all host threads, each step a bounded strided ray
    subset of the frame extrapolated to the frame; the C restatement of the
    same algorithm (oracle/hp_oracle.c) is timed beside it.  Falls back to
    the C port if the reference cannot be imported."""
    if rank != 0:
        return
    threads = host_threads()
    stride = args.cpu_stride
    vals, info, kind = [], None, "reference"
    for _ in range(args.steps):
        r = reference_numba_run(w, stride, threads)
        if r is None:
            kind = "port"
            break
        vals.append(r[0])
        info = r[1]
    port_vals = []
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_run(w, stride * 4, threads)
    for _ in range(1 if kind == "reference" else args.steps):
        v, pinfo = cpu_run(w, stride, threads)
        port_vals.append(v)
    if kind == "port":
        vals, info = port_vals, pinfo
    value = statistics.median(vals)
    port = statistics.median(port_vals)
    sample = (f"full build + every {stride}th ray ({info['m_sub']} rays) of the frame through query+sample on "
              f"{threads} threads (interleaved chunks), extrapolated to {w['m']} rays; " +
              ("the reference's own numba path (hashpoint from baseline/_ref: hash_index.build, "
               "query_batch_arrays, sample_batch_arrays)" if kind == "reference" else
               "C restatement of the reference kernels (oracle/hp_oracle.c)") + f"; {cpu_model()}")
    line = {
        "impl": "reference", "metric": "rays/sec (search+primary-surface sampling)",
        "value": value, "unit": "rays/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * w["m"] / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": describe(w), "rays": w["m"], "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": threads, "kind": kind, "sample": sample,
                         "c_port_rays_per_s": port},
        "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU leg
def local_device():
    import torch
    return int(os.environ.get("LOCAL_RANK", 0)) % max(torch.cuda.device_count(), 1)



def row_bands(w, world, rank):
    """Contiguous ray range of this rank (whole image rows, cost-balanced by
    the slots each ray's window scans, from the device index's table; every
    rank computes the same split)."""
    import torch

    from paper_2404_14044_b200 import device as dv
    from paper_2404_14044_b200.shard import balanced_row_bands
    dev = torch.device("cuda", local_device())
    idx = dv.build(torch.from_numpy(np.ascontiguousarray(w["cloud"].positions)).to(dev), w["cam"], w["cfg"].pad)
    lo, hi = balanced_row_bands(None, w["cam"], w["cfg"].pad, world, table_count=idx.table_count)[rank]
    W = w["cam"].width
    return lo * W, hi * W


def run_ours(args, w, rank, world, dist):
    import torch

    import paper_2404_14044_b200 as hp
    from paper_2404_14044_b200 import _lib, device as dv, pipeline
    from paper_2404_14044_b200.shard import gather_samples

    dev = torch.device("cuda", local_device())
    torch.cuda.set_device(dev)
    r0, r1 = row_bands(w, world, rank) if world > 1 else (0, w["m"])
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    xyz = up(w["cloud"].positions)
    col = up(w["cloud"].colors)
    rays = [up(w["pixels"][r0:r1]), up(w["dirs"][r0:r1]), up(w["t_near"][r0:r1]),
            up(w["t_far"][r0:r1]), up(w["slopes"][r0:r1])]
    scfg = hp.SamplerConfig()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    render = w["name"] == "cfg5"
    if render:
        from paper_2404_14044_b200.pointnerf import PointNeRFMLP, render_step
        mlp = PointNeRFMLP(w["cloud"].count, seed=0, device_=dev)

    # a row band (N > 1): the index holds only the points its rays can reach
    band_rows = None
    if world > 1 and r1 > r0:
        v = w["pixels"][r0:r1, 1]
        band_rows = (int(v.min()), int(v.max()) + 1)

    def step(timer=None):
        fr = pipeline.frame_device(xyz, col, w["cam"], w["cfg"], *rays, scfg, True, timer, emit_knn=render,
                                   rows=band_rows)
        if render:  # the full render step: aggregation MLP + compositing of this rank's rays
            fr.image = render_step(mlp, fr.samples, rays[1], w["cam"].origin, xyz, rays[0], rays[3],
                                   w["cam"].width, w["cam"].height)
        if world > 1:
            gather_samples(fr.samples[:9], dist)
        return fr

    for _ in range(args.warmup):
        fr = step()
    torch.cuda.synchronize()
    times, stage_tot, kern_tot = [], {}, {}
    launches0 = _lib.launch_count()
    _lib.timing_enable(True)
    _lib.timing_collect()
    smi = ClockSampler(dev.index)
    with smi:
        for _ in range(args.steps):
            flush.fill_(1.0)
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            timer = pipeline.StageTimer()
            dv.TIMER = timer
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fr = step(timer)
            e1.record()
            dv.TIMER = None
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            for k, v in timer.spans().items():
                stage_tot[k] = stage_tot.get(k, 0.0) + v
            for k, (v, c) in _lib.timing_collect().items():
                a, b = kern_tot.get(k, (0.0, 0))
                kern_tot[k] = (a + v, b + c)
    _lib.timing_enable(False)
    launches = _lib.launch_count() - launches0
    # parity gate on the last timed frame's own output
    parity = "skipped"
    if rank == 0 and not args.no_parity:
        parity = parity_gate(w, fr.samples[:9], r0, r1, PARITY_STRIDE.get(w["name"], 53))
    ms = statistics.mean(times)
    if dist is not None:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    stages = {k: v / args.steps for k, v in stage_tot.items()}
    QR_total = (fr.Q, fr.R)
    if dist is not None:  # whole-job candidate / sample counts
        qr = torch.tensor([fr.Q, fr.R], device=dev, dtype=torch.int64)
        dist.all_reduce(qr)
        QR_total = (int(qr[0]), int(qr[1]))

    # end-to-end through the public host-buffer API (pinned host inputs); at
    # N > 1 every rank runs its band concurrently, max time over ranks
    # one more (untimed) frame for the prefix kernel's bytes: Σ prefix length
    pipeline.TRACK_PREFIX_LEN = True
    pipeline.FLAG_REASONS.clear()
    plen_fr = step()
    pipeline.TRACK_PREFIX_LEN = False
    flag_reasons = [int(x) for x in sum(pipeline.FLAG_REASONS).cpu()] if pipeline.FLAG_REASONS else None
    e2e = None
    if not args.no_e2e and not render:
        e2e = run_e2e(args, w, r0, r1, dist)
    if rank != 0:
        return
    m_total = w["m"]
    value = m_total / (ms / 1e3)
    n, P = w["cloud"].count, fr.index.padded_width * fr.index.padded_height
    Q, R = QR_total
    bb, bq, bs = frame_bytes(n, fr.index.n_in, P, m_total, Q, R)
    peak, peak_kind = measured_peaks()
    # per-kernel algorithmic bytes of this rank's frame (inputs read once,
    # outputs written once).  Sort classes by the match counts.
    n_in = fr.index.n_in
    m_loc, q_loc, r_loc = r1 - r0, fr.Q, fr.R
    qs = np.diff(fr.query[0].cpu().numpy()) if fr.query is not None else np.zeros(0, np.int64)
    cls = {"k_query_sort": (qs > 0) & (qs <= 2048), "k_query_sort_large": qs > 2048}
    st = plen_fr.prefix_len.cpu().numpy() if plen_fr.prefix_len is not None else np.zeros(4, np.int64)
    plen, q_cut, q_whole, hit = (int(x) for x in st)
    kbytes = {
        # the query layout alone: xyz in, counts / scan / row pointers, 100 B out per placed point
        "hp_build": 24 * n + 16 * P + 4 * (P + 1) + 4 * n + 100 * n_in,
        "k_query_bound": 64 * m_loc + 4 * (P + 1) + 8 * m_loc,
        # rays in (64 B), row pointers, the fp32 copies (16 B / point), 8 B per
        # match out, per-ray counts / head counts / key bounds / probes / scanned
        "k_head_scan": 64 * m_loc + 4 * (P + 1) + 16 * n_in + 8 * q_loc + 56 * m_loc,
        # the cut rays' keys and slots (4 + 4 B / match) in, their selected
        # slots (4 B each, ~ the cut rays' head) and per-ray selection (16 B) out
        "k_head_select": 8 * q_cut + 4 * max(plen - q_whole, 0) + 16 * m_loc,
        # slots of whole rays (scratch) and of cut rays (the selection), exact
        # records (32 B / point, once), heads out (t, id32, dist: 20 B) and
        # per-ray inputs / outputs
        "k_head_sort": 4 * q_whole + 4 * max(plen - q_whole, 0) + 32 * n_in + 20 * plen + 112 * hit,
        "k_sample_plan": 8 * (m_loc + 1) + 16 * plen + 8 * m_loc + 24 * m_loc,
        "k_emit": 8 * (m_loc + 1) + 52 * r_loc + 24 * r_loc + 72 * r_loc,
    }
    for k, sel in cls.items():  # read the unsorted matches (20 B), write the CSR (24 B)
        kbytes[k] = 44 * int(qs[sel].sum()) + 24 * int(sel.sum())
    kern = {k: (v / args.steps, c // args.steps) for k, (v, c) in kern_tot.items()}
    top = max((k for k in kern if k in kbytes), key=lambda k: kern[k][0])
    t_top = kern[top][0] / max(kern[top][1], 1)
    b_top = kbytes[top] / max(kern[top][1], 1)
    achieved = b_top / (t_top / 1e3) / 1e9 if t_top > 0 else 0.0
    # the committed ncu capture is of the default command (cfg2, 1 GPU)
    traffic, traffic_src = ncu_traffic(top) if (args.workload == "cfg2" and world == 1) else (None, None)
    line = {
        "metric": "rays/sec (search+primary-surface sampling)", "value": value, "unit": "rays/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded reference scene generators)",
        "config": {"workload": describe(w), "rays": m_total, "n_points": n,
                   "n_indexed": fr.index.n_in, "Q": Q, "R": R, "P": P,
                   "l2": "flushed between timed steps (256 MB write)",
                   "parallelism": f"row bands x{world}" if world > 1 else "single GPU",
                   "ray_chunks": fr.chunks, "prefix_mode": fr.prefix, "head_resorted_rays": fr.resorted,
                   "full_path_rays": fr.flagged,
                   "flag_reasons": flag_reasons,
                   "parity_gate": parity},
        "roofline": {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes": b_top, "traffic_source": traffic_src,
                     "peak_source": peak_kind},
        "frame_roofline": {"bytes": bb + bq + bs, "achieved_gbs": (bb + bq + bs) / (ms / 1e3) / 1e9,
                           "frac": (bb + bq + bs) / (ms / 1e3) / 1e9 / peak,
                           # a path that never materialises the query CSR,
                           # reported beside B_frame, not divided by it
                           "b_fused": 24 * n + 64 * fr.index.n_in + 32 * P + 96 * m_total + 48 * R
                           if fr.prefix else None,
                           "head_len": plen if plen_fr.prefix_len is not None else None},
        "stages_ms": {k: round(v, 4) for k, v in stages.items()},
        "kernels_ms": {k: round(v[0], 4) for k, v in sorted(kern.items(), key=lambda x: -x[1][0])},
        "kernels_gbs": {k: round(kbytes[k] / (kern[k][0] / 1e3) / 1e9, 1) for k in kern if k in kbytes
                        and kern[k][0] > 0},
        "gpu_launches": launches,
        "clocks": smi.summary(),
    }
    if render:  # the MLP kernels against the tensor-core peak
        R_all, Kn = fr.R, scfg.k_neighbors
        flops = {"k_mlp_agg": R_all * Kn * 2 * (64 * 128 + 128 * 128), "k_mlp_head": R_all * 2 * (128 * 64 + 64 * 4)}
        tf_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]) \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1590.0
        line["mlp_roofline"] = {
            "bound": "tensor", "unit": "TFLOP/s", "peak": tf_peak, "peak_source": "measured bf16 burst (cuBLAS)",
            "kernels": {k: {"ms": kern[k][0], "flop": f, "achieved": f / (kern[k][0] / 1e3) / 1e12,
                            "frac": f / (kern[k][0] / 1e3) / 1e12 / tf_peak} for k, f in flops.items() if k in kern},
            "rows": R_all * Kn, "samples": R_all, "k": Kn}
        line["config"]["workload"] = ("cfg5: cfg2 search + primary-surface sampling (K=8 neighbours emitted) + "
                                      "Point-NeRF aggregation MLP (bf16 tcgen05: 64->128->128 per neighbour, "
                                      "weighted sum, 128->64->4 head) + volume compositing; random-init weights")
    if e2e is not None:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1:
        v, info = cpu_run(w, args.cpu_stride, host_threads())
        ref = reference_numba_run(w, args.cpu_stride, host_threads()) if w["name"] != "cfg5" else None
        line["cpu_baseline"] = {"value": v, "unit": "rays/s", "cores": host_threads(), "kind": "port",
                                "sample": f"full build + every {args.cpu_stride}th ray "
                                          f"({info['m_sub']} rays) through query+sample, "
                                          f"extrapolated; oracle/hp_oracle.c; {cpu_model()}"}
        if ref is not None:
            line["cpu_baseline"]["reference_numba"] = {
                "value": ref[0], "unit": "rays/s", "cores": host_threads(), "kind": "reference",
                "sample": f"the reference's own numba path (baseline/_ref hashpoint), same subset "
                          f"({ref[1]['m_sub']} rays), interleaved chunks over the host threads"}
    print(json.dumps(line), flush=True)


def run_e2e(args, w, r0, r1, dist=None):
    """End to end through the public host-buffer API: numpy / pinned host
    inputs in, numpy out, copies inside the timed region.  N = 1:
    pipeline.search_and_sample (rays from the host) and
    search_and_sample_view (rays on the device); N > 1:
    shard.search_and_sample_distributed (every rank its band, the tiles
    gathered to rank 0 inside the timed region), max over ranks."""
    import torch

    from paper_2404_14044_b200 import pipeline, shard
    m = r1 - r0
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731

    class PinnedCloud:  # PointCloud-like view over pinned host tensors
        positions = pin(w["cloud"].positions)
        colors = pin(w["cloud"].colors)
    cloud = PinnedCloud()
    cam = w["cam"]
    tn, tf = w["t_near"], w["t_far"]
    if dist is not None:
        times, out = [], None
        for i in range(args.warmup + args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = shard.search_and_sample_distributed(cloud, cam, w["cfg"], float(tn[0]), float(tf[0]), dist)
            torch.cuda.synchronize()
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
        sec = statistics.mean(times)
        h2d = cloud.positions.numel() * 8 + cloud.colors.numel() * 8 + 8 * m
        d2h = sum(int(x.nbytes) for x in out) if out is not None else 0
        dev = torch.device("cuda", torch.cuda.current_device())
        t = torch.tensor([sec, h2d, d2h], device=dev, dtype=torch.float64)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return {"value": w["m"] / float(mx[0]), "unit": "rays/s", "h2d_bytes_per_step": int(t[1]),
                "d2h_bytes_per_step": int(t[2]),
                "api": "paper_2404_14044_b200.shard.search_and_sample_distributed (numpy in on every rank, the "
                       "view's 9-tuple out on rank 0; row bands, device rays, gather to rank 0)"}
    warm = max(args.warmup, 3)  # the host-buffer path reaches its steady allocator state after a few calls

    def timed(cl, px, dr, a, b):
        times, out = [], None
        for i in range(warm + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = pipeline.search_and_sample(cl, cam, w["cfg"], px, dr, a, b)
            torch.cuda.synchronize()
            if i >= warm:
                times.append(time.perf_counter() - t0)
        return statistics.mean(times), out

    # headline: plain numpy arrays in (pageable; the library stages them
    # through pinned memory with host threads), numpy out
    sec, out = timed(w["cloud"], w["pixels"][r0:r1], w["dirs"][r0:r1], tn[r0:r1], tf[r0:r1])
    # the same with pinned torch tensors in (what a caller that keeps its
    # buffers pinned pays)
    psec, _ = timed(cloud, pin(w["pixels"][r0:r1]), pin(w["dirs"][r0:r1]), pin(tn[r0:r1]), pin(tf[r0:r1]))
    h2d = (cloud.positions.numel() * 8 + cloud.colors.numel() * 8 + 16 * m + 24 * m + 8 * m + 8 * m
           + 8 * m)
    d2h = sum(int(x.nbytes) for x in out)
    res = {"value": w["m"] / sec, "unit": "rays/s", "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "api": "paper_2404_14044_b200.pipeline.search_and_sample "
                                                 "(numpy arrays in / numpy out)",
           "pinned_inputs": {"value": w["m"] / psec, "unit": "rays/s",
                             "api": "the same call with pinned CPU torch tensors in"}}
    if (w["m"] == cam.width * cam.height and np.all(tn == tn[0]) and np.all(tf == tf[0])
            and np.array_equal(w["pixels"][[0, -1]], [[0, 0], [cam.width - 1, cam.height - 1]])):
        # the same frame as a whole view from plain numpy inputs (pageable
        # copies): rays generated on the device, only the cloud goes up
        npcloud = w["cloud"]
        vt = []
        for i in range(warm + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            vout = pipeline.search_and_sample_view(npcloud, cam, w["cfg"], float(tn[0]), float(tf[0]))
            torch.cuda.synchronize()
            if i >= warm:
                vt.append(time.perf_counter() - t0)
        vsec = statistics.mean(vt)
        res["view"] = {"value": w["m"] / vsec, "unit": "rays/s",
                       "h2d_bytes_per_step": int(npcloud.positions.nbytes + npcloud.colors.nbytes + 8 * m),
                       "d2h_bytes_per_step": int(sum(int(x.nbytes) for x in vout)),
                       "api": "paper_2404_14044_b200.pipeline.search_and_sample_view (numpy arrays in: the "
                              "camera's ray grid and slopes on the device; numpy out)"}
    return res


def rays_of(samples, rays):
    """The listed rays' part of a sampler 9-tuple (device tensors) as numpy,
    CSR offsets rebased (the same layout the oracle returns for those rays)."""
    off = samples[0].cpu().numpy()
    rays = np.asarray(rays, np.int64)
    lo, hi = off[rays], off[rays + 1]
    rows = np.concatenate([np.arange(a, b) for a, b in zip(lo, hi)]) if len(rays) else np.zeros(0, np.int64)
    idx = torch_index(rows, samples[1].device)
    out = [np.concatenate([[0], np.cumsum(hi - lo)]).astype(np.int64)]
    for k in range(1, 7):
        out.append(samples[k][idx].cpu().numpy())
    col = samples[7]
    out.append(col[idx].cpu().numpy() if col.shape[0] else np.zeros((0, 3)))
    out.append(samples[8][torch_index(rays, samples[8].device)].cpu().numpy())
    return out


def torch_index(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(dev)


def same_samples(got, ref, colors=True):
    """Bit-exact r_off / ids / t / dist / udf (and so the primary-surface point,
    the first retained candidate of each ray); alpha / w / colour / t_end
    within rtol 1e-12 (exp() of CUDA vs glibc may differ by an ulp)."""
    ok = all(np.array_equal(got[k], ref[k]) for k in range(5))
    ok &= all(np.allclose(got[k], ref[k], rtol=1e-12, atol=1e-300) for k in (5, 6, 8))
    if colors:
        ok &= np.allclose(got[7], ref[7], rtol=1e-12, atol=1e-300)
    return bool(ok)


def oracle_samples(cloud, cam, cfg, pixels, dirs, tn, tf, slopes, build=None):
    """The reference algorithm (C oracle) on the given rays: build, query, sample."""
    from oracle import oracle as orc
    from paper_2404_14044_b200.sampler import SamplerConfig
    b = build if build is not None else orc.build(cloud.positions, cam, cfg.pad)
    px = np.ascontiguousarray(pixels)
    q = orc.query(b["table_start"], b["table_count"], b["slot_x"], b["slot_y"], b["slot_z"],
                  b["reordered_ids"], cam.width + 2 * cfg.pad, cfg.pad, px[:, 0], px[:, 1],
                  dirs, cam.origin, tn, tf, slopes, threads=host_threads())
    sc = SamplerConfig()
    s = orc.sample(*q[:4], slopes, sc.k_neighbors, sc.beta * sc.beta, sc.gamma, True,
                   sc.epsilon, sc.tau_min, cloud.colors, threads=host_threads())
    return s, int(q[0][-1])


def parity_gate(w, samples, r0, r1, stride):
    """Fairness gate of the reference bench (bench.py:114-134): the TIMED
    frame's own output (the last timed step's samples of rays [r0, r1)) on
    every stride-th ray against the oracle; refuses the number on a mismatch."""
    sel = np.arange(r0, r1, stride)
    got = rays_of(samples, sel - r0)
    ref, Q = oracle_samples(w["cloud"], w["cam"], w["cfg"], w["pixels"][sel], w["dirs"][sel],
                            w["t_near"][sel], w["t_far"][sel], w["slopes"][sel])
    if not same_samples(got, ref):
        raise SystemExit("parity gate failed: the timed frame differs from the oracle; number rejected")
    return (f"pass (timed frame, every {stride}th ray: {len(sel)} rays, Q={Q}, R={len(ref[1])}; "
            "ids/t/dist/udf/primary bit-exact, alpha/w/colour/t_end rtol 1e-12)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + ["cfg3"], default="cfg2")
    ap.add_argument("--cpu-stride", type=int, default=None,
                    help="every k-th ray for the CPU legs (default per workload)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--views", type=int, default=None, help="cfg3: number of the 64 views to run")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.workload == "cfg3":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "cfg3 reference arm not provided "
                              "(64 views x 307k rays on the host CPU); see cfg2"}), flush=True)
            return
        dist = None
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_device())
            dist.init_process_group(os.environ.get("HP_DIST_BACKEND", "nccl"))
        run_views(args, rank, world, dist)
        if dist is not None:
            dist.destroy_process_group()
        return
    w = make_workload(args.workload)
    if args.cpu_stride is None:
        args.cpu_stride = CPU_STRIDE.get(args.workload, 97)
    if args.impl == "reference":
        run_reference(args, w, rank, world)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_device())
        # HP_DIST_BACKEND=gloo: functional check of the N > 1 path on a box
        # with fewer GPUs than ranks (no NCCL); never used for a bench number
        dist.init_process_group(os.environ.get("HP_DIST_BACKEND", "nccl"))
    run_ours(args, w, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
