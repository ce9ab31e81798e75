#!/usr/bin/env python
"""bench.py — the driver's benchmark contract for the octree build + octree
ray-casting hot path (BASELINE.json metric: frame ms & Gsamples/s, 3-ch
1920x1080; octree build GB/s; at 1/2/4/8 GPUs).

Workload (BASELINE.json configs[1], the largest single-GPU config): a
synthetic SPIM-shaped ("S") 3-channel 1024^3 uint16 volume,
32^3 bricks, homogeneity threshold 0, built on the device from
device-resident z-slabs (Octree.insert_channels) + fill_borders; then
1920x1080 DVR frames with per-channel transfer functions, one clipping
plane, early termination 0.99, step 0.5 voxel, LOD bias 0, camera at 2.5x
the extent (voxtree cli.default_scene).  A "step" is one full frame.

  value      pos-samples / s of the whole job (Gsamples/s), device time of the
             render (+ NCCL strip gather for N > 1), CUDA events, max over ranks
  e2e        the same through the public drop-in API with host output
             (OutOfCoreRenderer.render_fullframe -> float64 (H, W, 4) numpy, the
             reference's return type; SortFirstRenderer to_host for N > 1)
  build      device-resident slab ingest GB/s (+ host-slab e2e GB/s)
  roofline   render kernel: 48 B gathered per pos-sample (8 corners x 3 ch x
             2 B) / average kernel duration vs measured HBM copy bandwidth

`--impl reference` times the reference's own CPU implementation (the
unmodified voxtree package from baseline/_ref; the oracle port when that is
absent) on a bounded sample of the same workload on all host cores.
"""

from __future__ import annotations

import argparse
import ctypes as ct
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = (1024, 1024, 1024)
CHANNELS = 3
FMT = "uint16"
BRICK = 32
VIEWPORT = (1920, 1080)
CLIP_FRAC = 0.8
COLORS = ((1.0, 0.25, 0.2), (0.2, 1.0, 0.3), (0.25, 0.45, 1.0))
BYTES_PER_POS_SAMPLE = 8 * CHANNELS * 2  # 8 trilinear corners x C x uint16
L2_FLUSH_BYTES = 512 << 20
FALLBACK_HBM_GBS = 6650.0
WORKLOAD = ("cfg2: synthetic SPIM-shaped 3-ch uint16 volume (1024^3 by default), 32^3 bricks, tau=0, "
            "full octree build + fill_borders; 1920x1080 DVR frame, per-channel TFs, "
            "1 clip plane, ET 0.99, step 0.5 voxel, LOD bias 0")


def scene_for(mod, dims, viewport, lod_bias=0.0, mode="dvr", precision=None):
    """The bench scene, built from either our package's or the reference's
    render module (identical constructors, render/settings.py:70-84)."""
    cx, cy, cz = (d / 2.0 for d in dims)
    extent = float(max(dims))
    cam = mod.Camera(position=(cx, cy, -2.5 * extent), look_at=(cx, cy, cz), up=(0, 1, 0),
                     width=viewport[0], height=viewport[1])
    tfs = [mod.TransferFunction([(0.0, 0, 0, 0, 0), (0.12, 0, 0, 0, 0), (1.0, *col, 0.4)])
           for col in COLORS[:CHANNELS]]
    clips = mod.ClipSet((mod.ClipPlane((0.0, 0.0, 1.0), CLIP_FRAC * dims[2]),))
    st = mod.RenderSettings(mode=mode, early_termination_alpha=0.99, lod_bias=lod_bias)
    if precision is not None:  # B200 extension of RenderSettings
        st.precision = precision
    return mod.Scene(cam, st, tfs, clips)


# ---------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------

def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBps"):
            if k in d:
                return float(d[k]), "measured"
    except (OSError, ValueError):
        pass
    return FALLBACK_HBM_GBS, "fallback"


class Clocks:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            rows = open(self.path).read().strip().splitlines()
        except OSError:
            rows = []
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if self.path:
            os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def traffic_from_profiles(kernel):
    """dram bytes per launch from the committed ncu summary (profiles/)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(kernel)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # VT_DIST_BACKEND=gloo (test only): several ranks may share one GPU, so
    # the multi-rank path can be exercised on a single-GPU box
    backend = os.environ.get("VT_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_1407_2074_b200 import (BrickPoolConfig, DeviceState, Octree, VolumeDescriptor,
                                      _lib)
    from paper_1407_2074_b200 import render as R
    from paper_1407_2074_b200.render.sharded import SortFirstRenderer

    dims = tuple(args.dims)
    desc = VolumeDescriptor(dims=dims, channels=CHANNELS, sample_format=FMT)
    cfg = BrickPoolConfig(brick_dims=(BRICK,) * 3, homogeneity_threshold=0)
    geo_bricks = expected_bricks(dims, BRICK)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    def tree_on_stream(t):
        _lib.call("vt_tree_set_stream", t.handle, ct.c_void_p(stream.cuda_stream))

    # ---- synthetic volume: each rank synthesises (untimed) only the z-slab
    # it ingests; the z-slab sharded build (slab_build.py) inserts it, one
    # all-gather exchanges level <= k node records and every rank ends with
    # the full tree (the replicated pool the sort-first render reads) ----
    from paper_1407_2074_b200.slab_build import build_sharded, slab_plan
    Z, Y, X = dims[2], dims[1], dims[0]
    plan = slab_plan(expected_geometry(dims, BRICK), world)
    sz0, sz1 = plan.slabs[rank]
    vol = torch.empty((max(0, sz1 - sz0), Y, X, CHANNELS), dtype=torch.uint16, device="cuda")
    if sz1 > sz0:
        _lib.call("vt_synth", ct.c_void_p(vol.data_ptr()), 1, _lib.i32x3(dims), CHANNELS, 2, 0,
                  sz0, sz1, ct.c_void_p(stream.cuda_stream))
    raw_bytes = X * Y * Z * CHANNELS * 2  # whole job (all ranks)

    def build(src):
        tree = Octree(desc, cfg, reserve_slots=geo_bricks)
        tree_on_stream(tree)
        torch.cuda.synchronize()
        barrier()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        # device-resident volume: the rank's whole slab is one insertion;
        # host (pinned) volume: brick-layer slabs, so H2D overlaps the build
        slab = max(BRICK, sz1 - sz0) if hasattr(src, "is_cuda") else BRICK
        build_sharded(tree, lambda a, b: src[a - sz0:b - sz0], slab_z=slab, fill_borders=False)
        e1.record(stream)
        tree.finalize()
        tree.fill_borders()
        tree.sync()
        e2.record(stream)
        torch.cuda.synchronize()
        return tree, e0.elapsed_time(e1), e1.elapsed_time(e2)

    # untimed warm-up build (first launches load kernel modules, encode
    # tensor maps, page-lock staging), then three timed builds: the median
    # (by total time) is reported, the last tree is kept for rendering
    wt, _, _ = build(vol)
    wt.close()
    del wt
    torch.cuda.empty_cache()
    runs = []
    for rep in range(3):
        tree, b_ms, f_ms = build(vol)
        runs.append((b_ms + f_ms, b_ms, f_ms))
        if rep < 2:
            tree.close()
            del tree
            torch.cuda.empty_cache()
    _, build_ms, border_ms = sorted(runs)[1]
    pool_bytes = tree.brick_count * cfg.brick_nbytes(desc)
    # every rank must hold the same tree after the sharded build
    ck = tree.checksum()
    replicas_identical = True
    if world > 1:
        cks = [None] * world
        dist.all_gather_object(cks, ck)
        replicas_identical = all(c == ck for c in cks)
    # host-slab (pinned) build through the same public call: e2e ingest
    host = vol.cpu().pin_memory() if args.build_e2e else None
    del vol
    torch.cuda.empty_cache()
    build_e2e_ms = None
    if host is not None:
        # one untimed pass first (staging-pool growth, first H2D of the
        # pinned block), then the timed one, as for the device builds
        for _ in range(2):
            t2, build_e2e_ms, _ = build(host.numpy())
            t2.close()
            del t2
        del host
        torch.cuda.empty_cache()

    dev = DeviceState(tree, resident_all=True)
    scene = scene_for(R, dims, tuple(args.viewport), precision=args.precision)
    sfr = SortFirstRenderer(dev, strip_rows=args.strip_rows)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")

    def frame(sc):
        img, cnt = sfr.render_fullframe(sc, out_kind=R.raycast.OUT_RGBA8)
        return cnt

    times, kms, samples, skipped = [], [], 0, 0
    launches = 0
    with Clocks(local) as clk:
        for it in range(args.warmup + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            cnt = frame(scene)
            e1.record(stream)
            torch.cuda.synchronize()
            if it >= args.warmup:
                times.append(e0.elapsed_time(e1))
                rms = ct.c_double()
                _lib.call("vt_last_kernel_ms", tree.handle, ct.byref(rms), None)
                kms.append(rms.value)
                samples += cnt.samples
                skipped += cnt.samples_skipped
                launches += 1
    clocks = clk.summary()
    rdev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor(times, dtype=torch.float64, device=rdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.sum())
    frame_ms = total_ms / args.steps
    value = samples / (total_ms * 1e-3) / 1e9
    kernel_ms = statistics.mean(kms)
    samples_per_frame = samples / args.steps
    computed_per_frame = (samples - skipped) / args.steps

    # LOD sweep (one flushed frame each, rank-max)
    sweep = {}
    for bias in (-1.0, 0.0, 1.0, 2.0, 3.0):
        sc = scene_for(R, dims, tuple(args.viewport), lod_bias=bias, precision=args.precision)
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cnt = frame(sc)
        e1.record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=rdev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt[0])
        sweep[f"{bias:+.0f}"] = {"frame_ms": round(ms, 3), "samples": cnt.samples,
                                 "gsamples_s": round(cnt.samples / (ms * 1e-3) / 1e9, 3)}

    # e2e: public drop-in API, float64 image to host every frame
    W, H = args.viewport
    e2e_times, e2e_samples = [], 0
    rr = R.OutOfCoreRenderer(dev)
    for it in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if world == 1:
            img, cnt = rr.render_fullframe(scene)
        else:
            img, cnt = sfr.render_fullframe(scene, out_kind=R.raycast.OUT_F64, to_host=True)
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= args.warmup:
            e2e_times.append(e0.elapsed_time(e1))
            e2e_samples += cnt.samples
    t = torch.tensor(e2e_times, dtype=torch.float64, device=rdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = e2e_samples / (float(t.sum()) * 1e-3) / 1e9

    # build numbers: max over ranks (each rank builds its replica)
    bt = torch.tensor([build_ms, border_ms, build_e2e_ms or 0.0], dtype=torch.float64,
                      device=rdev)
    if world > 1:
        dist.all_reduce(bt, op=dist.ReduceOp.MAX)
    build_ms, border_ms, build_e2e_ms = (float(v) for v in bt.tolist())

    if rank == 0:
        peak, peak_kind = hbm_peak()
        # only the samples the kernel actually reconstructs gather bricks
        achieved = computed_per_frame / max(world, 1) * BYTES_PER_POS_SAMPLE / (kernel_ms * 1e-3) / 1e9
        # the build = insertion + fill_borders (ingest_bulk, ingest.py:182-224)
        total_build_ms = build_ms + border_ms
        build_gbs = raw_bytes / (total_build_ms * 1e-3) / 1e9
        build_alg = (raw_bytes + pool_bytes) / (total_build_ms * 1e-3) / 1e9
        out = {
            "metric": "Gsamples/s (3-ch pos-samples, 1920x1080 frame); frame ms; octree build GB/s",
            "value": round(value, 4),
            "unit": "Gsamples/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(frame_ms, 4),
            "frame_ms": round(frame_ms, 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f32 reconstruction / f64 accumulation",
            "data": "synthetic (SPIM-shaped S volume, generated on device, seed 0)",
            "config": {"workload": WORKLOAD, "dims": list(dims), "channels": CHANNELS,
                       "sample_format": FMT, "brick": BRICK, "viewport": list(args.viewport),
                       "parallelism": f"sort-first strips x{world} (strip_rows={args.strip_rows})"
                       if world > 1 else "single GPU",
                       "l2": f"flushed between frames (512 MB write); pool "
                             f"{pool_bytes / 1e9:.1f} GB vs 126 MB L2"},
            "samples_per_frame": int(samples_per_frame),
            "samples_computed_per_frame": int(computed_per_frame),
            "samples_note": "samples = the reference's RenderCounters.samples (identical); "
                            "computed = samples minus those the exact empty-space skip "
                            "accounted without reconstructing (TF alpha provably 0)",
            "render_kernel_ms": round(kernel_ms, 4),
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "traffic": traffic_from_profiles("k_render_fullframe"),
                         "model": "48 B gathered per computed pos-sample / avg render kernel "
                                  "ms (rank 0)"},
            "e2e": {"value": round(e2e_value, 4), "unit": "Gsamples/s",
                    "h2d_bytes_per_step": ct.sizeof(_lib.vt_scene),
                    "d2h_bytes_per_step": W * H * 4 * 8 + 48,
                    "api": "OutOfCoreRenderer.render_fullframe -> float64 (H,W,4) page-locked host "
                           "frame (N=1: the kernel writes it over PCIe)"
                    if world == 1 else "SortFirstRenderer.render_fullframe(to_host=True)"},
            "build": {"raw_gb": round(raw_bytes / 1e9, 3), "pool_gb": round(pool_bytes / 1e9, 3),
                      "bricks": tree.brick_count, "build_ms": round(total_build_ms, 2),
                      "build_runs_ms": [round(r[0], 2) for r in runs],
                      "insert_ms": round(build_ms, 2),
                      "fill_borders_ms": round(border_ms, 2),
                      "gbs_raw": round(build_gbs, 2),
                      "roofline": {"achieved": round(build_alg, 2), "peak": peak,
                                   "frac": round(build_alg / peak, 4), "unit": "GB/s",
                                   "model": "(raw + pool bytes) / (insert + fill_borders) time"},
                      "e2e_gbs_raw": round(raw_bytes / (build_e2e_ms * 1e-3) / 1e9, 2)
                      if build_e2e_ms else None,
                      "e2e_api": "Octree.insert_channels(pinned host slabs, 32 z each)",
                      "sharding": f"z-slab x{world}, level-k={plan.level} records all-gathered"
                      if world > 1 else "single GPU",
                      "tree_checksum": f"{ck:016x}", "replicas_identical": replicas_identical},
            "lod_sweep": sweep,
            "clocks": clocks,
        }
        if world == 1 and args.stream:
            out["stream"] = stream_ingest(args, peak)
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(out), flush=True)
    if world > 1:
        barrier()
        dist.destroy_process_group()


STREAM_DIMS = (2048, 2048, 64)  # cfg3's slice shape, two brick layers


def stream_ingest(args, peak):
    """cfg3-shaped slice stream (ingest_stream's VSTR order: per z, one
    single-channel 2048x2048 block per channel) through Octree.insert_block
    from device-resident slices, then finalize + fill_borders; CUDA events on
    the tree's stream around the whole sequence (host gaps included)."""
    import torch
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib
    dims = STREAM_DIMS
    X, Y, Z = dims
    st = torch.cuda.current_stream()
    vol = torch.empty((Z, Y, X, CHANNELS), dtype=torch.uint16, device="cuda")
    _lib.call("vt_synth", ct.c_void_p(vol.data_ptr()), 1, _lib.i32x3(dims), CHANNELS, 2, 0, 0, Z,
              ct.c_void_p(st.cuda_stream))
    planes = [vol[..., c].contiguous() for c in range(CHANNELS)]
    del vol
    desc = VolumeDescriptor(dims=dims, channels=CHANNELS, sample_format=FMT)
    cfg = BrickPoolConfig(brick_dims=(BRICK,) * 3, homogeneity_threshold=0)
    res = None
    for rep in range(2):  # warm-up, then timed
        tree = Octree(desc, cfg, reserve_slots=expected_bricks(dims, BRICK))
        _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(st.cuda_stream))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for z in range(Z):
            for c in range(CHANNELS):
                tree.insert_block(c, (0, 0, z), planes[c][z:z + 1])
        tree.finalize()
        tree.fill_borders()
        tree.sync()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        raw = X * Y * Z * CHANNELS * 2
        pool = tree.brick_count * cfg.brick_nbytes(desc)
        res = {"workload": f"cfg3-shaped slice stream {X}x{Y}x{Z} x{CHANNELS} uint16, one "
                           "single-channel slice per insert_block (VSTR order), device-resident "
                           "slices, + finalize + fill_borders",
               "inserts": Z * CHANNELS, "ms": round(ms, 2),
               "gbs_raw": round(raw / (ms * 1e-3) / 1e9, 2),
               "roofline": {"achieved": round((raw + pool) / (ms * 1e-3) / 1e9, 2), "peak": peak,
                            "frac": round((raw + pool) / (ms * 1e-3) / 1e9 / peak, 4),
                            "unit": "GB/s", "model": "(raw + pool bytes) / stream time"},
               "tree_checksum": f"{tree.checksum():016x}"}
        tree.close()
        del tree
    del planes
    torch.cuda.empty_cache()
    return res


def expected_geometry(dims, m):
    from paper_1407_2074_b200 import BrickPoolConfig, TreeGeometry, VolumeDescriptor
    desc = VolumeDescriptor(dims=dims, channels=CHANNELS, sample_format=FMT)
    return TreeGeometry.build(desc, BrickPoolConfig(brick_dims=(m,) * 3))


def expected_bricks(dims, m):
    from paper_1407_2074_b200 import BrickPoolConfig, TreeGeometry, VolumeDescriptor
    desc = VolumeDescriptor(dims=dims, channels=CHANNELS, sample_format=FMT)
    geo = TreeGeometry.build(desc, BrickPoolConfig(brick_dims=(m,) * 3))
    n = 0
    for lvl in range(geo.depth + 1):
        sc = 1 << lvl
        n += math.prod(-(-d // (m * sc)) for d in dims)
    return n


# ---------------------------------------------------------------------------
# reference (CPU) arm and the cpu_baseline leg
# ---------------------------------------------------------------------------

CPU_DIMS = (128, 128, 128)
CPU_VIEW_BASE = (192, 108)


def _reference_modules():
    """The unmodified reference (baseline/_ref), else the oracle port."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "voxtree")):
        sys.path.insert(0, ref)
        try:
            import voxtree  # noqa: F401
            from voxtree import render as vr
            return "reference", vr
        except Exception:
            sys.path.remove(ref)
    return "port", None


_CPU_STATE = {}


def _cpu_setup():
    """Build the bounded-sample tree with the reference (or the oracle)."""
    if "tree" in _CPU_STATE:
        return _CPU_STATE
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import voxtree_oracle as vo
    kind, vr = _reference_modules()
    vol = vo.synth_spim(CPU_DIMS, CHANNELS, 65535, seed=0)
    t0 = time.perf_counter()
    if kind == "reference":
        from voxtree.device import DeviceState, RenderMode
        from voxtree.octree import Octree
        from voxtree.volume import BrickPoolConfig, VolumeDescriptor
        tmp = tempfile.mkdtemp(prefix="vtx_ref_")
        desc = VolumeDescriptor(dims=CPU_DIMS, channels=CHANNELS, sample_format=FMT)
        cfg = BrickPoolConfig(brick_dims=(BRICK,) * 3, homogeneity_threshold=0)
        tree = Octree.create(desc, cfg, os.path.join(tmp, "pool.vxbp"))
        for c in range(CHANNELS):
            for z0 in range(0, CPU_DIMS[2], BRICK):
                tree.insert_block(c, (0, 0, z0), np.ascontiguousarray(vol[z0:z0 + BRICK, :, :, c]))
        t_ins = time.perf_counter() - t0
        tree.finalize()
        tree.fill_borders()
        dev = DeviceState(tree, slot_count=tree.brick_count + 8)
        for n in tree.iter_nodes():
            if n.brick is not None:
                dev.flag_buffer[n.index] |= 2
        dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), 1e9)
        _CPU_STATE.update(kind=kind, tree=tree, renderer=vr.OutOfCoreRenderer(dev), mod=vr)
    else:
        ot = vo.OracleTree(CPU_DIMS, (BRICK,) * 3, channels=CHANNELS, fmt=FMT, threshold=0)
        for c in range(CHANNELS):
            for z0 in range(0, CPU_DIMS[2], BRICK):
                ot.insert(c, (0, 0, z0), vol[z0:z0 + BRICK, :, :, c])
        t_ins = time.perf_counter() - t0
        ot.finished = True
        ot.fill_borders()
        nb, bb, _ = vo.resident_buffers(ot)
        _CPU_STATE.update(kind=kind, tree=ot, renderer=vo.OracleRenderer(ot, nb, bb), mod=None)
    _CPU_STATE["build_gbs"] = vol.nbytes / t_ins / 1e9
    return _CPU_STATE


def _cpu_render(view, tile):
    """Render rows [y0, y1) of the sample frame; returns pos-samples."""
    st = _cpu_setup()
    if st["kind"] == "reference":
        sc = scene_for(st["mod"], CPU_DIMS, view)
        sess = st["renderer"].start_refinement(sc, tile=tile)
        while not sess.run_pass():
            pass
        return int(sess.counters.samples)
    import voxtree_oracle as vo
    from paper_1407_2074_b200 import render as R  # scene constructors only (host)
    sc = scene_for(R, CPU_DIMS, view)
    spec = vo.SceneSpec(position=sc.camera.position, look_at=sc.camera.look_at,
                        width=view[0], height=view[1], lod_bias=0.0,
                        tfs=[tf.control_points() for tf in sc.transfer_functions],
                        clips=[(p.normal, p.offset) for p in sc.clips],
                        early_termination_alpha=0.99)
    _, cnt = st["renderer"].render_fullframe(spec, tile=tile)
    return int(cnt["samples"])


def _cpu_worker(job):
    view, tile = job
    return _cpu_render(view, tile)


def cpu_baseline(args):
    """Single-core reference render of the bounded sample (cpu_baseline leg)."""
    st = _cpu_setup()
    view = CPU_VIEW_BASE
    t0 = time.perf_counter()
    samples = _cpu_render(view, (0, 0, view[0], view[1]))
    dt = time.perf_counter() - t0
    return {"value": round(samples / dt / 1e9, 8), "unit": "Gsamples/s", "cores": 1,
            "kind": st["kind"],
            "sample": f"S volume {CPU_DIMS[0]}^3 x3 uint16, 32^3 bricks, same scene at "
                      f"{view[0]}x{view[1]}, all bricks resident: {samples} pos-samples "
                      f"in {dt:.2f} s",
            "build_gbs_raw": round(st["build_gbs"], 5)}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    view = (CPU_VIEW_BASE[0] * 2, CPU_VIEW_BASE[1] * 2)
    rows = max(1, -(-view[1] // (cores * 4)))  # small row tiles: dynamic load balance
    jobs = [(view, (0, y, view[0], min(view[1], y + rows))) for y in range(0, view[1], rows)]
    ctx = mp.get_context("fork")
    _cpu_setup()  # build once, inherited by the forked workers
    times, samples = [], 0
    with ctx.Pool(cores) as pool:
        for it in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            s = sum(pool.map(_cpu_worker, jobs, chunksize=1))
            dt = time.perf_counter() - t0
            if it >= args.warmup:
                times.append(dt)
                samples += s
    total = sum(times)
    v = samples / total / 1e9
    st = _CPU_STATE
    sample = (f"S volume {CPU_DIMS[0]}^3 x3 uint16, 32^3 bricks, same scene at {view[0]}x{view[1]} "
              f"split in {len(jobs)} row tiles over {cores} processes, all bricks resident")
    print(json.dumps({
        "impl": "reference", "metric": "Gsamples/s (3-ch pos-samples, 1920x1080 frame); frame ms; "
        "octree build GB/s", "value": round(v, 8), "unit": "Gsamples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": sample},
        "cpu_baseline": {"value": round(v, 8), "unit": "Gsamples/s", "cores": cores,
                         "kind": st["kind"], "sample": sample},
        "e2e": {"value": round(v, 8), "unit": "Gsamples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "build_gbs_raw": round(st["build_gbs"], 5)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--dims", type=int, nargs=3, default=list(DIMS))
    ap.add_argument("--viewport", type=int, nargs=2, default=list(VIEWPORT))
    ap.add_argument("--strip-rows", type=int, default=8)
    ap.add_argument("--precision", choices=("fp64", "fp32"), default="fp64",
                    help="sample reconstruction precision (RenderSettings.precision)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-build-e2e", dest="build_e2e", action="store_false")
    ap.add_argument("--no-stream", dest="stream", action="store_false",
                    help="skip the cfg3-shaped slice-stream ingest measurement")
    args = ap.parse_args()
    if args.warmup < 3:  # timing rule: at least 3 untimed warm-up steps
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
