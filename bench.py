#!/usr/bin/env python
"""bench.py — the driver's benchmark contract for the octree build + octree
ray-casting hot path (BASELINE.json metric: frame ms & Gsamples/s, 3-ch
1920x1080; octree build GB/s; at 1/2/4/8 GPUs).

Workload (N=1 default, BASELINE.json configs[2], the north-star set): the
synthetic SPIM-shaped ("S") 3-channel 2048x2048x1000 uint16
volume (25.2 GB raw; 32^3 bricks, homogeneity threshold 0, pool 35.3 GB),
which fits one B200.  It lives in HBM as planar (C, Z, Y, X) slices, the
layout a VSTR slice stream lands in (ingest_stream, ingest.py:306-358):

  stream              every (z, channel) slice in VSTR order through
                      Octree.insert_planar (= insert_block per slice), one
                      call per brick layer, + finalize + fill_borders: build
                      GB/s and its roofline fraction (1 + pool/raw bytes per
                      raw byte)
  stream_interleaved  the same stream with a 1920x1080 frame after every 50 z
                      (mirror refresh + render timed separately)
  stream_e2e          host -> tree: pinned host frames of the first 256 z
  value               Gsamples/s of 1920x1080 DVR frames of the final tree
                      (per-channel transfer functions, one clipping plane,
                      ET 0.99, step 0.5 voxel, LOD bias 0, camera at 2.5x the
                      extent as voxtree cli.default_scene); a "step" is one
                      frame; device time (CUDA events), L2 flushed between
                      frames, max over ranks
  e2e                 the same through the public drop-in API with host output
                      (OutOfCoreRenderer.render_fullframe -> float64 (H, W, 4)
                      numpy, the reference's return type)
  roofline            render kernel: 48 B gathered per reconstructed pos-sample
                      (8 corners x 3 ch x 2 B) / average kernel duration vs the
                      measured HBM copy bandwidth
  cfg2                secondary leg: configs[1] (1024^3 x 3 uint16), one-call
                      device build + 1080p frames

N > 1 (torchrun): the same volume built z-slab sharded (each rank inserts
its slab, one all-gather of level-k node records) and rendered sort-first
(interleaved strips, NCCL gather to rank 0).  `--workload cfg2` selects
configs[1] instead.

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

CHANNELS = 3
FMT = "uint16"
BRICK = 32
VIEWPORT = (1920, 1080)
CLIP_FRAC = 0.8
COLORS = ((1.0, 0.25, 0.2), (0.2, 1.0, 0.3), (0.25, 0.45, 1.0))
BYTES_PER_POS_SAMPLE = 8 * CHANNELS * 2  # 8 trilinear corners x C x uint16
L2_FLUSH_BYTES = 512 << 20
STREAM_CHUNK = 2 * BRICK  # slices per insert_planar call: a pair of brick layers
FALLBACK_HBM_GBS = 6650.0
_SCENE = ("1920x1080 DVR frame, per-channel TFs, 1 clip plane, ET 0.99, step 0.5 voxel, "
          "LOD bias 0")
WORKLOADS = {
    "cfg3": {"dims": (2048, 2048, 1000),
             "desc": "cfg3: synthetic SPIM-shaped 3-ch uint16 2048x2048x1000 (25.2 GB), 32^3 "
                     "bricks, tau=0, streamed slice-wise in VSTR order (device-resident planar "
                     "slices) + fill_borders, interleaved 1080p renders every 50 z; " + _SCENE},
    "cfg2": {"dims": (1024, 1024, 1024),
             "desc": "cfg2: synthetic SPIM-shaped 3-ch uint16 1024^3, 32^3 bricks, tau=0, "
                     "full octree build + fill_borders; " + _SCENE},
}
WORKLOAD = WORKLOADS["cfg3"]["desc"]


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

def _setup_dist():
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

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    return world, rank, local, backend, barrier


def _rank_max(vals, world, backend):
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def _synth(dims, z0, z1, stream):
    """(z1 - z0, Y, X, C) interleaved S volume on the device (vt_synth ==
    oracle synth_spim, hash-checked in tests/test_gpu_build.py)."""
    import torch
    from paper_1407_2074_b200 import _lib
    v = torch.empty((max(0, z1 - z0), dims[1], dims[0], CHANNELS), dtype=torch.uint16,
                    device="cuda")
    if z1 > z0:
        _lib.call("vt_synth", ct.c_void_p(v.data_ptr()), 1, _lib.i32x3(dims), CHANNELS, 2, 0,
                  z0, z1, ct.c_void_p(stream.cuda_stream))
    return v


def _synth_planar(dims, stream, z0=0, z1=None, pin=False):
    """(C, z1 - z0, Y, X) planar S volume: the layout a VSTR slice stream
    lands in (one frame per channel per z); device, or pinned host."""
    import torch
    z1 = dims[2] if z1 is None else z1
    X, Y = dims[0], dims[1]
    if pin:
        out = torch.empty((CHANNELS, z1 - z0, Y, X), dtype=torch.uint16, pin_memory=True)
    else:
        out = torch.empty((CHANNELS, z1 - z0, Y, X), dtype=torch.uint16, device="cuda")
    step = 64
    for a in range(z0, z1, step):
        b = min(z1, a + step)
        tmp = _synth(dims, a, b, stream)
        out[:, a - z0:b - z0].copy_(tmp.permute(3, 0, 1, 2))
        del tmp
    torch.cuda.synchronize()
    return out


class _Ev:
    """CUDA events on the bench stream around a region (device time)."""

    def __init__(self, stream):
        import torch
        self.s = stream
        self.a = torch.cuda.Event(enable_timing=True)
        self.b = torch.cuda.Event(enable_timing=True)

    def __enter__(self):
        self.a.record(self.s)
        return self

    def __exit__(self, *exc):
        self.b.record(self.s)

    def ms(self):
        return self.a.elapsed_time(self.b)


def leg_stream(P, dims, stream, peak):
    """Device-resident VSTR slice stream: every (z, channel) frame of the
    planar volume P through Octree.insert_planar, one call per brick layer,
    then finalize + fill_borders (ingest_stream, ingest.py:306-358); CUDA
    events around the whole sequence (host gaps included)."""
    import torch
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib
    desc = VolumeDescriptor(dims=dims, channels=CHANNELS, sample_format=FMT)
    cfg = BrickPoolConfig(brick_dims=(BRICK,) * 3, homogeneity_threshold=0)
    Z = dims[2]
    raw = dims[0] * dims[1] * Z * CHANNELS * 2
    res, runs = None, []
    for rep in range(3):  # warm-up, then two timed runs (best reported, both listed)
        tree = Octree(desc, cfg, reserve_slots=expected_bricks(dims, BRICK))
        _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize()
        with _Ev(stream) as ev:
            for z0 in range(0, Z, STREAM_CHUNK):
                tree.insert_planar(P[:, z0:min(Z, z0 + STREAM_CHUNK)], z0)
            with _Ev(stream) as evb:
                tree.finalize()
                tree.fill_borders()
                tree.sync()
        torch.cuda.synchronize()
        ms = ev.ms()
        pool = tree.brick_count * cfg.brick_nbytes(desc)
        groups, in_place, _ = tree.stream_counts()
        run = {"ms": round(ms, 3), "fill_borders_ms": round(evb.ms(), 3)}
        if rep == 0:
            tree.close()
            del tree
            continue
        if res is None or ms < res["ms"]:
            alg = (raw + pool) / (ms * 1e-3) / 1e9
            res = {"workload": f"{dims[0]}x{dims[1]}x{Z} x{CHANNELS} uint16 S volume, planar "
                               "(C, Z, Y, X) in HBM, every (z, channel) slice in VSTR order "
                               "through Octree.insert_planar (= insert_block per slice), one "
                               f"call per {STREAM_CHUNK} slices, + finalize + fill_borders",
                   "slices": Z * CHANNELS, "ms": round(ms, 3),
                   "fill_borders_ms": round(evb.ms(), 3),
                   "raw_gb": round(raw / 1e9, 3), "pool_gb": round(pool / 1e9, 3),
                   "gbs_raw": round(raw / (ms * 1e-3) / 1e9, 2),
                   "layer_groups": groups, "layers_read_in_place": in_place,
                   "roofline": {"achieved": round(alg, 2), "peak": peak,
                                "frac": round(alg / peak, 4), "unit": "GB/s",
                                "model": "(raw + pool bytes) / stream time (SURVEY 8d: "
                                         "1 + pool/raw B per raw byte)"},
                   "tree_checksum": f"{tree.checksum():016x}"}
        runs.append(round(ms, 3))
        res["runs_ms"] = list(runs)
        tree.close()
        del tree
        torch.cuda.empty_cache()
    return res


def leg_stream_interleaved(P, dims, stream, viewport, every_z, precision):
    """The stream again with a 1920x1080 frame after every `every_z` slices
    (a FrameService-style live view: refresh the mirror — flush, incremental
    brick maxima — then render); returns the numbers and the final tree."""
    import torch
    from paper_1407_2074_b200 import (BrickPoolConfig, DeviceState, Octree, VolumeDescriptor,
                                      _lib)
    from paper_1407_2074_b200 import render as R
    desc = VolumeDescriptor(dims=dims, channels=CHANNELS, sample_format=FMT)
    cfg = BrickPoolConfig(brick_dims=(BRICK,) * 3, homogeneity_threshold=0)
    Z = dims[2]
    tree = Octree(desc, cfg, reserve_slots=expected_bricks(dims, BRICK))
    _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(stream.cuda_stream))
    dev = DeviceState(tree, resident_all=True)
    rr = R.OutOfCoreRenderer(dev)
    scene = scene_for(R, dims, viewport, precision=precision)
    ins, fl, ref, fr, slots, nev = [], [], [], [], [], []
    torch.cuda.synchronize()
    with _Ev(stream) as tot:
        for z0 in range(0, Z, every_z):
            z1 = min(Z, z0 + every_z)
            with _Ev(stream) as e1:
                tree.insert_planar(P[:, z0:z1], z0)
            with _Ev(stream) as e2:
                tree.flush()
            with _Ev(stream) as e3:
                nev.append(dev.refresh())
            with _Ev(stream) as e4:
                img, cnt = rr.render_fullframe(scene, out_kind=R.raycast.OUT_RGBA8)
            ins.append(e1)
            fl.append(e2)
            ref.append(e3)
            fr.append((e4, cnt.samples))
            slots.append(dev.bmax_stats()[1])
        tree.finalize()
        tree.fill_borders()
        tree.sync()
    torch.cuda.synchronize()
    ins_ms = [e.ms() for e in ins]
    fl_ms = [e.ms() for e in fl]
    ref_ms = [e.ms() for e in ref]
    fr_ms = [e.ms() for e, _ in fr]
    out = {"every_z": every_z, "frames": len(fr_ms),
           "total_ms": round(tot.ms(), 2),
           "ingest_ms": round(sum(ins_ms), 2),
           "tree_flush_ms_mean": round(statistics.mean(fl_ms), 3),
           "tree_flush_ms_max": round(max(fl_ms), 3),
           "mirror_refresh_ms_mean": round(statistics.mean(ref_ms), 3),
           "mirror_refresh_ms_max": round(max(ref_ms), 3),
           "events_per_refresh_mean": int(statistics.mean(nev)),
           "bmax_slots_per_refresh_mean": int(statistics.mean(slots)),
           "frame_ms_mean": round(statistics.mean(fr_ms), 3),
           "frame_ms_max": round(max(fr_ms), 3),
           "samples_last_frame": int(fr[-1][1]),
           "note": "tree flush = the open brick layer's received planes built by the leaf "
                   "kernel + pyramid propagation of everything inserted since the last frame "
                   "(what any reader of the tree pays, octree.py:323-397 leaves the tree complete "
                   "after every insert_block); mirror refresh = apply the queued change events "
                   "(DeviceState.refresh, in-library), node-buffer repack, brick maxima of the "
                   "slots not written by the leaf kernel; frame = render kernel + RGBA8 "
                   "copy-out"}
    dev.close()
    return out, tree


def leg_frames(tree, dims, viewport, args, stream, barrier, world, rank, backend, sweep=True):
    """K flushed 1080p frames (sort-first strips over the ranks), the LOD
    sweep and the e2e frames through the public API."""
    import torch
    from paper_1407_2074_b200 import DeviceState, _lib
    from paper_1407_2074_b200 import render as R
    from paper_1407_2074_b200.render.sharded import SortFirstRenderer
    dev = DeviceState(tree, resident_all=True)
    scene = scene_for(R, dims, tuple(viewport), precision=args.precision)
    sfr = SortFirstRenderer(dev, strip_rows=args.strip_rows)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")

    def frame(sc):
        img, cnt = sfr.render_fullframe(sc, out_kind=R.raycast.OUT_RGBA8)
        return cnt

    times, kms, samples, skipped, launches = [], [], 0, 0, 0
    with Clocks(torch.cuda.current_device()) as clk:
        for it in range(args.warmup + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            with _Ev(stream) as ev:
                cnt = frame(scene)
            torch.cuda.synchronize()
            if it >= args.warmup:
                times.append(ev.ms())
                rms = ct.c_double()
                _lib.call("vt_last_kernel_ms", tree.handle, ct.byref(rms), None)
                kms.append(rms.value)
                samples += cnt.samples
                skipped += cnt.samples_skipped
                launches += 1
    clocks = clk.summary()
    t = _rank_max(times, world, backend)
    total_ms = sum(t)
    out = {"frame_ms": total_ms / args.steps,
           "value": samples / (total_ms * 1e-3) / 1e9,
           "kernel_ms": statistics.mean(kms),
           "samples_per_frame": samples / args.steps,
           "computed_per_frame": (samples - skipped) / args.steps,
           "launches": launches, "clocks": clocks}
    if sweep:
        sw = {}
        for bias in (-1.0, 0.0, 1.0, 2.0, 3.0):
            sc = scene_for(R, dims, tuple(viewport), lod_bias=bias, precision=args.precision)
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            with _Ev(stream) as ev:
                cnt = frame(sc)
            torch.cuda.synchronize()
            ms = _rank_max([ev.ms()], world, backend)[0]
            sw[f"{bias:+.0f}"] = {"frame_ms": round(ms, 3), "samples": cnt.samples,
                                  "gsamples_s": round(cnt.samples / (ms * 1e-3) / 1e9, 3)}
        out["lod_sweep"] = sw
    # e2e: public drop-in API, float64 image to host every frame
    e2e_times, e2e_samples = [], 0
    rr = R.OutOfCoreRenderer(dev)
    for it in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        with _Ev(stream) as ev:
            if world == 1:
                img, cnt = rr.render_fullframe(scene)
            else:
                img, cnt = sfr.render_fullframe(scene, out_kind=R.raycast.OUT_F64, to_host=True)
        torch.cuda.synchronize()
        if it >= args.warmup:
            e2e_times.append(ev.ms())
            e2e_samples += cnt.samples
    t = _rank_max(e2e_times, world, backend)
    out["e2e_value"] = e2e_samples / (sum(t) * 1e-3) / 1e9
    dev.close()
    return out


def leg_4k(tree, dims, args, stream, barrier, world, rank, backend):
    """configs[3]: the 24 GB set rendered at 3840x2160, sort-first strips over
    the ranks with the NCCL tile gather (RGBA8 to rank 0); L2 flushed,
    CUDA-event device time, max over ranks."""
    import torch
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200 import render as R
    from paper_1407_2074_b200.render.sharded import SortFirstRenderer
    dev = DeviceState(tree, resident_all=True)
    vp = (3840, 2160)
    scene = scene_for(R, dims, vp, precision=args.precision)
    sfr = SortFirstRenderer(dev, strip_rows=args.strip_rows)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    times, samples = [], 0
    steps = max(3, args.steps // 2)
    for it in range(args.warmup + steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        with _Ev(stream) as ev:
            img, cnt = sfr.render_fullframe(scene, out_kind=R.raycast.OUT_RGBA8)
        torch.cuda.synchronize()
        if it >= args.warmup:
            times.append(ev.ms())
            samples += cnt.samples
    t = _rank_max(times, world, backend)
    ms = sum(t) / steps
    dev.close()
    return {"viewport": list(vp), "frame_ms": round(ms, 4),
            "gsamples_s": round(samples / (sum(t) * 1e-3) / 1e9, 3),
            "samples_per_frame": int(samples / steps), "frames": steps,
            "parallelism": f"sort-first strips x{world}, gather to rank 0" if world > 1
            else "single GPU"}


def leg_whole_build(dims, stream, barrier, world, rank, backend, host_e2e):
    """Whole-volume device build (z-slab sharded over the ranks): each rank
    inserts its slab in one Octree.insert_channels call (ingest_bulk),
    one all-gather of level-k records, fill_borders; median of three."""
    import torch
    import torch.distributed as dist
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib
    from paper_1407_2074_b200.slab_build import build_sharded, slab_plan
    desc = VolumeDescriptor(dims=dims, channels=CHANNELS, sample_format=FMT)
    cfg = BrickPoolConfig(brick_dims=(BRICK,) * 3, homogeneity_threshold=0)
    plan = slab_plan(expected_geometry(dims, BRICK), world)
    sz0, sz1 = plan.slabs[rank]
    vol = _synth(dims, sz0, sz1, stream)
    raw_bytes = dims[0] * dims[1] * dims[2] * CHANNELS * 2

    def build(src):
        tree = Octree(desc, cfg, reserve_slots=expected_bricks(dims, BRICK))
        _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize()
        barrier()
        with _Ev(stream) as e1:
            slab = max(BRICK, sz1 - sz0) if hasattr(src, "is_cuda") else BRICK
            build_sharded(tree, lambda a, b: src[a - sz0:b - sz0], slab_z=slab,
                          fill_borders=False)
        with _Ev(stream) as e2:
            tree.finalize()
            tree.fill_borders()
            tree.sync()
        torch.cuda.synchronize()
        return tree, e1.ms(), e2.ms()

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
    ck = tree.checksum()
    replicas_identical = True
    if world > 1:
        cks = [None] * world
        dist.all_gather_object(cks, ck)
        replicas_identical = all(c == ck for c in cks)
    build_e2e_ms = None
    if host_e2e:
        host = vol.cpu().pin_memory()
        del vol
        torch.cuda.empty_cache()
        for _ in range(2):
            t2, build_e2e_ms, _ = build(host.numpy())
            t2.close()
            del t2
        del host
    else:
        del vol
    torch.cuda.empty_cache()
    build_ms, border_ms, build_e2e_ms = _rank_max([build_ms, border_ms, build_e2e_ms or 0.0],
                                                  world, backend)
    total = build_ms + border_ms
    alg = (raw_bytes + pool_bytes) / (total * 1e-3) / 1e9
    peak, _ = hbm_peak()
    info = {"raw_gb": round(raw_bytes / 1e9, 3), "pool_gb": round(pool_bytes / 1e9, 3),
            "bricks": tree.brick_count, "build_ms": round(total, 2),
            "build_runs_ms": [round(r[0], 2) for r in runs],
            "insert_ms": round(build_ms, 2), "fill_borders_ms": round(border_ms, 2),
            "gbs_raw": round(raw_bytes / (total * 1e-3) / 1e9, 2),
            "roofline": {"achieved": round(alg, 2), "peak": peak, "frac": round(alg / peak, 4),
                         "unit": "GB/s",
                         "model": "(raw + pool bytes) / (insert + fill_borders) time"},
            "e2e_gbs_raw": round(raw_bytes / (build_e2e_ms * 1e-3) / 1e9, 2)
            if build_e2e_ms else None,
            "e2e_api": "Octree.insert_channels(pinned host slabs, 32 z each)",
            "api": "Octree.insert_channels(device-resident slab) [z-slab sharded: "
                   "slab_build.build_sharded]",
            "sharding": f"z-slab x{world}, level-k={plan.level} records all-gathered"
            if world > 1 else "single GPU",
            "tree_checksum": f"{ck:016x}", "replicas_identical": replicas_identical}
    return tree, info


def leg_brick_sweep(stream, peak, dims=(1024, 1024, 1024)):
    """configs[4] on one GPU: the whole-volume slice-ingest / downsample build
    (one Octree.insert_channels of a device-resident volume + fill_borders)
    at brick edges 16, 32, 64 — GB/s and roofline fraction per brick size
    (the z-slab sharding over 8 GPUs splits exactly this work)."""
    import torch
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib
    desc = VolumeDescriptor(dims=dims, channels=CHANNELS, sample_format=FMT)
    vol = _synth(dims, 0, dims[2], stream)
    raw = dims[0] * dims[1] * dims[2] * CHANNELS * 2
    out = {}
    for m in (16, 32, 64):
        cfg = BrickPoolConfig(brick_dims=(m,) * 3, homogeneity_threshold=0)
        runs = []
        for rep in range(3):
            tree = Octree(desc, cfg, reserve_slots=expected_bricks(dims, m))
            _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(stream.cuda_stream))
            torch.cuda.synchronize()
            with _Ev(stream) as ev:
                tree.insert_channels((0, 0, 0), vol)
                tree.finalize()
                tree.fill_borders()
                tree.sync()
            torch.cuda.synchronize()
            if rep:
                runs.append(ev.ms())
            pool = tree.brick_count * cfg.brick_nbytes(desc)
            bricks = tree.brick_count
            tree.close()
            del tree
            torch.cuda.empty_cache()
        ms = min(runs)
        out[f"{m}^3"] = {"ms": round(ms, 3), "bricks": bricks, "pool_gb": round(pool / 1e9, 3),
                         "gbs_raw": round(raw / (ms * 1e-3) / 1e9, 1),
                         "roofline_frac": round((raw + pool) / (ms * 1e-3) / 1e9 / peak, 4),
                         "runs_ms": [round(r, 3) for r in runs]}
    del vol
    torch.cuda.empty_cache()
    out["workload"] = (f"{dims[0]}x{dims[1]}x{dims[2]} x{CHANNELS} uint16 S volume, device "
                       "resident, one insert_channels + fill_borders, tau 0")
    return out


def leg_stream_host(dims, stream, nz):
    """End-to-end host -> tree ingest of the first nz slices: pinned planar
    host frames through Octree.insert_planar (H2D inside the timed region)."""
    import torch
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib
    H = _synth_planar(dims, stream, 0, nz, pin=True)
    desc = VolumeDescriptor(dims=dims, channels=CHANNELS, sample_format=FMT)
    cfg = BrickPoolConfig(brick_dims=(BRICK,) * 3, homogeneity_threshold=0)
    raw = dims[0] * dims[1] * nz * CHANNELS * 2
    best = None
    for rep in range(2):
        tree = Octree(desc, cfg, reserve_slots=expected_bricks(dims, BRICK))
        _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with _Ev(stream) as ev:
            for z0 in range(0, nz, BRICK):
                tree.insert_planar(H[:, z0:min(nz, z0 + BRICK)], z0)
            tree.sync()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if rep and (best is None or ev.ms() < best[0]):
            best = (ev.ms(), wall)
        tree.close()
        del tree
    del H
    torch.cuda.empty_cache()
    return {"sample": f"first {nz} slices x {CHANNELS} channels ({raw / 1e9:.2f} GB), pinned "
                      "host planar frames, one insert_planar call per brick layer",
            "ms": round(best[0], 2), "gbs_raw": round(raw / (best[0] * 1e-3) / 1e9, 2),
            "wall_ms": round(best[1] * 1e3, 2),
            "h2d_bytes": raw}


def leg_vstr(dims, stream, nz):
    """The VSTR wire protocol end to end (ingest.py:306-358): the first nz
    slices of the volume as encoded slab frames (header + CRC32, one frame
    per (z, channel)) in host memory, through ingest_stream — frame parsing,
    CRC checks, H2D and the build inside the timed region (finalize +
    fill_borders included); the pipelined reader vs the reference's
    per-frame loop (workers=0)."""
    import io
    import torch
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib
    from paper_1407_2074_b200.ingest import (encode_end, encode_handshake, encode_slab,
                                             ingest_stream, read_handshake)
    sub = (dims[0], dims[1], nz)
    desc = VolumeDescriptor(dims=sub, channels=CHANNELS, sample_format=FMT)
    parts = [encode_handshake(desc)]
    for z0 in range(0, nz, 32):
        v = _synth(dims, z0, min(nz, z0 + 32), stream).cpu().numpy()
        for z in range(v.shape[0]):
            for c in range(CHANNELS):
                parts.append(encode_slab(desc, c, (0, 0, z0 + z), v[z:z + 1, :, :, c]))
        del v
    parts.append(encode_end())
    blob = b"".join(parts)
    del parts
    raw = dims[0] * dims[1] * nz * CHANNELS * 2
    cfg = BrickPoolConfig(brick_dims=(BRICK,) * 3, homogeneity_threshold=0)
    out = {"sample": f"first {nz} slices x {CHANNELS} channels of the cfg3 volume as "
                     f"{nz * CHANNELS} VSTR frames ({len(blob) / 1e9:.2f} GB in host memory)",
           "wire_bytes": len(blob)}
    for name, workers in (("pipelined", None), ("per_frame", 0)):
        best = None
        for rep in range(2 if workers is None else 1):
            tree = Octree(desc, cfg)
            _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(stream.cuda_stream))
            s = io.BytesIO(blob)
            read_handshake(s)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = ingest_stream(s, tree, workers=workers)
            tree.sync()
            ms = (time.perf_counter() - t0) * 1e3
            if best is None or ms < best:
                best = ms
            ck = f"{tree.checksum():016x}"
            tree.drain_event_arrays()
            tree.close()
        out[name] = {"ms": round(best, 2), "gbs_raw": round(raw / (best * 1e-3) / 1e9, 3),
                     "slabs": res.slabs, "tree_checksum": ck}
    out["identical"] = out["pipelined"]["tree_checksum"] == out["per_frame"]["tree_checksum"]
    del blob
    return out


def leg_tau(stream, peak):
    """Threshold > 0 builds (the paper's default homogeneity threshold, 5% of
    the format maximum: per-insertion propagation and the reference's exact
    prune, octree.py:456-493): cfg1 (256^3 x 3 uint8) as 32-z slabs and as a
    VSTR slice stream, and a cfg3-shaped crop (2048 x 2048 x 64 x 3 uint16)
    slice stream; device-resident S volumes, wall time with a device sync
    (host control plane included), best of two runs after a warm-up."""
    import torch
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib
    out = {}
    cases = [("cfg1_slabs", (256, 256, 256), "uint8", "slabs"),
             ("cfg1_stream", (256, 256, 256), "uint8", "stream"),
             ("cfg3_crop_stream", (2048, 2048, 64), "uint16", "stream")]
    for name, dims, fmt, mode in cases:
        X, Y, Z = dims
        sb = 1 if fmt == "uint8" else 2
        fmax = 255 if sb == 1 else 65535
        V = torch.empty((Z, Y, X, CHANNELS), dtype=torch.uint8 if sb == 1 else torch.uint16,
                        device="cuda")
        _lib.call("vt_synth", ct.c_void_p(V.data_ptr()), 1, _lib.i32x3(dims), CHANNELS, sb, 0, 0,
                  Z, ct.c_void_p(stream.cuda_stream))
        P = V.permute(3, 0, 1, 2).contiguous() if mode == "stream" else None
        torch.cuda.synchronize()
        desc = VolumeDescriptor(dims=dims, channels=CHANNELS, sample_format=fmt)
        cfg = BrickPoolConfig(brick_dims=(BRICK,) * 3, homogeneity_threshold=0.05 * fmax)
        raw = X * Y * Z * CHANNELS * sb
        runs, res = [], None
        for rep in range(3):
            tree = Octree(desc, cfg)
            _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(stream.cuda_stream))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            n = 0
            for z0 in range(0, Z, BRICK):
                z1 = min(Z, z0 + BRICK)
                if mode == "slabs":
                    tree.insert_channels((0, 0, z0), V[z0:z1])
                    n += 1
                else:
                    tree.insert_planar(P[:, z0:z1], z0)
                    n += (z1 - z0) * CHANNELS
            tree.finalize()
            tree.fill_borders()
            tree.sync()
            ms = (time.perf_counter() - t0) * 1e3
            if rep > 0:
                runs.append(round(ms, 2))
                pool = tree.brick_count * cfg.brick_nbytes(desc)
                if res is None or ms < res["ms"]:
                    res = {"dims": list(dims), "format": fmt, "tau": 0.05 * fmax,
                           "insertions": n, "ms": round(ms, 2),
                           "gbs_raw": round(raw / (ms * 1e-3) / 1e9, 3),
                           "roofline_frac": round((raw + pool) / (ms * 1e-3) / 1e9 / peak, 5),
                           "bricks": tree.brick_count, "pruned_bricks": tree.pruned_bricks,
                           "tree_checksum": f"{tree.checksum():016x}"}
            tree.drain_event_arrays()
            tree.close()
        res["runs_ms"] = runs
        res["api"] = ("Octree.insert_channels per 32-z slab" if mode == "slabs" else
                      "Octree.insert_planar (= insert_block per (z, channel) slice, VSTR order)")
        out[name] = res
        del V, P
        torch.cuda.empty_cache()
    out["note"] = ("wall time incl. finalize + fill_borders; every insertion propagates and prunes "
                   "before the next (the reference's history-dependent semantics), so a slice "
                   "stream is bound by per-insertion launch + sync latency, not HBM")
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    world, rank, local, backend, barrier = _setup_dist()
    from paper_1407_2074_b200 import _lib
    stream = torch.cuda.current_stream()
    peak, peak_kind = hbm_peak()
    wl = WORKLOADS[args.workload]
    dims = tuple(args.dims) if args.dims else wl["dims"]
    viewport = tuple(args.viewport)
    extra = {}
    if world == 1 and args.workload == "cfg3":
        P = _synth_planar(dims, stream)
        stream_res = leg_stream(P, dims, stream, peak) if args.stream else None
        inter, tree = leg_stream_interleaved(P, dims, stream, viewport, args.render_every,
                                             args.precision)
        del P
        torch.cuda.empty_cache()
        build_info = None
        extra["stream"] = stream_res
        extra["stream_interleaved"] = inter
    else:
        tree, build_info = leg_whole_build(dims, stream, barrier, world, rank, backend,
                                           host_e2e=args.build_e2e)
    fr = leg_frames(tree, dims, viewport, args, stream, barrier, world, rank, backend)
    if args.workload == "cfg3" and args.uhd:
        extra["cfg4_3840x2160"] = leg_4k(tree, dims, args, stream, barrier, world, rank, backend)
    pool_bytes = tree.brick_count * tree.config.brick_nbytes(tree.descriptor)
    tree_ck = f"{tree.checksum():016x}"
    tree.close()
    del tree
    torch.cuda.empty_cache()
    if world == 1 and args.workload == "cfg3" and args.build_e2e:
        extra["stream_e2e"] = leg_stream_host(dims, stream, min(dims[2], 256))
    if world == 1 and args.workload == "cfg3" and args.build_e2e:
        extra["stream_vstr_e2e"] = leg_vstr(dims, stream, min(dims[2], 128))
    if world == 1 and args.workload == "cfg3" and args.secondary:
        extra["cfg5_brick_sweep"] = leg_brick_sweep(stream, peak)
    if world == 1 and args.workload == "cfg3" and args.tau:
        extra["tau"] = leg_tau(stream, peak)
    if world == 1 and args.workload == "cfg3" and args.secondary:
        d2 = WORKLOADS["cfg2"]["dims"]
        t2, b2 = leg_whole_build(d2, stream, barrier, world, rank, backend, host_e2e=False)
        f2 = leg_frames(t2, d2, viewport, args, stream, barrier, world, rank, backend,
                        sweep=False)
        t2.close()
        del t2
        torch.cuda.empty_cache()
        extra["cfg2"] = {"workload": WORKLOADS["cfg2"]["desc"], "frame_ms": round(f2["frame_ms"], 4),
                         "gsamples_s": round(f2["value"], 3),
                         "render_kernel_ms": round(f2["kernel_ms"], 4),
                         "samples_per_frame": int(f2["samples_per_frame"]),
                         "samples_computed_per_frame": int(f2["computed_per_frame"]),
                         "e2e_gsamples_s": round(f2["e2e_value"], 3), "build": b2}
    if rank == 0:
        achieved = fr["computed_per_frame"] / max(world, 1) * BYTES_PER_POS_SAMPLE / (
            fr["kernel_ms"] * 1e-3) / 1e9
        W, H = viewport
        out = {
            "metric": "Gsamples/s (3-ch pos-samples, 1920x1080 frame); frame ms; octree build GB/s",
            "value": round(fr["value"], 4),
            "unit": "Gsamples/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(fr["frame_ms"], 4),
            "frame_ms": round(fr["frame_ms"], 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f32 reconstruction / f64 accumulation",
            "data": "synthetic (SPIM-shaped S volume, generated on device, seed 0)",
            "config": arm_config(args, dims, world),
            "samples_per_frame": int(fr["samples_per_frame"]),
            "samples_computed_per_frame": int(fr["computed_per_frame"]),
            "samples_note": "samples = the reference's RenderCounters.samples (identical); "
                            "computed = samples minus those the exact empty-space skip "
                            "accounted without reconstructing (TF alpha provably 0)",
            "render_kernel_ms": round(fr["kernel_ms"], 4),
            "gpu_launches": fr["launches"],
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "traffic": traffic_from_profiles("k_render_fullframe"),
                         "model": "48 B gathered per computed pos-sample / avg render kernel "
                                  "ms (rank 0)"},
            "e2e": {"value": round(fr["e2e_value"], 4), "unit": "Gsamples/s",
                    "h2d_bytes_per_step": ct.sizeof(_lib.vt_scene),
                    "d2h_bytes_per_step": W * H * 4 * 8 + 48,
                    "api": "OutOfCoreRenderer.render_fullframe -> float64 (H,W,4) page-locked host "
                           "frame (N=1: the kernel writes it over PCIe)"
                    if world == 1 else "SortFirstRenderer.render_fullframe(to_host=True)"},
            "tree_checksum": tree_ck,
            "lod_sweep": fr.get("lod_sweep"),
            "clocks": fr["clocks"],
        }
        if build_info is not None:
            out["build"] = build_info
        out.update(extra)
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(out), flush=True)
    if world > 1:
        barrier()
        dist.destroy_process_group()


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


def arm_config(args, dims, world):
    """The `config` object both arms print (ours and --impl reference): the
    workload, its shape and the frame; the reference arm's bounded CPU sample
    is described in its cpu_baseline.sample, not here."""
    wl = WORKLOADS[args.workload]
    W, H = args.viewport
    stored = (BRICK + 2) ** 3 * CHANNELS * 2
    pool = expected_bricks(dims, BRICK) * stored
    return {"workload": wl["desc"], "dims": list(dims), "channels": CHANNELS,
            "sample_format": FMT, "brick": BRICK, "viewport": [W, H],
            "parallelism": f"sort-first strips x{world} (strip_rows={args.strip_rows})"
            if world > 1 else "single GPU",
            "l2": f"flushed between frames (512 MB write); pool {pool / 1e9:.1f} GB vs 126 MB L2"}


# ---------------------------------------------------------------------------
# reference (CPU) arm and the cpu_baseline leg
# ---------------------------------------------------------------------------

# bounded sample of the workload for the CPU reference: the central 128^3
# sub-box of the cfg3 S volume (the same voxel values), the bench scene
# around it
CPU_DIMS = (128, 128, 128)
CPU_CROP = (960, 960, 436)  # x, y, z origin of the sub-box in the 2048x2048x1000 volume
CPU_VIEW_BASE = (192, 108)


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return None


def _cpu_volume():
    import voxtree_oracle as vo
    x0, y0, z0 = CPU_CROP
    d = WORKLOADS["cfg3"]["dims"]
    return vo.synth_spim(d, CHANNELS, 65535, seed=0, z0=z0, z1=z0 + CPU_DIMS[2], y0=y0,
                         y1=y0 + CPU_DIMS[1], x0=x0, x1=x0 + CPU_DIMS[0])


def _cpu_sample_text(view, extra=""):
    return (f"central {CPU_DIMS[0]}^3 sub-box of the cfg3 S volume (origin {CPU_CROP}), 32^3 "
            f"bricks, tau 0, the bench scene around it at {view[0]}x{view[1]}, all bricks "
            f"resident{extra}")


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
    vol = _cpu_volume()
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
            "kind": st["kind"], "cpu_model": _cpu_model(), "nproc": os.cpu_count(),
            "sample": _cpu_sample_text(view, f": {samples} pos-samples in {dt:.2f} s"),
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
    wl = WORKLOADS[args.workload]
    dims = tuple(args.dims) if args.dims else wl["dims"]
    sample = _cpu_sample_text(view, f", split in {len(jobs)} row tiles over {cores} processes "
                                    "(tile-restricted RefinementSession each)")
    print(json.dumps({
        "impl": "reference", "metric": "Gsamples/s (3-ch pos-samples, 1920x1080 frame); frame ms; "
        "octree build GB/s", "value": round(v, 8), "unit": "Gsamples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": arm_config(args, dims, world),
        "cpu_baseline": {"value": round(v, 8), "unit": "Gsamples/s", "cores": cores,
                         "kind": st["kind"], "cpu_model": _cpu_model(), "sample": sample},
        "e2e": {"value": round(v, 8), "unit": "Gsamples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "build_gbs_raw": round(st["build_gbs"], 5)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="cfg3")
    ap.add_argument("--dims", type=int, nargs=3, default=None,
                    help="override the workload's volume extent (x y z)")
    ap.add_argument("--viewport", type=int, nargs=2, default=list(VIEWPORT))
    ap.add_argument("--strip-rows", type=int, default=8)
    ap.add_argument("--render-every", type=int, default=50,
                    help="slices between the interleaved renders of the stream leg")
    ap.add_argument("--precision", choices=("fp64", "fp32"), default="fp64",
                    help="sample reconstruction precision (RenderSettings.precision)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-uhd", dest="uhd", action="store_false",
                    help="skip the 3840x2160 (configs[3]) frames")
    ap.add_argument("--no-tau", dest="tau", action="store_false",
                    help="skip the threshold > 0 build leg")
    ap.add_argument("--no-build-e2e", dest="build_e2e", action="store_false")
    ap.add_argument("--no-stream", dest="stream", action="store_false",
                    help="skip the pure stream-ingest measurement")
    ap.add_argument("--no-secondary", dest="secondary", action="store_false",
                    help="skip the cfg2 secondary leg")
    args = ap.parse_args()
    if args.warmup < 3:  # timing rule: at least 3 untimed warm-up steps
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
