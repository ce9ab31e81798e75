"""Render A/B: the bench's 1080p DVR frame (L2 flushed, CUDA events, kernel
time from vt_last_kernel_ms) on a device-built volume, for the library named
by VT_LIB (default: the in-tree build).  Prints one JSON line.

    VT_LIB=/path/libvtx_variant.so python tools/ab_render.py [--dims X Y Z] [--frames N]
"""
import argparse
import ctypes as ct
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1407_2074_b200 import (BrickPoolConfig, DeviceState, Octree,  # noqa: E402
                                  VolumeDescriptor, _lib)
from paper_1407_2074_b200 import render as R  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=3, default=[1024, 1024, 1024])
ap.add_argument("--frames", type=int, default=10)
ap.add_argument("--precision", default="fp64")
ap.add_argument("--ess", default=None)
a = ap.parse_args()
dims = tuple(a.dims)
st = torch.cuda.current_stream()
desc = VolumeDescriptor(dims=dims, channels=3, sample_format="uint16")
cfg = BrickPoolConfig(brick_dims=(32,) * 3, homogeneity_threshold=0)
tree = Octree(desc, cfg, reserve_slots=bench.expected_bricks(dims, 32))
_lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(st.cuda_stream))
for z0 in range(0, dims[2], 256):
    v = bench._synth(dims, z0, min(dims[2], z0 + 256), st)
    tree.insert_channels((0, 0, z0), v)
    tree.sync()
    del v
tree.finalize()
tree.fill_borders()
tree.sync()
dev = DeviceState(tree, resident_all=True)
rr = R.OutOfCoreRenderer(dev)
scene = bench.scene_for(R, dims, bench.VIEWPORT, precision=a.precision)
if a.ess:
    scene.settings.empty_space_skip = a.ess
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
ms, kms = [], []
for it in range(3 + a.frames):
    flush.zero_()
    torch.cuda.synchronize()
    with bench._Ev(st) as ev:
        img, cnt = rr.render_fullframe(scene, out_kind=R.raycast.OUT_RGBA8)
    torch.cuda.synchronize()
    if it >= 3:
        ms.append(ev.ms())
        r = ct.c_double()
        _lib.call("vt_last_kernel_ms", tree.handle, ct.byref(r), None)
        kms.append(r.value)
print(json.dumps({"lib": os.environ.get("VT_LIB", "in-tree"), "frame_ms": round(statistics.median(ms), 4),
                  "kernel_ms": round(statistics.median(kms), 4), "samples": cnt.samples,
                  "skipped": cnt.samples_skipped, "checksum": int(img.astype("u8").sum())}))
