"""Phase timing of the bench's interleaved leg (cfg3 stream with a 1080p
frame after every 50 z): per interval, wall time of insert / drain events /
apply (repack + brick maxima) / render with a device sync between phases
(profiling only).  VT_HOST_PROFILE=1 adds libvtx's host phase table.

    python tools/prof_interleaved.py [X Y Z] [--every 50] [--intervals N]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as ct  # noqa: E402

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1407_2074_b200 import (BrickPoolConfig, DeviceState, Octree,  # noqa: E402
                                  VolumeDescriptor, _lib)
from paper_1407_2074_b200 import render as R  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("dims", type=int, nargs="*", default=[2048, 2048, 1000])
ap.add_argument("--every", type=int, default=50)
ap.add_argument("--intervals", type=int, default=0)
a = ap.parse_args()
dims = tuple(a.dims)
st = torch.cuda.current_stream()
P = bench._synth_planar(dims, st)
desc = VolumeDescriptor(dims=dims, channels=3, sample_format="uint16")
cfg = BrickPoolConfig(brick_dims=(32,) * 3, homogeneity_threshold=0)
tree = Octree(desc, cfg, reserve_slots=bench.expected_bricks(dims, 32))
_lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(st.cuda_stream))
dev = DeviceState(tree, resident_all=True)
rr = R.OutOfCoreRenderer(dev)
scene = bench.scene_for(R, dims, bench.VIEWPORT)


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return r, (t1 - t0) * 1e3, (time.perf_counter() - t0) * 1e3


rows = []
Z = dims[2]
for k, z0 in enumerate(range(0, Z, a.every)):
    if a.intervals and k >= a.intervals:
        break
    z1 = min(Z, z0 + a.every)
    _, hi, wi = timed(lambda: tree.insert_planar(P[:, z0:z1], z0))
    nev, hd, wd = timed(dev.refresh)
    kinds = range(nev)
    _, ha, wa = timed(lambda: None)
    _, hr, wr = timed(lambda: rr.render_fullframe(scene, out_kind=R.raycast.OUT_RGBA8))
    rows.append((z0, wi, hi, wd, len(kinds), wa, ha, dev.bmax_stats()[1], wr))
    print(f"z {z0:4d}: insert {wi:6.2f} (host {hi:6.2f})  refresh {wd:5.2f} (host {hd:5.2f}, {len(kinds)} ev, "
          f"bmax slots {rows[-1][7]})  frame {wr:6.2f}",
          flush=True)
n = len(rows)
print(f"mean: insert {sum(r[1] for r in rows) / n:.2f}  refresh {sum(r[3] for r in rows) / n:.2f}  "
      f"frame {sum(r[8] for r in rows) / n:.2f} ms")
dev.close()
tree.close()
