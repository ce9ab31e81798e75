"""Phase timing of the device-resident VSTR slice stream (the bench's stream
leg) and of a whole-volume insert_channels build: wall time per phase with a
device synchronisation between phases (profiling only — the bench times
without those syncs).  VT_HOST_PROFILE=1 adds libvtx's host phase table.

    python tools/prof_stream3.py [X Y Z] [--layers-per-call K] [--whole]
"""
import argparse
import ctypes as ct
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("dims", type=int, nargs="*", default=[2048, 2048, 1000])
ap.add_argument("--layers-per-call", type=int, default=2)
ap.add_argument("--whole", action="store_true", help="also an insert_channels build")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
X, Y, Z = a.dims
C, M = 3, 32
dims = (X, Y, Z)
desc = VolumeDescriptor(dims=dims, channels=C, sample_format="uint16")
cfg = BrickPoolConfig(brick_dims=(M,) * 3, homogeneity_threshold=0)
st = torch.cuda.current_stream()
P = torch.empty((C, Z, Y, X), dtype=torch.uint16, device="cuda")
for z0 in range(0, Z, 64):
    z1 = min(Z, z0 + 64)
    tmp = torch.empty((z1 - z0, Y, X, C), dtype=torch.uint16, device="cuda")
    _lib.call("vt_synth", ct.c_void_p(tmp.data_ptr()), 1, _lib.i32x3(dims), C, 2, 0, z0, z1,
              ct.c_void_p(st.cuda_stream))
    P[:, z0:z1].copy_(tmp.permute(3, 0, 1, 2))
    del tmp
torch.cuda.synchronize()
raw = X * Y * Z * C * 2


def wall(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) * 1e3, (time.perf_counter() - t0) * 1e3


for rep in range(a.reps):
    tree = Octree(desc, cfg, reserve_slots=200000)
    _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(st.cuda_stream))
    step = M * a.layers_per_call
    calls = []

    def ingest():
        for z0 in range(0, Z, step):
            t = time.perf_counter()
            tree.insert_planar(P[:, z0:min(Z, z0 + step)], z0)
            calls.append((time.perf_counter() - t) * 1e3)

    h_ing, w_ing = wall(ingest)
    h_fl, w_fl = wall(tree.sync)
    tree.finalize()
    h_fb, w_fb = wall(tree.fill_borders)
    h_s, w_s = wall(tree.sync)
    tot = w_ing + w_fl + w_fb + w_s
    print(f"stream rep {rep}: ingest host {h_ing:.1f} / wall {w_ing:.1f} ms "
          f"(per call host min {min(calls):.2f} max {max(calls):.2f} ms), "
          f"flush {w_fl:.1f}, fill_borders host {h_fb:.1f} / wall {w_fb:.1f}, sync {w_s:.1f}; "
          f"total {tot:.1f} ms = {raw / tot / 1e6:.1f} GB/s raw; groups {tree.stream_counts()}",
          flush=True)
    tree.close()
    del tree
    torch.cuda.empty_cache()

if a.whole:
    V = P.permute(1, 2, 3, 0).contiguous()
    del P
    torch.cuda.empty_cache()
    for rep in range(a.reps):
        tree = Octree(desc, cfg, reserve_slots=200000)
        _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(st.cuda_stream))
        h_i, w_i = wall(lambda: tree.insert_channels((0, 0, 0), V))
        h_fl, w_fl = wall(tree.sync)
        tree.finalize()
        h_fb, w_fb = wall(tree.fill_borders)
        tot = w_i + w_fl + w_fb
        print(f"whole rep {rep}: insert host {h_i:.1f} / wall {w_i:.1f}, flush {w_fl:.1f}, "
              f"fill_borders host {h_fb:.1f} / wall {w_fb:.1f}; total {tot:.1f} ms = "
              f"{raw / tot / 1e6:.1f} GB/s raw", flush=True)
        tree.close()
        del tree
        torch.cuda.empty_cache()
