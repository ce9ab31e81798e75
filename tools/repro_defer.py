"""Checksum of slice-wise (deferred layers) + slab builds vs a bulk build."""
import ctypes as ct
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
SL = int(sys.argv[2]) if len(sys.argv) > 2 else 128  # z handled slice by slice
M, C = 32, 3
dims = (N, N, N)
vol = torch.empty((N, N, N, C), dtype=torch.uint16, device="cuda")
_lib.call("vt_synth", ct.c_void_p(vol.data_ptr()), 1, _lib.i32x3(dims), C, 2, 0, 0, N,
          ct.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()


def tree():
    return Octree(VolumeDescriptor(dims=dims, channels=C, sample_format="uint16"),
                  BrickPoolConfig(brick_dims=(M,) * 3, homogeneity_threshold=0))


def fin(t, tag):
    t.finalize()
    t.fill_borders()
    print(tag, hex(t.checksum()), t.dense_counts(), flush=True)


a = tree()
a.insert_channels((0, 0, 0), vol)
fin(a, "bulk")
for mode in ("slices+slabs", "slices only", "slices, sync mid"):
    t = tree()
    zs = SL if mode != "slices only" else N
    for z in range(zs):
        for c in range(C):
            t.insert_block(c, (0, 0, z), vol[z:z + 1, :, :, c].contiguous())
        if mode == "slices, sync mid" and z == 40:
            t.sync()
    for z in range(zs, N, M):
        t.insert_channels((0, 0, z), vol[z:z + M])
    fin(t, mode)
