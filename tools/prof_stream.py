"""Slice-wise (VSTR-order) ingest speed: per z, per channel, one (1, Y, X)
insert_block from device memory; cfg3's 2048x2048 planes (depth from argv)."""
import ctypes as ct
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib  # noqa: E402

X = Y = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
Z = int(sys.argv[2]) if len(sys.argv) > 2 else 128
C = 3
dims = (X, Y, Z)
desc = VolumeDescriptor(dims=dims, channels=C, sample_format="uint16")
cfg = BrickPoolConfig(brick_dims=(32,) * 3, homogeneity_threshold=0)
vol = torch.empty((Z, Y, X, C), dtype=torch.uint16, device="cuda")
st = torch.cuda.current_stream()
_lib.call("vt_synth", ct.c_void_p(vol.data_ptr()), 1, _lib.i32x3(dims), C, 2, 0, 0, Z,
          ct.c_void_p(st.cuda_stream))
planes = [vol[:, :, :, c].contiguous() for c in range(C)]  # channel-major planes
torch.cuda.synchronize()
for rep in range(2):
    tree = Octree(desc, cfg, reserve_slots=200000)
    _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(st.cuda_stream))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for z in range(Z):
        for c in range(C):
            tree.insert_block(c, (0, 0, z), planes[c][z:z + 1])
    t1 = time.perf_counter()
    tree.finalize()
    tree.fill_borders()
    tree.sync()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    raw = X * Y * Z * C * 2
    print(f"rep {rep}: inserts {1e3*(t1-t0):.1f} ms host, total {1e3*(t2-t0):.1f} ms, "
          f"{raw/(t2-t0)/1e9:.1f} GB/s raw, checksum {tree.checksum():x}")
    tree.close()
