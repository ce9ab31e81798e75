"""Per-channel slice build vs fused slabs at larger sizes (device synth)."""
import ctypes as ct
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib

N = int(sys.argv[1]); M = int(sys.argv[2]); nsl = int(sys.argv[3]); C = 3
dims = (N, N, N)
vol = torch.empty((N, N, N, C), dtype=torch.uint16, device="cuda")
_lib.call("vt_synth", ct.c_void_p(vol.data_ptr()), 1, _lib.i32x3(dims), C, 2, 0, 0, N,
          ct.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
desc = VolumeDescriptor(dims=dims, channels=C, sample_format="uint16")
cfg = BrickPoolConfig(brick_dims=(M,) * 3, homogeneity_threshold=0)
a = Octree(desc, cfg)
for z in range(0, N, M):
    a.insert_channels((0, 0, z), vol[z:z + M])
b = Octree(desc, cfg)
for z in range(nsl):
    for c in range(C):
        b.insert_block(c, (0, 0, z), vol[z:z + 1, :, :, c].contiguous())
for z in range(nsl, N, M):
    b.insert_channels((0, 0, z), vol[z:z + M])
for t in (a, b):
    t.finalize(); t.fill_borders()
print(N, M, nsl, "checksums equal", a.checksum() == b.checksum())
ia, fa, sa, _ = a.export(with_bricks=False)
ib, fb, sb, _ = b.export(with_bricks=False)
print("idx", np.array_equal(ia, ib), "flags", np.array_equal(fa, fb))
d = np.argwhere(sa != sb)
print("stat diffs", len(d))
rows = np.unique(d[:, 0]) if len(d) else []
geo = a.geometry
for r in rows[:6]:
    i = int(ia[r])
    print("node", i, "level", geo.level_of_index(i), "lo", geo.box_lo_of_index(i), "a", sa[r].tolist(), "b", sb[r].tolist())
if len(rows):
    i = int(ia[rows[0]])
    ba = a.read_brick(i); bb = b.read_brick(i)
    w = np.argwhere(ba != bb)
    print("brick voxels differ", len(w), w[:8].tolist())
