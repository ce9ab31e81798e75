"""Find the first difference between a fused-slab build and a per-channel
slice build (tau 0) — debugging aid."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import voxtree_oracle as vo
from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor

dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (32, 32, 64)
M = int(sys.argv[4]) if len(sys.argv) > 4 else 8
C = 3
vol = vo.synth_spim(dims, C, 65535, seed=0)
desc = VolumeDescriptor(dims=dims, channels=C, sample_format="uint16")
cfg = BrickPoolConfig(brick_dims=(M,) * 3, homogeneity_threshold=0)
a = Octree(desc, cfg)
for z in range(0, dims[2], M):
    a.insert_channels((0, 0, z), vol[z:z + M])
b = Octree(desc, cfg)
for z in range(dims[2]):
    for c in range(C):
        b.insert_block(c, (0, 0, z), vol[z:z + 1, :, :, c])
for t in (a, b):
    t.finalize(); t.fill_borders()
print("checksums", a.checksum(), b.checksum())
ia, fa, sa, ba = a.export()
ib, fb, sb, bb = b.export()
print("nodes", len(ia), len(ib), "equal idx", np.array_equal(ia, ib), "flags", np.array_equal(fa, fb))
d = np.argwhere(sa != sb)
print("stat diffs", len(d), d[:10])
for r in np.unique(d[:, 0])[:5]:
    print("node", ia[r], "a", sa[r].tolist(), "b", sb[r].tolist())
bd = [k for k in range(len(ba)) if not np.array_equal(ba[k], bb[k])]
print("brick diffs", len(bd), bd[:10])
if bd:
    k = bd[0]
    w = np.argwhere(ba[k] != bb[k])
    print("first brick", k, "voxels differ", len(w), w[:10].tolist())
    print(ba[k][tuple(w[0][:3])], bb[k][tuple(w[0][:3])])
ot = vo.OracleTree(dims, (M,) * 3, channels=C, fmt="uint16", threshold=0)
for z in range(dims[2]):
    for c in range(C):
        ot.insert(c, (0, 0, z), vol[z:z + 1, :, :, c])
ot.finished = True
ot.fill_borders()
print("oracle digest vs a/b:", vo.digest(ot))
