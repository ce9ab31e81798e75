import sys, numpy as np
sys.path.insert(0, '.')
from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor
dims = tuple(int(v) for v in sys.argv[1:4]); b = int(sys.argv[4])
vol = np.random.default_rng(0).integers(0, 65535, size=(dims[2], dims[1], dims[0], 3), dtype=np.uint16)
t = Octree(VolumeDescriptor(dims=dims, channels=3, sample_format="uint16"), BrickPoolConfig(brick_dims=(b,)*3, homogeneity_threshold=0))
t.insert_channels((0, 0, 0), vol)
t.sync()
print("ok", t.dense_counts())
