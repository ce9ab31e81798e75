"""Tree checksum of the cfg2 whole-volume build under the current env
switches (GPU box helper: run it with different VT_* settings and compare)."""
import ctypes as ct
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dims = (N, N, N)
desc = VolumeDescriptor(dims=dims, channels=3, sample_format="uint16")
cfg = BrickPoolConfig(brick_dims=(32,) * 3, homogeneity_threshold=0)
vol = torch.empty((N, N, N, 3), dtype=torch.uint16, device="cuda")
_lib.call("vt_synth", ct.c_void_p(vol.data_ptr()), 1, _lib.i32x3(dims), 3, 2, 0, 0, N, None)
torch.cuda.synchronize()
tree = Octree(desc, cfg, reserve_slots=40000)
tree.insert_channels((0, 0, 0), vol)
tree.finalize()
tree.fill_borders()
tree.sync()
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("VT_"))
print(f"{tag or 'defaults'}: checksum {tree.checksum()}")
