"""Host-slab (pinned) build through Octree.insert_channels, 32 z per call —
bench.py's build e2e leg in isolation (GPU box helper)."""
import ctypes as ct
import os
import sys
import time

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
host = vol.cpu().pin_memory().numpy()
del vol
for rep in range(3):
    tree = Octree(desc, cfg, reserve_slots=40000)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for z in range(0, N, 32):
        tree.insert_channels((0, 0, z), host[z:z + 32])
    tree.sync()
    t1 = time.perf_counter()
    print(f"{os.environ.get('AB_TAG', '')}: host-slab build {1e3 * (t1 - t0):.1f} ms = "
          f"{host.nbytes / (t1 - t0) / 1e9:.1f} GB/s")
    tree.close()
