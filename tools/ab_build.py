"""Median cfg2 build time (insert + finalize + fill_borders, CUDA events) of
one process; run it under different env settings to A/B host/device changes
(GPU box helper)."""
import ctypes as ct
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 7
dims = (N, N, N)
desc = VolumeDescriptor(dims=dims, channels=3, sample_format="uint16")
cfg = BrickPoolConfig(brick_dims=(32,) * 3, homogeneity_threshold=0)
vol = torch.empty((N, N, N, 3), dtype=torch.uint16, device="cuda")
st = torch.cuda.current_stream() if os.environ.get("AB_DEFAULT_STREAM") == "1" else torch.cuda.Stream()
_lib.call("vt_synth", ct.c_void_p(vol.data_ptr()), 1, _lib.i32x3(dims), 3, 2, 0, 0, N,
          ct.c_void_p(st.cuda_stream))
torch.cuda.synchronize()
ins, tot = [], []
for rep in range(REPS + 1):
    tree = Octree(desc, cfg, reserve_slots=40000)
    _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(st.cuda_stream))
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    with torch.cuda.stream(st):
        e0.record(st)
        tree.insert_channels((0, 0, 0), vol)
        tree.sync()
        e1.record(st)
        tree.finalize()
        tree.fill_borders()
        tree.sync()
        e2.record(st)
    torch.cuda.synchronize()
    if rep:
        ins.append(e0.elapsed_time(e1))
        tot.append(e0.elapsed_time(e2))
    tree.close()
print(f"{os.environ.get('AB_TAG', '')}: insert {statistics.median(ins):.2f} ms  "
      f"build {statistics.median(tot):.2f} ms  (min {min(tot):.2f})")
