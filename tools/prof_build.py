"""Host/device time breakdown of the cfg2 slab build (GPU box helper)."""
import cProfile
import ctypes as ct
import os
import pstats
import resource
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib  # noqa: E402

if os.environ.get("PROF_MALLOPT", "0") == "1":
    libc = ct.CDLL("libc.so.6")
    libc.mallopt(-3, 32 << 20)   # M_MMAP_THRESHOLD
    libc.mallopt(-1, 512 << 20)  # M_TRIM_THRESHOLD
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
SLAB = int(sys.argv[2]) if len(sys.argv) > 2 else 32
dims = (N, N, N)
desc = VolumeDescriptor(dims=dims, channels=3, sample_format="uint16")
cfg = BrickPoolConfig(brick_dims=(32,) * 3, homogeneity_threshold=0)
vol = torch.empty((N, N, N, 3), dtype=torch.uint16, device="cuda")
st = torch.cuda.current_stream()
_lib.call("vt_synth", ct.c_void_p(vol.data_ptr()), 1, _lib.i32x3(dims), 3, 2, 0, 0, N,
          ct.c_void_p(st.cuda_stream))
torch.cuda.synchronize()
for rep in range(2):
    tree = Octree(desc, cfg, reserve_slots=40000)
    _lib.call("vt_tree_set_stream", tree.handle, ct.c_void_p(st.cuda_stream))
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    tins = 0.0
    f0 = resource.getrusage(resource.RUSAGE_SELF).ru_minflt
    for z0 in range(0, N, SLAB):
        a = time.perf_counter()
        tree.insert_channels((0, 0, z0), vol[z0:z0 + SLAB])
        tins += time.perf_counter() - a
    print(f"minor faults during inserts: {resource.getrusage(resource.RUSAGE_SELF).ru_minflt - f0}")
    a = time.perf_counter()
    tree.sync()
    tsync = time.perf_counter() - a
    if os.environ.get("PROF_BORDERS", "0") == "1":
        tree.finalize()
        tree.fill_borders()
        tree.sync()
    pr.disable()
    t1 = time.perf_counter()
    print(f"rep {rep}: total {1e3*(t1-t0):.1f} ms  inserts {1e3*tins:.1f} ms  final sync {1e3*tsync:.1f} ms")
    if rep == 1:
        pstats.Stats(pr).sort_stats("tottime").print_stats(12)
    tree.close()
