import ctypes as ct, sys, os, time
sys.path.insert(0, '/root/repo')
import torch, bench
from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor, _lib
dims=(1024,1024,1024); M=int(sys.argv[1]) if len(sys.argv)>1 else 16
st=torch.cuda.current_stream()
vol=bench._synth(dims,0,dims[2],st)
desc=VolumeDescriptor(dims=dims,channels=3,sample_format="uint16")
cfg=BrickPoolConfig(brick_dims=(M,)*3,homogeneity_threshold=0)
for rep in range(2):
    t=Octree(desc,cfg,reserve_slots=bench.expected_bricks(dims,M))
    _lib.call("vt_tree_set_stream",t.handle,ct.c_void_p(st.cuda_stream))
    torch.cuda.synchronize(); t0=time.perf_counter()
    t.insert_channels((0,0,0),vol); h1=time.perf_counter()
    t.sync(); t1=time.perf_counter()
    t.finalize(); t.fill_borders(); h2=time.perf_counter(); t.sync(); t2=time.perf_counter()
    print(f"rep {rep}: insert host {1e3*(h1-t0):.2f} wall {1e3*(t1-t0):.2f}  borders host {1e3*(h2-t1):.2f} wall {1e3*(t2-t1):.2f}", flush=True)
    t.close()
