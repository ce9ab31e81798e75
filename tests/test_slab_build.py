"""z-slab sharded build (paper_1407_2074_b200/slab_build.py).

CPU: the slab plan (level-k alignment, contiguous cover) and the vectorised
node geometry.  GPU: G ranks simulated in one process — each tree inserts
only its slab, exports its level <= k records, merges everyone else's — and
every merged tree must be byte-identical (VXOC/VXBP digests after
fill_borders) to the single-GPU build of the whole volume."""

import numpy as np
import pytest

from paper_1407_2074_b200 import BrickPoolConfig, TreeGeometry, VolumeDescriptor
from paper_1407_2074_b200.slab_build import _levels_and_z, slab_plan


@pytest.mark.parametrize("dims,brick,world", [((64, 48, 128), (8, 8, 8), 4),
                                              ((1024, 1024, 1024), (32, 32, 32), 8),
                                              ((2048, 2048, 1000), (32, 32, 32), 8),
                                              ((32, 32, 40), (8, 8, 8), 3),
                                              ((16, 16, 8), (8, 8, 8), 4),
                                              ((64, 64, 64), (16, 16, 16), 1)])
def test_slab_plan_aligned_cover(dims, brick, world):
    geo = TreeGeometry.build(VolumeDescriptor(dims=dims), BrickPoolConfig(brick_dims=brick))
    plan = slab_plan(geo, world)
    assert len(plan.slabs) == world
    z = 0
    for z0, z1 in plan.slabs:
        assert z0 == z and z1 >= z0
        assert z0 % plan.layer_voxels == 0
        z = z1
    assert z == dims[2]
    layers = -(-dims[2] // plan.layer_voxels)
    if layers >= world:
        assert all(z1 > z0 for z0, z1 in plan.slabs)


def test_levels_and_z_match_geometry():
    geo = TreeGeometry.build(VolumeDescriptor(dims=(40, 24, 70)), BrickPoolConfig(brick_dims=(8, 8, 8)))
    idx = np.arange(geo.node_capacity)
    lvl, z = _levels_and_z(geo, idx)
    for i in range(0, geo.node_capacity, 7):
        assert lvl[i] == geo.level_of_index(i)
        assert z[i] == geo.box_lo_of_index(i)[2]


@pytest.mark.gpu
@pytest.mark.parametrize("dims,brick,world,channels,fmt", [
    ((40, 24, 70), (8, 8, 8), 4, 2, "uint8"),
    ((64, 48, 128), (8, 8, 8), 4, 3, "uint16"),
    ((48, 40, 96), (16, 8, 8), 3, 1, "uint16"),
])
def test_sharded_build_matches_single_gpu(dims, brick, world, channels, fmt, tmp_path):
    import voxtree_oracle as vo
    from gpu_helpers import digest
    from paper_1407_2074_b200 import Octree
    from paper_1407_2074_b200.slab_build import export_records, merge_records, slab_records
    fmax = 255 if fmt == "uint8" else 65535
    vol = vo.synth_spim(dims, channels, fmax, seed=5)
    desc = VolumeDescriptor(dims=dims, channels=channels, sample_format=fmt)
    cfg = BrickPoolConfig(brick_dims=brick, homogeneity_threshold=0)

    ref = Octree(desc, cfg)
    for z in range(0, dims[2], brick[2]):
        ref.insert_channels((0, 0, z), vol[z:z + brick[2]])
    ref.finalize()
    ref.fill_borders()
    want = digest(ref, tmp_path, "ref")

    plan = slab_plan(ref.geometry, world)
    trees, recs = [], []
    for r in range(world):
        t = Octree(desc, cfg)
        z0, z1 = plan.slabs[r]
        for z in range(z0, z1, brick[2]):
            t.insert_channels((0, 0, z), vol[z:min(z1, z + brick[2])])
        t.sync()
        trees.append(t)
        recs.append(export_records(t, slab_records(t, plan, z0, z1), device_bricks=(r % 2 == 0)) +
                    (t.inserted_voxels,))
    import torch
    for r, t in enumerate(trees):
        others = [recs[q] for q in range(world) if q != r]
        bricks = [o[3] if hasattr(o[3], "data_ptr") else torch.as_tensor(o[3]).cuda() for o in others]
        merge_records(t, np.concatenate([o[0] for o in others]),
                      np.concatenate([o[1] for o in others]),
                      np.concatenate([o[2] for o in others]), torch.cat(bricks),
                      sum(o[4] for o in others))
        t.finalize()
        t.fill_borders()
        assert t.node_count == ref.node_count
        assert t.brick_count == ref.brick_count
        assert t.inserted_voxels == ref.inserted_voxels
        assert digest(t, tmp_path, f"r{r}") == want, f"rank {r} differs"


class _Desc:
    channels = 2


class _Cfg:
    @staticmethod
    def brick_nbytes(desc):
        return 6


class _FakeTree:
    descriptor = _Desc()
    config = _Cfg()


def _gather_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    from paper_1407_2074_b200.slab_build import _all_gather_records
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 2 + rank  # ragged record counts
        idx = np.arange(n, dtype=np.int64) + 100 * rank
        flags = np.full(n, 9 + rank, np.int32)
        stats = np.arange(n * 2 * 5, dtype=np.int32).reshape(n, 2, 5) + rank
        nb = rank + 1
        bricks = torch.arange(nb * 6, dtype=torch.uint8) + rank
        parts = _all_gather_records(idx, flags, stats, bricks, 1000 + rank, _FakeTree(), None)
        ok = len(parts) == world
        for r, (i, f, s, b, ins) in enumerate(parts):
            ok &= np.array_equal(i, np.arange(2 + r) + 100 * r)
            ok &= bool(np.all(f == 9 + r)) and s.shape == (2 + r, 2, 5)
            ok &= np.array_equal(s, np.arange((2 + r) * 10).reshape(2 + r, 2, 5) + r)
            ok &= torch.equal(b, torch.arange((r + 1) * 6, dtype=torch.uint8) + r)
            ok &= ins == 1000 + r
        q.put(bool(ok))
    finally:
        dist.destroy_process_group()


def test_record_all_gather_gloo():
    """the one exchange step: ragged per-rank records over a world-3 group"""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert all(q.get(timeout=5) for _ in range(3))
