"""Multi-rank path on the GPU: two processes sharing one B200
(torch.distributed over gloo — the only GPU a test box has), each running
the real z-slab sharded build (slab_build.build_sharded: own slab, record
all-gather, vt_tree_merge) and the real sort-first renderer
(SortFirstRenderer: vt_render_strips + gather to rank 0 + counter
all-reduce).  Rank 0 compares against a single-process build and frame of
the same volume: identical tree checksum on every rank, identical image
(bit for bit) and counters."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

DIMS = (96, 80, 160)  # five 32-z slabs of 16^3 bricks
BRICK = 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene(R):
    import scenarios
    from gpu_helpers import to_scene
    spec = dict(scenarios.camera_for(DIMS, (72, 52), 1.8), mode="dvr", sampling_step=None,
                early_termination_alpha=0.99, lod_bias=0.0, tfs=scenarios.spim_tfs(3),
                clips=[((0.0, 0.0, 1.0), 120.0)])
    return to_scene(spec)


def _volume():
    import voxtree_oracle as vo
    return vo.synth_spim(DIMS, 3, 65535, seed=4)


def _tree():
    from gpu_helpers import make_tree
    return make_tree(dict(dims=DIMS, brick=(BRICK,) * 3, threshold=0, fmt="uint16", channels=3))


def _worker(rank, world, port, strip_rows, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    sys.path.insert(0, os.path.dirname(here))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1407_2074_b200 import DeviceState
        from paper_1407_2074_b200 import render as R
        from paper_1407_2074_b200.render.sharded import SortFirstRenderer
        from paper_1407_2074_b200.slab_build import build_sharded
        vol = torch.from_numpy(np.ascontiguousarray(_volume())).cuda()
        tree = _tree()
        plan = build_sharded(tree, lambda z0, z1: vol[z0:z1].contiguous())
        ck = tree.checksum()
        dev = DeviceState(tree, resident_all=True)
        sfr = SortFirstRenderer(dev, strip_rows=strip_rows)
        img, cnt = sfr.render_fullframe(_scene(R), out_kind=R.raycast.OUT_F64, to_host=True)
        out = {"rank": rank, "checksum": ck, "slabs": [list(s) for s in plan.slabs],
               "counters": {f: int(getattr(cnt, f)) for f in cnt.__dataclass_fields__}}
        if rank == 0:
            np.save(os.path.join(os.environ["VT_TEST_TMP"], "sharded.npy"), img)
        else:
            out["img_none"] = img is None
        q.put(out)
        dev.close()
        tree.close()
    finally:
        dist.destroy_process_group()


def _reference(tmp_path):
    """The single-process reference: one bulk build, one full frame."""
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    from paper_1407_2074_b200 import render as R
    vol = _volume()
    t = _tree()
    t.insert_channels((0, 0, 0), vol)
    t.finalize()
    t.fill_borders()
    img, cnt = OutOfCoreRenderer(DeviceState(t, resident_all=True)).render_fullframe(_scene(R))
    return t.checksum(), img, cnt


def _nccl_worker(port, q):
    """One NCCL rank (NCCL will not put two ranks on one GPU) playing both
    slabs of a two-slab plan: slab 1's records go through the real NCCL
    device collectives of the sharded build (`_all_gather_records`: meta
    all-gather, record and brick all_gather_into_tensor on device buffers)
    and are merged into the slab-0 tree; the frame is then rendered as two
    sort-first strip sets whose parts and counters go through NCCL gather /
    all-reduce on device tensors."""
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    sys.path.insert(0, os.path.dirname(here))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_1407_2074_b200 import DeviceState
        from paper_1407_2074_b200 import render as R
        from paper_1407_2074_b200.render.sharded import SortFirstRenderer, assemble
        from paper_1407_2074_b200 import slab_build as sb
        vol = torch.from_numpy(np.ascontiguousarray(_volume())).cuda()
        plan = sb.slab_plan(_tree().geometry, 2)
        trees = []
        for z0, z1 in plan.slabs:
            t = _tree()
            for z in range(z0, z1, 32):
                t.insert_channels((0, 0, z), vol[z:min(z1, z + 32)].contiguous())
            t.sync()
            trees.append(t)
        z0, z1 = plan.slabs[1]
        idx, flags, stats, bricks = sb.export_records(trees[1], sb.slab_records(trees[1], plan, z0, z1))
        parts = sb._all_gather_records(idx, flags, stats, bricks, trees[1].inserted_voxels,
                                       trees[1], None)
        assert len(parts) == 1 and parts[0][3].is_cuda
        assert np.array_equal(parts[0][0], idx) and np.array_equal(parts[0][2], stats)
        t = trees[0]
        sb.merge_records(t, *parts[0])
        t.finalize()
        t.fill_borders()
        ck = t.checksum()
        dev = DeviceState(t, resident_all=True)
        scene = _scene(R)
        # two virtual ranks' strips, rendered then exchanged through NCCL
        locs, cnts = [], []
        for r in range(2):
            sfr = SortFirstRenderer(dev, strip_rows=8)
            sfr.world, sfr.rank = 2, r
            loc, c = sfr.render_part(scene, R.raycast.OUT_F64)
            locs.append(loc.clone())
            cnts.append(c)
        torch.cuda.synchronize()
        g = torch.stack(locs)
        out = torch.empty_like(g)
        dist.all_gather_into_tensor(out.view(-1), g.view(-1))
        fields = list(cnts[0].__dataclass_fields__)
        v = torch.tensor([[getattr(c, f) for f in fields] for c in cnts], dtype=torch.int64,
                         device="cuda").sum(0)
        dist.all_reduce(v)
        img = assemble(out, scene.camera.height, 8)
        np.save(os.path.join(os.environ["VT_TEST_TMP"], "nccl.npy"), img.cpu().numpy())
        q.put({"backend": dist.get_backend(), "checksum": ck,
               "counters": dict(zip(fields, (int(x) for x in v.tolist())))})
        dev.close()
        for tt in trees:
            tt.close()
    finally:
        dist.destroy_process_group()


def test_nccl_sharded_build_exchange_and_sort_first_render(tmp_path):
    from gpu_helpers import counters_dict
    os.environ["VT_TEST_TMP"] = str(tmp_path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    ref_ck, img, cnt = _reference(tmp_path)
    assert res["backend"] == "nccl"
    assert res["checksum"] == ref_ck
    assert res["counters"] == counters_dict(cnt)
    got = np.load(os.path.join(str(tmp_path), "nccl.npy"))
    assert got.shape == img.shape and np.array_equal(got, img)


@pytest.mark.parametrize("strip_rows", [8, 5])
def test_two_ranks_sharded_build_and_sort_first_render(tmp_path, strip_rows):
    from gpu_helpers import counters_dict
    os.environ["VT_TEST_TMP"] = str(tmp_path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, strip_rows, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res.sort(key=lambda r: r["rank"])
    ref_ck, img, cnt = _reference(tmp_path)
    assert res[0]["slabs"] != [[0, DIMS[2]]]  # really split in z
    for r in res:
        assert r["checksum"] == ref_ck, r["rank"]
        assert r["counters"] == counters_dict(cnt), r["rank"]
    assert res[1]["img_none"]
    got = np.load(os.path.join(str(tmp_path), "sharded.npy"))
    assert got.shape == img.shape
    assert np.array_equal(got, img)
