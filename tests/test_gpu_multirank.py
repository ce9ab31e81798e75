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


@pytest.mark.parametrize("strip_rows", [8, 5])
def test_two_ranks_sharded_build_and_sort_first_render(tmp_path, strip_rows):
    from gpu_helpers import counters_dict
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    from paper_1407_2074_b200 import render as R
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
    # the single-process reference: one bulk build, one full frame
    vol = _volume()
    t = _tree()
    t.insert_channels((0, 0, 0), vol)
    t.finalize()
    t.fill_borders()
    ref_ck = t.checksum()
    img, cnt = OutOfCoreRenderer(DeviceState(t, resident_all=True)).render_fullframe(_scene(R))
    assert res[0]["slabs"] != [[0, DIMS[2]]]  # really split in z
    for r in res:
        assert r["checksum"] == ref_ck, r["rank"]
        assert r["counters"] == counters_dict(cnt), r["rank"]
    assert res[1]["img_none"]
    got = np.load(os.path.join(str(tmp_path), "sharded.npy"))
    assert got.shape == img.shape
    assert np.array_equal(got, img)
