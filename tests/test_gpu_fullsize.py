"""Parity at BASELINE.json's full sizes through size-independent properties
(the CPU oracle cannot build a 1024^3 or 2048x2048x1000 tree in test time).

* Build (cfg2, cfg3, cfg5): at homogeneity threshold 0 every brick is a pure
  function of the data, so every insertion order and every
  sharding must give the same tree — compared with the device digest
  ``Octree.checksum`` (structure + statistics + a hash of every brick).  The
  root statistics are checked against a direct reduction of the volume.
* Render (cfg2, 1920x1080): the exact empty-space skip changes no pixel and
  no counter; sort-first strips and tiles reassemble the full frame; the FP32
  reconstruction path stays within the north-star tolerance of 1/255.
"""

import ctypes as ct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1.0 / 255.0


def _synth(dims, C, z0=0, z1=None, fmt="uint16"):
    import torch
    from paper_1407_2074_b200 import _lib
    z1 = dims[2] if z1 is None else z1
    dt = torch.uint16 if fmt == "uint16" else torch.uint8
    vol = torch.empty((z1 - z0, dims[1], dims[0], C), dtype=dt, device="cuda")
    _lib.call("vt_synth", ct.c_void_p(vol.data_ptr()), 1, _lib.i32x3(dims), C,
              2 if fmt == "uint16" else 1, 0, z0, z1,
              ct.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return vol


def _tree(dims, C, brick, fmt="uint16"):
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor
    desc = VolumeDescriptor(dims=dims, channels=C, sample_format=fmt)
    cfg = BrickPoolConfig(brick_dims=(brick,) * 3, homogeneity_threshold=0)
    return Octree(desc, cfg)


def _expected_bricks(dims, m):
    from paper_1407_2074_b200 import BrickPoolConfig, TreeGeometry, VolumeDescriptor
    geo = TreeGeometry.build(VolumeDescriptor(dims=dims), BrickPoolConfig(brick_dims=(m,) * 3))
    return sum(int(np.prod([-(-d // (m << lvl)) for d in dims])) for lvl in range(geo.depth + 1))


def _finish(t):
    t.finalize()
    t.fill_borders()
    return t.checksum()


def _sharded_sim(dims, C, brick, vol, world):
    """world ranks in one process: slab inserts, record exchange, merge"""
    import torch
    from paper_1407_2074_b200.slab_build import (export_records, merge_records, slab_plan,
                                                  slab_records)
    trees = [_tree(dims, C, brick) for _ in range(world)]
    plan = slab_plan(trees[0].geometry, world)
    recs = []
    for r, t in enumerate(trees):
        z0, z1 = plan.slabs[r]
        for z in range(z0, z1, brick):
            t.insert_channels((0, 0, z), vol[z:min(z1, z + brick)])
        t.sync()
        recs.append(export_records(t, slab_records(t, plan, z0, z1)) + (t.inserted_voxels,))
    out = []
    for r in (0, world - 1):
        others = [recs[q] for q in range(world) if q != r]
        merge_records(trees[r], np.concatenate([o[0] for o in others]),
                      np.concatenate([o[1] for o in others]),
                      np.concatenate([o[2] for o in others]),
                      torch.cat([o[3] for o in others]), sum(o[4] for o in others))
        out.append(_finish(trees[r]))
    for t in trees:
        t.close()
    return out


def test_cfg2_build_order_and_sharding_independent():
    """1024^3 x 3 uint16, 32^3 bricks: 32-z slabs == one bulk insert ==
    per-channel single slices == 4-way z-slab sharded build"""
    import torch
    dims, C, M = (1024, 1024, 1024), 3, 32
    vol = _synth(dims, C)
    a = _tree(dims, C, M)
    for z in range(0, dims[2], M):
        a.insert_channels((0, 0, z), vol[z:z + M])
    want = _finish(a)
    assert a.brick_count == _expected_bricks(dims, M) == 37449
    # subtree extrema of the root == the volume's (octree.py:265-277)
    root = a.root
    for c in range(C):
        ch = vol[..., c].to(torch.int32)
        assert root.sub_min[c] == int(ch.min()) and root.sub_max[c] == int(ch.max())
        del ch
    a.close()
    b = _tree(dims, C, M)
    b.insert_channels((0, 0, 0), vol)
    assert _finish(b) == want
    b.close()
    c3 = _tree(dims, C, M)
    for z in range(0, 256):  # the first 8 brick layers slice by slice, per channel
        for ch in range(C):
            c3.insert_block(ch, (0, 0, z), vol[z:z + 1, :, :, ch].contiguous())
    for z in range(256, dims[2], M):
        c3.insert_channels((0, 0, z), vol[z:z + M])
    assert _finish(c3) == want
    c3.close()
    assert _sharded_sim(dims, C, M, vol, 4) == [want, want]


@pytest.mark.parametrize("brick", [16, 32, 64])
def test_cfg5_sharded_build_brick_sweep(brick):
    """z-slab sharded build (8 ranks simulated) over brick sizes 16^3-64^3"""
    dims, C = (512, 512, 512), 3
    vol = _synth(dims, C)
    t = _tree(dims, C, brick)
    for z in range(0, dims[2], brick):
        t.insert_channels((0, 0, z), vol[z:z + brick])
    want = _finish(t)
    assert t.brick_count == _expected_bricks(dims, brick)
    t.close()
    assert _sharded_sim(dims, C, brick, vol, 8) == [want, want]


def test_cfg3_spim_slice_stream_equals_slabs():
    """2048x2048x1000 x 3 uint16 (25 GB) streamed slice-wise in VSTR order
    (per z: channel 0, 1, 2) == brick-layer slabs"""
    import torch
    dims, C, M = (2048, 2048, 1000), 3, 32
    vol = _synth(dims, C)
    a = _tree(dims, C, M)
    for z in range(0, dims[2], M):
        a.insert_channels((0, 0, z), vol[z:z + M])
    want = _finish(a)
    assert a.brick_count == _expected_bricks(dims, M)
    a.close()
    torch.cuda.empty_cache()
    s = _tree(dims, C, M)
    for z in range(dims[2]):
        plane = vol[z:z + 1]
        for ch in range(C):
            s.insert_block(ch, (0, 0, z), plane[..., ch].contiguous())
    assert _finish(s) == want
    s.close()
    torch.cuda.empty_cache()
    # the bench's stream: planar (C, Z, Y, X) slices, one insert_planar call
    # per brick-layer pair (fused pairs, parent shells from the leaf kernel,
    # eager z seams)
    P = vol.permute(3, 0, 1, 2).contiguous()
    del vol
    torch.cuda.empty_cache()
    s = _tree(dims, C, M)
    for z in range(0, dims[2], 2 * M):
        s.insert_planar(P[:, z:z + 2 * M], z)
    assert s.stream_counts()[0] == (dims[2] + M - 1) // M
    assert _finish(s) == want
    s.close()


@pytest.fixture(scope="module")
def cfg2_render():
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200 import render as R
    dims, C, M = (1024, 1024, 1024), 3, 32
    vol = _synth(dims, C)
    t = _tree(dims, C, M)
    for z in range(0, dims[2], M):
        t.insert_channels((0, 0, z), vol[z:z + M])
    t.finalize()
    t.fill_borders()
    del vol
    dev = DeviceState(t, resident_all=True)
    yield dev, (lambda **kw: bench.scene_for(R, dims, (1920, 1080), **kw)), R
    dev.close()
    t.close()


def _counters(c):
    return {f: int(getattr(c, f)) for f in c.__dataclass_fields__}


def test_cfg2_empty_space_skip_is_exact(cfg2_render):
    dev, scene, R = cfg2_render
    rr = R.OutOfCoreRenderer(dev)
    outs = {}
    for mode in ("off", "bricks", "subbricks"):
        sc = scene()
        sc.settings.empty_space_skip = mode
        img, cnt = rr.render_fullframe(sc)
        outs[mode] = (img, _counters(cnt), cnt.samples_skipped, dev.read_flags(clear=True))
    ref_img, ref_cnt, skipped, ref_flags = outs["off"]
    assert skipped == 0 and ref_cnt["samples"] > 0
    for mode in ("bricks", "subbricks"):
        img, cnt, sk, fl = outs[mode]
        assert np.array_equal(img, ref_img), mode
        assert cnt == ref_cnt, mode
        assert np.array_equal(fl, ref_flags), mode
        assert sk > 0


def test_cfg2_strips_tiles_and_fp32(cfg2_render):
    import torch
    from paper_1407_2074_b200 import _lib
    from paper_1407_2074_b200.render.raycast import OUT_F64, scene_to_vt
    from paper_1407_2074_b200.render.sharded import assemble, part_rows
    dev, scene, R = cfg2_render
    rr = R.OutOfCoreRenderer(dev)
    sc = scene()
    full, fcnt = rr.render_fullframe(sc)
    # 8-way sort-first strips reassemble the frame exactly
    G, strip = 8, 8
    rows = part_rows(1080, strip, G)
    parts, total = [], 0
    for p in range(G):
        buf = torch.empty((rows, 1920, 4), dtype=torch.float64, device="cuda")
        cnt = _lib.vt_counters()
        s = scene_to_vt(sc, dev.octree.descriptor)
        _lib.call("vt_render_strips", dev.handle, ct.byref(s), strip, G, p,
                  ct.c_void_p(buf.data_ptr()), OUT_F64, 1, ct.byref(cnt))
        parts.append(buf)
        total += cnt.samples
    assert np.array_equal(assemble(torch.stack(parts), 1080, strip).cpu().numpy(), full)
    assert total == fcnt.samples
    tile, _ = rr.render_tile(sc, (700, 300, 1300, 800))
    assert np.array_equal(tile, full[300:800, 700:1300])
    f32 = scene(precision="fp32")
    img32, c32 = rr.render_fullframe(f32)
    assert float(np.max(np.abs(img32 - full))) <= TOL
    assert abs(c32.samples - fcnt.samples) <= 1e-4 * fcnt.samples
