"""Slice-stream ingest on the GPU: Octree.insert_many (vt_tree_insert_many)
and the deferred brick layers of per-slice insert_block calls must give the
tree, queued change events and VXOC/VXBP files of the general path (dense
build off) — ingest_stream's frame loop, ingest.py:306-358, over
Octree.insert_block, octree.py:323-397.

Covers: layers read in place from a planar (C, Z, Y, X) device array (4-D
TMA tensor map) for 1-4 channels, layers gathered from separate device
slices or host slices, 8-bit samples (interleaving fallback), blocks of
several planes, batches that end inside a layer, and readers (a node query,
a render) in the middle of a layer, which materialise the received planes
and keep the layer open."""

import numpy as np
import pytest

from gpu_helpers import make_tree

pytestmark = pytest.mark.gpu


def _vol(dims, C, fmt, seed=0):
    import voxtree_oracle as vo
    return vo.synth_spim(dims, C, 65535 if fmt == "uint16" else 255, seed=seed)


def _spec(dims, C, fmt, brick):
    return dict(dims=dims, brick=(brick,) * 3, threshold=0, fmt=fmt, channels=C)


def _ops(vol, zc=1):
    Z, C = vol.shape[0], vol.shape[3]
    return [(c, (0, 0, z), vol[z:z + zc, :, :, c]) for z in range(0, Z, zc) for c in range(C)]


def _state(tree):
    from paper_1407_2074_b200.serialize import octree_digests
    ev = tree.drain_events()
    a = octree_digests(tree)
    tree.finalize()
    tree.fill_borders()
    b = octree_digests(tree)
    return (ev.kinds.tolist(), ev.indices.tolist()), a, b, tree.checksum()


def _general(spec, ops):
    t = make_tree(spec)
    t.dense_build = False
    for c, o, v in ops:
        t.insert_block(c, o, v)
    return _state(t)


def _planar(vol):
    import torch
    return torch.as_tensor(np.ascontiguousarray(np.moveaxis(vol, 3, 0))).cuda()


@pytest.mark.parametrize("C", [1, 2, 3, 4])
def test_insert_many_planar_in_place(C):
    dims, brick = (64, 40, 40), 16
    vol = _vol(dims, C, "uint16", seed=C)
    spec = _spec(dims, C, "uint16", brick)
    want = _general(spec, _ops(vol))
    pv = _planar(vol)
    t = make_tree(spec)
    t.insert_many([(c, (0, 0, z), pv[c, z:z + 1]) for z in range(dims[2]) for c in range(C)])
    groups, in_place, _ = t.stream_counts()
    assert groups == 3 and in_place == 3
    assert _state(t) == want


@pytest.mark.parametrize("source", ["separate", "host", "chunks3"])
def test_insert_many_gathered(source):
    import torch
    dims, C, brick = (64, 40, 40), 3, 16
    vol = _vol(dims, C, "uint16", seed=11)
    spec = _spec(dims, C, "uint16", brick)
    zc = 3 if source == "chunks3" else 1
    want = _general(spec, _ops(vol, zc))
    t = make_tree(spec)
    ops = _ops(vol, zc)
    if source in ("separate", "chunks3"):
        ops = [(c, o, torch.as_tensor(np.ascontiguousarray(v)).cuda()) for c, o, v in ops]
    t.insert_many(ops)
    assert _state(t) == want


def test_insert_many_uint8_fallback():
    dims, C, brick = (48, 40, 36), 3, 8
    vol = _vol(dims, C, "uint8", seed=3)
    spec = _spec(dims, C, "uint8", brick)
    want = _general(spec, _ops(vol))
    pv = _planar(vol)
    t = make_tree(spec)
    t.insert_many([(c, (0, 0, z), pv[c, z:z + 1]) for z in range(dims[2]) for c in range(C)])
    assert t.stream_counts()[0] == 5
    assert _state(t) == want


@pytest.mark.parametrize("batch,read_every", [(7, 0), (7, 2), (50, 1), (1, 5)])
def test_batches_ending_inside_layers_and_mid_layer_readers(batch, read_every):
    """batches of `batch` blocks; after every `read_every`-th batch a reader
    (node query + a small render) forces the partial layer out"""
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    import scenarios
    from gpu_helpers import to_scene
    dims, C, brick = (64, 40, 40), 3, 16
    vol = _vol(dims, C, "uint16", seed=5)
    spec = _spec(dims, C, "uint16", brick)
    ops = _ops(vol)
    want = _general(spec, ops)
    pv = _planar(vol)
    dev_ops = [(c, o, pv[c, o[2]:o[2] + 1]) for c, o, _ in ops]
    t = make_tree(spec)
    sc = to_scene(dict(scenarios.camera_for(dims, (12, 10)), mode="dvr", sampling_step=None,
                       early_termination_alpha=0.99, lod_bias=0.0, tfs=scenarios.spim_tfs(C),
                       clips=[]))
    for k, b0 in enumerate(range(0, len(dev_ops), batch)):
        if batch == 1:
            t.insert_block(*dev_ops[b0])
        else:
            t.insert_many(dev_ops[b0:b0 + batch])
        if read_every and k % read_every == read_every - 1:
            t.root  # node query: flush
            img, cnt = OutOfCoreRenderer(DeviceState(t, resident_all=True)).render_fullframe(sc)
            assert cnt.samples > 0
    assert _state(t) == want


def test_mid_layer_render_matches_general_path_state():
    """a render halfway through a layer sees exactly the general path's tree"""
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    import scenarios
    from gpu_helpers import to_scene
    dims, C, brick = (64, 40, 40), 3, 16
    vol = _vol(dims, C, "uint16", seed=8)
    spec = _spec(dims, C, "uint16", brick)
    ops = _ops(vol)[:3 * 21 + 2]  # layer 1 half received, last z partial in channels
    pv = _planar(vol)
    sc = to_scene(dict(scenarios.camera_for(dims, (24, 20)), mode="dvr", sampling_step=None,
                       early_termination_alpha=0.99, lod_bias=0.0, tfs=scenarios.spim_tfs(C),
                       clips=[]))
    g = make_tree(spec)
    g.dense_build = False
    for op in ops:
        g.insert_block(*op)
    t = make_tree(spec)
    t.insert_many([(c, o, pv[c, o[2]:o[2] + 1]) for c, o, _ in ops])
    assert t.checksum() == g.checksum()
    ig, cg = OutOfCoreRenderer(DeviceState(g, resident_all=True)).render_fullframe(sc)
    it, ct_ = OutOfCoreRenderer(DeviceState(t, resident_all=True)).render_fullframe(sc)
    assert np.array_equal(ig, it) and cg == ct_
    # the layer stays open: the rest of the stream completes it
    rest = _ops(vol)[len(ops):]
    for op in rest:
        g.insert_block(*op)
    t.insert_many([(c, o, pv[c, o[2]:o[2] + 1]) for c, o, _ in rest])
    assert _state(t) == _state(g)


def test_insert_many_errors_after_prefix():
    """an invalid block raises after the blocks before it are inserted"""
    dims, C, brick = (32, 16, 16), 2, 8
    vol = _vol(dims, C, "uint16", seed=1)
    spec = _spec(dims, C, "uint16", brick)
    ops = _ops(vol)[:5]
    t = make_tree(spec)
    bad = (0, (0, 0, 15), np.zeros((2, 16, 32), np.uint16))  # z 15..16 outside
    with pytest.raises(ValueError):
        t.insert_many(ops + [bad])
    g = make_tree(spec)
    g.dense_build = False
    for op in ops:
        g.insert_block(*op)
    assert t.checksum() == g.checksum()
    with pytest.raises(ValueError):
        t.insert_many([(5, (0, 0, 0), vol[:1, :, :, 0])])


def test_interleaved_renders_incremental_maxima_exact():
    """renders between stream batches (one zero-copy mirror for the whole
    stream): the brick maxima are refreshed for the written slots only, and
    the exact empty-space skip still changes no pixel, counter or flag"""
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    import scenarios
    from gpu_helpers import counters_dict, to_scene
    dims, C, brick = (64, 48, 80), 3, 16
    vol = _vol(dims, C, "uint16", seed=21)
    spec = _spec(dims, C, "uint16", brick)
    pv = _planar(vol)
    ops = [(c, (0, 0, z), pv[c, z:z + 1]) for z in range(dims[2]) for c in range(C)]
    t = make_tree(spec)
    dev = DeviceState(t, resident_all=True)
    r = OutOfCoreRenderer(dev)
    spec_sc = dict(scenarios.camera_for(dims, (40, 32)), mode="dvr", sampling_step=None,
                   early_termination_alpha=0.99, lod_bias=0.0, tfs=scenarios.spim_tfs(C),
                   clips=[])
    seen = []
    for b0 in range(0, len(ops), 3 * 10):  # a render every 10 z
        t.insert_many(ops[b0:b0 + 30])
        dev.refresh()
        out = {}
        for mode in ("off", "bricks", "subbricks"):
            sc = to_scene(spec_sc)
            sc.settings.empty_space_skip = mode
            img, cnt = r.render_fullframe(sc)
            out[mode] = (img, counters_dict(cnt), dev.read_flags(clear=True))
        for mode in ("bricks", "subbricks"):
            assert np.array_equal(out[mode][0], out["off"][0]), (b0, mode)
            assert out[mode][1] == out["off"][1], (b0, mode)
            assert np.array_equal(out[mode][2], out["off"][2]), (b0, mode)
        seen.append(dev.bmax_stats())
    inc, last = seen[-1]
    assert inc >= len(seen) - 1
    assert 0 < last < t.brick_count
    # and the final tree equals the general path's
    t.finalize()
    t.fill_borders()
    g = make_tree(spec)
    g.dense_build = False
    for c, o, _ in ops:
        g.insert_block(c, o, vol[o[2]:o[2] + 1, :, :, c])
    g.finalize()
    g.fill_borders()
    assert t.checksum() == g.checksum()
    img, cnt = r.render_fullframe(to_scene(spec_sc))
    dg = DeviceState(g, resident_all=True)
    img2, cnt2 = OutOfCoreRenderer(dg).render_fullframe(to_scene(spec_sc))
    assert np.array_equal(img, img2) and counters_dict(cnt) == counters_dict(cnt2)


@pytest.mark.parametrize("where", ["device", "host"])
def test_insert_planar_slabs(where):
    """Octree.insert_planar: VSTR-order slabs of a planar array, in slabs that
    do and do not align with brick layers"""
    dims, C, brick = (64, 40, 40), 3, 16
    vol = _vol(dims, C, "uint16", seed=31)
    spec = _spec(dims, C, "uint16", brick)
    want = _general(spec, _ops(vol))
    planar = np.ascontiguousarray(np.moveaxis(vol, 3, 0))
    src = _planar(vol) if where == "device" else planar
    t = make_tree(spec)
    for z0, z1 in ((0, 16), (16, 21), (21, 40)):
        t.insert_planar(src[:, z0:z1], z0)
    assert t.stream_counts()[0] >= 1
    assert _state(t) == want


@pytest.mark.parametrize("reader", [False, True])
def test_layer_pairs_with_interior_parents(reader):
    """insert_planar in brick-layer pairs over a volume whose level-1
    parents have interior x/y neighbours: the pair's leaf kernel writes those
    parents' x/y shells and the slab seams their z shells; fill_borders skips
    them.  Same tree (checksum, VXOC/VXBP after fill_borders) as the general
    path, also with a reader (which resets every prefilled shell) mid-stream."""
    from paper_1407_2074_b200.serialize import octree_digests
    dims, C, brick = (224, 192, 160), 3, 16
    vol = _vol(dims, C, "uint16", seed=9)
    spec = _spec(dims, C, "uint16", brick)
    pv = _planar(vol)
    t = make_tree(spec)
    for z in range(0, dims[2], 4 * brick):
        t.insert_planar(pv[:, z:z + 4 * brick], z)
        if reader and z == 4 * brick:
            t.checksum()  # a reader between pairs: prefilled shells published
    t.finalize()
    t.fill_borders()
    g = make_tree(spec)
    g.dense_build = False
    for z in range(dims[2]):
        for c in range(C):
            g.insert_block(c, (0, 0, z), vol[z:z + 1, :, :, c])
    g.finalize()
    g.fill_borders()
    assert t.checksum() == g.checksum()
    assert octree_digests(t) == octree_digests(g)
