"""Threshold-0 dense build (csrc/dense_build.cu) against the general
incremental path of the same library (which is pinned to the unmodified
reference by test_gpu_build.py's golden digests and events).

The dense path must be invisible: the same insertion sequence with
``Octree.dense_build`` on and off gives byte-identical VXOC/VXBP digests,
device checksums, per-node records (flags, slots, statistics), brick
payloads and change events — before and after ``fill_borders``, with flushes
(reads) in the middle of a layer sequence, mixed with general-path
insertions, at partial bricks, non-split axes, 1-4 channels, u8 and u16.
"""

import numpy as np
import pytest

from gpu_helpers import digest

pytestmark = pytest.mark.gpu


def _tree(dims, C, brick, fmt, dense, bg=0):
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor
    desc = VolumeDescriptor(dims=dims, channels=C, sample_format=fmt, background_value=bg)
    cfg = BrickPoolConfig(brick_dims=brick, homogeneity_threshold=0)
    t = Octree(desc, cfg)
    t.dense_build = dense
    return t


def _volume(dims, C, fmt, seed):
    rng = np.random.default_rng(seed)
    hi = 256 if fmt == "uint8" else 65536
    vol = rng.integers(0, hi, size=(dims[2], dims[1], dims[0], C), dtype=np.int64)
    # smooth regions too, so means and extrema are not all trivially saturated
    vol[: dims[2] // 2, : dims[1] // 2] //= 7
    return vol.astype(fmt)


def _nodes(t):
    out = []
    for n in t.iter_nodes():
        out.append((n.index, n.level, n._flags, n._slot, tuple(n.avg), tuple(n.smin),
                    tuple(n.smax), None if n.sub_min is None else tuple(n.sub_min),
                    None if n.sub_max is None else tuple(n.sub_max)))
    return out


def _bricks(t):
    return {n.index: t.store.read_brick(n.brick).tobytes() for n in t.iter_nodes()
            if n.brick is not None}


def _events(batch):
    return list(zip(batch.kinds.tolist(), batch.indices.tolist()))


def _run(dims, C, brick, fmt, ops, dense, bg=0):
    """ops: ("slab", z0, z1) fused all-channel full-x/y block | ("box", c, origin, size)
    single-channel block | ("sync",) | ("borders",)"""
    t = _tree(dims, C, brick, fmt, dense, bg)
    vol = _volume(dims, C, fmt, seed=hash((dims, C, fmt)) & 0xFFFF)
    evs, snaps = [], []
    for op in ops:
        if op[0] == "slab":
            _, z0, z1 = op
            evs.append(_events(t.insert_channels((0, 0, z0), vol[z0:z1])))
        elif op[0] == "box":
            _, c, o, s = op
            blk = vol[o[2]:o[2] + s[2], o[1]:o[1] + s[1], o[0]:o[0] + s[0], c]
            evs.append(_events(t.insert_block(c, o, np.ascontiguousarray(blk))))
        elif op[0] == "sync":
            t.sync()
            snaps.append((t.checksum(), _nodes(t)))
        elif op[0] == "borders":
            t.finalize()
            t.fill_borders()
            evs.append(_events(t.drain_events()))
    t.sync()
    return t, evs, snaps


def _slabs(dims, mz, step=1):
    zs = list(range(0, dims[2], mz * step)) + [dims[2]]
    return [("slab", a, b) for a, b in zip(zs[:-1], zs[1:])]


CASES = {
    # name: dims, C, brick, fmt, ops
    "partial_u16_c3": ((40, 36, 50), 3, (8, 8, 8), "uint16", None),
    "bulk_u8_c1": ((64, 64, 64), 1, (16, 16, 16), "uint8", [("slab", 0, 64)]),
    "odd_u16_c4": ((17, 9, 33), 4, (8, 8, 8), "uint16", None),
    "nonsplit_z_u8_c2": ((30, 20, 12), 2, (8, 4, 16), "uint8", None),
    "nonsplit_xy_u16_c3": ((6, 8, 40), 3, (8, 8, 8), "uint16", None),
    "two_layer_slabs_u16_c2": ((48, 40, 72), 2, (8, 8, 8), "uint16", "step2"),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_dense_equals_general(name, tmp_path):
    dims, C, brick, fmt, ops = CASES[name]
    if ops is None:
        ops = _slabs(dims, brick[2])
    elif ops == "step2":
        ops = _slabs(dims, brick[2], step=2)
    ops = list(ops) + [("sync",), ("borders",)]
    ta, ea, sa = _run(dims, C, brick, fmt, ops, dense=False)
    tb, eb, sb = _run(dims, C, brick, fmt, ops, dense=True)
    leaf_inserts = tb.dense_counts()[0]
    assert leaf_inserts == sum(1 for o in ops if o[0] == "slab")
    assert ta.dense_counts() == (0, 0, 0)
    assert eb == ea
    assert sb == sa
    assert _nodes(tb) == _nodes(ta)
    assert _bricks(tb) == _bricks(ta)
    assert tb.checksum() == ta.checksum()
    assert digest(tb, tmp_path, "b") == digest(ta, tmp_path, "a")


def test_dense_interleaved_flushes_and_general_inserts(tmp_path):
    """Reads between layers (parents with incomplete subtrees go through the
    general path), general-path boxes over dense leaves and over fresh
    leaves, then dense layers again."""
    dims, C, brick, fmt = (32, 24, 56), 3, (8, 8, 8), "uint16"
    ops = [("slab", 0, 8), ("sync",),
           ("slab", 8, 16), ("box", 1, (3, 2, 9), (20, 7, 5)), ("sync",),
           ("box", 0, (0, 0, 16), (32, 24, 3)),      # partial layer: general path
           ("slab", 24, 40), ("sync",),
           ("box", 2, (1, 1, 16), (9, 9, 8)),
           ("slab", 40, 56), ("sync",),
           ("box", 0, (0, 0, 19), (32, 24, 5)), ("box", 1, (0, 0, 16), (32, 24, 8)),
           ("box", 2, (0, 0, 16), (32, 24, 8)), ("sync",),
           ("borders",)]
    ta, ea, sa = _run(dims, C, brick, fmt, ops, dense=False)
    tb, eb, sb = _run(dims, C, brick, fmt, ops, dense=True)
    # 4 dense slabs + the partial single-channel layer a later slab closes
    # (materialised by the dense leaf kernel, missing planes = seeds)
    assert tb.dense_counts()[0] == 5
    assert eb == ea
    assert sb == sa
    assert _nodes(tb) == _nodes(ta)
    assert _bricks(tb) == _bricks(ta)
    assert digest(tb, tmp_path, "b") == digest(ta, tmp_path, "a")


def test_dense_background_and_device_source(tmp_path):
    """Non-zero background (shells, out-of-volume octants) and a device
    (torch) source block; odd row alignment of 16-bit words."""
    import torch
    dims, C, brick, fmt = (34, 18, 20), 3, (8, 8, 4), "uint16"
    vol = _volume(dims, C, fmt, seed=7)
    res = []
    for dense in (False, True):
        t = _tree(dims, C, brick, fmt, dense, bg=4321)
        dv = torch.from_numpy(vol.view(np.int16)).cuda().view(torch.uint16)
        for z0 in range(0, dims[2], 4):
            t.insert_channels((0, 0, z0), dv[z0:z0 + 4])
        t.finalize()
        t.fill_borders()
        t.sync()
        res.append((t.checksum(), _nodes(t), _bricks(t), digest(t, tmp_path, str(dense)),
                    t.dense_counts()))
    assert res[1][4][0] == 5 and res[0][4] == (0, 0, 0)
    assert res[1][:4] == res[0][:4]


def test_dense_matches_oracle_small():
    """Direct check against the CPU oracle (not only the general path)."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle"))
    import voxtree_oracle as vo
    dims, C, brick = (24, 20, 16), 3, (8, 8, 8)
    vol = vo.synth_spim(dims, C, 65535, seed=3)
    t = _tree(dims, C, brick, "uint16", True)
    t.insert_channels((0, 0, 0), vol)
    t.finalize()
    t.fill_borders()
    t.sync()
    assert t.dense_counts()[0] == 1
    ot = vo.OracleTree(dims, brick, channels=C, fmt="uint16", threshold=0)
    for c in range(C):
        ot.insert(c, (0, 0, 0), vol[..., c])
    ot.finished = True
    ot.fill_borders()
    assert t.brick_count == len(ot.bricks)
    assert sorted(n.index for n in t.iter_nodes()) == sorted(ot.exists)
    for n in t.iter_nodes():
        i = n.index
        assert list(n.avg) == list(ot.avg[i]) and list(n.smin) == list(ot.smin[i])
        assert list(n.smax) == list(ot.smax[i])
        if n.brick is not None:
            assert np.array_equal(t.store.read_brick(n.brick), ot.bricks[n.index]), n.index


PREFILL_CASES = {
    # dims, C, brick, slab height (in bricks), bg
    "cfg_like_slabs": ((64, 48, 40), 3, (8, 8, 8), 1, 0),
    "two_layer_slabs_bg": ((48, 40, 72), 2, (8, 8, 8), 2, 17),
    "bulk_partial": ((40, 36, 50), 3, (8, 8, 8), 100, 0),
    "bulk_pow2_bg": ((64, 64, 64), 3, (8, 8, 8), 100, 5),
    # complete leaf grids in one insertion (parent slots by BFS rank, leaves
    # as one BFS range), incl. the compile-time 32x32 copy for C = 1, 2, 4
    "grid_b32_c1": ((128, 128, 64), 1, (32, 32, 32), 100, 0),
    "grid_b32_c2": ((64, 64, 64), 2, (32, 32, 32), 100, 9),
    "grid_b32_c4": ((64, 64, 128), 4, (32, 32, 32), 100, 0),
    "grid_b16_c2": ((64, 64, 64), 2, (16, 16, 16), 100, 0),
    "nonsplit_z": ((32, 16, 6), 3, (8, 8, 8), 1, 3),
    # whole volumes whose interior level-1 parents get their x/y shells from
    # the leaf kernel and their z shells from parent seams
    "bulk_interior_parents": ((96, 80, 64), 3, (8, 8, 8), 100, 0),
    "bulk_interior_parents_bg": ((112, 88, 72), 2, (8, 8, 8), 100, 13),
    "grid_b16_interior": ((160, 128, 96), 3, (16, 16, 16), 100, 0),
    "brick16_c4": ((64, 32, 48), 4, (16, 16, 16), 1, 0),
}


@pytest.mark.parametrize("name", sorted(PREFILL_CASES))
def test_dense_prefilled_shells_fast_borders(name, tmp_path):
    """Leaf shells written at insertion (TMA tile with halo) + fill_borders
    patching only the owed z-shells: byte-identical to the general path."""
    dims, C, brick, step, bg = PREFILL_CASES[name]
    ops = _slabs(dims, brick[2], step=step) + [("borders",)]
    ta, ea, _ = _run(dims, C, brick, "uint16", ops, dense=False, bg=bg)
    tb, eb, _ = _run(dims, C, brick, "uint16", ops, dense=True, bg=bg)
    assert tb.dense_counts()[2] == 1, "fill_borders did not take the prefilled-shell path"
    assert eb == ea
    assert _nodes(tb) == _nodes(ta)
    assert _bricks(tb) == _bricks(ta)
    assert digest(tb, tmp_path, "b") == digest(ta, tmp_path, "a")


@pytest.mark.parametrize("dims,whole", [((32, 24, 40), False), ((32, 24, 40), True),
                                        ((40, 36, 50), True), ((64, 64, 64), True),
                                        ((96, 80, 64), True)])
def test_prefilled_shells_read_as_background_before_fill_borders(tmp_path, dims, whole):
    """Before fill_borders a prefilled shell is the reference's background to
    every reader (read_brick, export, checksum, device mirror).  A whole-volume
    insertion also computes the parents' shells and owes their background
    (Tree::upper_borders / owed_shells): the same contract."""
    from paper_1407_2074_b200 import DeviceState
    C, brick = 3, (8, 8, 8)
    ops = [("slab", 0, dims[2])] if whole else _slabs(dims, brick[2])
    ta, _, _ = _run(dims, C, brick, "uint16", ops, dense=False)
    tb, _, _ = _run(dims, C, brick, "uint16", ops, dense=True)
    assert _bricks(tb) == _bricks(ta)
    assert tb.checksum() == ta.checksum()
    assert digest(tb, tmp_path, "b") == digest(ta, tmp_path, "a")
    tc, _, _ = _run(dims, C, brick, "uint16", ops, dense=True)
    DeviceState(tc, resident_all=True)  # mirror first, then read
    assert _bricks(tc) == _bricks(ta)
    for t in (ta, tb, tc):
        t.finalize()
        t.fill_borders()
    assert tb.dense_counts()[2] == 0 and tc.dense_counts()[2] == 0
    assert _bricks(tb) == _bricks(ta) == _bricks(tc)


def _run_stream(dims, C, brick, blocks, dense, snap_at=(), bg=0):
    """blocks: (z, dz, channel) single-channel full-x/y blocks in order, or
    ("box", c, origin, size) general blocks; a checksum read after the block
    indices in snap_at (a reader materialises a partial deferred layer)."""
    t = _tree(dims, C, brick, "uint16", dense, bg)
    vol = _volume(dims, C, "uint16", seed=11)
    evs, snaps = [], []
    for i, b in enumerate(blocks):
        if b[0] == "box":
            _, c, o, sz = b
            blk = vol[o[2]:o[2] + sz[2], o[1]:o[1] + sz[1], o[0]:o[0] + sz[0], c]
            evs.append(_events(t.insert_block(c, o, np.ascontiguousarray(blk))))
        else:
            z, dz, c = b
            evs.append(_events(t.insert_block(c, (0, 0, z),
                                              np.ascontiguousarray(vol[z:z + dz, :, :, c]))))
        if i in snap_at:
            snaps.append((t.checksum(), _nodes(t)))
    t.finalize()
    t.fill_borders()
    t.sync()
    return t, evs, snaps


def _vstr_order(dims, C, dz=1):
    return [(z, min(dz, dims[2] - z), c) for z in range(0, dims[2], dz) for c in range(C)]


STREAM_CASES = {
    "vstr_slices": ((48, 40, 50), 3, (8, 8, 8), "vstr", ()),
    "vstr_slices_reads": ((40, 32, 40), 3, (8, 8, 8), "vstr", (5, 40, 41, 77)),
    "vstr_two_slice_blocks": ((32, 24, 36), 2, (8, 8, 8), "vstr2", (9,)),
    "channel_major": ((32, 24, 24), 3, (8, 8, 8), "chmajor", ()),
    "shuffled_in_layer": ((32, 32, 32), 3, (8, 8, 8), "shuffled", (30,)),
    "general_block_between": ((32, 32, 24), 3, (8, 8, 8), "mixed", ()),
    "brick16_c4": ((64, 32, 40), 4, (16, 16, 16), "vstr", (70,)),
}


@pytest.mark.parametrize("name", sorted(STREAM_CASES))
def test_deferred_stream_layers_equal_general(name, tmp_path):
    """Slice streams (ingest_stream's VSTR order) through the deferred
    brick-layer path == the general path, with reads in the middle of layers
    (materialisation), other orders and general blocks in between."""
    dims, C, brick, kind, snaps = STREAM_CASES[name]
    if kind == "vstr":
        blocks = _vstr_order(dims, C)
    elif kind == "vstr2":
        blocks = _vstr_order(dims, C, dz=2)
    elif kind == "chmajor":
        blocks = [(z, 1, c) for c in range(C) for z in range(dims[2])]
    elif kind == "shuffled":
        rng = np.random.default_rng(5)
        blocks = []
        for z0 in range(0, dims[2], brick[2]):
            layer = [(z, 1, c) for z in range(z0, min(dims[2], z0 + brick[2])) for c in range(C)]
            rng.shuffle(layer)
            blocks += [tuple(int(v) for v in b) for b in layer]
    else:
        blocks = _vstr_order(dims, C)
        blocks.insert(13, ("box", 1, (3, 4, 2), (9, 7, 3)))
        blocks.insert(40, ("box", 0, (0, 0, 9), (32, 32, 1)))
    ta, ea, sa = _run_stream(dims, C, brick, blocks, dense=False, snap_at=snaps)
    tb, eb, sb = _run_stream(dims, C, brick, blocks, dense=True, snap_at=snaps)
    assert eb == ea
    assert sb == sa
    assert _nodes(tb) == _nodes(ta)
    assert _bricks(tb) == _bricks(ta)
    assert digest(tb, tmp_path, "b") == digest(ta, tmp_path, "a")
    if kind in ("vstr", "vstr2") and not snaps:
        # every layer completed without a reader: all built by the dense kernel
        assert tb.dense_counts()[0] == -(-dims[2] // brick[2])
