"""GPU parity at the BASELINE configs against golden vectors made by the
UNMODIFIED reference (tests/golden/make_golden_cfg.py, scenarios in
tests/cfg_scenarios.py):

* cfg1 (256^3 x 3 uint8, 32^3 bricks, tau 0 and 12.75): whole-volume and
  VSTR-order slice-stream builds — per-insertion change events (sha256),
  node/brick/prune counts, VXOC/VXBP digests before and after fill_borders;
  the slice stream also through Octree.insert_many (batched, planar device
  slices and host slices); the 512x512 DVR frame with the clip z <= 200:
  image (<= 1e-6 against the reference's float64 frame stored as float32;
  north-star tolerance 1/255), RGBA8, counters, used/requested flag sets,
  and the node buffer after the reference's upload policy made every brick
  resident (device.py:241-360).
* cfg2 (1024^3 x 3 uint16, the bench's build and 1920x1080 frame): VXOC/VXBP
  digests of the bench's one-call device build; three 64x64 tiles through
  the tile-restricted RefinementSession (render/raycast.py:309-315): pixels,
  counters and flag sets.
* cfg3 crop (256^2 x 64 of the 2048^2 x 1000 SPIM volume, VSTR order, tau 0
  and 3276.75): events and digests, per-slice and batched.
"""

import json
import os

import numpy as np
import pytest

import cfg_scenarios as cs
from gpu_helpers import counters_dict, make_tree, to_scene

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(part):
    with open(os.path.join(GOLD, f"golden_{part}.json")) as fh:
        g = json.load(fh)
    p = os.path.join(GOLD, f"renders_{part}.npz")
    return g, (np.load(p) if os.path.exists(p) else None)


G1, R1 = _load("cfg1")
G2, R2 = _load("cfg2")
G3, _ = _load("cfg3")

_VOL = {}


def _cfg1_vol():
    if "cfg1" not in _VOL:
        _VOL["cfg1"] = cs.cfg1_volume()
    return _VOL["cfg1"]


def _cfg3_vol():
    if "cfg3" not in _VOL:
        _VOL["cfg3"] = cs.cfg3_crop_volume()
    return _VOL["cfg3"]


def _digests(tree):
    from paper_1407_2074_b200.serialize import octree_digests
    return list(octree_digests(tree))


def _build_per_insert(spec, ops):
    tree = make_tree(spec)
    per = []
    for c, o, v in ops:
        ev = tree.insert_block(c, o, v)
        per.append((ev.kinds, ev.indices))
    tree.drain_events()
    return tree, per


def _check_build(tree, per, gold):
    assert cs.events_digest(per) == (gold["events_sha256"], gold["events_total"])
    assert tree.node_count == gold["node_count"]
    assert tree.brick_count == gold["brick_count"]
    assert tree.pruned_bricks == gold["pruned_bricks"]
    assert _digests(tree) == gold["digest_unfinished"]
    tree.finalize()
    tree.fill_borders()
    assert len(tree.drain_events()) == gold["border_events"]
    assert _digests(tree) == gold["digest_final"]


# ---------------------------------------------------------------------------
# cfg1
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", sorted(G1["builds"]))
def test_cfg1_build_vs_reference(name):
    mode, tau = name.split("_")
    spec = cs.tree_spec(cs.CFG1, cs.CFG1_TAUS[tau])
    tree, per = _build_per_insert(spec, cs.ops(_cfg1_vol(), mode))
    _check_build(tree, per, G1["builds"][name])


def _planar_device(vol):
    import torch
    # (C, Z, Y, X): every slice of a channel plane is an affine view
    return torch.as_tensor(np.ascontiguousarray(np.moveaxis(vol, 3, 0))).cuda()


@pytest.mark.parametrize("source", ["device_planar", "device_separate", "host"])
@pytest.mark.parametrize("tau", sorted(cs.CFG1_TAUS))
def test_cfg1_stream_insert_many(tau, source):
    """the slice stream through Octree.insert_many: the reference's digests
    and exactly the queued events of the per-slice insert_block loop"""
    import torch
    vol = _cfg1_vol()
    spec = cs.tree_spec(cs.CFG1, cs.CFG1_TAUS[tau])
    ref_tree, per = _build_per_insert(spec, cs.ops(vol, "stream"))
    want_k = np.concatenate([p[0] for p in per])
    want_i = np.concatenate([p[1] for p in per])
    tree = make_tree(spec)
    if source == "device_planar":
        pv = _planar_device(vol)
        blocks = [(c, (0, 0, z), pv[c, z:z + 1]) for z in range(vol.shape[0]) for c in range(3)]
    elif source == "device_separate":
        blocks = [(c, o, torch.as_tensor(np.ascontiguousarray(v)).cuda())
                  for c, o, v in cs.ops(vol, "stream")]
    else:
        blocks = cs.ops(vol, "stream")
    tree.insert_many(blocks)
    ev = tree.drain_events()
    assert np.array_equal(ev.kinds, want_k) and np.array_equal(ev.indices, want_i)
    assert isinstance(ev, list) and len(ev) == len(want_k)
    assert ev[:7] + ev[-7:] == _as_events((want_k[:7], want_i[:7])) + _as_events(
        (want_k[-7:], want_i[-7:]))
    gold = G1["builds"][f"stream_{tau}"]
    assert tree.brick_count == gold["brick_count"]
    assert tree.pruned_bricks == gold["pruned_bricks"]
    assert _digests(tree) == gold["digest_unfinished"]
    tree.finalize()
    tree.fill_borders()
    assert _digests(tree) == gold["digest_final"]
    groups, _, _ = tree.stream_counts()
    if tau == "tau0":
        assert groups == -(-vol.shape[0] // 32)  # every brick layer in one dense insertion
    del ref_tree


def _as_events(p):
    from paper_1407_2074_b200 import ChangeEvent, ChangeKind
    return [ChangeEvent(ChangeKind(int(k)), int(i)) for k, i in zip(*p)]


def _all_resident_policy(tree):
    """the reference's recipe: request every brick, run the
    upload policy, clear the flags"""
    import hashlib
    import torch
    from paper_1407_2074_b200 import DeviceState, RenderMode
    dev = DeviceState(tree, slot_count=tree.brick_count + 8)
    idx, fl = tree.node_indices(with_flags=True)
    bricked = idx[(fl & 8) != 0]
    fb = dev.flag_buffer
    fb[torch.as_tensor(bricked, device=fb.device)] |= 2
    plan = dev.process_flags(RenderMode.FULLFRAME)
    assert dev.upload_bricks(plan, 1e9) == len(bricked)
    dev.read_flags(clear=True)
    sha = hashlib.sha256(dev.node_buffer_host().astype("<u8").tobytes()).hexdigest()
    return dev, sha


@pytest.mark.parametrize("tau", sorted(cs.CFG1_TAUS))
def test_cfg1_render_vs_reference(tau):
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    gold = G1["renders"][f"frame_{tau}"]
    gb = G1["builds"][gold["build"]]
    spec = cs.tree_spec(cs.CFG1, cs.CFG1_TAUS[tau])
    tree, _ = _build_per_insert(spec, cs.ops(_cfg1_vol(), "bulk"))
    tree.finalize()
    tree.fill_borders()
    scene = to_scene(cs.scene_spec(cs.CFG1["dims"], **cs.CFG1_SCENE))
    ref = R1[f"frame_{tau}/image"].astype(np.float64)
    ref8 = R1[f"frame_{tau}/image_u8"]
    # the reference's bounded-residency mirror, every brick uploaded by its policy
    dev, sha = _all_resident_policy(tree)
    assert sha == gb["node_buffer_sha256"]
    for d in (dev, DeviceState(tree, resident_all=True)):
        img, cnt = OutOfCoreRenderer(d).render_fullframe(scene)
        err = float(np.max(np.abs(img - ref)))
        assert err <= 1.0 / 255.0
        assert err <= 1e-6, f"max err {err}"  # float32-stored golden
        img8 = np.clip(np.round(img * 255), 0, 255).astype(np.uint8)
        assert int(np.max(np.abs(img8.astype(int) - ref8.astype(int)))) <= 1
        assert counters_dict(cnt) == gold["counters"]
        assert cs.flag_sets(d.read_flags(clear=True)) == gold["flags"]


# ---------------------------------------------------------------------------
# cfg3 crop stream
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("tau", sorted(cs.CFG3_TAUS))
def test_cfg3_crop_stream_vs_reference(tau):
    vol = _cfg3_vol()
    spec = cs.tree_spec(cs.CFG3C, cs.CFG3_TAUS[tau])
    gold = G3["builds"][f"stream_{tau}"]
    tree, per = _build_per_insert(spec, cs.ops(vol, "stream"))
    _check_build(tree, per, gold)
    # batched, from one planar device array (read in place at tau 0)
    t2 = make_tree(spec)
    pv = _planar_device(vol)
    t2.insert_many([(c, (0, 0, z), pv[c, z:z + 1]) for z in range(vol.shape[0]) for c in range(3)])
    ev = t2.drain_events()
    assert len(ev) == gold["events_total"]
    assert _digests(t2) == gold["digest_unfinished"]
    t2.finalize()
    t2.fill_borders()
    assert _digests(t2) == gold["digest_final"]
    if tau == "tau0":
        assert t2.stream_counts()[:2] == (2, 2)  # two layers, both read in place


# ---------------------------------------------------------------------------
# cfg2: the bench's tree and frame
# ---------------------------------------------------------------------------

_CFG2 = {}


def _cfg2_tree():
    if "tree" in _CFG2:
        return _CFG2["tree"]
    import ctypes as ct
    import torch
    from paper_1407_2074_b200 import _lib
    spec = dict(cs.CFG2)
    dims = spec["dims"]
    vol = torch.empty((dims[2], dims[1], dims[0], 3), dtype=torch.uint16, device="cuda")
    _lib.call("vt_synth", ct.c_void_p(vol.data_ptr()), 1, _lib.i32x3(dims), 3, 2, 0, 0, dims[2],
              ct.c_void_p(torch.cuda.current_stream().cuda_stream))
    tree = make_tree(spec)
    tree.insert_channels((0, 0, 0), vol)  # the bench's device build
    tree.finalize()
    tree.fill_borders()
    tree.sync()
    del vol
    torch.cuda.empty_cache()
    _CFG2["tree"] = tree
    return tree


def test_cfg2_build_digest_vs_reference():
    gold = G2["builds"]["slabs_tau0"]
    tree = _cfg2_tree()
    assert tree.brick_count == gold["brick_count"] and tree.node_count == gold["node_count"]
    assert _digests(tree) == gold["digest_final"]


@pytest.mark.parametrize("name", [t[0] for t in cs.CFG2_TILES])
def test_cfg2_tile_vs_reference(name):
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    gold = G2["renders"][name]
    tile, bias = tuple(gold["tile"]), gold["lod_bias"]
    tree = _cfg2_tree()
    dev = DeviceState(tree, resident_all=True)
    dev.read_flags(clear=True)
    r = OutOfCoreRenderer(dev)
    scene = to_scene(cs.scene_spec(cs.CFG2["dims"], cs.CFG2_VIEWPORT, lod_bias=bias,
                                   clip_z=cs.CFG2_CLIP_Z), "refinement")
    sess = r.start_refinement(scene, tile=tile)
    while not sess.run_pass():
        pass
    assert sess.passes == gold["passes"]
    img = sess.image()
    x0, y0, x1, y1 = tile
    err = float(np.max(np.abs(img[y0:y1, x0:x1] - R2[name + "/tile"])))
    assert err <= 1.0 / 255.0
    assert err <= 1e-9, f"max err {err}"
    out = img.copy()
    out[y0:y1, x0:x1] = 0
    assert float(np.max(out)) == gold["outside_max"]
    assert counters_dict(sess.counters) == gold["counters"]
    assert cs.flag_sets(dev.read_flags(clear=True)) == gold["flags"]
    # the full 1920x1080 frame (the bench's render) agrees on the tile
    full, _ = r.render_fullframe(to_scene(cs.scene_spec(cs.CFG2["dims"], cs.CFG2_VIEWPORT,
                                                        lod_bias=bias, clip_z=cs.CFG2_CLIP_Z)))
    assert float(np.max(np.abs(full[y0:y1, x0:x1] - R2[name + "/tile"]))) <= 1e-9
