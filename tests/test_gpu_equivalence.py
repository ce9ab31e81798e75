"""The reference's equivalence tests (tests/test_equivalence.py and the
render properties of tests/test_render.py / tests/test_properties.py),
restated through the drop-in API on the GPU: refinement to completion vs the
in-core level-0 oracle (render/oracle.py:26-88, restated in
oracle/voxtree_oracle.py:render_reference_volume), with clips and channel
transforms; full frame == refinement when everything is resident; the
converged image independent of the brick-buffer size; bounded refinement
progress with one slot; monotone AVG fallbacks under uploads; a collapsed
homogeneous volume rendered from its AVG; tile restriction; an orbit that
stops uploading; flag soundness.  Tolerance: the reference's TOL = 1e-5."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5
COLORS = [(1.0, 0.2, 0.1), (0.1, 1.0, 0.2), (0.2, 0.1, 1.0), (1.0, 1.0, 0.2)]


def _tfs(channels):
    from paper_1407_2074_b200.render import TransferFunction
    return [TransferFunction([(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, *COLORS[c], 0.5)])
            for c in range(channels)]


def build_tree(volume, brick, *, threshold=0, bg=0, transforms=None, fill=True):
    """tests/helpers.py:11-29: an octree over a (z, y, x[, c]) uint8 volume."""
    from gpu_helpers import make_tree
    if volume.ndim == 3:
        volume = volume[..., None]
    dz, dy, dx, nc = volume.shape
    t = make_tree(dict(dims=(dx, dy, dz), brick=brick, threshold=threshold, fmt="uint8",
                       channels=nc, bg=bg, transforms=transforms, page_bricks=16,
                       ram_page_limit=64))
    for c in range(nc):
        t.insert_block(c, (0, 0, 0), np.ascontiguousarray(volume[..., c]))
    t.finalize()
    if fill:
        t.fill_borders()
    return t


def make_scene(dims, *, mode="dvr", strategy="refinement", viewport=(24, 24), tfs=None,
               clips=None, channels=1, lod_bias=-64.0, distance_scale=2.5, early=0.99):
    """tests/helpers.py:32-48."""
    from paper_1407_2074_b200.render import (Camera, RenderSettings, Scene, TransferFunction)
    center = tuple(d / 2 for d in dims)
    cam = Camera(position=(center[0], center[1], -distance_scale * max(dims)), look_at=center,
                 up=(0, 1, 0), fov_y=np.pi / 4, width=viewport[0], height=viewport[1])
    st = RenderSettings(mode=mode, strategy=strategy, lod_bias=lod_bias,
                        early_termination_alpha=early)
    if tfs is None:
        tfs = [TransferFunction.ramp(max_alpha=0.6) for _ in range(channels)]
    sc = Scene(camera=cam, settings=st, transfer_functions=tfs)
    if clips is not None:
        sc.clips = clips
    return sc


def refine_to_completion(renderer, device, scene, max_passes=1000):
    """tests/helpers.py:51-61."""
    from paper_1407_2074_b200 import RenderMode
    session = renderer.start_refinement(scene)
    while not session.run_pass():
        plan = device.process_flags(RenderMode.REFINEMENT)
        uploaded = device.upload_bricks(plan, budget_ms=1e9)
        assert uploaded or plan, "refinement stalled"
        assert session.passes < max_passes
    return session


def oracle_image(volume, tree, scene):
    """ReferenceRenderer(volume, desc).render(scene) (render/oracle.py:26-88)."""
    import voxtree_oracle as vo
    d = tree.descriptor
    ot = vo.OracleTree(d.dims, tree.config.brick_dims, channels=d.channels, fmt="uint8",
                       bg=d.background_value, threshold=0, spacing=d.spacing,
                       transforms=d.channel_transforms)
    cam, st = scene.camera, scene.settings
    spec = vo.SceneSpec(position=cam.position, look_at=cam.look_at, up=cam.up, fov_y=cam.fov_y,
                        width=cam.width, height=cam.height, mode=st.mode,
                        sampling_step=st.sampling_step,
                        early_termination_alpha=st.early_termination_alpha,
                        lod_bias=st.lod_bias,
                        tfs=[tf.control_points() for tf in scene.transfer_functions],
                        clips=[(p.normal, p.offset) for p in scene.clips])
    return vo.render_reference_volume(volume, ot, spec)


def _vol(seed, size, channels):
    return np.random.default_rng(seed).integers(0, 255, size=(size, size, size, channels),
                                                dtype=np.uint8)


@pytest.mark.parametrize("channels", [1, 2, 3])
@pytest.mark.parametrize("mode", ["dvr", "mip"])
def test_completed_refinement_matches_oracle(channels, mode):
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    vol = _vol(channels * 10 + (mode == "mip"), 16, channels)
    tree = build_tree(vol, (4, 4, 4))
    dev = DeviceState(tree, slot_count=80)
    scene = make_scene((16, 16, 16), mode=mode, channels=channels, tfs=_tfs(channels),
                       viewport=(20, 20))
    session = refine_to_completion(OutOfCoreRenderer(dev), dev, scene)
    assert np.max(np.abs(session.image() - oracle_image(vol, tree, scene))) <= TOL


def test_refinement_matches_oracle_with_clip_planes():
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import ClipPlane, ClipSet, OutOfCoreRenderer
    vol = _vol(42, 16, 2)
    tree = build_tree(vol, (4, 4, 4))
    dev = DeviceState(tree, slot_count=80)
    clips = ClipSet((ClipPlane((1.0, 0.0, 0.0), 10.0), ClipPlane((0.0, -1.0, 0.0), -3.0)))
    scene = make_scene((16, 16, 16), channels=2, tfs=_tfs(2), viewport=(20, 20), clips=clips)
    session = refine_to_completion(OutOfCoreRenderer(dev), dev, scene)
    assert np.max(np.abs(session.image() - oracle_image(vol, tree, scene))) <= TOL


def test_refinement_matches_oracle_with_channel_translation():
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    vol = _vol(43, 16, 2)
    tr = np.stack([np.eye(4), np.eye(4)])
    tr[1, 0, 3] = 1.0
    tree = build_tree(vol, (4, 4, 4), transforms=tr)
    dev = DeviceState(tree, slot_count=80)
    scene = make_scene((16, 16, 16), channels=2, tfs=_tfs(2), viewport=(20, 20))
    session = refine_to_completion(OutOfCoreRenderer(dev), dev, scene)
    assert np.max(np.abs(session.image() - oracle_image(vol, tree, scene))) <= TOL


def test_identity_transforms_bit_identical_to_disabled():
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    vol = _vol(44, 8, 2)
    scene = make_scene((8, 8, 8), channels=2, tfs=_tfs(2), viewport=(12, 12))
    images = []
    for tr in (None, np.stack([np.eye(4), np.eye(4)])):
        tree = build_tree(vol, (4, 4, 4), transforms=tr)
        dev = DeviceState(tree, slot_count=40)
        images.append(refine_to_completion(OutOfCoreRenderer(dev), dev, scene).image())
    assert np.array_equal(images[0], images[1])


def test_translation_against_constructed_ground_truth():
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    base = np.random.default_rng(45).integers(0, 255, size=(8, 8, 9), dtype=np.uint8)
    vol = np.zeros((8, 8, 8, 2), dtype=np.uint8)
    vol[..., 0] = base[:, :, :8]
    vol[..., 1] = base[:, :, 1:]
    tr = np.stack([np.eye(4), np.eye(4)])
    tr[1, 0, 3] = -1.0
    tree = build_tree(vol, (4, 4, 4), transforms=tr)
    dev = DeviceState(tree, slot_count=80)
    tf = _tfs(1)
    scene = make_scene((8, 8, 8), channels=2, viewport=(20, 20), tfs=[tf[0], tf[0]],
                       distance_scale=1.25)
    image = refine_to_completion(OutOfCoreRenderer(dev), dev, scene).image()
    dup = np.stack([vol[..., 0], vol[..., 0]], axis=-1)
    oracle = oracle_image(dup, build_tree(dup, (4, 4, 4)), scene)
    assert np.max(np.abs(image[:, 7:14] - oracle[:, 7:14])) <= 1e-5
    assert oracle[:, 7:14, 3].max() > 0.5


def test_fullframe_equals_refinement_when_all_resident():
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    tree = build_tree(_vol(46, 16, 1), (4, 4, 4))
    dev = DeviceState(tree, slot_count=80)
    r = OutOfCoreRenderer(dev)
    scene = make_scene((16, 16, 16), viewport=(16, 16))
    session = refine_to_completion(r, dev, scene)
    full, counters = r.render_fullframe(scene)
    assert counters.avg_fallbacks == 0 and counters.coarse_fallbacks == 0
    assert np.array_equal(full, session.image())


def test_converged_image_invariant_to_buffer_size():
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    tree = build_tree(_vol(47, 16, 1), (4, 4, 4))
    scene = make_scene((16, 16, 16), viewport=(12, 12))
    images, passes = [], []
    for slots in (1, 64):
        dev = DeviceState(tree, slot_count=slots)
        s = refine_to_completion(OutOfCoreRenderer(dev), dev, scene)
        images.append(s.image())
        passes.append(s.passes)
    assert np.array_equal(images[0], images[1])
    assert passes[0] > passes[1]


def test_refinement_progress_bounded_with_single_slot():
    from paper_1407_2074_b200 import DeviceState, RenderMode
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    tree = build_tree(_vol(48, 16, 1), (4, 4, 4))
    dev = DeviceState(tree, slot_count=1)
    session = OutOfCoreRenderer(dev).start_refinement(make_scene((16, 16, 16), viewport=(8, 8)))
    prev = None
    while not session.run_pass():
        remaining = int(np.sum(session.rays.n_steps - session.rays.k))
        if prev is not None:
            assert remaining < prev
        prev = remaining
        dev.upload_bricks(dev.process_flags(RenderMode.REFINEMENT), budget_ms=1e9)
        assert session.passes <= tree.brick_count + 5
    assert session.passes <= tree.brick_count + 5


def test_fullframe_avg_fallbacks_monotone_under_uploads():
    from paper_1407_2074_b200 import DeviceState, RenderMode
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    tree = build_tree(_vol(49, 16, 1), (4, 4, 4))
    dev = DeviceState(tree, slot_count=16)
    r = OutOfCoreRenderer(dev)
    scene = make_scene((16, 16, 16), viewport=(12, 12), lod_bias=0.0)
    counts = []
    for _ in range(8):
        _, c = r.render_fullframe(scene)
        counts.append(c.avg_fallbacks)
        dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), budget_ms=1e9)
    assert all(b <= a for a, b in zip(counts, counts[1:]))
    assert counts[-1] == 0


def test_homogeneous_volume_renders_from_avg_with_empty_buffer():
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer, TransferFunction
    tree = build_tree(np.full((8, 8, 8), 180, dtype=np.uint8), (4, 4, 4), threshold=2)
    assert tree.brick_count == 0
    dev = DeviceState(tree, slot_count=1)
    tf = TransferFunction.constant(0.3, 0.6, 0.9, 1.0)
    image, c = OutOfCoreRenderer(dev).render_fullframe(
        make_scene((8, 8, 8), viewport=(9, 9), tfs=[tf]))
    assert c.avg_fallbacks == 0
    assert image[4, 4, :3] == pytest.approx([0.3, 0.6, 0.9], abs=1e-9)
    assert image[4, 4, 3] == pytest.approx(1.0)


def test_pruning_disabled_at_zero_threshold_matches_forced_off():
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    vol = _vol(50, 8, 1)
    vol[:4] = 60
    scene = make_scene((8, 8, 8), viewport=(10, 10))
    images = []
    for dense in (True, False):  # the B200 dense build on / forced off
        tree = build_tree(vol, (4, 4, 4), threshold=0)
        tree.dense_build = dense
        assert tree.pruned_bricks == 0
        dev = DeviceState(tree, slot_count=40)
        images.append(refine_to_completion(OutOfCoreRenderer(dev), dev, scene).image())
    assert np.array_equal(images[0], images[1])


def test_refinement_tile_restricts_to_rectangle():
    from paper_1407_2074_b200 import DeviceState, RenderMode
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    tree = build_tree(_vol(51, 16, 1), (4, 4, 4))
    dev = DeviceState(tree, slot_count=80)
    r = OutOfCoreRenderer(dev)
    scene = make_scene((16, 16, 16), viewport=(16, 16))
    full = refine_to_completion(r, dev, scene).image()
    session = r.start_refinement(scene, tile=(4, 4, 12, 12))
    while not session.run_pass():
        dev.upload_bricks(dev.process_flags(RenderMode.REFINEMENT), budget_ms=1e9)
    tiled = session.image()
    assert np.array_equal(tiled[4:12, 4:12], full[4:12, 4:12])
    outside = np.ones((16, 16), dtype=bool)
    outside[4:12, 4:12] = False
    assert np.all(tiled[outside] == 0.0)


def test_orbit_reaches_stable_brick_configuration():
    from paper_1407_2074_b200 import DeviceState, RenderMode
    from paper_1407_2074_b200.render import Camera, OutOfCoreRenderer
    tree = build_tree(_vol(52, 16, 1), (4, 4, 4))
    dev = DeviceState(tree, slot_count=128)
    r = OutOfCoreRenderer(dev)
    scene = make_scene((16, 16, 16), viewport=(12, 12), lod_bias=0.0)
    per_frame = []
    for i in range(12):
        a = 2 * np.pi * i / 12
        scene.camera = Camera(position=(8 + 40 * np.sin(a), 8.0, 8 - 40 * np.cos(a)),
                              look_at=(8, 8, 8), up=(0, 1, 0), width=12, height=12)
        before = dev.uploads
        r.render_fullframe(scene)
        dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), budget_ms=1e9)
        per_frame.append(dev.uploads - before)
    assert sum(per_frame[6:]) == 0, per_frame


def test_flag_soundness_after_fullframe_pass():
    """tests/test_properties.py:139-170: a cold pass sets only requested bits,
    on non-homogeneous non-resident nodes; a warm pass sets used bits only on
    resident bricks."""
    from paper_1407_2074_b200 import DeviceState, RenderMode
    from paper_1407_2074_b200.device import FLAG_REQUESTED, FLAG_USED
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    vol = np.random.default_rng(0).integers(0, 255, size=(16, 16, 16), dtype=np.uint8)
    tree = build_tree(vol, (4, 4, 4))
    dev = DeviceState(tree, slot_count=8)
    r = OutOfCoreRenderer(dev)
    scene = make_scene((16, 16, 16), viewport=(10, 10))
    r.render_fullframe(scene)
    flags = dev.read_flags()
    assert not (flags & ~np.uint8(3)).any()
    assert not (flags & FLAG_USED).any()
    requested = np.flatnonzero(flags & FLAG_REQUESTED)
    assert requested.size > 0
    nb = dev.node_buffer_host()
    for idx in requested:
        e = int(nb[idx])
        assert e & 2 and not e & 1
    dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), budget_ms=1e9)
    r.render_fullframe(scene)
    flags = dev.read_flags()
    used = np.flatnonzero(flags & FLAG_USED)
    assert used.size > 0
    nb = dev.node_buffer_host()
    for idx in used:
        assert int(nb[idx]) & 1
