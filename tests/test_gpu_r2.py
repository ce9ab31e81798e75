"""GPU parity, round 2: channel-transform renders and the residency policy
against golden vectors made by the UNMODIFIED reference
(tests/golden/make_golden_r2.py, scenarios in tests/r2_scenarios.py), plus
the reference's own DeviceState policy tests (tests/test_device.py:98-290,
tests/test_acceptance.py:321-396) restated through the drop-in API.

Tolerance: images max |GPU - reference| <= 1/255 per RGBA component
(north_star); asserted <= 1e-9 (FP64 kernel).  Counters, flags, plans,
node buffers (sha256 of the Fig. 4 entries) and slot tables identical."""

import hashlib
import json
import os

import numpy as np
import pytest

import r2_scenarios as r2
from gpu_helpers import counters_dict, digest, make_tree, to_scene

pytestmark = pytest.mark.gpu

TOL = 1.0 / 255.0
GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "golden_r2.json")) as fh:
    GOLDEN = json.load(fh)
RENDERS = np.load(os.path.join(GOLD, "renders_r2.npz"))


def node_sha(dev):
    return hashlib.sha256(dev.node_buffer_host().astype("<u8").tobytes()).hexdigest()


def plan_list(plan):
    return [[int(i.node_index), int(i.slot), None if i.evicts is None else int(i.evicts)]
            for i in plan]


_TREES = {}


def xf_tree(name):
    if name not in _TREES:
        b = r2.xf_trees()[name]
        tree = make_tree(b["tree"])
        for c, o, v in b["ops"]:
            tree.insert_block(c, o, np.ascontiguousarray(v))
        tree.drain_events()
        tree.finalize()
        tree.fill_borders()
        tree.drain_events()
        _TREES[name] = tree
    return _TREES[name]


# -- channel transforms --------------------------------------------------------

@pytest.mark.parametrize("name", list(r2.xf_trees()))
def test_transform_tree_digest(name, tmp_path):
    tree = xf_tree(name)
    g = GOLDEN["builds"][name]
    assert (tree.node_count, tree.brick_count) == (g["node_count"], g["brick_count"])
    assert digest(tree, str(tmp_path), name) == g["digest"]


@pytest.mark.parametrize("name", list(r2.xf_cases()))
def test_transform_render_vs_reference(name):
    from paper_1407_2074_b200 import DeviceState, RenderMode
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    rc = r2.xf_cases()[name]
    gold = GOLDEN["renders"][name]
    tree = xf_tree(rc["build"])
    scene = to_scene(rc["scene"], rc["strategy"])
    if rc["resident"] == "all":
        dev = DeviceState(tree, resident_all=True)
    elif rc["resident"] == "slots":
        dev = DeviceState(tree, slot_count=rc["slots"])
    else:
        dev = DeviceState(tree, slot_count=tree.brick_count + 8)
    r = OutOfCoreRenderer(dev)
    if rc["strategy"] == "fullframe":
        img, cnt = r.render_fullframe(scene)
        err = float(np.max(np.abs(img - RENDERS[name + "/image"])))
        assert err <= TOL and err <= 1e-9, f"{name}: max err {err}"
        assert counters_dict(cnt) == gold["counters"]
        assert np.array_equal(dev.read_flags(), RENDERS[name + "/flags"])
        if rc["resident"] == "none":
            plan = dev.process_flags(RenderMode.FULLFRAME)
            assert plan_list(plan) == gold["plan"]
            dev.upload_bricks(plan, 1e9)
            img2, cnt2 = r.render_fullframe(scene)
            assert float(np.max(np.abs(img2 - RENDERS[name + "/image2"]))) <= 1e-9
            assert counters_dict(cnt2) == gold["counters2"]
            assert np.array_equal(dev.read_flags(), RENDERS[name + "/flags2"])
            dev.check_consistency()
    else:
        sess = r.start_refinement(scene, tile=rc.get("tile"))
        plans = []
        while not sess.run_pass():
            plan = dev.process_flags(RenderMode.REFINEMENT)
            plans.append(plan_list(plan))
            dev.upload_bricks(plan, 1e9)
            assert sess.passes <= 500
        assert plans == gold["plans"]
        assert sess.passes == gold["passes"]
        assert counters_dict(sess.counters) == gold["counters"]
        err = float(np.max(np.abs(sess.image() - RENDERS[name + "/image"])))
        assert err <= 1e-9, f"{name}: max err {err}"
        dev.check_consistency()


# -- residency: the 1/64 full-frame guarantee (tests/test_acceptance.py:321-348) --

def test_fullframe_one_sixty_fourth_guarantee_vs_reference(tmp_path):
    from paper_1407_2074_b200 import DeviceState, RenderMode
    from paper_1407_2074_b200.render import OutOfCoreRenderer
    gold = GOLDEN["ff64"]
    tree = make_tree(r2.ff64_tree())
    tree.insert_block(0, (0, 0, 0), r2.ff64_volume())
    tree.finalize()
    tree.fill_borders()
    tree.drain_events()
    assert digest(tree, str(tmp_path), "ff64") == gold["digest"]
    payload = tree.store.payload_nbytes
    slots = max(1, (payload // 64) // tree.config.brick_nbytes(tree.descriptor))
    assert (payload, slots) == (gold["payload"], gold["slots"])
    dev = DeviceState(tree, slot_count=slots)
    r = OutOfCoreRenderer(dev)
    fallbacks = []
    for i, g in enumerate(gold["frames"]):
        img, cnt = r.render_fullframe(to_scene(r2.ff64_scene_spec(i), "fullframe"))
        plan = dev.process_flags(RenderMode.FULLFRAME)
        done = dev.upload_bricks(plan, budget_ms=1e9)
        assert counters_dict(cnt) == g["counters"], i
        assert plan_list(plan) == g["plan"], i
        assert done == g["uploaded"]
        assert node_sha(dev) == g["node_sha"], i
        assert dev.pending_requests == g["pending"]
        if f"ff64/{i}" in RENDERS:
            assert float(np.max(np.abs(img - RENDERS[f"ff64/{i}"]))) <= 1e-9, i
        fallbacks.append(cnt.avg_fallbacks)
    assert all(f == 0 for f in fallbacks[2:]), fallbacks
    dev.check_consistency()


# -- residency: apply_events over a pruning tree (device.py:205-237) ------------

def test_apply_events_sequence_vs_reference():
    from paper_1407_2074_b200.device import FLAG_REQUESTED, DeviceState, RenderMode
    gold = GOLDEN["events"]
    tree = make_tree(r2.events_tree())
    dev = DeviceState(tree, slot_count=4)
    for step, ((origin, block), g) in enumerate(zip(r2.events_ops(), gold["steps"])):
        tree.insert_block(0, origin, block)
        evs = tree.drain_events()
        assert [[int(e.kind), int(e.node_index)] for e in evs] == g["events"], step
        dev.apply_events(evs)
        assert node_sha(dev) == g["after_apply"], step
        idx, fl = tree.node_indices(with_flags=True)
        from paper_1407_2074_b200 import _lib
        bricked = sorted(int(i) for i, f in zip(idx, fl) if f & _lib.NODE_BRICK)
        req = r2.events_requests(step, bricked)
        assert req == g["requests"], step
        fb = dev.flag_buffer
        for i in req:
            fb[i] |= FLAG_REQUESTED
        plan = dev.process_flags(RenderMode.FULLFRAME)
        assert plan_list(plan) == g["plan"], step
        assert dev.upload_bricks(plan, budget_ms=1e9) == g["uploaded"]
        assert node_sha(dev) == g["node_sha"], step
        assert sorted([k, v] for k, v in dev._node_slot.items()) == g["resident"], step
        assert dev.pending_requests == g["pending"]
        assert dev.evictions == g["evictions"]
        dev.check_consistency()
    assert (tree.node_count, tree.brick_count) == (gold["node_count"], gold["brick_count"])
    assert node_sha(DeviceState(tree, slot_count=4)) == gold["rebuilt_sha"]


# -- the reference's DeviceState tests (tests/test_device.py), restated ---------

def _make_tree(threshold=0):
    return make_tree(dict(dims=(16, 16, 16), brick=(4, 4, 4), threshold=threshold,
                          fmt="uint8", page_bricks=8, ram_page_limit=8))


def _full_tree():
    tree = _make_tree(0)
    vol = np.random.default_rng(2).integers(0, 255, (16, 16, 16), dtype=np.uint8)
    tree.insert_block(0, (0, 0, 0), vol)
    return tree


def test_empty_event_list_leaves_buffer_unchanged():
    from paper_1407_2074_b200 import DeviceState
    dev = DeviceState(_make_tree(), slot_count=4)
    before = dev.node_buffer_host().copy()
    dev.apply_events([])
    assert np.array_equal(dev.node_buffer_host(), before)


def test_incremental_events_match_from_scratch_rebuild():
    from paper_1407_2074_b200 import DeviceState
    rng = np.random.default_rng(0)
    tree = _make_tree(threshold=12)
    dev = DeviceState(tree, slot_count=4)
    for _ in range(10):
        origin = rng.integers(0, 12, size=3)
        size = rng.integers(1, 5, size=3)
        block = rng.integers(0, 255, size=tuple(reversed(size)), dtype=np.uint8)
        tree.insert_block(0, tuple(int(v) for v in origin), block)
        dev.apply_events(tree.drain_events())
    rebuilt = DeviceState(tree, slot_count=4)
    assert np.array_equal(dev.node_buffer_host(), rebuilt.node_buffer_host())
    dev.check_consistency()


def test_update_event_drops_resident_brick():
    from paper_1407_2074_b200.device import FLAG_REQUESTED, DeviceState, RenderMode
    from paper_1407_2074_b200.device import unpack_node
    tree = _make_tree()
    vol = np.random.default_rng(1).integers(0, 255, (16, 16, 16), dtype=np.uint8)
    tree.insert_block(0, (0, 0, 0), vol)
    dev = DeviceState(tree, slot_count=4)
    dev.apply_events(tree.drain_events())
    leaf = tree.find_node((0.5, 0.5, 0.5), 0)
    dev.flag_buffer[leaf.index] |= FLAG_REQUESTED
    plan = dev.process_flags(RenderMode.FULLFRAME)
    assert dev.upload_bricks(plan, budget_ms=1000) == 1
    assert unpack_node(int(dev.node_buffer_host()[leaf.index]), 1).in_buffer
    tree.insert_block(0, (0, 0, 0), vol[:4, :4, :4])
    dev.apply_events(tree.drain_events())
    assert not unpack_node(int(dev.node_buffer_host()[leaf.index]), 1).in_buffer
    assert dev.resident_bricks == 0
    dev.check_consistency()


def test_no_requests_empty_plan_flags_cleared():
    from paper_1407_2074_b200.device import FLAG_USED, DeviceState, RenderMode
    dev = DeviceState(_full_tree(), slot_count=4)
    dev.flag_buffer[5] |= FLAG_USED
    assert dev.process_flags(RenderMode.FULLFRAME) == []
    assert not dev.read_flags().any()


def test_fullframe_coarse_request_evicts_used_fine_brick():
    from paper_1407_2074_b200.device import FLAG_REQUESTED, FLAG_USED, DeviceState, RenderMode
    dev = DeviceState(_full_tree(), slot_count=3)
    for idx in (9, 10, 11):
        dev.flag_buffer[idx] |= FLAG_REQUESTED
    dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), budget_ms=1000)
    assert dev.resident_bricks == 3
    for idx in (9, 10, 11):
        dev.flag_buffer[idx] |= FLAG_USED
    assert dev.process_flags(RenderMode.FULLFRAME) == []
    fb = dev.flag_buffer
    fb[9] |= FLAG_USED
    fb[12] |= FLAG_REQUESTED
    fb[13] |= FLAG_REQUESTED
    fb[1] |= FLAG_REQUESTED
    plan = dev.process_flags(RenderMode.FULLFRAME)
    assert [i.node_index for i in plan] == [1, 12, 13]
    assert plan[0].evicts == 9
    assert {plan[1].evicts, plan[2].evicts} == {10, 11}


def test_fullframe_defers_when_residents_are_coarser():
    from paper_1407_2074_b200.device import FLAG_REQUESTED, FLAG_USED, DeviceState, RenderMode
    dev = DeviceState(_full_tree(), slot_count=2)
    for idx in (1, 2):
        dev.flag_buffer[idx] |= FLAG_REQUESTED
    dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), budget_ms=1000)
    assert dev.resident_bricks == 2
    fb = dev.flag_buffer
    fb[1] |= FLAG_USED
    fb[2] |= FLAG_USED
    fb[9] |= FLAG_REQUESTED
    fb[10] |= FLAG_REQUESTED
    assert dev.process_flags(RenderMode.FULLFRAME) == []
    assert dev.pending_requests == 2
    assert dev.resident_bricks == 2


def test_refinement_replaces_all_slots():
    from paper_1407_2074_b200.device import FLAG_REQUESTED, FLAG_USED, DeviceState, RenderMode
    dev = DeviceState(_full_tree(), slot_count=2)
    for idx in (1, 2):
        dev.flag_buffer[idx] |= FLAG_REQUESTED
    dev.upload_bricks(dev.process_flags(RenderMode.REFINEMENT), budget_ms=1000)
    fb = dev.flag_buffer
    fb[1] |= FLAG_USED
    fb[2] |= FLAG_USED
    fb[9] |= FLAG_REQUESTED
    fb[10] |= FLAG_REQUESTED
    plan = dev.process_flags(RenderMode.REFINEMENT)
    assert len(plan) == 2
    dev.upload_bricks(plan, budget_ms=1000)
    assert set(dev._node_slot) == {9, 10}
    dev.check_consistency()


def test_deferred_requests_rise_with_age():
    from paper_1407_2074_b200.device import FLAG_REQUESTED, DeviceState, RenderMode
    dev = DeviceState(_full_tree(), slot_count=1)
    dev.flag_buffer[9] |= FLAG_REQUESTED
    plan = dev.process_flags(RenderMode.FULLFRAME)
    assert [i.node_index for i in plan] == [9]
    dev.upload_bricks(plan, budget_ms=0)
    fb = dev.flag_buffer
    fb[9] |= FLAG_REQUESTED
    fb[10] |= FLAG_REQUESTED
    plan = dev.process_flags(RenderMode.FULLFRAME)
    assert [i.node_index for i in plan][0] == 9


class _FakeClock:
    def __init__(self):
        self.t = 0.0

    def __call__(self):
        return self.t


def _upload_with_cost(budget_ms, item_cost_s=0.040, items=5, slots=None):
    """tests/test_device.py:256-275: the store's acquire is monkeypatched to
    advance a fake clock, exactly as the reference's test does."""
    from paper_1407_2074_b200.device import FLAG_REQUESTED, DeviceState, RenderMode
    tree = _full_tree()
    dev = DeviceState(tree, slot_count=slots or items)
    clock = _FakeClock()
    original = tree.store.acquire

    def slow_acquire(loc, blocking=True):
        clock.t += item_cost_s
        return original(loc, blocking)

    tree.store.acquire = slow_acquire
    for idx in range(9, 9 + items):
        dev.flag_buffer[idx] |= FLAG_REQUESTED
    plan = dev.process_flags(RenderMode.FULLFRAME)
    assert len(plan) == items
    done = dev.upload_bricks(plan, budget_ms=budget_ms, clock=clock)
    tree.store.acquire = original
    return done, clock.t


def test_zero_budget_defers_everything():
    done, _ = _upload_with_cost(0)
    assert done == 0


def test_budget_150ms_runs_three_to_four_items():
    done, elapsed = _upload_with_cost(150)
    assert 3 <= done <= 4
    assert elapsed * 1000 <= 150 + 40


@pytest.mark.parametrize("budget", [50, 150, 200])
def test_budget_overshoot_bounded_by_one_item(budget):
    done, elapsed = _upload_with_cost(budget)
    assert elapsed * 1000 <= budget + 40
    assert done >= 1


@pytest.mark.parametrize("budget_ms", [50, 150, 200])
def test_upload_budget_bounded_acceptance(budget_ms):
    """tests/test_acceptance.py:353-384 (10 requests, 16 slots)."""
    _, elapsed = _upload_with_cost(budget_ms, items=10, slots=16)
    assert elapsed * 1000 <= budget_ms + 40


def test_unavailable_brick_is_skipped_and_stays_requested():
    """BrickStore.acquire returning None (all pages pinned) skips the item
    (device.py:336-339)."""
    from paper_1407_2074_b200.device import FLAG_REQUESTED, DeviceState, RenderMode
    tree = _full_tree()
    dev = DeviceState(tree, slot_count=4)
    original = tree.store.acquire
    tree.store.acquire = lambda loc, blocking=True: None if loc.node_index == 10 else \
        original(loc, blocking)
    for idx in (9, 10, 11):
        dev.flag_buffer[idx] |= FLAG_REQUESTED
    done = dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), budget_ms=1e9)
    tree.store.acquire = original
    assert done == 2 and dev.unavailable_skips == 1
    assert set(dev._node_slot) == {9, 11} and dev.pending_requests == 1
    dev.check_consistency()


def test_uploaded_entry_valid_before_next_pass():
    from paper_1407_2074_b200.device import FLAG_REQUESTED, DeviceState, RenderMode
    from paper_1407_2074_b200.device import unpack_node
    tree = _full_tree()
    dev = DeviceState(tree, slot_count=2)
    dev.flag_buffer[9] |= FLAG_REQUESTED
    dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), budget_ms=1000)
    entry = unpack_node(int(dev.node_buffer_host()[9]), 1)
    assert entry.in_buffer
    assert dev.slot_owner[entry.slot] == 9
    node = tree.node_by_index(9)
    assert np.array_equal(dev.brick_buffer[entry.slot].cpu().numpy(),
                          tree.store.read_brick(node.brick))


# -- resident_all refresh consumes events in the library (vt_mirror_apply_queued) --

def test_resident_all_refresh_equals_drain_and_apply():
    """DeviceState.refresh() on a zero-copy mirror == apply_events(
    drain_events()): same node buffer, deleted nodes' feedback flags
    cleared, and the queue is empty afterwards (device.py:205-237)."""
    from paper_1407_2074_b200.device import FLAG_REQUESTED, FLAG_USED, DeviceState
    trees = []
    for _ in range(2):
        t = make_tree(r2.events_tree())
        trees.append((t, DeviceState(t, resident_all=True)))
    for step, (origin, block) in enumerate(r2.events_ops()):
        for t, dev in trees:
            fb = dev.flag_buffer
            fb[:] = FLAG_USED | FLAG_REQUESTED  # every node flagged
            t.insert_block(0, origin, block)
        (ta, da), (tb, db) = trees
        evs = tb.drain_events()
        db.apply_events(evs)
        n = da.refresh()
        assert n == len(evs), step
        assert len(ta.drain_events()) == 0
        assert node_sha(da) == node_sha(db), step
        fa, fbb = da.read_flags(), db.read_flags()
        assert np.array_equal(fa, fbb), step
        deleted = [int(e.node_index) for e in evs if int(e.kind) == 2]
        assert all(fa[i] == 0 for i in deleted), step
