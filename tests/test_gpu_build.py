"""GPU parity of the octree build (libvtx via the drop-in Octree API):
byte-identical VXOC/VXBP digests, identical change events, node counts,
prune counts and Fig. 4 node buffers versus golden vectors from the
unmodified reference (tests/golden/, made by make_golden.py) and versus the
CPU oracle on larger seeded cases.  Bit-exact is the bar (integer work)."""

import hashlib
import json
import os

import numpy as np
import pytest

import scenarios
from gpu_helpers import build_scenario, digest, make_tree

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "golden.json")) as fh:
    GOLDEN = json.load(fh)


@pytest.mark.parametrize("name", list(scenarios.SCENARIOS))
def test_build_bit_exact_vs_reference(name, tmp_path):
    gold = GOLDEN["builds"][name]
    sc, tree, events = build_scenario(name)
    assert events == gold["events"]
    assert tree.node_count == gold["node_count"]
    assert tree.pruned_bricks == gold["pruned_bricks"]
    assert tree.brick_count == gold["brick_count"]
    assert [int(i) for i in tree.node_indices()] == gold["nodes"]
    assert digest(tree, tmp_path, "a") == gold["digest_unfinished"]
    from paper_1407_2074_b200 import DeviceState
    dev = DeviceState(tree, slot_count=1)
    nb = dev.node_buffer_host()
    assert hashlib.sha256(nb.astype("<u8").tobytes()).hexdigest() == gold["node_buffer_sha256"]
    dev.close()
    tree.finalize()
    tree.fill_borders()
    ev = tree.drain_events()
    assert [[int(e.kind), e.node_index] for e in ev] == gold["border_events"]
    assert digest(tree, tmp_path, "b") == gold["digest_final"]


def test_fig3_golden_walk():  # test_octree.py:128-213
    from paper_1407_2074_b200 import Octree
    sc = scenarios.scenario("fig3")
    tree = make_tree(sc["tree"])
    c, o, v = sc["ops"][0]
    ev = tree.insert_block(c, o, v)
    assert [e.node_index for e in ev if e.kind == 1] == [1, 2, 9, 10]
    x = lambda n: tree.read_brick(n)[1, 1, 1:5, 0].tolist()  # noqa: E731
    assert x(9) == [1, 5, 2, 0] and x(1) == [3, 1, 0, 0] and x(0) == [2, 0, 0, 0]
    for c, o, v in sc["ops"][1:3]:
        tree.insert_block(c, o, v)
    assert tree.pruned_bricks == 2
    leaf, parent = tree.node_by_index(10), tree.node_by_index(1)
    assert leaf.brick is None and leaf.avg == [3] and parent.brick is None and parent.avg == [3]
    assert tree.node_by_index(9).smin == [1] and tree.node_by_index(9).smax == [5]
    tree.insert_block(*sc["ops"][3])
    assert x(0) == [3, 3, 3, 3] and x(17) == [2, 2, 4, 4] and x(18) == [2, 4, 3, 3]
    assert tree.node_count == 7


def test_halfsample_block_device_vs_oracle():
    import voxtree_oracle as vo
    from paper_1407_2074_b200.octree import halfsample_block
    rng = np.random.default_rng(0)
    for _ in range(60):
        mz, my, mx = (int(rng.choice([2, 4, 6])), int(rng.choice([1, 2, 4])),
                      int(rng.choice([2, 4, 8])))
        C = int(rng.integers(1, 4))
        split = (mx > 1, my > 1, mz > 1)
        v = rng.integers(0, 65535, size=(mz, my, mx, C)).astype(np.int64)
        ext = (int(rng.integers(0, mx + 1)), int(rng.integers(0, my + 1)),
               int(rng.integers(0, mz + 1)))
        assert np.array_equal(halfsample_block(v, ext, split, 11),
                              vo.halfsample(v, ext, split, 11))
    # known answers (test_octree.py:66-84)
    v = np.array([2, 4, 100, 100]).reshape(1, 1, 4, 1)
    assert halfsample_block(v, (3, 1, 1), (True, False, False), 7)[0, 0, :, 0].tolist() == [3, 100]
    assert halfsample_block(v, (2, 1, 1), (True, False, False), 7)[0, 0, :, 0].tolist() == [3, 7]


def _oracle_from_ops(spec, ops):
    import voxtree_oracle as vo
    t = vo.OracleTree(**spec)
    for c, o, v in ops:
        t.insert(c, o, v)
    return t


@pytest.mark.parametrize("seed", range(4))
def test_random_partitions_tau0_equal_bulk(seed, tmp_path):
    """acceptance criterion 3 (test_acceptance.py:130-158) at 64^3 x 3 u16."""
    rng = np.random.default_rng(100 + seed)
    vol = rng.integers(0, 65535, size=(64, 64, 64, 3), dtype=np.uint16)
    spec = dict(dims=(64, 64, 64), brick=(16, 16, 16), threshold=0, fmt="uint16", channels=3)
    bulk = make_tree(spec)
    bulk.insert_channels((0, 0, 0), vol)
    ref = digest(bulk, tmp_path, "bulk")
    part = make_tree(spec)
    for c in range(3):
        for (x0, y0, z0), (x1, y1, z1) in scenarios._partition(rng, (64, 64, 64), cuts=3):
            part.insert_block(c, (x0, y0, z0), vol[z0:z1, y0:y1, x0:x1, c])
    assert digest(part, tmp_path, "part") == ref
    import voxtree_oracle as vo
    ot = _oracle_from_ops(spec, [(c, (0, 0, 0), vol[..., c]) for c in range(3)])
    assert list(vo.digest(ot)) == ref


@pytest.mark.parametrize("seed", range(3))
def test_random_sequences_tau_positive_vs_oracle(seed, tmp_path):
    """tau > 0: history-dependent semantics replayed insertion by insertion."""
    import voxtree_oracle as vo
    rng = np.random.default_rng(7 + seed)
    spec = dict(dims=(40, 33, 24), brick=(8, 8, 8), threshold=float(rng.integers(5, 60)),
                fmt="uint8", channels=2, bg=int(rng.integers(0, 20)))
    ops = []
    for _ in range(30):
        o = tuple(int(rng.integers(0, d)) for d in spec["dims"])
        s = tuple(int(rng.integers(1, d - oo + 1)) for d, oo in zip(spec["dims"], o))
        s = tuple(min(v, 12) for v in s)
        base = int(rng.integers(0, 200))
        span = int(rng.choice([1, 3, 30, 120]))
        vals = (base + rng.integers(0, span, size=s[::-1])).clip(0, 255).astype(np.uint8)
        ops.append((int(rng.integers(0, 2)), o, vals))
    gpu = make_tree(spec)
    for c, o, v in ops:
        gpu.insert_block(c, o, v)
    ot = _oracle_from_ops(spec, ops)
    assert gpu.node_count == ot.node_count and gpu.pruned_bricks == ot.pruned_bricks
    assert digest(gpu, tmp_path, "g") == list(vo.digest(ot))
    gpu.finalize()
    gpu.fill_borders()
    ot.finished = True
    ot.fill_borders()
    assert digest(gpu, tmp_path, "g2") == list(vo.digest(ot))


def test_slice_stream_spim_tau_vs_oracle(tmp_path):
    """SPIM-shaped stream, slice by slice and channel-interleaved (VSTR order)
    at tau = 5%: the order-dependent case must replay exactly."""
    import voxtree_oracle as vo
    vol = vo.synth_spim((64, 64, 48), 3, 65535, seed=0)
    spec = dict(dims=(64, 64, 48), brick=(16, 16, 16), threshold=None, fmt="uint16", channels=3)
    ops = [(c, (0, 0, z), vol[z:z + 1, :, :, c]) for z in range(48) for c in range(3)]
    gpu = make_tree(spec)
    for c, o, v in ops:
        gpu.insert_block(c, o, v)
    ot = _oracle_from_ops(spec, ops)
    assert gpu.pruned_bricks == ot.pruned_bricks
    assert digest(gpu, tmp_path, "s") == list(vo.digest(ot))


def test_insert_channels_matches_successive_inserts(tmp_path):
    import voxtree_oracle as vo
    vol = vo.synth_spim((48, 40, 36), 3, 255, seed=7)
    for thr in (0, None):
        spec = dict(dims=(48, 40, 36), brick=(8, 8, 8), threshold=thr, fmt="uint8", channels=3)
        a = make_tree(spec)
        ev_a = []
        for z in range(0, 36, 8):
            ev_a += a.insert_channels((0, 0, z), vol[z:z + 8])
        b = make_tree(spec)
        ev_b = []
        for z in range(0, 36, 8):
            for c in range(3):
                ev_b += b.insert_block(c, (0, 0, z), vol[z:z + 8, :, :, c])
        assert ev_a == ev_b
        assert digest(a, tmp_path, "a") == digest(b, tmp_path, "b")


def test_device_input_matches_host_input(tmp_path):
    import torch
    import voxtree_oracle as vo
    vol = vo.synth_uniform((32, 32, 32), 2, 65535, seed=3)
    spec = dict(dims=(32, 32, 32), brick=(8, 8, 8), threshold=0, fmt="uint16", channels=2)
    a = make_tree(spec)
    a.insert_channels((0, 0, 0), vol)
    b = make_tree(spec)
    b.insert_channels((0, 0, 0), torch.from_numpy(vol.astype(np.int32)).cuda().to(torch.uint16))
    assert digest(a, tmp_path, "h") == digest(b, tmp_path, "d")


def test_synth_kernel_matches_oracle():
    import ctypes as ct
    import torch
    import voxtree_oracle as vo
    from paper_1407_2074_b200 import _lib
    dims = (70, 33, 20)
    for kind, fn in ((0, vo.synth_uniform), (1, vo.synth_spim)):
        for sb, fmax in ((1, 255), (2, 65535)):
            want = fn(dims, 3, fmax, seed=5, z0=4, z1=17)
            t = torch.empty(want.size, dtype=torch.uint8 if sb == 1 else torch.uint16,
                            device="cuda")
            _lib.call("vt_synth", ct.c_void_p(t.data_ptr()), kind, _lib.i32x3(dims), 3, sb, 5,
                      4, 17, None)
            torch.cuda.synchronize()
            got = t.cpu().numpy().reshape(want.shape)
            assert np.array_equal(got, want), (kind, sb)


def test_save_load_roundtrip(tmp_path):
    from paper_1407_2074_b200 import load_octree, save_octree
    sc, tree, _ = build_scenario("ragged_2ch", borders=True)
    a = digest(tree, tmp_path, "a")
    loaded = load_octree(os.path.join(tmp_path, "a.vxoc"), os.path.join(tmp_path, "a.vxbp"))
    assert digest(loaded, tmp_path, "c") == a
    assert loaded.node_count == tree.node_count and loaded.brick_count == tree.brick_count


def test_errors_mirror_reference():
    sc = scenarios.scenario("fig3")
    tree = make_tree(sc["tree"])
    with pytest.raises(ValueError):
        tree.insert_block(1, (0, 0, 0), np.zeros((1, 1, 1), np.uint8))
    with pytest.raises(ValueError):
        tree.insert_block(0, (14, 0, 0), np.zeros((1, 1, 4), np.uint8))
    with pytest.raises(ValueError):
        tree.insert_block(0, (0, 0, 0), np.zeros((1, 4), np.uint8))
