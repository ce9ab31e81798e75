"""Pin the CPU oracle (oracle/voxtree_oracle.py) to the unmodified
reference: golden vectors in tests/golden/ were produced by
tests/golden/make_golden.py running /root/reference, plus the reference's own
known-answer tests (pkg/tests/test_octree.py, test_device.py, test_render.py)."""

import hashlib
import json
import os

import numpy as np
import pytest

import scenarios
import voxtree_oracle as vo

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "golden.json")) as fh:
    GOLDEN = json.load(fh)
RENDERS = np.load(os.path.join(GOLD, "renders.npz"))


def oracle_tree(name):
    sc = scenarios.scenario(name)
    t = vo.OracleTree(**sc["tree"])
    events = [[list(e) for e in t.insert(c, o, v)] for c, o, v in sc["ops"]]
    return sc, t, events


# -- known answers from the reference's own tests --------------------------------

def test_halfsample_known_answers():  # test_octree.py:66-84
    v = np.array([2, 4, 6, 8]).reshape(1, 1, 4, 1)
    assert vo.halfsample(v, (4, 1, 1), (True, False, False), 0)[0, 0, :, 0].tolist() == [3, 7]
    v = np.array([0, 0, 0, 0, 8, 8, 8, 8]).reshape(2, 2, 2, 1)
    assert vo.halfsample(v, (2, 2, 2), (True,) * 3, 0)[0, 0, 0, 0] == 4
    v = np.array([2, 4, 100, 100]).reshape(1, 1, 4, 1)
    assert vo.halfsample(v, (3, 1, 1), (True, False, False), 7)[0, 0, :, 0].tolist() == [3, 100]
    assert vo.halfsample(v, (2, 1, 1), (True, False, False), 7)[0, 0, :, 0].tolist() == [3, 7]


def test_homogeneity_strict():  # test_octree.py:104-110
    assert vo.homogeneous([3], [3], 1) and not vo.homogeneous([1], [5], 1)
    assert not vo.homogeneous([7], [7], 0)


def test_geometry_known_answers():  # test_octree.py:123-128, test_device.py:70-72
    g = vo.Geo((1004, 1002, 1611), (64, 64, 64))
    assert g.depth == 5 and g.virtual == (2048, 2048, 2048)
    assert (8 ** 8 - 1) // 7 * 8 == 19_173_960
    g = vo.Geo((20, 16, 16), (8, 16, 16))
    assert g.virtual == (32, 16, 16)
    assert [g.level_of(i) for i in (0, 1, 8, 9, 72)] == [2, 1, 1, 0, 0]


def test_fig3_structure():  # test_acceptance.py:50-85
    _, t, _ = oracle_tree("fig3")
    assert t.nodes() == [0, 1, 2, 9, 10, 17, 18]
    assert sorted(t.bricks) == [0, 2, 9, 17, 18]
    assert t.bricks[17][1, 1, 1:5, 0].tolist() == [2, 2, 4, 4]


def test_quantization_bound():  # test_acceptance.py:231-239
    worst = max(abs(round(vo.quantize(v, 3, 65535) * 65535 / 8191) - v) for v in range(0, 65536, 7))
    assert worst <= 4


# -- golden vectors from the unmodified reference --------------------------------

@pytest.mark.parametrize("name", list(scenarios.SCENARIOS))
def test_build_matches_reference(name):
    gold = GOLDEN["builds"][name]
    sc, t, events = oracle_tree(name)
    assert events == gold["events"]
    assert t.node_count == gold["node_count"]
    assert t.pruned_bricks == gold["pruned_bricks"]
    assert t.nodes() == gold["nodes"]
    assert sorted(t.bricks) == gold["bricks"]
    assert list(vo.digest(t)) == gold["digest_unfinished"]
    nb = vo.node_buffer(t)
    assert hashlib.sha256(nb.astype("<u8").tobytes()).hexdigest() == gold["node_buffer_sha256"]
    if sc["borders"]:
        t.finished = True
        n0 = len(t.events)
        t.fill_borders()
        assert [list(e) for e in t.events[n0:]] == gold["border_events"]
        assert list(vo.digest(t)) == gold["digest_final"]


def _built(name):
    sc, t, _ = oracle_tree(name)
    t.finished = True
    t.fill_borders()
    return t


@pytest.mark.parametrize("name", list(scenarios.RENDER_CASES))
def test_render_matches_reference(name):
    rc = scenarios.render_case(name)
    gold = GOLDEN["renders"][name]
    t = _built(rc["build"])
    spec = vo.SceneSpec(**rc["scene"])
    if rc["resident"] == "all":
        nb, bb, _ = vo.resident_buffers(t)
    else:
        nb, bb = vo.node_buffer(t), np.zeros((1,) + t._stored_shape(), t.dtype)
    r = vo.OracleRenderer(t, nb, bb)
    st = r.start(spec, rc["tile"])
    _, cnt = r.run(st, spec, fullframe=rc["strategy"] == "fullframe")
    img = r.image(st, spec, cnt if rc["strategy"] == "fullframe" else None)
    ref = RENDERS[name + "/image"]
    assert np.max(np.abs(img - ref)) <= 1e-12
    assert cnt == gold["counters"]
    if rc["strategy"] == "fullframe":
        assert np.array_equal(r.flags, RENDERS[name + "/flags"])
    if rc["resident"] == "none":
        # second pass with the reference's upload plan resident
        _, _, slots_all = vo.resident_buffers(t)
        res = {i: slots_all[i] for i, _slot in gold["plan"]}
        nb2 = vo.node_buffer(t, res)
        _, bb2, _ = vo.resident_buffers(t)
        r2 = vo.OracleRenderer(t, nb2, bb2)
        img2, cnt2 = r2.render_fullframe(spec)
        assert np.max(np.abs(img2 - RENDERS[name + "/image2"])) <= 1e-12
        assert cnt2 == gold["counters2"]
        assert np.array_equal(r2.flags, RENDERS[name + "/flags2"])


def test_synthetic_generators_deterministic():
    a = vo.synth_spim((40, 24, 20), 3, 65535, seed=3)
    b = np.concatenate([vo.synth_spim((40, 24, 20), 3, 65535, seed=3, z0=z, z1=z + 5)
                        for z in range(0, 20, 5)])
    assert np.array_equal(a, b)
    u = vo.synth_uniform((16, 8, 4), 2, 255, seed=1)
    assert u.dtype == np.uint8 and u.max() <= 255
