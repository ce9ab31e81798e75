"""CPU: the oracle's channel-transform sampler branch (render/raycast.py:
258-276) and its builds pinned to the round-2 reference goldens
(tests/golden/make_golden_r2.py).  Oracle = test infrastructure only."""

import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))

import r2_scenarios as r2  # noqa: E402
import voxtree_oracle as vo  # noqa: E402

GOLD = os.path.join(HERE, "golden")
with open(os.path.join(GOLD, "golden_r2.json")) as fh:
    GOLDEN = json.load(fh)
RENDERS = np.load(os.path.join(GOLD, "renders_r2.npz"))


def _tree(name):
    b = r2.xf_trees()[name]
    t = vo.OracleTree(**b["tree"])
    for c, o, v in b["ops"]:
        t.insert(c, o, np.ascontiguousarray(v))
    t.finished = True
    t.fill_borders()
    return t


@pytest.mark.parametrize("name", list(r2.xf_trees()))
def test_oracle_transform_tree_digest(name):
    t = _tree(name)
    g = GOLDEN["builds"][name]
    assert t.node_count == g["node_count"]
    assert list(vo.digest(t)) == g["digest"]


@pytest.mark.parametrize("name", [k for k, v in r2.xf_cases().items()
                                  if v["resident"] == "all"])
def test_oracle_transform_render(name):
    rc = r2.xf_cases()[name]
    t = _tree(rc["build"])
    nb, bb, _ = vo.resident_buffers(t)
    r = vo.OracleRenderer(t, nb, bb)
    img, cnt = r.render_fullframe(vo.SceneSpec(**rc["scene"]))
    assert np.max(np.abs(img - RENDERS[name + "/image"])) <= 1e-12
    assert cnt == GOLDEN["renders"][name]["counters"]
    assert np.array_equal(r.flags, RENDERS[name + "/flags"])


def test_golden_r2_residency_invariants():
    """The reference's own acceptance claims hold in the recorded goldens:
    zero AVG fallbacks after warm-up at 1/64 of the payload, and the
    incremental node buffer equals a from-scratch rebuild."""
    fb = [f["counters"]["avg_fallbacks"] for f in GOLDEN["ff64"]["frames"]]
    assert fb[0] > 0 and all(f == 0 for f in fb[2:])
    ev = GOLDEN["events"]
    kinds = {k for s in ev["steps"] for k, _ in s["events"]}
    assert kinds == {1, 2, 3}, kinds  # created, deleted and updated all exercised
