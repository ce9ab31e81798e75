"""Generate golden vectors by running the UNMODIFIED reference (voxtree, pure
Python) on the shared scenarios.  Runs only in the build container, where
/root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.json (digests, events, counts, counters) and
tests/golden/renders.npz (images + feedback flags).  Nothing on the GPU box
reads /root/reference; tests consume only these committed files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import scenarios  # noqa: E402
from voxtree.device import DeviceState, RenderMode  # noqa: E402
from voxtree.octree import Octree  # noqa: E402
from voxtree.render import (Camera, ClipPlane, ClipSet, OutOfCoreRenderer,  # noqa: E402
                            RenderSettings, Scene, TransferFunction)
from voxtree.serialize import save_octree  # noqa: E402
from voxtree.volume import BrickPoolConfig, VolumeDescriptor  # noqa: E402


def ref_tree(tmp, spec, tag):
    desc = VolumeDescriptor(dims=spec["dims"], channels=spec.get("channels", 1),
                            sample_format=spec.get("fmt", "uint8"),
                            spacing=spec.get("spacing", (1.0, 1.0, 1.0)),
                            background_value=spec.get("bg", 0))
    cfg = BrickPoolConfig(brick_dims=spec["brick"], homogeneity_threshold=spec["threshold"])
    return Octree.create(desc, cfg, os.path.join(tmp, f"{tag}.pool"))


def digest(tree, tmp, tag):
    o, p = os.path.join(tmp, f"{tag}.vxoc"), os.path.join(tmp, f"{tag}.vxbp")
    save_octree(tree, o, p)
    with open(o, "rb") as fo, open(p, "rb") as fp:
        return [hashlib.sha256(fo.read()).hexdigest(), hashlib.sha256(fp.read()).hexdigest()]


def build(tmp, name):
    sc = scenarios.scenario(name)
    tree = ref_tree(tmp, sc["tree"], name)
    events = []
    for c, origin, values in sc["ops"]:
        evs = tree.insert_block(c, origin, values)
        events.append([[int(e.kind), int(e.node_index)] for e in evs])
    tree.drain_events()
    out = dict(events=events, digest_unfinished=digest(tree, tmp, name + "_a"),
               node_count=tree.node_count, pruned_bricks=tree.pruned_bricks,
               brick_count=tree.brick_count,
               nodes=sorted(n.index for n in tree.iter_nodes()),
               bricks=sorted(n.index for n in tree.iter_nodes() if n.brick is not None))
    if sc["borders"]:
        tree.finalize()
        tree.fill_borders()
        out["border_events"] = [[int(e.kind), int(e.node_index)] for e in tree.drain_events()]
        out["digest_final"] = digest(tree, tmp, name + "_b")
    dev = DeviceState(tree, slot_count=1)
    out["node_buffer_sha256"] = hashlib.sha256(dev.node_buffer.astype("<u8").tobytes()).hexdigest()
    return tree, out


def to_scene(spec, strategy):
    cam = Camera(position=spec["position"], look_at=spec["look_at"], up=spec["up"],
                 fov_y=spec["fov_y"], width=spec["width"], height=spec["height"])
    st = RenderSettings(mode=spec["mode"], strategy=strategy,
                        sampling_step=spec["sampling_step"],
                        early_termination_alpha=spec["early_termination_alpha"],
                        lod_bias=spec["lod_bias"])
    tfs = [TransferFunction(p) for p in spec["tfs"]]
    clips = ClipSet(tuple(ClipPlane(tuple(n), o) for n, o in spec["clips"]))
    return Scene(camera=cam, settings=st, transfer_functions=tfs, clips=clips)


def counters_dict(c):
    return {f: int(getattr(c, f)) for f in c.__dataclass_fields__}


def render(tmp, name, trees, arrays):
    rc = scenarios.render_case(name)
    tree = trees[rc["build"]]
    scene = to_scene(rc["scene"], rc["strategy"])
    dev = DeviceState(tree, slot_count=tree.brick_count + 8)
    r = OutOfCoreRenderer(dev)
    out = {}
    if rc["resident"] == "all":
        for n in tree.iter_nodes():
            if n.brick is not None:
                dev.flag_buffer[n.index] |= 2
        dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), 1e9)
    if rc["strategy"] == "fullframe":
        img, cnt = r.render_fullframe(scene)
        arrays[name + "/image"] = img
        arrays[name + "/flags"] = dev.flag_buffer.copy()
        out["counters"] = counters_dict(cnt)
        if rc["resident"] == "none":
            plan = dev.process_flags(RenderMode.FULLFRAME)
            out["plan"] = [[i.node_index, i.slot] for i in plan]
            dev.upload_bricks(plan, 1e9)
            img2, cnt2 = r.render_fullframe(scene)
            arrays[name + "/image2"] = img2
            arrays[name + "/flags2"] = dev.flag_buffer.copy()
            out["counters2"] = counters_dict(cnt2)
    else:
        sess = r.start_refinement(scene, tile=rc["tile"])
        passes = 0
        while not sess.run_pass():
            dev.upload_bricks(dev.process_flags(RenderMode.REFINEMENT), 1e9)
            passes += 1
        arrays[name + "/image"] = sess.image()
        out["counters"] = counters_dict(sess.counters)
        out["passes"] = sess.passes
    return out


def main():
    golden = {"builds": {}, "renders": {}}
    arrays = {}
    trees = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name in scenarios.SCENARIOS:
            tree, out = build(tmp, name)
            trees[name] = tree
            golden["builds"][name] = out
            print("build", name, out["node_count"], out["brick_count"], out["pruned_bricks"])
        for name in scenarios.RENDER_CASES:
            golden["renders"][name] = render(tmp, name, trees, arrays)
            print("render", name, golden["renders"][name]["counters"])
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(golden, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "renders.npz"), **arrays)


if __name__ == "__main__":
    main()
