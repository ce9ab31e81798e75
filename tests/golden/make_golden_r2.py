"""Round-2 golden vectors, made by running the UNMODIFIED reference (voxtree,
pure Python) in the build container:

    python tests/golden/make_golden_r2.py

Scenarios: tests/r2_scenarios.py.  Writes tests/golden/golden_r2.json and
tests/golden/renders_r2.npz.  Nothing on the GPU box reads /root/reference;
tests/test_gpu_r2.py consumes only these committed files.  ~1 min here.
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

import r2_scenarios as r2  # noqa: E402
from voxtree.device import FLAG_REQUESTED, DeviceState, RenderMode  # noqa: E402
from voxtree.octree import Octree  # noqa: E402
from voxtree.render import (Camera, ClipPlane, ClipSet, OutOfCoreRenderer,  # noqa: E402
                            RenderSettings, Scene, TransferFunction)
from voxtree.serialize import save_octree  # noqa: E402
from voxtree.volume import BrickPoolConfig, VolumeDescriptor  # noqa: E402


def ref_tree(tmp, spec, tag):
    desc = VolumeDescriptor(dims=spec["dims"], channels=spec.get("channels", 1),
                            sample_format=spec["fmt"], spacing=spec.get("spacing", (1, 1, 1)),
                            background_value=spec.get("bg", 0),
                            channel_transforms=spec.get("transforms"))
    cfg = BrickPoolConfig(brick_dims=spec["brick"], homogeneity_threshold=spec["threshold"],
                          page_bricks=spec.get("page_bricks", 64),
                          ram_page_limit=spec.get("ram_page_limit", 64))
    return Octree.create(desc, cfg, os.path.join(tmp, f"{tag}.pool"))


def digest(tree, tmp, tag):
    o, p = os.path.join(tmp, f"{tag}.vxoc"), os.path.join(tmp, f"{tag}.vxbp")
    save_octree(tree, o, p)
    out = []
    for f in (o, p):
        with open(f, "rb") as fh:
            out.append(hashlib.sha256(fh.read()).hexdigest())
        os.unlink(f)
    return out


def to_scene(spec, strategy):
    cam = Camera(position=spec["position"], look_at=spec["look_at"], up=spec["up"],
                 fov_y=spec["fov_y"], width=spec["width"], height=spec["height"])
    st = RenderSettings(mode=spec["mode"], strategy=strategy, sampling_step=spec["sampling_step"],
                        early_termination_alpha=spec["early_termination_alpha"],
                        lod_bias=spec["lod_bias"])
    return Scene(camera=cam, settings=st,
                 transfer_functions=[TransferFunction(p) for p in spec["tfs"]],
                 clips=ClipSet(tuple(ClipPlane(tuple(n), o) for n, o in spec["clips"])))


def counters_dict(c):
    return {f: int(getattr(c, f)) for f in c.__dataclass_fields__}


def node_sha(dev):
    return hashlib.sha256(np.asarray(dev.node_buffer).astype("<u8").tobytes()).hexdigest()


def plan_list(plan):
    return [[int(i.node_index), int(i.slot), None if i.evicts is None else int(i.evicts)]
            for i in plan]


def part_transforms(tmp, gold, arrays):
    trees = {}
    for name, b in r2.xf_trees().items():
        tree = ref_tree(tmp, b["tree"], name)
        for c, o, v in b["ops"]:
            tree.insert_block(c, o, np.ascontiguousarray(v))
        tree.drain_events()
        tree.finalize()
        tree.fill_borders()
        tree.drain_events()
        trees[name] = tree
        gold["builds"][name] = dict(node_count=tree.node_count, brick_count=tree.brick_count,
                                    digest=digest(tree, tmp, name))
        print("build", name, tree.node_count, tree.brick_count, flush=True)
    for name, rc in r2.xf_cases().items():
        tree = trees[rc["build"]]
        scene = to_scene(rc["scene"], rc["strategy"])
        out = {}
        if rc["resident"] == "slots":
            dev = DeviceState(tree, slot_count=rc["slots"])
        else:
            dev = DeviceState(tree, slot_count=tree.brick_count + 8)
        if rc["resident"] == "all":
            for n in tree.iter_nodes():
                if n.brick is not None:
                    dev.flag_buffer[n.index] |= FLAG_REQUESTED
            dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), 1e9)
        r = OutOfCoreRenderer(dev)
        if rc["strategy"] == "fullframe":
            img, cnt = r.render_fullframe(scene)
            arrays[name + "/image"] = img
            arrays[name + "/flags"] = dev.flag_buffer.copy()
            out["counters"] = counters_dict(cnt)
            if rc["resident"] == "none":
                plan = dev.process_flags(RenderMode.FULLFRAME)
                out["plan"] = plan_list(plan)
                dev.upload_bricks(plan, 1e9)
                img2, cnt2 = r.render_fullframe(scene)
                arrays[name + "/image2"] = img2
                arrays[name + "/flags2"] = dev.flag_buffer.copy()
                out["counters2"] = counters_dict(cnt2)
        else:
            sess = r.start_refinement(scene, tile=rc.get("tile"))
            plans = []
            while not sess.run_pass():
                plan = dev.process_flags(RenderMode.REFINEMENT)
                plans.append(plan_list(plan))
                dev.upload_bricks(plan, 1e9)
                if sess.passes > 500:
                    raise RuntimeError("refinement did not converge")
            arrays[name + "/image"] = sess.image()
            out["counters"] = counters_dict(sess.counters)
            out["passes"] = sess.passes
            out["plans"] = plans
        gold["renders"][name] = out
        print("render", name, out["counters"]["samples"], flush=True)


def part_ff64(tmp, gold, arrays):
    """tests/test_acceptance.py:321-348: a brick buffer of 1/64 of the
    payload, 24-frame orbit, full-frame mode, uploads with unbounded budget."""
    vol = r2.ff64_volume()
    spec = r2.ff64_tree()
    tree = ref_tree(tmp, spec, "ff64")
    tree.insert_block(0, (0, 0, 0), vol)
    tree.finalize()
    tree.fill_borders()
    tree.drain_events()
    payload = tree.store.payload_nbytes
    brick_nbytes = tree.config.brick_nbytes(tree.descriptor)
    slots = max(1, (payload // 64) // brick_nbytes)
    dev = DeviceState(tree, slot_count=slots)
    r = OutOfCoreRenderer(dev)
    frames = []
    for i in range(24):
        scene = to_scene(r2.ff64_scene_spec(i), "fullframe")
        img, cnt = r.render_fullframe(scene)
        plan = dev.process_flags(RenderMode.FULLFRAME)
        done = dev.upload_bricks(plan, budget_ms=1e9)
        frames.append(dict(counters=counters_dict(cnt), plan=plan_list(plan), uploaded=done,
                           node_sha=node_sha(dev), pending=dev.pending_requests))
        if i in (0, 1, 2, 12, 23):
            arrays[f"ff64/{i}"] = img
    gold["ff64"] = dict(slots=int(slots), payload=int(payload), frames=frames,
                        digest=digest(tree, tmp, "ff64"))
    print("ff64 slots", slots, [f["counters"]["avg_fallbacks"] for f in frames], flush=True)


def part_events(tmp, gold):
    """apply_events over a pruning tree with resident bricks (device.py:205-237)."""
    tree = ref_tree(tmp, r2.events_tree(), "events")
    dev = DeviceState(tree, slot_count=4)
    steps = []
    for step, (origin, block) in enumerate(r2.events_ops()):
        tree.insert_block(0, origin, block)
        evs = tree.drain_events()
        dev.apply_events(evs)
        after_apply = node_sha(dev)
        bricked = sorted(n.index for n in tree.iter_nodes() if n.brick is not None)
        req = r2.events_requests(step, bricked)
        for i in req:
            dev.flag_buffer[i] |= FLAG_REQUESTED
        plan = dev.process_flags(RenderMode.FULLFRAME)
        done = dev.upload_bricks(plan, budget_ms=1e9)
        steps.append(dict(events=[[int(e.kind), int(e.node_index)] for e in evs],
                          after_apply=after_apply, requests=req, plan=plan_list(plan),
                          uploaded=done, node_sha=node_sha(dev),
                          resident=sorted([int(k), int(v)] for k, v in dev._node_slot.items()),
                          pending=dev.pending_requests, evictions=dev.evictions))
    rebuilt = DeviceState(tree, slot_count=4)
    gold["events"] = dict(steps=steps, rebuilt_sha=node_sha(rebuilt),
                          node_count=tree.node_count, brick_count=tree.brick_count)
    print("events", [len(s["events"]) for s in steps], flush=True)


def main():
    gold = {"builds": {}, "renders": {}}
    arrays = {}
    with tempfile.TemporaryDirectory() as tmp:
        part_transforms(tmp, gold, arrays)
        part_ff64(tmp, gold, arrays)
        part_events(tmp, gold)
    with open(os.path.join(HERE, "golden_r2.json"), "w") as fh:
        json.dump(gold, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "renders_r2.npz"), **arrays)


if __name__ == "__main__":
    main()
