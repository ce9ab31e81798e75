"""Shared helpers for the GPU parity tests: build device trees from the
shared scenarios through the drop-in API, digest them with save_octree."""

from __future__ import annotations

import hashlib
import os

import numpy as np

import scenarios


def make_tree(spec, **kw):
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor
    desc = VolumeDescriptor(dims=spec["dims"], channels=spec.get("channels", 1),
                            sample_format=spec.get("fmt", "uint8"),
                            spacing=spec.get("spacing", (1.0, 1.0, 1.0)),
                            background_value=spec.get("bg", 0),
                            channel_transforms=spec.get("transforms"))
    cfg = BrickPoolConfig(brick_dims=spec["brick"], homogeneity_threshold=spec["threshold"],
                          page_bricks=spec.get("page_bricks", 64),
                          ram_page_limit=spec.get("ram_page_limit", 64))
    return Octree(desc, cfg, **kw)


def build_scenario(name, borders=False):
    sc = scenarios.scenario(name)
    tree = make_tree(sc["tree"])
    events = []
    for c, o, v in sc["ops"]:
        evs = tree.insert_block(c, o, v)
        events.append([[int(e.kind), int(e.node_index)] for e in evs])
    tree.drain_events()
    if borders:
        tree.finalize()
        tree.fill_borders()
    return sc, tree, events


def digest(tree, tmp_path, tag):
    from paper_1407_2074_b200 import save_octree
    o, p = os.path.join(tmp_path, f"{tag}.vxoc"), os.path.join(tmp_path, f"{tag}.vxbp")
    save_octree(tree, o, p)
    with open(o, "rb") as fo, open(p, "rb") as fp:
        return [hashlib.sha256(fo.read()).hexdigest(), hashlib.sha256(fp.read()).hexdigest()]


def to_scene(spec, strategy="fullframe"):
    from paper_1407_2074_b200.render import (Camera, ClipPlane, ClipSet, RenderSettings, Scene,
                                             TransferFunction)
    cam = Camera(position=spec["position"], look_at=spec["look_at"], up=spec["up"],
                 fov_y=spec["fov_y"], width=spec["width"], height=spec["height"])
    st = RenderSettings(mode=spec["mode"], strategy=strategy, sampling_step=spec["sampling_step"],
                        early_termination_alpha=spec["early_termination_alpha"],
                        lod_bias=spec["lod_bias"])
    return Scene(cam, st, [TransferFunction(p) for p in spec["tfs"]],
                 ClipSet(tuple(ClipPlane(tuple(n), o) for n, o in spec["clips"])))


def counters_dict(c):
    return {f: int(getattr(c, f)) for f in c.__dataclass_fields__}
