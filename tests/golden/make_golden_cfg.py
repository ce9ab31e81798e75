"""Golden vectors at the BASELINE configs, made by running the UNMODIFIED
reference (voxtree, pure Python) in the build container:

    python tests/golden/make_golden_cfg.py cfg1|cfg2|cfg3 [--out DIR]

Scenarios are defined in tests/cfg_scenarios.py.  Writes
tests/golden/golden_<part>.json (+ renders_<part>.npz).  Nothing on the GPU
box reads /root/reference; the GPU tests (tests/test_gpu_cfg.py) consume only
these committed files.  Wall time here: cfg1 ~4 min, cfg2 ~15 min, cfg3 ~1 min.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import cfg_scenarios as cs  # noqa: E402
from voxtree.device import DeviceState, RenderMode  # noqa: E402
from voxtree.octree import Octree  # noqa: E402
from voxtree.render import (Camera, ClipPlane, ClipSet, OutOfCoreRenderer,  # noqa: E402
                            RenderSettings, Scene, TransferFunction)
from voxtree.serialize import save_octree  # noqa: E402
from voxtree.volume import BrickPoolConfig, VolumeDescriptor  # noqa: E402


def ref_tree(tmp, spec, tag):
    desc = VolumeDescriptor(dims=spec["dims"], channels=spec["channels"],
                            sample_format=spec["fmt"])
    cfg = BrickPoolConfig(brick_dims=spec["brick"], homogeneity_threshold=spec["threshold"],
                          page_bricks=spec["page_bricks"], ram_page_limit=spec["ram_page_limit"])
    return Octree.create(desc, cfg, os.path.join(tmp, f"{tag}.pool"))


def file_sha(path):
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for blk in iter(lambda: fh.read(1 << 24), b""):
            h.update(blk)
    return h.hexdigest()


def digest(tree, tmp, tag):
    o, p = os.path.join(tmp, f"{tag}.vxoc"), os.path.join(tmp, f"{tag}.vxbp")
    save_octree(tree, o, p)
    out = [file_sha(o), file_sha(p)]
    os.unlink(o)
    os.unlink(p)
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


def insert_all(tree, ops):
    per = []
    for c, origin, values in ops:
        evs = tree.insert_block(c, origin, np.ascontiguousarray(values))
        per.append(([int(e.kind) for e in evs], [int(e.node_index) for e in evs]))
    tree.drain_events()
    return cs.events_digest(per)


def tree_record(tree, tmp, tag, ev):
    out = dict(events_sha256=ev[0], events_total=ev[1], node_count=tree.node_count,
               brick_count=tree.brick_count, pruned_bricks=tree.pruned_bricks,
               digest_unfinished=digest(tree, tmp, tag + "_a"))
    tree.finalize()
    tree.fill_borders()
    out["border_events"] = len(tree.drain_events())
    out["digest_final"] = digest(tree, tmp, tag + "_b")
    return out


def resident_device(tree):
    dev = DeviceState(tree, slot_count=tree.brick_count + 8)
    for n in tree.iter_nodes():
        if n.brick is not None:
            dev.flag_buffer[n.index] |= 2
    dev.upload_bricks(dev.process_flags(RenderMode.FULLFRAME), 1e9)
    dev.flag_buffer[:] = 0
    dev.node_sha256 = hashlib.sha256(dev.node_buffer.astype("<u8").tobytes()).hexdigest()
    return dev


def part_cfg1(tmp):
    gold, arrays = {"builds": {}, "renders": {}}, {}
    vol = cs.cfg1_volume()
    for tau_name, tau in cs.CFG1_TAUS.items():
        spec = cs.tree_spec(cs.CFG1, tau)
        for mode in cs.CFG1_MODES:
            name = f"{mode}_{tau_name}"
            t0 = time.time()
            tree = ref_tree(tmp, spec, name)
            ev = insert_all(tree, cs.ops(vol, mode))
            t_ins = time.time() - t0
            rec = tree_record(tree, tmp, name, ev)
            rec["reference_seconds"] = round(t_ins, 2)
            gold["builds"][name] = rec
            print("cfg1 build", name, rec["brick_count"], rec["pruned_bricks"], f"{t_ins:.1f}s",
                  flush=True)
            if mode == "bulk":
                dev = resident_device(tree)
                gold["builds"][name]["node_buffer_sha256"] = dev.node_sha256
                sp = cs.scene_spec(cs.CFG1["dims"], **cs.CFG1_SCENE)
                t0 = time.time()
                img, cnt = OutOfCoreRenderer(dev).render_fullframe(to_scene(sp, "fullframe"))
                dt = time.time() - t0
                rname = f"frame_{tau_name}"
                arrays[rname + "/image"] = img.astype(np.float32)
                arrays[rname + "/image_u8"] = np.clip(np.round(img * 255), 0, 255).astype(np.uint8)
                gold["renders"][rname] = dict(build=name, counters=counters_dict(cnt),
                                              flags=cs.flag_sets(dev.flag_buffer),
                                              image_sha256=hashlib.sha256(
                                                  img.astype("<f8").tobytes()).hexdigest(),
                                              reference_seconds=round(dt, 2))
                print("cfg1 render", rname, counters_dict(cnt), f"{dt:.1f}s", flush=True)
    return gold, arrays


def part_cfg2(tmp):
    gold, arrays = {"builds": {}, "renders": {}}, {}
    spec = dict(cs.CFG2)
    tree = ref_tree(tmp, spec, "cfg2")
    t0 = time.time()
    per = []
    M = spec["brick"][2]
    for z0 in range(0, spec["dims"][2], M):
        slab = cs.cfg2_volume_slab(z0, z0 + M)
        for c in range(3):
            evs = tree.insert_block(c, (0, 0, z0), np.ascontiguousarray(slab[..., c]))
            per.append(([int(e.kind) for e in evs], [int(e.node_index) for e in evs]))
        print("cfg2 slab", z0, f"{time.time() - t0:.0f}s", flush=True)
    tree.drain_events()
    t_ins = time.time() - t0
    rec = dict(node_count=tree.node_count, brick_count=tree.brick_count,
               pruned_bricks=tree.pruned_bricks, reference_seconds=round(t_ins, 1))
    tree.finalize()
    t0 = time.time()
    tree.fill_borders()
    tree.drain_events()
    rec["fill_borders_seconds"] = round(time.time() - t0, 1)
    rec["digest_final"] = digest(tree, tmp, "cfg2_b")
    gold["builds"]["slabs_tau0"] = rec
    print("cfg2 build", rec, flush=True)
    dev = resident_device(tree)
    rec["node_buffer_sha256"] = dev.node_sha256
    r = OutOfCoreRenderer(dev)
    for name, tile, bias in cs.CFG2_TILES:
        sp = cs.scene_spec(spec["dims"], cs.CFG2_VIEWPORT, lod_bias=bias, clip_z=cs.CFG2_CLIP_Z)
        dev.flag_buffer[:] = 0
        t0 = time.time()
        sess = r.start_refinement(to_scene(sp, "refinement"), tile=tile)
        while not sess.run_pass():
            dev.upload_bricks(dev.process_flags(RenderMode.REFINEMENT), 1e9)
        dt = time.time() - t0
        x0, y0, x1, y1 = tile
        img = sess.image()
        arrays[name + "/tile"] = img[y0:y1, x0:x1].copy()
        outside = img.copy()
        outside[y0:y1, x0:x1] = 0
        gold["renders"][name] = dict(tile=list(tile), lod_bias=bias, passes=sess.passes,
                                     counters=counters_dict(sess.counters),
                                     flags=cs.flag_sets(dev.flag_buffer),
                                     outside_max=float(np.max(outside)),
                                     reference_seconds=round(dt, 1))
        print("cfg2 tile", name, counters_dict(sess.counters), f"{dt:.1f}s", flush=True)
    return gold, arrays


def part_cfg3(tmp):
    gold = {"builds": {}, "renders": {}}
    vol = cs.cfg3_crop_volume()
    for tau_name, tau in cs.CFG3_TAUS.items():
        spec = cs.tree_spec(cs.CFG3C, tau)
        name = f"stream_{tau_name}"
        t0 = time.time()
        tree = ref_tree(tmp, spec, name)
        ev = insert_all(tree, cs.ops(vol, "stream"))
        t_ins = time.time() - t0
        rec = tree_record(tree, tmp, name, ev)
        rec["reference_seconds"] = round(t_ins, 2)
        gold["builds"][name] = rec
        print("cfg3 crop", name, rec["brick_count"], rec["pruned_bricks"], f"{t_ins:.1f}s",
              flush=True)
    return gold, {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("part", choices=("cfg1", "cfg2", "cfg3"))
    ap.add_argument("--out", default=HERE)
    a = ap.parse_args()
    fn = {"cfg1": part_cfg1, "cfg2": part_cfg2, "cfg3": part_cfg3}[a.part]
    with tempfile.TemporaryDirectory(dir="/tmp") as tmp:
        gold, arrays = fn(tmp)
    with open(os.path.join(a.out, f"golden_{a.part}.json"), "w") as fh:
        json.dump(gold, fh, indent=1, sort_keys=True)
    if arrays:
        np.savez_compressed(os.path.join(a.out, f"renders_{a.part}.npz"), **arrays)


if __name__ == "__main__":
    main()
