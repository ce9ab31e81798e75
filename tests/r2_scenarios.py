"""Round-2 golden scenarios, shared by tests/golden/make_golden_r2.py (run
against the UNMODIFIED reference in the build container) and the GPU parity
tests (tests/test_gpu_r2.py).  Inputs are regenerated from seeds; only the
expected outputs are committed (tests/golden/golden_r2.json, renders_r2.npz).

* channel-transform renders — the transformed sampler branch
  (render/raycast.py:258-276, transform_points) in full-frame DVR, MIP with
  a clip plane and anisotropic spacing, bounded-residency refinement, and a
  threshold > 0 tree;
* residency — the 1/64 full-frame guarantee orbit
  (tests/test_acceptance.py:321-348) with every plan and counter recorded;
  an apply_events sequence over a pruning tree with resident bricks
  (device.py:205-237, tests/test_device.py:98-150)."""

from __future__ import annotations

import numpy as np

import scenarios


def transforms_a():
    tr = np.stack([np.eye(4)] * 3)
    tr[1, 0, 3] = 1.0
    tr[2, :3, :3] = [[0.99, 0.01, 0.0], [0.0, 1.0, 0.02], [0.0, 0.0, 1.01]]
    tr[2, 2, 3] = -0.5
    return tr


def transforms_b():
    """Small rotation about z for channel 1, a shear + shift for channel 2."""
    tr = np.stack([np.eye(4)] * 3)
    a = np.deg2rad(3.0)
    tr[1, :2, :2] = [[np.cos(a), -np.sin(a)], [np.sin(a), np.cos(a)]]
    tr[1, :3, 3] = [0.75, -0.5, 0.25]
    tr[2, 0, 2] = 0.03
    tr[2, 1, 3] = 1.25
    return tr


def _vol_u16(seed, dims, C):
    from voxtree_oracle import synth_spim  # oracle/ on sys.path (tests only)
    return synth_spim(dims, C, 65535, seed=seed)


def xf_trees():
    """name -> dict(tree=spec, ops=[(c, origin, values)])"""
    out = {}
    rng = np.random.default_rng(3)
    vol = rng.integers(0, 255, size=(32, 32, 32, 3), dtype=np.uint8)
    out["xf_u8"] = dict(
        tree=dict(dims=(32, 32, 32), brick=(8, 8, 8), threshold=0, fmt="uint8", channels=3,
                  transforms=transforms_a()),
        ops=[(c, (0, 0, 0), vol[..., c]) for c in range(3)])
    dims = (40, 36, 28)
    v = _vol_u16(5, dims, 3)
    ops = [(c, (0, 0, z), v[z:z + 7, :, :, c]) for z in range(0, 28, 7) for c in range(3)]
    out["xf_u16_aniso"] = dict(
        tree=dict(dims=dims, brick=(8, 8, 8), threshold=0, fmt="uint16", channels=3,
                  spacing=(1.0, 0.5, 2.0), bg=11, transforms=transforms_b()),
        ops=ops)
    from voxtree_oracle import synth_spim
    w = synth_spim((48, 40, 36), 3, 255, seed=7)
    out["xf_spim_tau"] = dict(
        tree=dict(dims=(48, 40, 36), brick=(8, 8, 8), threshold=None, fmt="uint8", channels=3,
                  transforms=transforms_a()),
        ops=[(c, (0, 0, z), w[z:z + 8, :, :, c]) for c in range(3) for z in range(0, 36, 8)])
    return out


def _scene(tree, viewport, **kw):
    C = tree.get("channels", 1)
    spacing = tree.get("spacing", (1.0, 1.0, 1.0))
    spec = dict(scenarios.camera_for(tree["dims"], viewport, kw.pop("dist", 2.5), spacing),
                mode=kw.pop("mode", "dvr"), sampling_step=kw.pop("step", None),
                early_termination_alpha=kw.pop("early", 0.99), lod_bias=kw.pop("lod_bias", 0.0),
                tfs=kw.pop("tfs", scenarios.ramp_tfs(C)), clips=list(kw.pop("clips", ())))
    assert not kw, kw
    return spec


def xf_cases():
    """name -> dict(build, scene, strategy, resident, tile, slots)"""
    t = {k: v["tree"] for k, v in xf_trees().items()}
    return {
        "xf_u8_dvr": dict(build="xf_u8", scene=_scene(t["xf_u8"], (24, 24), lod_bias=-64.0),
                          strategy="fullframe", resident="all"),
        "xf_u8_dvr_lod": dict(build="xf_u8", scene=_scene(t["xf_u8"], (20, 18), lod_bias=0.5,
                                                          dist=1.6),
                              strategy="fullframe", resident="all"),
        "xf_u16_mip_clip": dict(build="xf_u16_aniso",
                                scene=_scene(t["xf_u16_aniso"], (28, 22), mode="mip",
                                             clips=[((0.0, 0.0, 1.0), 30.0)]),
                                strategy="fullframe", resident="all"),
        "xf_u16_dvr_cold": dict(build="xf_u16_aniso",
                                scene=_scene(t["xf_u16_aniso"], (20, 16), lod_bias=0.0,
                                             tfs=scenarios.spim_tfs(3)),
                                strategy="fullframe", resident="none"),
        "xf_u16_refine": dict(build="xf_u16_aniso",
                              scene=_scene(t["xf_u16_aniso"], (20, 20), lod_bias=-1.0),
                              strategy="refinement", resident="slots", slots=12,
                              tile=(3, 2, 17, 19)),
        "xf_spim_tau_dvr": dict(build="xf_spim_tau",
                                scene=_scene(t["xf_spim_tau"], (32, 24), tfs=scenarios.spim_tfs(3)),
                                strategy="fullframe", resident="all"),
    }


# ---------------------------------------------------------------------------
# residency
# ---------------------------------------------------------------------------

def ff64_volume():
    return np.random.default_rng(19).integers(0, 65535, size=(64, 64, 64), dtype=np.uint16)


def ff64_tree():
    return dict(dims=(64, 64, 64), brick=(16, 16, 16), threshold=0, fmt="uint16", channels=1,
                page_bricks=8, ram_page_limit=64)


def ff64_scene_spec(i):
    """Frame i of the 24-frame orbit (tests/test_acceptance.py:321-348;
    tests/helpers.py:32-48 make_scene: TransferFunction.ramp(max_alpha=0.6))."""
    center = np.array([32.0, 32.0, 32.0])
    radius = 2.5 * 64
    angle = 2 * np.pi * i / 24
    pos = center + radius * np.array([np.sin(angle), 0.0, -np.cos(angle)])
    return dict(position=tuple(float(v) for v in pos), look_at=(32.0, 32.0, 32.0),
                up=(0.0, 1.0, 0.0), fov_y=np.pi / 4, width=24, height=24, mode="dvr",
                sampling_step=None, early_termination_alpha=0.99, lod_bias=0.0,
                tfs=[[(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, 0.6)]], clips=[])


def events_tree():
    return dict(dims=(16, 16, 16), brick=(4, 4, 4), threshold=12, fmt="uint8", channels=1,
                page_bricks=8, ram_page_limit=8)


def events_ops():
    """(origin, block) per step: random blocks, then a uniform overwrite
    that collapses a subtree (NODE_DELETED events), then refills."""
    rng = np.random.default_rng(0)
    out = []
    for _ in range(10):
        origin = tuple(int(v) for v in rng.integers(0, 12, size=3))
        size = rng.integers(1, 5, size=3)
        out.append((origin, rng.integers(0, 255, size=tuple(int(s) for s in reversed(size)),
                                         dtype=np.uint8)))
    out.append(((0, 0, 0), rng.integers(0, 255, size=(16, 16, 16), dtype=np.uint8)))
    out.append(((0, 0, 0), np.full((8, 8, 8), 90, np.uint8)))
    out.append(((8, 8, 8), np.full((8, 8, 8), 200, np.uint8)))
    out.append(((4, 4, 4), rng.integers(0, 255, size=(6, 6, 6), dtype=np.uint8)))
    return out


def events_requests(step, bricked):
    """Deterministic REQUESTED set for a step from the sorted bricked nodes."""
    if not bricked:
        return []
    n = len(bricked)
    return sorted({bricked[(7 * step) % n], bricked[(7 * step + 3) % n], bricked[-1 - step % n]})
