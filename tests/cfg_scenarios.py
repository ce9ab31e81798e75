"""BASELINE-config parity scenarios (BASELINE.json configs[0..2]) shared by the
golden generator that runs the UNMODIFIED reference in the build container
(tests/golden/make_golden_cfg.py) and the GPU parity tests
(tests/test_gpu_cfg.py).  Volumes are the seeded SPIM-shaped 'S' data
(SURVEY §8d), regenerated on both sides; only expected outputs are committed
(tests/golden/golden_cfg.json, renders_cfg.npz).

* cfg1: 256^3 x 3 uint8, 32^3 bricks, tau in {0, 0.05*fmax}, built as three
  whole-volume inserts (tests/helpers.py:24-25) and as the VSTR-order slice
  stream (per z: one single-channel slice per channel, ingest.py:306-358);
  512x512 DVR with the clip z <= 200, every brick resident.
* cfg2: 1024^3 x 3 uint16, 32^3 bricks, tau 0 — the bench's 1920x1080 frame
  (bench.py scene_for), checked on 64x64 tiles through the reference's
  tile-restricted RefinementSession (render/raycast.py:309-315).
* cfg3 crop: the 256x256x64 sub-box (x, y 896..1152, z 448..512) of the
  2048x2048x1000 SPIM volume streamed slice-wise in VSTR order, tau 0 and
  0.05*fmax ("digest parity on a 256^2 x 64 crop stream").
"""

from __future__ import annotations

import hashlib

import numpy as np

COLORS = ((1.0, 0.25, 0.2), (0.2, 1.0, 0.3), (0.25, 0.45, 1.0))  # bench.py COLORS


def spim_tfs():
    return [[(0.0, 0.0, 0.0, 0.0, 0.0), (0.12, 0.0, 0.0, 0.0, 0.0), (1.0, *col, 0.4)]
            for col in COLORS]


def scene_spec(dims, viewport, lod_bias=0.0, clip_z=None, mode="dvr"):
    """cli.default_scene-style camera (cli.py:55-63): 2.5x the extent in front
    of the centre along +z, fov 45 deg; the bench scene (bench.py scene_for)."""
    cx, cy, cz = (d / 2.0 for d in dims)
    ext = float(max(dims))
    return dict(position=(cx, cy, -2.5 * ext), look_at=(cx, cy, cz), up=(0.0, 1.0, 0.0),
                fov_y=np.pi / 4, width=viewport[0], height=viewport[1], mode=mode,
                sampling_step=None, early_termination_alpha=0.99, lod_bias=lod_bias,
                tfs=spim_tfs(), clips=[] if clip_z is None else [((0.0, 0.0, 1.0), float(clip_z))])


# ---------------------------------------------------------------------------
# cfg1
# ---------------------------------------------------------------------------

CFG1 = dict(dims=(256, 256, 256), brick=(32, 32, 32), fmt="uint8", channels=3,
            page_bricks=16, ram_page_limit=64)
CFG1_TAUS = {"tau0": 0, "tau5": None}  # None = 0.05 * fmax = 12.75 (volume.py:136-139)
CFG1_MODES = ("bulk", "stream")
CFG1_SCENE = dict(viewport=(512, 512), lod_bias=0.0, clip_z=200.0)


def cfg1_volume():
    import voxtree_oracle as vo
    return vo.synth_spim(CFG1["dims"], 3, 255, seed=0)


def ops(vol, mode, z_chunk=1):
    """Insertion sequence: 'bulk' = one whole-volume insert per channel;
    'stream' = VSTR order, per z one (z_chunk, Y, X) block per channel."""
    C = vol.shape[3]
    if mode == "bulk":
        return [(c, (0, 0, 0), vol[..., c]) for c in range(C)]
    Z = vol.shape[0]
    return [(c, (0, 0, z), vol[z:z + z_chunk, :, :, c]) for z in range(0, Z, z_chunk)
            for c in range(C)]


def tree_spec(base, threshold):
    d = dict(base)
    d["threshold"] = threshold
    return d


# ---------------------------------------------------------------------------
# cfg2
# ---------------------------------------------------------------------------

CFG2 = dict(dims=(1024, 1024, 1024), brick=(32, 32, 32), fmt="uint16", channels=3,
            threshold=0, page_bricks=16, ram_page_limit=4096)
CFG2_VIEWPORT = (1920, 1080)
CFG2_CLIP_Z = 0.8 * 1024  # bench.py CLIP_FRAC
# (name, tile (x0, y0, x1, y1), lod_bias): the frame centre, a tile across the
# side faces' silhouette, the centre one LOD coarser
CFG2_TILES = (("center", (928, 508, 992, 572), 0.0),
              ("side", (1150, 508, 1214, 572), 0.0),
              ("center_lod1", (928, 508, 992, 572), 1.0))


def cfg2_volume_slab(z0, z1):
    import voxtree_oracle as vo
    return vo.synth_spim(CFG2["dims"], 3, 65535, seed=0, z0=z0, z1=z1)


# ---------------------------------------------------------------------------
# cfg3 crop
# ---------------------------------------------------------------------------

CFG3_DIMS = (2048, 2048, 1000)
CFG3_CROP = dict(x=(896, 1152), y=(896, 1152), z=(448, 512))
CFG3C = dict(dims=(256, 256, 64), brick=(32, 32, 32), fmt="uint16", channels=3,
             page_bricks=16, ram_page_limit=64)
CFG3_TAUS = {"tau0": 0, "tau5": None}  # None = 3276.75


def cfg3_crop_volume():
    import voxtree_oracle as vo
    c = CFG3_CROP
    return vo.synth_spim(CFG3_DIMS, 3, 65535, seed=0, z0=c["z"][0], z1=c["z"][1],
                         y0=c["y"][0], y1=c["y"][1], x0=c["x"][0], x1=c["x"][1])


# ---------------------------------------------------------------------------
# digests
# ---------------------------------------------------------------------------

def events_digest(per_insert):
    """sha256 over every insertion's events: int64 [n, kinds..., indices...]
    per insertion, in order.  ``per_insert`` holds (kinds, indices) arrays."""
    h = hashlib.sha256()
    n_total = 0
    for kinds, idx in per_insert:
        kinds = np.asarray(kinds, np.int64)
        idx = np.asarray(idx, np.int64)
        h.update(np.concatenate([[len(kinds)], kinds, idx]).astype("<i8").tobytes())
        n_total += len(kinds)
    return h.hexdigest(), n_total


def flag_sets(flags):
    f = np.asarray(flags)
    return {"used": np.nonzero(f & 1)[0].tolist(), "requested": np.nonzero(f & 2)[0].tolist()}
