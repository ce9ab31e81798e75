"""Deterministic build / render scenarios shared by the golden-vector
generator (run against the unmodified reference), the oracle pin tests and
the GPU parity tests.  Everything is regenerated from seeds, so only the
expected outputs are committed under tests/golden/."""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# build scenarios: (tree kwargs, list of insert ops, fill_borders)
#   op = (channel, origin (x,y,z), shape (dz,dy,dx), generator)
# ---------------------------------------------------------------------------

FIG3_BLOCKS = [((0, 0, 0), [1, 5, 2]), ((6, 0, 0), [3, 3, 2, 2]),
               ((3, 0, 0), [4, 3, 3]), ((10, 0, 0), [4, 4, 2, 4, 3, 3])]


def _rand(seed, shape, lo, hi, dtype):
    return np.random.default_rng(seed).integers(lo, hi, size=shape, dtype=dtype)


def _partition(rng, dims, cuts=2):
    cs = []
    for a in range(3):
        c = sorted(set([0, dims[a]] + list(rng.integers(1, dims[a], size=cuts)))) if dims[a] > 1 \
            else [0, dims[a]]
        cs.append(c)
    boxes = []
    for i in range(len(cs[0]) - 1):
        for j in range(len(cs[1]) - 1):
            for k in range(len(cs[2]) - 1):
                boxes.append(((cs[0][i], cs[1][j], cs[2][k]),
                              (cs[0][i + 1], cs[1][j + 1], cs[2][k + 1])))
    rng.shuffle(boxes)
    return boxes


def scenario(name):
    """Returns dict(tree=..., ops=[(channel, origin, ndarray)], borders=bool)."""
    S = SCENARIOS[name]
    return S()


def _fig3():
    ops = [(0, o, np.asarray(v, np.uint8).reshape(1, 1, -1)) for o, v in FIG3_BLOCKS]
    return dict(tree=dict(dims=(16, 1, 1), brick=(4, 1, 1), threshold=1, fmt="uint8"),
                ops=ops, borders=True)


def _seeding():
    ops = [(0, (0, 0, 0), np.asarray([50, 51, 50, 51], np.uint8).reshape(1, 1, 4)),
           (0, (0, 0, 0), np.asarray([99], np.uint8).reshape(1, 1, 1))]
    return dict(tree=dict(dims=(8, 1, 1), brick=(4, 1, 1), threshold=3, fmt="uint8"),
                ops=ops, borders=True)


def _history_r9(order):
    a = (0, (0, 0, 0), np.asarray([10, 12, 12, 12, 12, 12, 12, 12], np.uint8).reshape(1, 1, 8))
    b = (0, (4, 0, 0), np.asarray([40, 90, 40, 90], np.uint8).reshape(1, 1, 4))
    a2 = (0, (0, 0, 0), np.asarray([10, 12, 12, 12], np.uint8).reshape(1, 1, 4))
    ops = [a, b] if order == "A" else [b, a2]
    return dict(tree=dict(dims=(16, 1, 1), brick=(4, 1, 1), threshold=3, fmt="uint8"),
                ops=ops, borders=True)


def _random_blocks_u8():
    rng = np.random.default_rng(3)
    ops = []
    for _ in range(8):
        origin = tuple(int(v) for v in rng.integers(0, 12, size=3))
        size = tuple(int(v) for v in rng.integers(1, 6, size=3))
        ops.append((0, origin, rng.integers(0, 255, size=size[::-1], dtype=np.uint8)))
    return dict(tree=dict(dims=(16, 16, 16), brick=(4, 4, 4), threshold=12, fmt="uint8"),
                ops=ops, borders=True)


def _halfbg_slices():
    vol = _rand(9, (16, 16, 16), 0, 255, np.uint8)
    vol[:, :8, :] = 0
    ops = [(0, (0, 0, z), vol[z:z + 1]) for z in range(16)]
    return dict(tree=dict(dims=(16, 16, 16), brick=(4, 4, 4), threshold=12, fmt="uint8"),
                ops=ops, borders=True)


def _bulk3_u16_tau0():
    vol = _rand(7, (32, 32, 32, 3), 0, 65535, np.uint16)
    ops = [(c, (0, 0, 0), vol[..., c]) for c in range(3)]
    return dict(tree=dict(dims=(32, 32, 32), brick=(8, 8, 8), threshold=0, fmt="uint16",
                          channels=3), ops=ops, borders=True)


def _partition3_u16_tau0():
    vol = _rand(7, (32, 32, 32, 3), 0, 65535, np.uint16)
    rng = np.random.default_rng(1000)
    ops = []
    for c in range(3):
        for (x0, y0, z0), (x1, y1, z1) in _partition(rng, (32, 32, 32)):
            ops.append((c, (x0, y0, z0), vol[z0:z1, y0:y1, x0:x1, c]))
    return dict(tree=dict(dims=(32, 32, 32), brick=(8, 8, 8), threshold=0, fmt="uint16",
                          channels=3), ops=ops, borders=True)


def _ragged_2ch():
    # non-brick-multiple extents, anisotropic bricks, background 3, tau 500
    rng = np.random.default_rng(11)
    dims = (20, 13, 9)
    vol = rng.integers(0, 65535, size=(9, 13, 20, 2), dtype=np.uint16)
    vol[:, :6, :, 1] = 1000 + (vol[:, :6, :, 1] % 300)
    ops = []
    for c in (0, 1):
        for (x0, y0, z0), (x1, y1, z1) in _partition(rng, dims, cuts=1):
            ops.append((c, (x0, y0, z0), vol[z0:z1, y0:y1, x0:x1, c]))
    return dict(tree=dict(dims=dims, brick=(4, 6, 4), threshold=500, fmt="uint16",
                          channels=2, bg=3, spacing=(1.0, 1.0, 2.0)), ops=ops, borders=True)


def _flat_2d():
    vol = _rand(5, (1, 24, 40), 0, 255, np.uint8)
    vol[0, :12, :20] = 77
    ops = [(0, (0, 0, 0), vol[:, :, :17]), (0, (17, 0, 0), vol[:, :, 17:])]
    return dict(tree=dict(dims=(40, 24, 1), brick=(8, 4, 1), threshold=4, fmt="uint8"),
                ops=ops, borders=True)


def _spim_slices_tau():
    from voxtree_oracle import synth_spim  # oracle/ on sys.path (tests only)
    vol = synth_spim((64, 48, 32), 2, 65535, seed=0)
    ops = []
    for z in range(32):
        for c in range(2):
            ops.append((c, (0, 0, z), vol[z:z + 1, :, :, c]))
    return dict(tree=dict(dims=(64, 48, 32), brick=(8, 8, 8), threshold=None, fmt="uint16",
                          channels=2), ops=ops, borders=True)


def _spim_bulk_u8_tau():
    from voxtree_oracle import synth_spim
    vol = synth_spim((48, 40, 36), 3, 255, seed=7)
    ops = [(c, (0, 0, z), vol[z:z + 8, :, :, c]) for c in range(3) for z in range(0, 36, 8)]
    return dict(tree=dict(dims=(48, 40, 36), brick=(8, 8, 8), threshold=None, fmt="uint8",
                          channels=3), ops=ops, borders=True)


def _collapse_uniform():
    ops = [(0, (0, 0, 0), np.full((8, 8, 8), 200, np.uint8))]
    return dict(tree=dict(dims=(8, 8, 8), brick=(4, 4, 4), threshold=2, fmt="uint8"),
                ops=ops, borders=True)


def _overwrite():
    vol = _rand(5, (16, 16, 16), 0, 255, np.uint8)
    ops = [(0, (0, 0, 0), vol), (0, (4, 4, 4), vol[4:12, 4:12, 4:12]),
           (0, (2, 3, 5), _rand(6, (3, 4, 5), 0, 255, np.uint8))]
    return dict(tree=dict(dims=(16, 16, 16), brick=(8, 8, 8), threshold=12, fmt="uint8"),
                ops=ops, borders=True)


SCENARIOS = {
    "fig3": _fig3,
    "seeding": _seeding,
    "history_A": lambda: _history_r9("A"),
    "history_B": lambda: _history_r9("B"),
    "random_blocks_u8": _random_blocks_u8,
    "halfbg_slices": _halfbg_slices,
    "bulk3_u16_tau0": _bulk3_u16_tau0,
    "partition3_u16_tau0": _partition3_u16_tau0,
    "ragged_2ch": _ragged_2ch,
    "flat_2d": _flat_2d,
    "spim_slices_tau": _spim_slices_tau,
    "spim_bulk_u8_tau": _spim_bulk_u8_tau,
    "collapse_uniform": _collapse_uniform,
    "overwrite": _overwrite,
}

# ---------------------------------------------------------------------------
# render scenarios: (build scenario, scene spec kwargs, strategy)
# ---------------------------------------------------------------------------

COLORS = [(1.0, 0.2, 0.1), (0.1, 1.0, 0.2), (0.2, 0.1, 1.0), (1.0, 1.0, 0.2)]


def ramp_tfs(C, alpha=0.5):
    return [[(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, *COLORS[c], alpha)] for c in range(C)]


def spim_tfs(C):
    return [[(0.0, 0.0, 0.0, 0.0, 0.0), (0.12, 0.0, 0.0, 0.0, 0.0), (1.0, *COLORS[c], 0.4)]
            for c in range(C)]


def camera_for(dims, viewport, distance_scale=2.5, spacing=(1.0, 1.0, 1.0)):
    ext = [d * s for d, s in zip(dims, spacing)]
    center = tuple(e / 2 for e in ext)
    return dict(position=(center[0], center[1], -distance_scale * max(ext)), look_at=center,
                up=(0.0, 1.0, 0.0), fov_y=np.pi / 4, width=viewport[0], height=viewport[1])


def render_case(name):
    return RENDER_CASES[name]()


def _rc(build, viewport=(24, 20), mode="dvr", lod_bias=-64.0, clips=(), tfs=None,
        early=0.99, step=None, dist=2.5, tile=None, strategy="fullframe", resident="all"):
    sc = scenario(build)
    t = sc["tree"]
    C = t.get("channels", 1)
    spacing = t.get("spacing", (1.0, 1.0, 1.0))
    spec = dict(camera_for(t["dims"], viewport, dist, spacing), mode=mode,
                sampling_step=step, early_termination_alpha=early, lod_bias=lod_bias,
                tfs=tfs if tfs is not None else ramp_tfs(C), clips=list(clips))
    return dict(build=build, scene=spec, tile=tile, strategy=strategy, resident=resident)


RENDER_CASES = {
    "bulk3_dvr_lod0": lambda: _rc("bulk3_u16_tau0", lod_bias=-64.0),
    "bulk3_mip": lambda: _rc("bulk3_u16_tau0", mode="mip"),
    "bulk3_lod_bias0": lambda: _rc("bulk3_u16_tau0", viewport=(20, 20), lod_bias=0.0),
    "bulk3_lod_bias2_clip": lambda: _rc("bulk3_u16_tau0", lod_bias=2.0,
                                        clips=[((0.0, 0.0, 1.0), 20.0), ((1.0, 0.0, 0.0), 25.0)]),
    "ragged_dvr_clip": lambda: _rc("ragged_2ch", lod_bias=0.0,
                                   clips=[((0.0, -1.0, 0.0), -3.0)]),
    "spim_u8_dvr": lambda: _rc("spim_bulk_u8_tau", viewport=(32, 24), lod_bias=0.0,
                               tfs=spim_tfs(3)),
    "spim_u8_mip_near": lambda: _rc("spim_bulk_u8_tau", viewport=(32, 24), mode="mip",
                                    dist=1.25, lod_bias=1.0),
    "halfbg_noet": lambda: _rc("halfbg_slices", early=None, lod_bias=0.5),
    "flat2d_dvr": lambda: _rc("flat_2d", viewport=(16, 16), lod_bias=0.0),
    "random_u8_tile_refine": lambda: _rc("random_blocks_u8", viewport=(20, 20),
                                         tile=(4, 3, 15, 17), strategy="refinement"),
    "bulk3_cold_fullframe": lambda: _rc("bulk3_u16_tau0", viewport=(16, 16), lod_bias=0.0,
                                        resident="none"),
}
