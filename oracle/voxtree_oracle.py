"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference ``voxtree`` hot path (octree build,
border fill, VXOC/VXBP serialization, Fig. 4 node entries, octree ray
casting).  It exists to CHECK the CUDA product path and to time the
reference algorithm on host cores (``bench.py`` cpu_baseline / ``--impl
reference``).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``
may import it; the product package never does.

Parity pin: every function below is checked against golden vectors produced
by the unmodified reference (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src`` in the build container and commits the results
under ``tests/golden/``), and against the reference's own known-answer tests
(Fig. 3 walk, half-sample vectors, seeding, borders).  See
``tests/test_oracle_golden.py``.

The tree state is kept the way the GPU engine keeps it — flat, keyed by the
breadth-first node index — rather than as linked node objects.
Citations are relative to /root/reference/pkg/src/voxtree/.
"""

from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# geometry  (volume.py:155-260)
# ---------------------------------------------------------------------------


def virtual_dims(dims, brick):
    """Shared-depth padding to M*2^N per split axis (volume.py:155-179)."""
    ns = []
    for d, m in zip(dims, brick):
        n, ext = 0, m
        while ext < d:
            ext, n = ext * 2, n + 1
        ns.append(n)
    depth = max(ns)
    virt = tuple(m if n == 0 else m << depth for m, n in zip(brick, ns))
    return virt, depth


class Geo:
    """Complete-tree BFS geometry (volume.py:182-260)."""

    def __init__(self, dims, brick):
        self.dims = tuple(int(v) for v in dims)
        self.brick = tuple(int(v) for v in brick)
        self.virtual, self.depth = virtual_dims(self.dims, self.brick)
        self.split = tuple(v > m for v, m in zip(self.virtual, self.brick))
        self.capacity = (8 ** (self.depth + 1) - 1) // 7
        self.real_octants = [k for k in range(8)
                             if all(self.split[a] or not (k >> a) & 1 for a in range(3))]
        # first BFS index of each depth d (d = depth - level)
        self.level_start = [(8 ** d - 1) // 7 for d in range(self.depth + 2)]

    def extent(self, level):
        return tuple(m << level if s else m for m, s in zip(self.brick, self.split))

    def scale(self, level):
        return tuple(1 << level if s else 1 for s in self.split)

    def level_of(self, index):
        d = 0
        while index >= self.level_start[d + 1]:
            d += 1
        return self.depth - d

    def path(self, index):
        ks = []
        while index > 0:
            ks.append((index - 1) % 8)
            index = (index - 1) // 8
        return ks[::-1]

    def box_lo(self, index):
        lo = [0, 0, 0]
        level = self.depth
        for k in self.path(index):
            half = self.extent(level - 1)
            for a in range(3):
                if (k >> a) & 1:
                    lo[a] += half[a]
            level -= 1
        return tuple(lo)

    def octant(self, point, lo, level):
        half = self.extent(level - 1)
        return sum(1 << a for a in range(3)
                   if self.split[a] and point[a] >= lo[a] + half[a])

    def in_volume(self, lo, level):
        ext = self.extent(level)
        return all(lo[a] < self.dims[a] and lo[a] + ext[a] > 0 for a in range(3))

    def in_extent(self, lo, level):
        """(cx, cy, cz) in-volume interior counts (octree.py:190-199)."""
        sc = self.scale(level)
        return tuple(int(min(max(-(-(self.dims[a] - lo[a]) // sc[a]), 0), self.brick[a]))
                     for a in range(3))


# ---------------------------------------------------------------------------
# integer kernels  (octree.py:53-99)
# ---------------------------------------------------------------------------


def round_mean(sums, counts):
    """(2*sum + n) // (2n): exact rational mean, ties up (octree.py:53-55)."""
    s = np.asarray(sums, dtype=np.int64)
    n = np.asarray(counts, dtype=np.int64)
    return (2 * s + n) // (2 * n)


def halfsample(values, in_extent, split, bg):
    """2x2x2 (split axes only) mean over in-volume sources; bg where a parent
    voxel has none (octree.py:58-92).  values: (mz, my, mx, C)."""
    mz, my, mx, nc = values.shape
    cx, cy, cz = in_extent
    kx, ky, kz = (2 if split[0] else 1), (2 if split[1] else 1), (2 if split[2] else 1)
    masked = np.zeros((mz, my, mx, nc), dtype=np.int64)
    masked[:cz, :cy, :cx] = values[:cz, :cy, :cx]
    oz, oy, ox = mz // kz, my // ky, mx // kx
    sums = masked.reshape(oz, kz, oy, ky, ox, kx, nc).sum(axis=(1, 3, 5))
    cnt_x = np.clip(cx - kx * np.arange(ox), 0, kx)
    cnt_y = np.clip(cy - ky * np.arange(oy), 0, ky)
    cnt_z = np.clip(cz - kz * np.arange(oz), 0, kz)
    cnt = (cnt_z[:, None, None] * cnt_y[None, :, None] * cnt_x[None, None, :])[..., None]
    mean = (2 * sums + cnt) // (2 * np.maximum(cnt, 1))
    return np.where(cnt > 0, mean, np.int64(bg))


def homogeneous(lo, hi, tau):
    """strict max - min < tau on every channel (octree.py:95-99)."""
    return all((h - l) < tau for l, h in zip(lo, hi))


# ---------------------------------------------------------------------------
# incremental octree build  (octree.py:143-614)
# ---------------------------------------------------------------------------

CREATED, DELETED, UPDATED = 1, 2, 3


class OracleTree:
    """Flat BFS-indexed octree state.  ``bricks[i]`` is the stored brick
    (Mz+2, My+2, Mx+2, C) of node i; ``kids`` holds nodes with children."""

    def __init__(self, dims, brick, channels=1, fmt="uint8", bg=0, threshold=0.0,
                 spacing=(1.0, 1.0, 1.0), transforms=None, page_bricks=64,
                 ram_page_limit=64):
        self.geo = Geo(dims, brick)
        if self.geo.depth > 8:
            raise ValueError("tree deeper than 9 levels")
        self.C = int(channels)
        self.fmt = fmt
        self.dtype = np.dtype(np.uint8 if fmt == "uint8" else np.uint16)
        self.fmax = 255 if fmt == "uint8" else 65535
        self.bg = int(bg)
        self.tau = float(threshold) if threshold is not None else 0.05 * self.fmax
        self.spacing = tuple(float(s) for s in spacing)
        self.transforms = None if transforms is None else np.asarray(transforms, np.float64)
        self.page_bricks = page_bricks
        self.ram_page_limit = ram_page_limit
        self.exists = {0}
        self.kids = set()
        self.bricks: dict[int, np.ndarray] = {}
        self.in_vol = {0: True}
        bgv = [self.bg] * self.C
        self.avg = {0: list(bgv)}
        self.smin = {0: list(bgv)}
        self.smax = {0: list(bgv)}
        self.sub = {0: (list(bgv), list(bgv))}
        self.pruned_bricks = 0
        self.events: list[tuple[int, int]] = []
        self.finished = False
        self.borders_filled = False

    # -- helpers ------------------------------------------------------------
    @property
    def node_count(self):
        return len(self.exists)

    def level(self, i):
        return self.geo.level_of(i)

    def children(self, i):
        if i not in self.kids:
            return []
        return [8 * i + 1 + k for k in self.geo.real_octants]

    def _stored_shape(self):
        m = self.geo.brick
        return (m[2] + 2, m[1] + 2, m[0] + 2, self.C)

    def _create_children(self, i):
        """octree.py:209-223 — all real octants at once, seeded with the
        parent's current AVG when in-volume."""
        if i in self.kids:
            return
        self.kids.add(i)
        lvl = self.level(i)
        lo = self.geo.box_lo(i)
        for k in self.geo.real_octants:
            c = 8 * i + 1 + k
            clo = self.geo.box_lo(c)
            inv = self.geo.in_volume(clo, lvl - 1)
            seed = list(self.avg[i]) if inv else [self.bg] * self.C
            self.exists.add(c)
            self.in_vol[c] = inv
            self.avg[c] = list(seed)
            self.smin[c] = list(seed)
            self.smax[c] = list(seed)
            self.sub[c] = (list(seed), list(seed)) if inv else None
            self.events.append((CREATED, c))
        del lo

    def _alloc_brick(self, i):
        """octree.py:225-241 — bg everywhere, node AVG over in-volume interior."""
        if i in self.bricks:
            return False
        b = np.full(self._stored_shape(), self.bg, dtype=self.dtype)
        cx, cy, cz = self.geo.in_extent(self.geo.box_lo(i), self.level(i))
        b[1:1 + cz, 1:1 + cy, 1:1 + cx, :] = np.asarray(self.avg[i], dtype=self.dtype)
        self.bricks[i] = b
        return True

    def _stats(self, i):
        """octree.py:248-263 (+ sub for leaves / childless nodes)."""
        cx, cy, cz = self.geo.in_extent(self.geo.box_lo(i), self.level(i))
        if 0 in (cx, cy, cz):
            return
        reg = self.bricks[i][1:1 + cz, 1:1 + cy, 1:1 + cx, :].reshape(-1, self.C)
        n = cx * cy * cz
        self.smin[i] = [int(v) for v in reg.min(axis=0)]
        self.smax[i] = [int(v) for v in reg.max(axis=0)]
        self.avg[i] = [int(v) for v in round_mean(reg.sum(axis=0, dtype=np.int64), n)]
        if self.level(i) == 0 or i not in self.kids:
            self.sub[i] = (list(self.smin[i]), list(self.smax[i]))

    def _aggregate(self, i):
        """octree.py:265-277."""
        lo = hi = None
        for c in self.children(i):
            s = self.sub[c]
            if s is None:
                continue
            if lo is None:
                lo, hi = list(s[0]), list(s[1])
            else:
                lo = [min(a, b) for a, b in zip(lo, s[0])]
                hi = [max(a, b) for a, b in zip(hi, s[1])]
        if lo is not None:
            self.sub[i] = (lo, hi)

    def _octant_values(self, c):
        """octree.py:281-306 — child's contribution to its parent."""
        g = self.geo
        mx, my, mz = g.brick
        lvl = self.level(c)
        cx, cy, cz = g.in_extent(g.box_lo(c), lvl)
        if c in self.bricks:
            inner = self.bricks[c][1:1 + mz, 1:1 + my, 1:1 + mx, :]
            return halfsample(inner, (cx, cy, cz), g.split, self.bg)
        kx, ky, kz = (2 if g.split[0] else 1), (2 if g.split[1] else 1), (2 if g.split[2] else 1)
        out = np.full((mz // kz, my // ky, mx // kx, self.C), self.bg, dtype=np.int64)
        out[:-(-cz // kz), :-(-cy // ky), :-(-cx // kx), :] = self.avg[c]
        return out

    def _write_octant(self, p, c):
        """octree.py:308-319."""
        g = self.geo
        mx, my, mz = g.brick
        k = (c - 1) % 8
        blk = self._octant_values(c)
        ox = mx // 2 if (k & 1 and g.split[0]) else 0
        oy = my // 2 if (k & 2 and g.split[1]) else 0
        oz = mz // 2 if (k & 4 and g.split[2]) else 0
        bz, by, bx = blk.shape[:3]
        self.bricks[p][1 + oz:1 + oz + bz, 1 + oy:1 + oy + by, 1 + ox:1 + ox + bx, :] = blk

    def _leaf_for(self, gx, gy, gz):
        """octree.py:399-409."""
        g = self.geo
        pt = (gx * g.brick[0] + 0.5, gy * g.brick[1] + 0.5, gz * g.brick[2] + 0.5)
        i, lvl, lo = 0, g.depth, (0, 0, 0)
        while lvl > 0:
            self._create_children(i)
            k = g.octant(pt, lo, lvl)
            i = 8 * i + 1 + k
            lo = g.box_lo(i)
            lvl -= 1
        self._alloc_brick(i)
        return i

    def insert(self, channel, origin, values):
        """octree.py:323-397 — one channel's (dz, dy, dx) cuboid at origin."""
        if not 0 <= channel < self.C:
            raise ValueError("channel out of range")
        origin = tuple(int(v) for v in origin)
        values = np.asarray(values)
        if values.ndim != 3:
            raise ValueError("block values must be 3-D")
        bd = (values.shape[2], values.shape[1], values.shape[0])
        g = self.geo
        for a in range(3):
            if origin[a] < 0 or origin[a] + bd[a] > g.dims[a]:
                raise ValueError("block outside volume")
        values = values.astype(self.dtype, copy=False)
        start = len(self.events)
        touched = [set() for _ in range(g.depth + 1)]
        updated = set()
        m = g.brick
        lo_g = [origin[a] // m[a] for a in range(3)]
        hi_g = [(origin[a] + bd[a] - 1) // m[a] for a in range(3)]
        for gz in range(lo_g[2], hi_g[2] + 1):
            for gy in range(lo_g[1], hi_g[1] + 1):
                for gx in range(lo_g[0], hi_g[0] + 1):
                    leaf = self._leaf_for(gx, gy, gz)
                    llo = g.box_lo(leaf)
                    s = [max(origin[a], llo[a]) for a in range(3)]
                    e = [min(origin[a] + bd[a], llo[a] + m[a]) for a in range(3)]
                    self.bricks[leaf][1 + s[2] - llo[2]:1 + e[2] - llo[2],
                                      1 + s[1] - llo[1]:1 + e[1] - llo[1],
                                      1 + s[0] - llo[0]:1 + e[0] - llo[0], channel] = \
                        values[s[2] - origin[2]:e[2] - origin[2],
                               s[1] - origin[1]:e[1] - origin[1],
                               s[0] - origin[0]:e[0] - origin[0]]
                    self._stats(leaf)
                    touched[0].add(leaf)
                    updated.add(leaf)
        for lvl in range(1, g.depth + 1):
            groups: dict[int, list[int]] = {}
            for c in touched[lvl - 1]:
                groups.setdefault((c - 1) // 8, []).append(c)
            for p in sorted(groups):
                fresh = self._alloc_brick(p)
                for c in (self.children(p) if fresh else sorted(groups[p])):
                    self._write_octant(p, c)
                self._stats(p)
                self._aggregate(p)
                touched[lvl].add(p)
                updated.add(p)
        deleted: set[int] = set()
        self._prune(touched, updated, deleted)
        for i in sorted(updated):
            if i not in deleted:
                self.events.append((UPDATED, i))
        return self.events[start:]

    def _drop_brick(self, i):
        if i in self.bricks:
            del self.bricks[i]
            self.pruned_bricks += 1

    def _delete_below(self, i, deleted):
        """octree.py:482-493 — post-order deletion."""
        for c in self.children(i):
            if c in self.kids:
                self._delete_below(c, deleted)
            self._drop_brick(c)
            self.exists.discard(c)
            for d in (self.in_vol, self.avg, self.smin, self.smax, self.sub):
                d.pop(c, None)
            deleted.add(c)
            self.events.append((DELETED, c))
        self.kids.discard(i)

    def _prune(self, touched, updated, deleted):
        """octree.py:456-480."""
        g, tau = self.geo, self.tau
        for lvl in range(g.depth + 1):
            for i in sorted(touched[lvl]):
                if i == 0 or i not in self.bricks:
                    continue
                if homogeneous(self.smin[i], self.smax[i], tau):
                    self._drop_brick(i)
                    updated.add(i)
        for lvl in range(1, g.depth + 1):
            for i in sorted(touched[lvl]):
                if i == 0 or i not in self.kids:
                    continue
                s = self.sub[i]
                if s is None or homogeneous(s[0], s[1], tau):
                    self._delete_below(i, deleted)
                    updated.add(i)
        s = self.sub[0]
        if (s is None or homogeneous(s[0], s[1], tau)) and (0 in self.kids or 0 in self.bricks):
            if 0 in self.kids:
                self._delete_below(0, deleted)
            self._drop_brick(0)
            updated.add(0)

    # -- queries --------------------------------------------------------------
    def find(self, point, target_level=0):
        """octree.py:497-505."""
        g = self.geo
        i, lvl, lo = 0, g.depth, (0, 0, 0)
        while lvl > target_level and i in self.kids:
            i = 8 * i + 1 + g.octant(point, lo, lvl)
            lo = g.box_lo(i)
            lvl -= 1
        return i

    def nodes(self):
        return sorted(self.exists)

    # -- borders (octree.py:540-614) ---------------------------------------------
    def fill_borders(self):
        g = self.geo
        m = g.brick
        for i in sorted(self.bricks):
            lvl = self.level(i)
            sc = g.scale(lvl)
            lo = g.box_lo(i)
            mlo = [lo[a] // sc[a] for a in range(3)]
            mvirt = [-(-g.virtual[a] // sc[a]) for a in range(3)]
            dst = self.bricks[i]
            for sz in range(3):
                for sy in range(3):
                    for sx in range(3):
                        if (sx, sy, sz) == (1, 1, 1):
                            continue
                        loc, glb, out = [], [], False
                        for a, s in enumerate((sx, sy, sz)):
                            if s == 1:
                                loc.append((1, 1 + m[a]))
                                glb.append(mlo[a])
                            else:
                                l0 = 0 if s == 0 else 1 + m[a]
                                g0 = mlo[a] - 1 if s == 0 else mlo[a] + m[a]
                                loc.append((l0, l0 + 1))
                                glb.append(g0)
                                out = out or g0 < 0 or g0 >= mvirt[a]
                        view = dst[loc[2][0]:loc[2][1], loc[1][0]:loc[1][1], loc[0][0]:loc[0][1], :]
                        if out:
                            view[...] = self.bg
                            continue
                        pt = tuple((glb[a] + 0.5) * sc[a] for a in range(3))
                        nb = self.find(pt, lvl)
                        if self.level(nb) != lvl or nb not in self.bricks:
                            view[...] = np.asarray(self.avg[nb], dtype=self.dtype)
                            continue
                        nlo = g.box_lo(nb)
                        nm = [nlo[a] // sc[a] for a in range(3)]
                        sl = [slice(1 + glb[a] - nm[a], 1 + glb[a] - nm[a] + (loc[a][1] - loc[a][0]))
                              for a in range(3)]
                        view[...] = self.bricks[nb][sl[2], sl[1], sl[0], :]
            self.events.append((UPDATED, i))
        self.borders_filled = True


# ---------------------------------------------------------------------------
# VXOC / VXBP bytes  (serialize.py:61-125, paging.py:200-380)
# ---------------------------------------------------------------------------

_FMT_CODE = {"uint8": 1, "uint16": 2}


def serialize(t: OracleTree):
    """(vxoc_bytes, vxbp_bytes) exactly as save_octree writes them."""
    g = t.geo
    bricked = [i for i in t.nodes() if i in t.bricks]
    brick_nbytes = int(np.prod(t._stored_shape())) * t.dtype.itemsize
    pb = t.page_bricks
    npages = -(-len(bricked) // pb)
    sb = t._stored_shape()
    pool = [struct.pack("<4sIIQIIIHHQQ12x", b"VXBP", 1, pb, brick_nbytes,
                        sb[0], sb[1], sb[2], t.C, _FMT_CODE[t.fmt], npages,
                        (64 + npages * (pb * brick_nbytes + 4)) if npages else 0)]
    for p in range(npages):
        page = bytearray(pb * brick_nbytes)
        for s, i in enumerate(bricked[p * pb:(p + 1) * pb]):
            page[s * brick_nbytes:(s + 1) * brick_nbytes] = \
                np.ascontiguousarray(t.bricks[i], dtype=t.dtype.newbyteorder("<")).tobytes()
        pool.append(bytes(page))
        pool.append(struct.pack("<I", zlib.crc32(bytes(page))))
    if npages:
        bits = np.zeros(npages * pb, dtype=np.uint8)
        bits[:len(bricked)] = 1
        pool.append(np.packbits(bits, bitorder="little").tobytes())
    flags = (1 if t.transforms is not None else 0) | (2 if t.finished else 0) | \
        (4 if t.borders_filled else 0)
    meta = [struct.pack("<4sI", b"VXOC", 1),
            struct.pack("<3IHH3dIB3x", *g.dims, t.C, _FMT_CODE[t.fmt], *t.spacing, t.bg, flags)]
    if t.transforms is not None:
        meta.append(np.asarray(t.transforms, dtype="<f8").tobytes())
    meta.append(struct.pack("<3IdIII", *g.brick, t.tau, 1, pb, t.ram_page_limit))
    nodes = t.nodes()
    meta.append(struct.pack("<IQ", g.depth, len(nodes)))
    canon = {i: divmod(s, pb) for s, i in enumerate(bricked)}
    for i in nodes:
        nf = (1 if i in t.bricks else 0) | (2 if i in t.kids else 0) | (4 if t.in_vol[i] else 0)
        meta.append(struct.pack("<QBB2x", i, t.level(i), nf))
        sub = t.sub[i]
        for c in range(t.C):
            meta.append(struct.pack("<5I", t.smin[i][c], t.smax[i][c], t.avg[i][c],
                                    sub[0][c] if sub else 0, sub[1][c] if sub else 0))
        meta.append(struct.pack("<II", *canon.get(i, (0xFFFFFFFF, 0xFFFFFFFF))))
    return b"".join(meta), b"".join(pool)


def digest(t: OracleTree):
    import hashlib
    a, b = serialize(t)
    return hashlib.sha256(a).hexdigest(), hashlib.sha256(b).hexdigest()


# ---------------------------------------------------------------------------
# Fig. 4 node entries  (device.py:47-99, 168-203)
# ---------------------------------------------------------------------------


def quantize(v, C, fmax):
    qmax = (1 << (40 // C)) - 1
    return int(round(v * qmax / fmax))


def pack_entry(resident, not_homog, child_ptr, slot, avgs, C):
    if not 0 <= child_ptr < (1 << 22):
        raise OverflowError("child pointer exceeds 22 bits")
    e = (1 if resident else 0) | (2 if not_homog else 0) | (child_ptr << 2)
    if resident:
        if not 0 <= slot < (1 << 32):
            raise OverflowError("slot exceeds 32 bits")
        return e | (slot << 24)
    w = 40 // C
    for c, q in enumerate(avgs):
        if not 0 <= q < (1 << w):
            raise OverflowError("AVG exceeds field")
        e |= q << (24 + c * w)
    return e


def node_buffer(t: OracleTree, slots: dict | None = None):
    """uint64[capacity]; ``slots`` maps node index -> brick-buffer slot for
    resident bricks (device.py:168-178, 193-203)."""
    slots = slots or {}
    nb = np.zeros(t.geo.capacity, dtype=np.uint64)
    for i in t.nodes():
        ptr = i + 1 if i in t.kids else 0
        if i in slots:
            nb[i] = pack_entry(True, i in t.bricks, ptr, slots[i], (), t.C)
        else:
            nb[i] = pack_entry(False, i in t.bricks, ptr, None,
                               [quantize(v, t.C, t.fmax) for v in t.avg[i]], t.C)
    return nb


def resident_buffers(t: OracleTree):
    """Every brick resident, slots in BFS order (the all-resident mirror)."""
    bricked = [i for i in t.nodes() if i in t.bricks]
    slots = {i: s for s, i in enumerate(bricked)}
    shape = (max(1, len(bricked)),) + t._stored_shape()
    bb = np.zeros(shape, dtype=t.dtype)
    for i, s in slots.items():
        bb[s] = t.bricks[i]
    return node_buffer(t, slots), bb, slots


# ---------------------------------------------------------------------------
# ray casting  (render/camera.py, core.py, transfer.py, raycast.py)
# ---------------------------------------------------------------------------


@dataclass
class SceneSpec:
    """Plain-data scene: camera, settings, per-channel TF points, clips."""
    position: tuple
    look_at: tuple
    up: tuple = (0.0, 1.0, 0.0)
    fov_y: float = np.pi / 4
    width: int = 16
    height: int = 16
    mode: str = "dvr"
    sampling_step: float | None = None
    reference_step: float | None = None
    early_termination_alpha: float | None = 0.99
    lod_bias: float = 0.0
    tfs: list = field(default_factory=list)       # per channel: [(x, r, g, b, a), ...]
    clips: list = field(default_factory=list)     # [((nx, ny, nz), offset), ...]


def _unit(v):
    n = np.linalg.norm(v)
    if n == 0:
        raise ValueError("zero-length camera vector")
    return v / n


def camera_basis(s: SceneSpec):
    pos = np.asarray(s.position, dtype=np.float64)
    fwd = _unit(np.asarray(s.look_at, dtype=np.float64) - pos)
    right = _unit(np.cross(fwd, np.asarray(s.up, dtype=np.float64)))
    return pos, fwd, right, np.cross(right, fwd)


def camera_rays(s: SceneSpec):
    """camera.py:41-53."""
    pos, fwd, right, up = camera_basis(s)
    th = np.tan(s.fov_y / 2.0)
    xs = (2.0 * (np.arange(s.width) + 0.5) / s.width - 1.0) * th * (s.width / s.height)
    ys = (1.0 - 2.0 * (np.arange(s.height) + 0.5) / s.height) * th
    px, py = np.meshgrid(xs, ys)
    d = fwd[None, :] + px.reshape(-1, 1) * right[None, :] + py.reshape(-1, 1) * up[None, :]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return pos.reshape(1, 3), d


def ray_bounds(origin, dirs, box_hi, clips):
    """core.py:34-67."""
    hi = np.asarray(box_hi, dtype=np.float64)
    t0 = np.zeros(len(dirs))
    t1 = np.full(len(dirs), np.inf)
    for a in range(3):
        o, d = origin[..., a], dirs[:, a]
        with np.errstate(divide="ignore", invalid="ignore"):
            ta, tb = (0.0 - o) / d, (hi[a] - o) / d
        par = d == 0
        ins = (o >= 0.0) & (o <= hi[a])
        t0 = np.maximum(t0, np.where(par, np.where(ins, -np.inf, np.inf), np.minimum(ta, tb)))
        t1 = np.minimum(t1, np.where(par, np.where(ins, np.inf, -np.inf), np.maximum(ta, tb)))
    for normal, offset in clips:
        n = np.asarray(normal, dtype=np.float64)
        num = offset - origin @ n
        den = dirs @ n
        with np.errstate(divide="ignore", invalid="ignore"):
            tc = num / den
        keep = (den == 0) & (num >= 0)
        kill = (den == 0) & (num < 0)
        up = den > 0
        t1 = np.where(up, np.minimum(t1, tc), t1)
        t0 = np.where(~up & ~keep & ~kill, np.maximum(t0, tc), t0)
        t1 = np.where(kill, -np.inf, t1)
    return t0, t1, t0 < t1


def tf_lookup(points, x):
    """transfer.py:12-41 — np.interp per component on sorted points."""
    pts = sorted((float(p[0]), tuple(float(v) for v in p[1:])) for p in points)
    xs = np.asarray([p[0] for p in pts])
    rgba = np.asarray([p[1] for p in pts])
    flat = np.asarray(x, dtype=np.float64).reshape(-1)
    return np.stack([np.interp(flat, xs, rgba[:, j]) for j in range(4)], axis=1)


class OracleRenderer:
    """Octree ray caster over (node_buffer, brick_buffer) — raycast.py:53-339.

    Per-ray state (k, acc, mip, terminated) lives in ``state`` so refinement
    passes can resume; ``flags`` is the feedback byte buffer."""

    def __init__(self, t: OracleTree, nb, bb, flags=None):
        self.t, self.g = t, t.geo
        self.nb, self.bb = nb, bb
        self.flags = np.zeros(t.geo.capacity, np.uint8) if flags is None else flags
        self.spacing = np.asarray(t.spacing, np.float64)
        self.dims = np.asarray(self.g.dims, np.float64)
        self.box_hi = self.dims * self.spacing
        sp = np.asarray(self.g.split)
        self.base_voxel = float(np.min(self.spacing[sp] if sp.any() else self.spacing))
        self.ext = np.asarray([self.g.extent(l) for l in range(self.g.depth + 1)], np.float64)
        self.scl = np.asarray([self.g.scale(l) for l in range(self.g.depth + 1)], np.float64)
        tr = t.transforms
        self.transforms = None
        if tr is not None and any(not np.allclose(tr[c], np.eye(4)) for c in range(t.C)):
            self.transforms = tr

    # counters: samples, tf_lookups, avg_fallbacks, coarse_fallbacks, requested, used
    def new_counters(self):
        return dict(samples=0, tf_lookups=0, avg_fallbacks=0, coarse_fallbacks=0,
                    bricks_requested=0, bricks_used_marks=0)

    def start(self, s: SceneSpec, tile=None):
        o, d = camera_rays(s)
        step = float(s.sampling_step) if s.sampling_step is not None else 0.5 * float(np.min(self.spacing))
        t0, t1, hit = ray_bounds(o, d, self.box_hi, s.clips)
        span = np.maximum(t1 - t0, 0.0)
        n = len(d)
        st = dict(origin=o, dirs=d, step=step, t0=np.where(hit, t0, 0.0),
                  n=np.where(hit, np.ceil(span / step - 1e-12), 0).astype(np.int64),
                  k=np.zeros(n, np.int64), susp=np.zeros(n, bool),
                  rgb=np.zeros((n, 3)), a=np.zeros(n), mip=np.zeros((n, self.t.C)),
                  term=np.zeros(n, bool))
        if tile is not None:
            x0, y0, x1, y1 = tile
            cols, rows = np.meshgrid(np.arange(s.width), np.arange(s.height))
            st["n"][(~((cols >= x0) & (cols < x1) & (rows >= y0) & (rows < y1))).reshape(-1)] = 0
        return st

    def _mark(self, idx, flag):
        if idx.size:
            np.bitwise_or.at(self.flags, idx, np.uint8(flag))

    def _descend(self, pv, target):
        """raycast.py:86-123."""
        n = len(pv)
        idx = np.zeros(n, np.int64)
        lvl = np.full(n, self.g.depth, np.int64)
        lo = np.zeros((n, 3))
        a1 = np.full(n, -1, np.int64)
        a1l = np.zeros(n, np.int64)
        a1lo = np.zeros((n, 3))
        a2, a2l, a2lo = a1.copy(), a1l.copy(), a1lo.copy()
        split = np.asarray(self.g.split)
        for _ in range(self.g.depth):
            ptr = ((self.nb[idx] >> np.uint64(2)) & np.uint64(0x3FFFFF)).astype(np.int64)
            mv = np.flatnonzero((ptr != 0) & (lvl > target))
            if mv.size == 0:
                break
            half = self.ext[lvl[mv] - 1]
            bits = (pv[mv] >= lo[mv] + half) & split[None, :]
            k = bits[:, 0] * 1 + bits[:, 1] * 2 + bits[:, 2] * 4
            a2[mv], a2l[mv], a2lo[mv] = a1[mv], a1l[mv], a1lo[mv]
            a1[mv], a1l[mv], a1lo[mv] = idx[mv], lvl[mv], lo[mv]
            idx[mv] = 8 * (ptr[mv] - 1) + 1 + k
            lo[mv] = lo[mv] + bits * half
            lvl[mv] -= 1
        return idx, lvl, lo, (a1, a1l, a1lo), (a2, a2l, a2lo)

    def _avg(self, e, c):
        w = 40 // self.t.C
        q = ((e >> np.uint64(24 + c * w)) & np.uint64((1 << w) - 1)).astype(np.float64)
        return np.round(q * float(self.t.fmax) / float((1 << w) - 1))

    def _trilerp(self, e, lvl, lo, pv, c):
        slot = ((e >> np.uint64(24)) & np.uint64(0xFFFFFFFF)).astype(np.int64)
        m = np.asarray(self.g.brick, np.int64)
        f = (pv - lo) / self.scl[lvl] + 0.5
        f = np.clip(f, 0.0, m + 1.0) if self.t.borders_filled else np.clip(f, 1.0, m.astype(np.float64))
        i0 = np.clip(np.floor(f).astype(np.int64), 0, m)
        w1 = np.clip(f - i0, 0.0, 1.0)
        w0 = 1.0 - w1
        v = np.zeros(len(pv))
        for dz in (0, 1):
            wz = w1[:, 2] if dz else w0[:, 2]
            for dy in (0, 1):
                wy = w1[:, 1] if dy else w0[:, 1]
                for dx in (0, 1):
                    wx = w1[:, 0] if dx else w0[:, 0]
                    v += wz * wy * wx * self.bb[slot, i0[:, 2] + dz, i0[:, 1] + dy,
                                                i0[:, 0] + dx, c].astype(np.float64)
        return v

    def _resolve(self, pv, target, chans, fullframe, cnt):
        """raycast.py:167-238."""
        idx, lvl, lo, anc1, anc2 = self._descend(pv, target)
        e = self.nb[idx]
        res = (e & np.uint64(1)) != 0
        nh = (e & np.uint64(2)) != 0
        miss = nh & ~res
        vals = np.empty((len(pv), len(chans)))
        hm, rm = np.flatnonzero(~nh), np.flatnonzero(res)
        for j, c in enumerate(chans):
            if hm.size:
                vals[hm, j] = self._avg(e[hm], c)
            if rm.size:
                vals[rm, j] = self._trilerp(e[rm], lvl[rm], lo[rm], pv[rm], c)
        self._mark(idx[rm], 1)
        cnt["bricks_used_marks"] += rm.size
        mm = np.flatnonzero(miss)
        self._mark(idx[mm], 2)
        cnt["bricks_requested"] += mm.size
        if mm.size and fullframe:
            todo = mm
            for ai, al, alo in (anc1, anc2):
                if todo.size == 0:
                    break
                ok = ai[todo] >= 0
                cand, rest = todo[ok], todo[~ok]
                if cand.size == 0:
                    todo = rest
                    continue
                ae = self.nb[ai[cand]]
                ares = (ae & np.uint64(1)) != 0
                amiss = ((ae & np.uint64(2)) != 0) & ~ares
                req = cand[amiss]
                self._mark(ai[req], 2)
                cnt["bricks_requested"] += req.size
                hit = cand[ares]
                if hit.size:
                    for j, c in enumerate(chans):
                        vals[hit, j] = self._trilerp(self.nb[ai[hit]], al[hit], alo[hit], pv[hit], c)
                    self._mark(ai[hit], 1)
                    cnt["bricks_used_marks"] += hit.size
                    cnt["coarse_fallbacks"] += hit.size
                todo = np.sort(np.concatenate([rest, cand[~ares]]))
            if todo.size:
                for j, c in enumerate(chans):
                    vals[todo, j] = self._avg(e[todo], c)
                cnt["avg_fallbacks"] += todo.size
            miss[:] = False
        return vals, miss

    def _lod(self, p, s, basis):
        cam, fwd = basis[0], basis[1]
        z = (p - cam) @ fwd
        fp = np.maximum(z, 1e-12) * (2.0 * np.tan(s.fov_y / 2.0) / s.height)
        fp = fp * (2.0 ** s.lod_bias)
        with np.errstate(divide="ignore"):
            lv = np.floor(np.log2(np.maximum(fp / self.base_voxel, 1e-300)))
        return np.clip(lv, 0, self.g.depth).astype(np.int64)

    def _sample(self, p, s, basis, fullframe, cnt):
        """raycast.py:242-278."""
        C = self.t.C
        out = np.full((len(p), C), float(self.t.bg))
        miss = np.zeros(len(p), bool)
        groups = [(list(range(C)), None)] if self.transforms is None else \
            [([c], self.transforms[c]) for c in range(C)]
        for chans, mat in groups:
            q = p if mat is None else p @ mat[:3, :3].T + mat[:3, 3]
            pv = q / self.spacing
            sel = np.flatnonzero(np.all((pv >= 0.0) & (pv <= self.dims), axis=1))
            if sel.size == 0:
                continue
            target = self._lod(q[sel], s, basis)
            v, m = self._resolve(np.clip(pv[sel], 0.0, self.dims - 1e-9), target, chans,
                                 fullframe, cnt)
            out[np.ix_(sel, chans)] = v
            miss[sel] |= m
        return out, miss

    def run(self, st, s: SceneSpec, fullframe=True, cnt=None):
        """core.py:162-187 march; returns True if any ray suspended."""
        cnt = self.new_counters() if cnt is None else cnt
        basis = camera_basis(s)
        ref = s.reference_step if s.reference_step else st["step"]
        corr = st["step"] / ref
        fmax = float(self.t.fmax)
        st["susp"][:] = False
        while True:
            idx = np.flatnonzero(~st["term"] & ~st["susp"] & (st["k"] < st["n"]))
            if idx.size == 0:
                break
            t = st["t0"][idx] + st["k"][idx] * st["step"]
            p = st["origin"] + t[:, None] * st["dirs"][idx]
            vals, miss = self._sample(p, s, basis, fullframe, cnt)
            cnt["samples"] += idx.size
            if miss.any():
                st["susp"][idx[miss]] = True
                idx, vals = idx[~miss], vals[~miss]
            if idx.size == 0:
                continue
            if s.mode == "mip":
                st["mip"][idx] = np.maximum(st["mip"][idx], vals)
            else:
                srgb = np.zeros((idx.size, 3))
                trans = np.ones(idx.size)
                for c, pts in enumerate(s.tfs):
                    rgba = tf_lookup(pts, vals[:, c] / fmax)
                    cnt["tf_lookups"] += idx.size
                    al = 1.0 - (1.0 - rgba[:, 3]) ** corr
                    srgb += rgba[:, :3] * al[:, None]
                    trans *= 1.0 - al
                np.clip(srgb, 0.0, 1.0, out=srgb)
                w = 1.0 - st["a"][idx]
                st["rgb"][idx] += w[:, None] * srgb
                st["a"][idx] += w * (1.0 - trans)
                lim = s.early_termination_alpha
                if lim is not None and lim < 1.0:
                    st["term"][idx] |= st["a"][idx] >= lim
            st["k"][idx] += 1
        return bool(st["susp"].any()), cnt

    def image(self, st, s: SceneSpec, cnt=None):
        """core.py:137-155."""
        if s.mode == "mip":
            n = len(st["mip"])
            rgb = np.zeros((n, 3))
            trans = np.ones(n)
            for c, pts in enumerate(s.tfs):
                rgba = tf_lookup(pts, st["mip"][:, c] / float(self.t.fmax))
                if cnt is not None:
                    cnt["tf_lookups"] += n
                rgb += rgba[:, :3] * rgba[:, 3:4]
                trans *= 1.0 - rgba[:, 3]
            np.clip(rgb, 0.0, 1.0, out=rgb)
            flat = np.concatenate([rgb, (1.0 - trans)[:, None]], axis=1)
        else:
            flat = np.concatenate([st["rgb"], st["a"][:, None]], axis=1)
        return flat.reshape(s.height, s.width, 4)

    def render_fullframe(self, s: SceneSpec, tile=None):
        st = self.start(s, tile)
        _, cnt = self.run(st, s, True)
        return self.image(st, s, cnt), cnt


def render_reference_volume(volume, t: OracleTree, s: SceneSpec):
    """In-core level-0 oracle (render/oracle.py:26-88): background-padded
    volume, f = pvox + 0.5, same march/composite."""
    if volume.ndim == 3:
        volume = volume[..., None]
    padded = np.pad(volume, ((1, 1), (1, 1), (1, 1), (0, 0)), constant_values=t.bg)

    class _Vol(OracleRenderer):
        def _sample(self, p, s, basis, fullframe, cnt):
            out = np.full((len(p), self.t.C), float(self.t.bg))
            for c in range(self.t.C):
                q = p if self.transforms is None else \
                    p @ self.transforms[c][:3, :3].T + self.transforms[c][:3, 3]
                pv = q / self.spacing
                sel = np.flatnonzero(np.all((pv >= 0.0) & (pv <= self.dims), axis=1))
                if sel.size == 0:
                    continue
                f = pv[sel] + 0.5
                i0 = np.clip(np.floor(f).astype(np.int64), 0, self.dims.astype(np.int64))
                w1 = np.clip(f - i0, 0.0, 1.0)
                w0 = 1.0 - w1
                v = np.zeros(sel.size)
                for dz in (0, 1):
                    wz = w1[:, 2] if dz else w0[:, 2]
                    for dy in (0, 1):
                        wy = w1[:, 1] if dy else w0[:, 1]
                        for dx in (0, 1):
                            wx = w1[:, 0] if dx else w0[:, 0]
                            v += wz * wy * wx * padded[i0[:, 2] + dz, i0[:, 1] + dy,
                                                       i0[:, 0] + dx, c].astype(np.float64)
                out[sel, c] = v
            return out, np.zeros(len(p), bool)

    r = _Vol(t, None, None)
    st = r.start(s)
    r.run(st, s, True)
    return r.image(st, s)


# ---------------------------------------------------------------------------
# synthetic volumes (shared integer formula; CUDA twin in the product's
# synth kernel, hash-checked in tests)
# ---------------------------------------------------------------------------

_M32 = np.uint64(0xFFFFFFFF)


def hash4(x, y, z, c, seed):
    """32-bit integer mix of (x, y, z, c, seed) — identical bit ops in CUDA."""
    h = (np.asarray(x, np.uint64) * np.uint64(0x9E3779B1)) & _M32
    h ^= (np.asarray(y, np.uint64) * np.uint64(0x85EBCA77)) & _M32
    h = (h * np.uint64(0xC2B2AE3D)) & _M32
    h ^= (np.asarray(z, np.uint64) * np.uint64(0x27D4EB2F)) & _M32
    h ^= (np.asarray(c, np.uint64) * np.uint64(0x165667B1) + np.uint64(seed)) & _M32
    h ^= h >> np.uint64(15)
    h = (h * np.uint64(0x2C1B3C6D)) & _M32
    h ^= h >> np.uint64(12)
    h = (h * np.uint64(0x297A2D39)) & _M32
    h ^= h >> np.uint64(15)
    return h


def synth_uniform(dims, C, fmax, seed=0, z0=0, z1=None):
    """'U' data: hash & fmax — x-fastest (z, y, x, C) for z in [z0, z1)."""
    dx, dy, dz = dims
    z1 = dz if z1 is None else z1
    z, y, x = np.meshgrid(np.arange(z0, z1), np.arange(dy), np.arange(dx), indexing="ij")
    out = np.empty((z1 - z0, dy, dx, C), dtype=np.uint8 if fmax == 255 else np.uint16)
    for c in range(C):
        out[..., c] = (hash4(x, y, z, c, seed) % np.uint64(fmax + 1)).astype(out.dtype)
    return out


def synth_spim(dims, C, fmax, seed=0, z0=0, z1=None, y0=0, y1=None, x0=0, x1=None):
    """'S' data: integer-only SPIM-like specimen: noisy
    background, ellipsoidal specimen, per-channel blob lattice of 32^3 cells.
    Returns the sub-box [z0, z1) x [y0, y1) x [x0, x1) of the volume of
    extent ``dims`` (a crop keeps the full volume's specimen geometry)."""
    dx, dy, dz = dims
    z1 = dz if z1 is None else z1
    y1 = dy if y1 is None else y1
    x1 = dx if x1 is None else x1
    z, y, x = np.meshgrid(np.arange(z0, z1, dtype=np.int64), np.arange(y0, y1, dtype=np.int64),
                          np.arange(x0, x1, dtype=np.int64), indexing="ij")
    big = fmax > 255
    amp = 40000 if big else 220
    base = 100 if big else 8
    noise_mask = 15 if big else 3
    out = np.empty((z1 - z0, y1 - y0, x1 - x0, C), dtype=np.uint16 if big else np.uint8)
    # ellipsoid: sum((2p - d)^2 * 400 / d^2) <= 81*4 ... integer form
    ex = (2 * x - dx) ** 2 * 10000 // max(dx * dx, 1)
    ey = (2 * y - dy) ** 2 * 10000 // max(dy * dy, 1)
    ez = (2 * z - dz) ** 2 * 10000 // max(dz * dz, 1)
    inside = (ex + ey + ez) <= 8100  # semi-axes 0.45 * dims
    cx, cy, cz = x >> 5, y >> 5, z >> 5
    lx, ly, lz = (x & 31) - 16, (y & 31) - 16, (z & 31) - 16
    d2 = lx * lx + ly * ly + lz * lz
    for c in range(C):
        v = base + (hash4(x, y, z, c, seed) & np.uint64(noise_mask)).astype(np.int64)
        hc = hash4(cx, cy, cz, c + 7, seed)
        has = (hc % np.uint64(4)) == 0
        r = 4 + ((hc >> np.uint64(8)) % np.uint64(9)).astype(np.int64)
        r2 = r * r
        blob = amp * np.maximum(0, r2 - d2) // r2
        v = v + np.where(inside & has, blob, 0)
        out[..., c] = np.clip(v, 0, fmax).astype(out.dtype)
    return out
