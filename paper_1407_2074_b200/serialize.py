"""VXOC metadata + canonical VXBP pool export/import — the reference's
persistence format (serialize.py:61-206, paging.py:60-380), written from a
device tree through vt_tree_export / read through vt_tree_import.

Byte layout is the reference's, so a tree built on the GPU and one built by
voxtree from the same insertion sequence serialize to identical files
(the digest parity harness).  Bricks are copied out of HBM in batches; the
page CRCs and bitmap are computed here on the host (file I/O is host work).
"""

from __future__ import annotations

import os
import struct
import tempfile
import zlib

import numpy as np

from . import _lib
from .octree import Octree
from .volume import BrickPoolConfig, VolumeDescriptor

MAGIC = b"VXOC"
VERSION = 1
POOL_MAGIC = b"VXBP"

_HEAD = struct.Struct("<4sI")
_DESC = struct.Struct("<3IHH3dIB3x")
_CONF = struct.Struct("<3IdIII")
_TREE = struct.Struct("<IQ")
_NODE = struct.Struct("<QBB2x")
_CHAN = struct.Struct("<5I")
_LOC = struct.Struct("<II")
_POOL_HEAD = struct.Struct("<4sIIQIIIHHQQ12x")
_CRC = struct.Struct("<I")
_NO_BRICK = 0xFFFFFFFF
_FMT_CODES = {"uint8": 1, "uint16": 2}
_FMT_NAMES = {v: k for k, v in _FMT_CODES.items()}
_F_TRANSFORMS, _F_FINISHED, _F_BORDERS = 1, 2, 4
_N_BRICK, _N_CHILDREN, _N_INVOL = 1, 2, 4


def _write_atomic(path, chunks) -> None:
    folder = os.path.dirname(os.path.abspath(path)) or "."
    fd, tmp = tempfile.mkstemp(dir=folder, prefix=".vx-")
    try:
        with os.fdopen(fd, "wb") as fh:
            for c in chunks:
                fh.write(c)
            fh.flush()
            os.fsync(fh.fileno())
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _pool_chunks(n, batches, page_bricks: int, brick_shape, channels: int, dtype):
    """Chunks of a freshly written, flushed VXBP holding n bricks, taken in
    order from ``batches`` (arrays of whole bricks) — BrickStore.create +
    allocate/write_brick + flush, paging.py:120-380."""
    dt = np.dtype(dtype).newbyteorder("<")
    nbytes = int(np.prod(brick_shape)) * channels * dt.itemsize
    pages = -(-n // page_bricks)
    stride = page_bricks * nbytes + _CRC.size
    footer = _POOL_HEAD.size + pages * stride if pages else 0
    yield _POOL_HEAD.pack(POOL_MAGIC, 1, page_bricks, nbytes, *brick_shape, channels,
                          _FMT_CODES[np.dtype(dtype).name], pages, footer)
    page, cur, done = bytearray(), 0, 0
    for b in batches:
        flat = np.ascontiguousarray(b, dtype=dt).reshape(len(b), -1).view(np.uint8)
        pos = 0
        while pos < len(flat):
            take = min(page_bricks - cur, len(flat) - pos)
            page += flat[pos:pos + take].tobytes()
            cur += take
            pos += take
            done += take
            if cur == page_bricks:
                yield bytes(page)
                yield _CRC.pack(zlib.crc32(page))
                page, cur = bytearray(), 0
    if page:
        page += bytes(page_bricks * nbytes - len(page))
        yield bytes(page)
        yield _CRC.pack(zlib.crc32(page))
    assert done == n, (done, n)
    if pages:
        bits = np.zeros(pages * page_bricks, np.uint8)
        bits[:n] = 1
        yield np.packbits(bits, bitorder="little").tobytes()


def pool_bytes(bricks: np.ndarray, page_bricks: int, brick_shape, channels: int, dtype):
    """Chunks of a freshly written, flushed VXBP holding ``bricks`` in order."""
    return list(_pool_chunks(len(bricks), [bricks] if len(bricks) else [], page_bricks,
                             brick_shape, channels, dtype))


def _octree_chunks(tree: Octree, idx, flags, stats):
    """VXOC metadata chunks (serialize.py:92-124)."""
    desc, cfg = tree.descriptor, tree.config
    hdr = 0
    if desc.channel_transforms is not None:
        hdr |= _F_TRANSFORMS
    if tree.construction_finished:
        hdr |= _F_FINISHED
    if tree.borders_filled:
        hdr |= _F_BORDERS
    parts = [_HEAD.pack(MAGIC, VERSION),
             _DESC.pack(*desc.dims, desc.channels, _FMT_CODES[desc.sample_format],
                        *desc.spacing, desc.background_value, hdr)]
    if desc.channel_transforms is not None:
        parts.append(np.asarray(desc.channel_transforms, dtype="<f8").tobytes())
    parts.append(_CONF.pack(*cfg.brick_dims, tree.threshold, cfg.overlap,
                            cfg.page_bricks, cfg.ram_page_limit))
    parts.append(_TREE.pack(tree.geometry.depth, len(idx)))
    geo = tree.geometry
    canon = 0
    for r, i in enumerate(idx):
        f = int(flags[r])
        nf = (_N_BRICK if f & _lib.NODE_BRICK else 0) | \
            (_N_CHILDREN if f & _lib.NODE_CHILDREN else 0) | \
            (_N_INVOL if f & _lib.NODE_IN_VOLUME else 0)
        parts.append(_NODE.pack(int(i), geo.level_of_index(int(i)), nf))
        inv = bool(f & _lib.NODE_IN_VOLUME)
        for c in range(desc.channels):
            a, lo, hi, slo, shi = (int(v) for v in stats[r, c])
            parts.append(_CHAN.pack(lo, hi, a, slo if inv else 0, shi if inv else 0))
        if f & _lib.NODE_BRICK:
            parts.append(_LOC.pack(*divmod(canon, cfg.page_bricks)))
            canon += 1
        else:
            parts.append(_LOC.pack(_NO_BRICK, _NO_BRICK))
    return parts


def _brick_batches(tree: Octree, bricked, batch: int):
    for k in range(0, len(bricked), batch):
        yield tree.export(indices=bricked[k:k + batch])[3]


def save_octree(tree: Octree, octree_path, pool_path, *, batch: int = 4096) -> None:
    """Persist the tree and a canonically compacted copy of its pool
    (serialize.py:61-125); bricks leave HBM in batches."""
    desc, cfg = tree.descriptor, tree.config
    with tree.lock:
        idx, flags, stats, _ = tree.export(with_bricks=False)
        bricked = idx[(flags & _lib.NODE_BRICK) != 0]
        _write_atomic(pool_path, _pool_chunks(len(bricked), _brick_batches(tree, bricked, batch),
                                              cfg.page_bricks,
                                              tuple(reversed(cfg.stored_brick_dims)),
                                              desc.channels, desc.dtype))
        _write_atomic(octree_path, _octree_chunks(tree, idx, flags, stats))


def octree_digests(tree: Octree, *, batch: int = 4096) -> tuple[str, str]:
    """sha256 of the VXOC and VXBP files save_octree would write, without
    writing them (the digest parity harness at BASELINE sizes)."""
    import hashlib
    desc, cfg = tree.descriptor, tree.config
    with tree.lock:
        idx, flags, stats, _ = tree.export(with_bricks=False)
        bricked = idx[(flags & _lib.NODE_BRICK) != 0]
        hp = hashlib.sha256()
        for c in _pool_chunks(len(bricked), _brick_batches(tree, bricked, batch), cfg.page_bricks,
                              tuple(reversed(cfg.stored_brick_dims)), desc.channels, desc.dtype):
            hp.update(c)
        ho = hashlib.sha256()
        for c in _octree_chunks(tree, idx, flags, stats):
            ho.update(c)
        return ho.hexdigest(), hp.hexdigest()


def load_octree(octree_path, pool_path, *, ram_page_limit: int | None = None,
                device: int = 0) -> Octree:
    """Rebuild a device tree from VXOC + VXBP (serialize.py:128-206)."""
    with open(octree_path, "rb") as fh:
        raw = fh.read()
    off = 0
    magic, version = _HEAD.unpack_from(raw, off)
    off += _HEAD.size
    if magic != MAGIC:
        raise ValueError(f"{octree_path} is not an octree metadata file")
    if version != VERSION:
        raise ValueError(f"unsupported octree file version {version}")
    dx, dy, dz, nc, fmt, sx, sy, sz, bg, hdr = _DESC.unpack_from(raw, off)
    off += _DESC.size
    transforms = None
    if hdr & _F_TRANSFORMS:
        transforms = np.frombuffer(raw, "<f8", nc * 16, off).reshape(nc, 4, 4).copy()
        off += nc * 128
    desc = VolumeDescriptor(dims=(dx, dy, dz), channels=nc, sample_format=_FMT_NAMES[fmt],
                            spacing=(sx, sy, sz), background_value=bg,
                            channel_transforms=transforms)
    bx, by, bz, thr, overlap, page_bricks, ram_pages = _CONF.unpack_from(raw, off)
    off += _CONF.size
    # the file's ram_page_limit is kept (it is part of the VXOC header); the
    # reference passes an override only to its paging store's RAM cache
    # (serialize.py:128-206), which the HBM pool does not have, so the
    # argument is accepted and ignored
    del ram_page_limit
    cfg = BrickPoolConfig(brick_dims=(bx, by, bz), homogeneity_threshold=thr, overlap=overlap,
                          page_bricks=page_bricks, ram_page_limit=ram_pages)
    depth, count = _TREE.unpack_from(raw, off)
    off += _TREE.size
    idx = np.empty(count, np.int64)
    flags = np.empty(count, np.int32)
    stats = np.empty((count, nc, 5), np.int32)
    locs = []
    for r in range(count):
        i, _lvl, nf = _NODE.unpack_from(raw, off)
        off += _NODE.size
        idx[r] = i
        flags[r] = (_lib.NODE_EXISTS | (_lib.NODE_BRICK if nf & _N_BRICK else 0) |
                    (_lib.NODE_CHILDREN if nf & _N_CHILDREN else 0) |
                    (_lib.NODE_IN_VOLUME if nf & _N_INVOL else 0))
        for c in range(nc):
            lo, hi, a, slo, shi = _CHAN.unpack_from(raw, off)
            off += _CHAN.size
            stats[r, c] = (a, lo, hi, slo, shi)
        page, slot = _LOC.unpack_from(raw, off)
        off += _LOC.size
        if nf & _N_BRICK:
            locs.append((page, slot))
    bricks = _read_pool(pool_path, locs, desc, cfg)
    tree = Octree(desc, cfg, None, device=device, reserve_slots=max(1, len(locs)))
    if tree.geometry.depth != depth:
        raise ValueError("octree depth mismatch with descriptor/config")
    import ctypes as ct
    _lib.call("vt_tree_import", tree.handle, count, _lib.ptr(idx, ct.c_int64),
              _lib.ptr(flags, ct.c_int32),
              _lib.ptr(np.ascontiguousarray(stats), ct.c_int32),
              ct.c_void_p(bricks.ctypes.data) if len(locs) else None,
              1 if hdr & _F_FINISHED else 0, 1 if hdr & _F_BORDERS else 0, 0)
    return tree


def _read_pool(path, locs, desc, cfg):
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _POOL_HEAD.size:
        raise _lib.StoreIOError("brick pool header truncated")
    (magic, version, page_bricks, nbytes, bz, by, bx, nc, code, pages,
     _footer) = _POOL_HEAD.unpack_from(raw, 0)
    if magic != POOL_MAGIC:
        raise _lib.StoreIOError("not a brick pool file")
    if version != 1:
        raise _lib.StoreIOError(f"unsupported brick pool version {version}")
    dt = np.dtype(_FMT_NAMES.get(code, "uint8")).newbyteorder("<")
    stride = page_bricks * nbytes + _CRC.size
    out = np.empty((len(locs), bz, by, bx, nc), dtype=desc.dtype)
    checked = set()
    for r, (page, slot) in enumerate(locs):
        base = _POOL_HEAD.size + page * stride
        if page not in checked:
            body = raw[base:base + page_bricks * nbytes]
            (crc,) = _CRC.unpack_from(raw, base + page_bricks * nbytes)
            if len(body) < page_bricks * nbytes or zlib.crc32(body) != crc:
                raise _lib.StoreIOError(f"page {page} checksum mismatch")
            checked.add(page)
        b = raw[base + slot * nbytes: base + (slot + 1) * nbytes]
        out[r] = np.frombuffer(b, dt).reshape(bz, by, bx, nc)
    return out
