"""z-slab sharded octree build across the GPUs of one node (the
reference has no multi-process build — ``ingest_bulk`` runs one thread per
channel behind ``Octree.lock``, ingest.py:182-224).

Every rank holds a tree with the full geometry.  The volume's z extent is cut
into contiguous slabs of whole level-k node layers, k the highest level with
at least one layer per rank, so every node at a level <= k lies inside one
slab.  Each rank inserts only its slab: its nodes at levels <= k are then
final (at homogeneity threshold 0 every brick is a pure function of the data
under it).  One exchange — an all-gather of those node records (flags,
statistics, bricks) — gives every rank the complete set of level <= k
subtrees; ``vt_tree_merge`` splices the foreign ones in and recomputes every
ancestor above level k from all of its children, so each rank ends with the
tree a single-GPU build of the whole volume produces, byte for byte
(borders are filled afterwards on the merged tree).  The result is the
replicated pool sort-first rendering needs.

Threshold > 0 is refused: pruning is history dependent and
only the sequential insertion order defines it.
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np

from . import _lib

_STATS = 5


@dataclass(frozen=True)
class SlabPlan:
    level: int                      # k: nodes at levels <= k are slab-local
    layer_voxels: int               # z extent of one level-k node
    slabs: tuple                    # per rank: (z0, z1) voxel range (may be empty)


def slab_plan(geometry, world: int) -> SlabPlan:
    """Largest k with >= world level-k layers over the volume's z extent;
    layers are dealt out contiguously (rank r gets layers [r L / G, (r+1) L / G))."""
    dz = geometry.dims[2]
    mz = geometry.brick_dims[2]
    split_z = geometry.virtual[2] > mz
    best = 0
    if split_z:
        for k in range(geometry.depth + 1):
            layers = -(-dz // (mz << k))
            if layers >= world:
                best = k
    ext = (mz << best) if split_z else mz
    layers = -(-dz // ext)
    slabs = []
    for r in range(world):
        l0, l1 = r * layers // world, (r + 1) * layers // world
        slabs.append((min(dz, l0 * ext), min(dz, l1 * ext)))
    return SlabPlan(best, ext, tuple(slabs))


def _levels_and_z(geometry, idx: np.ndarray):
    """Vectorised level and box z-origin (level-0 voxels) of BFS indices."""
    idx = np.asarray(idx, np.int64)
    starts = [(8 ** d - 1) // 7 for d in range(geometry.depth + 2)]
    d = np.searchsorted(np.asarray(starts[1:]), idx, side="right")
    level = geometry.depth - d
    z = np.zeros_like(idx)
    cur = idx.copy()
    lvl = level.copy()
    mz = geometry.brick_dims[2]
    split_z = geometry.virtual[2] > mz
    for _ in range(geometry.depth):
        live = cur > 0
        k = (cur - 1) & 7
        if split_z:
            z += np.where(live & ((k >> 2) & 1).astype(bool), mz << lvl, 0)
        cur = np.where(live, (cur - 1) >> 3, 0)
        lvl = np.where(live, lvl + 1, lvl)
    return level, z


def slab_records(tree, plan: SlabPlan, z0: int, z1: int):
    """Indices of this rank's final nodes: levels <= k inside [z0, z1)."""
    idx = tree.node_indices()
    if z1 <= z0:
        return idx[:0]
    level, z = _levels_and_z(tree.geometry, idx)
    keep = (level <= plan.level) & (z >= z0) & (z < z1) & (idx > 0)
    return idx[keep]


def export_records(tree, indices, device_bricks: bool = True):
    """(indices, VT_NODE_* flags, stats (n, C, 5) int32, bricks) with the
    bricks of the bricked records in record order — a CUDA uint8 tensor
    (device_bricks) or a numpy array."""
    idx = np.ascontiguousarray(indices, np.int64)
    n = len(idx)
    C = tree.descriptor.channels
    flags = np.empty(n, np.int32)
    stats = np.empty((n, C, _STATS), np.int32)
    _lib.call("vt_tree_export_nodes", tree.handle, n, _lib.ptr(idx, ct.c_int64),
              _lib.ptr(flags, ct.c_int32), _lib.ptr(stats, ct.c_int32), None, 0)
    nb = int(np.count_nonzero(flags & _lib.NODE_BRICK))
    bb = tree.config.brick_nbytes(tree.descriptor)
    if device_bricks:
        import torch
        bricks = torch.empty(max(1, nb) * bb, dtype=torch.uint8, device="cuda")
        ptr, kind = ct.c_void_p(bricks.data_ptr()), _lib.VT_MEM_DEVICE
    else:
        bricks = np.empty(max(1, nb) * bb, np.uint8)
        ptr, kind = ct.c_void_p(bricks.ctypes.data), _lib.VT_MEM_HOST
    if nb:
        _lib.call("vt_tree_export_nodes", tree.handle, n, _lib.ptr(idx, ct.c_int64), None, None,
                  ptr, kind)
    return idx, flags, stats, bricks[:nb * bb]


def merge_records(tree, idx, flags, stats, bricks, inserted_voxels: int = 0) -> None:
    """Splice records (``export_records`` layout) into ``tree`` and recompute
    all levels above them (vt_tree_merge)."""
    idx = np.ascontiguousarray(idx, np.int64)
    flags = np.ascontiguousarray(flags, np.int32)
    stats = np.ascontiguousarray(stats, np.int32)
    if hasattr(bricks, "data_ptr"):
        ptr, kind = ct.c_void_p(bricks.data_ptr() if bricks.numel() else 0), _lib.VT_MEM_DEVICE
    else:
        bricks = np.ascontiguousarray(bricks)
        ptr, kind = ct.c_void_p(bricks.ctypes.data if bricks.size else 0), _lib.VT_MEM_HOST
    with tree.lock:
        _lib.call("vt_tree_merge", tree.handle, len(idx), _lib.ptr(idx, ct.c_int64),
                  _lib.ptr(flags, ct.c_int32), _lib.ptr(stats, ct.c_int32), ptr, kind,
                  int(inserted_voxels))


def build_sharded(tree, source, group=None, slab_z=32, fill_borders=True) -> SlabPlan:
    """Build ``tree`` on every rank of ``group`` from ``source(z0, z1)`` —
    a callable returning the (z1 - z0, Y, X, C) block of the volume (device
    tensor or numpy) — inserting only this rank's slab, then exchanging node
    records with one all-gather over NCCL (see module doc)."""
    import torch
    import torch.distributed as dist
    if tree.threshold > 0:
        raise ValueError("the z-slab sharded build needs homogeneity threshold 0 "
                         "(pruning is defined by the sequential insertion order)")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    plan = slab_plan(tree.geometry, world)
    z0, z1 = plan.slabs[rank]
    for z in range(z0, z1, slab_z):
        tree.insert_channels((0, 0, z), source(z, min(z1, z + slab_z)))
    tree.sync()
    if world > 1:
        own = slab_records(tree, plan, z0, z1)
        idx, flags, stats, bricks = export_records(tree, own)
        ins = tree.inserted_voxels
        parts = _all_gather_records(idx, flags, stats, bricks, ins, tree, group)
        others = [p for r, p in enumerate(parts) if r != rank]
        if others:
            cat = lambda k: np.concatenate([p[k] for p in others])  # noqa: E731
            merge_records(tree, cat(0), cat(1), cat(2),
                          torch.cat([p[3] for p in others]) if others else bricks,
                          sum(p[4] for p in others))
    if fill_borders:
        tree.finalize()
        tree.fill_borders()
    tree.sync()
    return plan


def _all_gather_records(idx, flags, stats, bricks, inserted, tree, group):
    """One all-gather of every rank's records (padded to the largest)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out_dev = bricks.device
    # NCCL exchanges device buffers; other backends (gloo tests) via host
    dev = out_dev if dist.get_backend(group) == "nccl" else torch.device("cpu")
    bricks = bricks.to(dev)
    C = tree.descriptor.channels
    bb = tree.config.brick_nbytes(tree.descriptor)
    meta = torch.tensor([len(idx), bricks.numel() // bb, inserted], dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    metas = [m.tolist() for m in metas]
    nmax = max(m[0] for m in metas)
    bmax = max(m[1] for m in metas)
    rec = torch.zeros((nmax, 2 + C * _STATS), dtype=torch.int64, device=dev)
    n = len(idx)
    if n:
        rec[:n, 0] = torch.as_tensor(idx, device=dev)
        rec[:n, 1] = torch.as_tensor(flags.astype(np.int64), device=dev)
        rec[:n, 2:] = torch.as_tensor(stats.reshape(n, -1).astype(np.int64), device=dev)
    recs = torch.empty((world * rec.shape[0], rec.shape[1]), dtype=rec.dtype, device=dev)
    dist.all_gather_into_tensor(recs, rec, group=group)
    recs = recs.reshape((world,) + tuple(rec.shape))
    pad = torch.zeros(max(1, bmax) * bb, dtype=torch.uint8, device=dev)
    pad[:bricks.numel()] = bricks
    allb = torch.empty(world * pad.numel(), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(allb, pad, group=group)
    allb = allb.reshape(world, pad.numel())
    out = []
    recs = recs.cpu().numpy()
    for r, (nr, br, ins) in enumerate(metas):
        rr = recs[r, :nr]
        out.append((rr[:, 0].astype(np.int64), rr[:, 1].astype(np.int32),
                    rr[:, 2:].astype(np.int32).reshape(nr, C, _STATS),
                    allb[r, :br * bb].to(out_dev), ins))
    return out
