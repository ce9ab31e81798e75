"""Incremental octree over a device-resident (HBM) brick pool — drop-in for
voxtree.octree (octree.py:143-614).

``Octree`` keeps the reference's constructor, ``insert_block`` /
``finalize`` / ``fill_borders`` / ``drain_events`` / ``find_node`` /
``node_by_index`` / ``iter_nodes`` API, exceptions and events.  All data
work runs in libvtx (csrc/): the host keeps only the lock the reference
holds (octree.py:153) and the event list.  Node objects returned by the
queries are snapshots (the reference hands out live objects; callers in the
reference only read them).
"""

from __future__ import annotations

import ctypes as ct
import os
import sys
import threading
from collections.abc import Sequence
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _lib
from .volume import BrickPoolConfig, TreeGeometry, VolumeDescriptor


class ChangeKind(IntEnum):
    NODE_CREATED = 1
    NODE_DELETED = 2
    NODE_UPDATED = 3


@dataclass(frozen=True)
class ChangeEvent:
    kind: ChangeKind
    node_index: int


@dataclass(frozen=True)
class BrickLocator:
    """Handle of a node's brick: the node index plus its HBM pool slot."""
    node_index: int
    slot: int


def round_mean(sums, counts):
    """(2*sum + n) // (2n), ties up (octree.py:53-55) — host helper for
    scalar bookkeeping; the bulk means are computed on the device."""
    s = np.asarray(sums, dtype=np.int64)
    n = np.asarray(counts, dtype=np.int64)
    return (2 * s + n) // (2 * n)


def halfsample_block(values: np.ndarray, in_extent, split, background: int) -> np.ndarray:
    """halfsample_block (octree.py:58-92) executed by the device kernel."""
    v = np.ascontiguousarray(values, dtype=np.int32)
    if v.ndim != 4:
        raise ValueError("values must be (mz, my, mx, C)")
    mz, my, mx, nc = v.shape
    k = [2 if s else 1 for s in split]
    out = np.empty((mz // k[2], my // k[1], mx // k[0], nc), dtype=np.int32)
    shape = (ct.c_int32 * 4)(mz, my, mx, nc)
    _lib.call("vt_halfsample", _lib.ptr(v, ct.c_int32), shape, _lib.i32x3(in_extent),
              _lib.i32x3([1 if s else 0 for s in split]), int(background),
              _lib.ptr(out, ct.c_int32), 0)
    return out.astype(np.int64)


def classify_homogeneous(smin, smax, threshold: float):
    """Per-channel ``max - min < threshold`` and the overall verdict
    (octree.py:95-99)."""
    per = [(hi - lo) < threshold for lo, hi in zip(smin, smax)]
    return per, all(per)


_EV_TABLES: dict = {}  # ChangeKind value -> object array of interned events by node index


def _event_table(kind: int, n: int) -> np.ndarray:
    tbl = _EV_TABLES.get(kind)
    if tbl is None or len(tbl) < n:
        new = np.empty(max(n, 2 * (0 if tbl is None else len(tbl)), 1024), dtype=object)
        if tbl is not None:
            new[:len(tbl)] = tbl
        _EV_TABLES[kind] = tbl = new
    return tbl


def _events_from_arrays(kinds: np.ndarray, idx: np.ndarray) -> list:
    """ChangeEvent objects for packed (kind, index) arrays.  ChangeEvent is a
    frozen dataclass, so equal events can be shared: each (kind, index) is
    built once per process and a batch is a vectorised gather."""
    n = len(kinds)
    if n == 0:
        return []
    out = np.empty(n, dtype=object)
    for k in np.unique(kinds).tolist():
        m = kinds == k
        ii = idx[m]
        tbl = _event_table(k, int(ii.max()) + 1)
        vals = tbl[ii]
        miss = np.flatnonzero(np.equal(vals, None))
        if miss.size:
            kind = ChangeKind(k)
            for u in np.unique(ii[miss]).tolist():
                tbl[u] = ChangeEvent(kind, u)
            vals = tbl[ii]
        out[m] = vals
    return out.tolist()


class EventList(list):
    """What insert_block / drain_events return (octree.py:180-183, 393-395):
    a real ``list`` of ChangeEvent.  The library's packed form is kept as
    ``kinds`` / ``indices`` numpy arrays (B200 extension for bulk consumers
    such as DeviceState.apply_events); any in-place change of the list
    recomputes them from the elements."""

    def __init__(self, items=(), *, kinds=None, indices=None):
        if kinds is not None:
            kinds = np.asarray(kinds, np.int32)
            indices = np.asarray(indices, np.int64)
            super().__init__(_events_from_arrays(kinds, indices))
            self._arr = (kinds, indices)
        else:
            super().__init__(items)
            self._arr = None

    @classmethod
    def from_arrays(cls, kinds, indices) -> "EventList":
        return cls(kinds=kinds, indices=indices)

    @staticmethod
    def concat(batches) -> "EventList":
        batches = [b for b in batches if len(b)]
        if not batches:
            return EventList()
        if len(batches) == 1:
            return batches[0]
        return EventList.from_arrays(np.concatenate([b.kinds for b in batches]),
                                     np.concatenate([b.indices for b in batches]))

    def _arrays(self):
        if self._arr is None or len(self._arr[0]) != len(self):
            self._arr = (np.fromiter((int(e.kind) for e in self), np.int32, len(self)),
                         np.fromiter((int(e.node_index) for e in self), np.int64, len(self)))
        return self._arr

    @property
    def kinds(self) -> np.ndarray:
        return self._arrays()[0]

    @property
    def indices(self) -> np.ndarray:
        return self._arrays()[1]

    def _dirty(self):
        self._arr = None


def _mutator(name):
    base = getattr(list, name)

    def fn(self, *a, **kw):
        self._arr = None
        return base(self, *a, **kw)
    fn.__name__ = name
    return fn


for _m in ("__setitem__", "__delitem__", "__iadd__", "__imul__", "append", "extend", "insert",
           "pop", "remove", "clear", "sort", "reverse"):
    setattr(EventList, _m, _mutator(_m))

EventBatch = EventList  # round-1 name


class EventArrays(Sequence):
    """The change events of a bulk B200 insertion (insert_channels): a
    read-only sequence of ChangeEvent over the packed ``kinds`` /
    ``indices`` arrays, so a whole-volume insertion (hundreds of thousands
    of events) costs no Python objects until a caller iterates it.  The
    reference-API calls (insert_block, drain_events) return EventList."""

    __slots__ = ("kinds", "indices")

    def __init__(self, kinds, indices):
        self.kinds = np.asarray(kinds, np.int32)
        self.indices = np.asarray(indices, np.int64)

    def __len__(self):
        return len(self.kinds)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return EventArrays(self.kinds[i], self.indices[i])
        return ChangeEvent(ChangeKind(int(self.kinds[i])), int(self.indices[i]))

    def __eq__(self, other):
        if isinstance(other, (EventArrays, EventList)):
            return (np.array_equal(self.kinds, other.kinds)
                    and np.array_equal(self.indices, other.indices))
        try:
            return list(self) == list(other)
        except TypeError:
            return NotImplemented

    def to_list(self) -> "EventList":
        return EventList.from_arrays(self.kinds, self.indices)

    def __repr__(self):
        return f"EventArrays({len(self)} events)"


class OctreeNode:
    """Snapshot of one node (OctreeNode, octree.py:102-140)."""

    __slots__ = ("_tree", "level", "index", "box_lo", "avg", "smin", "smax", "sub_min",
                 "sub_max", "in_volume", "_flags", "_slot")

    def __init__(self, tree: "Octree", index: int, rec: _lib.vt_node):
        C = tree.descriptor.channels
        self._tree = tree
        self.index = index
        self.level = int(rec.level)
        self.box_lo = tuple(int(v) for v in rec.box_lo)
        self._flags = int(rec.flags)
        self._slot = int(rec.slot)
        st = [[int(rec.stats[c][s]) for s in range(5)] for c in range(C)]
        self.avg = [st[c][0] for c in range(C)]
        self.smin = [st[c][1] for c in range(C)]
        self.smax = [st[c][2] for c in range(C)]
        self.in_volume = bool(self._flags & _lib.NODE_IN_VOLUME)
        self.sub_min = [st[c][3] for c in range(C)] if self.in_volume else None
        self.sub_max = [st[c][4] for c in range(C)] if self.in_volume else None

    @property
    def brick(self):
        return BrickLocator(self.index, self._slot) if self._flags & _lib.NODE_BRICK else None

    @property
    def has_children(self) -> bool:
        return bool(self._flags & _lib.NODE_CHILDREN)

    @property
    def children(self):
        if not self.has_children:
            return None
        geo = self._tree.geometry
        out = [None] * 8
        for k in geo.real_octants:
            out[k] = self._tree.node_by_index(8 * self.index + 1 + k)
        return out

    def child_nodes(self):
        return [c for c in (self.children or []) if c is not None]

    def __repr__(self):
        kind = "brick" if self.brick else "avg"
        return f"<node {self.index} L{self.level} {kind} avg={self.avg}>"


class _BrickHandle:
    """BrickHandle (paging.py:54-60) over the HBM pool."""

    __slots__ = ("_store", "loc")

    def __init__(self, store: "_PoolView", loc: BrickLocator):
        self._store, self.loc = store, loc

    @property
    def data(self) -> np.ndarray:
        return self._store.read_brick(self.loc)


class _PoolView:
    """``tree.store`` facade: brick reads go to HBM (BrickStore.read_brick,
    paging.py:398-403)."""

    page_faults = 0  # the pool is HBM-resident: nothing is ever paged in

    def __init__(self, tree: "Octree"):
        self._tree = tree

    def read_brick(self, loc: BrickLocator) -> np.ndarray:
        return self._tree.read_brick(loc.node_index)

    def acquire(self, loc: BrickLocator, blocking: bool = True) -> "_BrickHandle":
        """BrickStore.acquire (paging.py:248-290): every brick of the HBM
        pool is always available, so this never returns None; the handle's
        ``data`` reads the brick on demand (DeviceState.upload_bricks copies
        pool -> brick buffer on the device and never touches it)."""
        return _BrickHandle(self, loc)

    def release(self, handle: "_BrickHandle") -> None:
        pass

    @property
    def live_bricks(self) -> int:
        return self._tree.brick_count

    @property
    def payload_nbytes(self) -> int:
        t = self._tree
        return t.brick_count * t.config.brick_nbytes(t.descriptor)

    def close(self) -> None:
        pass


class Octree:
    """Incrementally constructed octree with its brick pool in HBM."""

    def __init__(self, desc: VolumeDescriptor, cfg: BrickPoolConfig, store=None, *,
                 device: int = 0, reserve_slots: int = 0):
        self.descriptor = desc
        self.config = cfg
        self.geometry = TreeGeometry.build(desc, cfg)
        self.threshold = cfg.resolve_threshold(desc)
        self.lock = threading.RLock()
        self._closed = False
        d = _lib.vt_tree_desc()
        d.dims[:] = list(desc.dims)
        d.channels = desc.channels
        d.sample_bytes = desc.dtype.itemsize
        d.background = desc.background_value
        d.brick[:] = list(cfg.brick_dims)
        d.threshold = float(self.threshold)
        d.reserve_slots = int(reserve_slots)
        d.device = int(device)
        self.device = int(device)
        h = ct.c_void_p()
        _lib.call("vt_tree_create", ct.byref(d), ct.byref(h))
        self._h = h
        self._dense = os.environ.get("VT_DENSE", "1") != "0"
        self._ev_cap = 4096
        self.store = _PoolView(self)

    # -- factories ---------------------------------------------------------
    @classmethod
    def create(cls, desc: VolumeDescriptor, cfg: BrickPoolConfig, pool_path=None, **kw):
        """Octree.create (octree.py:166-176); the pool lives in HBM, so
        ``pool_path`` is accepted for signature compatibility only."""
        return cls(desc, cfg, None, **kw)

    def close(self):
        if not self._closed and self._h:
            _lib.call("vt_tree_destroy", self._h)
            self._closed = True

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- events --------------------------------------------------------------
    def drain_event_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        """B200 extension: drain_events as packed (kinds int32, indices
        int64) arrays — no Python object per event (a 2048^2 slice of 32^3
        bricks updates ~5.5k nodes).  Events stay queued in the library until
        drained, as in the reference (octree.py:180-183)."""
        with self.lock:
            n = ct.c_int64()
            _lib.call("vt_tree_event_count", self._h, ct.byref(n))
            kinds = np.empty(n.value, np.int32)
            idx = np.empty(n.value, np.int64)
            if n.value:
                got, more = ct.c_int64(), ct.c_int32()
                _lib.call("vt_tree_take_events", self._h, _lib.ptr(kinds, ct.c_int32),
                          _lib.ptr(idx, ct.c_int64), n.value, ct.byref(got), ct.byref(more))
            return kinds, idx

    def drain_events(self) -> "EventList":
        """Every queued change event, oldest first (octree.py:180-183)."""
        return EventList.from_arrays(*self.drain_event_arrays())

    # -- insertion -------------------------------------------------------------
    def insert_block(self, channel: int, origin, values) -> EventList:
        """Octree.insert_block (octree.py:323-397).  ``values`` (dz, dy, dx)
        numpy array (host) or a CUDA tensor/array exposing
        ``__cuda_array_interface__`` (device, stream-ordered)."""
        desc = self.descriptor
        if not 0 <= channel < desc.channels:
            raise ValueError(f"channel {channel} out of range")
        return self._insert(int(channel), origin, values, 3)

    def insert_channels(self, origin, values) -> "EventArrays":
        """All channels at once: values (dz, dy, dx, C) interleaved; same
        tree and events as C successive insert_block calls (returned as a
        lazy EventArrays sequence)."""
        return self._insert(-1, origin, values, 4)

    def insert_many(self, blocks) -> None:
        """B200 extension (vt_tree_insert_many): insert ``blocks`` — an
        iterable of ``(channel, origin, values)`` as insert_block takes them —
        in one library call.  The tree and the queued change events
        (drain_events) are exactly those of calling insert_block on each in
        order (ingest_stream's frame loop, ingest.py:306-358); only the
        per-call return lists are not built.  Consecutive device or host
        blocks are batched; at threshold 0 the single-channel full-x/y blocks
        that complete a brick layer become one dense insertion, read in place
        when they are slices of one planar (C, Z, Y, X) device array."""
        desc = self.descriptor
        run, run_kind, keep, cstream = [], None, [], 0

        def flush_run():
            nonlocal run, keep
            if not run:
                return
            arr = (_lib.vt_block * len(run))(*run)
            _lib.call("vt_tree_insert_many", self._h, len(run), arr, run_kind,
                      ct.c_void_p(cstream))
            run, keep = [], []

        with self.lock:
            for channel, origin, values in blocks:
                if not 0 <= int(channel) < desc.channels:
                    flush_run()
                    raise ValueError(f"channel {channel} out of range")
                src, kind, shape, k, cs = self._source(values, 3)
                if run and kind != run_kind:
                    flush_run()
                run_kind, cstream = kind, cs
                o = [int(v) for v in origin]
                b = _lib.vt_block()
                b.channel = int(channel)
                b.origin[:] = o
                b.dims[:] = [shape[2], shape[1], shape[0]]
                b.samples = src
                run.append(b)
                keep.append(k)
            flush_run()

    _BLOCK_DTYPE = np.dtype([("channel", "<i4"), ("origin", "<i4", 3), ("dims", "<i4", 3),
                             ("pad", "<i4"), ("samples", "<u8")])

    def insert_planar(self, values, z0: int = 0) -> None:
        """B200 extension: a slab of a slice stream in VSTR order.  ``values``
        is a (C, dz, Y, X) planar block (CUDA tensor or host array) holding
        planes z0 .. z0+dz of every channel over the full x/y extent; the
        tree and queued events are those of
        ``insert_block(c, (0, 0, z0 + z), values[c, z:z + 1])`` for each z,
        for each channel c (ingest_stream's frame order, ingest.py:306-358),
        issued as one vt_tree_insert_many call without per-slice Python work."""
        desc = self.descriptor
        torch = sys.modules.get("torch")
        if torch is not None and isinstance(values, torch.Tensor) and values.is_cuda:
            want = torch.uint8 if desc.dtype == np.uint8 else torch.uint16
            if values.dtype != want:
                raise ValueError(f"planar block must be {want}")
            if values.dim() != 4 or values.stride(3) != 1 or values.stride(2) != values.shape[3]:
                raise ValueError("planar block must be (C, dz, Y, X) with contiguous planes")
            C, dz, Y, X = values.shape
            base, es = values.data_ptr(), values.element_size()
            cstr, zstr = values.stride(0) * es, values.stride(1) * es
            kind = _lib.VT_MEM_DEVICE
            cs = torch.cuda.current_stream(values.device).cuda_stream
            keep = values
        else:
            if torch is not None and isinstance(values, torch.Tensor):
                values = values.numpy()  # host tensor (pinned memory stays pinned)
            arr = np.asarray(values)
            if arr.dtype != desc.dtype:
                arr = arr.astype(desc.dtype)
            if arr.ndim != 4:
                raise ValueError("planar block must be (C, dz, Y, X)")
            isz = arr.itemsize
            if arr.strides[3] != isz or arr.strides[2] != arr.shape[3] * isz:
                arr = np.ascontiguousarray(arr)  # each (c, z) plane must be contiguous
            C, dz, Y, X = arr.shape
            base, cstr, zstr = arr.ctypes.data, arr.strides[0], arr.strides[1]
            kind, cs, keep = _lib.VT_MEM_HOST, 0, arr
        if C != desc.channels:
            raise ValueError("planar block must hold every channel")
        n = dz * C
        blk = np.zeros(n, self._BLOCK_DTYPE)
        z = np.repeat(np.arange(dz, dtype=np.int64), C)
        c = np.tile(np.arange(C, dtype=np.int64), dz)
        blk["channel"] = c
        blk["origin"][:, 2] = z0 + z
        blk["dims"][:] = (X, Y, 1)
        blk["samples"] = (base + c * cstr + z * zstr).astype(np.uint64)
        with self.lock:
            _lib.call("vt_tree_insert_many", self._h, n,
                      blk.ctypes.data_as(ct.POINTER(_lib.vt_block)), kind, ct.c_void_p(cs))
        del keep

    def stream_counts(self) -> tuple[int, int, int]:
        """(brick layers built by insert_many as one dense insertion, of which
        read in place, deferred layers of per-block slice streams)."""
        a, b, c = ct.c_int64(), ct.c_int64(), ct.c_int64()
        _lib.call("vt_tree_stream_counts", self._h, ct.byref(a), ct.byref(b), ct.byref(c))
        return int(a.value), int(b.value), int(c.value)

    def _insert(self, channel: int, origin, values, ndim: int) -> EventList:
        desc = self.descriptor
        origin = tuple(int(v) for v in origin)
        src, kind, shape, keep, cstream = self._source(values, ndim)
        if ndim == 4 and shape[3] != desc.channels:
            raise ValueError("last axis must hold every channel")
        bdims = (shape[2], shape[1], shape[0])
        for a in range(3):
            if origin[a] < 0 or origin[a] + bdims[a] > desc.dims[a]:
                raise ValueError(f"block [{origin} + {bdims}) outside volume {desc.dims}")
        with self.lock:
            # one library call: stream ordering, the insertion, its events
            cap = self._ev_cap
            kinds = np.empty(cap, np.int32)
            idx = np.empty(cap, np.int64)
            n = ct.c_int64()
            _lib.call("vt_tree_insert_ev", self._h, channel, _lib.i32x3(origin),
                      _lib.i32x3(bdims), src, kind, ct.c_void_p(cstream),
                      _lib.ptr(kinds, ct.c_int32), _lib.ptr(idx, ct.c_int64), cap,
                      ct.byref(n))
            total = int(n.value)
            if total > cap:
                # more events than the guess: copy them (they stay queued)
                kinds = np.empty(total, np.int32)
                idx = np.empty(total, np.int64)
                cnt = ct.c_int64()
                _lib.call("vt_tree_event_count", self._h, ct.byref(cnt))
                _lib.call("vt_tree_copy_events", self._h, cnt.value - total, total,
                          _lib.ptr(kinds, ct.c_int32), _lib.ptr(idx, ct.c_int64))
                self._ev_cap = min(1 << 20, 1 << (total - 1).bit_length())
            else:
                kinds, idx = kinds[:total], idx[:total]
            del keep  # device blocks: the caller's stream waits for our reads
            if channel < 0:
                return EventArrays(kinds, idx)
            return EventList.from_arrays(kinds, idx)

    def _source(self, values, ndim):
        """(pointer, memory kind, shape, keep-alive, caller stream handle)."""
        dt = self.descriptor.dtype
        torch = sys.modules.get("torch")
        is_tensor = torch is not None and isinstance(values, torch.Tensor)
        if is_tensor or getattr(values, "__cuda_array_interface__", None) is not None:
            import torch
            t = values if is_tensor else torch.as_tensor(values, device="cuda")
            if not t.is_cuda:
                values = t.numpy()
            else:
                if t.dim() != ndim:
                    raise ValueError(f"block values must be {ndim}-D")
                want = torch.uint8 if dt == np.uint8 else torch.uint16
                if t.dtype != want or not t.is_contiguous():
                    t = t.to(want).contiguous()
                # device work runs on the tree's stream, ordered after torch's
                # current stream (event wait, no host synchronisation)
                cs = torch.cuda.current_stream(t.device).cuda_stream
                return ct.c_void_p(t.data_ptr()), _lib.VT_MEM_DEVICE, tuple(t.shape), t, cs
        arr = np.asarray(values)
        if arr.ndim != ndim:
            raise ValueError("block values must be 3-D (z, y, x)" if ndim == 3 else
                             "block values must be 4-D (z, y, x, c)")
        arr = np.ascontiguousarray(arr.astype(dt, copy=False))
        return ct.c_void_p(arr.ctypes.data), _lib.VT_MEM_HOST, arr.shape, arr, 0

    # -- state ---------------------------------------------------------------
    def _info(self) -> _lib.vt_tree_info:
        info = _lib.vt_tree_info()
        _lib.call("vt_tree_info_get", self._h, ct.byref(info))
        return info

    @property
    def node_count(self) -> int:
        return int(self._info().node_count)

    @property
    def brick_count(self) -> int:
        return int(self._info().brick_count)

    @property
    def pruned_bricks(self) -> int:
        return int(self._info().pruned_bricks)

    @property
    def inserted_voxels(self) -> int:
        return int(self._info().inserted_voxels)

    @property
    def construction_finished(self) -> bool:
        return bool(self._info().finished)

    @property
    def borders_filled(self) -> bool:
        return bool(self._info().borders_filled)

    @property
    def root(self) -> OctreeNode:
        return self.node_by_index(0)

    def checksum(self) -> int:
        """Device-computed 64-bit digest of structure, statistics and every
        brick (vt_tree_checksum) — equal trees, equal digests."""
        out = ct.c_uint64()
        _lib.call("vt_tree_checksum", self._h, ct.byref(out))
        return int(out.value)

    @property
    def dense_build(self) -> bool:
        """B200 extension: threshold-0 dense build on (default) / off
        (vt_tree_set_dense).  Results are identical either way."""
        return self._dense

    @dense_build.setter
    def dense_build(self, on: bool) -> None:
        with self.lock:
            _lib.call("vt_tree_set_dense", self._h, 1 if on else 0)
            self._dense = bool(on)

    def dense_counts(self) -> tuple[int, int, int]:
        """(dense leaf insertions, dense parent recomputes, fill_borders calls
        served by prefilled leaf shells) so far."""
        a, b, c = ct.c_int64(), ct.c_int64(), ct.c_int64()
        _lib.call("vt_tree_dense_counts", self._h, ct.byref(a), ct.byref(b), ct.byref(c))
        return int(a.value), int(b.value), int(c.value)

    def use_stream(self, stream) -> None:
        """Run this tree's device work on ``stream`` (a torch.cuda.Stream or
        a raw cudaStream_t handle)."""
        h = getattr(stream, "cuda_stream", stream)
        _lib.call("vt_tree_set_stream", self._h, ct.c_void_p(int(h)))

    def flush(self) -> None:
        """B200 extension: enqueue deferred device work (an open slice
        layer's received planes, pending propagation) without a host wait."""
        with self.lock:
            _lib.call("vt_tree_flush", self._h)

    def sync(self) -> None:
        """Complete deferred device work (tau == 0 batches)."""
        _lib.call("vt_tree_sync", self._h)

    # -- finalization ----------------------------------------------------------
    def finalize(self) -> None:
        with self.lock:
            _lib.call("vt_tree_finalize", self._h)

    def fill_borders(self) -> None:
        """octree.py:540-549; emits NODE_UPDATED per brick."""
        with self.lock:
            _lib.call("vt_tree_fill_borders", self._h)

    def fill_borders_async(self) -> threading.Thread:
        th = threading.Thread(target=self.fill_borders, name="border-fill", daemon=True)
        th.start()
        return th

    # -- lookup ------------------------------------------------------------------
    def node_by_index(self, index: int) -> OctreeNode | None:
        rec = _lib.vt_node()
        ex = ct.c_int32()
        _lib.call("vt_tree_node", self._h, int(index), ct.byref(rec), ct.byref(ex))
        return OctreeNode(self, int(index), rec) if ex.value else None

    def find_node(self, point, target_level: int = 0) -> OctreeNode:
        p = (ct.c_double * 3)(*[float(v) for v in point])
        out = ct.c_int64()
        _lib.call("vt_tree_find_node", self._h, p, int(target_level), ct.byref(out))
        return self.node_by_index(out.value)

    def node_indices(self, with_flags: bool = False):
        n = ct.c_int64()
        _lib.call("vt_tree_list_nodes", self._h, None, None, 0, ct.byref(n))
        idx = np.empty(n.value, np.int64)
        fl = np.empty(n.value, np.int32)
        _lib.call("vt_tree_list_nodes", self._h, _lib.ptr(idx, ct.c_int64),
                  _lib.ptr(fl, ct.c_int32), n.value, ct.byref(n))
        return (idx, fl) if with_flags else idx

    def iter_nodes(self):
        """Breadth-first (== ascending index) snapshots (octree.py:507-513)."""
        idx, flags, stats, _ = self.export(with_bricks=False)
        geo = self.geometry
        for r, i in enumerate(idx):
            rec = _lib.vt_node()
            rec.flags = int(flags[r])
            rec.level = geo.level_of_index(int(i))
            rec.box_lo[:] = list(geo.box_lo_of_index(int(i)))
            rec.slot = -1
            for c in range(self.descriptor.channels):
                for s in range(5):
                    rec.stats[c][s] = int(stats[r, c, s])
            yield OctreeNode(self, int(i), rec)

    def read_brick(self, index: int) -> np.ndarray:
        cfg, desc = self.config, self.descriptor
        bz, by, bx = tuple(reversed(cfg.stored_brick_dims))
        out = np.empty((bz, by, bx, desc.channels), dtype=desc.dtype)
        _lib.call("vt_tree_read_brick", self._h, int(index), ct.c_void_p(out.ctypes.data))
        return out

    def export(self, indices=None, with_bricks=True):
        """Bulk snapshot for serialization: (indices, VT_NODE_* flags, stats
        (n, C, 5) as [avg, smin, smax, sub_min, sub_max], bricks of the
        bricked nodes in index order)."""
        all_idx, all_fl = self.node_indices(with_flags=True)
        if indices is None:
            idx, flags = all_idx, all_fl
        else:
            idx = np.asarray(indices, np.int64)
            lut = dict(zip(all_idx.tolist(), all_fl.tolist()))
            flags = np.asarray([lut[int(i)] for i in idx], np.int32)
        C = self.descriptor.channels
        stats = np.empty((len(idx), C, 5), np.int32)
        nbrick = int(np.count_nonzero(flags & _lib.NODE_BRICK))
        bricks = None
        if with_bricks:
            bz, by, bx = tuple(reversed(self.config.stored_brick_dims))
            bricks = np.empty((nbrick, bz, by, bx, C), dtype=self.descriptor.dtype)
        _lib.call("vt_tree_export", self._h, len(idx), _lib.ptr(idx, ct.c_int64),
                  _lib.ptr(stats, ct.c_int32),
                  ct.c_void_p(bricks.ctypes.data) if bricks is not None and nbrick else None)
        return idx, flags, stats, bricks
