"""Sort-first multi-GPU full-frame rendering (no reference
counterpart — the reference renders on one CPU thread, raycast.py:282-290).

One process per GPU, each holding a full replica of the node buffer and the
brick pool (``DeviceState(tree, resident_all=True)``).  The frame is cut
into horizontal strips of ``strip_rows`` rows; rank r renders strips
r, r + G, r + 2G, ... (interleaving balances the per-GPU sample load, which
is concentrated where the specimen projects) with ONE launch of the fused
ray-casting kernel (``vt_render_strips``), then the compact strip buffers
are gathered to the root rank over NCCL and re-interleaved there.  The six
render counters are summed with an all-reduce.  Rays are independent and
the pool is read-only during a pass, so there is no other exchange.
"""

from __future__ import annotations

import ctypes as ct

import numpy as np

from .. import _lib
from .core import RenderCounters
from .raycast import OUT_F32, OUT_F64, OUT_RGBA8, scene_to_vt

_TORCH_DTYPE = {OUT_F64: "float64", OUT_F32: "float32", OUT_RGBA8: "uint8"}


def part_rows(height: int, strip_rows: int, n_parts: int) -> int:
    """Rows of one part's compact buffer: ceil(strips / n_parts) whole strips
    (vt_strip_part_rows; the padding rows past the frame are zero)."""
    if n_parts <= 1:
        return height
    strips = -(-height // strip_rows)
    return -(-strips // n_parts) * strip_rows


def frame_rows_of_part(height: int, strip_rows: int, n_parts: int, part: int) -> np.ndarray:
    """Frame row index of every row of ``part``'s compact buffer (-1 = pad)."""
    if n_parts <= 1:
        return np.arange(height)
    rows = part_rows(height, strip_rows, n_parts)
    jl = np.arange(rows)
    s = jl // strip_rows
    j = (s * n_parts + part) * strip_rows + jl % strip_rows
    return np.where(j < height, j, -1)


def assemble(parts, height: int, strip_rows: int):
    """Re-interleave gathered part buffers (G, rows, W, 4) into the frame:
    strip s of the frame is strip s // G of part s % G."""
    import torch
    stacked = parts if isinstance(parts, torch.Tensor) else torch.stack(list(parts))
    g, rows, w, ch = stacked.shape
    if g == 1:
        return stacked[0, :height]
    per = rows // strip_rows
    x = stacked.reshape(g, per, strip_rows, w, ch).permute(1, 0, 2, 3, 4)
    return x.reshape(per * g * strip_rows, w, ch)[:height]


class SortFirstRenderer:
    """Full-frame render of one Scene across the ranks of ``group``
    (torch.distributed, backend nccl on B200).  ``render_fullframe`` returns
    the assembled image on ``root`` (a CUDA tensor, or a host numpy array with
    ``to_host=True``) and None elsewhere, plus the globally summed
    RenderCounters on every rank."""

    def __init__(self, device, group=None, strip_rows: int = 8, root: int = 0):
        import torch.distributed as dist
        self.device = device
        self.group = group
        self.strip_rows = int(strip_rows)
        self.root = int(root)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.descriptor = device.octree.descriptor if device is not None else None
        self._bufs = {}

    def _buffer(self, key, shape, dtype, device="cuda"):
        import torch
        b = self._bufs.get(key)
        if (b is None or tuple(b.shape) != tuple(shape) or b.dtype != dtype
                or b.device != torch.device(device)):
            b = torch.empty(shape, dtype=dtype, device=device)
            self._bufs[key] = b
        return b

    def render_part(self, scene, out_kind: int = OUT_RGBA8):
        """This rank's strips: a (part_rows, W, 4) CUDA tensor + counters."""
        import torch
        cam = scene.camera
        rows = part_rows(cam.height, self.strip_rows, self.world)
        dtype = getattr(torch, _TORCH_DTYPE[out_kind])
        local = self._buffer("local", (rows, cam.width, 4), dtype)
        s = scene_to_vt(scene, self.descriptor)
        cnt = _lib.vt_counters()
        # stream ordering both ways, no host synchronisation: the tree's
        # stream after torch's (the buffer), torch's after the render (the
        # gather reads it)
        self.device.order_after_torch()
        _lib.call("vt_render_strips", self.device.handle, ct.byref(s), self.strip_rows,
                  self.world, self.rank, ct.c_void_p(local.data_ptr()), out_kind, 1,
                  ct.byref(cnt))
        _lib.call("vt_tree_signal_stream", self.device.octree.handle,
                  ct.c_void_p(torch.cuda.current_stream().cuda_stream))
        return local, RenderCounters.from_vt(cnt)

    def gather(self, local):
        """Gather every part to root and re-interleave (root only)."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return local
        parts = None
        # NCCL gathers device buffers directly; other backends stage via host
        src = local if dist.get_backend(self.group) == "nccl" else local.cpu()
        if self.rank == self.root:
            parts = self._buffer("parts", (self.world,) + tuple(src.shape), src.dtype,
                                 src.device)
            plist = list(parts.unbind(0))
        dist.gather(src, plist if self.rank == self.root else None, dst=self.root,
                    group=self.group)
        if self.rank != self.root:
            return None
        return parts.to(local.device)

    def reduce_counters(self, cnt: RenderCounters) -> RenderCounters:
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return cnt
        fields = list(RenderCounters.__dataclass_fields__)
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        v = torch.tensor([getattr(cnt, f) for f in fields] + [cnt.samples_skipped],
                         dtype=torch.int64, device=dev)
        dist.all_reduce(v, group=self.group)
        vals = v.tolist()
        out = RenderCounters(**{f: int(x) for f, x in zip(fields, vals)})
        out.samples_skipped = int(vals[-1])
        return out

    def render_fullframe(self, scene, out_kind: int = OUT_RGBA8, to_host: bool = False):
        local, cnt = self.render_part(scene, out_kind)
        parts = self.gather(local)
        cnt = self.reduce_counters(cnt)
        if parts is None:
            return None, cnt
        img = assemble(parts if self.world > 1 else local[None], scene.camera.height,
                       self.strip_rows)
        if to_host:
            img = img.cpu().numpy()
        return img, cnt
