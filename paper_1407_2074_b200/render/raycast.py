"""Octree ray caster — drop-in for voxtree.render.raycast (raycast.py:53-339).

``OutOfCoreRenderer.render_fullframe`` launches the fused full-frame kernel
(ray setup + march + finalize in one pass); ``RefinementSession`` keeps the
per-ray state (k, accumulated colour, maxima, terminated/suspended) in HBM
between passes.  No CPU path exists.
"""

from __future__ import annotations

import ctypes as ct

import numpy as np

from .. import _lib
from ..device import DeviceState
from .core import RenderCounters
from .settings import Scene

OUT_F64, OUT_F32, OUT_RGBA8 = 0, 1, 2


def host_image(shape, dtype):
    """Output array for a frame: page-locked when torch is present (its
    caching host allocator recycles the block once the array is dropped), so
    the device-to-host copy runs at full PCIe speed."""
    try:
        import torch
        if torch.cuda.is_available():
            tdt = {np.float64: torch.float64, np.float32: torch.float32,
                   np.uint8: torch.uint8}[dtype]
            return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    except ImportError:
        pass
    return np.empty(shape, dtype=dtype)


_BASIS_CACHE: dict = {}


def _camera_frame(cam):
    """(basis, tan_half, footprint) of ``cam``, memoised on the pose: the
    numpy results are reused as-is, so the packed values stay bit-identical
    while an unchanged camera costs one tuple hash per frame."""
    # raw bytes, so -0.0 and 0.0 (equal as floats) stay distinct keys
    key = (np.array([*cam.position, *cam.look_at, *cam.up, cam.fov_y],
                    dtype=np.float64).tobytes(), cam.height)
    hit = _BASIS_CACHE.get(key)
    if hit is None:
        if len(_BASIS_CACHE) > 64:
            _BASIS_CACHE.clear()
        hit = (cam.basis(), float(np.tan(cam.fov_y / 2.0)), float(cam.pixel_footprint_scale()))
        _BASIS_CACHE[key] = hit
    return hit


def scene_to_vt(scene: Scene, descriptor) -> _lib.vt_scene:
    """Pack a Scene for the kernel.  Transcendental / BLAS-dependent camera
    constants are computed with numpy exactly as the reference computes them
    (camera.py:33-57, settings.py:60-67)."""
    cam, st = scene.camera, scene.settings
    C = descriptor.channels
    if len(scene.transfer_functions) != C:
        raise ValueError(f"need one transfer function per channel ({C})")
    s = _lib.vt_scene()
    (pos, fwd, right, up), s.tan_half, s.footprint_scale = _camera_frame(cam)
    s.position[:] = pos.tolist()
    s.fwd[:] = fwd.tolist()
    s.right[:] = right.tolist()
    s.up[:] = up.tolist()
    s.aspect = cam.width / cam.height
    s.width, s.height = int(cam.width), int(cam.height)
    s.mode_mip = 1 if st.mode == "mip" else 0
    s.precision = 1 if getattr(st, "precision", "fp64") == "fp32" else 0
    s.empty_skip = {None: 0, "off": 1, "bricks": 2, "subbricks": 3}[
        getattr(st, "empty_space_skip", None)]
    step = st.resolve_step(descriptor.spacing)
    s.step = step
    s.corr_exp = st.opacity_exponent(step)
    et = st.early_termination_alpha
    s.et_limit = -1.0 if et is None else float(et)
    s.lod_scale = float(2.0 ** st.lod_bias)
    tf_x = np.ctypeslib.as_array(s.tf_x)
    tf_rgba = np.ctypeslib.as_array(s.tf_rgba)
    for c, tf in enumerate(scene.transfer_functions):
        xs = np.asarray(tf.xs, dtype=np.float64)
        n = len(xs)
        s.tf_count[c] = n
        tf_x[c, :n] = xs
        tf_rgba[c, :n] = np.asarray(tf.rgba, dtype=np.float64)
    planes = list(scene.clips)
    s.n_clips = len(planes)
    for q, p in enumerate(planes):
        s.clip_normal[q][:] = [float(v) for v in p.normal]
        s.clip_offset[q] = float(p.offset)
    s.spacing[:] = list(descriptor.spacing)
    s.has_transforms = 1 if descriptor.has_channel_transforms else 0
    if s.has_transforms:
        tr = np.ctypeslib.as_array(s.transforms)
        for c in range(C):
            m = np.asarray(descriptor.channel_transforms[c], dtype=np.float64)
            tr[c] = m[:3, :4].reshape(-1)
    return s


class OutOfCoreRenderer:
    """Full-frame and refinement passes over a DeviceState (raycast.py:53-295)."""

    def __init__(self, device: DeviceState):
        self.device = device
        self.descriptor = device.octree.descriptor
        self.geometry = device.octree.geometry
        self.channels = self.descriptor.channels

    def render_fullframe(self, scene: Scene, out_kind: int = OUT_F64):
        """One complete pass; returns ((H, W, 4) image, RenderCounters)."""
        s = scene_to_vt(scene, self.descriptor)
        cam = scene.camera
        dtype = {OUT_F64: np.float64, OUT_F32: np.float32, OUT_RGBA8: np.uint8}[out_kind]
        img = host_image((cam.height, cam.width, 4), dtype)
        cnt = _lib.vt_counters()
        self.device.order_after_torch()
        _lib.call("vt_render_fullframe", self.device.handle, ct.byref(s),
                  ct.c_void_p(img.ctypes.data), out_kind, 0, ct.byref(cnt))
        return img, RenderCounters.from_vt(cnt)

    def render_tile(self, scene: Scene, rect, out_kind: int = OUT_F64):
        """Pixels [x0,x1) x [y0,y1) of the full-frame image (sort-first tile)."""
        s = scene_to_vt(scene, self.descriptor)
        x0, y0, x1, y1 = (int(v) for v in rect)
        dtype = {OUT_F64: np.float64, OUT_F32: np.float32, OUT_RGBA8: np.uint8}[out_kind]
        img = np.empty((y1 - y0, x1 - x0, 4), dtype=dtype)
        cnt = _lib.vt_counters()
        r = (ct.c_int32 * 4)(x0, y0, x1, y1)
        self.device.order_after_torch()
        _lib.call("vt_render_tile", self.device.handle, ct.byref(s), r,
                  ct.c_void_p(img.ctypes.data), out_kind, 0, ct.byref(cnt))
        return img, RenderCounters.from_vt(cnt)

    def start_refinement(self, scene: Scene, tile=None) -> "RefinementSession":
        return RefinementSession(self, scene, tile=tile)


class _RayView:
    """``session.rays`` view: n_steps / k / suspended copied from HBM."""

    def __init__(self, session: "RefinementSession"):
        self._s = session

    def _state(self):
        n = self._s._n
        k = np.empty(n, np.int64)
        ns = np.empty(n, np.int64)
        sus = np.empty(n, np.uint8)
        _lib.call("vt_rays_state", self._s._h, _lib.ptr(k, ct.c_int64),
                  _lib.ptr(ns, ct.c_int64), ct.c_void_p(sus.ctypes.data))
        return k, ns, sus.astype(bool)

    @property
    def k(self):
        return self._state()[0]

    @property
    def n_steps(self):
        return self._state()[1]

    @property
    def suspended(self):
        return self._state()[2]


class RefinementSession:
    """Progressive refinement with per-ray state cached in HBM between
    passes (raycast.py:298-339); complete when a pass requests nothing."""

    def __init__(self, renderer: OutOfCoreRenderer, scene: Scene, tile=None):
        self.renderer = renderer
        self.scene = scene
        self.scene_key = scene.key()
        s = scene_to_vt(scene, renderer.descriptor)
        cam = scene.camera
        self._n = cam.width * cam.height
        h = ct.c_void_p()
        t = None
        if tile is not None:
            x0, y0, x1, y1 = (int(v) for v in tile)
            t = (ct.c_int32 * 4)(max(0, x0), max(0, y0), min(cam.width, x1), min(cam.height, y1))
        renderer.device.order_after_torch()
        _lib.call("vt_rays_create", renderer.device.handle, ct.byref(s), t, ct.byref(h))
        self._h = h
        self.rays = _RayView(self)
        self.counters = RenderCounters()
        self.passes = 0
        self.complete = False
        self._last_suspended = 0

    def __del__(self):
        try:
            if self._h:
                _lib.call("vt_rays_destroy", self._h)
                self._h = None
        except Exception:
            pass

    def run_pass(self) -> bool:
        if self.complete:
            return True
        cnt = _lib.vt_counters()
        sus = ct.c_int64()
        self.renderer.device.order_after_torch()
        _lib.call("vt_rays_march", self._h, 1, ct.byref(cnt), ct.byref(sus))
        self.passes += 1
        pc = RenderCounters.from_vt(cnt)
        self.counters = self.counters.merged(pc)
        self._last_suspended = int(sus.value)
        self.complete = pc.bricks_requested == 0
        return self.complete

    @property
    def suspended_rays(self) -> int:
        return self._last_suspended

    def image(self) -> np.ndarray:
        cam = self.scene.camera
        out = np.empty((cam.height, cam.width, 4), np.float64)
        cnt = _lib.vt_counters()
        _lib.call("vt_rays_image", self._h, ct.c_void_p(out.ctypes.data), ct.byref(cnt))
        return out
