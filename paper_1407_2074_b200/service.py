"""The caller side of the render path: the interactive frame service and the
orbit benchmark protocol, on the B200 tree / mirror / renderer.

Mirrors ``voxtree.service`` (service.py:74-349) and ``voxtree.cli bench``
(cli.py:209-252) — same class, method names, control-message schema, status
JSON, frame wire format and loop semantics — so a viewer or script written
against the reference drives this package unchanged:

* ``FrameService.step`` (service.py:222-261): pending change events go to the
  device mirror (``DeviceState.apply_events``, a device-side repack of the
  node buffer); a changed scene or tree restarts the loop; full-frame passes
  repeat until one requested no brick and uploaded nothing ("stable"), then
  a refinement session runs pass by pass and its image replaces the shown one
  only when complete.  The brick buffer defaults to the reference's bounded
  one (512 MiB, flag-driven uploads); ``resident_all=True`` (B200 extension)
  makes the HBM pool the brick buffer, so the first pass is already stable.
* ``handle_control`` (service.py:127-183): camera, transfer_function,
  clip_planes, mode, strategy, reset_refinement, abort_ingest, ping,
  get_settings; every message answered with an ack / nack echoing its id.
* Frames: 16-byte header (frame id, width, height, format 1 = PNG RGBA) +
  PNG (service.py:45-61); status JSON after every frame (service.py:271-286).
* ``serve``: the websocket transport (service.py:320-349), optional — the
  ``websockets`` package is imported only when it is called.

``orbit_bench`` is the paper's interactive benchmark protocol
(``voxtree bench``, cli.py:209-252): a full orbit of
full-frame passes around the volume centre at 2.5x its extent.
"""

from __future__ import annotations

import io
import json
import struct
import threading
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .device import DeviceState, RenderMode
from .ingest import ingest_stream
from .octree import Octree
from .render import (Camera, ClipPlane, ClipSet, OutOfCoreRenderer, RenderSettings, Scene,
                     TransferFunction, image_to_rgba8)

FRAME_HEADER = struct.Struct("<IIII")  # frame id, width, height, pixel format
PIXEL_FORMAT_PNG_RGBA = 1


def encode_frame(frame_id: int, image: np.ndarray) -> bytes:
    """Header + PNG of the RGBA8 conversion of a float (H, W, 4) image."""
    from PIL import Image
    rgba = image_to_rgba8(image)
    png = io.BytesIO()
    Image.fromarray(rgba, "RGBA").save(png, format="PNG")
    h, w = rgba.shape[:2]
    return FRAME_HEADER.pack(frame_id, w, h, PIXEL_FORMAT_PNG_RGBA) + png.getvalue()


def decode_frame(blob: bytes):
    """(frame_id, width, height, format, RGBA8 array) of an encoded frame."""
    from PIL import Image
    fid, w, h, fmt = FRAME_HEADER.unpack_from(blob, 0)
    return fid, w, h, fmt, np.asarray(Image.open(io.BytesIO(blob[FRAME_HEADER.size:])))


@dataclass
class _Client:
    """One viewer: a bounded outbox — a slow viewer loses its oldest frames,
    the render loop never waits for it."""
    queue: deque = field(default_factory=lambda: deque(maxlen=8))
    ready: threading.Event = field(default_factory=threading.Event)
    closed: bool = False

    def push(self, payload) -> None:
        self.queue.append(payload)
        self.ready.set()


def _default_camera(desc, viewport) -> Camera:
    centre = tuple(d * s / 2.0 for d, s in zip(desc.dims, desc.spacing))
    extent = max(d * s for d, s in zip(desc.dims, desc.spacing))
    return Camera(position=(centre[0], centre[1], -2.5 * extent), look_at=centre, up=(0, 1, 0),
                  width=viewport[0], height=viewport[1])


class FrameService:
    """Render loop + session state, independent of the transport."""

    def __init__(self, tree: Octree, *, viewport=(256, 256),
                 brick_budget_bytes: int | None = None, slot_count: int | None = None,
                 upload_budget_ms: float = 150.0, idle_sleep: float = 0.02,
                 resident_all: bool = False):
        self.tree = tree
        if resident_all:
            # B200 extension: the HBM pool is the brick buffer
            self.device = DeviceState(tree, resident_all=True)
        else:
            opts = {k: v for k, v in (("brick_budget_bytes", brick_budget_bytes),
                                      ("slot_count", slot_count)) if v is not None}
            self.device = DeviceState(tree, **opts)
        self.renderer = OutOfCoreRenderer(self.device)
        self.upload_budget_ms = upload_budget_ms
        self.idle_sleep = idle_sleep
        desc = tree.descriptor
        self._lock = threading.Lock()
        self._camera = _default_camera(desc, viewport)
        self._tfs = [TransferFunction.ramp(max_alpha=0.8) for _ in range(desc.channels)]
        self._clips = ClipSet()
        self._settings = RenderSettings(strategy="refinement")
        self._version = 0          # bumped by every accepted control
        self._shown_version = -1   # the version the loop last restarted for
        self._session = None
        self._stable = False       # a full-frame pass requested / uploaded nothing
        self.frame_id = 0
        self.refinement_complete = False
        self._clients: list[_Client] = []
        self._stop = threading.Event()
        self._ingest_abort = threading.Event()
        self._ingest_thread: threading.Thread | None = None
        self._render_thread: threading.Thread | None = None

    # -- scene ----------------------------------------------------------------
    def current_scene(self) -> Scene:
        with self._lock:
            return Scene(camera=self._camera, settings=self._settings,
                         transfer_functions=list(self._tfs), clips=self._clips)

    def _with_settings(self, **changes) -> RenderSettings:
        s = self._settings
        kw = dict(mode=s.mode, strategy=s.strategy, sampling_step=s.sampling_step,
                  early_termination_alpha=s.early_termination_alpha, lod_bias=s.lod_bias)
        kw.update(changes)
        return RenderSettings(**kw)

    # -- control messages -----------------------------------------------------
    def _ctl_camera(self, m):
        cam = self._camera
        vp = m.get("viewport", [cam.width, cam.height])
        self._camera = Camera(position=tuple(m.get("position", cam.position)),
                              look_at=tuple(m.get("look_at", cam.look_at)),
                              up=tuple(m.get("up", cam.up)),
                              fov_y=float(np.deg2rad(m["fov_deg"])) if "fov_deg" in m
                              else cam.fov_y,
                              width=int(vp[0]), height=int(vp[1]))

    def _ctl_transfer_function(self, m):
        c = int(m["channel"])
        if not 0 <= c < self.tree.descriptor.channels:
            raise ValueError(f"channel {c} out of range")
        self._tfs[c] = TransferFunction(m["points"])

    def _ctl_clip_planes(self, m):
        self._clips = ClipSet(tuple(ClipPlane(tuple(p[:3]), float(p[3]))
                                    for p in m.get("planes", [])))

    def _ctl_mode(self, m):
        self._settings = self._with_settings(mode=m["mode"])

    def _ctl_strategy(self, m):
        self._settings = self._with_settings(strategy=m["strategy"])

    def _ctl_reset_refinement(self, m):
        pass  # the version bump restarts the loop

    def _ctl_abort_ingest(self, m):
        self._ingest_abort.set()

    def handle_control(self, message: str) -> dict:
        """Apply one JSON control message; the ack / nack reply echoes its id."""
        msg = None
        try:
            msg = json.loads(message)
            if not isinstance(msg, dict) or "type" not in msg:
                raise ValueError("control message must be an object with a type")
            kind = msg["type"]
            if kind == "ping":
                return {"type": "ack", "id": msg.get("id")}
            if kind == "get_settings":
                with self._lock:
                    return {"type": "settings", "id": msg.get("id"), **self._settings_dict()}
            handler = getattr(self, f"_ctl_{kind}", None) if isinstance(kind, str) else None
            if handler is None:
                raise ValueError(f"unknown control type {kind!r}")
            with self._lock:
                handler(msg)
                self._version += 1
            return {"type": "ack", "id": msg.get("id")}
        except Exception as exc:  # a bad message is answered, never fatal
            mid = msg.get("id") if isinstance(msg, dict) else None
            return {"type": "nack", "id": mid, "error": str(exc)}

    def _settings_dict(self) -> dict:
        cam = self._camera
        return {"camera": {"position": list(cam.position), "look_at": list(cam.look_at),
                           "up": list(cam.up), "fov_deg": float(np.rad2deg(cam.fov_y)),
                           "viewport": [cam.width, cam.height]},
                "mode": self._settings.mode, "strategy": self._settings.strategy,
                "transfer_functions": [tf.control_points() for tf in self._tfs],
                "clip_planes": [[*p.normal, p.offset] for p in self._clips]}

    # -- live ingest ------------------------------------------------------------
    def attach_ingest(self, stream) -> threading.Thread:
        """Consume a VSTR stream (after its handshake) while rendering."""
        t = threading.Thread(target=lambda: ingest_stream(
            stream, self.tree, should_stop=self._ingest_abort.is_set), name="ingest", daemon=True)
        self._ingest_thread = t
        t.start()
        return t

    @property
    def ingest_active(self) -> bool:
        return self._ingest_thread is not None and self._ingest_thread.is_alive()

    def construction_progress(self) -> float:
        desc = self.tree.descriptor
        return min(100.0, 100.0 * self.tree.inserted_voxels / (desc.voxel_count * desc.channels))

    # -- render loop -------------------------------------------------------------
    def step(self) -> bool:
        """One loop iteration; True when a frame was broadcast."""
        events = self.tree.drain_events()
        if len(events):
            self.device.apply_events(events)
        scene = self.current_scene()
        with self._lock:
            version = self._version
        if len(events) or version != self._shown_version:
            self._shown_version = version
            self._session = None
            self._stable = False
            self.refinement_complete = False

        if not self._stable:
            image, counters = self.renderer.render_fullframe(scene)
            plan = self.device.process_flags(RenderMode.FULLFRAME)
            uploaded = self.device.upload_bricks(plan, self.upload_budget_ms)
            self._stable = counters.bricks_requested == 0 and uploaded == 0
            self._broadcast(image)
            return True

        if self._settings.strategy != "refinement" or self.refinement_complete:
            return False
        if self._session is None:
            self._session = self.renderer.start_refinement(scene)
        if self._session.run_pass():
            self.refinement_complete = True
            self._broadcast(self._session.image())
            return True
        self.device.upload_bricks(self.device.process_flags(RenderMode.REFINEMENT),
                                  self.upload_budget_ms)
        self._push_all(self._status_json())
        return False

    def _push_all(self, payload) -> None:
        for client in list(self._clients):
            client.push(payload)

    def _broadcast(self, image: np.ndarray) -> None:
        self.frame_id += 1
        frame = encode_frame(self.frame_id, image)
        status = self._status_json()
        for client in list(self._clients):
            client.push(frame)
            client.push(status)

    def _status_json(self) -> str:
        return json.dumps({"type": "status", "frame_id": self.frame_id,
                           "construction_pct": round(self.construction_progress(), 2),
                           "bricks_resident": self.device.resident_bricks,
                           "refinement_complete": self.refinement_complete,
                           "ingest_active": self.ingest_active,
                           "mode": self._settings.mode, "strategy": self._settings.strategy})

    def run(self) -> None:
        while not self._stop.is_set():
            if not self.step() and not self.ingest_active:
                time.sleep(self.idle_sleep)

    def start(self) -> None:
        self._render_thread = threading.Thread(target=self.run, name="render-loop", daemon=True)
        self._render_thread.start()

    def stop(self) -> None:
        self._stop.set()
        self._ingest_abort.set()
        if self._render_thread is not None:
            self._render_thread.join(timeout=5)

    # -- viewers -----------------------------------------------------------------
    def register_client(self) -> _Client:
        client = _Client()
        self._clients.append(client)
        with self._lock:
            self._version += 1  # a new viewer gets a fresh frame
        return client

    def unregister_client(self, client: _Client) -> None:
        client.closed = True
        if client in self._clients:
            self._clients.remove(client)


def serve(service: FrameService, host: str = "127.0.0.1", port: int = 8765):
    """Websocket transport (service.py:320-349): binary frames and status
    JSON out, control JSON in, one sender thread per viewer."""
    from websockets.sync.server import serve as ws_serve

    def handler(conn):
        client = service.register_client()

        def sender():
            while not client.closed:
                client.ready.wait(0.25)
                client.ready.clear()
                while client.queue:
                    try:
                        conn.send(client.queue.popleft())
                    except Exception:
                        client.closed = True
                        return

        out = threading.Thread(target=sender, daemon=True)
        out.start()
        try:
            for message in conn:
                if isinstance(message, str):
                    conn.send(json.dumps(service.handle_control(message)))
        finally:
            service.unregister_client(client)

    service.start()
    try:
        with ws_serve(handler, host, port) as server:
            server.serve_forever()
    finally:
        service.stop()


def orbit_bench(tree: Octree, *, frames: int = 100, orbit_degrees: float = 360.0,
                viewport=(128, 128), scene: Scene | None = None,
                brick_budget_bytes: int = 512 * 1024 * 1024, budget_ms: float = 150.0,
                resident_all: bool = False) -> dict:
    """The paper's interactive benchmark (``voxtree bench``, cli.py:209-252):
    ``frames`` full-frame passes on an orbit in the x-z plane around the
    volume centre at 2.5x the largest extent, bricks uploaded between frames
    under ``budget_ms``.  Times are wall clock per render call (the reference
    protocol); returns its summary numbers."""
    desc = tree.descriptor
    vw, vh = int(viewport[0]), int(viewport[1])
    device = (DeviceState(tree, resident_all=True) if resident_all
              else DeviceState(tree, brick_budget_bytes=int(brick_budget_bytes)))
    renderer = OutOfCoreRenderer(device)
    if scene is None:
        scene = Scene(_default_camera(desc, (vw, vh)), RenderSettings(),
                      [TransferFunction.ramp(max_alpha=0.8) for _ in range(desc.channels)])
    centre = np.array([d * s / 2.0 for d, s in zip(desc.dims, desc.spacing)])
    radius = 2.5 * max(d * s for d, s in zip(desc.dims, desc.spacing))
    times, fallbacks = [], []
    uploads0 = device.uploads
    for i in range(frames):
        a = np.deg2rad(orbit_degrees) * i / frames
        pos = centre + radius * np.array([np.sin(a), 0.0, -np.cos(a)])
        scene.camera = Camera(position=tuple(pos), look_at=tuple(centre), up=(0, 1, 0),
                              fov_y=scene.camera.fov_y, width=vw, height=vh)
        t0 = time.perf_counter()
        _, counters = renderer.render_fullframe(scene)
        times.append(time.perf_counter() - t0)
        fallbacks.append(counters.avg_fallbacks)
        device.upload_bricks(device.process_flags(RenderMode.FULLFRAME), budget_ms)
    ms = np.asarray(times) * 1e3
    return {"frames": frames, "mean_ms": float(ms.mean()),
            "p50_ms": float(np.percentile(ms, 50)), "p95_ms": float(np.percentile(ms, 95)),
            "fps": float(1e3 / ms.mean()), "avg_fallbacks_first": int(fallbacks[0]),
            "avg_fallbacks_last": int(fallbacks[-1]),
            "bricks_uploaded": int(device.uploads - uploads0)}
