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


def _png(rgba: np.ndarray) -> bytes:
    from PIL import Image
    sink = io.BytesIO()
    Image.fromarray(rgba, "RGBA").save(sink, format="PNG")
    return sink.getvalue()


def encode_frame(frame_id: int, image: np.ndarray) -> bytes:
    """Header + PNG of the RGBA8 conversion of a float (H, W, 4) image."""
    rgba = image_to_rgba8(image)
    head = FRAME_HEADER.pack(frame_id, rgba.shape[1], rgba.shape[0], PIXEL_FORMAT_PNG_RGBA)
    return head + _png(rgba)


def decode_frame(blob: bytes):
    """(frame_id, width, height, format, RGBA8 array) of an encoded frame."""
    from PIL import Image
    head = FRAME_HEADER.unpack_from(blob, 0)
    pixels = np.asarray(Image.open(io.BytesIO(memoryview(blob)[FRAME_HEADER.size:])))
    return (*head, pixels)


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


@dataclass
class _SceneState:
    """What a viewer controls; ``version`` counts accepted changes."""
    camera: Camera
    tfs: list
    clips: ClipSet
    settings: RenderSettings
    version: int = 0

    def as_scene(self) -> Scene:
        return Scene(camera=self.camera, settings=self.settings,
                     transfer_functions=list(self.tfs), clips=self.clips)

    def restyled(self, **changes) -> RenderSettings:
        s = self.settings
        base = {f: getattr(s, f) for f in ("mode", "strategy", "sampling_step",
                                            "reference_step", "early_termination_alpha",
                                            "lod_bias", "precision", "empty_space_skip")}
        base.update(changes)
        return RenderSettings(**base)

    def describe(self) -> dict:
        c = self.camera
        cam = {"position": list(c.position), "look_at": list(c.look_at), "up": list(c.up),
               "fov_deg": float(np.rad2deg(c.fov_y)), "viewport": [c.width, c.height]}
        return {"camera": cam, "mode": self.settings.mode, "strategy": self.settings.strategy,
                "transfer_functions": [tf.control_points() for tf in self.tfs],
                "clip_planes": [[*p.normal, p.offset] for p in self.clips]}


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
        nch = tree.descriptor.channels
        self._lock = threading.Lock()
        self._state = _SceneState(camera=_default_camera(tree.descriptor, viewport),
                                  tfs=[TransferFunction.ramp(max_alpha=0.8) for _ in range(nch)],
                                  clips=ClipSet(), settings=RenderSettings(strategy="refinement"))
        self._shown_version = -1   # the scene version the loop last restarted for
        self._session = None       # refinement session of the shown scene
        self._stable = False       # a full-frame pass requested / uploaded nothing
        self.frame_id = 0
        self.refinement_complete = False
        self._clients: list[_Client] = []
        self._stop = threading.Event()
        self._ingest_abort = threading.Event()
        self._ingest_thread: threading.Thread | None = None
        self._render_thread: threading.Thread | None = None

    @property
    def _settings(self) -> RenderSettings:
        return self._state.settings

    def current_scene(self) -> Scene:
        with self._lock:
            return self._state.as_scene()

    # -- control messages (one handler per message type) ---------------------
    def _on_camera(self, m):
        cam = self._state.camera
        w, h = m.get("viewport", [cam.width, cam.height])
        fov = float(np.deg2rad(m["fov_deg"])) if "fov_deg" in m else cam.fov_y
        self._state.camera = Camera(position=tuple(m.get("position", cam.position)),
                                    look_at=tuple(m.get("look_at", cam.look_at)),
                                    up=tuple(m.get("up", cam.up)), fov_y=fov,
                                    width=int(w), height=int(h))

    def _on_transfer_function(self, m):
        ch = int(m["channel"])
        if ch < 0 or ch >= self.tree.descriptor.channels:
            raise ValueError(f"channel {ch} out of range")
        self._state.tfs[ch] = TransferFunction(m["points"])

    def _on_clip_planes(self, m):
        planes = [ClipPlane(tuple(q[:3]), float(q[3])) for q in m.get("planes", [])]
        self._state.clips = ClipSet(tuple(planes))

    def _on_mode(self, m):
        self._state.settings = self._state.restyled(mode=m["mode"])

    def _on_strategy(self, m):
        self._state.settings = self._state.restyled(strategy=m["strategy"])

    def _on_reset_refinement(self, m):
        """Nothing to change: the version bump restarts the loop."""

    def _on_abort_ingest(self, m):
        self._ingest_abort.set()

    def handle_control(self, message: str) -> dict:
        """Apply one JSON control message; the ack / nack reply echoes its id."""
        msg = None
        try:
            msg = json.loads(message)
            if not isinstance(msg, dict) or "type" not in msg:
                raise ValueError("control message must be an object with a type")
            kind, mid = msg["type"], msg.get("id")
            if kind == "ping":
                return {"type": "ack", "id": mid}
            if kind == "get_settings":
                with self._lock:
                    return {"type": "settings", "id": mid, **self._state.describe()}
            apply = getattr(self, f"_on_{kind}", None) if isinstance(kind, str) else None
            if apply is None:
                raise ValueError(f"unknown control type {kind!r}")
            with self._lock:
                apply(msg)
                self._state.version += 1
            return {"type": "ack", "id": mid}
        except Exception as exc:  # a bad message is answered, never fatal
            return {"type": "nack", "id": msg.get("id") if isinstance(msg, dict) else None,
                    "error": str(exc)}

    # -- live ingest ------------------------------------------------------------
    def attach_ingest(self, stream) -> threading.Thread:
        """Consume a VSTR stream (after its handshake) while rendering."""
        def consume():
            ingest_stream(stream, self.tree, should_stop=self._ingest_abort.is_set)

        self._ingest_thread = threading.Thread(target=consume, name="ingest", daemon=True)
        self._ingest_thread.start()
        return self._ingest_thread

    @property
    def ingest_active(self) -> bool:
        th = self._ingest_thread
        return bool(th and th.is_alive())

    def construction_progress(self) -> float:
        d = self.tree.descriptor
        done = self.tree.inserted_voxels / float(d.voxel_count * d.channels)
        return min(100.0, 100.0 * done)

    # -- render loop -------------------------------------------------------------
    def _sync_changes(self) -> Scene:
        """Apply pending tree events to the mirror; a scene or data change
        restarts the loop.  Returns the scene to draw."""
        events = self.tree.drain_events()
        changed = len(events) > 0
        if changed:
            self.device.apply_events(events)
        with self._lock:
            scene, version = self._state.as_scene(), self._state.version
        if changed or version != self._shown_version:
            self._shown_version = version
            self._session, self._stable, self.refinement_complete = None, False, False
        return scene

    def _fullframe(self, scene: Scene) -> None:
        image, counters = self.renderer.render_fullframe(scene)
        uploaded = self.device.upload_bricks(self.device.process_flags(RenderMode.FULLFRAME),
                                             self.upload_budget_ms)
        self._stable = counters.bricks_requested == 0 and uploaded == 0
        self._broadcast(image)

    def _refine(self, scene: Scene) -> bool:
        if self._session is None:
            self._session = self.renderer.start_refinement(scene)
        if not self._session.run_pass():
            self.device.upload_bricks(self.device.process_flags(RenderMode.REFINEMENT),
                                      self.upload_budget_ms)
            self._push_all(self._status_json())
            return False
        self.refinement_complete = True
        self._broadcast(self._session.image())
        return True

    def step(self) -> bool:
        """One loop iteration; True when a frame was broadcast."""
        scene = self._sync_changes()
        if not self._stable:
            self._fullframe(scene)
            return True
        if self._settings.strategy == "refinement" and not self.refinement_complete:
            return self._refine(scene)
        return False

    def _push_all(self, payload) -> None:
        for client in list(self._clients):
            client.push(payload)

    def _broadcast(self, image: np.ndarray) -> None:
        self.frame_id += 1
        for payload in (encode_frame(self.frame_id, image), self._status_json()):
            self._push_all(payload)

    def _status_json(self) -> str:
        s = self._settings
        return json.dumps({"type": "status", "frame_id": self.frame_id,
                           "construction_pct": round(self.construction_progress(), 2),
                           "bricks_resident": self.device.resident_bricks,
                           "refinement_complete": self.refinement_complete,
                           "ingest_active": self.ingest_active, "mode": s.mode,
                           "strategy": s.strategy})

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
            self._state.version += 1  # a new viewer gets a fresh frame
        return client

    def unregister_client(self, client: _Client) -> None:
        client.closed = True
        if client in self._clients:
            self._clients.remove(client)


def serve(service: FrameService, host: str = "127.0.0.1", port: int = 8765):
    """Websocket transport (service.py:320-349): per viewer, a sender thread
    drains its outbox (binary frames, status text) while the connection's
    text messages are answered as controls."""
    from websockets.sync.server import serve as ws_serve

    def pump(conn, client: _Client) -> None:
        while not client.closed:
            if not client.ready.wait(0.25):
                continue
            client.ready.clear()
            try:
                while client.queue:
                    conn.send(client.queue.popleft())
            except Exception:  # the viewer went away
                client.closed = True

    def session(conn) -> None:
        client = service.register_client()
        threading.Thread(target=pump, args=(conn, client), daemon=True).start()
        try:
            for message in conn:
                if isinstance(message, str):
                    conn.send(json.dumps(service.handle_control(message)))
        finally:
            service.unregister_client(client)

    service.start()
    try:
        with ws_serve(session, host, port) as server:
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
    extent = np.asarray(desc.dims, np.float64) * np.asarray(desc.spacing, np.float64)
    centre = extent / 2.0
    angles = np.deg2rad(orbit_degrees) * np.arange(frames) / frames
    ring = centre + 2.5 * extent.max() * np.stack(
        [np.sin(angles), np.zeros_like(angles), -np.cos(angles)], axis=1)
    times, fallbacks = [], []
    uploads0 = device.uploads
    for pos in ring:
        scene.camera = Camera(position=tuple(float(v) for v in pos),
                              look_at=tuple(float(v) for v in centre), up=(0, 1, 0),
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
