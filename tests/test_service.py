"""The caller side of the render path: FrameService
(voxtree service.py:74-349) and the orbit benchmark (cli.py:209-252).

CPU: the frame wire format (16-byte header + PNG, service.py:45-61).
GPU: control acks / nacks, the loop's full-frame -> refinement progression
(its frames equal the renderer's own images), live VSTR ingest through the
service, the orbit protocol.
"""

import io
import json

import numpy as np
import pytest


def test_frame_wire_format_roundtrip():
    from paper_1407_2074_b200.render import image_to_rgba8
    from paper_1407_2074_b200.service import FRAME_HEADER, decode_frame, encode_frame
    img = np.random.default_rng(0).random((12, 17, 4))
    blob = encode_frame(42, img)
    fid, w, h, fmt, rgba = decode_frame(blob)
    assert (fid, w, h, fmt) == (42, 17, 12, 1)
    assert FRAME_HEADER.size == 16
    assert np.array_equal(rgba, image_to_rgba8(img))


def _service(**kw):
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor
    from paper_1407_2074_b200.service import FrameService
    dims, C = (32, 24, 20), 2
    vol = np.random.default_rng(3).integers(0, 255, size=(dims[2], dims[1], dims[0], C),
                                            dtype=np.uint8)
    vol[:, :8] = 3
    tree = Octree(VolumeDescriptor(dims=dims, channels=C, sample_format="uint8"),
                  BrickPoolConfig(brick_dims=(8, 8, 8), homogeneity_threshold=0))
    tree.insert_channels((0, 0, 0), vol)
    tree.finalize()
    tree.fill_borders()
    return FrameService(tree, viewport=(40, 30), **kw), tree


@pytest.mark.gpu
def test_control_messages_ack_nack():
    svc, _ = _service()
    assert svc.handle_control(json.dumps({"type": "ping", "id": 7})) == {"type": "ack", "id": 7}
    r = svc.handle_control(json.dumps({"type": "camera", "id": 1, "fov_deg": 30,
                                       "viewport": [20, 10]}))
    assert r == {"type": "ack", "id": 1}
    st = svc.handle_control(json.dumps({"type": "get_settings", "id": 2}))
    assert st["camera"]["viewport"] == [20, 10] and abs(st["camera"]["fov_deg"] - 30) < 1e-9
    assert st["strategy"] == "refinement" and len(st["transfer_functions"]) == 2
    bad = svc.handle_control(json.dumps({"type": "transfer_function", "id": 3, "channel": 9,
                                         "points": [[0, 0, 0, 0, 0], [1, 1, 1, 1, 1]]}))
    assert bad["type"] == "nack" and bad["id"] == 3 and "out of range" in bad["error"]
    assert svc.handle_control(json.dumps({"type": "warp", "id": 4}))["type"] == "nack"
    assert svc.handle_control("not json")["type"] == "nack"
    assert svc.handle_control(json.dumps({"type": "clip_planes", "id": 5,
                                          "planes": [[0, 0, 1, 10.0]]}))["type"] == "ack"
    assert svc.handle_control(json.dumps({"type": "mode", "id": 6, "mode": "mip"}))["type"] == "ack"
    assert svc.current_scene().settings.mode == "mip"


@pytest.mark.gpu
@pytest.mark.parametrize("resident_all", [False, True])
def test_loop_fullframe_then_refinement(resident_all):
    from paper_1407_2074_b200.render import image_to_rgba8
    from paper_1407_2074_b200.service import decode_frame
    svc, _ = _service(resident_all=resident_all, slot_count=None if resident_all else 16)
    client = svc.register_client()
    frames = []
    for _ in range(200):
        if svc.step():
            frames.append([p for p in client.queue if isinstance(p, bytes)][-1])
        if svc.refinement_complete:
            break
    assert svc.refinement_complete and frames
    status = json.loads([p for p in client.queue if isinstance(p, str)][-1])
    assert status["refinement_complete"] and status["construction_pct"] == 100.0
    # the final broadcast is the refinement image of the current scene
    ref = svc.renderer.start_refinement(svc.current_scene())
    while not ref.run_pass():
        pass
    fid, w, h, fmt, rgba = decode_frame(frames[-1])
    assert (w, h) == (40, 30) and fid == svc.frame_id
    assert np.array_equal(rgba, image_to_rgba8(ref.image()))
    # a control message restarts the loop with a full-frame pass
    svc.handle_control(json.dumps({"type": "reset_refinement", "id": 9}))
    assert svc.step() and not svc.refinement_complete


@pytest.mark.gpu
def test_live_ingest_through_the_service(tmp_path):
    from paper_1407_2074_b200 import BrickPoolConfig, Octree, VolumeDescriptor
    from paper_1407_2074_b200.ingest import (encode_end, encode_handshake, encode_slab,
                                             read_handshake)
    from paper_1407_2074_b200.service import FrameService
    dims, C = (16, 16, 16), 2
    desc = VolumeDescriptor(dims=dims, channels=C, sample_format="uint8")
    vol = np.random.default_rng(4).integers(0, 255, size=(16, 16, 16, C), dtype=np.uint8)
    blob = encode_handshake(desc)
    for z in range(16):
        for c in range(C):
            blob += encode_slab(desc, c, (0, 0, z), vol[z:z + 1, :, :, c])
    blob += encode_end()
    s = io.BytesIO(blob)
    read_handshake(s)
    tree = Octree(desc, BrickPoolConfig(brick_dims=(8, 8, 8), homogeneity_threshold=0))
    svc = FrameService(tree, viewport=(24, 24), resident_all=True)
    svc.attach_ingest(s).join(timeout=60)
    assert not svc.ingest_active and svc.construction_progress() == 100.0
    assert tree.borders_filled
    produced = svc.step()
    assert produced and svc.frame_id == 1
    ref = Octree(desc, BrickPoolConfig(brick_dims=(8, 8, 8), homogeneity_threshold=0))
    ref.insert_channels((0, 0, 0), vol)
    ref.finalize()
    ref.fill_borders()
    assert tree.checksum() == ref.checksum()


@pytest.mark.gpu
def test_orbit_bench_protocol():
    from paper_1407_2074_b200.service import orbit_bench
    _, tree = _service()
    r = orbit_bench(tree, frames=8, viewport=(32, 32))
    assert r["frames"] == 8 and r["mean_ms"] > 0 and r["p95_ms"] >= r["p50_ms"]
    r2 = orbit_bench(tree, frames=4, viewport=(32, 32), resident_all=True)
    assert r2["avg_fallbacks_first"] == 0 and r2["bricks_uploaded"] == 0
