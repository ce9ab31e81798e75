"""Ingest entry points (paper_1407_2074_b200/ingest.py) — the reference's
test_ingest.py behaviours.  CPU: sidecars, raw sources and the VSTR wire
format, pinned to bytes the unmodified reference encoder produced
(tests/golden/vstr_stream.bin).  GPU: bulk and streamed ingestion build
byte-identical trees; NACK / corrupt / abort semantics."""

import hashlib
import io
import json
import os

import numpy as np
import pytest

from paper_1407_2074_b200 import BrickPoolConfig, VolumeDescriptor
from paper_1407_2074_b200.ingest import (ProtocolError, RawVolumeSource, encode_abort,
                                         encode_end, encode_handshake, encode_slab,
                                         ingest_bulk, ingest_stream, read_handshake,
                                         read_sidecar, write_sidecar)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def write_raw(tmp_path, arr, name):
    p = tmp_path / name
    arr.astype(arr.dtype.newbyteorder("<")).tofile(p)
    return p


def make_source(tmp_path, vol, fmt="uint8", bg=0, interleaved=False):
    dz, dy, dx, nc = vol.shape
    desc = VolumeDescriptor(dims=(dx, dy, dz), channels=nc, sample_format=fmt,
                            background_value=bg)
    if interleaved:
        files = write_raw(tmp_path, vol, "all.raw")
    else:
        files = [write_raw(tmp_path, vol[..., c], f"ch{c}.raw") for c in range(nc)]
    side = tmp_path / "vol.txt"
    write_sidecar(side, desc, files)
    return RawVolumeSource.from_sidecar(side)


# -- CPU ---------------------------------------------------------------------------

def test_sidecar_roundtrip(tmp_path):
    tr = np.stack([np.eye(4), np.eye(4)])
    tr[1, 2, 3] = -2.5
    desc = VolumeDescriptor(dims=(8, 6, 4), channels=2, sample_format="uint16",
                            spacing=(1.0, 2.0, 0.5), background_value=3, channel_transforms=tr)
    side = tmp_path / "v.txt"
    write_sidecar(side, desc, ["a.raw", "b.raw"])
    got, files, inter = read_sidecar(side)
    assert got.dims == desc.dims and got.channels == 2 and got.sample_format == "uint16"
    assert got.spacing == desc.spacing and got.background_value == 3
    assert np.array_equal(got.channel_transforms, tr)
    assert not inter and [os.path.basename(f) for f in files] == ["a.raw", "b.raw"]


def test_raw_source_size_mismatch_rejected(tmp_path):
    vol = np.zeros((4, 4, 4, 1), np.uint8)
    src = make_source(tmp_path, vol)
    with open(src.files[0], "ab") as fh:
        fh.write(b"x")
    with pytest.raises(ValueError):
        RawVolumeSource.from_sidecar(tmp_path / "vol.txt")


def test_interleaved_source_channel_extraction(tmp_path):
    vol = np.random.default_rng(1).integers(0, 255, size=(3, 4, 5, 2), dtype=np.uint8)
    src = make_source(tmp_path, vol, interleaved=True)
    assert src.interleaved
    for c in range(2):
        assert np.array_equal(src.read_channel(c), vol[..., c])
    assert np.array_equal(src.read_interleaved(), vol)


def test_handshake_roundtrip():
    tr = np.stack([np.eye(4)] * 3)
    tr[2, 1, 3] = 4.0
    desc = VolumeDescriptor(dims=(9, 8, 7), channels=3, sample_format="uint8",
                            spacing=(0.5, 1.0, 3.0), background_value=2, channel_transforms=tr)
    got = read_handshake(io.BytesIO(encode_handshake(desc)))
    assert got.dims == desc.dims and got.channels == 3 and got.spacing == desc.spacing
    assert got.background_value == 2 and np.array_equal(got.channel_transforms, tr)


@pytest.mark.parametrize("blob", [b"NOPE\x01\x00", b"VS", b"VSTR\x02\x00" + b"\0" * 40])
def test_bad_handshakes_rejected(blob):
    with pytest.raises(ProtocolError):
        read_handshake(io.BytesIO(blob))


def test_wire_format_matches_reference_encoder():
    """bytes from the unmodified reference encoder decode to the same values,
    and our encoder reproduces them byte for byte"""
    blob = open(os.path.join(GOLD, "vstr_stream.bin"), "rb").read()
    exp = json.load(open(os.path.join(GOLD, "vstr_stream.json")))
    s = io.BytesIO(blob)
    desc = read_handshake(s)
    assert list(desc.dims) == exp["dims"] and desc.channels == 2
    assert list(desc.spacing) == exp["spacing"] and desc.background_value == 7
    assert desc.channel_transforms[1, 0, 3] == exp["transform1_03"]
    a = np.asarray(exp["slab_a"], np.uint16)
    b = np.asarray(exp["slab_b"], np.uint16)
    mine = (encode_handshake(desc) + encode_slab(desc, 0, (0, 0, 0), a) +
            encode_slab(desc, 1, (2, 1, 3), b) + encode_slab(desc, 0, (5, 0, 0), b) +
            encode_end())
    assert mine == blob


# -- GPU ---------------------------------------------------------------------------

def _tree(desc, threshold=0, brick=(4, 4, 4)):
    from paper_1407_2074_b200 import Octree
    return Octree(desc, BrickPoolConfig(brick_dims=brick, homogeneity_threshold=threshold,
                                        page_bricks=16, ram_page_limit=64))


def _digest(tree, tmp_path, tag):
    from paper_1407_2074_b200 import save_octree
    o, p = tmp_path / f"{tag}.vxoc", tmp_path / f"{tag}.vxbp"
    save_octree(tree, o, p)
    return hashlib.sha256(o.read_bytes()).hexdigest(), hashlib.sha256(p.read_bytes()).hexdigest()


@pytest.mark.gpu
@pytest.mark.parametrize("threshold", [0, 12])
def test_bulk_ingest_matches_direct_insertion(tmp_path, threshold):
    vol = np.random.default_rng(2).integers(0, 255, size=(12, 10, 9, 2), dtype=np.uint8)
    vol[:, :5] = 4
    src = make_source(tmp_path, vol)
    t = _tree(src.descriptor, threshold)
    rep = ingest_bulk(src, t)
    ref = _tree(src.descriptor, threshold)
    for c in range(2):
        for z0 in range(0, 12, 4):
            ref.insert_block(c, (0, 0, z0), vol[z0:z0 + 4, :, :, c])
    ref.finalize()
    ref.fill_borders()
    assert _digest(t, tmp_path, "a") == _digest(ref, tmp_path, "b")
    assert rep.brick_count == ref.brick_count and rep.raw_bytes == vol.nbytes
    assert rep.payload_ratio > 0 and "bricks" in rep.summary()


@pytest.mark.gpu
@pytest.mark.parametrize("threshold", [0, 12])
def test_stream_equals_bulk(tmp_path, threshold):
    vol = np.random.default_rng(3).integers(0, 255, size=(8, 8, 8, 2), dtype=np.uint8)
    src = make_source(tmp_path, vol)
    bulk = _tree(src.descriptor, threshold)
    ingest_bulk(src, bulk)
    desc = src.descriptor
    blob = encode_handshake(desc)
    for c in range(2):
        for z0 in range(0, 8, 4):
            blob += encode_slab(desc, c, (0, 0, z0), vol[z0:z0 + 4, :, :, c])
    blob += encode_end()
    s = io.BytesIO(blob)
    st = _tree(read_handshake(s), threshold)
    res = ingest_stream(s, st)
    assert res.slabs == 4 and not res.aborted
    assert _digest(st, tmp_path, "s") == _digest(bulk, tmp_path, "b")


@pytest.mark.gpu
def test_duplicate_slab_is_idempotent(tmp_path):
    vol = np.random.default_rng(4).integers(0, 255, size=(8, 8, 8, 1), dtype=np.uint8)
    desc = VolumeDescriptor(dims=(8, 8, 8), channels=1, sample_format="uint8")
    one = encode_handshake(desc) + encode_slab(desc, 0, (0, 0, 0), vol[..., 0]) + encode_end()
    two = (encode_handshake(desc) + encode_slab(desc, 0, (0, 0, 0), vol[..., 0]) * 2 +
           encode_end())
    digests = []
    for tag, blob in (("one", one), ("two", two)):
        s = io.BytesIO(blob)
        t = _tree(read_handshake(s))
        ingest_stream(s, t)
        digests.append(_digest(t, tmp_path, tag))
    assert digests[0] == digests[1]


@pytest.mark.gpu
def test_out_of_bounds_slab_nacked_stream_continues(tmp_path):
    desc = VolumeDescriptor(dims=(8, 8, 8), channels=1, sample_format="uint8")
    good = np.full((4, 8, 8), 9, np.uint8)
    nacks = []
    blob = (encode_handshake(desc) + encode_slab(desc, 0, (0, 0, 6), good) +
            encode_slab(desc, 3, (0, 0, 0), good) + encode_slab(desc, 0, (0, 0, 0), good) +
            encode_end())
    s = io.BytesIO(blob)
    t = _tree(read_handshake(s))
    res = ingest_stream(s, t, on_nack=nacks.append)
    assert res.rejected == 2 and res.slabs == 1 and len(nacks) == 2
    assert t.borders_filled


@pytest.mark.gpu
def test_corrupt_payload_drops_connection():
    desc = VolumeDescriptor(dims=(8, 8, 8), channels=1, sample_format="uint8")
    frame = bytearray(encode_slab(desc, 0, (0, 0, 0), np.ones((1, 8, 8), np.uint8)))
    frame[-1] ^= 0xFF
    s = io.BytesIO(encode_handshake(desc) + bytes(frame))
    t = _tree(read_handshake(s))
    with pytest.raises(ProtocolError):
        ingest_stream(s, t)


@pytest.mark.gpu
def test_abort_keeps_partial_tree_renderable():
    from paper_1407_2074_b200 import DeviceState
    from paper_1407_2074_b200.render import (Camera, OutOfCoreRenderer, RenderSettings, Scene,
                                             TransferFunction)
    desc = VolumeDescriptor(dims=(8, 8, 8), channels=1, sample_format="uint8")
    blob = (encode_handshake(desc) +
            encode_slab(desc, 0, (0, 0, 0), np.full((4, 8, 8), 200, np.uint8)) +
            encode_abort() + encode_slab(desc, 0, (0, 0, 4), np.full((4, 8, 8), 9, np.uint8)))
    s = io.BytesIO(blob)
    t = _tree(read_handshake(s))
    res = ingest_stream(s, t)
    assert res.aborted and res.slabs == 1 and t.borders_filled
    dev = DeviceState(t, resident_all=True)
    cam = Camera(position=(4.0, 4.0, -20.0), look_at=(4.0, 4.0, 4.0), width=8, height=8)
    img, cnt = OutOfCoreRenderer(dev).render_fullframe(
        Scene(cam, RenderSettings(), [TransferFunction.ramp(max_alpha=0.5)]))
    assert cnt.samples > 0 and img[..., 3].max() > 0
