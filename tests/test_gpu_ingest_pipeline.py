"""The pipelined VSTR ingest (reader thread + pinned brick-layer-pair buffers
+ pooled CRC32 + one insert_many per pair) against the reference's
per-frame loop (ingest.py:306-358, `workers=0` here): the same tree (VXOC /
VXBP after fill_borders), the same queued change events, the same result
counters — with NACKed slabs, repeated slices, general blocks between
slices, an abort, a checksum error and should_stop() in the middle of a
pair, at threshold 0 and > 0."""

import io

import numpy as np
import pytest

from gpu_helpers import digest, make_tree

pytestmark = pytest.mark.gpu

DIMS, C, BRICK = (96, 80, 72), 3, 16


def _vol(seed=3):
    import voxtree_oracle as vo
    return vo.synth_spim(DIMS, C, 65535, seed=seed)


def _spec(threshold=0):
    return dict(dims=DIMS, brick=(BRICK,) * 3, threshold=threshold, fmt="uint16", channels=C)


def _stream(desc, frames, tail="end"):
    from paper_1407_2074_b200.ingest import encode_abort, encode_end, encode_handshake
    blob = [encode_handshake(desc)] + frames
    if tail == "end":
        blob.append(encode_end())
    elif tail == "abort":
        blob.append(encode_abort())
    s = io.BytesIO(b"".join(blob))
    return s


def _frames(desc, vol, extra=()):
    """VSTR slice order; `extra` inserts (index, frame bytes) at positions."""
    from paper_1407_2074_b200.ingest import encode_slab
    out = []
    for z in range(DIMS[2]):
        for c in range(C):
            out.append(encode_slab(desc, c, (0, 0, z), vol[z:z + 1, :, :, c]))
    for i, f in sorted(extra, key=lambda e: -e[0]):
        out.insert(i, f)
    return out


def _run(spec, blob_fn, workers, **kw):
    from paper_1407_2074_b200.ingest import ingest_stream, read_handshake
    t = make_tree(spec)
    s = blob_fn(t.descriptor)
    read_handshake(s)
    err = None
    try:
        res = ingest_stream(s, t, workers=workers, **kw)
    except Exception as exc:  # noqa: BLE001 - compared between the two paths
        res, err = None, type(exc).__name__
        t.finalize()
        t.fill_borders()
    ev = t.drain_event_arrays()
    return t, res, err, ev


def _same(a, b, tmp_path):
    (ta, ra, ea, eva), (tb, rb, eb, evb) = a, b
    assert ea == eb
    if ra is not None:
        assert (ra.slabs, ra.rejected, ra.aborted, ra.nacks) == \
               (rb.slabs, rb.rejected, rb.aborted, rb.nacks)
    assert np.array_equal(eva[0], evb[0]) and np.array_equal(eva[1], evb[1])
    assert ta.checksum() == tb.checksum()
    assert digest(ta, str(tmp_path), "a") == digest(tb, str(tmp_path), "b")


@pytest.mark.parametrize("threshold", [0, None])
def test_pipelined_stream_equals_per_frame(tmp_path, threshold):
    from paper_1407_2074_b200.ingest import encode_slab
    vol = _vol()
    spec = _spec(threshold)

    def blob(desc):
        other = vol[10:14, 20:50, 5:60, 1]
        extra = [(7, encode_slab(desc, 1, (5, 20, 10), other)),          # general block
                 (40, encode_slab(desc, 0, (0, 0, 70), vol[:3, :, :, 0])),  # out of bounds
                 (41, encode_slab(desc, 5, (0, 0, 3), vol[3:4, :, :, 0])),  # bad channel
                 (100, encode_slab(desc, 2, (0, 0, 30), vol[31:32, :, :, 2]))]  # repeat z 30
        return _stream(desc, _frames(desc, vol, extra))

    a = _run(spec, blob, 0)
    b = _run(spec, blob, 4)
    assert b[1].rejected == 2 and b[1].slabs == DIMS[2] * C + 2
    _same(a, b, tmp_path)


@pytest.mark.parametrize("cut", [1, 50, 95, 150])
def test_pipelined_abort_and_stop_mid_pair(tmp_path, cut):
    vol = _vol(seed=8)
    spec = _spec()

    def blob(desc):
        return _stream(desc, _frames(desc, vol)[:cut], tail="abort")

    _same(_run(spec, blob, 0), _run(spec, blob, 3), tmp_path)
    calls = {"n": 0}

    def stop_after():
        calls["n"] += 1
        return calls["n"] > cut

    def blob_full(desc):
        return _stream(desc, _frames(desc, vol))

    a = _run(spec, blob_full, 0, should_stop=stop_after)
    calls["n"] = 0
    b = _run(spec, blob_full, 3, should_stop=stop_after)
    assert a[1].aborted and b[1].aborted and a[1].slabs == b[1].slabs == cut
    _same(a, b, tmp_path)


def test_pipelined_checksum_error_inserts_the_frames_before(tmp_path):
    vol = _vol(seed=5)
    spec = _spec()

    def blob(desc):
        fr = _frames(desc, vol)
        bad = bytearray(fr[130])
        bad[-1] ^= 0xFF  # payload byte: the CRC no longer matches
        fr[130] = bytes(bad)
        return _stream(desc, fr)

    a = _run(spec, blob, 0)
    b = _run(spec, blob, 4)
    assert a[2] == "ProtocolError"
    _same(a, b, tmp_path)
