"""Wire-format golden for the VSTR slab stream: bytes produced by the
UNMODIFIED reference encoder (voxtree.ingest) — run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_vstr_golden.py

Writes tests/golden/vstr_stream.bin (handshake with channel transforms, two
slab frames, an out-of-bounds frame, end marker) and vstr_stream.json (the
decoded expectations)."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from voxtree.ingest import encode_end, encode_handshake, encode_slab  # noqa: E402
from voxtree.volume import VolumeDescriptor  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

tr = np.stack([np.eye(4), np.eye(4)])
tr[1, 0, 3] = 1.5
desc = VolumeDescriptor(dims=(6, 5, 4), channels=2, sample_format="uint16",
                        spacing=(1.0, 0.5, 2.0), background_value=7, channel_transforms=tr)
rng = np.random.default_rng(11)
a = rng.integers(0, 65535, size=(2, 5, 6), dtype=np.uint16)
b = rng.integers(0, 65535, size=(1, 3, 4), dtype=np.uint16)
blob = (encode_handshake(desc) + encode_slab(desc, 0, (0, 0, 0), a) +
        encode_slab(desc, 1, (2, 1, 3), b) + encode_slab(desc, 0, (5, 0, 0), b) + encode_end())
with open(os.path.join(HERE, "vstr_stream.bin"), "wb") as fh:
    fh.write(blob)
with open(os.path.join(HERE, "vstr_stream.json"), "w") as fh:
    json.dump({"dims": [6, 5, 4], "channels": 2, "format": "uint16", "spacing": [1.0, 0.5, 2.0],
               "background": 7, "transform1_03": 1.5, "slab_a": a.tolist(), "slab_b": b.tolist(),
               "nbytes": len(blob)}, fh)
print("wrote", len(blob), "bytes")
