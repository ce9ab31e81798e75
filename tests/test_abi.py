"""CPU-side checks of the drop-in boundary: libvtx.so loads without a GPU
and exports every entry point include/vtx.h declares; the ctypes signature
table covers the header; host-side config validation mirrors the
reference's errors (voxtree/volume.py)."""

import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vtx.h")
LIB = os.path.join(ROOT, "paper_1407_2074_b200", "libvtx.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vt_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1407_2074_b200 import _lib
    L = _lib.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (vt_[a-z_0-9]+)", out))
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    assert L.vt_abi_version() == 1


def test_ctypes_table_covers_header():
    from paper_1407_2074_b200 import _lib
    skip = {"vt_last_error", "vt_abi_version"}
    assert sorted(set(declared()) - skip) == sorted(_lib.SIGNATURES)


def test_struct_sizes_match_header():
    """ctypes struct layouts == the C structs (compiled probe)."""
    from paper_1407_2074_b200 import _lib
    probe = os.path.join(ROOT, "build", "sizes")
    os.makedirs(os.path.dirname(probe), exist_ok=True)
    src = probe + ".c"
    with open(src, "w") as fh:
        fh.write('#include <stdio.h>\n#include "vtx.h"\nint main(){printf("%zu %zu %zu %zu %zu\\n",'
                 'sizeof(vt_tree_desc),sizeof(vt_tree_info),sizeof(vt_node),sizeof(vt_scene),'
                 'sizeof(vt_counters));return 0;}\n')
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", probe], check=True)
    sizes = [int(v) for v in subprocess.run([probe], capture_output=True, text=True,
                                            check=True).stdout.split()]
    import ctypes as ct
    assert sizes == [ct.sizeof(_lib.vt_tree_desc), ct.sizeof(_lib.vt_tree_info),
                     ct.sizeof(_lib.vt_node), ct.sizeof(_lib.vt_scene),
                     ct.sizeof(_lib.vt_counters)]


def test_error_mapping():
    from paper_1407_2074_b200 import _lib
    _lib.lib()
    with pytest.raises(ValueError):
        d = _lib.vt_tree_desc()
        d.dims[:] = [8, 8, 8]
        d.channels = 9  # rejected before any CUDA call
        d.sample_bytes = 1
        d.brick[:] = [4, 4, 4]
        import ctypes as ct
        h = ct.c_void_p()
        _lib.call("vt_tree_create", ct.byref(d), ct.byref(h))


def test_volume_validation_mirrors_reference():
    from paper_1407_2074_b200 import BrickPoolConfig, TreeGeometry, VolumeDescriptor, virtual_dims
    with pytest.raises(ValueError):
        VolumeDescriptor(dims=(0, 1, 1))
    with pytest.raises(ValueError):
        VolumeDescriptor(dims=(4, 4, 4), channels=5)
    with pytest.raises(ValueError):
        BrickPoolConfig(brick_dims=(3, 4, 4))
    assert virtual_dims((1004, 1002, 1611), (64, 64, 64)) == ((2048, 2048, 2048), 5)
    assert virtual_dims((20, 16, 16), (8, 16, 16)) == ((32, 16, 16), 2)
    assert virtual_dims((16, 1, 1), (4, 1, 1)) == ((16, 1, 1), 2)
    assert virtual_dims((2048, 2048, 1000), (32, 32, 32)) == ((2048, 2048, 2048), 6)
    g = TreeGeometry.build(VolumeDescriptor(dims=(16, 16, 16)), BrickPoolConfig(brick_dims=(4, 4, 4)))
    assert g.node_capacity == 73 and g.level_of_index(9) == 0
    assert g.box_lo_of_index(8 * 1 + 1 + 7) == (4, 4, 4)  # child 7 of node 1 (level 0)
    assert g.box_lo_of_index(72) == (12, 12, 12)  # last level-0 node
    with pytest.raises(ValueError):
        TreeGeometry.build(VolumeDescriptor(dims=(4096, 1, 1)), BrickPoolConfig(brick_dims=(2, 1, 1)))


def test_geometry_matches_oracle():
    import voxtree_oracle as vo
    from paper_1407_2074_b200 import BrickPoolConfig, TreeGeometry, VolumeDescriptor
    rng = np.random.default_rng(0)
    for _ in range(50):
        dims = tuple(int(v) for v in rng.integers(1, 300, 3))
        brick = tuple(int(v) for v in rng.choice([1, 2, 4, 8, 16, 32], 3))
        og = vo.Geo(dims, brick)
        if og.depth > 8:
            continue
        g = TreeGeometry.build(VolumeDescriptor(dims=dims), BrickPoolConfig(brick_dims=brick))
        assert g.virtual == og.virtual and g.depth == og.depth
        for i in rng.integers(0, og.capacity, 20):
            assert g.box_lo_of_index(int(i)) == og.box_lo(int(i))
            assert g.level_of_index(int(i)) == og.level_of(int(i))
