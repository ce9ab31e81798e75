"""ctypes binding of libvtx.so (include/vtx.h).

The product path has no CPU fallback: if the shared library is missing or
cannot be loaded, every entry point raises ``RuntimeError`` naming the
build command.  Status codes map to the reference's exception types
(include/vtx.h conventions).
"""

from __future__ import annotations

import ctypes as ct
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# VT_LIB: an alternate build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("VT_LIB") or os.path.join(HERE, "libvtx.so")

VT_OK, VT_EINVAL, VT_EOVERFLOW, VT_ENOMEM, VT_ECUDA, VT_ESTATE, VT_EIO = range(7)
VT_MEM_HOST, VT_MEM_DEVICE = 0, 1
NODE_EXISTS, NODE_CHILDREN, NODE_IN_VOLUME, NODE_BRICK = 1, 2, 4, 8
MAX_TF_POINTS = 16


class StoreIOError(Exception):
    """Disk failure or corruption in the brick-pool file (paging.py:37-38)."""


class vt_tree_desc(ct.Structure):
    _fields_ = [("dims", ct.c_int32 * 3), ("channels", ct.c_int32),
                ("sample_bytes", ct.c_int32), ("background", ct.c_int32),
                ("brick", ct.c_int32 * 3), ("threshold", ct.c_double),
                ("reserve_slots", ct.c_int64), ("device", ct.c_int32)]


class vt_tree_info(ct.Structure):
    _fields_ = [("node_count", ct.c_int64), ("brick_count", ct.c_int64),
                ("pruned_bricks", ct.c_int64), ("inserted_voxels", ct.c_int64),
                ("capacity", ct.c_int64), ("pool_slots", ct.c_int64), ("depth", ct.c_int32),
                ("virtual_dims", ct.c_int32 * 3), ("finished", ct.c_int32),
                ("borders_filled", ct.c_int32)]


class vt_node(ct.Structure):
    _fields_ = [("flags", ct.c_int32), ("level", ct.c_int32), ("box_lo", ct.c_int32 * 3),
                ("slot", ct.c_int32), ("stats", (ct.c_int32 * 5) * 4)]


class vt_scene(ct.Structure):
    _fields_ = [("position", ct.c_double * 3), ("fwd", ct.c_double * 3),
                ("right", ct.c_double * 3), ("up", ct.c_double * 3),
                ("tan_half", ct.c_double), ("aspect", ct.c_double),
                ("footprint_scale", ct.c_double), ("width", ct.c_int32), ("height", ct.c_int32),
                ("mode_mip", ct.c_int32), ("step", ct.c_double), ("corr_exp", ct.c_double),
                ("et_limit", ct.c_double), ("lod_scale", ct.c_double),
                ("tf_count", ct.c_int32 * 4), ("tf_x", (ct.c_double * MAX_TF_POINTS) * 4),
                ("tf_rgba", ((ct.c_double * 4) * MAX_TF_POINTS) * 4),
                ("n_clips", ct.c_int32), ("clip_normal", (ct.c_double * 3) * 3),
                ("clip_offset", ct.c_double * 3), ("spacing", ct.c_double * 3),
                ("has_transforms", ct.c_int32), ("transforms", (ct.c_double * 12) * 4),
                ("precision", ct.c_int32), ("empty_skip", ct.c_int32)]


class vt_counters(ct.Structure):
    _fields_ = [("samples", ct.c_int64), ("tf_lookups", ct.c_int64),
                ("avg_fallbacks", ct.c_int64), ("coarse_fallbacks", ct.c_int64),
                ("bricks_requested", ct.c_int64), ("bricks_used_marks", ct.c_int64),
                ("samples_skipped", ct.c_int64)]


class vt_block(ct.Structure):
    _fields_ = [("channel", ct.c_int32), ("origin", ct.c_int32 * 3), ("dims", ct.c_int32 * 3),
                ("pad", ct.c_int32), ("samples", ct.c_void_p)]


P = ct.c_void_p
I32, I64, U32 = ct.c_int32, ct.c_int64, ct.c_uint32
PI32, PI64 = ct.POINTER(ct.c_int32), ct.POINTER(ct.c_int64)

# name -> argtypes (all return vt_status)
SIGNATURES = {
    "vt_tree_create": [ct.POINTER(vt_tree_desc), ct.POINTER(P)],
    "vt_tree_destroy": [P],
    "vt_tree_set_stream": [P, P],
    "vt_tree_insert": [P, I32, PI32, PI32, P, I32],
    "vt_tree_insert_channels": [P, PI32, PI32, P, I32],
    "vt_tree_insert_ev": [P, I32, PI32, PI32, P, I32, P, PI32, PI64, I64, PI64],
    "vt_tree_insert_many": [P, I64, ct.POINTER(vt_block), I32, P],
    "vt_tree_stream_counts": [P, PI64, PI64, PI64],
    "vt_tree_publish_halos": [P],
    "vt_mirror_bmax_stats": [P, PI64, PI64],
    "vt_tree_take_events": [P, PI32, PI64, I64, PI64, PI32],
    "vt_tree_copy_events": [P, I64, I64, PI32, PI64],
    "vt_tree_event_count": [P, PI64],
    "vt_tree_checksum": [P, ct.POINTER(ct.c_uint64)],
    "vt_tree_export_nodes": [P, I64, PI64, PI32, PI32, P, I32],
    "vt_tree_merge": [P, I64, PI64, PI32, PI32, P, I32, I64],
    "vt_tree_wait_stream": [P, P],
    "vt_tree_signal_stream": [P, P],
    "vt_tree_set_dense": [P, I32],
    "vt_tree_dense_counts": [P, PI64, PI64, PI64],
    "vt_tree_finalize": [P],
    "vt_tree_fill_borders": [P],
    "vt_tree_sync": [P],
    "vt_tree_flush": [P],
    "vt_tree_info_get": [P, ct.POINTER(vt_tree_info)],
    "vt_tree_node": [P, I64, ct.POINTER(vt_node), PI32],
    "vt_tree_list_nodes": [P, PI64, PI32, I64, PI64],
    "vt_tree_find_node": [P, ct.POINTER(ct.c_double), I32, PI64],
    "vt_tree_read_brick": [P, I64, P],
    "vt_tree_export": [P, I64, PI64, PI32, P],
    "vt_tree_import": [P, I64, PI64, PI32, PI32, P, I32, I32, I64],
    "vt_halfsample": [PI32, PI32, PI32, PI32, I32, PI32, I32],
    "vt_mirror_create": [P, I64, ct.POINTER(P)],
    "vt_mirror_destroy": [P],
    "vt_mirror_buffers": [P, ct.POINTER(P), ct.POINTER(P), ct.POINTER(P), PI64, PI64],
    "vt_mirror_set_resident": [P, I64, PI64, PI32, I32],
    "vt_mirror_repack": [P],
    "vt_mirror_apply_queued": [P, PI64, PI64],
    "vt_mirror_read_flags": [P, P, I32],
    "vt_rays_create": [P, ct.POINTER(vt_scene), PI32, ct.POINTER(P)],
    "vt_rays_destroy": [P],
    "vt_rays_march": [P, I32, ct.POINTER(vt_counters), PI64],
    "vt_rays_image": [P, P, ct.POINTER(vt_counters)],
    "vt_rays_state": [P, PI64, PI64, P],
    "vt_render_fullframe": [P, ct.POINTER(vt_scene), P, I32, I32, ct.POINTER(vt_counters)],
    "vt_render_tile": [P, ct.POINTER(vt_scene), PI32, P, I32, I32, ct.POINTER(vt_counters)],
    "vt_render_strips": [P, ct.POINTER(vt_scene), I32, I32, I32, P, I32, I32,
                         ct.POINTER(vt_counters)],
    "vt_strip_part_rows": [I32, I32, I32],
    "vt_synth": [P, I32, PI32, I32, I32, U32, I32, I32, P],
    "vt_last_kernel_ms": [P, ct.POINTER(ct.c_double), ct.POINTER(ct.c_double)],
}

_lib = None


def lib():
    """Load libvtx.so once; raise loudly if it is absent (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libvtx.so not built at {LIB_PATH}; run `make -C paper_1407_2074_b200/csrc` "
            "or __graft_entry__.build() (there is no CPU fallback)")
    L = ct.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ct.c_int32
    L.vt_last_error.restype = ct.c_char_p
    L.vt_last_error.argtypes = []
    L.vt_abi_version.restype = ct.c_int32
    _lib = L
    return L


def check(status: int) -> None:
    if status == VT_OK:
        return
    msg = lib().vt_last_error().decode("utf-8", "replace")
    if status == VT_EINVAL:
        raise ValueError(msg)
    if status == VT_EOVERFLOW:
        raise OverflowError(msg)
    if status == VT_EIO:
        raise StoreIOError(msg)
    raise RuntimeError(f"libvtx error {status}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def i32x3(v):
    return (ct.c_int32 * 3)(*[int(x) for x in v])


def ptr(a, ctype):
    """ctypes pointer to a contiguous numpy array."""
    return a.ctypes.data_as(ct.POINTER(ctype))
