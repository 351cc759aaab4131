"""ctypes binding of libts_b200.so (the C ABI in include/ts_b200.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
fallback: if the shared object is missing the import fails loudly, and
every compute entry point needs a CUDA device.  ctypes releases the GIL for
the duration of each call, so the reference's threaded callers
(server.py:49-56) keep running concurrently.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# TS_LIB_PATH: a profiling build of the same sources (make PROFILE=1,
# scripts only); the product always loads the in-tree library
LIB_PATH = os.environ.get("TS_LIB_PATH") or os.path.join(HERE, "libts_b200.so")

P = C.c_void_p
I32 = C.c_int
I64 = C.c_int64
F64 = C.c_double
SZ = C.c_size_t

# ts_tile_desc (include/ts_b200.h) as a numpy structured dtype
TILE_DESC = np.dtype([
    ("file_offset", "<i8"), ("file_size", "<i8"),
    ("point_data_offset", "<i8"), ("point_count", "<i8"),
    ("las_stride", "<i8"), ("chunk_size", "<u4"), ("format", "<i4"),
    ("record_length", "<i4"), ("compressed", "<i4"),
    ("scale", "<f8", (3,)), ("offset", "<f8", (3,)),
    ("image_base", "<i8"), ("table_pos", "<i8")], align=True)
assert TILE_DESC.itemsize == 120
TABLE_POS_IN_IMAGE = -2

# name -> (restype, argtypes); every symbol include/ts_b200.h declares
SIGNATURES = {
    "ts_version": (C.c_char_p, []),
    "ts_device_count": (I32, []),
    "ts_launch_count": (C.c_uint64, []),
    "ts_record_size": (I32, [I32]),
    "ts_chunk_counts": (I32, [P, P, I32, P, P, P]),
    "ts_chunk_decode_scratch": (SZ, [I32]),
    "ts_chunk_decode": (I32, [P, P, I32, P, P, P, P, P, P, P]),
    "ts_extract_chunk_points": (I32, [P, P, I32, P, P, P, P, P, P, P, P]),
    "ts_lazdec_scratch": (SZ, [I64]),
    "ts_lazdec": (I32, [P, P, I32, P, P, P, P, P, I64, P, P, P, P]),
    "ts_positions": (I32, [P, I64, I32, P, P, P, P]),
    "ts_colors": (I32, [P, I64, I32, I32, P, P, P]),
    "ts_index_build": (I32, [P, I64, I64, I64, I64, I64, P, P, P, P]),
    "ts_gather_count": (I32, [P, P, P, P, I64, I64, I64, I64, P, I32, F64,
                              P, P]),
    "ts_gather_fill": (I32, [P, P, P, P, P, I64, I64, I64, I64, P, I32, F64,
                             P, P, P, P, P, P, P, P]),
    "ts_nearest": (I32, [P, I64, P, I64, P, P]),
    "ts_cell_keys": (I32, [P, I64, P, P]),
    "ts_triangulate_scratch": (SZ, [I64, I32]),
    "ts_triangulate": (I32, [P, P, I32, P, P, P, P, P]),
    "ts_raster": (I32, [P, P, P, P, P, P, P, P, I32, I32, P, P, P, P, P, P,
                        P, P, P]),
    "ts_weights_create": (I32, [P, SZ, I32, C.POINTER(P)]),
    "ts_weights_destroy": (I32, [P]),
    "ts_weights_is_identity": (I32, [P]),
    "ts_refine_workspace": (SZ, [P, I32]),
    "ts_refine": (I32, [P, P, I32, P, P, P, P]),
    "ts_conv2d": (I32, [P, I32, I32, I32, I32, P, I32, I32, P, I32, I32, I32, P,
                        P]),
    "ts_bake_workspace": (SZ, [I32]),
    "ts_bake_bin_scratch": (SZ, [I64, I32, I32]),
    "ts_bake_bin": (I32, [P, P, I64, F64, F64, I32, I32, P, P, P, P]),
    "ts_bake": (I32, [P, P, I64, P, I32, P, P, P, F64, F64, I32, I32, P, P, P,
                      P, P, P, P, P]),
    "ts_wire_record_size": (SZ, [I32]),
    "ts_wire_heightmaps": (I32, [P, P, P, P, I32, I32, P, P]),
    "ts_render_points": (I32, [P, P, I64, P, C.c_uint32, P, P]),
    "ts_render_heightmaps_scratch": (SZ, [I32]),
    "ts_render_heightmaps": (I32, [P, P, P, P, P, I32, P, P, P, P]),
    "ts_render_resolve": (I32, [P, I64, P, P, P, P]),
    "ts_bbox_areas": (I32, [P, I64, P, P, P, P, P]),
    "ts_incircle_sign": (I32, [P, P, P, P]),
    "ts_orient_sign": (I32, [P, P, P]),
    "ts_predicates_device": (I32, [P, I64, I32, P, P]),
}

_LIB = None


def lib():
    """The loaded library; raises if it has not been built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -c 'import "
                f"__graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB
