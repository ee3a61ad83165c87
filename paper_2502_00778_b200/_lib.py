"""ctypes bindings of the two native libraries of the package.

* ``lib/libdualmesh.so``  -- the product: C-ABI of include/dm_capi.h over the
  sm_100a kernels.  Loading it never needs a GPU; every compute entry point
  fails with ``DM_ERR_CUDA`` when no sm_100 device is present.  There is no
  Python or CPU fallback: if the library is missing, import of the engine
  raises.
* ``lib/libdm_meshgen.so`` -- SPEC meshgen (synthetic input grids).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBDIR = os.path.join(_HERE, "lib")

P = C.c_void_p
I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
U64P = C.POINTER(C.c_uint64)
U8P = C.POINTER(C.c_uint8)
I8P = C.POINTER(C.c_int8)
DP = C.POINTER(C.c_double)
FP = C.POINTER(C.c_float)
i32, i64, dbl, u64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64

DM_OK = 0
DM_ERR_INVALID_ARG = -1
DM_ERR_MESH_EDGE_MISMATCH = -2
DM_ERR_EDGE_ABSENT = -3
DM_ERR_CUDA = -4
DM_ERR_OOM = -5
DM_ERR_STATE = -6
DM_ERR_UNSUPPORTED = -7

DM_NAV_TRADITIONAL = 0
DM_NAV_DUALFREE = 1
DM_VOL_EDGE = 0
DM_VOL_ELEMENT = 1
DM_VARIANT_GATHER = 0
DM_VARIANT_SCATTER = 1
DM_VARIANT_GATHER_ELEM = 2
DM_VARIANT_GATHER_FACES = 3
DM_VARIANT_GATHER_EXACT = 4

DM_VCOUNT = 8

# name -> (restype, argtypes); mirrors include/dm_capi.h exactly.
CAPI = {
    "dm_version": (C.c_int, []),
    "dm_status_string": (C.c_char_p, [C.c_int]),
    "dm_create": (C.c_int, [C.POINTER(P), C.c_int]),
    "dm_destroy": (None, [P]),
    "dm_last_error": (C.c_char_p, [P]),
    "dm_set_mesh": (C.c_int, [P, C.c_int, DP, i64, I32P, i64, I32P, i64]),
    "dm_set_coords": (C.c_int, [P, DP]),
    "dm_set_coords_device": (C.c_int, [P, P]),
    "dm_gen_tri_square": (C.c_int, [P, C.c_int, C.c_uint64, C.c_double, C.c_uint64]),
    "dm_gen_tet_box": (C.c_int, [P, C.c_int, C.c_int, C.c_int, DP, C.c_int, C.c_double,
                                 C.c_uint64]),
    "dm_gen_permute": (C.c_int, [P, C.c_uint64, C.c_uint64]),
    "dm_get_mesh": (C.c_int, [P, DP, I32P, I32P]),
    "dm_mesh_sizes": (C.c_int, [P, C.POINTER(C.c_int), I64P, I64P, I64P]),
    "dm_build_edges": (C.c_int, [P, I64P]),
    "dm_get_edges": (C.c_int, [P, I32P, U64P]),
    "dm_get_e2l": (C.c_int, [P, I32P]),
    "dm_get_incidence": (C.c_int, [P, I32P, I32P]),
    "dm_edge_of": (C.c_int, [P, I32P, I32P, i64, I32P]),
    "dm_navs": (C.c_int, [P, C.c_int, C.c_int]),
    "dm_volumes": (C.c_int, [P, C.c_int]),
    "dm_get_navs": (C.c_int, [P, DP]),
    "dm_get_volumes": (C.c_int, [P, DP]),
    "dm_put_navs": (C.c_int, [P, DP]),
    "dm_put_volumes": (C.c_int, [P, DP]),
    "dm_metrics_host": (C.c_int, [P, DP, C.c_int, C.c_int, C.c_int, DP, DP]),
    "dm_metrics_host_async": (C.c_int, [P, DP, C.c_int, C.c_int, C.c_int, DP, DP]),
    "dm_check_closure": (C.c_int, [P, DP, DP]),
    "dm_check_linear_exactness": (C.c_int, [P, DP, DP, DP]),
    "dm_check_total_volume": (C.c_int, [P, DP, DP, DP]),
    "dm_corrupt_nav": (C.c_int, [P, i64, dbl]),
    "dm_max_face_area": (C.c_int, [P, DP]),
    "dm_max_element_volume": (C.c_int, [P, DP]),
    "dm_total_volume": (C.c_int, [P, DP]),
    "dm_boundary_node_mask": (C.c_int, [P, U8P]),
    "dm_validate": (C.c_int, [P, I8P, I64P, I64P]),
    "dm_validate_list": (C.c_int, [P, C.c_int, I64P, i64, I64P]),
    "dm_derive_boundary": (C.c_int, [P, I64P]),
    "dm_get_derived_boundary": (C.c_int, [P, I32P]),
    "dm_stream": (C.c_int, [P, C.POINTER(P)]),
    "dm_device_views": (C.c_int, [P, P]),
    "dm_sync": (C.c_int, [P]),
    "dm_set_timing": (C.c_int, [P, C.c_int]),
    "dm_get_timings": (C.c_int, [P, FP, C.c_int]),
    "dm_get_step_timings": (C.c_int, [P, FP, C.c_int, C.POINTER(C.c_int)]),
    "dm_kernel_launches": (C.c_int64, [P]),
    "dm_plan_info": (C.c_int, [P, I64P]),
    "dm_plan_side_edges": (C.c_int, [P, I64P]),
    "dm_plan_bytes": (C.c_int, [P, I64P]),
    "dm_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(P)]),
    "dm_mesh_file_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), I64P, I64P, I64P,
                                    C.POINTER(C.c_int), DP, I32P, I32P, C.c_char_p, C.c_int64]),
    "dm_mesh_file_write": (C.c_int, [C.c_char_p, C.c_int, DP, C.c_int64, I32P, C.c_int64, I32P,
                                     C.c_int64]),
    "dm_mesh_checksum": (C.c_uint64, [C.c_int, DP, C.c_int64, I32P, C.c_int64, I32P, C.c_int64]),
    "dm_metrics_file_write": (C.c_int, [C.c_char_p, C.c_int, I32P, C.c_int64, DP, DP, C.c_int64,
                                        C.c_int, C.c_int, C.c_uint64]),
    "dm_host_free": (C.c_int, [P]),
}

MESHGEN = {
    "dmg_tri_square_sizes": (None, [C.c_int, I64P, I64P, I64P]),
    "dmg_tri_square": (C.c_int, [C.c_int, u64, dbl, u64, DP, I32P, I32P]),
    "dmg_tet_box_sizes": (None, [C.c_int, C.c_int, C.c_int, I64P, I64P, I64P]),
    "dmg_tet_box": (C.c_int, [C.c_int, C.c_int, C.c_int, DP, C.c_int, dbl, u64, DP, I32P, I32P]),
    "dmg_bl_z": (C.c_int, [C.c_int, dbl, dbl, DP]),
    "dmg_permute": (C.c_int, [C.c_int, i64, i64, i64, u64, u64, DP, I32P, I32P]),
    "dmg_first_inverted": (C.c_int64, [C.c_int, i64, DP, I32P]),
    "dmg_flip23": (C.c_int64, [i64, DP, i64, I32P, i64, u64, I32P]),
}

_cache: dict[str, C.CDLL] = {}


def _load(name: str, table: dict) -> C.CDLL:
    if name in _cache:
        return _cache[name]
    path = os.path.join(LIBDIR, name)
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the sm_100a library first "
            "(python -c 'import __graft_entry__ as g; g.build()' or `make`). "
            "There is no CPU fallback.")
    lib = C.CDLL(path)
    for sym, (res, args) in table.items():
        fn = getattr(lib, sym)
        fn.restype = res
        fn.argtypes = args
    _cache[name] = lib
    return lib


def capi() -> C.CDLL:
    return _load("libdualmesh.so", CAPI)


def meshgen() -> C.CDLL:
    return _load("libdm_meshgen.so", MESHGEN)


def ptr(a, ctype):
    """ctypes pointer to a contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))
