"""ctypes binding of libslcs.so (include/slcs.h).

This is the binding a Python host uses; INTEGRATION.md shows the equivalent
C++ shim for the reference executor.  There is deliberately no fallback: if
the CUDA library is missing or no GPU is present, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# SLCS_LIB_PATH: an alternative build of the same sources (A/B measurements only)
LIB_PATH = os.environ.get("SLCS_LIB_PATH") or os.path.join(HERE, "libslcs.so")
HEADER = os.path.join(HERE, "..", "include", "slcs.h")

_lib = None

vp = C.c_void_p
pvp = C.POINTER(C.c_void_p)
i32 = C.c_int
i64 = C.c_int64
dbl = C.c_double
sz = C.c_size_t
cstr = C.c_char_p

_SIGS = {
    "slcs_abi_version": (i32, []),
    "slcs_last_error": (cstr, []),
    "slcs_ctx_create": (i32, [i32, vp, pvp]),
    "slcs_ctx_destroy": (i32, [vp]),
    "slcs_ctx_synchronize": (i32, [vp]),
    "slcs_ctx_stream": (vp, [vp]),
    "slcs_ctx_launch_count": (i64, [vp]),
    "slcs_image_upload": (i32, [vp, i32, i32, i32, i32, vp, pvp]),
    "slcs_image_from_device": (i32, [vp, i32, i32, i32, i32, vp, pvp]),
    "slcs_image_download": (i32, [vp, vp, vp, sz]),
    "slcs_image_to_device": (i32, [vp, vp, vp, sz]),
    "slcs_random_mask": (i32, [vp, i32, i32, C.c_longlong, C.c_uint64, dbl, pvp]),
    "slcs_random_u16": (i32, [vp, i32, i32, C.c_longlong, C.c_uint64, pvp]),
    "slcs_image_retain": (i32, [vp]),
    "slcs_image_release": (i32, [vp]),
    "slcs_image_info": (i32, [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32),
                              C.POINTER(i32)]),
    "slcs_image_storage": (i32, [vp, pvp, C.POINTER(sz), C.POINTER(sz)]),
    "slcs_threshold": (i32, [vp, i32, vp, dbl, pvp]),
    "slcs_not": (i32, [vp, vp, pvp]),
    "slcs_and": (i32, [vp, vp, vp, pvp]),
    "slcs_or": (i32, [vp, vp, vp, pvp]),
    "slcs_near": (i32, [vp, vp, pvp]),
    "slcs_near_k": (i32, [vp, vp, i32, pvp]),
    "slcs_interior": (i32, [vp, vp, pvp]),
    "slcs_interior_k": (i32, [vp, vp, i32, pvp]),
    "slcs_volume": (i32, [vp, vp, C.POINTER(i64)]),
    "slcs_volume_async": (i32, [vp, vp, vp]),
    "slcs_png_load": (i32, [vp, cstr, pvp]),
    "slcs_near_k_halo": (i32, [vp, vp, i32, i32, vp, i32, vp, i32, pvp]),
    "slcs_band_record_bytes": (sz, [i32, i32]),
    "slcs_ccl_border_record": (i32, [vp, vp, vp]),
    "slcs_band_ccl_relabel": (i32, [vp, vp, i32, i32, vp, vp, vp]),
    "slcs_ccl_band_begin": (i32, [vp, vp, vp, vp]),
    "slcs_ccl_band_begin_reach": (i32, [vp, vp, vp]),
    "slcs_reach_prepare_labels": (i32, [vp, vp, vp, vp]),
    "slcs_ccl_band_finish": (i32, [vp, i32, i32, vp, vp, vp]),
    "slcs_ccl_job_destroy": (i32, [vp]),
    "slcs_reach_border_record": (i32, [vp, vp]),
    "slcs_band_reach_merge": (i32, [vp, i32, i32, vp]),
    "slcs_png_decode": (i32, [vp, vp, sz, pvp]),
    "slcs_png_save": (i32, [vp, vp, cstr]),
    "slcs_label_color": (None, [C.c_uint32, vp]),
    "slcs_ccl": (i32, [vp, vp, pvp]),
    "slcs_reach": (i32, [vp, vp, vp, pvp]),
    "slcs_maxvol": (i32, [vp, vp, pvp]),
    "slcs_reach_prepare": (i32, [vp, vp, vp, pvp]),
    "slcs_reach_row": (i32, [vp, i32, vp, vp]),
    "slcs_reach_set_flags": (i32, [vp, i32, vp]),
    "slcs_reach_finish": (i32, [vp, i32, pvp]),
    "slcs_reach_state_destroy": (i32, [vp]),
    "slcs_image_rows": (i32, [vp, vp, i32, i32, pvp]),
    "slcs_image_vstack": (i32, [vp, i32, C.POINTER(vp), pvp]),
    "slcs_h_threshold": (i32, [vp, i32, vp, i32, i32, dbl, vp]),
    "slcs_h_not": (i32, [vp, vp, i32, i32, vp]),
    "slcs_h_and": (i32, [vp, vp, vp, i32, i32, vp]),
    "slcs_h_or": (i32, [vp, vp, vp, i32, i32, vp]),
    "slcs_h_dilate": (i32, [vp, vp, i32, i32, vp]),
    "slcs_h_count_true": (i32, [vp, vp, i32, i32, C.POINTER(i64)]),
    "slcs_h_ccl_label": (i32, [vp, vp, i32, i32, vp]),
    "slcs_h_reach": (i32, [vp, vp, vp, i32, i32, vp]),
    "slcs_program_create": (i32, [vp, i32, C.POINTER(cstr), C.POINTER(dbl), C.POINTER(cstr),
                                  C.POINTER(i32), C.POINTER(i32), pvp]),
    "slcs_program_destroy": (i32, [vp]),
    "slcs_program_bind": (i32, [vp, cstr, vp]),
    "slcs_program_run": (i32, [vp, i32]),
    "slcs_program_set_input_host": (i32, [vp, cstr, i32, i32, i32, i32, vp]),
    "slcs_program_download": (i32, [vp, i32, vp, sz]),
    "slcs_program_result": (i32, [vp, i32, C.POINTER(i32), pvp, C.POINTER(dbl)]),
    "slcs_program_task_state": (i32, [vp, i32, C.POINTER(i32), C.POINTER(cstr)]),
    "slcs_program_task_time": (i32, [vp, i32, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "slcs_program_launches": (i32, [vp, C.POINTER(i32)]),
    "slcs_program_plan": (cstr, [vp]),
}


def header_symbols() -> list[str]:
    """Every function declared in include/slcs.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(slcs_[a-z0-9_]+)\s*\(", text)))


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the SLCS path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L
