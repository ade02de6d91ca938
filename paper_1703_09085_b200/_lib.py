"""ctypes declarations of libhm (include/hm.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libhm.so")

HM_OK, HM_EINVAL, HM_ENOMEM, HM_ECUDA, HM_EPIVOT, HM_ESTRUCT, HM_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
STATUS = {0: "HM_OK", -1: "HM_EINVAL", -2: "HM_ENOMEM", -3: "HM_ECUDA", -4: "HM_EPIVOT",
          -5: "HM_ESTRUCT", -6: "HM_EUNSUPPORTED"}

P_i32 = C.POINTER(C.c_int32)
P_i64 = C.POINTER(C.c_int64)
P_f64 = C.POINTER(C.c_double)


class HostDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("nclusters", C.c_int32),
        ("cl_start", P_i32), ("cl_size", P_i32), ("cl_son0", P_i32), ("cl_nsons", P_i32),
        ("cl_level", P_i32), ("cl_bbox", P_f64),
        ("nblocks", C.c_int32),
        ("bl_row", P_i32), ("bl_col", P_i32), ("bl_kind", P_i32), ("bl_son0", P_i32),
        ("bl_nsons", P_i32), ("bl_rank", P_i32), ("bl_off", P_i64),
        ("factors", P_f64), ("nfactors", C.c_int64),
        ("dense", P_f64), ("ndense", C.c_int64),
        ("perm", P_i64),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("nclusters", C.c_int32), ("nblocks", C.c_int32), ("nadm", C.c_int32),
        ("ndense", C.c_int32), ("depth", C.c_int32),
        ("max_rank", C.c_int32),
        ("mean_rank", C.c_double),
        ("factor_doubles", C.c_int64), ("dense_doubles", C.c_int64),
        ("addproduct_calls", C.c_int64), ("evaluated_terms", C.c_int64),
        ("truncations", C.c_int64), ("trunc_cols", C.c_int64), ("merges", C.c_int64),
        ("dense_adds", C.c_int64), ("levels", C.c_int64), ("kernel_launches", C.c_int64),
        ("flops_trunc", C.c_double), ("flops_eval", C.c_double), ("flops_dense", C.c_double),
        ("bytes_trunc", C.c_double), ("bytes_eval", C.c_double), ("bytes_dense", C.c_double),
        ("min_pivot", C.c_double),
    ]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class Allocator(C.Structure):
    """hm_allocator (include/hm.h): stream-ordered device memory hook."""
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", C.c_void_p)]


HM_NPROF = 32


class Prof(C.Structure):
    _fields_ = [
        ("name", (C.c_char * 24) * HM_NPROF),
        ("ms", C.c_double * HM_NPROF),
        ("launches", C.c_int64 * HM_NPROF),
        ("flops", C.c_double * HM_NPROF),
        ("bytes", C.c_double * HM_NPROF),
        ("count", C.c_int32),
    ]


EXPORTS = [
    "hm_version", "hm_ctx_create", "hm_ctx_destroy", "hm_last_error", "hm_sync", "hm_trim", "hm_build", "hm_build_nrm",
    "hm_import", "hm_export", "hm_export_sizes", "hm_export_into", "hm_clone", "hm_free", "hm_addmul", "hm_addmul_std",
    "hm_lr", "hm_chol", "hm_inv",
    "hm_matvec_thin", "hm_solve_thin", "hm_precond_error", "hm_stats", "hm_profile_enable", "hm_profile_reset", "hm_profile_get",
    "hm_test_trunc_batched", "hm_test_eval_batched",
    "hm_flush_capture", "hm_flush_capture_info", "hm_flush_replay", "hm_flush_capture_free",
]


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(
            f"libhm not built: {path} is missing.  Run `make -C paper_1703_09085_b200` or "
            "__graft_entry__.build().  There is no CPU fallback.")
    lib = C.CDLL(path)
    vp = C.c_void_p
    sig = {
        "hm_version": (C.c_char_p, []),
        "hm_ctx_create": (C.c_int, [C.c_int, vp, vp, C.POINTER(vp)]),
        "hm_ctx_destroy": (C.c_int, [vp]),
        "hm_last_error": (C.c_char_p, [vp]),
        "hm_sync": (C.c_int, [vp]),
        "hm_trim": (C.c_int, [vp]),
        "hm_build": (C.c_int, [vp, P_f64, P_f64, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double,
                               C.POINTER(vp), P_i64]),
        "hm_build_nrm": (C.c_int, [vp, P_f64, P_f64, P_f64, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double,
                                   C.POINTER(vp), P_i64]),
        "hm_import": (C.c_int, [vp, C.POINTER(HostDesc), C.POINTER(vp)]),
        "hm_export": (C.c_int, [vp, vp, C.POINTER(HostDesc)]),
        "hm_export_sizes": (C.c_int, [vp, vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "hm_export_into": (C.c_int, [vp, vp, C.POINTER(HostDesc), vp, vp]),
        "hm_clone": (C.c_int, [vp, vp, C.POINTER(vp)]),
        "hm_free": (C.c_int, [vp, vp]),
        "hm_addmul": (C.c_int, [vp, C.c_double, vp, vp, vp, C.c_double]),
        "hm_addmul_std": (C.c_int, [vp, C.c_double, vp, vp, vp, C.c_double]),
        "hm_lr": (C.c_int, [vp, vp, C.c_double]),
        "hm_inv": (C.c_int, [vp, vp, C.c_double]),
        "hm_chol": (C.c_int, [vp, vp, C.c_double, C.c_double]),
        "hm_matvec_thin": (C.c_int, [vp, vp, C.c_int, C.c_double, vp, C.c_int64, C.c_double, vp,
                                     C.c_int64, C.c_int]),
        "hm_solve_thin": (C.c_int, [vp, vp, C.c_int, vp, C.c_int64, C.c_int]),
        "hm_precond_error": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_uint64, P_f64]),
        "hm_stats": (C.c_int, [vp, vp, C.POINTER(Stats)]),
        "hm_profile_enable": (C.c_int, [vp, C.c_int]),
        "hm_profile_reset": (C.c_int, [vp]),
        "hm_profile_get": (C.c_int, [vp, C.POINTER(Prof)]),
        "hm_test_trunc_batched": (C.c_int, [vp, C.c_int, P_i32, P_i32, P_i32, vp, P_i64, vp, P_i64,
                                            vp, P_i64, vp, P_i64, C.c_double, P_i32, P_f64]),
        "hm_test_eval_batched": (C.c_int, [vp, vp, C.c_int, P_i32, P_i32, P_f64, vp, P_i64, P_i32, vp, P_i64,
                                           P_i32, P_i32, C.c_double]),
        "hm_flush_capture": (C.c_int, [vp, C.c_uint64]),
        "hm_flush_capture_info": (C.c_int, [vp, C.c_int, P_i64, P_i32, P_i32, P_i32, P_i32, C.POINTER(C.c_int)]),
        "hm_flush_replay": (C.c_int, [vp, C.c_int, C.c_double, C.c_int, P_f64, P_i64]),
        "hm_flush_capture_free": (C.c_int, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib
