"""ctypes binding of libhcinfer.so (include/hcinfer.h).  Argument marshalling only: every
step of the compensated linear runs in the library's sm_100a kernels.  There is no CPU
fallback — if the shared library is missing the import of the binding fails loudly."""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HC_LIB_PATH") or os.path.join(_PKG, "libhcinfer.so")   # override: dev variant builds

HC_OK, HC_ERR_CONFIG, HC_ERR_STATE, HC_ERR_NUMERIC, HC_ERR_RUNTIME = 0, 2, 3, 4, 5
QKV, O, UPGATE, DOWN = 0, 1, 2, 3
OUT_F32, OUT_BF16 = 0, 1
GLUE_NONE, GLUE_SILU_MUL = 0, 1
FACTORS_BF16, FACTORS_FP8 = 0, 1


class HCError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[hc_status {code}] {msg}")
        self.code = code


class hc_sens(C.Structure):
    _fields_ = [("layer", C.c_int32), ("window_kind", C.c_int32), ("slot", C.c_int32), ("expert", C.c_int32),
                ("n_sigma", C.c_int32), ("sigma", C.POINTER(C.c_double)), ("phi", C.c_double),
                ("n_salient", C.c_int32), ("n_total", C.c_int32), ("D_matrix", C.c_double), ("gate", C.c_double)]


class hc_budget(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("D_layer", C.POINTER(C.c_double)), ("top_k_layers", C.c_int32),
                ("tau", C.c_double), ("k0", C.c_int32), ("r_std", C.c_double * 4),
                ("two_stage_mode", C.c_int32), ("moe_k", C.c_int32)]


class hc_matrix_desc(C.Structure):
    _fields_ = [("layer", C.c_int32), ("window_kind", C.c_int32), ("slot", C.c_int32), ("expert", C.c_int32),
                ("N", C.c_int32), ("K", C.c_int32), ("bits", C.c_int32), ("group", C.c_int32),
                ("codes", C.c_void_p), ("scales", C.c_void_p), ("zeros", C.c_void_p),
                ("U", C.c_void_p), ("V", C.c_void_p),
                ("r_stored", C.c_int32), ("r_alloc", C.c_int32), ("row_begin", C.c_int32), ("row_end", C.c_int32),
                ("glue", C.c_int32), ("factor_dtype", C.c_int32), ("u_scale", C.c_void_p), ("v_scale", C.c_void_p)]


# (name, restype, argtypes) — every symbol include/hcinfer.h declares
SIGNATURES = [
    ("hc_version", C.c_char_p, []),
    ("hc_set_option", C.c_int, [C.c_char_p, C.c_int32]),
    ("hc_peer_region", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    ("hc_peer_ipc_handle", C.c_int, [C.c_void_p, C.c_void_p]),
    ("hc_peer_connect", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    ("hc_peer_set", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    ("hc_calib_svd", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                               C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p]),
    ("hc_calib_salience", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_void_p, C.c_void_p,
                                    C.c_void_p]),
    ("hc_calib_r_std", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_void_p]),
    ("hc_get_option", C.c_int, [C.c_char_p, C.c_void_p]),
    ("hc_last_error", C.c_char_p, []),
    ("hc_allocate_ranks", C.c_int, [C.POINTER(hc_sens), C.c_int32, C.POINTER(hc_budget), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    ("hc_create", C.c_int, [C.POINTER(C.c_void_p), C.c_int32]),
    ("hc_destroy", C.c_int, [C.c_void_p]),
    ("hc_load_layer", C.c_int, [C.c_void_p, C.POINTER(hc_matrix_desc), C.c_int32, C.c_void_p]),
    ("hc_set_rank", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    ("hc_window_rows", C.c_int64, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32]),
    ("hc_compensated_linear", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                        C.c_void_p, C.c_int32, C.c_void_p]),
    ("hc_stack_forward", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    ("hc_moe_forward", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                                 C.c_void_p, C.c_void_p]),
    ("hc_moe_set_dynamic_ranks", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32]),
    ("hc_moe_last_ranks", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]),
    ("hc_nccl_unique_id", C.c_int, [C.c_void_p]),
    ("hc_set_comm", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]),
    ("hc_repacked_bytes", C.c_size_t, [C.c_int32, C.c_int32, C.c_int32]),
    ("hc_repack_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    ("hc_unpack_repacked_host", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_void_p]),
    ("hc_unshard_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python __graft_entry__.py build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int):
    if status != HC_OK:
        raise HCError(status, lib().hc_last_error().decode(errors="replace"))
