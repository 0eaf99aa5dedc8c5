"""ctypes declarations for libngsgd.so (include/ngsgd.h).  Argument marshalling only.

The library is built in-tree (``python -m paper_1410_7455_b200.build``).  There is no
fallback: if the shared object is missing or fails to load, importing this module
raises, so nothing can silently run a CPU path.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libngsgd.so")

c_int32, c_int64, c_float, c_double, c_void_p = (ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                                                  ctypes.c_double, ctypes.c_void_p)

STATUS = {0: "NG_OK", 1: "NG_EINVAL", 2: "NG_ESHAPE", 3: "NG_ENONFINITE", 4: "NG_ELABEL", 5: "NG_ECUDA",
          6: "NG_ENCCL", 7: "NG_ENOTPD", 8: "NG_ESTATE", 9: "NG_ENOMEM"}


class NgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class NgsgdConfig(ctypes.Structure):
    _fields_ = [("rank", c_int32), ("alpha", c_float), ("s_samples", c_float), ("update_period", c_int32),
                ("always_update_first", c_int32), ("epsilon", c_float), ("precision", c_int32)]


class NgsgdStateHost(ctypes.Structure):
    _fields_ = [("dim", c_int32), ("rank", c_int32), ("t", c_int32), ("initialized", c_int32), ("rho", c_double),
                ("d", ctypes.POINTER(c_double)), ("w", ctypes.POINTER(c_float)), ("last_updated", c_int32),
                ("last_floored", c_int32), ("last_reorth_checked", c_int32), ("last_reorthogonalized", c_int32),
                ("last_jacobi_sweeps", c_int32)]


class NnetConfig(ctypes.Structure):
    _fields_ = [("input_dim", c_int32), ("num_hidden", c_int32), ("hidden_dim", c_int32), ("pnorm_group", c_int32),
                ("num_classes", c_int32), ("max_minibatch", c_int32), ("precond", c_int32), ("ng_in", NgsgdConfig),
                ("ng_out", NgsgdConfig), ("precision", c_int32), ("seed", ctypes.c_uint64), ("renorm", c_int32)]


class NnetInput(ctypes.Structure):
    _fields_ = [("frames", c_void_p), ("format", c_int32), ("ld", c_int64), ("lo", c_void_p), ("step", c_void_p),
                ("rows", c_void_p), ("labels", c_void_p)]


class NnetUpdateStats(ctypes.Structure):
    _fields_ = [("alpha_t", c_float * 16), ("gamma_in", c_float * 16), ("gamma_out", c_float * 16),
                ("updated_in", c_int32 * 16), ("updated_out", c_int32 * 16)]


class ProfileStats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64 * 16), ("ms", c_double * 16), ("flops", c_double * 16),
                ("bytes", c_double * 16)]


PROF_GROUPS = ["fwd_gemm", "bwd_gemm", "upd_gemm", "ng_proj", "ng_apply", "ng_refresh", "ng_init", "elemwise",
               "average", "ng_eig"]

# name -> (restype, argtypes); every symbol include/ngsgd.h declares
SIGNATURES = {
    "ng_last_error": (ctypes.c_char_p, []),
    "ng_version": (ctypes.c_char_p, []),
    "ngsgd_config_default": (None, [ctypes.POINTER(NgsgdConfig), c_int32]),
    "ngsgd_create": (c_int32, [c_int32, c_int32, ctypes.POINTER(NgsgdConfig), c_void_p, ctypes.POINTER(c_void_p)]),
    "ngsgd_destroy": (c_int32, [c_void_p]),
    "ngsgd_precondition": (c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_void_p, c_void_p, c_int32]),
    "ngsgd_get_state": (c_int32, [c_void_p, ctypes.POINTER(NgsgdStateHost)]),
    "ngsgd_join": (c_int32, [c_void_p]),
    "nnet_join": (c_int32, [c_void_p]),
    "ngsgd_set_state": (c_int32, [c_void_p, ctypes.POINTER(NgsgdStateHost)]),
    "nnet_create": (c_int32, [ctypes.POINTER(NnetConfig), c_void_p, ctypes.POINTER(c_void_p)]),
    "nnet_destroy": (c_int32, [c_void_p]),
    "nnet_forward_backward": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_int32, ctypes.POINTER(c_double)]),
    "nnet_objective_async": (c_int32, [c_void_p, c_void_p]),
    "nnet_update": (c_int32, [c_void_p, c_float, c_float, ctypes.POINTER(NnetUpdateStats)]),
    "nnet_num_layers": (c_int32, [c_void_p, ctypes.POINTER(c_int32)]),
    "nnet_layer_shape": (c_int32, [c_void_p, c_int32, ctypes.POINTER(c_int32), ctypes.POINTER(c_int32)]),
    "nnet_get_params": (c_int32, [c_void_p, c_int32, c_void_p, c_int64]),
    "nnet_set_params": (c_int32, [c_void_p, c_int32, c_void_p, c_int64]),
    "nnet_get_ngsgd": (c_int32, [c_void_p, c_int32, c_int32, ctypes.POINTER(c_void_p)]),
    "nnet_comm_id_bytes": (c_int32, []),
    "nnet_comm_get_unique_id": (c_int32, [c_void_p]),
    "nnet_comm_init": (c_int32, [c_void_p, c_void_p, c_int32, c_int32]),
    "nnet_average": (c_int32, [c_void_p, c_int32]),
    "ng_debug_tree_avg": (c_int32, [c_int32, c_int64, c_void_p, c_void_p, c_void_p]),
    "ng_profile_enable": (c_int32, [ctypes.c_uint32]),
    "ng_profile_read": (c_int32, [ctypes.POINTER(ProfileStats)]),
    "ng_kernel_launches": (ctypes.c_int64, []),
    "ng_debug_gemm_tf32": (c_int32, [c_int32, c_int32, c_int32, c_void_p, c_int64, c_int32, c_void_p, c_int64,
                                     c_int32, c_void_p, c_int64, c_int32, c_int32, c_void_p]),
    "ng_debug_gemm_tc": (c_int32, [c_int32, c_int32, c_int32, c_void_p, c_int64, c_int32, c_void_p, c_int64,
                                   c_int32, c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p]),
    "nnet_forward_backward_ex": (c_int32, [c_void_p, ctypes.POINTER(NnetInput), c_int32, ctypes.POINTER(c_double)]),
    "ng_compress_frames": (c_int32, [c_int32, c_int32, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                                     c_void_p]),
    "nnet_arena_size": (c_int32, [c_void_p, ctypes.POINTER(c_int64)]),
    "nnet_copy_arena": (c_int32, [c_void_p, c_void_p, c_int32]),
    "nnet_set_combination": (c_int32, [c_void_p, ctypes.POINTER(c_void_p), c_int32, ctypes.POINTER(c_float)]),
    "nnet_combination_grad": (c_int32, [c_void_p, ctypes.POINTER(c_void_p), c_int32, ctypes.POINTER(c_double)]),
    "nnet_select_best": (c_int32, [c_void_p, c_double, ctypes.POINTER(c_int32)]),
    "nnet_average_local": (c_int32, [ctypes.POINTER(c_void_p), c_int32]),
    "ngsimple_create": (c_int32, [c_int32, c_int32, c_float, c_void_p, ctypes.POINTER(c_void_p)]),
    "ngsimple_destroy": (c_int32, [c_void_p]),
    "ngsimple_precondition": (c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_void_p, c_void_p]),
    "ngsimple_read_flags": (c_int32, [c_void_p]),
    "ng_debug_eig_tri": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ng_debug_tri_fail": (c_int32, [c_void_p, c_void_p]),
    "ng_debug_refresh_times": (c_int32, [c_void_p, c_void_p]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1410_7455_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(code: int) -> None:
    if code != 0:
        raise NgError(code, lib.ng_last_error().decode())
