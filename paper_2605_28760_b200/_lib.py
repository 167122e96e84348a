"""ctypes binding of libzob200.so (include/zob200.h).

The shared library is the product: there is no CPU or Triton fallback.  If it
is missing (not built) or cannot initialise a B200, calls raise loudly.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, DimensionError, InputError, ScoringAbort

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libzob200.so")

ZO_OK, ZO_ERR_CONFIG, ZO_ERR_DIMENSION, ZO_ERR_INPUT, ZO_ERR_ABORT, ZO_ERR_CUDA, ZO_ERR_INTERNAL = range(7)
PREC_FP16, PREC_BF16, PREC_FP32 = 0, 1, 2
EST_LOZO, EST_FACTORIZED, EST_DENSE = 0, 1, 2
SCOPE_LORA_ONLY, SCOPE_FULL = 0, 1
ARCH_ZOSERVE, ARCH_OPT = 0, 1

_lib = None
_lock = threading.Lock()


class ZoModelDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "vocab", "dim", "n_layers", "n_heads", "prompt_len", "opt_len", "max_batch", "rank",
        "estimator", "precision", "device", "scope", "arch", "max_pos")]


# (name, restype, argtypes) for every symbol include/zob200.h declares
_c = ctypes
_P = _c.c_void_p
SIGNATURES = [
    ("zo_last_error", _c.c_char_p, []),
    ("zo_version", _c.c_int, []),
    ("zo_create", _c.c_int, [_c.POINTER(_P), _c.POINTER(ZoModelDesc)]),
    ("zo_destroy", _c.c_int, [_P]),
    ("zo_set_stream", _c.c_int, [_P, _P]),
    ("zo_synchronize", _c.c_int, [_P]),
    ("zo_num_matrices", _c.c_int, [_P]),
    ("zo_matrix_info", _c.c_int, [_P, _c.c_int, _c.c_char_p, _c.c_int, _c.POINTER(_c.c_int64),
                                  _c.POINTER(_c.c_int64)]),
    ("zo_device_bytes", _c.c_int, [_P, _c.POINTER(_c.c_uint64)]),
    ("zo_init_params", _c.c_int, [_P, _c.c_uint64, _c.c_double]),
    ("zo_upload_matrix", _c.c_int, [_P, _c.c_char_p, _P, _c.c_int64, _c.c_int64]),
    ("zo_download_matrix", _c.c_int, [_P, _c.c_char_p, _P, _c.c_int64, _c.c_int64]),
    ("zo_upload_vector", _c.c_int, [_P, _c.c_char_p, _P, _c.c_int64]),
    ("zo_download_vector", _c.c_int, [_P, _c.c_char_p, _P, _c.c_int64]),
    ("zo_sample_u", _c.c_int, [_P, _c.c_uint64, _c.c_uint64]),
    ("zo_sample_v", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32]),
    ("zo_sample_stream", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_int64, _P]),
    ("zo_slot_count", _c.c_int, [_P, _c.c_int32, _c.POINTER(_c.c_int64)]),
    ("zo_get_slot", _c.c_int, [_P, _c.c_int32, _P, _c.c_int64]),
    ("zo_set_slot", _c.c_int, [_P, _c.c_int32, _P, _c.c_int64]),
    ("zo_set_window", _c.c_int, [_P, _c.c_int64]),
    ("zo_set_update_mode", _c.c_int, [_P, _c.c_int32]),
    ("zo_set_schedule", _c.c_int, [_P, _c.c_int32]),
    ("zo_slot_snapshot", _c.c_int, [_P, _c.c_int32, _c.c_int32]),
    ("zo_slot_snapshot_wait", _c.c_int, [_P, _c.c_int32, _c.c_int32, _P]),
    ("zo_sampler_flags", _c.c_int, [_P, _c.POINTER(_c.c_uint32)]),
    ("zo_prepare_probe", _c.c_int, [_P, _c.c_double, _c.c_int32]),
    ("zo_score", _c.c_int, [_P, _P, _P, _c.c_int32, _c.c_int32, _P]),
    ("zo_score_options", _c.c_int, [_P, _P, _P, _c.c_int32, _c.c_int32, _P]),
    ("zo_coefficient", _c.c_int, [_P, _c.c_int32, _c.c_double, _c.c_double, _c.c_int32, _P]),
    ("zo_set_coefficient", _c.c_int, [_P, _P]),
    ("zo_update_u", _c.c_int, [_P]),
    ("zo_fold", _c.c_int, [_P]),
    ("zo_update_dense", _c.c_int, [_P, _c.c_double]),
    ("zo_update_vectors", _c.c_int, [_P, _c.c_double]),
    ("zo_step", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_double, _c.c_double, _c.c_int32,
                           _P, _P, _c.c_int32, _P]),
    ("zo_step_async", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_double, _c.c_double,
                                 _c.c_int32, _P, _P, _c.c_int32]),
    ("zo_fold_async", _c.c_int, [_P]),
    ("zo_step_graph", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_double, _c.c_double,
                                 _c.c_int32, _P, _P, _c.c_int32]),
    ("zo_step_score_async", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_double, _P, _P,
                                       _c.c_int32]),
    ("zo_step_apply_async", _c.c_int, [_P, _c.c_double, _c.c_double, _c.c_int32, _c.c_int32]),
    ("zo_read_out4", _c.c_int, [_P, _P]),
    ("zo_graph_kernel_count", _c.c_int, [_P, _c.POINTER(_c.c_int32), _c.POINTER(_c.c_int32)]),
    ("zo_qdir_score_async", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_int32, _c.c_int32,
                                       _c.c_double, _c.c_double, _c.c_int32, _P, _P, _c.c_int32]),
    ("zo_out4_io", _c.c_int, [_P, _P, _c.c_int32]),
    ("zo_qdir_apply_async", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_double, _P]),
    ("zo_step_score_graph", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_double, _P, _P,
                                       _c.c_int32]),
    ("zo_step_apply_graph", _c.c_int, [_P, _c.c_double, _c.c_double, _c.c_int32, _c.c_int32]),
    ("zo_qdir_score_graph", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_int32, _c.c_int32,
                                       _c.c_double, _c.c_double, _c.c_int32, _P, _P, _c.c_int32]),
    ("zo_qdir_apply_graph", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_double, _P]),
    ("zo_split_graph_kernels", _c.c_int, [_P, _P]),
    ("zo_baseline_directions", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32]),
    ("zo_baseline_pass", _c.c_int, [_P, _c.c_int32, _c.c_double, _c.c_int32]),
    ("zo_baseline_update", _c.c_int, [_P, _c.c_double, _c.c_int32]),
    ("zo_baseline_step_async", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_double, _c.c_double,
                                          _c.c_int32, _c.c_int32, _P, _P, _c.c_int32]),
    ("zo_last_step_ms", _c.c_int, [_P, _c.POINTER(_c.c_float)]),
    ("zo_fnv1a64", _c.c_uint64, [_P, _c.c_uint64, _c.c_uint64]),
    ("zo_bench_gemm", _c.c_int, [_P, _c.c_int32, _c.c_int32, _c.c_int32, _c.POINTER(_c.c_float),
                                 _c.POINTER(_c.c_double)]),
    ("zo_nll_io", _c.c_int, [_P, _P, _c.c_int32, _c.c_int32]),
    ("zo_trace_gemm", _c.c_int, [_P, _c.c_int32, _c.c_int32, _P, _c.c_int32, _c.POINTER(_c.c_int32)]),
    ("zo_profile_step", _c.c_int, [_P, _c.c_uint64, _c.c_uint64, _c.c_int32, _c.c_double, _c.c_double, _P, _P,
                                   _c.c_int32, _c.POINTER(_c.c_float)]),
    ("zo_test_gemm", _c.c_int, [_c.c_int32] * 6 + [_P, _P, _P]),
    ("zo_test_gemm_tf32x3", _c.c_int, [_c.c_int32] * 3 + [_P, _P, _P]),
    ("zo_digest_chain", _c.c_uint64, [_c.POINTER(_c.c_char_p), _P, _c.POINTER(_c.c_int64),
                                      _c.POINTER(_c.c_int64), _c.c_int32, _c.c_uint64]),
]


def lib():
    """Load libzob200.so (fails loudly when the CUDA extension is missing)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"libzob200.so not built ({LIB_PATH}); run `python -m paper_2605_28760_b200.build`. "
                        "There is no CPU fallback.")
                L = ctypes.CDLL(LIB_PATH)
                for name, res, args in SIGNATURES:
                    f = getattr(L, name)
                    f.restype = res
                    f.argtypes = args
                _lib = L
    return _lib


_EXC = {
    ZO_ERR_CONFIG: ConfigError,
    ZO_ERR_DIMENSION: DimensionError,
    ZO_ERR_INPUT: InputError,
    ZO_ERR_ABORT: ScoringAbort,
}


def check(code: int) -> None:
    if code != ZO_OK:
        msg = lib().zo_last_error().decode("utf-8", "replace")
        raise _EXC.get(code, RuntimeError)(msg)
