"""ctypes loader for liblatecache_b200.so (the in-tree C-ABI library).

There is no fallback: if the shared library is missing, importing the package
raises ImportError; engine calls on a machine without an sm_100 GPU raise
CudaError from the library itself.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblatecache_b200.so")

LC_OK = 0
LC_ERR_INVALID_ARGUMENT = 1
LC_ERR_RUNTIME = 2
LC_ERR_INFEASIBLE_PLAN = 3
LC_ERR_CUDA = 4

LC_PREC_BF16X3 = 0
LC_PREC_BF16 = 1
LC_SERVE_SHADOW = 1
LC_SERVE_NO_GRAPH = 2


class InfeasiblePlanError(ValueError):
    """simulate_model's invalid_argument for a plan failing check_constraints (serving.cpp:23-29)."""


class CudaError(RuntimeError):
    """Device failure (no sm_100 GPU, CUDA error)."""


class CnnOpDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("in_", C.c_int), ("out", C.c_int), ("res", C.c_int),
        ("C", C.c_int), ("H", C.c_int), ("W", C.c_int), ("Cout", C.c_int), ("k", C.c_int),
        ("stride", C.c_int), ("pad", C.c_int), ("relu", C.c_int), ("tap", C.c_int),
        ("w", C.POINTER(C.c_double)), ("w_len", C.c_longlong),
        ("scale", C.POINTER(C.c_double)), ("shift", C.POINTER(C.c_double)),
    ]


class AdaptConfig(C.Structure):  # lc_adapt_config
    _fields_ = [
        ("sample_rate", C.c_double), ("window_min", C.c_double), ("retrain_interval_min", C.c_double),
        ("recency_decay", C.c_double), ("mixin_fraction", C.c_double), ("epochs", C.c_int),
        ("learning_rate", C.c_double), ("retrain_pause_ms", C.c_double), ("tau", C.c_double),
        ("beta", C.c_double), ("w_fp", C.c_double), ("w_fn", C.c_double),
    ]


class RetrainEventC(C.Structure):  # lc_retrain_event
    _fields_ = [
        ("interval", C.c_int), ("time_min", C.c_double), ("window_size", C.c_longlong),
        ("mixin_size", C.c_longlong), ("applied", C.c_int), ("note", C.c_char * 160),
    ]


# lc_swap_hook: void (*)(void* ctx, double swap_time_min)
SWAP_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_double)


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2101_07344_b200` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    I, LL, D, U64 = C.c_int, C.c_longlong, C.c_double, C.c_uint64
    pI, pLL, pD, pF = C.POINTER(C.c_int), C.POINTER(C.c_longlong), C.POINTER(C.c_double), C.POINTER(C.c_float)
    sig = {
        "lc_last_error": (C.c_char_p, []),
        "lc_version": (C.c_char_p, []),
        "lc_free": (None, [P]),
        "lc_model_make_mlp": (I, [I, I, pI, I, I, U64, C.POINTER(P)]),
        "lc_model_load": (I, [C.c_char_p, C.c_size_t, C.POINTER(P)]),
        "lc_model_save": (I, [P, C.POINTER(P), C.POINTER(C.c_size_t)]),
        "lc_model_make_cnn": (I, [C.c_char_p, I, U64, C.POINTER(P)]),
        "lc_model_info": (I, [P, pI, pI, pLL]),
        "lc_model_tap": (I, [P, I, pI, pI, pI]),
        "lc_model_macs": (LL, [P, I]),
        "lc_model_free": (None, [P]),
        "lc_model_cnn_ops": (I, [P, pI, pI]),
        "lc_model_cnn_op": (I, [P, I, C.POINTER(CnnOpDesc)]),
        "lc_variant_build": (I, [I, I, C.c_char_p, LL, I, U64, C.POINTER(P)]),
        "lc_variant_load": (I, [C.c_char_p, C.c_size_t, C.POINTER(P)]),
        "lc_variant_save": (I, [P, C.POINTER(P), C.POINTER(C.c_size_t)]),
        "lc_variant_set_delta": (I, [P, D]),
        "lc_variant_info": (I, [P, pI, pI, pD, C.c_char_p, I]),
        "lc_variant_macs": (LL, [P]),
        "lc_variant_layer": (I, [P, I, I, pI, pI, pI, pI, pI, pI, C.POINTER(pD), pLL, C.POINTER(pD), pLL]),
        "lc_variant_set_selector_out": (I, [P, D, D]),
        "lc_variant_free": (None, [P]),
        "lc_plan_check": (I, [C.c_char_p, C.c_char_p, pD, I, D, D, pI, pI, pI, I, pI, C.POINTER(P)]),
        "lc_gen_workload": (I, [I, D, D, D, D, U64, pI, LL, I, pLL, pLL, pI, pD, LL]),
        "lc_nearest_rank": (D, [pD, LL, D]),
        "lc_engine_create": (I, [I, P, C.POINTER(P), I, I, I, C.POINTER(P)]),
        "lc_engine_destroy": (I, [P]),
        "lc_engine_set_delta": (I, [P, I, D]),
        "lc_engine_set_selector_out": (I, [P, I, D, D]),
        "lc_engine_input": (I, [P, C.POINTER(P)]),
        "lc_serve_batch": (I, [P, pF, I, C.c_uint, pI, pI, pI, pF, pF, pD]),
        "lc_serve_device": (I, [P, I, C.c_uint]),
        "lc_engine_sync": (I, [P]),
        "lc_engine_results": (I, [P, I, pI, pI, pI, pF, pF, pD]),
        "lc_engine_read_tap": (I, [P, pF, I, I, pF]),
        "lc_engine_counts": (I, [P, pI]),
        "lc_lookup_batch": (I, [P, I, pF, I, pI, pI, pF, pF, pF]),
        "lc_measure_metrics": (I, [P, pF, I, pD, I, C.POINTER(C.c_longlong)]),
        "lc_serve_submit": (I, [P, pF, I, C.c_uint, pI]),
        "lc_engine_layer_times": (I, [P, pF, I, C.c_uint, pD, pD]),
        "lc_model_save_binary": (I, [P, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
        "lc_model_load_binary": (I, [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p)]),
        "lc_variant_save_binary": (I, [P, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
        "lc_variant_load_binary": (I, [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p)]),
        "lc_serve_collect": (I, [P, I, I, pI, pI, pI, pF, pF, pD]),
        "lc_tune_delta": (I, [P, pF, I, C.c_double, pD, I, pD, I]),
        "lc_train_predictor": (I, [I, P, pD, C.c_longlong, pD, I, I, pD, D, D, I, I, C.c_uint64, D, D]),
        "lc_train_selector": (I, [I, P, pD, C.c_longlong, pD, I, I, pD, D, D, I, I, C.c_uint64, D, D]),
        "lc_engine_update_variant": (I, [P, P]),
        "lc_run_adaptation": (I, [P, pF, I, pD, pI, I, C.POINTER(AdaptConfig), C.POINTER(pD), pD, I, C.c_uint64, I,
                                  pI, pI, pI, pD, C.POINTER(RetrainEventC), I, pI]),
        "lc_engine_variant": (I, [P, I, C.POINTER(P)]),
        "lc_engine_set_swap_hook": (I, [P, SWAP_HOOK, P]),
        "lc_engine_time": (I, [P, I, C.c_uint, I, pD]),
        "lc_engine_kernel_count": (I, [P, C.c_uint, I]),
        "lc_engine_profile": (I, [P, I, C.c_uint, I, pI, pI, pD, pD, pD]),
        "lc_serve_timed": (I, [P, I, C.c_uint, pD]),
        "lc_engine_stage_input": (I, [P, P, I, I]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status == LC_OK:
        return
    msg = lib.lc_last_error().decode("utf-8", "replace")
    if status == LC_ERR_INFEASIBLE_PLAN:
        raise InfeasiblePlanError(msg)
    if status == LC_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == LC_ERR_CUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


def take_bytes(ptr: C.c_void_p, n: C.c_size_t) -> bytes:
    try:
        return C.string_at(ptr, n.value)
    finally:
        lib.lc_free(ptr)


def take_string(ptr: C.c_void_p, n: C.c_size_t) -> str:
    try:
        return C.string_at(ptr, n.value).decode()
    finally:
        lib.lc_free(ptr)


EXPORTED_SYMBOLS = [
    "lc_last_error", "lc_version", "lc_free", "lc_model_make_mlp", "lc_model_load", "lc_model_save",
    "lc_model_make_cnn", "lc_model_info", "lc_model_tap", "lc_model_macs", "lc_model_free", "lc_model_cnn_ops",
    "lc_model_cnn_op", "lc_variant_build", "lc_variant_load", "lc_variant_save", "lc_variant_set_delta",
    "lc_variant_info", "lc_variant_macs", "lc_variant_layer", "lc_variant_set_selector_out", "lc_variant_free",
    "lc_plan_check", "lc_gen_workload", "lc_nearest_rank", "lc_engine_create", "lc_engine_destroy",
    "lc_engine_set_delta", "lc_engine_set_selector_out", "lc_engine_input", "lc_serve_batch", "lc_serve_device",
    "lc_engine_sync", "lc_engine_results", "lc_engine_counts", "lc_lookup_batch", "lc_engine_time",
    "lc_engine_kernel_count", "lc_engine_profile", "lc_serve_timed", "lc_engine_stage_input",
    "lc_measure_metrics", "lc_tune_delta", "lc_train_predictor", "lc_train_selector", "lc_engine_update_variant",
    "lc_run_adaptation", "lc_engine_variant", "lc_serve_submit", "lc_serve_collect", "lc_engine_layer_times",
    "lc_model_save_binary", "lc_model_load_binary", "lc_variant_save_binary", "lc_variant_load_binary",
    "lc_engine_read_tap", "lc_engine_set_swap_hook",
]
