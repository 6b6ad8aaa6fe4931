"""ctypes binding of the C ABI in include/dfgtb.h (libdfgtb.so, built in-tree).

The product path: every call goes to the sm_100a library.  There is no CPU
fallback -- if libdfgtb.so is missing or fails to load, import raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DFGTB_LIB selects an alternative in-tree build (A/B experiments, tools/)
LIB_PATH = os.environ.get("DFGTB_LIB") or os.path.join(_HERE, "libdfgtb.so")

OK, EINVAL, ECUDA, ENOMEM = 0, 1, 2, 3

_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_I = C.POINTER(C.c_int)
_I64 = C.POINTER(C.c_int64)


class Config(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("leaf_threshold", C.c_int), ("p_max", C.c_int),
                ("cost_model", C.c_int), ("mode", C.c_int), ("local_pushdown", C.c_int)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "kernel_evaluations", "pairs_visited", "base_cases", "prunes_finite_diff",
        "prunes_farfield", "prunes_direct_local", "prunes_far_to_local", "levels",
        "pairs_covered")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class Timings(C.Structure):
    _fields_ = [(n, C.c_float) for n in (
        "tree_ms", "traverse_ms", "moments_ms", "local_ms", "base_ms", "farfield_ms", "final_ms",
        "total_ms", "base_f32_ms", "base_fp64_ms", "moments_build_ms")]

    def as_dict(self):
        return {n: float(getattr(self, n)) for n, _ in self._fields_}


class CvRow(C.Structure):
    _fields_ = [("scale", C.c_double), ("h", C.c_double), ("conv_h", C.c_double),
                ("lk_score", C.c_double), ("lk_clamped", C.c_int), ("ls_score", C.c_double),
                ("seconds", C.c_double), ("base_ms", C.c_double), ("base_pairs", C.c_uint64),
                ("kernel_evaluations", C.c_uint64), ("pairs_visited", C.c_uint64)]


# every symbol include/dfgtb.h declares (tests check the .so exports all of them)
EXPORTS = (
    "dfgtb_default_config", "dfgtb_create", "dfgtb_create_device", "dfgtb_create_f32",
    "dfgtb_compute_batch_f32", "dfgtb_destroy",
    "dfgtb_compute", "dfgtb_compute_device", "dfgtb_compute_batch", "dfgtb_last_stats",
    "dfgtb_last_timings",
    "dfgtb_p_max", "dfgtb_cv", "dfgtb_sweep", "dfgtb_lkcv_from_sums", "dfgtb_lscv_from_sums",
    "dfgtb_tree_nodes", "dfgtb_tree_height", "dfgtb_export_tree", "dfgtb_naive",
    "dfgtb_series_op", "dfgtb_dfma_peak", "dfgtb_mufu_exp_error", "dfgtb_f32_exp_error", "dfgtb_f32_terms", "dfgtb_last_base_split", "dfgtb_ex2_peak", "dfgtb_base_exp_mode", "dfgtb_device_count", "dfgtb_release_cached_memory",
    "dfgtb_stream", "dfgtb_choose_methods", "dfgtb_box_bounds", "dfgtb_sweep_best",
    "dfgtb_launch_count", "dfgtb_last_error", "dfgtb_guard_check", "dfgtb_guard_selftest",
)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    V = C.c_void_p
    sz = C.c_size_t
    sig = {
        "dfgtb_default_config": (None, [C.POINTER(Config)]),
        "dfgtb_create": (C.c_int, [_D, sz, sz, C.POINTER(Config), C.POINTER(V)]),
        "dfgtb_create_device": (C.c_int, [V, sz, sz, C.POINTER(Config), C.POINTER(V)]),
        "dfgtb_create_f32": (C.c_int, [_F, sz, sz, C.POINTER(Config), C.POINTER(V)]),
        "dfgtb_compute_batch_f32": (C.c_int, [V, _F, sz, _D, sz, _D, C.POINTER(Stats)]),
        "dfgtb_destroy": (None, [V]),
        "dfgtb_compute": (C.c_int, [V, _D, sz, C.c_double, _D, C.POINTER(Stats)]),
        "dfgtb_compute_device": (C.c_int, [V, V, sz, C.c_double, V, C.POINTER(Stats)]),
        "dfgtb_compute_batch": (C.c_int, [V, _D, sz, _D, sz, _D, C.POINTER(Stats)]),
        "dfgtb_last_stats": (C.c_int, [V, C.POINTER(Stats)]),
        "dfgtb_last_timings": (C.c_int, [V, C.POINTER(Timings)]),
        "dfgtb_p_max": (C.c_int, [V]),
        "dfgtb_cv": (C.c_int, [V, C.c_double, C.c_double, C.POINTER(CvRow)]),
        "dfgtb_sweep": (C.c_int, [V, _D, sz, C.c_double, C.c_int, C.POINTER(CvRow)]),
        "dfgtb_lkcv_from_sums": (C.c_int, [sz, sz, C.c_double, _D, _D, _I]),
        "dfgtb_lscv_from_sums": (C.c_int, [sz, sz, C.c_double, _D, C.c_double, _D, _D]),
        "dfgtb_tree_nodes": (C.c_int, [V]),
        "dfgtb_tree_height": (C.c_int, [V]),
        "dfgtb_export_tree": (C.c_int, [V, _I, _D, _D, _D, _D, _I, _I, _I, _D, _I64, _I]),
        "dfgtb_naive": (C.c_int, [_D, sz, _D, sz, sz, C.c_double, _D]),
        "dfgtb_series_op": (C.c_int, [C.c_int, sz, C.c_int, _D, sz, _D, _D, C.c_double, C.c_int,
                                      _D]),
        "dfgtb_dfma_peak": (C.c_double, []),
        "dfgtb_mufu_exp_error": (C.c_double, []),
        "dfgtb_f32_exp_error": (C.c_double, []),
        "dfgtb_last_base_split": (C.c_int, [V, _I, _I, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "dfgtb_f32_terms": (C.c_int, [sz, _D, _D, _D, sz, _D]),
        "dfgtb_ex2_peak": (C.c_double, []),
        "dfgtb_base_exp_mode": (C.c_int, [V]),
        "dfgtb_device_count": (C.c_int, []),
        "dfgtb_release_cached_memory": (None, []),
        "dfgtb_stream": (C.c_size_t, [V]),
        "dfgtb_choose_methods": (C.c_int, [sz, _D, _I]),
        "dfgtb_sweep_best": (C.c_int, [C.POINTER(CvRow), sz, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
        "dfgtb_box_bounds": (C.c_int, [sz, sz, _D, _D]),
        "dfgtb_launch_count": (C.c_uint64, [V]),
        "dfgtb_last_error": (C.c_char_p, []),
        "dfgtb_guard_check": (C.c_int, []),
        "dfgtb_guard_selftest": (C.c_int, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


class _Lib:
    """The loaded libdfgtb.so, opened on first use.

    Importing the package checks that the library exists (no CPU fallback) but does
    not map it: processes that only need the package's host helpers (e.g. the
    datagen of bench.py's reference arm) never load the CUDA library.
    """

    _lib = None

    def __getattr__(self, name):
        if _Lib._lib is None:
            _Lib._lib = _load()
        return getattr(_Lib._lib, name)

    @property
    def loaded(self) -> bool:
        return _Lib._lib is not None


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                      "(or __graft_entry__.build()); there is no CPU fallback")
lib = _Lib()


def check(rc: int) -> None:
    """Raise the Python analogue of the reference's exception for a return code."""
    if rc == OK:
        return
    msg = (lib.dfgtb_last_error() or b"").decode()
    if rc == EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)
