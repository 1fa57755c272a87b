"""Loader for the sm_100a library `_lib/libzxs_b200.so` (C ABI: include/zxs_b200.h).

There is no CPU fallback: if the library is missing, importing the product
API raises. Build it with `python -c "import __graft_entry__ as g; g.build()"`
or `make -C paper_2604_01059_b200/csrc`.
"""
from __future__ import annotations

import ctypes
import os

from . import zxs_format as _fmt

LIB_PATH = os.environ.get("ZXS_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                         "libzxs_b200.so")

ZXS_OK, ZXS_INVALID_ARGUMENT, ZXS_RUNTIME_ERROR, ZXS_CUDA_ERROR, ZXS_OUT_OF_MEMORY, ZXS_UNSUPPORTED = range(6)

_u64p = ctypes.POINTER(ctypes.c_uint64)
_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_vp = ctypes.c_void_p


class SamplerInfo(ctypes.Structure):
    """ctypes mirror of `zxs_sampler_info`."""

    _fields_ = [(n, ctypes.c_uint32) for n in (
        "mode", "num_outputs", "num_detectors", "num_observables", "f_width", "num_mechanisms",
        "num_direct", "num_components", "max_chain", "fwords")] + [
        ("num_terms", ctypes.c_uint64), ("num_factors", ctypes.c_uint64),
        ("num_selector_bits", ctypes.c_uint64), ("philox_blocks_per_shot", ctypes.c_uint64),
        ("device_bytes", ctypes.c_uint64), ("device", ctypes.c_int), ("monomial", ctypes.c_int),
        ("num_mono_components", ctypes.c_uint32), ("num_mono_forms", ctypes.c_uint32),
        ("num_mono_records", ctypes.c_uint64), ("num_mono_dead_terms", ctypes.c_uint64),
        ("num_mono_loads", ctypes.c_uint64), ("num_tab_entries", ctypes.c_uint64),
        ("num_mono_negligible_terms", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


class SampleOptions(ctypes.Structure):
    """ctypes mirror of `zxs_sample_options`."""

    _fields_ = [("force_dense", ctypes.c_uint32), ("reserved", ctypes.c_uint32), ("sparse_threshold", ctypes.c_double)]


# (name, restype, argtypes) for every symbol include/zxs_b200.h declares
SIGNATURES = (
    ("zxs_last_error", ctypes.c_char_p, []),
    ("zxs_abi_version", ctypes.c_uint32, []),
    ("zxs_sampler_create", ctypes.c_int, [ctypes.POINTER(_fmt.ModelDesc), ctypes.c_int, ctypes.POINTER(_vp)]),
    ("zxs_sampler_destroy", None, [_vp]),
    ("zxs_sampler_get_info", ctypes.c_int, [_vp, ctypes.POINTER(SamplerInfo)]),
    ("zxs_sample", ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u64p, _vp]),
    ("zxs_sample_opts", ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.POINTER(SampleOptions), _u64p, _vp]),
    ("zxs_sparse_eligible", ctypes.c_int, [_vp, ctypes.POINTER(SampleOptions), ctypes.POINTER(ctypes.c_int)]),
    ("zxs_sample_device", ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _vp,
                                         ctypes.c_uint64, _vp, _vp]),
    ("zxs_count_device", ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _vp, _vp]),
    ("zxs_count", ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u64p, _vp]),
    ("zxs_check_errors", ctypes.c_int, [_vp, _vp]),
    ("zxs_kernel_timing", ctypes.c_int, [_vp, ctypes.c_int]),
    ("zxs_kernel_times", ctypes.c_int, [_vp, _dp, _u64p]),
    ("zxs_kernel_times_n", ctypes.c_int, [_vp, _dp, _u64p, ctypes.c_uint32]),
    ("zxs_dedup_stats", ctypes.c_int, [_vp, ctypes.c_int, _u64p]),
    ("zxs_tie_count", ctypes.c_int, [_vp, ctypes.c_int, _u64p]),
    ("zxs_encoded_bytes", ctypes.c_uint64, [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                            ctypes.c_uint32]),
    ("zxs_encode_shots_device", ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                               ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _vp, _vp]),
    ("zxs_sample_encoded", ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.POINTER(SampleOptions), ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_uint32, _u8p, _vp]),
    ("zxs_sample_error_batch", ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u64p]),
    ("zxs_eval_batch", ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.c_uint32, _u64p, ctypes.c_uint32,
                                      ctypes.c_uint64, _dp, _dp]),
    ("zxs_eval_batch_mono", ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.c_uint32, _u64p, ctypes.c_uint32,
                                           ctypes.c_uint64, _dp]),
    ("zxs_sample_given_f", ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u64p, _dp,
                                          _u64p]),
    ("zxs_probability_of", ctypes.c_int, [_vp, _u8p, ctypes.c_uint32, _dp]),
    ("zxs_imag_health", ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, _dp]),
    ("zxs_probability_of_at", ctypes.c_int, [_vp, _u8p, ctypes.c_uint32, _u8p, ctypes.c_uint32, _dp]),
    ("zxs_philox_uniform", ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                          ctypes.c_uint64, _dp]),
    ("zxs_measure_philox_peak", ctypes.c_int, [ctypes.c_int, _dp]),
    ("zxs_measure_fp64_peak", ctypes.c_int, [ctypes.c_int, _dp]),
    ("zxs_measure_smem_peak", ctypes.c_int, [ctypes.c_int, _dp]),
    ("zxs_debug_heavy_layout", ctypes.c_int, [ctypes.POINTER(_fmt.ModelDesc), ctypes.c_uint64,
                                              ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint64, _u64p]),
    ("zxs_debug_mono_layout", ctypes.c_int, [ctypes.POINTER(_fmt.ModelDesc), ctypes.c_uint64,
                                             ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint64, _u64p]),
)

_lib = None


def lib():
    """The loaded library; raises if it was not built (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"sm_100a sampler library not built: {LIB_PATH}. Run __graft_entry__.build() "
                "(there is no CPU fallback).")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            if os.environ.get("ZXS_B200_LIB") and not hasattr(L, name):
                continue  # an older A/B build (tests/test_abi.py checks the product library's exports)
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.zxs_abi_version() != 2:
            raise RuntimeError("libzxs_b200.so ABI version mismatch")
        _lib = L
    return _lib


def check(status: int):
    """Maps C-ABI status codes to the reference's exception classes."""
    if status == ZXS_OK:
        return
    msg = lib().zxs_last_error().decode()
    if status == ZXS_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if status == ZXS_OUT_OF_MEMORY:
        raise MemoryError(msg)
    if status == ZXS_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)  # std::runtime_error / CUDA failures
