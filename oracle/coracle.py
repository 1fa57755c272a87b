"""ctypes wrapper over oracle/_ref/libzxs_oracle.so — TEST INFRASTRUCTURE ONLY.

The C restatement of the sampler (oracle/zxs_oracle.c) run on the flattened
model arrays. Used as the checker in tests and as bench.py's `cpu_baseline`
"port" leg when the reference library is absent; never by the product.
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))
from paper_2604_01059_b200 import zxs_format  # noqa: E402  (pure-python file format, no GPU code)

LIB_PATH = os.path.join(_HERE, "_ref", "libzxs_oracle.so")
_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_dp = ctypes.POINTER(ctypes.c_double)
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"C oracle not built: {LIB_PATH} (run `make -C oracle`)")
        L = ctypes.CDLL(LIB_PATH)
        D = ctypes.POINTER(zxs_format.ModelDesc)
        L.zo_philox_block.argtypes = [_u32p, _u32p, _u32p]
        L.zo_philox_block.restype = None
        L.zo_uniform_at.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]
        L.zo_uniform_at.restype = ctypes.c_double
        L.zo_sample_error_batch.argtypes = [D, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u64p]
        L.zo_sample_error_batch.restype = None
        L.zo_eval_batch.argtypes = [D, ctypes.c_uint32, _u64p, ctypes.c_uint32, ctypes.c_uint64, _dp]
        L.zo_eval_batch.restype = ctypes.c_double
        L.zo_sample.argtypes = [D, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u64p, _dp, _u64p]
        L.zo_sample.restype = ctypes.c_int
        L.zo_encode.argtypes = [_u64p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                ctypes.c_int, ctypes.POINTER(ctypes.c_uint8), ctypes.c_uint64]
        L.zo_encode.restype = ctypes.c_longlong
        _lib = L
    return _lib


def philox_block(ctr, key) -> list[int]:
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().zo_philox_block(c, k, o)
    return list(o)


def uniform_at(seed: int, stream: int, index: int) -> float:
    return lib().zo_uniform_at(seed, stream, index)


def encode(cols: np.ndarray, shots: int, fmt: int, first_output: int = 0, output_count: int = 0xFFFFFFFF) -> bytes:
    """encode_shots (encode.cpp:22-48) of a [num_outputs][ceil(shots/64)] record."""
    cols = np.ascontiguousarray(cols, np.uint64)
    cap = shots * (cols.shape[0] + 1) + 16
    buf = np.zeros(cap, np.uint8)
    n = lib().zo_encode(cols.ctypes.data_as(_u64p), cols.shape[0], shots, first_output, output_count, fmt,
                        buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), cap)
    if n < 0:
        raise ValueError("encode: invalid arguments")
    return buf[:n].tobytes()


class OracleModel:
    def __init__(self, arrays: dict):
        self.arrays = {k: np.ascontiguousarray(v) for k, v in arrays.items()}
        self.desc = zxs_format.make_desc(self.arrays)
        h = self.arrays["header"]
        self.num_outputs, self.f_width = int(h[3]), int(h[4])
        self.num_positions = int(self.arrays["comp_outputs"].size)

    @classmethod
    def load(cls, path: str) -> "OracleModel":
        return cls(zxs_format.load(path))

    def sample(self, shots: int, seed: int, first_shot: int = 0, fcols=None, uniforms=None) -> np.ndarray:
        out = np.zeros((self.num_outputs, (shots + 63) // 64), np.uint64)
        fp = up = None
        if fcols is not None:
            fcols = np.ascontiguousarray(fcols, np.uint64)
            fp = fcols.ctypes.data_as(_u64p)
        if uniforms is not None:
            uniforms = np.ascontiguousarray(uniforms, np.float64)
            up = uniforms.ctypes.data_as(_dp)
        rc = lib().zo_sample(ctypes.byref(self.desc), seed, first_shot, shots, fp, up, out.ctypes.data_as(_u64p))
        if rc:
            raise RuntimeError("autoregressive ratio outside [0, 1]: numeric breakdown")
        return out

    def sample_error_batch(self, shots: int, seed: int, first_shot: int = 0) -> np.ndarray:
        out = np.zeros((self.f_width, (shots + 63) // 64), np.uint64)
        lib().zo_sample_error_batch(ctypes.byref(self.desc), seed, first_shot, shots, out.ctypes.data_as(_u64p))
        return out

    def eval_batch(self, tensor: int, params: np.ndarray, shots: int):
        params = np.ascontiguousarray(params, np.uint64)
        vals = np.zeros(shots, np.float64)
        mi = lib().zo_eval_batch(ctypes.byref(self.desc), tensor, params.ctypes.data_as(_u64p), params.shape[0],
                                 shots, vals.ctypes.data_as(_dp))
        return vals, mi
