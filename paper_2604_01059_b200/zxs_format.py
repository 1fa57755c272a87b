"""`.zxs` files: a flattened zxsim::CompiledSampler as named numpy arrays.

The same container as include/zxs_flat.hpp (C++ writer/reader): magic
"ZXS1\\0\\0\\0\\0", u32 n_arrays, then per array u32 name_len, name, u32 dtype
(0 u8, 1 u32, 2 i64, 3 f64, 4 u64), u64 count, raw little-endian data padded to
8 bytes. The arrays are exactly the fields of `zxs_model_desc`
(include/zxs_b200.h), which mirrors CompiledSampler
(/root/reference/proj/include/zxsim/compile.hpp:59-72).
"""
from __future__ import annotations

import ctypes
import struct

import numpy as np

_DTYPES = {0: np.uint8, 1: np.uint32, 2: np.int64, 3: np.float64, 4: np.uint64}
_CODES = {np.dtype(v): k for k, v in _DTYPES.items()}

# name -> dtype, in file order (zxs_flat.hpp FlatModel::visit)
FIELDS = (
    ("header", np.uint32),
    ("base_offset", np.uint32),
    ("mech_vec_begin", np.uint32),
    ("vec_bit_begin", np.uint32),
    ("vec_bits", np.uint32),
    ("mech_probability", np.float64),
    ("mech_table_begin", np.uint32),
    ("table", np.float64),
    ("direct_output", np.uint32),
    ("direct_flip_const", np.uint8),
    ("direct_bit_begin", np.uint32),
    ("direct_bits", np.uint32),
    ("comp_out_begin", np.uint32),
    ("comp_outputs", np.uint32),
    ("comp_num_magic", np.uint32),
    ("comp_chi", np.uint64),
    ("comp_tensor_begin", np.uint32),
    ("tensor_param_width", np.uint32),
    ("tensor_exponent_halves", np.int64),
    ("tensor_term_begin", np.uint64),
    ("term_c", np.float64),
    ("term_factor_begin", np.uint64),
    ("factor_table", np.uint32),
    ("factor_u_begin", np.uint64),
    ("factor_u_bits", np.uint32),
    ("factor_v_begin", np.uint64),
    ("factor_v_bits", np.uint32),
    ("h_table", np.float64),
    ("h_alpha", np.float64),
    ("h_beta", np.float64),
)


def load(path: str) -> dict:
    """Reads a .zxs file (or a gzip- / xz-compressed .zxs.gz / .zxs.xz)."""
    if path.endswith(".gz"):
        import gzip
        with gzip.open(path, "rb") as fp:
            data = fp.read()
    elif path.endswith(".xz"):
        import lzma
        with lzma.open(path, "rb") as fp:
            data = fp.read()
    else:
        with open(path, "rb") as fp:
            data = fp.read()
    if data[:4] != b"ZXS1":
        raise ValueError(f"not a .zxs file: {path}")
    (n,) = struct.unpack_from("<I", data, 8)
    off = 12
    arrays = {}
    for _ in range(n):
        (ln,) = struct.unpack_from("<I", data, off)
        name = data[off + 4: off + 4 + ln].decode()
        code, count = struct.unpack_from("<IQ", data, off + 4 + ln)
        dt = np.dtype(_DTYPES[code])
        start = off + 4 + ln + 12
        nbytes = count * dt.itemsize
        arrays[name] = np.frombuffer(data, dt, count, start).copy()
        used = 4 + ln + 12 + nbytes
        off += used + ((8 - used % 8) % 8)
    for name, dt in FIELDS:
        if name not in arrays or arrays[name].dtype != np.dtype(dt):
            raise ValueError(f".zxs array missing or mistyped: {name}")
    return arrays


def save(path: str, arrays: dict):
    with open(path, "wb") as fp:
        fp.write(b"ZXS1\0\0\0\0")
        fp.write(struct.pack("<I", len(FIELDS)))
        for name, dt in FIELDS:
            a = np.ascontiguousarray(arrays[name], dt)
            nb = name.encode()
            fp.write(struct.pack("<I", len(nb)) + nb + struct.pack("<IQ", _CODES[np.dtype(dt)], a.size))
            fp.write(a.tobytes())
            used = 4 + len(nb) + 12 + a.nbytes
            fp.write(b"\0" * ((8 - used % 8) % 8))


# ---------------------------------------------------------------- C-ABI view
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class ModelDesc(ctypes.Structure):
    """ctypes mirror of `zxs_model_desc` (include/zxs_b200.h)."""

    _fields_ = [
        ("abi_version", ctypes.c_uint32), ("mode", ctypes.c_uint32),
        ("num_detectors", ctypes.c_uint32), ("num_observables", ctypes.c_uint32),
        ("num_outputs", ctypes.c_uint32), ("f_width", ctypes.c_uint32),
        ("num_base_offset", ctypes.c_uint32), ("base_offset", _u32p),
        ("num_mechanisms", ctypes.c_uint32), ("mech_vec_begin", _u32p),
        ("num_vectors", ctypes.c_uint32), ("vec_bit_begin", _u32p), ("vec_bits", _u32p),
        ("mech_probability", _dp), ("mech_table_begin", _u32p), ("table", _dp),
        ("num_direct", ctypes.c_uint32), ("direct_output", _u32p), ("direct_flip_const", _u8p),
        ("direct_bit_begin", _u32p), ("direct_bits", _u32p),
        ("num_components", ctypes.c_uint32), ("comp_out_begin", _u32p), ("comp_outputs", _u32p),
        ("comp_num_magic", _u32p), ("comp_chi", _u64p), ("comp_tensor_begin", _u32p),
        ("num_tensors", ctypes.c_uint32), ("tensor_param_width", _u32p),
        ("tensor_exponent_halves", _i64p), ("tensor_term_begin", _u64p),
        ("num_terms", ctypes.c_uint64), ("term_c", _dp), ("term_factor_begin", _u64p),
        ("num_factors", ctypes.c_uint64), ("factor_table", _u32p),
        ("factor_u_begin", _u64p), ("factor_u_bits", _u32p),
        ("factor_v_begin", _u64p), ("factor_v_bits", _u32p),
        ("num_h_tables", ctypes.c_uint32), ("h_table", _dp), ("h_alpha", _dp), ("h_beta", _dp),
        ("flags", ctypes.c_uint32),
    ]


_PTR = {np.dtype(np.uint32): _u32p, np.dtype(np.uint64): _u64p, np.dtype(np.int64): _i64p,
        np.dtype(np.float64): _dp, np.dtype(np.uint8): _u8p}


def make_desc(arrays: dict) -> ModelDesc:
    """Builds the C struct over `arrays` (which must outlive the struct's use)."""
    d = ModelDesc()
    hdr = arrays["header"]
    d.abi_version = 2
    d.mode, d.num_detectors, d.num_observables, d.num_outputs, d.f_width = (int(x) for x in hdr[:5])
    d.flags = int(hdr[5]) if hdr.size > 5 else 0  # ZXS_MODEL_* (absent in older files)
    for name, dt in FIELDS[1:]:
        a = arrays[name]
        assert a.dtype == np.dtype(dt) and a.flags.c_contiguous, name
        setattr(d, name, a.ctypes.data_as(_PTR[a.dtype]))
    d.num_base_offset = arrays["base_offset"].size
    d.num_mechanisms = arrays["mech_vec_begin"].size - 1
    d.num_vectors = arrays["vec_bit_begin"].size - 1
    d.num_direct = arrays["direct_output"].size
    d.num_components = arrays["comp_out_begin"].size - 1
    d.num_tensors = arrays["tensor_param_width"].size
    d.num_terms = arrays["term_factor_begin"].size - 1
    d.num_factors = arrays["factor_table"].size
    d.num_h_tables = arrays["h_alpha"].size
    return d
