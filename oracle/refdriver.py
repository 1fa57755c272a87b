"""ctypes wrapper over oracle/_ref/libzxsim_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the unmodified reference (zxsim, /root/reference/proj/src)
compiled in place by oracle/Makefile, plus oracle/ref_driver.cpp. It is the
checker the CUDA path is compared against; only tests/, __graft_entry__.smoke()
and bench.py's reference / cpu_baseline legs may load it. Never imported by the
product package.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libzxsim_ref.so")
# The same library with the front-end's cat5 normalisation fixed (oracle/Makefile
# `fixed`): only ever used to COMPILE a circuit to a .zxs file, which the
# unmodified library then loads, samples and evaluates.
FIXED_LIB_PATH = os.path.join(_HERE, "_ref", "libzxsim_fixed.so")
_fixed_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run `make -C oracle`)")
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        L.zr_last_error.restype = ctypes.c_char_p
        L.zr_compile.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(vp)]
        L.zr_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
        L.zr_save.argtypes = [vp, ctypes.c_char_p]
        L.zr_free.argtypes = [vp]
        L.zr_free.restype = None
        L.zr_info.argtypes = [vp, _u64p]
        L.zr_format_stats.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
        L.zr_sample.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                ctypes.c_uint32, ctypes.c_int, _u64p]
        L.zr_sample_opts.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double, _u64p]
        L.zr_sample_opts.restype = ctypes.c_int
        L.zr_sample_rb.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_uint64, ctypes.c_uint32, _u64p]
        L.zr_sample_given_f.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                        _u64p, _dp, _u64p]
        L.zr_sample_error_batch.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                            _u64p]
        L.zr_eval_batch.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32, _u64p, ctypes.c_uint32,
                                    ctypes.c_uint64, _dp, _dp]
        L.zr_probability_of_at.argtypes = [vp, _u8p, _u8p, _dp]
        L.zr_probability_of.argtypes = [vp, _u8p, _dp]
        L.zr_uniform_at.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]
        L.zr_uniform_at.restype = ctypes.c_double
        L.zr_encode.argtypes = [_u64p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                                ctypes.c_char_p, ctypes.c_uint64, _u64p]
        L.zr_plan.argtypes = [ctypes.c_char_p, ctypes.c_int, _u64p]
        L.zr_oracle_distribution.argtypes = [ctypes.c_char_p, ctypes.c_int, _u64p, _dp, ctypes.c_uint64, _u64p]
        _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().zr_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _ptr(a, t=_u64p):
    return a.ctypes.data_as(t)


INFO_KEYS = ("mode", "num_detectors", "num_observables", "num_outputs", "f_width",
             "num_mechanisms", "num_direct", "num_components", "num_joint", "max_chain",
             "num_terms", "num_factors", "chi", "num_magic", "pure_clifford_deterministic",
             "separation_complete")


class RefModel:
    """A zxsim::CompiledSampler held by the reference library."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def compile(cls, text: str, mode: int = 0) -> "RefModel":
        h = ctypes.c_void_p()
        _check(lib().zr_compile(text.encode(), mode, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def compile_fixed(cls, text: str, mode: int = 0) -> "RefModel":
        """Compiled by the front-end with the cat5 fix (decompose.cpp:106), then
        handed to the unmodified library through the lossless .zxs round trip."""
        import tempfile
        with tempfile.NamedTemporaryFile(suffix=".zxs") as tmp:
            compile_fixed_to(text, mode, tmp.name)
            return cls.load(tmp.name)

    @classmethod
    def load(cls, path: str) -> "RefModel":
        h = ctypes.c_void_p()
        if path.endswith((".gz", ".xz")):  # the C++ loader reads plain .zxs: inflate to a temp file
            import gzip
            import lzma
            import shutil
            import tempfile
            with tempfile.NamedTemporaryFile(suffix=".zxs") as tmp:
                with (gzip.open(path, "rb") if path.endswith(".gz") else lzma.open(path, "rb")) as src:
                    shutil.copyfileobj(src, tmp, 1 << 24)
                tmp.flush()
                _check(lib().zr_load(os.fsencode(tmp.name), ctypes.byref(h)))
        else:
            _check(lib().zr_load(os.fsencode(path), ctypes.byref(h)))
        return cls(h)

    def save(self, path: str):
        _check(lib().zr_save(self._h, os.fsencode(path)))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.zr_free(self._h)
            self._h = None

    @property
    def info(self) -> dict:
        a = np.zeros(16, np.uint64)
        _check(lib().zr_info(self._h, _ptr(a)))
        return {k: int(v) for k, v in zip(INFO_KEYS, a)}

    def stats(self) -> str:
        buf = ctypes.create_string_buffer(1 << 16)
        _check(lib().zr_format_stats(self._h, buf, len(buf)))
        return buf.value.decode()

    def sample(self, shots: int, seed: int, batch_size: int = 65536, threads: int = 0,
               force_dense: bool = True) -> np.ndarray:
        """The reference's sample_detectors/measurements: [num_outputs][words] u64."""
        n = self.info["num_outputs"]
        out = np.zeros((n, (shots + 63) // 64), np.uint64)
        _check(lib().zr_sample(self._h, shots, seed, batch_size, threads, int(force_dense), _ptr(out)))
        return out

    def sample_opts(self, shots: int, seed: int, sparse_threshold: float = 8.0, force_dense: bool = False) -> np.ndarray:
        """sample_* with the options that select the sparse path (sampler.cpp:104-117)."""
        n = self.info["num_outputs"]
        out = np.zeros((n, (shots + 63) // 64), np.uint64)
        _check(lib().zr_sample_opts(self._h, shots, seed, int(force_dense), sparse_threshold, _ptr(out)))
        return out

    def sample_rb(self, shots: int, seed: int, first_shot: int = 0, batch_size: int = 65536,
                  threads: int = 0) -> np.ndarray:
        """run_batch restatement (per-component widths, any first_shot)."""
        n = self.info["num_outputs"]
        out = np.zeros((n, (shots + 63) // 64), np.uint64)
        _check(lib().zr_sample_rb(self._h, seed, first_shot, shots, batch_size, threads, _ptr(out)))
        return out

    def sample_given_f(self, fcols: np.ndarray, shots: int, seed: int = 0, first_shot: int = 0,
                       uniforms: np.ndarray | None = None) -> np.ndarray:
        n = self.info["num_outputs"]
        out = np.zeros((n, (shots + 63) // 64), np.uint64)
        fcols = np.ascontiguousarray(fcols, np.uint64)
        up = None
        if uniforms is not None:
            uniforms = np.ascontiguousarray(uniforms, np.float64)
            up = _ptr(uniforms, _dp)
        _check(lib().zr_sample_given_f(self._h, seed, first_shot, shots, _ptr(fcols), up, _ptr(out)))
        return out

    def sample_error_batch(self, shots: int, seed: int, first_shot: int = 0) -> np.ndarray:
        fw = self.info["f_width"]
        out = np.zeros((fw, (shots + 63) // 64), np.uint64)
        _check(lib().zr_sample_error_batch(self._h, seed, first_shot, shots, _ptr(out)))
        return out

    def eval_batch(self, component: int, chain_pos: int, params: np.ndarray, shots: int):
        params = np.ascontiguousarray(params, np.uint64)
        vals = np.zeros(shots, np.float64)
        mi = ctypes.c_double(0.0)
        _check(lib().zr_eval_batch(self._h, component, chain_pos, _ptr(params), params.shape[0],
                                   shots, _ptr(vals, _dp), ctypes.byref(mi)))
        return vals, mi.value

    def probability_of_at(self, outcome, f) -> float:
        o = np.ascontiguousarray(outcome, np.uint8)
        fa = np.ascontiguousarray(f, np.uint8)
        out = ctypes.c_double()
        _check(lib().zr_probability_of_at(self._h, _ptr(o, _u8p), _ptr(fa, _u8p), ctypes.byref(out)))
        return out.value

    def probability_of(self, outcome) -> float:
        o = np.ascontiguousarray(outcome, np.uint8)
        out = ctypes.c_double()
        _check(lib().zr_probability_of(self._h, _ptr(o, _u8p), ctypes.byref(out)))
        return out.value


def fixed_available() -> bool:
    return os.path.exists(FIXED_LIB_PATH)


def compile_fixed_to(text: str, mode: int, path: str) -> None:
    """Compile with the fixed front-end and write the .zxs model to `path`."""
    global _fixed_lib
    if _fixed_lib is None:
        if not fixed_available():
            raise RuntimeError(f"fixed front-end not built: {FIXED_LIB_PATH} (run `make -C oracle fixed`)")
        L = ctypes.CDLL(FIXED_LIB_PATH)
        vp = ctypes.c_void_p
        L.zr_last_error.restype = ctypes.c_char_p
        L.zr_compile.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(vp)]
        L.zr_save.argtypes = [vp, ctypes.c_char_p]
        L.zr_free.argtypes = [vp]
        L.zr_free.restype = None
        _fixed_lib = L
    h = ctypes.c_void_p()
    if _fixed_lib.zr_compile(text.encode(), mode, ctypes.byref(h)) != 0:
        raise RuntimeError(_fixed_lib.zr_last_error().decode())
    try:
        if _fixed_lib.zr_save(h, os.fsencode(path)) != 0:
            raise RuntimeError(_fixed_lib.zr_last_error().decode())
    finally:
        _fixed_lib.zr_free(h)


def plan(text: str, mode: int = 0) -> dict:
    """Front-end probe (lower, simplify, plan_decomposition; no tensors)."""
    out = np.zeros(5, np.uint64)
    _check(lib().zr_plan(text.encode(), mode, _ptr(out)))
    return dict(zip(("num_magic", "chi", "vertices", "e_params", "channels"), (int(x) for x in out)))


def oracle_distribution(text: str, mode: int = 0) -> dict:
    """The reference's exact statevector oracle: {outcome key: probability}."""
    cap = 1 << 16
    keys = np.zeros(cap, np.uint64)
    probs = np.zeros(cap, np.float64)
    n = ctypes.c_uint64()
    _check(lib().zr_oracle_distribution(text.encode(), mode, _ptr(keys), _ptr(probs, _dp), cap, ctypes.byref(n)))
    m = min(n.value, cap)
    return {int(k): float(p) for k, p in zip(keys[:m], probs[:m])}


def uniform_at(seed: int, stream: int, index: int) -> float:
    return lib().zr_uniform_at(seed, stream, index)


def encode(cols: np.ndarray, shots: int, fmt: int) -> bytes:
    cols = np.ascontiguousarray(cols, np.uint64)
    width = cols.shape[0]
    cap = shots * (width + 1) + 16
    buf = ctypes.create_string_buffer(cap)
    written = ctypes.c_uint64()
    _check(lib().zr_encode(_ptr(cols), width, shots, fmt, buf, cap, ctypes.byref(written)))
    return buf.raw[: written.value]


def fnv1a64(cols: np.ndarray) -> str:
    """SURVEY Appendix C hash: FNV-1a-64 over every column word, LE bytes."""
    data = np.ascontiguousarray(cols, np.uint64).tobytes()
    h = 0xCBF29CE484222325
    # vectorised over bytes would need a scan; chunk through python for moderate sizes
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
