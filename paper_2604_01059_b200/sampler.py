"""Host-side mirror of the reference sampler API, backed by the sm_100a library.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/zxsim/sampler.hpp and phase_terms.hpp:

    reference (C++)                                   here
    ---------------------------------------------     -----------------------------------------
    struct SamplerOptions        sampler.hpp:32-38    SamplerOptions
    struct SampleRecord          sampler.hpp:22-30    SampleRecord (columns: [width][words] u64)
    sample_detectors             sampler.hpp:57-58    sample_detectors(cs, shots, opt)
    sample_measurements          sampler.hpp:59-60    sample_measurements(cs, shots, opt)
    sample_error_batch           sampler.hpp:54-55    sample_error_batch(cs, seed, first_shot, shots)
    eval_batch                   phase_terms.hpp:82   eval_batch(cs, component, chain_pos, params, shots)
    probability_of_at            sampler.hpp:67-68    probability_of_at(cs, outcome, f_assignment)
    Philox::uniform_at           rng.hpp:31-41        philox_uniform(seed, stream, first_index, n)

std::invalid_argument surfaces as ValueError, std::runtime_error as
RuntimeError. `CompiledSampler` is the flattened zxsim::CompiledSampler
(compile.hpp:59-72) uploaded to one GPU; every computation runs on the device.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native, zxs_format

MODE_DETECTORS = 0
MODE_MEASUREMENTS = 1

_u64p = ctypes.POINTER(ctypes.c_uint64)
_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


@dataclass
class SamplerOptions:
    """sampler.hpp:32-38. seed, sparse_threshold and force_dense select the bits
    exactly as in the reference (dense path, or the sparse geometric path for
    pure-Clifford deterministic single-mechanism models, sampler.cpp:104-147);
    batch_size and threads do not change them and are accepted for signature
    compatibility."""

    seed: int = 0
    batch_size: int = 65536
    threads: int = 0
    sparse_threshold: float = 8.0
    force_dense: bool = False


@dataclass
class SampleRecord:
    """sampler.hpp:22-30: column-major bits, shot s at bit s&63 of word s>>6."""

    shots: int = 0
    width: int = 0
    columns: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.uint64))

    def get(self, shot: int, output: int) -> bool:
        return bool((int(self.columns[output, shot >> 6]) >> (shot & 63)) & 1)


@dataclass
class BatchEvalResult:
    """phase_terms.hpp:75-78."""

    values: np.ndarray
    max_imag_ratio: float = 0.0


class CompiledSampler:
    """A flattened compiled sampler resident on one GPU."""

    def __init__(self, arrays: dict, device: int = 0):
        L = _native.lib()
        self.arrays = {k: np.ascontiguousarray(v) for k, v in arrays.items()}
        desc = zxs_format.make_desc(self.arrays)
        h = ctypes.c_void_p()
        _native.check(L.zxs_sampler_create(ctypes.byref(desc), device, ctypes.byref(h)))
        self._h = h
        info = _native.SamplerInfo()
        _native.check(L.zxs_sampler_get_info(self._h, ctypes.byref(info)))
        self.info = info.as_dict()
        self.device = device
        hdr = self.arrays["header"]
        self.mode, self.num_detectors, self.num_observables, self.num_outputs, self.f_width = (int(x) for x in hdr[:5])
        cob = self.arrays["comp_out_begin"]
        self.components = [self.arrays["comp_outputs"][cob[i]:cob[i + 1]].tolist() for i in range(len(cob) - 1)]

    @classmethod
    def load(cls, path: str, device: int = 0) -> "CompiledSampler":
        return cls(zxs_format.load(path), device)

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().zxs_sampler_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def num_chain_positions(self) -> int:
        return sum(len(c) for c in self.components)

    # ---- device-resident entry points (bench / multi-GPU) --------------
    def sample_device(self, seed: int, first_shot: int, shots: int, columns_ptr: int, ld_words: int,
                      counts_ptr: int = 0, stream: int = 0):
        """Asynchronous on `stream`; columns/counts are device pointers."""
        _native.check(_native.lib().zxs_sample_device(self._h, seed, first_shot, shots, columns_ptr or None,
                                                      ld_words, counts_ptr or None, stream or None))

    def count_device(self, seed: int, first_shot: int, shots: int, counts_ptr: int, stream: int = 0):
        _native.check(_native.lib().zxs_count_device(self._h, seed, first_shot, shots, counts_ptr, stream or None))

    def check_errors(self, stream: int = 0):
        _native.check(_native.lib().zxs_check_errors(self._h, stream or None))

    def kernel_timing(self, enable: bool):
        """Start (clearing) / stop per-kernel CUDA-event timing of every launch."""
        _native.check(_native.lib().zxs_kernel_timing(self._h, 1 if enable else 0))

    def kernel_times(self) -> dict:
        """{kernel: (total ms, launches)} for shot_kernel, heavy_kernel, mono_kernel and the
        deduplicated path's dedup_eval_kernel and its per-shot/reduction kernels (dedup_aux)."""
        names = ("shot_kernel", "heavy_kernel", "mono_kernel", "dedup_eval_kernel", "dedup_aux")
        ms = (ctypes.c_double * len(names))()
        n = (ctypes.c_uint64 * len(names))()
        _native.check(_native.lib().zxs_kernel_times_n(self._h, ms, n, len(names)))
        return {k: (ms[i], int(n[i])) for i, k in enumerate(names)}

    def mono_chain_positions(self) -> int:
        """Autoregressive positions of the components on the large-chi integer path (their draws
        run in the deduplicated / mono kernels, not in shot_kernel): zxs_debug_mono_layout with
        the sampler's threshold (ZXS_MONO_MIN_FACTORS / ZXS_HEAVY_MIN_FACTORS, default 2000)."""
        import os
        if not self.info["num_mono_components"]:
            return 0
        mf = int(os.environ.get("ZXS_MONO_MIN_FACTORS", os.environ.get("ZXS_HEAVY_MIN_FACTORS", "2000")))
        desc = zxs_format.make_desc(self.arrays)
        need = ctypes.c_uint64()
        L = _native.lib()
        _native.check(L.zxs_debug_mono_layout(ctypes.byref(desc), mf, None, 0, ctypes.byref(need)))
        buf = np.zeros(need.value, np.uint32)
        _native.check(L.zxs_debug_mono_layout(ctypes.byref(desc), mf, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                              buf.size, ctypes.byref(need)))
        n_comps = int(buf[4])
        return int(sum(int(buf[8 + 5 * i + 1]) for i in range(n_comps)))

    def dedup_stats(self, reset: bool = False) -> dict:
        """Counters of the deduplicated large-chi path (include/zxs_b200.h zxs_dedup_stats)."""
        out = (ctypes.c_uint64 * 6)()
        _native.check(_native.lib().zxs_dedup_stats(self._h, int(reset), out))
        return dict(zip(("batches", "fallbacks", "keys", "plane_load_bytes", "eval_launches", "enabled"),
                        (int(x) for x in out)))

    def tie_count(self, reset: bool = False) -> int:
        """Near-tie autoregressive draws of the integer paths since the last reset
        (include/zxs_b200.h zxs_tie_count): the only draws whose bit could differ
        from the reference's."""
        out = ctypes.c_uint64()
        _native.check(_native.lib().zxs_tie_count(self._h, int(reset), ctypes.byref(out)))
        return int(out.value)

    # ---- host-buffer entry points --------------------------------------
    def sample_into(self, expected_mode: int, seed: int, first_shot: int, shots: int, out: np.ndarray,
                    stream: int = 0) -> np.ndarray:
        """zxs_sample into a caller-owned [num_outputs][ceil(shots/64)] u64 array."""
        words = (shots + 63) // 64
        if out.dtype != np.uint64 or out.shape != (self.num_outputs, words) or not out.flags.c_contiguous:
            raise ValueError("output must be a C-contiguous uint64 array [num_outputs][ceil(shots/64)]")
        _native.check(_native.lib().zxs_sample(self._h, expected_mode, seed, first_shot, shots,
                                               out.ctypes.data_as(_u64p), stream or None))
        return out

    def count(self, seed: int, first_shot: int, shots: int) -> np.ndarray:
        out = np.zeros(self.num_outputs, np.uint64)
        _native.check(_native.lib().zxs_count(self._h, seed, first_shot, shots, out.ctypes.data_as(_u64p), None))
        return out


def _sample(cs: CompiledSampler, mode: int, shots: int, opt: SamplerOptions, first_shot: int = 0) -> SampleRecord:
    words = (shots + 63) // 64
    cols = np.zeros((cs.num_outputs, words), np.uint64)
    if cs.mode != mode:
        # same message and class as sampler.cpp:308-309 / 316-317
        raise ValueError("sampler was compiled in measurement mode" if cs.mode == MODE_MEASUREMENTS
                         else "sampler was compiled in detector mode")
    if shots and first_shot == 0:
        o = _native.SampleOptions(1 if opt.force_dense else 0, 0, float(opt.sparse_threshold))
        _native.check(_native.lib().zxs_sample_opts(cs.handle, mode, opt.seed, shots, ctypes.byref(o),
                                                    cols.ctypes.data_as(_u64p), None))
    elif shots:
        cs.sample_into(mode, opt.seed, first_shot, shots, cols)  # dense path, any global shot range
    return SampleRecord(shots=shots, width=cs.num_outputs, columns=cols)


def sparse_eligible(cs: CompiledSampler, opt: SamplerOptions | None = None) -> bool:
    """sampler.cpp:104-117: would sample_* take the sparse geometric path?"""
    opt = opt or SamplerOptions()
    o = _native.SampleOptions(1 if opt.force_dense else 0, 0, float(opt.sparse_threshold))
    e = ctypes.c_int()
    _native.check(_native.lib().zxs_sparse_eligible(cs.handle, ctypes.byref(o), ctypes.byref(e)))
    return bool(e.value)


def sample_detectors(cs: CompiledSampler, shots: int, opt: SamplerOptions | None = None,
                     first_shot: int = 0) -> SampleRecord:
    """sampler.hpp:57-58. `first_shot` (extension) samples the global shot
    range [first_shot, first_shot+shots): bits equal the reference's for those
    shot indices."""
    return _sample(cs, MODE_DETECTORS, shots, opt or SamplerOptions(), first_shot)


def sample_measurements(cs: CompiledSampler, shots: int, opt: SamplerOptions | None = None,
                        first_shot: int = 0) -> SampleRecord:
    """sampler.hpp:59-60."""
    return _sample(cs, MODE_MEASUREMENTS, shots, opt or SamplerOptions(), first_shot)


def count_outputs(cs: CompiledSampler, shots: int, seed: int = 0, first_shot: int = 0) -> np.ndarray:
    """Per-output number of set bits over the shot range (logical-error and
    detector counts for sweeps that do not materialise records)."""
    return cs.count(seed, first_shot, shots)


def sample_error_batch(cs: CompiledSampler, seed: int, first_shot: int, shots: int) -> np.ndarray:
    """sampler.hpp:54-55: the f-columns ParamBatch [f_width][ceil(shots/64)]."""
    out = np.zeros((cs.f_width, (shots + 63) // 64), np.uint64)
    _native.check(_native.lib().zxs_sample_error_batch(cs.handle, seed, first_shot, shots,
                                                       out.ctypes.data_as(_u64p)))
    return out


def eval_batch(cs: CompiledSampler, component: int, chain_pos: int, params: np.ndarray,
               shots: int) -> BatchEvalResult:
    """phase_terms.hpp:82 on chain tensor `chain_pos` (0 = normalization,
    1+j = marginals[j]) of `component`; params is a ParamBatch
    [param_cols][ceil(shots/64)] u64."""
    params = np.ascontiguousarray(params, np.uint64)
    if params.ndim != 2 or params.shape[1] != (shots + 63) // 64:
        raise ValueError("params must be [param_cols][ceil(shots/64)]")
    vals = np.zeros(shots, np.float64)
    mi = ctypes.c_double(0.0)
    _native.check(_native.lib().zxs_eval_batch(cs.handle, component, chain_pos, params.ctypes.data_as(_u64p),
                                               params.shape[0], shots, vals.ctypes.data_as(_dp), ctypes.byref(mi)))
    return BatchEvalResult(vals, mi.value)


def eval_batch_mono(cs: CompiledSampler, component: int, chain_pos: int, params: np.ndarray,
                    shots: int) -> np.ndarray:
    """eval_batch evaluated by the integer monomial kernel that samples
    large-chi components (zxs_mono.cuh): the reference's values up to its
    own rounding of the h tables. NotImplementedError if the component is
    not on that path."""
    params = np.ascontiguousarray(params, np.uint64)
    if params.ndim != 2 or params.shape[1] != (shots + 63) // 64:
        raise ValueError("params must be [param_cols][ceil(shots/64)]")
    vals = np.zeros(shots, np.float64)
    _native.check(_native.lib().zxs_eval_batch_mono(cs.handle, component, chain_pos, params.ctypes.data_as(_u64p),
                                                    params.shape[0], shots, vals.ctypes.data_as(_dp)))
    return vals


def sample_given_f(cs: CompiledSampler, fcols: np.ndarray, shots: int, seed: int = 0, first_shot: int = 0,
                   uniforms: np.ndarray | None = None) -> np.ndarray:
    """run_batch (sampler.cpp:51-102) driven by injected noise: f-columns
    [f_width][words] and optionally the autoregressive uniforms
    [sum of chain lengths][shots]. Returns [num_outputs][words]."""
    fcols = np.ascontiguousarray(fcols, np.uint64)
    out = np.zeros((cs.num_outputs, (shots + 63) // 64), np.uint64)
    up = None
    if uniforms is not None:
        uniforms = np.ascontiguousarray(uniforms, np.float64)
        if uniforms.shape != (cs.num_chain_positions, shots):
            raise ValueError("uniforms must be [sum of chain lengths][shots]")
        up = uniforms.ctypes.data_as(_dp)
    _native.check(_native.lib().zxs_sample_given_f(cs.handle, seed, first_shot, shots,
                                                   fcols.ctypes.data_as(_u64p), up, out.ctypes.data_as(_u64p)))
    return out


def probability_of_at(cs: CompiledSampler, outcome, f_assignment) -> float:
    """sampler.hpp:67-68 (sampler.cpp:360-368), evaluated on the device."""
    o = np.ascontiguousarray(np.asarray(outcome, np.uint8))
    f = np.ascontiguousarray(np.asarray(f_assignment, np.uint8))
    out = ctypes.c_double()
    _native.check(_native.lib().zxs_probability_of_at(cs.handle, o.ctypes.data_as(_u8p), o.size,
                                                      f.ctypes.data_as(_u8p), f.size, ctypes.byref(out)))
    return out.value


FORMAT_01, FORMAT_B8 = 0, 1  # ShotFormat::ascii01 / b8 (encode.hpp:25)


def sample_encoded(cs: CompiledSampler, shots: int, opt: SamplerOptions | None = None, fmt: int = FORMAT_B8,
                   first_output: int = 0, output_count: int = 0xFFFFFFFF, first_shot: int = 0,
                   mode: int | None = None) -> bytes:
    """The CLI's write path, fused on the device (zxsim.cpp:142-163):
    encode_shots(sample_detectors/measurements(cs, shots, opt), fmt, first_output, output_count)."""
    opt = opt or SamplerOptions()
    mode = cs.mode if mode is None else mode
    n = _native.lib().zxs_encoded_bytes(cs.num_outputs, shots, first_output, output_count, fmt)
    out = np.zeros(max(n, 1), np.uint8)
    o = _native.SampleOptions(1 if opt.force_dense else 0, 0, float(opt.sparse_threshold))
    _native.check(_native.lib().zxs_sample_encoded(cs.handle, mode, opt.seed, first_shot, shots, ctypes.byref(o), fmt,
                                                   first_output, output_count, out.ctypes.data_as(_u8p), None))
    return out[:n].tobytes()


def encode_shots(columns: np.ndarray, shots: int, fmt: int = FORMAT_B8, first_output: int = 0,
                 output_count: int = 0xFFFFFFFF, device: int = 0) -> bytes:
    """encode_shots (encode.hpp:29) of a host record [num_outputs][ceil(shots/64)], run on the GPU."""
    import torch
    cols = np.ascontiguousarray(columns, np.uint64)
    nout, words = cols.shape
    if words < (shots + 63) // 64:
        raise ValueError("record has fewer words than ceil(shots/64)")
    n = _native.lib().zxs_encoded_bytes(nout, shots, first_output, output_count, fmt)
    if n == 0 and shots:
        if first_output > nout or fmt not in (FORMAT_01, FORMAT_B8):
            raise ValueError("encode_shots: invalid arguments")
        return b""
    dev = torch.device("cuda", device)
    dcols = torch.from_numpy(cols.view(np.int64)).to(dev)
    dout = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev)
    _native.check(_native.lib().zxs_encode_shots_device(dcols.data_ptr(), words, nout, shots, first_output,
                                                        output_count, fmt, dout.data_ptr(), st.cuda_stream))
    return dout[:n].cpu().numpy().tobytes()


def probability_of(cs: CompiledSampler, outcome) -> float:
    """sampler.hpp:64 (sampler.cpp:370-429): exact outcome probability; leaves on the device."""
    o = np.ascontiguousarray(np.asarray(outcome, np.uint8))
    out = ctypes.c_double()
    _native.check(_native.lib().zxs_probability_of(cs.handle, o.ctypes.data_as(_u8p), o.size, ctypes.byref(out)))
    return out.value


def imag_health(cs: CompiledSampler, samples: int = 4096, seed: int = 1) -> np.ndarray:
    """Per component, max |Im P| / |P| over random parameter vectors (phase_terms.cpp:134-141;
    SURVEY finding 3: the reference never checks it)."""
    out = np.zeros(max(len(cs.components), 1), np.float64)
    _native.check(_native.lib().zxs_imag_health(cs.handle, samples, seed, out.ctypes.data_as(_dp)))
    return out[:len(cs.components)]


def measure_philox_peak(device: int = 0) -> float:
    """Philox4x32-10 blocks/s of the draw code alone (same-op-mix roofline)."""
    out = ctypes.c_double()
    _native.check(_native.lib().zxs_measure_philox_peak(device, ctypes.byref(out)))
    return out.value


def measure_fp64_peak(device: int = 0) -> float:
    """FP64 DMUL+DADD ops/s of the exact contraction's op mix (heavy_kernel roofline)."""
    out = ctypes.c_double()
    _native.check(_native.lib().zxs_measure_fp64_peak(device, ctypes.byref(out)))
    return out.value


def measure_smem_peak(device: int = 0) -> float:
    """Shared-memory bytes/s of conflict-free LDS + XOR (mono_kernel roofline)."""
    out = ctypes.c_double()
    _native.check(_native.lib().zxs_measure_smem_peak(device, ctypes.byref(out)))
    return out.value


def philox_uniform(seed: int, stream: int, first_index: int, n: int, device: int = 0) -> np.ndarray:
    """Philox(seed, stream).uniform_at(first_index + i), i < n, on the device."""
    out = np.zeros(n, np.float64)
    _native.check(_native.lib().zxs_philox_uniform(device, seed, stream, first_index, n,
                                                   out.ctypes.data_as(_dp)))
    return out
