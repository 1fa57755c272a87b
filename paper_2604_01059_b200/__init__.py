"""B200 (sm_100a) shot sampler for zxsim compiled samplers (Tsim hot path).

The reference front-end (circuit parse, ZX simplification, stabilizer-rank
compile) produces a CompiledSampler on the host; this package uploads its
flattened form (`.zxs`, see zxs_format) to a GPU and runs the per-shot
pipeline — Philox error draw, f = T.e, term contraction, autoregressive bit
loop — as hand-written sm_100a kernels behind the C ABI in include/zxs_b200.h.
"""
from .sampler import (  # noqa: F401
    FORMAT_01,
    FORMAT_B8,
    MODE_DETECTORS,
    MODE_MEASUREMENTS,
    BatchEvalResult,
    CompiledSampler,
    SampleRecord,
    SamplerOptions,
    count_outputs,
    encode_shots,
    eval_batch,
    eval_batch_mono,
    imag_health,
    measure_fp64_peak,
    measure_philox_peak,
    measure_smem_peak,
    philox_uniform,
    probability_of,
    probability_of_at,
    sample_detectors,
    sample_encoded,
    sample_error_batch,
    sample_given_f,
    sample_measurements,
    sparse_eligible,
)

__all__ = [
    "FORMAT_01", "FORMAT_B8", "encode_shots", "sample_encoded", "MODE_DETECTORS", "MODE_MEASUREMENTS", "BatchEvalResult", "CompiledSampler", "SampleRecord",
    "SamplerOptions", "count_outputs", "eval_batch", "eval_batch_mono", "imag_health", "measure_fp64_peak", "measure_philox_peak", "measure_smem_peak",
    "philox_uniform", "probability_of", "probability_of_at",
    "sample_detectors", "sample_error_batch", "sample_given_f", "sample_measurements", "sparse_eligible",
]
