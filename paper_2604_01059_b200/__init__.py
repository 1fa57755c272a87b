"""B200 (sm_100a) shot sampler for zxsim compiled samplers (Tsim hot path).

The reference front-end (circuit parse, ZX simplification, stabilizer-rank
compile) produces a CompiledSampler on the host; this package uploads its
flattened form (`.zxs`, see zxs_format) to a GPU and runs the per-shot
pipeline — Philox error draw, f = T.e, term contraction, autoregressive bit
loop — as hand-written sm_100a kernels behind the C ABI in include/zxs_b200.h.
"""
from .sampler import (  # noqa: F401
    MODE_DETECTORS,
    MODE_MEASUREMENTS,
    BatchEvalResult,
    CompiledSampler,
    SampleRecord,
    SamplerOptions,
    count_outputs,
    eval_batch,
    eval_batch_mono,
    measure_fp64_peak,
    measure_philox_peak,
    philox_uniform,
    probability_of_at,
    sample_detectors,
    sample_error_batch,
    sample_given_f,
    sample_measurements,
)

__all__ = [
    "MODE_DETECTORS", "MODE_MEASUREMENTS", "BatchEvalResult", "CompiledSampler", "SampleRecord",
    "SamplerOptions", "count_outputs", "eval_batch", "eval_batch_mono", "measure_fp64_peak", "measure_philox_peak", "philox_uniform", "probability_of_at",
    "sample_detectors", "sample_error_batch", "sample_given_f", "sample_measurements",
]
