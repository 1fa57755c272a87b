/*
 * zxs_b200.h — C ABI of the B200 (sm_100a) shot sampler for zxsim compiled samplers.
 *
 * This is the drop-in boundary for the reference's shot-sampling hot path
 * (/root/reference/proj). The reference front-end (parse_circuit, lower,
 * clifford_simplify, compile_circuit) stays on the host; its product, a
 * `zxsim::CompiledSampler` (proj/include/zxsim/compile.hpp:59-72), is flattened
 * into `zxs_model_desc` (plain arrays, no C++ types) and uploaded once. The
 * entry points below replace, one for one:
 *
 *   zxs_sample                 sample_detectors / sample_measurements
 *                              (proj/include/zxsim/sampler.hpp:57-60,
 *                               proj/src/sampler.cpp:119-210, 306-320)
 *   zxs_sample_device          same, output left in device memory (bench / chaining)
 *   zxs_count[_device]         per-output flip counts of the same shots (the
 *                              1e9-shot sweep; NCCL all-reduces these across GPUs)
 *   zxs_sample_error_batch     sample_error_batch (sampler.hpp:54-55, sampler.cpp:257-304)
 *   zxs_eval_batch             eval_batch (phase_terms.hpp:82, phase_terms.cpp:90-144)
 *   zxs_sample_given_f         run_batch (sampler.cpp:51-102) driven by injected
 *                              f-columns and (optionally) injected uniforms
 *   zxs_probability_of_at      probability_of_at (sampler.hpp:67-68, sampler.cpp:360-368)
 *   zxs_philox_uniform         Philox::uniform_at (proj/include/zxsim/rng.hpp:31-41)
 *
 * Bit layout of every column array is the reference's (sampler.hpp:22-30,
 * phase_terms.hpp:64-73): column-major, shot s at bit (s & 63) of 64-bit
 * word (s >> 6), little-endian; words per column = ceil(shots / 64); tail
 * bits beyond `shots` are zero.
 *
 * Error model: every call returns a zxs_status. ZXS_INVALID_ARGUMENT maps to
 * the reference's std::invalid_argument, ZXS_RUNTIME_ERROR to
 * std::runtime_error (e.g. "autoregressive ratio outside [0, 1]: numeric
 * breakdown", sampler.cpp:86-89); zxs_last_error() returns the message of the
 * calling thread's last failure. There is no CPU fallback: a missing GPU is
 * ZXS_CUDA_ERROR.
 */
#ifndef ZXS_B200_H_
#define ZXS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZXS_ABI_VERSION 2u

/* zxs_model_desc.flags */
#define ZXS_MODEL_PURE_CLIFFORD_DETERMINISTIC 1u /* CompiledSampler.stats.pure_clifford_deterministic (compile.cpp:324-325) */

typedef enum zxs_status {
    ZXS_OK = 0,
    ZXS_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    ZXS_RUNTIME_ERROR = 2,    /* std::runtime_error in the reference */
    ZXS_CUDA_ERROR = 3,       /* no device / launch failure */
    ZXS_OUT_OF_MEMORY = 4,
    ZXS_UNSUPPORTED = 5       /* shape outside the compiled kernel envelope */
} zxs_status;

typedef enum zxs_mode {
    ZXS_MODE_DETECTORS = 0,   /* SampleMode::detectors  (lowering.hpp:38) */
    ZXS_MODE_MEASUREMENTS = 1 /* SampleMode::measurements */
} zxs_mode;

/*
 * Flattened zxsim::CompiledSampler. Every *_begin array is a CSR offset
 * array with (count + 1) entries. All pointers are host memory, read only
 * during zxs_sampler_create.
 */
typedef struct zxs_model_desc {
    uint32_t abi_version; /* = ZXS_ABI_VERSION */
    uint32_t mode;        /* zxs_mode (compile.hpp:60) */
    uint32_t num_detectors, num_observables, num_outputs;
    uint32_t f_width; /* compile.hpp:64 */

    /* ErrorModel (error_model.hpp:40-44) */
    uint32_t num_base_offset;    /* base_offset as a list of set f indices */
    const uint32_t *base_offset;
    uint32_t num_mechanisms;
    const uint32_t *mech_vec_begin;  /* [num_mechanisms+1] -> f_vectors     */
    uint32_t num_vectors;
    const uint32_t *vec_bit_begin;   /* [num_vectors+1]    -> vec_bits      */
    const uint32_t *vec_bits;        /* set f indices of each f_vector      */
    const double *mech_probability;  /* [num_mechanisms] (singles)          */
    const uint32_t *mech_table_begin;/* [num_mechanisms+1] -> table (joints)*/
    const double *table;             /* joint tables, 2^k entries each      */

    /* DirectOutput (compile.hpp:26-30) */
    uint32_t num_direct;
    const uint32_t *direct_output;
    const uint8_t *direct_flip_const;
    const uint32_t *direct_bit_begin; /* [num_direct+1] */
    const uint32_t *direct_bits;

    /* AutoComponent (compile.hpp:35-41): outputs in chain order */
    uint32_t num_components;
    const uint32_t *comp_out_begin;   /* [num_components+1] */
    const uint32_t *comp_outputs;
    const uint32_t *comp_num_magic;   /* [num_components] */
    const uint64_t *comp_chi;         /* [num_components] */
    /* component c owns tensors comp_tensor_begin[c] .. comp_tensor_begin[c+1]-1:
       [normalization, marginals[0], ..., marginals[n_out-1]] */
    const uint32_t *comp_tensor_begin;/* [num_components+1] */

    /* PhaseTermTensors (phase_terms.hpp:39-47) */
    uint32_t num_tensors;
    const uint32_t *tensor_param_width;    /* [num_tensors] */
    const int64_t *tensor_exponent_halves; /* [num_tensors] */
    const uint64_t *tensor_term_begin;     /* [num_tensors+1] */
    /* PhaseTerm (phase_terms.hpp:27-37) */
    uint64_t num_terms;
    const double *term_c;                  /* [2*num_terms] (re, im)          */
    const uint64_t *term_factor_begin;     /* [num_terms+1]                   */
    uint64_t num_factors;
    const uint32_t *factor_table;          /* [num_factors] -> h-table index  */
    const uint64_t *factor_u_begin;        /* [num_factors+1] -> factor_u_bits */
    const uint32_t *factor_u_bits;         /* set param indices of u_k        */
    const uint64_t *factor_v_begin;        /* [num_factors+1] -> factor_v_bits */
    const uint32_t *factor_v_bits;         /* set param indices of v_k        */
    /* distinct h tables: h[(a<<1)|b] as (re, im), plus the phase pair they
       were built from (phase_terms.cpp:40-47, scalar.cpp:81-85) */
    uint32_t num_h_tables;
    const double *h_table;                 /* [8*num_h_tables]                */
    const double *h_alpha;                 /* [num_h_tables]                  */
    const double *h_beta;                  /* [num_h_tables]                  */

    /* ZXS_MODEL_* bits; gates the sparse geometric path (sampler.cpp:104-117) */
    uint32_t flags;
} zxs_model_desc;

/* SamplerOptions (sampler.hpp:32-38) fields that change the sampled bits.
   batch_size and threads do not (any batch split gives the same record). */
typedef struct zxs_sample_options {
    uint32_t force_dense;      /* default 0 */
    uint32_t reserved;
    double sparse_threshold;   /* default 8.0 */
} zxs_sample_options;

typedef enum zxs_format {
    ZXS_FORMAT_01 = 0, /* ShotFormat::ascii01 (encode.hpp:25) */
    ZXS_FORMAT_B8 = 1  /* ShotFormat::b8 */
} zxs_format;

typedef struct zxs_sampler zxs_sampler;

typedef struct zxs_sampler_info {
    uint32_t mode, num_outputs, num_detectors, num_observables, f_width;
    uint32_t num_mechanisms, num_direct, num_components, max_chain;
    uint32_t fwords;          /* 64-bit words of the per-shot f register file */
    uint64_t num_terms, num_factors, num_selector_bits;
    uint64_t philox_blocks_per_shot; /* num_mechanisms + sum of chain lengths */
    uint64_t device_bytes;    /* resident model bytes in HBM */
    int device;
    int monomial;             /* 1 if every h entry is an exact Clifford monomial */
    /* large-chi components lowered to the integer monomial path (zxs_mono.cuh) */
    uint32_t num_mono_components, num_mono_forms;
    uint64_t num_mono_records, num_mono_dead_terms;
    uint64_t num_mono_loads;  /* parameter-plane loads per 32-shot word per pass over the mono chains */
    uint64_t num_tab_entries; /* tabulated-chain ratio entries (small components, shot_kernel) */
    uint64_t num_mono_negligible_terms; /* terms with |c'| < 2^-40 of their tensor's largest (dropped) */
} zxs_sampler_info;

/* Message of the calling thread's last failed call ("" if none). */
const char *zxs_last_error(void);
uint32_t zxs_abi_version(void);

/* Uploads the model to `device` (cudaSetDevice ordinal). */
zxs_status zxs_sampler_create(const zxs_model_desc *desc, int device, zxs_sampler **out);
void zxs_sampler_destroy(zxs_sampler *s);
zxs_status zxs_sampler_get_info(const zxs_sampler *s, zxs_sampler_info *info);

/*
 * sample_detectors / sample_measurements for shots [first_shot, first_shot+shots)
 * (global shot indices: the output is a pure function of (model, seed, shot
 * index), so any split of the shot range gives the same bits).
 * `expected_mode` reproduces the reference's mode check (sampler.cpp:308-317).
 * host_columns: [num_outputs][ceil(shots/64)] uint64, written in full.
 * stream: a cudaStream_t, or NULL for the sampler's own stream. Synchronous.
 */
zxs_status zxs_sample(zxs_sampler *s, uint32_t expected_mode, uint64_t seed,
                      uint64_t first_shot, uint64_t shots, uint64_t *host_columns,
                      void *stream);

/*
 * sample_detectors / sample_measurements with the reference's options, whole
 * record from shot 0: when the model is pure-Clifford deterministic, every
 * mechanism is a single with p < 1 and the expected flips per shot are below
 * sparse_threshold (and !force_dense), the reference's sparse geometric path
 * (sampler.cpp:104-147, 214-255: per-mechanism geometric gaps on
 * RngStream(seed, m), constant outputs as all-ones words) runs on the device;
 * otherwise the dense path (same bits as zxs_sample). opts may be NULL
 * (defaults). Synchronous.
 */
zxs_status zxs_sample_opts(zxs_sampler *s, uint32_t expected_mode, uint64_t seed, uint64_t shots,
                           const zxs_sample_options *opts, uint64_t *host_columns, void *stream);

/* Near-tie draws since the last reset: autoregressive draws of the integer
 * (monomial / deduplicated) paths whose uniform fell within 1e-9 (relative)
 * of the ratio -- the only draws whose bit could differ from the reference's
 * (those paths reproduce the reference's values up to its own rounding of the
 * h tables). The exact paths never count. reset != 0 clears the count. */
zxs_status zxs_tie_count(zxs_sampler *s, int reset, uint64_t *out);

/* 1 if zxs_sample_opts would take the sparse geometric path (sparse_eligible). */
zxs_status zxs_sparse_eligible(const zxs_sampler *s, const zxs_sample_options *opts, int *eligible);

/*
 * Device-resident variant: dev_columns is device memory [num_outputs][ld_words]
 * uint64 with ld_words >= ceil(shots/64). dev_counts (nullable, device,
 * [num_outputs] uint64) is incremented by the per-output number of set bits.
 * Enqueued on `stream` (a cudaStream_t; NULL is the legacy default stream).
 * Calls on one sampler are serialised (its per-shot scratch is shared by
 * every entry point), so concurrent calls on different streams do not
 * overlap. Large-chi components on the deduplicated path synchronise the
 * stream once per batch (key counts); everything else returns without
 * waiting. Shots are processed in batches of at most 2^28. Errors in the
 * autoregressive ratio check are reported by the next zxs_check_errors /
 * synchronous call.
 */
zxs_status zxs_sample_device(zxs_sampler *s, uint64_t seed, uint64_t first_shot,
                             uint64_t shots, uint64_t *dev_columns, uint64_t ld_words,
                             uint64_t *dev_counts, void *stream);

/* Counts only (no bit record): dev_counts[num_outputs] += flips. Enqueued like zxs_sample_device. */
zxs_status zxs_count_device(zxs_sampler *s, uint64_t seed, uint64_t first_shot,
                            uint64_t shots, uint64_t *dev_counts, void *stream);
/* Host variant of the above: host_counts[num_outputs] is overwritten. Synchronous. */
zxs_status zxs_count(zxs_sampler *s, uint64_t seed, uint64_t first_shot, uint64_t shots,
                     uint64_t *host_counts, void *stream);

/*
 * Per-kernel device timing: zxs_kernel_timing(s, 1) clears and starts
 * recording CUDA events around every launch of the shot kernel [0], the
 * exact large-chi kernel [1] and the monomial kernel [2] (on the launch
 * stream); zxs_kernel_times sums their elapsed ms and launch counts.
 * zxs_kernel_timing(s, 0) stops. Used by bench.py for the roofline.
 */
zxs_status zxs_kernel_timing(zxs_sampler *s, int enable);
zxs_status zxs_kernel_times(zxs_sampler *s, double *ms /*[3]*/, uint64_t *launches /*[3]*/);
/* The same for the first n timing slots: [3] the deduplicated path's
 * contraction kernel (dedup_eval_kernel), [4] its per-shot and reduction
 * kernels (key hashing, autoregressive steps, segment folds, table clears). */
zxs_status zxs_kernel_times_n(zxs_sampler *s, double *ms, uint64_t *launches, uint32_t n);

/*
 * Counters of the deduplicated large-chi path (zxs_dedup.cuh): out[0] batches,
 * out[1] batches that fell back to the per-shot kernel (more distinct keys
 * than ZXS_DEDUP_MAX_KEYS), out[2] distinct keys evaluated (summed over chain
 * positions), out[3] algorithmic shared-memory plane-load bytes of those
 * evaluations, out[4] dedup_eval_kernel launches, out[5] 1 if the path is
 * enabled. reset != 0 clears the counters after reading.
 */
zxs_status zxs_dedup_stats(zxs_sampler *s, int reset, uint64_t *out /*[6]*/);

/* Synchronizes `stream` and reports (then clears) a device-side ratio breakdown. */
zxs_status zxs_check_errors(zxs_sampler *s, void *stream);

/*
 * encode_shots (proj/src/encode.cpp:22-48) of a device record on the device:
 * dev_columns [num_outputs][ld_words] -> dev_out, shot-major, outputs
 * [first_output, first_output + output_count) clamped to the record width as
 * the reference does. 01: per shot `width` chars + '\n'; b8: per shot
 * ceil(width/8) bytes, bit b % 8 of byte b / 8. zxs_encoded_bytes gives the
 * output size (0 for invalid arguments). Asynchronous on `stream`.
 */
uint64_t zxs_encoded_bytes(uint32_t num_outputs, uint64_t shots, uint32_t first_output,
                           uint32_t output_count, uint32_t format);
zxs_status zxs_encode_shots_device(const uint64_t *dev_columns, uint64_t ld_words, uint32_t num_outputs,
                                   uint64_t shots, uint32_t first_output, uint32_t output_count,
                                   uint32_t format, uint8_t *dev_out, void *stream);

/*
 * The CLI's sample path fused (zxsim.cpp:142-163):
 * write_output(encode_shots(sample_detectors/measurements(cs, shots, opts), fmt, first, count))
 * with sampling and encoding on the device and only the encoded bytes copied
 * to host_out (zxs_encoded_bytes(...) bytes). opts (nullable: defaults) as in
 * zxs_sample_opts; the sparse path applies to first_shot == 0. Synchronous.
 */
zxs_status zxs_sample_encoded(zxs_sampler *s, uint32_t expected_mode, uint64_t seed, uint64_t first_shot,
                              uint64_t shots, const zxs_sample_options *opts, uint32_t format,
                              uint32_t first_output, uint32_t output_count, uint8_t *host_out, void *stream);

/* f-columns after the dense error draw: host_fcols [f_width][ceil(shots/64)]. */
zxs_status zxs_sample_error_batch(zxs_sampler *s, uint64_t seed, uint64_t first_shot,
                                  uint64_t shots, uint64_t *host_fcols);

/*
 * eval_batch on one chain tensor of one component: chain_pos 0 is the
 * normalization, chain_pos 1+j the marginal of output j. host_params is a
 * ParamBatch: [param_cols][ceil(shots/64)] with param_cols >= the tensor's
 * param_width. host_values[shots] receives the real parts; max_imag_ratio
 * (nullable) the reference's max |Im|/|P| (phase_terms.cpp:137-141).
 */
zxs_status zxs_eval_batch(zxs_sampler *s, uint32_t component, uint32_t chain_pos,
                          const uint64_t *host_params, uint32_t param_cols, uint64_t shots,
                          double *host_values, double *max_imag_ratio);

/*
 * Same contract as zxs_eval_batch, evaluated by the integer monomial kernel
 * (zxs_mono.cuh) that samples large-chi components: the values equal the
 * reference's eval_batch up to the reference's own rounding of its h tables.
 * ZXS_UNSUPPORTED if the component is not on that path.
 */
zxs_status zxs_eval_batch_mono(zxs_sampler *s, uint32_t component, uint32_t chain_pos,
                               const uint64_t *host_params, uint32_t param_cols, uint64_t shots,
                               double *host_values);

/*
 * run_batch with the noise configuration injected: host_fcols
 * [f_width][ceil(shots/64)] replaces the Philox error draw. host_uniforms
 * (nullable) injects the autoregressive draws: [sum_c n_out(c)][shots]
 * doubles in (component, chain position) order; NULL uses Philox(seed,
 * auto_stream(c, pos)).uniform_at(first_shot + s) like the reference.
 * host_columns: [num_outputs][ceil(shots/64)].
 */
zxs_status zxs_sample_given_f(zxs_sampler *s, uint64_t seed, uint64_t first_shot,
                              uint64_t shots, const uint64_t *host_fcols,
                              const double *host_uniforms, uint64_t *host_columns);

/*
 * probability_of_at (sampler.cpp:360-368): outcome[num_outputs] and
 * f_assignment[f_width] as 0/1 bytes. Evaluated on the device.
 */
zxs_status zxs_probability_of_at(zxs_sampler *s, const uint8_t *outcome, uint32_t n_outcome,
                                 const uint8_t *f_assignment, uint32_t n_f, double *out);

/*
 * probability_of (sampler.hpp:64, sampler.cpp:370-429): exact P(outcome),
 * marginalised over every mechanism outcome. Same entropy guard (> 20 bits ->
 * ZXS_INVALID_ARGUMENT), same DFS order and Kahan summation as the reference;
 * each leaf's outcome_probability_given runs on the device.
 */
zxs_status zxs_probability_of(zxs_sampler *s, const uint8_t *outcome, uint32_t n_outcome, double *out);

/*
 * Health check of the compiled tensors (SURVEY finding 3): the reference
 * computes max |Im P| / |P| (phase_terms.cpp:134-141) but never checks it;
 * physically P is real. Evaluates every chain tensor with the exact kernel on
 * `samples` random parameter vectors; out[num_components] receives each
 * component's largest max|Im P| / max|Re P| over its chain tensors.
 */
zxs_status zxs_imag_health(zxs_sampler *s, uint64_t samples, uint64_t seed, double *out);

/* Philox4x32-10 uniform_at (rng.hpp:31-41) evaluated on the device, n draws
   at indices first_index .. first_index+n-1. */
zxs_status zxs_philox_uniform(int device, uint64_t seed, uint32_t stream, uint64_t first_index,
                              uint64_t n, double *host_out);

/* Diagnostic (host only, no GPU needed): the compact word streams the
   large-chi path (heavy_kernel) would evaluate for `desc`, components with
   >= min_factors factors. out[cap] receives, in u32 words: {n_words, n_chunks,
   n_tensor_bounds, zero_row, n_comps, n_components, 0, 0}, then per heavy
   component {ci, n_out, upos_base, out_begin, first_tensor}, the per-component
   heavy flags, the tensor -> first-chunk bounds, per chunk {word_begin,
   n_words, n_terms, 0}, and the words. *needed = total words (out may be NULL
   to query). */
zxs_status zxs_debug_heavy_layout(const zxs_model_desc *desc, uint64_t min_factors, uint32_t *out, uint64_t cap,
                                  uint64_t *needed);

/* Diagnostic (host only): the record streams of the integer monomial path
   (zxs_mono.cuh) for components with >= min_factors factors. out receives
   {n_words, n_chunks, n_tensor_bounds, n_dict, n_comps, n_components, 0, 0},
   per mono component {ci, n_out, upos_base, out_begin, first_tensor}, the
   per-component flags, tensor -> first-chunk bounds, chunks {word_begin,
   n_words, n_terms, 0}, the form dictionary (4 words per entry), the words. */
zxs_status zxs_debug_mono_layout(const zxs_model_desc *desc, uint64_t min_factors, uint32_t *out, uint64_t cap,
                                 uint64_t *needed);

/* Diagnostic: Philox4x32-10 blocks/s of this library's draw code (the shot
   kernel's Philox and filter compare, same launch shape, no memory traffic)
   on `device` -- the same-op-mix roofline of the error draw. */
zxs_status zxs_measure_philox_peak(int device, double *blocks_per_s);

/* Diagnostic: FP64 ops/s (DMUL + DADD, no FMA contraction, the exact
   contraction's op mix) of a register-resident kernel on `device` -- the
   roofline denominator of heavy_kernel. */
zxs_status zxs_measure_fp64_peak(int device, double *ops_per_s);

/* Diagnostic: shared-memory bytes/s of conflict-free 32-bit loads XORed into
   registers (mono_kernel's selector op mix) on `device` -- the roofline
   denominator of mono_kernel. */
zxs_status zxs_measure_smem_peak(int device, double *bytes_per_s);

#ifdef __cplusplus
}
#endif

#endif /* ZXS_B200_H_ */
