/*
 * oracle/zxs_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of
 * the reference's shot-sampling hot path over the flattened model arrays
 * (zxs_model_desc, include/zxs_b200.h). It is the checker, never the thing
 * measured or shipped: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may call it.
 *
 * Pinned against the reference library itself (oracle/_ref/libzxsim_ref.so,
 * the unmodified proj/src compiled in place) and the Random123 Philox KATs by
 * tests/test_oracle.py. Compiled with -ffp-contract=off so every complex
 * product is rounded like the reference's x86-64 build (no FMA).
 *
 * Each function cites the reference code it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "zxs_b200.h"

/* ---- Philox4x32-10 (proj/include/zxsim/rng.hpp:25-71) ---------------- */
void zo_philox_block(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int i = 0; i < 10; i++) { /* rng.hpp:62-66 */
        uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0; /* rng.hpp:49-54 */
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    memcpy(out, c, sizeof(c));
}

/* Philox(seed, stream).uniform_at(index)  (rng.hpp:27-41) */
double zo_uniform_at(uint64_t seed, uint32_t stream, uint64_t index) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32) ^ stream};
    uint32_t ctr[4] = {(uint32_t)index, (uint32_t)(index >> 32), 0x9e3779b9u, 0u};
    uint32_t r[4];
    zo_philox_block(ctr, key, r);
    uint64_t a = ((uint64_t)r[0] << 32) | r[1];
    return (double)(a >> 11) * 0x1.0p-53;
}

static inline int getbit(const uint64_t *col, uint64_t s) { return (int)((col[s >> 6] >> (s & 63)) & 1u); }
static inline void flipbit(uint64_t *col, uint64_t s) { col[s >> 6] ^= (uint64_t)1 << (s & 63); }

/* sample_error_batch (proj/src/sampler.cpp:257-304).
   fcols: [f_width][words], words = ceil(shots/64). */
void zo_sample_error_batch(const zxs_model_desc *d, uint64_t seed, uint64_t first_shot, uint64_t shots,
                           uint64_t *fcols) {
    const uint64_t words = (shots + 63) / 64;
    memset(fcols, 0, (size_t)d->f_width * words * 8);
    for (uint32_t i = 0; i < d->num_base_offset; i++) { /* 261-264 */
        uint64_t *col = fcols + (size_t)d->base_offset[i] * words;
        for (uint64_t w = 0; w < words; w++) col[w] = ~(uint64_t)0;
    }
    for (uint32_t m = 0; m < d->num_mechanisms; m++) {
        const uint32_t v0 = d->mech_vec_begin[m], nv = d->mech_vec_begin[m + 1] - v0;
        if (nv == 1) { /* single: 269-280 */
            const double p = d->mech_probability[m];
            for (uint64_t s = 0; s < shots; s++) {
                if (zo_uniform_at(seed, m, first_shot + s) < p) {
                    for (uint32_t b = d->vec_bit_begin[v0]; b < d->vec_bit_begin[v0 + 1]; b++) {
                        flipbit(fcols + (size_t)d->vec_bits[b] * words, s);
                    }
                }
            }
        } else if (nv > 1) { /* joint: inverse CDF, 281-302 */
            const uint32_t t0 = d->mech_table_begin[m], tn = d->mech_table_begin[m + 1] - t0;
            for (uint64_t s = 0; s < shots; s++) {
                const double u = zo_uniform_at(seed, m, first_shot + s);
                double acc = 0.0;
                uint32_t outcome = 0;
                for (uint32_t o = 0; o < tn; o++) {
                    acc += d->table[t0 + o];
                    if (u < acc) {
                        outcome = o;
                        break;
                    }
                }
                for (uint32_t b = 0; b < nv; b++) {
                    if ((outcome >> b) & 1u) {
                        for (uint32_t i = d->vec_bit_begin[v0 + b]; i < d->vec_bit_begin[v0 + b + 1]; i++) {
                            flipbit(fcols + (size_t)d->vec_bits[i] * words, s);
                        }
                    }
                }
            }
        }
    }
    if (shots & 63) { /* keep tail bits zero like a fresh ParamBatch */
        const uint64_t mask = ((uint64_t)1 << (shots & 63)) - 1;
        for (uint32_t f = 0; f < d->f_width; f++) fcols[(size_t)f * words + words - 1] &= mask;
    }
}

/* eval_batch (proj/src/phase_terms.cpp:90-144) on tensor t.
   params: [ncols][words]; values[shots]; returns max |Im|/|P|. */
double zo_eval_batch(const zxs_model_desc *d, uint32_t t, const uint64_t *params, uint32_t ncols, uint64_t shots,
                     double *values) {
    (void)ncols;
    const uint64_t words = (shots + 63) / 64;
    double *acc = calloc(2 * (shots ? shots : 1), sizeof(double));
    uint64_t *aw = malloc(8 * (words ? words : 1)), *bw = malloc(8 * (words ? words : 1));
    for (uint64_t term = d->tensor_term_begin[t]; term < d->tensor_term_begin[t + 1]; term++) {
        for (uint64_t s = 0; s < shots; s++) {
            double re = d->term_c[2 * term], im = d->term_c[2 * term + 1]; /* prod = c (106) */
            for (uint64_t k = d->term_factor_begin[term]; k < d->term_factor_begin[term + 1]; k++) {
                int a = 0, b = 0;
                for (uint64_t i = d->factor_u_begin[k]; i < d->factor_u_begin[k + 1]; i++)
                    a ^= getbit(params + (size_t)d->factor_u_bits[i] * words, s);
                for (uint64_t i = d->factor_v_begin[k]; i < d->factor_v_begin[k + 1]; i++)
                    b ^= getbit(params + (size_t)d->factor_v_bits[i] * words, s);
                const double *h = d->h_table + 8 * (size_t)d->factor_table[k] + 2 * ((a << 1) | b);
                /* prod *= h (122-127): (re + i im)(hr + i hi), products rounded separately */
                const double nr = re * h[0] - im * h[1];
                const double ni = re * h[1] + im * h[0];
                re = nr;
                im = ni;
            }
            acc[2 * s] += re; /* acc += prod (129-131) */
            acc[2 * s + 1] += im;
        }
    }
    (void)aw;
    (void)bw;
    double max_imag = 0.0;
    for (uint64_t s = 0; s < shots; s++) { /* 134-141 */
        values[s] = acc[2 * s];
        const double mag = hypot(acc[2 * s], acc[2 * s + 1]);
        if (mag > 0) {
            const double r = fabs(acc[2 * s + 1]) / (mag + 1e-300);
            if (r > max_imag) max_imag = r;
        }
    }
    free(acc);
    free(aw);
    free(bw);
    return max_imag;
}

/* run_batch (proj/src/sampler.cpp:51-102) over [first_shot, first_shot+shots)
   with one parameter batch per component (param width f_width + n_out).
   fcols_in (nullable) injects the f-columns, uniforms (nullable) the
   autoregressive draws [position][shots]. out: [num_outputs][words].
   Returns 0, or 2 on the reference's ratio breakdown (sampler.cpp:86-89). */
int zo_sample(const zxs_model_desc *d, uint64_t seed, uint64_t first_shot, uint64_t shots,
              const uint64_t *fcols_in, const double *uniforms, uint64_t *out) {
    const uint64_t words = (shots + 63) / 64;
    memset(out, 0, (size_t)d->num_outputs * words * 8);
    if (!shots) return 0;
    uint32_t max_out = 0;
    for (uint32_t c = 0; c < d->num_components; c++) {
        uint32_t n = d->comp_out_begin[c + 1] - d->comp_out_begin[c];
        if (n > max_out) max_out = n;
    }
    const uint32_t W = d->f_width + max_out;
    uint64_t *batch = calloc((size_t)(W ? W : 1) * words, 8);
    if (fcols_in) {
        memcpy(batch, fcols_in, (size_t)d->f_width * words * 8);
    } else {
        zo_sample_error_batch(d, seed, first_shot, shots, batch);
    }
    for (uint32_t i = 0; i < d->num_direct; i++) { /* 59-70 */
        uint64_t *dst = out + (size_t)d->direct_output[i] * words;
        for (uint64_t w = 0; w < words; w++) {
            uint64_t acc = d->direct_flip_const[i] ? ~(uint64_t)0 : 0;
            for (uint32_t b = d->direct_bit_begin[i]; b < d->direct_bit_begin[i + 1]; b++)
                acc ^= batch[(size_t)d->direct_bits[b] * words + w];
            dst[w] = acc;
        }
    }
    double *prev = malloc(8 * shots), *cur = malloc(8 * shots);
    int status = 0;
    uint32_t upos = 0;
    for (uint32_t ci = 0; ci < d->num_components && !status; ci++) { /* 73-101 */
        const uint32_t ob = d->comp_out_begin[ci], n = d->comp_out_begin[ci + 1] - ob;
        const uint32_t tb = d->comp_tensor_begin[ci];
        memset(batch + (size_t)d->f_width * words, 0, (size_t)max_out * words * 8); /* 75-78 */
        zo_eval_batch(d, tb, batch, W, shots, prev);
        for (uint32_t pos = 0; pos < n && !status; pos++, upos++) {
            zo_eval_batch(d, tb + 1 + pos, batch, W, shots, cur);
            const uint32_t stream = 0x80000000u ^ (ci << 12) ^ pos; /* 37-39 */
            uint64_t *dst = out + (size_t)d->comp_outputs[ob + pos] * words;
            for (uint64_t s = 0; s < shots; s++) {
                double ratio = cur[s] / prev[s];
                if (!(ratio > -1e-6 && ratio < 1.0 + 1e-6)) { /* 85-89 */
                    status = 2;
                    break;
                }
                ratio = (0.0 < ratio) ? ratio : 0.0; /* std::max(0.0, ratio) */
                ratio = (ratio < 1.0) ? ratio : 1.0; /* std::min(1.0, ratio) */
                const double u = uniforms ? uniforms[(size_t)upos * shots + s]
                                          : zo_uniform_at(seed, stream, first_shot + s);
                if (!(u < ratio)) { /* 91-96 */
                    flipbit(batch + (size_t)(d->f_width + pos) * words, s);
                    flipbit(dst, s);
                    prev[s] -= cur[s];
                } else {
                    prev[s] = cur[s];
                }
            }
        }
    }
    if (shots & 63) { /* 201-208 */
        const uint64_t mask = ((uint64_t)1 << (shots & 63)) - 1;
        for (uint32_t o = 0; o < d->num_outputs; o++) out[(size_t)o * words + words - 1] &= mask;
    }
    free(prev);
    free(cur);
    free(batch);
    return status;
}

/* ---- encode_shots (proj/src/encode.cpp:22-48) ------------------------- */
/* cols: [num_outputs][ceil(shots/64)]. Output range clamped as encode.cpp:23-25.
   format 0 = ascii01 (width chars + '\n' per shot, encode.cpp:27-35),
   1 = b8 (ceil(width/8) bytes per shot, bit b%8 of byte b/8, encode.cpp:37-46).
   Returns bytes written, or -1 if cap is too small / arguments invalid. */
long long zo_encode(const uint64_t *cols, uint32_t num_outputs, uint64_t shots, uint32_t first_output,
                    uint32_t output_count, int format, uint8_t *out, uint64_t cap) {
    if (first_output > num_outputs) return -1;
    uint32_t rest = num_outputs - first_output;
    uint32_t last = first_output + (output_count < rest ? output_count : rest);
    if (last > num_outputs) last = num_outputs;
    uint32_t width = last - first_output;
    uint64_t words = (shots + 63) / 64;
    uint64_t rb = format == 0 ? (uint64_t)width + 1 : ((uint64_t)width + 7) / 8;
    if (shots * rb > cap) return -1;
    memset(out, 0, shots * rb);
    for (uint64_t s = 0; s < shots; s++) {
        uint8_t *row = out + s * rb;
        for (uint32_t b = 0; b < width; b++) {
            int bit = (int)((cols[(uint64_t)(first_output + b) * words + (s >> 6)] >> (s & 63)) & 1u);
            if (format == 0) {
                row[b] = (uint8_t)(bit ? '1' : '0');
            } else if (bit) {
                row[b / 8] |= (uint8_t)(1u << (b % 8));
            }
        }
        if (format == 0) row[width] = '\n';
    }
    return (long long)(shots * rb);
}
