// zxs_kernels.cuh — the fused per-shot kernel and the verification kernels.
//
// One launch of shot_kernel runs the whole per-shot pipeline of the
// reference's run_batch (proj/src/sampler.cpp:51-102) for a range of shots:
//   (1) Philox4x32-10 draw of every error mechanism (sampler.cpp:266-303),
//   (2) f = T.e accumulated as XOR masks in the lane's f registers,
//   (3) warp transpose into 32-shot bit-sliced columns (ParamBatch layout),
//   (4) direct-output parities (sampler.cpp:59-70),
//   (5) the autoregressive chain per component with eval_batch
//       (phase_terms.cpp:90-144) evaluated in place (sampler.cpp:72-101),
//   (6) packed 32-shot output words and/or per-output flip counts.
// A warp owns a 32-shot tile; warps stride over tiles (persistent grid).
#pragma once

#include "zxs_device.cuh"

namespace zxs_dev {

struct LaunchArgs {
    DevModel m;
    const uint4 *mechs;      // [num_mech] {stream, entry_begin, entry_end, 0}
    const ulonglong2 *entries; // {lim, flip}
    uint64_t seed, first_shot, shots, n_tiles;
    uint32_t *out32;         // [num_outputs][ld32] (nullable)
    uint64_t ld32;
    unsigned long long *counts; // [num_outputs] (nullable)
    uint32_t *fcols_out;     // error-batch seam: [f_width][fcols_ld32] (nullable)
    uint64_t fcols_ld32;
    const uint32_t *fcols_in; // injected f: [f_width][fcols_ld32] (nullable)
    const double *uniforms;  // injected AR uniforms: [positions][uniforms_ld] (nullable)
    uint64_t uniforms_ld;
    unsigned long long *err; // [0] = flag, [1] = first failing shot
};

// eval_batch for one 32-shot tile: returns (Re, Im) of
// sum_t c_t prod_k h_tk[(a<<1)|b] for this lane's shot, accumulated in the
// reference's order (terms in order, factors in order, acc starts at 0).
__device__ __forceinline__ double2 eval_tensor(const DevModel &m, uint32_t t,
                                               const uint32_t *cols, uint32_t lane) {
    double2 acc = make_double2(0.0, 0.0);
    const uint32_t t0 = m.tensor_term_begin[t], t1 = m.tensor_term_begin[t + 1];
    for (uint32_t term = t0; term < t1; term++) {
        double2 prod = m.term_c[term];
        const uint32_t k0 = m.term_factor_begin[term], k1 = m.term_factor_begin[term + 1];
        for (uint32_t k = k0; k < k1; k++) {
            const Factor fr = m.factors[k];
            const uint16_t *s = m.selectors + fr.sel;
            uint32_t aw = 0, bw = 0;
            for (uint32_t i = 0; i < fr.nu; i++) aw ^= cols[s[i]];
            for (uint32_t i = 0; i < fr.nv; i++) bw ^= cols[s[fr.nu + i]];
            const uint32_t idx = (((aw >> lane) & 1u) << 1) | ((bw >> lane) & 1u);
            prod = cmul_rn(prod, m.h_table[4 * fr.table + idx]);
        }
        acc = cadd_rn(acc, prod);
    }
    return acc;
}

__device__ __forceinline__ void report_ratio_error(unsigned long long *err, uint64_t shot) {
    atomicOr(&err[0], 1ull);
    atomicMin(&err[1], (unsigned long long)shot);
}

template <int FW>
__global__ void __launch_bounds__(256) shot_kernel(const LaunchArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    const DevModel &m = a.m;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t warps = blockDim.x >> 5;
    unsigned long long *scount = reinterpret_cast<unsigned long long *>(smem);
    uint32_t *cols = smem + 2 * m.num_outputs + warp * m.col_stride;
    if (a.counts) {
        for (uint32_t o = threadIdx.x; o < m.num_outputs; o += blockDim.x) scount[o] = 0;
        __syncthreads();
    }
    const uint32_t seed_lo = uint32_t(a.seed), seed_hi = uint32_t(a.seed >> 32);
    const uint64_t stride = uint64_t(gridDim.x) * warps;

    for (uint64_t tile = uint64_t(blockIdx.x) * warps + warp; tile < a.n_tiles; tile += stride) {
        const uint64_t local = tile * 32 + lane;
        const bool valid = local < a.shots;
        const uint32_t vmask = __ballot_sync(kFull, valid);
        const uint64_t shot = a.first_shot + local;
        const uint32_t idx_lo = uint32_t(shot), idx_hi = uint32_t(shot >> 32);

        // ---- (1)-(3): f configuration as bit-sliced columns
        if (a.fcols_in) {
            for (uint32_t c = lane; c < m.f_width; c += 32) cols[c] = a.fcols_in[c * a.fcols_ld32 + tile];
        } else {
            uint64_t f[FW];
#pragma unroll
            for (int w = 0; w < FW; w++) f[w] = m.base_offset[w];
            for (uint32_t mi = 0; mi < m.num_mech; mi++) {
                const uint4 md = a.mechs[mi];
                const uint64_t r = philox_r01(seed_lo, seed_hi ^ md.x, idx_lo, idx_hi);
                uint32_t flip = kNoFlip;
                for (uint32_t e = md.y; e < md.z; e++) {
                    const ulonglong2 en = a.entries[e];
                    if (r <= en.x) {
                        flip = uint32_t(en.y);
                        break;
                    }
                }
                if (flip != kNoFlip) {
                    const uint64_t *mask = m.flip_mask + size_t(flip) * FW;
#pragma unroll
                    for (int w = 0; w < FW; w++) f[w] ^= mask[w];
                }
            }
#pragma unroll
            for (int w = 0; w < FW; w++) {
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const uint32_t base = uint32_t(w) * 64u + uint32_t(h) * 32u;
                    if (base < m.f_width) {
                        const uint32_t x = h ? uint32_t(f[w] >> 32) : uint32_t(f[w]);
                        cols[base + lane] = warp_transpose32(x, lane);
                    }
                }
            }
        }
        __syncwarp();
        if (a.fcols_out) {
            for (uint32_t c = lane; c < m.f_width; c += 32) a.fcols_out[c * a.fcols_ld32 + tile] = cols[c] & vmask;
            __syncwarp();
            continue;
        }

        // ---- (4): direct outputs, lane-parallel over outputs
        for (uint32_t d = lane; d < m.num_direct; d += 32) {
            const uint32_t od = m.direct_out[d];
            uint32_t w = (od >> 31) ? kFull : 0u;
            for (uint32_t b = m.direct_bit_begin[d]; b < m.direct_bit_begin[d + 1]; b++) w ^= cols[m.direct_bits[b]];
            w &= vmask;
            const uint32_t o = od & 0x7fffffffu;
            if (a.out32) a.out32[o * a.ld32 + tile] = w;
            if (a.counts && w) atomicAdd(&scount[o], (unsigned long long)__popc(w));
        }

        // ---- (5): autoregressive components
        uint32_t upos = 0;
        for (uint32_t ci = 0; ci < m.num_components; ci++) {
            const uint32_t ob = m.comp_out_begin[ci], n = m.comp_out_begin[ci + 1] - ob;
            const uint32_t tb = m.comp_tensor_begin[ci];
            for (uint32_t p = lane; p < n; p += 32) cols[m.f_width + p] = 0u;
            __syncwarp();
            double prev = eval_tensor(m, tb, cols, lane).x;
            for (uint32_t pos = 0; pos < n; pos++, upos++) {
                const double cur = eval_tensor(m, tb + 1 + pos, cols, lane).x;
                const double ratio = __ddiv_rn(cur, prev);
                if (!(ratio > -1e-6 && ratio < 1.0 + 1e-6) && valid) report_ratio_error(a.err, shot);
                double cl = (0.0 < ratio) ? ratio : 0.0;  // std::max(0.0, ratio)
                cl = (cl < 1.0) ? cl : 1.0;               // std::min(1.0, .)
                double u;
                if (a.uniforms) {
                    u = valid ? a.uniforms[upos * a.uniforms_ld + local] : 0.0;
                } else {
                    const uint32_t stream = 0x80000000u ^ (ci << 12) ^ pos;  // sampler.cpp:37-39
                    u = philox_uniform(philox_r01(seed_lo, seed_hi ^ stream, idx_lo, idx_hi));
                }
                const bool bit = !(u < cl);
                prev = bit ? __dsub_rn(prev, cur) : cur;
                const uint32_t word = __ballot_sync(kFull, bit) & vmask;
                if (lane == 0) {
                    cols[m.f_width + pos] = word;
                    const uint32_t o = m.comp_outputs[ob + pos];
                    if (a.out32) a.out32[o * a.ld32 + tile] = word;
                    if (a.counts && word) atomicAdd(&scount[o], (unsigned long long)__popc(word));
                }
                __syncwarp();
            }
        }
    }
    if (a.counts) {
        __syncthreads();
        for (uint32_t o = threadIdx.x; o < m.num_outputs; o += blockDim.x) {
            if (scount[o]) atomicAdd(&a.counts[o], scount[o]);
        }
    }
}

// eval_batch seam (phase_terms.cpp:90-144) over injected parameter columns.
__global__ void __launch_bounds__(256) eval_kernel(DevModel m, uint32_t tensor, const uint32_t *params,
                                                   uint64_t ld32, uint32_t ncols, uint32_t col_stride,
                                                   uint64_t shots, uint64_t n_tiles, double *values,
                                                   unsigned long long *max_imag_bits) {
    extern __shared__ __align__(16) uint32_t smem[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    uint32_t *cols = smem + warp * col_stride;
    for (uint64_t tile = uint64_t(blockIdx.x) * warps + warp; tile < n_tiles;
         tile += uint64_t(gridDim.x) * warps) {
        for (uint32_t c = lane; c < ncols; c += 32) cols[c] = params[c * ld32 + tile];
        __syncwarp();
        const uint64_t local = tile * 32 + lane;
        const double2 acc = eval_tensor(m, tensor, cols, lane);
        if (local < shots) {
            values[local] = acc.x;
            const double mag = hypot(acc.x, acc.y);
            if (mag > 0) {
                const double ratio = fabs(acc.y) / (mag + 1e-300);  // phase_terms.cpp:137-141
                atomicMax(max_imag_bits, (unsigned long long)__double_as_longlong(ratio));
            }
        }
        __syncwarp();
    }
}

__global__ void philox_kernel(uint64_t seed, uint32_t stream, uint64_t first, uint64_t n, double *out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t idx = first + i;
        out[i] = philox_uniform(philox_r01(uint32_t(seed), uint32_t(seed >> 32) ^ stream, uint32_t(idx),
                                           uint32_t(idx >> 32)));
    }
}

}  // namespace zxs_dev
