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
//   (6) packed output words and/or per-output flip counts.
//
// Work decomposition: a warp owns a tile of 64 consecutive shots (one 64-bit
// output word per output); lane l carries shots l and 32 + l (kS = 2), so
// the warp-uniform Philox key schedule of each mechanism is shared by two
// independent Philox chains per lane. Warps stride over tiles (persistent
// grid sized to the SM count).
//
// Mechanism records live in the kernel's parameter space when they fit
// (kParamMechs), so the per-mechanism threshold loads are uniform LDCU
// constant-bank reads and the loop index is the Philox stream (uniform
// datapath for the key schedule); larger models read them from global memory.
#pragma once

#include "zxs_device.cuh"

namespace zxs_dev {

constexpr int kS = 2;                 // shots per lane
constexpr int kTileShots = 32 * kS;   // shots per warp tile = one u64 word
constexpr uint32_t kParamMechs = 1920;

// One mechanism: the first scan entry inline; further entries (joint tables)
// in global memory at ext_begin[m] .. ext_begin[m] + n_extra.
struct __align__(16) MechRec {
    unsigned long long lim0;  // fire/hit iff r01 <= lim0
    uint32_t flip0;           // flip-set id of the first entry, or kNoFlip
    uint32_t n_extra;         // number of further entries
};

template <uint32_t N>
struct MechTable {
    MechRec rec[N];
};
static_assert(kS == 2, "output stores pack two 32-shot words");

struct LaunchArgs {
    DevModel m;
    uint32_t num_mech;             // reference mechanism count (streams 0..num_mech-1)
    const MechRec *mech_global;    // used when num_mech > kParamMechs
    const uint32_t *ext_begin;     // [num_mech]
    const ulonglong2 *ext;         // {lim, flip}
    uint64_t seed, first_shot, shots, n_tiles;
    uint32_t k0_round[10];         // seed_lo + i * 0x9E3779B9: Philox key-0 schedule (rng.hpp:64)
    uint32_t *out32;               // [num_outputs][ld32] (nullable)
    uint64_t ld32;
    unsigned long long *counts;    // [num_outputs] (nullable)
    uint32_t *fcols_out;           // error-batch seam: [f_width][fcols_ld32] (nullable)
    uint64_t fcols_ld32;
    const uint32_t *fcols_in;      // injected f: [f_width][fcols_ld32] (nullable)
    const double *uniforms;        // injected AR uniforms: [positions][uniforms_ld] (nullable)
    uint64_t uniforms_ld;
    unsigned long long *err;       // [0] = flag, [1] = first failing shot
};

// 32x32 -> 64 multiply as one mul.wide.u32 (IMAD.WIDE.U32); written in PTX
// because the C++ form lowers with extra adds of zero high words.
__device__ __forceinline__ void mul_wide(uint32_t a, uint32_t b, uint32_t &lo, uint32_t &hi) {
    asm("{\n\t.reg .b64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}" : "=r"(lo), "=r"(hi) : "r"(a), "r"(b));
}

// S Philox4x32-10 blocks sharing the key (seed_lo, seed_hi ^ stream): the
// reference's Philox(seed, stream).uniform2_at(idx) (rng.hpp:27-38) up to the
// (r0 << 32 | r1) word. Round structure per rng.hpp:44-56. The key-0 schedule
// depends only on the seed and is read from the launch parameters (constant
// bank operands of the LOP3s); the key-1 schedule depends on the stream.
template <int S>
__device__ __forceinline__ void philox_multi(const uint32_t (&k0r)[10], uint32_t k1, const uint32_t (&lo)[S],
                                             const uint32_t (&hi)[S], uint64_t (&r)[S]) {
    uint32_t c0[S], c1[S], c2[S], c3[S];
#pragma unroll
    for (int s = 0; s < S; s++) {
        c0[s] = lo[s];
        c1[s] = hi[s];
        c2[s] = 0x9e3779b9u;
        c3[s] = 0u;
    }
#pragma unroll
    for (int i = 0; i < 10; i++) {
#pragma unroll
        for (int s = 0; s < S; s++) {
            uint32_t h0, l0, h1, l1;
            mul_wide(c0[s], 0xD2511F53u, l0, h0);
            mul_wide(c2[s], 0xCD9E8D57u, l1, h1);
            const uint32_t n0 = h1 ^ c1[s] ^ k0r[i], n2 = h0 ^ c3[s] ^ k1;
            c0[s] = n0;
            c1[s] = l1;
            c2[s] = n2;
            c3[s] = l0;
        }
        k1 += 0xBB67AE85u;
    }
#pragma unroll
    for (int s = 0; s < S; s++) r[s] = (uint64_t(c0[s]) << 32) | c1[s];
}

// eval_batch (phase_terms.cpp:90-144) for the kS 32-shot sub-tiles of a warp
// tile: acc[s] = sum_t c_t prod_k h_tk[(a<<1)|b] for this lane's shot in
// sub-tile s, accumulated in the reference's order (terms in order, factors
// in order, acc starting at 0), every product and sum rounded separately.
__device__ __forceinline__ void eval_tensor(const DevModel &m, uint32_t t, const uint32_t *cols, uint32_t stride,
                                            uint32_t lane, double2 (&acc)[kS]) {
#pragma unroll
    for (int s = 0; s < kS; s++) acc[s] = make_double2(0.0, 0.0);
    const uint32_t t0 = m.tensor_term_begin[t], t1 = m.tensor_term_begin[t + 1];
    for (uint32_t term = t0; term < t1; term++) {
        const double2 c = m.term_c[term];
        double2 prod[kS];
#pragma unroll
        for (int s = 0; s < kS; s++) prod[s] = c;
        const uint32_t k0 = m.term_factor_begin[term], k1 = m.term_factor_begin[term + 1];
        for (uint32_t k = k0; k < k1; k++) {
            const Factor fr = m.factors[k];
            const uint16_t *sel = m.selectors + fr.sel;
            uint32_t aw[kS] = {}, bw[kS] = {};
            for (uint32_t i = 0; i < fr.nu; i++) {
                const uint32_t p = sel[i];
#pragma unroll
                for (int s = 0; s < kS; s++) aw[s] ^= cols[s * stride + p];
            }
            for (uint32_t i = 0; i < fr.nv; i++) {
                const uint32_t p = sel[fr.nu + i];
#pragma unroll
                for (int s = 0; s < kS; s++) bw[s] ^= cols[s * stride + p];
            }
            const double2 *h = m.h_table + 4 * fr.table;
#pragma unroll
            for (int s = 0; s < kS; s++) {
                const uint32_t idx = (((aw[s] >> lane) & 1u) << 1) | ((bw[s] >> lane) & 1u);
                prod[s] = cmul_rn(prod[s], h[idx]);
            }
        }
#pragma unroll
        for (int s = 0; s < kS; s++) acc[s] = cadd_rn(acc[s], prod[s]);
    }
}

__device__ __forceinline__ void report_ratio_error(unsigned long long *err, uint64_t shot) {
    atomicOr(&err[0], 1ull);
    atomicMin(&err[1], (unsigned long long)shot);
}

// Rare path of the mechanism draw: the flip set selected by each of the
// lane's two draws (first entry, then the rest of a joint table in order).
// Kept out of line so the divergent scan does not pull the draw loop's
// counters and Philox keys off the uniform datapath.
__device__ __noinline__ uint2 resolve_flips(uint64_t r0, uint64_t r1, MechRec md, const uint32_t *ext_begin,
                                            const ulonglong2 *ext, uint32_t mi) {
    uint32_t out[kS];
    const uint64_t r[kS] = {r0, r1};
#pragma unroll
    for (int s = 0; s < kS; s++) {
        uint32_t flip = kNoFlip;
        if (r[s] <= md.lim0) {
            flip = md.flip0;
        } else if (md.n_extra) {
            const uint32_t e0 = ext_begin[mi];
            for (uint32_t e = e0; e < e0 + md.n_extra; e++) {
                const ulonglong2 en = ext[e];
                if (r[s] <= en.x) {
                    flip = uint32_t(en.y);
                    break;
                }
            }
        }
        out[s] = flip;
    }
    return make_uint2(out[0], out[1]);
}

template <int FW, bool PARAM_MECHS>
__global__ void __launch_bounds__(128) shot_kernel(const __grid_constant__ LaunchArgs a,
                                                   const __grid_constant__ MechTable<PARAM_MECHS ? kParamMechs : 1> mt) {
    extern __shared__ __align__(16) uint32_t smem[];
    // One warp per CTA: the tile loop depends only on blockIdx, so the
    // compiler can keep loop counters, Philox keys and mechanism records in
    // uniform registers (UR) on the uniform datapath.
    const DevModel &m = a.m;
    const uint32_t lane = threadIdx.x;
    unsigned long long *scount = reinterpret_cast<unsigned long long *>(smem);
    uint32_t *cols = smem + 2 * m.num_outputs;
    if (a.counts) {
        for (uint32_t o = lane; o < m.num_outputs; o += 32) scount[o] = 0;
        __syncwarp();
    }
    const uint32_t seed_hi = uint32_t(a.seed >> 32);

    for (uint64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        uint64_t local[kS], shot[kS];
        uint32_t vmask[kS], idx_lo[kS], idx_hi[kS];
#pragma unroll
        for (int s = 0; s < kS; s++) {
            local[s] = tile * kTileShots + 32 * s + lane;
            vmask[s] = __ballot_sync(kFull, local[s] < a.shots);
            shot[s] = a.first_shot + local[s];
            idx_lo[s] = uint32_t(shot[s]);
            idx_hi[s] = uint32_t(shot[s] >> 32);
        }

        // ---- (1)-(3): f configuration as bit-sliced columns
        if (a.fcols_in) {
            for (uint32_t c = lane; c < m.f_width; c += 32) {
#pragma unroll
                for (int s = 0; s < kS; s++) cols[s * m.col_stride + c] = a.fcols_in[c * a.fcols_ld32 + tile * kS + s];
            }
        } else {
            uint64_t f[kS][FW];
#pragma unroll
            for (int w = 0; w < FW; w++) {
                const uint64_t b = m.base_offset[w];
#pragma unroll
                for (int s = 0; s < kS; s++) f[s][w] = b;
            }
            for (uint32_t mi = 0; mi < a.num_mech; mi++) {
                // No early-out for mechanisms that cannot flip anything: a
                // data-dependent `continue` here moves the key schedule off the
                // uniform datapath. Such records never fire (lim0 = 0, no flip).
                const MechRec md = PARAM_MECHS ? mt.rec[mi] : a.mech_global[mi];
                uint64_t r[kS];
                philox_multi<kS>(a.k0_round, seed_hi ^ mi, idx_lo, idx_hi, r);  // stream = mechanism index
                // Common case: every lane's draw resolves at the first entry with
                // no flip (no error). Anything else goes through one warp-uniform
                // branch, which keeps the loop (and the key schedule) uniform.
                bool busy = false;
#pragma unroll
                for (int s = 0; s < kS; s++) {
                    const bool hit0 = r[s] <= md.lim0;
                    busy |= hit0 ? (md.flip0 != kNoFlip) : (md.n_extra != 0);
                }
                if (__any_sync(kFull, busy)) {
                    const uint2 fl = resolve_flips(r[0], r[1], md, a.ext_begin, a.ext, mi);
                    const uint32_t flip[kS] = {fl.x, fl.y};
#pragma unroll
                    for (int s = 0; s < kS; s++) {
                        if (flip[s] != kNoFlip) {
                            const uint64_t *mask = m.flip_mask + size_t(flip[s]) * FW;
#pragma unroll
                            for (int w = 0; w < FW; w++) f[s][w] ^= mask[w];
                        }
                    }
                }
            }
#pragma unroll
            for (int s = 0; s < kS; s++) {
#pragma unroll
                for (int w = 0; w < FW; w++) {
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const uint32_t base = uint32_t(w) * 64u + uint32_t(h) * 32u;
                        if (base < m.f_width) {
                            const uint32_t x = h ? uint32_t(f[s][w] >> 32) : uint32_t(f[s][w]);
                            cols[s * m.col_stride + base + lane] = warp_transpose32(x, lane);
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (a.fcols_out) {
            for (uint32_t c = lane; c < m.f_width; c += 32) {
#pragma unroll
                for (int s = 0; s < kS; s++) a.fcols_out[c * a.fcols_ld32 + tile * kS + s] = cols[s * m.col_stride + c] & vmask[s];
            }
            __syncwarp();
            continue;
        }

        // ---- (4): direct outputs, lane-parallel over outputs
        for (uint32_t d = lane; d < m.num_direct; d += 32) {
            const uint32_t od = m.direct_out[d];
            uint32_t w[kS];
#pragma unroll
            for (int s = 0; s < kS; s++) w[s] = (od >> 31) ? kFull : 0u;
            for (uint32_t b = m.direct_bit_begin[d]; b < m.direct_bit_begin[d + 1]; b++) {
                const uint32_t fb = m.direct_bits[b];
#pragma unroll
                for (int s = 0; s < kS; s++) w[s] ^= cols[s * m.col_stride + fb];
            }
            const uint32_t o = od & 0x7fffffffu;
#pragma unroll
            for (int s = 0; s < kS; s++) w[s] &= vmask[s];
            if (a.out32) {
                *reinterpret_cast<uint2 *>(a.out32 + o * a.ld32 + tile * kS) = make_uint2(w[0], w[1]);
            }
            if (a.counts && (w[0] | w[1])) atomicAdd(&scount[o], (unsigned long long)(__popc(w[0]) + __popc(w[1])));
        }

        // ---- (5): autoregressive components
        uint32_t upos = 0;
        for (uint32_t ci = 0; ci < m.num_components; ci++) {
            const uint32_t ob = m.comp_out_begin[ci], n = m.comp_out_begin[ci + 1] - ob;
            const uint32_t tb = m.comp_tensor_begin[ci];
            for (uint32_t p = lane; p < n; p += 32) {
#pragma unroll
                for (int s = 0; s < kS; s++) cols[s * m.col_stride + m.f_width + p] = 0u;
            }
            __syncwarp();
            double2 acc[kS];
            double prev[kS];
            eval_tensor(m, tb, cols, m.col_stride, lane, acc);
#pragma unroll
            for (int s = 0; s < kS; s++) prev[s] = acc[s].x;
            for (uint32_t pos = 0; pos < n; pos++, upos++) {
                eval_tensor(m, tb + 1 + pos, cols, m.col_stride, lane, acc);
                uint64_t rr[kS];
                if (!a.uniforms) {
                    const uint32_t stream = 0x80000000u ^ (ci << 12) ^ pos;  // sampler.cpp:37-39
                    philox_multi<kS>(a.k0_round, seed_hi ^ stream, idx_lo, idx_hi, rr);
                }
                uint32_t word[kS];
#pragma unroll
                for (int s = 0; s < kS; s++) {
                    const bool valid = local[s] < a.shots;
                    const double cur = acc[s].x;
                    const double ratio = __ddiv_rn(cur, prev[s]);
                    if (!(ratio > -1e-6 && ratio < 1.0 + 1e-6) && valid) report_ratio_error(a.err, shot[s]);
                    double cl = (0.0 < ratio) ? ratio : 0.0;  // std::max(0.0, ratio)
                    cl = (cl < 1.0) ? cl : 1.0;               // std::min(1.0, .)
                    const double u = a.uniforms ? (valid ? a.uniforms[upos * a.uniforms_ld + local[s]] : 0.0)
                                                : philox_uniform(rr[s]);
                    const bool bit = !(u < cl);
                    prev[s] = bit ? __dsub_rn(prev[s], cur) : cur;
                    word[s] = __ballot_sync(kFull, bit) & vmask[s];
                }
                if (lane == 0) {
#pragma unroll
                    for (int s = 0; s < kS; s++) cols[s * m.col_stride + m.f_width + pos] = word[s];
                    const uint32_t o = m.comp_outputs[ob + pos];
                    if (a.out32) *reinterpret_cast<uint2 *>(a.out32 + o * a.ld32 + tile * kS) = make_uint2(word[0], word[1]);
                    if (a.counts && (word[0] | word[1])) {
                        atomicAdd(&scount[o], (unsigned long long)(__popc(word[0]) + __popc(word[1])));
                    }
                }
                __syncwarp();
            }
        }
    }
    if (a.counts) {
        __syncwarp();
        for (uint32_t o = lane; o < m.num_outputs; o += 32) {
            if (scount[o]) atomicAdd(&a.counts[o], scount[o]);
        }
    }
}

// eval_batch seam (phase_terms.cpp:90-144) over injected parameter columns,
// one 64-shot tile per warp in the same layout as the shot kernel.
__global__ void __launch_bounds__(256) eval_kernel(DevModel m, uint32_t tensor, const uint32_t *params,
                                                   uint64_t ld32, uint32_t ncols, uint32_t stride, uint64_t shots,
                                                   uint64_t n_tiles, double *values,
                                                   unsigned long long *max_imag_bits) {
    extern __shared__ __align__(16) uint32_t smem[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    uint32_t *cols = smem + warp * (kS * stride);
    for (uint64_t tile = uint64_t(blockIdx.x) * warps + warp; tile < n_tiles; tile += uint64_t(gridDim.x) * warps) {
        for (uint32_t c = lane; c < ncols; c += 32) {
#pragma unroll
            for (int s = 0; s < kS; s++) cols[s * stride + c] = params[c * ld32 + tile * kS + s];
        }
        __syncwarp();
        double2 acc[kS];
        eval_tensor(m, tensor, cols, stride, lane, acc);
#pragma unroll
        for (int s = 0; s < kS; s++) {
            const uint64_t local = tile * kTileShots + 32 * s + lane;
            if (local < shots) {
                values[local] = acc[s].x;
                const double mag = hypot(acc[s].x, acc[s].y);
                if (mag > 0) {
                    const double ratio = fabs(acc[s].y) / (mag + 1e-300);  // phase_terms.cpp:137-141
                    atomicMax(max_imag_bits, (unsigned long long)__double_as_longlong(ratio));
                }
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
