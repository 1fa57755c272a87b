// zxs_heavy.cuh — autoregressive chain of large-chi components.
//
// Components whose chain tensors hold many factors (the cultivation proxy:
// chi = 46,656 terms, ~3.1 M factors per tensor) are evaluated here instead of
// in the per-warp loop of shot_kernel. The arithmetic is the reference's
// eval_batch (phase_terms.cpp:90-144) in the reference's order, so results
// stay bit-identical; what changes is the data movement:
//
//  * Each tensor is re-encoded once (host) as a compact word stream: per term
//    {n_factors, c.re, c.im}, per factor a 32-bit header {table, |u|, |v|}
//    followed by the selector indices packed four per word (~12 B/factor
//    instead of ~30 B), cut into <= kChunkWords chunks on term boundaries.
//  * A CTA of kHeavyWarps warps owns 32 * kHS shots per warp (4096 shots per
//    CTA). Chunks are streamed HBM/L2 -> shared memory with cp.async.bulk
//    (1-D TMA) into two mbarrier-tracked buffers: the next chunk lands while
//    the current one is evaluated, and every fetched byte serves 4096 shots.
//  * Every warp walks the chunk with warp-uniform (broadcast) shared loads.
//    Parameters are held per lane as "byte planes": plane[p][lane] bit s is
//    parameter p of the lane's shot in sub-tile s, so one byte load + XOR per
//    selector yields the parities of all kHS = 8 shots of the lane, and the
//    h-table offset of shot s is ((a << 5 | b << 4) >> s) & 0x30.
#pragma once

#include "zxs_kernels.cuh"

namespace zxs_dev {

constexpr int kHS = 8;              // 32-shot words per warp (shots per lane)
constexpr int kHeavyWarps = 16;     // warps per CTA
constexpr uint32_t kChunkWords = 8192;  // 32 KiB per chunk buffer
constexpr int kMaxHeavyComps = 8;

struct HeavyComp {
    uint32_t ci;           // component index (Philox AR stream, sampler.cpp:37-39)
    uint32_t n_out;        // chain length
    uint32_t upos_base;    // first chain position of this component in the global position order
    uint32_t out_begin;    // into comp_outputs
    uint32_t first_tensor; // index into tensor_chunk_begin (chain order: norm, marg0, ...)
    uint32_t nf;           // monomial path: local f parameters (local nf + j = sampled bit j)
    uint32_t pmap_begin;   // monomial path: MonoArgs::param_map[pmap_begin + local] = raw parameter
};

struct HeavyArgs {
    uint64_t seed, first_shot, shots, n_cta_tiles;
    uint32_t k0_round[10];
    uint32_t f_width, col_words;    // col_words = f_width + max heavy chain length
    const uint32_t *fcols;          // [f_width][fcols_ld32] from shot_kernel
    uint64_t fcols_ld32;
    uint32_t *out32;                // [num_outputs][out_ld32] (nullable)
    uint64_t out_ld32;
    unsigned long long *counts;     // (nullable)
    const double *uniforms;         // injected AR uniforms (nullable)
    uint64_t uniforms_ld;
    unsigned long long *err;
    const uint32_t *words;          // chunk streams
    const uint4 *chunks;            // {word_begin, n_words (multiple of 4), n_terms, 0}
    const uint32_t *tensor_chunk_begin;
    uint32_t total_chunks;
    const uint32_t *comp_outputs;
    const double2 *htab;
    uint32_t n_tables;
    uint32_t n_comps;
    HeavyComp comps[kMaxHeavyComps];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "ZXS_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra ZXS_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D TMA: global -> shared, completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Issues the copy of chunk-sequence use `u` into buffer u & 1.
__device__ __forceinline__ void heavy_issue(const HeavyArgs &h, uint64_t u, uint32_t *buf0, uint64_t *bars) {
    const uint4 c = h.chunks[u % h.total_chunks];
    const uint32_t b = uint32_t(u & 1);
    mbar_expect_tx(&bars[b], c.y * 4u);
    bulk_g2s(buf0 + b * kChunkWords, h.words + c.x, c.y * 4u, &bars[b]);
}

// XOR of the lane's byte planes over `groups` groups of four selector byte
// offsets (padding selectors point at an all-zero plane row): bit s of the
// result is the selector parity of the lane's shot s.
__device__ __forceinline__ uint32_t heavy_parity(const uint4 *w4, uint32_t &q, uint32_t groups,
                                                 const uint8_t *planes) {
    uint32_t acc = 0;
    for (uint32_t g = 0; g < groups; g++) {
        const uint4 o = w4[q++];
        acc ^= uint32_t(*reinterpret_cast<const uint16_t *>(planes + o.x)) ^
               uint32_t(*reinterpret_cast<const uint16_t *>(planes + o.y));
        acc ^= uint32_t(*reinterpret_cast<const uint16_t *>(planes + o.z)) ^
               uint32_t(*reinterpret_cast<const uint16_t *>(planes + o.w));
    }
    return acc;
}

// Spreads the low 8 bits of v to the even bit positions 0, 2, ..., 14.
__device__ __forceinline__ uint32_t spread8(uint32_t v) {
    v = (v | (v << 4)) & 0x0F0Fu;
    v = (v | (v << 2)) & 0x3333u;
    return (v | (v << 1)) & 0x5555u;
}

__global__ void __launch_bounds__(kHeavyWarps * 32, 1) heavy_kernel(const __grid_constant__ HeavyArgs h) {
    extern __shared__ __align__(128) uint8_t hsm[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(hsm);
    uint32_t *buf0 = reinterpret_cast<uint32_t *>(hsm + 128);
    double2 *htab = reinterpret_cast<double2 *>(hsm + 128 + 2 * kChunkWords * 4);
    uint32_t *colsw = reinterpret_cast<uint32_t *>(htab + 4 * h.n_tables);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    // [param][lane] 16-bit planes: bit 2s = parameter of the lane's shot in sub-tile s
    uint16_t *planes = reinterpret_cast<uint16_t *>(colsw) + warp * h.col_words * 32;
    const uint8_t *my_planes = reinterpret_cast<const uint8_t *>(planes + lane);

    const uint64_t my_tiles = blockIdx.x < h.n_cta_tiles ? (h.n_cta_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const uint64_t total_uses = my_tiles * h.total_chunks;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (uint32_t i = threadIdx.x; i < 4 * h.n_tables; i += blockDim.x) htab[i] = h.htab[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint64_t u = 0; u < 2 && u < total_uses; u++) heavy_issue(h, u, buf0, bars);
    }
    const uint32_t seed_hi = uint32_t(h.seed >> 32);
    const uint32_t k2c = uint32_t(kP1c) ^ h.k0_round[1];
    uint64_t use = 0;

    for (uint64_t ct = blockIdx.x; ct < h.n_cta_tiles; ct += gridDim.x) {
        // first 32-bit word of this warp's shots; shot of (lane, s) = (w0 + s) * 32 + lane.
        // Per-shot Philox state is rebuilt at each autoregressive draw rather
        // than kept live across the factor loop (register pressure).
        const uint64_t w0 = (ct * kHeavyWarps + warp) * kHS;
        for (uint32_t p = 0; p < h.col_words; p++) {  // byte planes of the lane's 8 shots
            uint32_t byte = 0;
            if (p < h.f_width) {
#pragma unroll
                for (int s = 0; s < kHS; s++) {
                    const uint32_t col = (w0 + s < h.fcols_ld32) ? h.fcols[p * h.fcols_ld32 + w0 + s] : 0u;
                    byte |= ((col >> lane) & 1u) << s;
                }
            }
            planes[p * 32 + lane] = uint16_t(spread8(byte));
        }
        __syncwarp();

        for (uint32_t hc = 0; hc < h.n_comps; hc++) {
            const HeavyComp cd = h.comps[hc];
            double prev[kHS];
            for (uint32_t pos = 0; pos <= cd.n_out; pos++) {  // pos 0: normalization, pos j+1: marginal j
                const uint32_t t = cd.first_tensor + pos;
                double2 acc[kHS];
#pragma unroll
                for (int s = 0; s < kHS; s++) acc[s] = make_double2(0.0, 0.0);
                for (uint32_t c = h.tensor_chunk_begin[t]; c < h.tensor_chunk_begin[t + 1]; c++, use++) {
                    const uint32_t b = uint32_t(use & 1);
                    mbar_wait(&bars[b], uint32_t((use >> 1) & 1));
                    const uint32_t *w = buf0 + b * kChunkWords;
                    const uint32_t nterms = h.chunks[c].z;
                    uint32_t p = 0;
                    const uint4 *w4 = reinterpret_cast<const uint4 *>(w);
                    uint32_t q = 0;
                    for (uint32_t tt = 0; tt < nterms; tt++) {
                        const uint4 t0 = w4[q], t1 = w4[q + 1];  // {nfac, re.lo, re.hi, im.lo}, {im.hi, -, -, -}
                        q += 2;
                        const uint32_t nfac = t0.x;
                        const double2 cterm = make_double2(__hiloint2double(int(t0.z), int(t0.y)),
                                                           __hiloint2double(int(t1.x), int(t0.w)));
                        double2 prod[kHS];
#pragma unroll
                        for (int s = 0; s < kHS; s++) prod[s] = cterm;
                        for (uint32_t k = 0; k < nfac; k++) {
                            const uint32_t hdr = w4[q++].x;  // table | u groups << 8 | v groups << 16
                            const uint32_t av = heavy_parity(w4, q, (hdr >> 8) & 0xffu, my_planes);
                            const uint32_t bv = heavy_parity(w4, q, (hdr >> 16) & 0xffu, my_planes);
                            const char *ht = reinterpret_cast<const char *>(htab + 4 * (hdr & 0xffu));
                            // shot s: a at bit 2s+1, b at bit 2s -> h index (a<<1|b) * 16 bytes
                            const uint32_t z = (av << 1) | bv;
#pragma unroll
                            for (int s = 0; s < kHS; s++) {
                                const uint32_t off = (2 * s >= 4) ? ((z >> (2 * s - 4)) & 0x30u) : ((z << (4 - 2 * s)) & 0x30u);
                                const double2 hv = *reinterpret_cast<const double2 *>(ht + off);
                                prod[s] = cmul_rn(prod[s], hv);
                            }
                        }
#pragma unroll
                        for (int s = 0; s < kHS; s++) acc[s] = cadd_rn(acc[s], prod[s]);
                    }
                    __syncthreads();  // buffer b fully consumed by every warp
                    if (threadIdx.x == 0 && use + 2 < total_uses) heavy_issue(h, use + 2, buf0, bars);
                }
                if (pos == 0) {
#pragma unroll
                    for (int s = 0; s < kHS; s++) prev[s] = acc[s].x;
                    continue;
                }
                // autoregressive draw of output pos-1 (sampler.cpp:84-99)
                const uint32_t j = pos - 1;
                uint32_t rhi[kHS], rlo[kHS];
                if (!h.uniforms) {
                    PhiloxPre pre[kHS];
#pragma unroll
                    for (int s = 0; s < kHS; s++) {
                        const uint64_t shot = h.first_shot + (w0 + s) * 32 + lane;
                        pre[s] = philox_pre(uint32_t(shot), uint32_t(shot >> 32), h.k0_round[0]);
                    }
                    const uint32_t stream = 0x80000000u ^ (cd.ci << 12) ^ j;
                    philox_tail<kHS>(pre, seed_hi ^ stream, h.k0_round, k2c, h.k0_round[9], rhi, rlo);
                }
                uint32_t word[kHS];
#pragma unroll
                for (int s = 0; s < kHS; s++) {
                    const uint64_t local_s = (w0 + s) * 32 + lane;
                    const bool valid = local_s < h.shots;
                    const double cur = acc[s].x;
                    const double ratio = __ddiv_rn(cur, prev[s]);
                    if (!(ratio > -1e-6 && ratio < 1.0 + 1e-6) && valid) report_ratio_error(h.err, h.first_shot + local_s);
                    double cl = (0.0 < ratio) ? ratio : 0.0;
                    cl = (cl < 1.0) ? cl : 1.0;
                    const double u = h.uniforms ? (valid ? h.uniforms[(cd.upos_base + j) * h.uniforms_ld + local_s] : 0.0)
                                                : philox_uniform((uint64_t(rhi[s]) << 32) | rlo[s]);
                    const bool bit = !(u < cl);
                    prev[s] = bit ? __dsub_rn(prev[s], cur) : cur;
                    word[s] = __ballot_sync(kFull, bit && valid);
                }
                uint32_t byte = 0;
#pragma unroll
                for (int s = 0; s < kHS; s++) byte |= ((word[s] >> lane) & 1u) << s;
                planes[(h.f_width + j) * 32 + lane] = uint16_t(spread8(byte));
                if (lane == 0) {
                    const uint32_t o = h.comp_outputs[cd.out_begin + j];
                    unsigned long long ones = 0;
#pragma unroll
                    for (int s = 0; s < kHS; s++) {
                        if (h.out32 && w0 + s < min(h.out_ld32, 2 * ((h.shots + 63) / 64))) {
                            h.out32[o * h.out_ld32 + w0 + s] = word[s];
                        }
                        ones += __popc(word[s]);
                    }
                    if (h.counts && ones) atomicAdd(&h.counts[o], ones);
                }
                __syncwarp();
            }
            // reset this component's sampled-bit columns for the next component
            for (uint32_t j = 0; j < cd.n_out; j++) planes[(h.f_width + j) * 32 + lane] = 0;
            __syncwarp();
        }
    }
}

}  // namespace zxs_dev
