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
//  * Every warp walks the chunk with warp-uniform (broadcast) shared loads;
//    selector parities are XORs of bit-sliced parameter columns held in
//    shared memory, kHS 32-shot words per parameter read as uint4 vectors.
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

// XORs `count` selector columns from the packed byte stream into acc.
__device__ __forceinline__ void heavy_selectors(const uint32_t *w, uint32_t &p, uint32_t &sw, uint32_t &nb,
                                                uint32_t count, const uint4 *cols, uint32_t (&acc)[kHS]) {
    for (uint32_t i = 0; i < count; i++) {
        if (nb == 0) {
            sw = w[p++];
            nb = 4;
        }
        const uint32_t sel = sw & 0xffu;
        sw >>= 8;
        nb--;
        const uint4 *c = cols + sel * (kHS / 4);
#pragma unroll
        for (int q = 0; q < kHS / 4; q++) {
            const uint4 v = c[q];
            acc[4 * q + 0] ^= v.x;
            acc[4 * q + 1] ^= v.y;
            acc[4 * q + 2] ^= v.z;
            acc[4 * q + 3] ^= v.w;
        }
    }
}

__global__ void __launch_bounds__(kHeavyWarps * 32, 1) heavy_kernel(const __grid_constant__ HeavyArgs h) {
    extern __shared__ __align__(128) uint8_t hsm[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(hsm);
    uint32_t *buf0 = reinterpret_cast<uint32_t *>(hsm + 128);
    double2 *htab = reinterpret_cast<double2 *>(hsm + 128 + 2 * kChunkWords * 4);
    uint32_t *colsw = reinterpret_cast<uint32_t *>(htab + 4 * h.n_tables);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t *cols = colsw + warp * h.col_words * kHS;  // [param][kHS]
    const uint4 *cols4 = reinterpret_cast<const uint4 *>(cols);

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
        const uint64_t w0 = (ct * kHeavyWarps + warp) * kHS;  // first 32-bit word of this warp's shots
        uint64_t local[kHS];
        uint32_t vmask[kHS];
        PhiloxPre pre[kHS];
#pragma unroll
        for (int s = 0; s < kHS; s++) {
            local[s] = (w0 + s) * 32 + lane;
            vmask[s] = __ballot_sync(kFull, local[s] < h.shots);
            const uint64_t shot = h.first_shot + local[s];
            pre[s] = philox_pre(uint32_t(shot), uint32_t(shot >> 32), h.k0_round[0]);
        }
        for (uint32_t i = lane; i < h.col_words * kHS; i += 32) {
            const uint32_t p = i / kHS, s = i % kHS;
            cols[i] = (p < h.f_width && w0 + s < h.fcols_ld32) ? h.fcols[p * h.fcols_ld32 + w0 + s] : 0u;
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
                    for (uint32_t tt = 0; tt < nterms; tt++) {
                        const uint32_t nfac = w[p];
                        const double2 cterm = make_double2(__hiloint2double(int(w[p + 2]), int(w[p + 1])),
                                                           __hiloint2double(int(w[p + 4]), int(w[p + 3])));
                        p += 5;
                        double2 prod[kHS];
#pragma unroll
                        for (int s = 0; s < kHS; s++) prod[s] = cterm;
                        for (uint32_t k = 0; k < nfac; k++) {
                            const uint32_t hdr = w[p++];
                            uint32_t aw[kHS] = {}, bw[kHS] = {};
                            uint32_t sw = 0, nb = 0;
                            heavy_selectors(w, p, sw, nb, (hdr >> 8) & 0xffu, cols4, aw);
                            heavy_selectors(w, p, sw, nb, (hdr >> 16) & 0xffu, cols4, bw);
                            const double2 *ht = htab + 4 * (hdr & 0xffu);
#pragma unroll
                            for (int s = 0; s < kHS; s++) {
                                const uint32_t idx = (((aw[s] >> lane) & 1u) << 1) | ((bw[s] >> lane) & 1u);
                                prod[s] = cmul_rn(prod[s], ht[idx]);
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
                    const uint32_t stream = 0x80000000u ^ (cd.ci << 12) ^ j;
                    philox_tail<kHS>(pre, seed_hi ^ stream, h.k0_round, k2c, h.k0_round[9], rhi, rlo);
                }
                uint32_t word[kHS];
#pragma unroll
                for (int s = 0; s < kHS; s++) {
                    const bool valid = local[s] < h.shots;
                    const double cur = acc[s].x;
                    const double ratio = __ddiv_rn(cur, prev[s]);
                    if (!(ratio > -1e-6 && ratio < 1.0 + 1e-6) && valid) report_ratio_error(h.err, h.first_shot + local[s]);
                    double cl = (0.0 < ratio) ? ratio : 0.0;
                    cl = (cl < 1.0) ? cl : 1.0;
                    const double u = h.uniforms ? (valid ? h.uniforms[(cd.upos_base + j) * h.uniforms_ld + local[s]] : 0.0)
                                                : philox_uniform((uint64_t(rhi[s]) << 32) | rlo[s]);
                    const bool bit = !(u < cl);
                    prev[s] = bit ? __dsub_rn(prev[s], cur) : cur;
                    word[s] = __ballot_sync(kFull, bit) & vmask[s];
                }
                if (lane == 0) {
                    const uint32_t o = h.comp_outputs[cd.out_begin + j];
                    unsigned long long ones = 0;
#pragma unroll
                    for (int s = 0; s < kHS; s++) {
                        cols[(h.f_width + j) * kHS + s] = word[s];
                        if (h.out32 && w0 + s < h.out_ld32) h.out32[o * h.out_ld32 + w0 + s] = word[s];
                        ones += __popc(word[s]);
                    }
                    if (h.counts && ones) atomicAdd(&h.counts[o], ones);
                }
                __syncwarp();
            }
            // reset this component's sampled-bit columns for the next component
            for (uint32_t i = lane; i < cd.n_out * kHS; i += 32) cols[h.f_width * kHS + i] = 0u;
            __syncwarp();
        }
    }
}

}  // namespace zxs_dev
