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
constexpr uint32_t kParamMechs = 1536;

// Small chain tensors as a uniform program in the kernel parameter space:
// per factor the u / v selectors as 64-bit masks over the parameter columns
// (f bits, then the component's sampled bits), so eval reads descriptors with
// uniform constant-bank loads and walks selector bits on the uniform
// datapath instead of chasing global-memory CSR arrays. Used when every
// light (shot_kernel-evaluated) component fits (f_width + chain <= 64).
constexpr uint32_t kLightTensors = 48, kLightTerms = 160, kLightFactors = 320, kLightTables = 32;
// Tabulated chains: a light component whose parity forms over f are few
// (m_f of them) has its whole autoregressive chain precomputed on the host,
// exactly as the reference evaluates it (eval_batch order, IEEE ratio,
// sampler.cpp:84-99), as a table per chain position indexed by the m_f
// f-form parities and the bits sampled so far: the clamped ratio, NaN where
// the reference would throw. The device then forms m_f parities per shot and
// does one table load and one compare per position.
constexpr uint32_t kTabComps = 64, kTabForms = 192, kTabSel = 512;
struct TabProg {
    uint32_t comp[kTabComps];       // valid << 31 | m_f << 24 | first form
    uint32_t base[kTabComps];       // first table entry (position 0); position j at base + ((2^j - 1) << m_f)
    uint16_t form_sel_begin[kTabForms + 1];
    uint16_t form_sel[kTabSel];     // f indices of each form's selectors
};

struct LightProg {
    uint32_t valid, n_tables, tab_valid, pad;
    TabProg tab;
    uint32_t tensor_term[kLightTensors + 1];   // by model tensor index
    uint32_t term_factor[kLightTerms + 1];
    double2 term_c[kLightTerms];
    unsigned long long fu[kLightFactors], fv[kLightFactors];
    uint8_t ftable[kLightFactors];
};

// One mechanism: the first scan entry inline; further entries (joint tables)
// in global memory at ext_begin[m] .. ext_begin[m] + n_extra.
struct __align__(16) MechRec {
    unsigned long long lim0;  // fire/hit iff r01 <= lim0
    uint32_t flip0;           // flip-set id of the first entry, or kNoFlip
    uint32_t n_extra;         // number of further entries
};

// Fast filter of one mechanism, read every draw: the draw certainly needs no
// flip when ((r01 >> 32) ^ sense) < thr. sense = 0, thr = hi32(lim0) when the
// first entry is "no error" (joint tables); sense = ~0, thr = ~hi32(lim0) when
// the first entry flips and there are no further entries (singles); thr = 0
// (always take the exact path) otherwise. The exact comparison with the full
// MechRec runs only in the rare warp-uniform slow path.
struct MechFast {
    uint32_t thr, sense;
};

template <uint32_t N>
struct MechTable {
    MechFast fast[N];
    LightProg prog;
};

struct LaunchArgs {
    DevModel m;
    uint32_t num_mech;             // reference mechanism count (streams 0..num_mech-1)
    const MechRec *mech_global;    // [num_mech] full records (slow path)
    const MechFast *fast_global;   // [num_mech] filters, used when num_mech > kParamMechs
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
    uint32_t *heavy_fcols;         // f-columns for heavy_kernel: [f_width][heavy_ld32] (nullable)
    uint64_t heavy_ld32;
    void *heavy_fraw;              // per shot f word (f_width <= 64) for the deduplicated path's keys (nullable):
    uint32_t fraw_bytes;           // 4 (f_width <= 32) or 8 bytes per shot
    uint32_t *fcols_spare;         // host bookkeeping: where the f columns go if a batch must be redone
    uint32_t debug_ar_components;  // profiling only (ZXS_DEBUG_AR_COMPONENTS): evaluate this many components
    const double *tab;             // tabulated chains (LightProg.tab), clamped ratios / NaN
    // probability mode (outcome_probability_given, sampler.cpp:324-356): the
    // outcome bits are forced instead of drawn and prob[shot] receives
    // P(outcome | f) for the injected f of every shot. Every component runs
    // here (exact FP64 order), none is deferred to the large-chi kernels.
    const uint8_t *forced;         // [num_outputs] 0/1 (nullable)
    double *prob;                  // [shots]
};

// 32x32 -> 64 multiply as one mul.wide.u32 (IMAD.WIDE.U32); written in PTX
// because the C++ form lowers with extra adds of zero high words.
__device__ __forceinline__ void mul_wide(uint32_t a, uint32_t b, uint32_t &lo, uint32_t &hi) {
    asm("{\n\t.reg .b64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}" : "=r"(lo), "=r"(hi) : "r"(a), "r"(b));
}

constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u, kW1 = 0xBB67AE85u;
constexpr uint64_t kP1c = uint64_t(kM1) * 0x9e3779b9u;  // round-1 product of the constant counter word

// Mechanism-independent part of Philox rounds 1-2 for one shot index: with
// ctr = {idx_lo, idx_hi, 0x9e3779b9, 0} (rng.hpp:32-33), round 1's first
// product and round 2's first product depend only on the shot and key 0.
struct PhiloxPre {
    uint32_t a;   // hi32(M0 * idx_lo)
    uint32_t x;   // hi32(M0 * c0_1) ^ lo32(M0 * idx_lo)
    uint32_t l2;  // lo32(M0 * c0_1)
};

__device__ __forceinline__ PhiloxPre philox_pre(uint32_t idx_lo, uint32_t idx_hi, uint32_t k0_0) {
    uint32_t A, B, H2, L2;
    mul_wide(idx_lo, kM0, B, A);
    const uint32_t c0_1 = uint32_t(kP1c >> 32) ^ idx_hi ^ k0_0;
    mul_wide(c0_1, kM0, L2, H2);
    return PhiloxPre{A, H2 ^ B, L2};
}

// The rest of Philox4x32-10 for key (seed_lo, k1) (rng.hpp:44-68): 16 wide
// multiplies per block instead of 20. Returns r0 ^ (k9 ^ k0_round[9]) and r1,
// i.e. r0 itself when k9 == k0_round[9] (k9 may fold in a filter mask).
template <int S>
__device__ __forceinline__ void philox_tail(const PhiloxPre (&p)[S], uint32_t k1, const uint32_t (&k0r)[10],
                                            uint32_t k2c, uint32_t k9, uint32_t (&rhi)[S], uint32_t (&rlo)[S]) {
    uint32_t c0[S], c1[S], c2[S], c3[S];
    const uint32_t k1_1 = k1 + kW1;
#pragma unroll
    for (int s = 0; s < S; s++) {  // rounds 1 and 2
        uint32_t h, l;
        mul_wide(p[s].a ^ k1, kM1, l, h);
        c0[s] = h ^ k2c;  // hi32(M1 * c2_1) ^ lo32(kP1c) ^ k0r[1]
        c1[s] = l;
        c2[s] = p[s].x ^ k1_1;
        c3[s] = p[s].l2;
    }
    uint32_t k1i = k1 + 2 * kW1;
#pragma unroll
    for (int i = 2; i <= 8; i++) {  // rounds 3..9
#pragma unroll
        for (int s = 0; s < S; s++) {
            uint32_t h0, l0, h1, l1;
            mul_wide(c0[s], kM0, l0, h0);
            mul_wide(c2[s], kM1, l1, h1);
            const uint32_t n0 = h1 ^ c1[s] ^ k0r[i], n2 = h0 ^ c3[s] ^ k1i;
            c0[s] = n0;
            c1[s] = l1;
            c2[s] = n2;
            c3[s] = l0;
        }
        k1i += kW1;
    }
#pragma unroll
    for (int s = 0; s < S; s++) {  // round 10: only r0, r1 are used (rng.hpp:35)
        uint32_t h1, l1;
        mul_wide(c2[s], kM1, l1, h1);
        rhi[s] = h1 ^ c1[s] ^ k9;
        rlo[s] = l1;
    }
}

// eval_batch (phase_terms.cpp:90-144) for the kS 32-shot sub-tiles of a warp
// tile: acc[s] = sum_t c_t prod_k h_tk[(a<<1)|b] for this lane's shot in
// sub-tile s, accumulated in the reference's order (terms in order, factors
// in order, acc starting at 0), every product and sum rounded separately.
template <int S = kS>
__device__ __forceinline__ void eval_tensor(const DevModel &m, uint32_t t, const uint32_t *cols, uint32_t stride,
                                            uint32_t lane, double2 (&acc)[S]) {
#pragma unroll
    for (int s = 0; s < S; s++) acc[s] = make_double2(0.0, 0.0);
    const uint32_t t0 = m.tensor_term_begin[t], t1 = m.tensor_term_begin[t + 1];
    for (uint32_t term = t0; term < t1; term++) {
        const double2 c = m.term_c[term];
        double2 prod[S];
#pragma unroll
        for (int s = 0; s < S; s++) prod[s] = c;
        const uint32_t k0 = m.term_factor_begin[term], k1 = m.term_factor_begin[term + 1];
        for (uint32_t k = k0; k < k1; k++) {
            const Factor fr = m.factors[k];
            const uint16_t *sel = m.selectors + fr.sel;
            uint32_t aw[S] = {}, bw[S] = {};
            for (uint32_t i = 0; i < fr.nu; i++) {
                const uint32_t p = sel[i];
#pragma unroll
                for (int s = 0; s < S; s++) aw[s] ^= cols[s * stride + p];
            }
            for (uint32_t i = 0; i < fr.nv; i++) {
                const uint32_t p = sel[fr.nu + i];
#pragma unroll
                for (int s = 0; s < S; s++) bw[s] ^= cols[s * stride + p];
            }
            const double2 *h = m.h_table + 4 * fr.table;
#pragma unroll
            for (int s = 0; s < S; s++) {
                const uint32_t idx = (((aw[s] >> lane) & 1u) << 1) | ((bw[s] >> lane) & 1u);
                prod[s] = cmul_rn(prod[s], h[idx]);
            }
        }
#pragma unroll
        for (int s = 0; s < S; s++) acc[s] = cadd_rn(acc[s], prod[s]);
    }
}

// eval_tensor over the uniform LightProg: same products and sums in the
// reference's order (phase_terms.cpp:121-131); h tables staged in shared
// memory (sh, 4 entries per table), selected per lane by (a << 1) | b.
template <int S = kS>
__device__ __forceinline__ void eval_tensor_light(const LightProg &pg, uint32_t t, const uint32_t *cols,
                                                  uint32_t stride, uint32_t lane, const double2 *sh,
                                                  double2 (&acc)[S]) {
#pragma unroll
    for (int s = 0; s < S; s++) acc[s] = make_double2(0.0, 0.0);
    const uint32_t t0 = pg.tensor_term[t], t1 = pg.tensor_term[t + 1];
    for (uint32_t term = t0; term < t1; term++) {
        const double2 c = pg.term_c[term];
        double2 prod[S];
#pragma unroll
        for (int s = 0; s < S; s++) prod[s] = c;
        const uint32_t k0 = pg.term_factor[term], k1 = pg.term_factor[term + 1];
        for (uint32_t k = k0; k < k1; k++) {
            uint32_t aw[S] = {}, bw[S] = {};
            for (unsigned long long x = pg.fu[k]; x; x &= x - 1) {
                const uint32_t p = __ffsll((long long)x) - 1;
#pragma unroll
                for (int s = 0; s < S; s++) aw[s] ^= cols[s * stride + p];
            }
            for (unsigned long long x = pg.fv[k]; x; x &= x - 1) {
                const uint32_t p = __ffsll((long long)x) - 1;
#pragma unroll
                for (int s = 0; s < S; s++) bw[s] ^= cols[s * stride + p];
            }
            const double2 *h = sh + 4 * pg.ftable[k];
#pragma unroll
            for (int s = 0; s < S; s++) {
                const uint32_t idx = (((aw[s] >> lane) & 1u) << 1) | ((bw[s] >> lane) & 1u);
                prod[s] = cmul_rn(prod[s], h[idx]);
            }
        }
#pragma unroll
        for (int s = 0; s < S; s++) acc[s] = cadd_rn(acc[s], prod[s]);
    }
}

__device__ __forceinline__ void report_ratio_error(unsigned long long *err, uint64_t shot) {
    atomicOr(&err[0], 1ull);
    atomicMin(&err[1], (unsigned long long)shot);
}

// Near-tie draws of the integer (monomial / deduplicated) paths, whose values
// differ from the reference's by the reference's own rounding (<= 1e-12
// relative of the term-magnitude sum, tests/test_gpu_parity.py): a draw whose
// uniform lies within 1e-9 (relative) of the clamped ratio is one whose bit
// could differ from the reference's. Counted in err[2] (zxs_tie_count).
__device__ __forceinline__ void count_near_tie(unsigned long long *err, double u, double cl) {
    if (fabs(u - cl) <= 1e-9 * fmax(cl, 1e-300)) atomicAdd(&err[2], 1ull);
}

// Rare path of the mechanism draw: the flip set selected by each of the
// lane's two draws (first entry, then the rest of a joint table in order).
// Kept out of line so the divergent scan does not pull the draw loop's
// counters and Philox keys off the uniform datapath. Draws and results travel
// by value (registers under the ABI) rather than through arrays passed by
// reference (local memory).
template <int S>
struct DrawsS {
    uint64_t v[S];
};
template <int S>
struct FlipsS {
    uint32_t v[S];
};
template <int S>
__device__ __noinline__ FlipsS<S> resolve_flips(const DrawsS<S> r, MechRec md, const uint32_t *ext_begin,
                                                const ulonglong2 *ext, uint32_t mi) {
    FlipsS<S> out;
#pragma unroll
    for (int s = 0; s < S; s++) {
        uint32_t flip = kNoFlip;
        if (r.v[s] <= md.lim0) {
            flip = md.flip0;
        } else if (md.n_extra) {
            const uint32_t e0 = ext_begin[mi];
            for (uint32_t e = e0; e < e0 + md.n_extra; e++) {
                const ulonglong2 en = ext[e];
                if (r.v[s] <= en.x) {
                    flip = uint32_t(en.y);
                    break;
                }
            }
        }
        out.v[s] = flip;
    }
    return out;
}

// Stores the lane group's S consecutive 32-bit output words of a tile (row
// `row`, first word `w0`), only those below the row length `ld` (the last
// tile of a range may be partial).
template <int S>
__device__ __forceinline__ void store_words(uint32_t *row, uint64_t w0, uint64_t ld, const uint32_t (&w)[S]) {
    if constexpr (S == 2) {
        *reinterpret_cast<uint2 *>(row + w0) = make_uint2(w[0], w[1]);  // ld is even: always in range
    } else {
        if (w0 + S <= ld) {
            if ((reinterpret_cast<uintptr_t>(row + w0) & 15) == 0) {
                *reinterpret_cast<uint4 *>(row + w0) = make_uint4(w[0], w[1], w[2], w[3]);
            } else {  // odd 64-bit row pitch: rows are only 8-byte aligned
                *reinterpret_cast<uint2 *>(row + w0) = make_uint2(w[0], w[1]);
                *reinterpret_cast<uint2 *>(row + w0 + 2) = make_uint2(w[2], w[3]);
            }
        } else {
#pragma unroll
            for (int s = 0; s < S; s++) {
                if (w0 + s < ld) row[w0 + s] = w[s];
            }
        }
    }
}

template <int FW, bool PARAM_MECHS, int S>
#ifndef ZXS_MAXNREG
#define ZXS_MAXNREG 96
#endif
#ifndef ZXS_MAXNREG4
#define ZXS_MAXNREG4 128  // measured: 128 (80 B of spills) beats 144 / 160 without spills
#endif
__global__ void __maxnreg__(S == 4 ? ZXS_MAXNREG4 : ZXS_MAXNREG) shot_kernel(const __grid_constant__ LaunchArgs a,
                                                   const __grid_constant__ MechTable<PARAM_MECHS ? kParamMechs : 1> mt) {
    extern __shared__ __align__(16) uint32_t smem[];
    // One warp per CTA: the tile loop depends only on blockIdx, so the
    // compiler can keep loop counters, Philox keys and mechanism records in
    // uniform registers (UR) on the uniform datapath.
    const DevModel &m = a.m;
    const uint32_t lane = threadIdx.x;
    unsigned long long *scount = reinterpret_cast<unsigned long long *>(smem);
    const bool light = mt.prog.valid != 0;
    const uint32_t sh_off = (2 * m.num_outputs + 3) & ~3u;  // 16-byte aligned
    double2 *sh = reinterpret_cast<double2 *>(smem + sh_off);  // light h tables
    uint32_t *cols = smem + sh_off + (light ? 16 * mt.prog.n_tables : 0);
    if (light) {
        for (uint32_t i = lane; i < 4 * mt.prog.n_tables; i += 32) sh[i] = m.h_table[i];
        __syncwarp();
    }
    if (a.counts) {
        for (uint32_t o = lane; o < m.num_outputs; o += 32) scount[o] = 0;
        __syncwarp();
    }
    const uint32_t seed_hi = uint32_t(a.seed >> 32);
    const uint32_t k2c = uint32_t(kP1c) ^ a.k0_round[1];

    for (uint64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        uint64_t local[S], shot[S];
        uint32_t vmask[S];
        PhiloxPre pre[S];
#pragma unroll
        for (int s = 0; s < S; s++) {
            local[s] = tile * (32 * S) + 32 * s + lane;
            vmask[s] = __ballot_sync(kFull, local[s] < a.shots);
            shot[s] = a.first_shot + local[s];
            pre[s] = philox_pre(uint32_t(shot[s]), uint32_t(shot[s] >> 32), a.k0_round[0]);
        }

        // ---- (1)-(3): f configuration as bit-sliced columns
        if (a.fcols_in) {
            for (uint32_t c = lane; c < m.f_width; c += 32) {
#pragma unroll
                for (int s = 0; s < S; s++) {
                    const uint64_t wi = tile * S + s;
                    cols[s * m.col_stride + c] = wi < a.fcols_ld32 ? a.fcols_in[c * a.fcols_ld32 + wi] : 0u;
                }
            }
        } else {
            uint64_t f[S][FW];
#pragma unroll
            for (int w = 0; w < FW; w++) {
                const uint64_t b = m.base_offset[w];
#pragma unroll
                for (int s = 0; s < S; s++) f[s][w] = b;
            }
            for (uint32_t mi = 0; mi < a.num_mech; mi++) {
                // No early-out for mechanisms that cannot flip anything: a
                // data-dependent `continue` here moves the key schedule off the
                // uniform datapath. Such records never flip.
                const MechFast mf = PARAM_MECHS ? mt.fast[mi] : a.fast_global[mi];
                uint32_t rhi[S], rlo[S];
                philox_tail<S>(pre, seed_hi ^ mi, a.k0_round, k2c, a.k0_round[9] ^ mf.sense, rhi, rlo);
                // Common case: every lane's draw certainly resolves to "no flip"
                // (no error); anything else takes one warp-uniform branch, which
                // keeps the loop (and the key schedule) uniform.
                bool busy = false;
#pragma unroll
                for (int s = 0; s < S; s++) busy |= !(rhi[s] < mf.thr);
                if (__any_sync(kFull, busy)) {
                    const MechRec md = a.mech_global[mi];
                    DrawsS<S> rr;
#pragma unroll
                    for (int s = 0; s < S; s++) rr.v[s] = (uint64_t(rhi[s] ^ mf.sense) << 32) | rlo[s];
                    const FlipsS<S> flip = resolve_flips<S>(rr, md, a.ext_begin, a.ext, mi);
#pragma unroll
                    for (int s = 0; s < S; s++) {
                        if (flip.v[s] != kNoFlip) {
                            const uint64_t *mask = m.flip_mask + size_t(flip.v[s]) * FW;
#pragma unroll
                            for (int w = 0; w < FW; w++) f[s][w] ^= mask[w];
                        }
                    }
                }
            }
            if constexpr (FW == 1) {
                if (a.heavy_fraw) {  // lane = shot: coalesced 4- or 8-byte stores
#pragma unroll
                    for (int s = 0; s < S; s++) {
                        if (local[s] < a.shots) {
                            if (a.fraw_bytes == 4) {
                                static_cast<uint32_t *>(a.heavy_fraw)[local[s]] = uint32_t(f[s][0]);
                            } else {
                                static_cast<unsigned long long *>(a.heavy_fraw)[local[s]] = f[s][0];
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int s = 0; s < S; s++) {
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
        if (a.heavy_fcols) {
            for (uint32_t c = lane; c < m.f_width; c += 32) {
#pragma unroll
                for (int s = 0; s < S; s++) {
                    if (tile * S + s < a.heavy_ld32) a.heavy_fcols[c * a.heavy_ld32 + tile * S + s] = cols[s * m.col_stride + c];
                }
            }
        }
        if (a.fcols_out) {
            for (uint32_t c = lane; c < m.f_width; c += 32) {
#pragma unroll
                for (int s = 0; s < S; s++) {
                    if (tile * S + s < a.fcols_ld32) a.fcols_out[c * a.fcols_ld32 + tile * S + s] = cols[s * m.col_stride + c] & vmask[s];
                }
            }
            __syncwarp();
            continue;
        }

        // ---- (4): direct outputs, lane-parallel over outputs
        uint32_t mism[S] = {};  // probability mode: shots whose direct outputs differ from the outcome
        for (uint32_t d = lane; d < m.num_direct; d += 32) {
            const uint32_t od = m.direct_out[d];
            uint32_t w[S];
#pragma unroll
            for (int s = 0; s < S; s++) w[s] = (od >> 31) ? kFull : 0u;
            for (uint32_t b = m.direct_bit_begin[d]; b < m.direct_bit_begin[d + 1]; b++) {
                const uint32_t fb = m.direct_bits[b];
#pragma unroll
                for (int s = 0; s < S; s++) w[s] ^= cols[s * m.col_stride + fb];
            }
            const uint32_t o = od & 0x7fffffffu;
            if (a.forced) {
                const uint32_t want = a.forced[o] ? kFull : 0u;
#pragma unroll
                for (int s = 0; s < S; s++) mism[s] |= w[s] ^ want;
                continue;
            }
#pragma unroll
            for (int s = 0; s < S; s++) w[s] &= vmask[s];
            if (a.out32) store_words<S>(a.out32 + o * a.ld32, tile * S, a.ld32, w);
            if (a.counts) {
                uint32_t ones = 0;
#pragma unroll
                for (int s = 0; s < S; s++) ones += __popc(w[s]);
                if (ones) atomicAdd(&scount[o], (unsigned long long)ones);
            }
        }

        double pgiven[S];
        bool pzero[S];
#pragma unroll
        for (int s = 0; s < S; s++) {
            pgiven[s] = 1.0;
            pzero[s] = false;
        }
        if (a.forced) {
#pragma unroll
            for (int s = 0; s < S; s++) {
                mism[s] = __reduce_or_sync(kFull, mism[s]);
                pzero[s] = (mism[s] >> lane) & 1u;  // sampler.cpp:328-336: return 0.0 before any component
            }
        }

        // ---- (5): autoregressive components
        uint32_t upos = 0;
        const uint32_t ncomp_eval = min(m.num_components, a.debug_ar_components);
        for (uint32_t ci = 0; ci < ncomp_eval; ci++) {
            const uint32_t ob = m.comp_out_begin[ci], n = m.comp_out_begin[ci + 1] - ob;
            if (m.comp_heavy[ci] && !a.forced) {  // evaluated by heavy_kernel / mono_kernel
                upos += n;
                continue;
            }
            if (mt.prog.tab_valid && ci < kTabComps && (mt.prog.tab.comp[ci] >> 31) && !a.forced) {
                // ---- tabulated chain (TabProg): m_f form parities + sampled bits index the ratios
                const uint32_t cw = mt.prog.tab.comp[ci], mf = (cw >> 24) & 0x7fu, f0 = cw & 0xffffu;
                uint32_t idx[S] = {};
                for (uint32_t i = 0; i < mf; i++) {
                    uint32_t w[S] = {};
                    for (uint32_t q = mt.prog.tab.form_sel_begin[f0 + i]; q < mt.prog.tab.form_sel_begin[f0 + i + 1]; q++) {
                        const uint32_t pcol = mt.prog.tab.form_sel[q];
#pragma unroll
                        for (int s = 0; s < S; s++) w[s] ^= cols[s * m.col_stride + pcol];
                    }
#pragma unroll
                    for (int s = 0; s < S; s++) idx[s] |= ((w[s] >> lane) & 1u) << i;
                }
                const double *tabp = a.tab + mt.prog.tab.base[ci];
                for (uint32_t pos = 0; pos < n; pos++, upos++) {
                    uint32_t rhi[S], rlo[S];
                    if (!a.uniforms) {
                        const uint32_t stream = 0x80000000u ^ (ci << 12) ^ pos;  // sampler.cpp:37-39
                        philox_tail<S>(pre, seed_hi ^ stream, a.k0_round, k2c, a.k0_round[9], rhi, rlo);
                    }
                    const double *tj = tabp + ((size_t((1u << pos) - 1u)) << mf);
                    uint32_t word[S];
#pragma unroll
                    for (int s = 0; s < S; s++) {
                        const bool valid = local[s] < a.shots;
                        const double cl = __ldg(tj + idx[s]);
                        if (isnan(cl) && valid) report_ratio_error(a.err, shot[s]);  // sampler.cpp:86-89
                        const double u = a.uniforms ? (valid ? a.uniforms[upos * a.uniforms_ld + local[s]] : 0.0)
                                                    : philox_uniform((uint64_t(rhi[s]) << 32) | rlo[s]);
                        const bool bit = !(u < cl);
                        idx[s] |= uint32_t(bit) << (mf + pos);
                        word[s] = __ballot_sync(kFull, bit) & vmask[s];
                    }
                    if (lane == 0) {
                        const uint32_t o = m.comp_outputs[ob + pos];
                        if (a.out32) store_words<S>(a.out32 + o * a.ld32, tile * S, a.ld32, word);
                        if (a.counts) {
                            uint32_t ones = 0;
#pragma unroll
                            for (int s = 0; s < S; s++) ones += __popc(word[s]);
                            if (ones) atomicAdd(&scount[o], (unsigned long long)ones);
                        }
                    }
                }
                continue;
            }
            const uint32_t tb = m.comp_tensor_begin[ci];
            // the light program holds the non-heavy components' tensors only: a heavy one
            // evaluated here (probability mode) reads the global tensors
            const bool lightc = light && !m.comp_heavy[ci];
            for (uint32_t p = lane; p < n; p += 32) {
#pragma unroll
                for (int s = 0; s < S; s++) cols[s * m.col_stride + m.f_width + p] = 0u;
            }
            __syncwarp();
            double2 acc[S];
            double prev[S], norm[S];
            if (lightc) {
                eval_tensor_light<S>(mt.prog, tb, cols, m.col_stride, lane, sh, acc);
            } else {
                eval_tensor<S>(m, tb, cols, m.col_stride, lane, acc);
            }
#pragma unroll
            for (int s = 0; s < S; s++) {
                prev[s] = norm[s] = acc[s].x;
                // sampler.cpp:343-345
                if (a.forced && !pzero[s] && local[s] < a.shots && !(norm[s] > 0.0)) report_ratio_error(a.err, shot[s]);
            }
            for (uint32_t pos = 0; pos < n; pos++, upos++) {
                if (lightc) {
                    eval_tensor_light<S>(mt.prog, tb + 1 + pos, cols, m.col_stride, lane, sh, acc);
                } else {
                    eval_tensor<S>(m, tb + 1 + pos, cols, m.col_stride, lane, acc);
                }
                if (a.forced) {  // sampler.cpp:346-352: forced outcome bit
                    const uint32_t o = m.comp_outputs[ob + pos];
                    const bool bit = a.forced[o] != 0;
#pragma unroll
                    for (int s = 0; s < S; s++) prev[s] = bit ? __dsub_rn(prev[s], acc[s].x) : acc[s].x;
                    if (lane == 0) {
#pragma unroll
                        for (int s = 0; s < S; s++) cols[s * m.col_stride + m.f_width + pos] = bit ? kFull : 0u;
                    }
                    __syncwarp();
                    continue;
                }
                uint32_t rhi[S], rlo[S];
                if (!a.uniforms) {
                    const uint32_t stream = 0x80000000u ^ (ci << 12) ^ pos;  // sampler.cpp:37-39
                    philox_tail<S>(pre, seed_hi ^ stream, a.k0_round, k2c, a.k0_round[9], rhi, rlo);
                }
                uint32_t word[S];
#pragma unroll
                for (int s = 0; s < S; s++) {
                    const bool valid = local[s] < a.shots;
                    const double cur = acc[s].x;
                    const double ratio = __ddiv_rn(cur, prev[s]);
                    if (!(ratio > -1e-6 && ratio < 1.0 + 1e-6) && valid) report_ratio_error(a.err, shot[s]);
                    double cl = (0.0 < ratio) ? ratio : 0.0;  // std::max(0.0, ratio)
                    cl = (cl < 1.0) ? cl : 1.0;               // std::min(1.0, .)
                    const double u = a.uniforms ? (valid ? a.uniforms[upos * a.uniforms_ld + local[s]] : 0.0)
                                                : philox_uniform((uint64_t(rhi[s]) << 32) | rlo[s]);
                    const bool bit = !(u < cl);
                    prev[s] = bit ? __dsub_rn(prev[s], cur) : cur;
                    word[s] = __ballot_sync(kFull, bit) & vmask[s];
                }
                if (lane == 0) {
#pragma unroll
                    for (int s = 0; s < S; s++) cols[s * m.col_stride + m.f_width + pos] = word[s];
                    const uint32_t o = m.comp_outputs[ob + pos];
                    if (a.out32) store_words<S>(a.out32 + o * a.ld32, tile * S, a.ld32, word);
                    if (a.counts) {
                        uint32_t ones = 0;
#pragma unroll
                        for (int s = 0; s < S; s++) ones += __popc(word[s]);
                        if (ones) atomicAdd(&scount[o], (unsigned long long)ones);
                    }
                }
                __syncwarp();
            }
            if (a.forced) {
#pragma unroll
                for (int s = 0; s < S; s++) pgiven[s] = __dmul_rn(pgiven[s], __ddiv_rn(prev[s], norm[s]));  // sampler.cpp:353
            }
        }
        if (a.forced) {
#pragma unroll
            for (int s = 0; s < S; s++) {
                if (local[s] < a.shots) a.prob[local[s]] = pzero[s] ? 0.0 : pgiven[s];
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
                                                   unsigned long long *max_imag_bits, double *imag_values) {
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
                if (imag_values) imag_values[local] = acc[s].y;
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

// Same-op-mix roofline for the error draw: the shot kernel's Philox code
// (philox_pre once per tile, philox_tail + filter compare per mechanism,
// kS shots per lane, one warp per CTA) with no memory traffic at all.
__global__ void __maxnreg__(ZXS_MAXNREG) philox_peak_kernel(const __grid_constant__ LaunchArgs a, uint32_t nmech,
                                                            uint32_t tiles_per_cta, uint32_t *sink) {
    const uint32_t lane = threadIdx.x, seed_hi = uint32_t(a.seed >> 32);
    const uint32_t k2c = uint32_t(kP1c) ^ a.k0_round[1];
    uint32_t acc = 0;
    for (uint32_t t = 0; t < tiles_per_cta; t++) {
        PhiloxPre pre[kS];
#pragma unroll
        for (int s = 0; s < kS; s++) {
            const uint64_t shot = (uint64_t(blockIdx.x) * tiles_per_cta + t) * kTileShots + 32 * s + lane;
            pre[s] = philox_pre(uint32_t(shot), uint32_t(shot >> 32), a.k0_round[0]);
        }
        for (uint32_t mi = 0; mi < nmech; mi++) {
            uint32_t rhi[kS], rlo[kS];
            philox_tail<kS>(pre, seed_hi ^ mi, a.k0_round, k2c, a.k0_round[9], rhi, rlo);
            bool busy = false;
#pragma unroll
            for (int s = 0; s < kS; s++) busy |= !(rhi[s] < 0xffff0000u);
            if (__any_sync(kFull, busy)) acc ^= rlo[0] ^ rlo[1];
        }
    }
    if (acc == 0x9e3779b9u) sink[0] = acc;  // keeps the work observable
}

// Same-op-mix roofline for the exact contraction (heavy_kernel): independent
// chains of cmul_rn + cadd_rn (4 DMUL + 4 DADD, no FMA), 8 per thread.
__global__ void __launch_bounds__(256) fp64_peak_kernel(double2 h, uint32_t iters, double *sink) {
    double2 p[8];
#pragma unroll
    for (int i = 0; i < 8; i++) p[i] = make_double2(1.0 + 1e-3 * (threadIdx.x + i), 1e-3 * i);
    double2 acc = make_double2(0.0, 0.0);
    for (uint32_t it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            p[i] = cmul_rn(p[i], h);
            acc = cadd_rn(acc, p[i]);
        }
    }
    if (acc.x == 1.2345 && acc.y == 6.789) sink[0] = acc.x;  // keeps the work observable
}

// Same-op-mix roofline for mono_kernel's selector loads: conflict-free
// 32-bit shared loads (one 128 B wavefront per warp instruction) XORed into a
// register, addresses a per-lane base plus warp-uniform plane offsets.
__global__ void __launch_bounds__(256) smem_peak_kernel(uint32_t iters, uint32_t *sink) {
    __shared__ uint32_t planes[64 * 32];
    const uint32_t lane = threadIdx.x & 31u;
    for (uint32_t i = threadIdx.x; i < 64 * 32; i += blockDim.x) planes[i] = i * 0x9E3779B9u;
    __syncthreads();
    const char *lb = reinterpret_cast<const char *>(planes + lane);
    uint32_t acc = 0, off = 0;
    for (uint32_t it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 16; k++) acc ^= *reinterpret_cast<const uint32_t *>(lb + ((off + k * 5u) & 63u) * 128u);
        off += 7;
    }
    if (acc == 0x12345678u) sink[0] = acc;  // keeps the work observable
}

__global__ void philox_kernel(uint64_t seed, uint32_t stream, uint64_t first, uint64_t n, double *out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t idx = first + i;
        out[i] = philox_uniform(philox_r01(uint32_t(seed), uint32_t(seed >> 32) ^ stream, uint32_t(idx),
                                           uint32_t(idx >> 32)));
    }
}

}  // namespace zxs_dev
