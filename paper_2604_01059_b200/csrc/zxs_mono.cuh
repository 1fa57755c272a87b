// zxs_mono.cuh — integer (Clifford-monomial) contraction of large-chi components.
//
// Every h table the reference builds is h(a,b) = 1 + e^{i(al+a pi)} +
// e^{i(be+b pi)} - e^{i(al+be+a pi+b pi)} (phase_terms.cpp:40-47,
// scalar.cpp:81-85). When al, be are multiples of pi/2 (every table of every
// BASELINE circuit: the branches of decompose_magic are Clifford diagrams,
// SURVEY §8 a13), each entry is exactly 0 or 2^(m/2) w^k (w = e^{i pi/4}) with
// m fixed per table and k mod 2 fixed per table. So a term's product over its
// factors is c_t 2^(M/2) w^(K0) i^J, where M, K0 are per-term constants and
//   J = sum_k d_k(a_k, b_k) mod 4,   zero = OR_k z_k(a_k, b_k)
// depend on the shot only through the factor parities a_k = u_k.P, b_k = v_k.P.
// The host folds the constants into c'_t and lowers every factor to one
// record acting on three bit-sliced words per lane (32 shots each):
//   J0, J1  (J mod 4, two bit planes)   Z  (term is zero)
// and the per-term epilogue adds Re(c'_t i^J) = {re, -im, -re, im}[J] to the
// shot's FP64 accumulator for every non-zero shot, terms in the reference's
// order (phase_terms.cpp:129-131). This is the north star's "exact
// dyadic-phase accumulation": no floating-point work per factor at all; the
// values differ from the reference's only by the reference's own rounding of
// its h entries (~1e-16 relative), so sampled bits agree except at exact
// threshold ties (counted by the tests).
//
// Term sharing: consecutive terms share most of their factors (the
// cultivation proxy's terms are a product of six 6-way cat5 branches), so the
// host arranges each tensor's terms in a shared-prefix tree (zxs_api.cu
// mono_tree): a node's records are applied on top of its parent's (Z, J0,
// J1), kept per level in a small shared-memory stack, and leaves -- the
// terms, in the reference's order -- run the epilogue. This cuts the records
// evaluated per shot ~2.6x on that circuit.
//
// Work decomposition: lane = one 32-shot word (bit s = shot 32*w + s), a warp
// = 1024 shots, a CTA = kMonoWarps warps that walk the SAME record stream:
// chunks of the stream are fetched once per CTA with cp.async.bulk into a
// double buffer and read with warp-uniform (broadcast) shared loads. The
// parities a = u.P are formed from the lane's parameter planes in shared
// memory (plane[p][lane], conflict-free), selector lists coming from a form
// dictionary (distinct u/v lists of the component, 16 B per entry of up to
// seven pre-scaled plane offsets, read through L1).
#pragma once

#include "zxs_heavy.cuh"

namespace zxs_dev {

// Words per lane NW: 1 (32 shots per lane, 16 warps per SM) or 2 (64 shots per
// lane via 64-bit plane loads, 12 warps per SM: half the issue slots per shot
// for the parity work at 128 accumulator registers).
template <int NW>
struct MonoCfg;
template <>
struct MonoCfg<1> {
    static constexpr int kWarps = 16;
};
template <>
struct MonoCfg<2> {
    static constexpr int kWarps = 12;
};
constexpr int kMonoWarps = 16;               // upper bound of MonoCfg<NW>::kWarps (host sizing)
constexpr uint32_t kMonoChunkWords = 2048;   // 8 KiB per chunk buffer
// record word: kind << 28 | second form << kFormShiftB | first form (14-bit dictionary ids)
constexpr uint32_t kFormMask = 0x3fffu;
constexpr int kFormShiftB = 14;
constexpr uint32_t kFvFormBytes = 32 * 4;  // block form table (dedup_eval_kernel): fv[form][lane], 32-bit words
constexpr uint32_t kMonoNoForm = kFormMask;  // "no form" (parity 0) in the 14-bit form fields
constexpr int kMaxMonoComps = 8;
constexpr uint32_t kMonoMaxDepth = 8;        // levels of the shared-prefix term tree
constexpr uint32_t kMonoSegStart = 1u << 30; // node header flag: first node of a summation segment
constexpr uint32_t kDedupSegs = 2368;        // summation segments per tensor (148 SMs x 16 warps)

// record kinds (bits 28..31 of a record word; first form in bits 0..13,
// second form in bits 14..27; ids index the tensor's dictionary)
enum : uint32_t {
    kRecAdd = 0,    // J += a
    kRecSub = 1,    // J -= a
    kRecAdd2 = 2,   // J += 2a
    kRecZ = 3,      // Z |= a
    kRecZn = 4,     // Z |= ~a
    kRecGen = 15,   // two forms; next word: alpha | beta << 2 | gamma << 4 | zlut << 6
};

struct MonoArgs {
    uint64_t seed, first_shot, shots, n_cta_tiles;
    uint32_t k0_round[10];
    // planes per warp: [0, W) the current tensor's basis planes, all_plane = ALL (XOR of the W basis
    // planes), all_plane + 1 = ZERO (padding selectors), all_plane + 2 + j = raw sampled bit j
    uint32_t f_width, n_planes, all_plane;
    const uint32_t *tensor_width;     // [mono tensors] param width W
    const uint32_t *tensor_basis_begin;       // [mono tensors] first basis vector
    const unsigned long long *basis;  // basis vectors: masks over the component's local params
    const uint16_t *param_map;        // local param -> raw param (f column, or f_width + sampled bit)
    const uint32_t *fcols;            // [f_width][fcols_ld32] from shot_kernel
    uint64_t fcols_ld32;
    uint32_t *out32;                  // [num_outputs][out_ld32] (nullable)
    uint64_t out_ld32;
    unsigned long long *counts;       // (nullable)
    const double *uniforms;           // injected AR uniforms (nullable)
    uint64_t uniforms_ld;
    unsigned long long *err;
    double *scratch;                  // [3][n_cta_tiles * warps * shots per warp]: prev, cur, folded sum per shot
    const uint32_t *words;            // record streams
    const uint4 *chunks;              // {word_begin, n_words (multiple of 4), n_terms, 0}
    const uint32_t *tensor_chunk_begin;
    uint32_t total_chunks;
    const uint4 *dict;                // form dictionaries, one per tensor
    const uint32_t *tensor_dict_begin;  // [mono tensors + 1]
    uint32_t max_dict;                // largest per-tensor dictionary (entries staged in smem)
    uint32_t stack_depth;             // levels of (Z, J0, J1) kept per lane (deepest node + 1)
    const uint32_t *comp_outputs;
    // eval seam: evaluate one tensor and store the values (no chain)
    int eval_tensor;                  // -1: sample; else index into tensor_chunk_begin
    uint32_t eval_comp;               // eval: index into comps of the tensor's component
    double *eval_out;                 // [shots]
    uint32_t n_comps;
    HeavyComp comps[kMaxMonoComps];
};

// Bit-sliced words of NW x 32 shots.
template <int NW>
struct BW {
    uint32_t w[NW];
};
template <int NW>
__device__ __forceinline__ BW<NW> bw_zero() {
    BW<NW> r;
#pragma unroll
    for (int i = 0; i < NW; i++) r.w[i] = 0u;
    return r;
}
#define ZXS_BW_OP(NAME, EXPR)                                                   \
    template <int NW>                                                           \
    __device__ __forceinline__ BW<NW> NAME(const BW<NW> &a, const BW<NW> &b) { \
        BW<NW> r;                                                               \
        _Pragma("unroll") for (int i = 0; i < NW; i++) r.w[i] = (EXPR);        \
        return r;                                                               \
    }
ZXS_BW_OP(bw_xor, a.w[i] ^ b.w[i])
ZXS_BW_OP(bw_and, a.w[i] & b.w[i])
ZXS_BW_OP(bw_or, a.w[i] | b.w[i])
ZXS_BW_OP(bw_andn, ~a.w[i] & b.w[i])  // ~a & b
#undef ZXS_BW_OP
template <int NW>
__device__ __forceinline__ BW<NW> bw_not(const BW<NW> &a) {
    BW<NW> r;
#pragma unroll
    for (int i = 0; i < NW; i++) r.w[i] = ~a.w[i];
    return r;
}

// One plane of the lane: plane p of lane l at byte (p * 32 + l) * 4 * NW.
template <int NW>
__device__ __forceinline__ BW<NW> mono_plane(const char *lb, uint32_t p) {
    if constexpr (NW == 1) {
        BW<1> r;
        r.w[0] = *reinterpret_cast<const uint32_t *>(lb + (p << 7));
        return r;
    } else {
        const uint2 v = *reinterpret_cast<const uint2 *>(lb + (p << 8));
        BW<2> r;
        r.w[0] = v.x;
        r.w[1] = v.y;
        return r;
    }
}

// Parity words of dictionary form f for the lane's shots: XOR of the lane's
// parameter planes the entry lists. Entry layout (16 B): byte 0 = size class
// c (2c + 2 selector slots, 15 for c = 7) | 0x80 if the list continues in
// the next entry; bytes 1..15 = plane indices, unused slots naming the
// all-zero plane. Lists longer than half the tensor's width are stored
// complemented against the ALL plane. Each size class is straight-line code:
// every load of the entry is issued before the XOR tree consumes them (a
// selector costs a byte extract, an address IMAD, one LDS and half a 3-input
// XOR per word), and the warp takes one uniform branch per entry.
// Selector k (1..15) of entry e: plane index in byte k.
template <int NW>
__device__ __forceinline__ BW<NW> mono_sel(const uint4 &e, const char *lb, int k) {
    const uint32_t word = k < 4 ? e.x : k < 8 ? e.y : k < 12 ? e.z : e.w;
    return mono_plane<NW>(lb, __byte_perm(word, 0u, 0x4440u + uint32_t(k & 3)));
}

// XOR of the first N selectors of one entry (N a size class's slot count),
// or of two entries of the same class with all 2N loads issued together.
template <int NW, int N>
__device__ __forceinline__ BW<NW> mono_cls(const uint4 &e, const char *lb) {
    BW<NW> v[N];
#pragma unroll
    for (int k = 0; k < N; k++) v[k] = mono_sel<NW>(e, lb, k + 1);
#pragma unroll
    for (int st = 1; st < N; st <<= 1) {
#pragma unroll
        for (int k = 0; k + st < N; k += 2 * st) v[k] = bw_xor<NW>(v[k], v[k + st]);
    }
    return v[0];
}
template <int NW, int N>
__device__ __forceinline__ void mono_cls2(const uint4 &e0, const uint4 &e1, const char *lb, BW<NW> &r0, BW<NW> &r1) {
    BW<NW> v[N], u[N];
#pragma unroll
    for (int k = 0; k < N; k++) {
        v[k] = mono_sel<NW>(e0, lb, k + 1);
        u[k] = mono_sel<NW>(e1, lb, k + 1);
    }
#pragma unroll
    for (int st = 1; st < N; st <<= 1) {
#pragma unroll
        for (int k = 0; k + st < N; k += 2 * st) {
            v[k] = bw_xor<NW>(v[k], v[k + st]);
            u[k] = bw_xor<NW>(u[k], u[k + st]);
        }
    }
    r0 = v[0];
    r1 = u[0];
}

template <int NW>
__device__ __forceinline__ BW<NW> mono_entry(const uint4 e, const char *lb) {
    switch (e.x & 7u) {  // slots: 2, 4, 6, 8, 10, 12, 14, 15
        case 0: return mono_cls<NW, 2>(e, lb);
        case 1: return mono_cls<NW, 4>(e, lb);
        case 2: return mono_cls<NW, 6>(e, lb);
        case 3: return mono_cls<NW, 8>(e, lb);
        case 4: return mono_cls<NW, 10>(e, lb);
        case 5: return mono_cls<NW, 12>(e, lb);
        case 6: return mono_cls<NW, 14>(e, lb);
        default: return mono_cls<NW, 15>(e, lb);
    }
}

// Two single-entry forms of the same size class: one branch, 2N loads in flight
// (classes up to kPairMaxCls: the register budget of the 64-shot lanes).
constexpr uint32_t kPairMaxCls = 4;
template <int NW>
__device__ __forceinline__ void mono_entry2(const uint4 e0, const uint4 e1, const char *lb, BW<NW> &r0, BW<NW> &r1) {
    switch (e0.x & 7u) {
        case 0: mono_cls2<NW, 2>(e0, e1, lb, r0, r1); return;
        case 1: mono_cls2<NW, 4>(e0, e1, lb, r0, r1); return;
        case 2: mono_cls2<NW, 6>(e0, e1, lb, r0, r1); return;
        case 3: mono_cls2<NW, 8>(e0, e1, lb, r0, r1); return;
        default: mono_cls2<NW, 10>(e0, e1, lb, r0, r1); return;
    }
}

#ifndef ZXS_FORM_NOINLINE
#define ZXS_FORM_NOINLINE 0
#endif
template <int NW>
#if ZXS_FORM_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
BW<NW> mono_form(const uint4 *sd, uint32_t f, const char *lb) {
    uint4 e = sd[f];
    BW<NW> acc = mono_entry<NW>(e, lb);
    while (e.x & 0x80u) {
        e = sd[++f];
        acc = bw_xor<NW>(acc, mono_entry<NW>(e, lb));
    }
    return acc;
}

// J += c * x (mod 4) on the bit planes (J0, J1), c in 0..3.
template <int NW>
__device__ __forceinline__ void j_add(BW<NW> &j0, BW<NW> &j1, const BW<NW> &x, uint32_t c) {
#pragma unroll
    for (int i = 0; i < NW; i++) {
        const uint32_t xl = (c & 1u) ? x.w[i] : 0u;
        j1.w[i] ^= (j0.w[i] & xl) ^ ((c & 2u) ? x.w[i] : 0u);
        j0.w[i] ^= xl;
    }
}

// Groups of four one-form records per pass (NW = 1) cost instruction-cache
// misses in the term-parallel dedup_eval_kernel (16 warps walking different
// segments); pairs keep the hot loop small.
#ifndef ZXS_MONO_QUAD
#define ZXS_MONO_QUAD 0
#endif
constexpr bool kMonoQuad = ZXS_MONO_QUAD != 0;

// One-form records, forms of four (NW = 1, kMonoQuad) or two records formed
// together (independent shared loads in flight), then applied by kind.
#define ZXS_MONO_RUN(N, OP)                                                              \
    {                                                                                    \
        uint32_t i_ = 0;                                                                 \
        if constexpr (NW == 1 && kMonoQuad) {                                            \
            for (; i_ + 4 <= (N); i_ += 4) {                                             \
                const uint32_t r0_ = w[q + i_], r1_ = w[q + i_ + 1];                     \
                const uint32_t r2_ = w[q + i_ + 2], r3_ = w[q + i_ + 3];                 \
                const BW<NW> x0 = mono_form<NW>(sd, r0_ & kFormMask, pl);                   \
                const BW<NW> x1 = mono_form<NW>(sd, r1_ & kFormMask, pl);                   \
                const BW<NW> x2 = mono_form<NW>(sd, r2_ & kFormMask, pl);                   \
                const BW<NW> x3 = mono_form<NW>(sd, r3_ & kFormMask, pl);                   \
                OP(r0_, x0);                                                             \
                OP(r1_, x1);                                                             \
                OP(r2_, x2);                                                             \
                OP(r3_, x3);                                                             \
            }                                                                            \
        } else {                                                                         \
            for (; i_ + 2 <= (N); i_ += 2) {                                             \
                const uint32_t r0_ = w[q + i_], r1_ = w[q + i_ + 1];                     \
                const uint32_t fa_ = r0_ & kFormMask, fb_ = r1_ & kFormMask;                   \
                const uint4 ea_ = sd[fa_], eb_ = sd[fb_];                                \
                BW<NW> x0, x1;                                                           \
                if (((ea_.x ^ eb_.x) & 0x87u) == 0 && (ea_.x & 0x87u) <= kPairMaxCls) {  \
                    mono_entry2<NW>(ea_, eb_, pl, x0, x1);                               \
                } else {                                                                 \
                    x0 = mono_form<NW>(sd, fa_, pl);                                     \
                    x1 = mono_form<NW>(sd, fb_, pl);                                     \
                }                                                                        \
                OP(r0_, x0);                                                             \
                OP(r1_, x1);                                                             \
            }                                                                            \
        }                                                                                \
        for (; i_ < (N); i_++) {                                                         \
            const uint32_t r0_ = w[q + i_];                                              \
            const BW<NW> x0 = mono_form<NW>(sd, r0_ & kFormMask, pl);                       \
            OP(r0_, x0);                                                                 \
        }                                                                                \
        q += (N);                                                                        \
    }
#define ZXS_OP_ADD(x) { j1 = bw_xor<NW>(j1, bw_and<NW>(j0, x)); j0 = bw_xor<NW>(j0, x); }
// op of a record word r on (Z, J0, J1): the kind is warp-uniform (one uniform branch)
#define ZXS_OP_KIND(r, x)                  \
    switch ((r) >> 28) {                   \
        case kRecAdd: ZXS_OP_ADD(x); break; \
        case kRecSub: ZXS_OP_SUB(x); break; \
        case kRecAdd2: ZXS_OP_ADD2(x); break; \
        case kRecZ: ZXS_OP_Z(x); break;     \
        default: ZXS_OP_ZN(x); break;       \
    }
#define ZXS_OP_SUB(x) { j1 = bw_xor<NW>(j1, bw_andn<NW>(j0, x)); j0 = bw_xor<NW>(j0, x); }
#define ZXS_OP_ADD2(x) { j1 = bw_xor<NW>(j1, x); }
#define ZXS_OP_Z(x) { z = bw_or<NW>(z, x); }
#define ZXS_OP_ZN(x) { z = bw_or<NW>(z, bw_not<NW>(x)); }
#define ZXS_OP_ANY(r, x) ZXS_OP_KIND(r, x)

// Leaf epilogue: acc[s] += Re(c' i^J) = {re, -im, -re, im}[J] for the non-zero
// shots, in term order; the sign is a flip of the high word's sign bit.
template <int NW>
__device__ __forceinline__ void mono_leaf(double (&acc)[32 * NW], const BW<NW> &z, const BW<NW> &j0, const BW<NW> &j1,
                                          double re, double im) {
    const uint32_t re_lo = uint32_t(__double2loint(re)), re_hi = uint32_t(__double2hiint(re));
    const uint32_t im_lo = uint32_t(__double2loint(im)), im_hi = uint32_t(__double2hiint(im));
#pragma unroll
    for (int i = 0; i < NW; i++) {
        const uint32_t neg = j0.w[i] ^ j1.w[i];
#pragma unroll
        for (int s = 0; s < 32; s++) {
            const bool odd = (j0.w[i] >> s) & 1u;
            const uint32_t lo = odd ? im_lo : re_lo;
            const uint32_t hi = (odd ? im_hi : re_hi) ^ ((neg << (31 - s)) & 0x80000000u);
            if (!((z.w[i] >> s) & 1u)) {
                acc[i * 32 + s] = __dadd_rn(acc[i * 32 + s], __hiloint2double(int(hi), int(lo)));
            }
        }
    }
}

// Walks `nnodes` nodes of a record stream (node layout in zxs_api.cu
// encode_mono) on top of the per-level (Z, J0, J1) stack `stk`; leaves add
// Re(c' i^J) of their non-zero shots to acc. FOLD: a node flagged
// kMonoSegStart first folds the running segment sum into tot (tot += acc,
// acc = 0), so the tensor value is the canonical
//   ((0 + S_0) + S_1) + ... + S_{G-1},   S_k = segment k's terms in order
// that the deduplicated path (zxs_dedup.cuh) computes segment by segment.
template <int NW, bool FOLD>
__device__ __forceinline__ void mono_walk(const uint32_t *w, uint32_t nnodes, const uint4 *sd, const char *pl,
                                          BW<NW> *stk, double (&acc)[32 * NW], double *tot) {
    uint32_t q = 0;
    for (uint32_t nn = 0; nn < nnodes; nn++) {
        // node: {leaf << 31 | seg_start << 30 | depth << 24 | n_gen, n_add | n_sub << 8 | n_add2 << 16 | n_z << 24,
        // n_zn} [re, im], records grouped by kind
        const uint32_t h0 = w[q], h1 = w[q + 1], h2 = w[q + 2];
        const uint32_t depth = (h0 >> 24) & 0x3fu;
        const bool leaf = (h0 >> 31) != 0;
        if (FOLD && (h0 & kMonoSegStart)) {
            // eight at a time (compiler barriers keep the loads from being hoisted
            // together: the accumulators already fill the register file)
#pragma unroll
            for (int g = 0; g < 4 * NW; g++) {
                asm volatile("" ::: "memory");
                double t[8];
#pragma unroll
                for (int s = 0; s < 8; s++) t[s] = tot[8 * g + s];
#pragma unroll
                for (int s = 0; s < 8; s++) {
                    tot[8 * g + s] = __dadd_rn(t[s], acc[8 * g + s]);
                    acc[8 * g + s] = 0.0;
                }
            }
            asm volatile("" ::: "memory");
        }
        q += 3;
        double re = 0.0, im = 0.0;
        if (leaf) {
            re = __hiloint2double(int(w[q + 1]), int(w[q]));
            im = __hiloint2double(int(w[q + 3]), int(w[q + 2]));
            q += 4;
        }
        // state of the parent (depth - 1), or the empty product at the root
        BW<NW> z = bw_zero<NW>(), j0 = bw_zero<NW>(), j1 = bw_zero<NW>();
        if (depth) {
            const BW<NW> *ps = stk + (depth - 1) * 96;
            z = ps[0];
            j0 = ps[32];
            j1 = ps[64];
        }
        {
            // one-form records (any kind, ordered by size class): one copy of the
            // form code for all kinds keeps the kernel within the instruction cache
            const uint32_t ns = (h1 & 0xffu) + ((h1 >> 8) & 0xffu) + ((h1 >> 16) & 0xffu) + (h1 >> 24) + (h2 & 0xffu);
            ZXS_MONO_RUN(ns, ZXS_OP_ANY)
        }
        for (uint32_t g = 0; g < (h0 & 0xffu); g++) {  // two-form records
            const uint32_t r = w[q], gw = w[q + 1];
            q += 2;
            const uint32_t fa = r & kFormMask, fb = (r >> kFormShiftB) & kFormMask;
            const BW<NW> a = fa == kMonoNoForm ? bw_zero<NW>() : mono_form<NW>(sd, fa, pl);
            const BW<NW> bb = fb == kMonoNoForm ? bw_zero<NW>() : mono_form<NW>(sd, fb, pl);
            const uint32_t zl = gw >> 6;
#pragma unroll
            for (int i = 0; i < NW; i++) {
                z.w[i] |= ((zl & 1u) ? (~a.w[i] & ~bb.w[i]) : 0u) | ((zl & 2u) ? (~a.w[i] & bb.w[i]) : 0u) |
                          ((zl & 4u) ? (a.w[i] & ~bb.w[i]) : 0u) | ((zl & 8u) ? (a.w[i] & bb.w[i]) : 0u);
            }
            j_add<NW>(j0, j1, a, gw & 3u);
            j_add<NW>(j0, j1, bb, (gw >> 2) & 3u);
            j_add<NW>(j0, j1, bw_and<NW>(a, bb), (gw >> 4) & 3u);
        }
        if (!leaf) {
            BW<NW> *ns = stk + depth * 96;
            ns[0] = z;
            ns[32] = j0;
            ns[64] = j1;
            continue;
        }
        mono_leaf<NW>(acc, z, j0, j1, re, im);
    }
}

// KW warps per CTA: MonoCfg's, or 4 (the narrow variant, for components whose
// dictionary and parameter planes do not fit the wide CTA's shared memory).
template <int NW, int KW = MonoCfg<NW>::kWarps>
__global__ void __launch_bounds__(KW * 32, 1) mono_kernel(const __grid_constant__ MonoArgs h) {
    constexpr int kW = KW;
    constexpr uint32_t kLaneShots = 32 * NW;
    constexpr uint64_t kWarpShots = 32ull * kLaneShots;
    extern __shared__ __align__(128) uint8_t msm[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(msm);
    uint32_t *buf0 = reinterpret_cast<uint32_t *>(msm + 128);
    uint4 *sd = reinterpret_cast<uint4 *>(buf0 + 2 * kMonoChunkWords);  // the current tensor's dictionary
    // per warp: stack [depth][z, j0, j1][lane][NW], planes [p][lane][NW]
    uint32_t *stack_all = reinterpret_cast<uint32_t *>(sd + h.max_dict);
    uint32_t *planes_all = stack_all + kW * h.stack_depth * 3 * 32 * NW;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    BW<NW> *stk = reinterpret_cast<BW<NW> *>(stack_all + warp * h.stack_depth * 3 * 32 * NW) + lane;
    uint32_t *planes = planes_all + warp * h.n_planes * 32 * NW;  // [p][lane][NW]
    BW<NW> *myplanes = reinterpret_cast<BW<NW> *>(planes) + lane;  // plane p at myplanes[p * 32]
    const char *pl = reinterpret_cast<const char *>(myplanes);

    // chunk uses per CTA tile: every tensor of every component (or the one eval tensor)
    uint32_t chunks_per_tile = 0;
    if (h.eval_tensor >= 0) {
        chunks_per_tile = h.tensor_chunk_begin[h.eval_tensor + 1] - h.tensor_chunk_begin[h.eval_tensor];
    } else {
        for (uint32_t hc = 0; hc < h.n_comps; hc++) {
            const HeavyComp cd = h.comps[hc];
            chunks_per_tile += h.tensor_chunk_begin[cd.first_tensor + cd.n_out + 1] - h.tensor_chunk_begin[cd.first_tensor];
        }
    }
    const uint64_t my_tiles = blockIdx.x < h.n_cta_tiles ? (h.n_cta_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const uint64_t total_uses = my_tiles * chunks_per_tile;
    // chunk sequence of use u: tile-major, then tensors in chain order
    auto chunk_of_use = [&](uint64_t u) -> uint32_t {
        uint32_t r = uint32_t(u % chunks_per_tile);
        if (h.eval_tensor >= 0) return h.tensor_chunk_begin[h.eval_tensor] + r;
        for (uint32_t hc = 0; hc < h.n_comps; hc++) {
            const HeavyComp cd = h.comps[hc];
            const uint32_t c0 = h.tensor_chunk_begin[cd.first_tensor];
            const uint32_t n = h.tensor_chunk_begin[cd.first_tensor + cd.n_out + 1] - c0;
            if (r < n) return c0 + r;
            r -= n;
        }
        return 0;
    };
    auto issue = [&](uint64_t u) {
        const uint4 c = h.chunks[chunk_of_use(u)];
        const uint32_t b = uint32_t(u & 1);
        mbar_expect_tx(&bars[b], c.y * 4u);
        bulk_g2s(buf0 + b * kMonoChunkWords, h.words + c.x, c.y * 4u, &bars[b]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint64_t u = 0; u < 2 && u < total_uses; u++) issue(u);
    }
    const uint32_t seed_hi = uint32_t(h.seed >> 32);
    const uint32_t k2c = uint32_t(kP1c) ^ h.k0_round[1];
    uint64_t use = 0;

    for (uint64_t ct = blockIdx.x; ct < h.n_cta_tiles; ct += gridDim.x) {
        // the lane's NW consecutive 32-shot words: wrd .. wrd + NW - 1
        const uint64_t wrd = ((ct * kW + warp) * 32 + lane) * NW;
        for (uint32_t p = h.all_plane + 1; p < h.n_planes; p++) myplanes[p * 32] = bw_zero<NW>();  // ZERO, sampled bits
        __syncwarp();
        double *prev_g = h.scratch + wrd * 32;
        double *cur_g = h.scratch + (h.n_cta_tiles * kW * kWarpShots) + wrd * 32;
        double *tot_g = h.scratch + 2 * (h.n_cta_tiles * kW * kWarpShots) + wrd * 32;  // folded segment sums

        const uint32_t ncomp = h.eval_tensor >= 0 ? 1u : h.n_comps;
        for (uint32_t hc = 0; hc < ncomp; hc++) {
            const HeavyComp cd = h.comps[h.eval_tensor >= 0 ? h.eval_comp : hc];
            const uint32_t npos = h.eval_tensor >= 0 ? 1u : cd.n_out + 1;
            for (uint32_t pos = 0; pos < npos; pos++) {  // pos 0: normalization, pos j+1: marginal j
                const uint32_t t = h.eval_tensor >= 0 ? uint32_t(h.eval_tensor) : cd.first_tensor + pos;
                // this tensor's basis planes from the raw parameters (f columns from the
                // shot kernel's scratch, sampled bits so far from shared memory), and ALL
                {
                    const uint32_t W = min(h.tensor_width[t], h.all_plane);
                    const unsigned long long *bv = h.basis + h.tensor_basis_begin[t];
                    BW<NW> all = bw_zero<NW>();
                    for (uint32_t b = 0; b < W; b++) {
                        BW<NW> v = bw_zero<NW>();
                        for (unsigned long long x = bv[b]; x; x &= x - 1) {
                            const uint32_t p = __ldg(h.param_map + cd.pmap_begin + __ffsll((long long)x) - 1);  // raw
                            BW<NW> r;
                            if (p < h.f_width) {
#pragma unroll
                                for (int i = 0; i < NW; i++) {
                                    r.w[i] = wrd + i < h.fcols_ld32 ? __ldg(h.fcols + p * h.fcols_ld32 + wrd + i) : 0u;
                                }
                            } else {
                                r = myplanes[(h.all_plane + 2 + (p - h.f_width)) * 32];
                            }
                            v = bw_xor<NW>(v, r);
                        }
                        myplanes[b * 32] = v;
                        all = bw_xor<NW>(all, v);
                    }
                    myplanes[h.all_plane * 32] = all;
                }
                // stage the tensor's form dictionary (every warp is past the previous tensor)
                {
                    const uint32_t d0 = h.tensor_dict_begin[t], nd = h.tensor_dict_begin[t + 1] - d0;
                    for (uint32_t i = threadIdx.x; i < nd; i += blockDim.x) sd[i] = __ldg(h.dict + d0 + i);
                    __syncthreads();
                }
                double acc[kLaneShots];
#pragma unroll
                for (int s = 0; s < int(kLaneShots); s++) {
                    acc[s] = 0.0;
                    tot_g[s] = 0.0;
                }
                for (uint32_t c = h.tensor_chunk_begin[t]; c < h.tensor_chunk_begin[t + 1]; c++, use++) {
                    const uint32_t b = uint32_t(use & 1);
                    mbar_wait(&bars[b], uint32_t((use >> 1) & 1));
                    const uint32_t *w = buf0 + b * kMonoChunkWords;
#ifdef ZXS_MONO_NOFOLD  // A/B timing only: not the canonical order
                    mono_walk<NW, false>(w, h.chunks[c].z, sd, pl, stk, acc, tot_g);
#else
                    mono_walk<NW, true>(w, h.chunks[c].z, sd, pl, stk, acc, tot_g);
#endif
                    __syncthreads();  // buffer b fully consumed by every warp
                    if (threadIdx.x == 0 && use + 2 < total_uses) issue(use + 2);
                }
#pragma unroll
                for (int g = 0; g < int(kLaneShots) / 8; g++) {  // last segment, eight at a time
                    asm volatile("" ::: "memory");
                    double t[8];
#pragma unroll
                    for (int s = 0; s < 8; s++) t[s] = tot_g[8 * g + s];
#pragma unroll
                    for (int s = 0; s < 8; s++) acc[8 * g + s] = __dadd_rn(t[s], acc[8 * g + s]);
                }
                asm volatile("" ::: "memory");
                if (h.eval_tensor >= 0) {
#pragma unroll
                    for (int s = 0; s < int(kLaneShots); s++) {
                        if (wrd * 32 + s < h.shots) h.eval_out[wrd * 32 + s] = acc[s];
                    }
                    continue;
                }
                if (pos == 0) {
#pragma unroll
                    for (int s = 0; s < int(kLaneShots); s++) prev_g[s] = acc[s];
                    continue;
                }
#pragma unroll
                for (int s = 0; s < int(kLaneShots); s++) cur_g[s] = acc[s];
                // autoregressive draw of output pos-1 (sampler.cpp:84-99), one shot at a time
                const uint32_t j = pos - 1;
                const uint32_t stream = 0x80000000u ^ (cd.ci << 12) ^ j;  // sampler.cpp:37-39
                BW<NW> word = bw_zero<NW>();
                for (uint32_t s = 0; s < kLaneShots; s++) {
                    const uint64_t local = wrd * 32 + s;
                    const bool valid = local < h.shots;
                    const double cur = cur_g[s], pv = prev_g[s];
                    const double ratio = __ddiv_rn(cur, pv);
                    if (!(ratio > -1e-6 && ratio < 1.0 + 1e-6) && valid) report_ratio_error(h.err, h.first_shot + local);
                    double cl = (0.0 < ratio) ? ratio : 0.0;
                    cl = (cl < 1.0) ? cl : 1.0;
                    double u;
                    if (h.uniforms) {
                        u = valid ? h.uniforms[(cd.upos_base + j) * h.uniforms_ld + local] : 0.0;
                    } else {
                        const uint64_t shot = h.first_shot + local;
                        PhiloxPre pre[1] = {philox_pre(uint32_t(shot), uint32_t(shot >> 32), h.k0_round[0])};
                        uint32_t rhi[1], rlo[1];
                        philox_tail<1>(pre, seed_hi ^ stream, h.k0_round, k2c, h.k0_round[9], rhi, rlo);
                        u = philox_uniform((uint64_t(rhi[0]) << 32) | rlo[0]);
                    }
                    if (valid) count_near_tie(h.err, u, cl);
                    const bool bit = !(u < cl) && valid;
                    prev_g[s] = bit ? __dsub_rn(pv, cur) : cur;
#pragma unroll
                    for (int i = 0; i < NW; i++) {
                        if ((s >> 5) == uint32_t(i)) word.w[i] |= uint32_t(bit) << (s & 31);
                    }
                }
                myplanes[(h.all_plane + 2 + j) * 32] = word;
                const uint32_t o = h.comp_outputs[cd.out_begin + j];
#pragma unroll
                for (int i = 0; i < NW; i++) {
                    // bounded by this batch's record words (out_ld32 is the row stride)
                    if (h.out32 && wrd + i < min(h.out_ld32, 2 * ((h.shots + 63) / 64))) {
                        h.out32[o * h.out_ld32 + wrd + i] = word.w[i];
                    }
                }
                if (h.counts) {
                    uint32_t ones = 0;
#pragma unroll
                    for (int i = 0; i < NW; i++) ones += __popc(word.w[i]);
                    ones = __reduce_add_sync(kFull, ones);
                    if (lane == 0 && ones) atomicAdd(&h.counts[o], (unsigned long long)ones);
                }
                __syncwarp();
            }
            // reset this component's sampled-bit planes for the next component
            if (h.eval_tensor < 0) {
                for (uint32_t j = 0; j < cd.n_out; j++) myplanes[(h.all_plane + 2 + j) * 32] = bw_zero<NW>();
            }
            __syncwarp();
        }
    }
}

}  // namespace zxs_dev
