// zxs_device.cuh — device-side building blocks of the sm_100a shot sampler.
//
// Layout in HBM (built once by zxs_sampler_create, see zxs_api.cu):
//   * mechanism scan entries  (one per reachable table outcome)    u64 lim + u32 flip id
//   * flip masks              (FW u64 words per distinct flip set) f-space XOR masks
//   * direct outputs          CSR over f indices
//   * chain tensors           terms (c as double2, factor range) and factors
//                             (selector range + h-table id), selectors u16
//   * h tables                double2[4] per distinct table
// Per shot, the f register file lives in FW u64 registers of the lane that
// owns the shot (lane = shot within a 32-shot tile); after the draw it is
// transposed into 32-shot bit-sliced columns in shared memory, which is the
// reference's ParamBatch layout (phase_terms.hpp:64-73) at 32 shots per word.
#pragma once

#include <cstdint>

namespace zxs_dev {

constexpr uint32_t kNoFlip = 0xffffffffu;
constexpr uint32_t kFull = 0xffffffffu;

// ---------------------------------------------------------------- Philox
// Philox4x32-10 as in proj/include/zxsim/rng.hpp:25-71: key = {seed_lo,
// seed_hi ^ stream}, ctr = {idx_lo, idx_hi, 0x9e3779b9, 0}; returns the
// 64-bit (r0 << 32 | r1) whose top 53 bits are the reference's uniform_at
// mantissa (rng.hpp:35-37). Only r0/r1 are live after round 10, so the last
// round's second product is dead code.
__device__ __forceinline__ uint64_t philox_r01(uint32_t k0, uint32_t k1, uint32_t idx_lo,
                                               uint32_t idx_hi) {
    uint32_t c0 = idx_lo, c1 = idx_hi, c2 = 0x9e3779b9u, c3 = 0u;
#pragma unroll
    for (int i = 0; i < 10; i++) {
        uint64_t p0 = uint64_t(0xD2511F53u) * c0;
        uint64_t p1 = uint64_t(0xCD9E8D57u) * c2;
        uint32_t n0 = uint32_t(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = uint32_t(p1);
        uint32_t n2 = uint32_t(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = uint32_t(p0);
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return (uint64_t(c0) << 32) | c1;
}

// uniform_at (rng.hpp:37): (r >> 11) * 2^-53, exact in double.
__device__ __forceinline__ double philox_uniform(uint64_t r) {
    return __ull2double_rn(r >> 11) * 0x1.0p-53;
}

// ---------------------------------------------------------------- complex
// std::complex<double> operator*= / += as GCC emits them without FMA
// contraction (the reference is built for baseline x86-64): re = ac - bd,
// im = ad + bc, every product and sum rounded separately. The _rn
// intrinsics keep nvcc from fusing them, so the device reproduces the
// reference's eval_batch (phase_terms.cpp:121-131) bit for bit.
__device__ __forceinline__ double2 cmul_rn(double2 x, double2 h) {
    double2 r;
    r.x = __dsub_rn(__dmul_rn(x.x, h.x), __dmul_rn(x.y, h.y));
    r.y = __dadd_rn(__dmul_rn(x.x, h.y), __dmul_rn(x.y, h.x));
    return r;
}

__device__ __forceinline__ double2 cadd_rn(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

// ---------------------------------------------------------------- bits
// In-register 32x32 bit transpose across a warp: on entry lane i holds row
// i (bit j = element (i, j)); on exit lane j holds column j (bit i).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, uint32_t lane) {
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int st = 0; st < 5; st++) {
        const uint32_t s = 16u >> st;
        const uint32_t m = masks[st];
        uint32_t p = __shfl_xor_sync(kFull, x, s);
        x = (lane & s) ? ((x & ~m) | ((p & ~m) >> s)) : ((x & m) | ((p & m) << s));
    }
    return x;
}

// ---------------------------------------------------------------- model
struct Factor {
    uint32_t sel;    // first selector (u list, then v list) in `selectors`
    uint16_t nu, nv; // |u_k|, |v_k|
    uint32_t table;  // h-table id
    uint32_t pad;
};

struct DevModel {
    uint32_t f_width, fw, num_outputs, num_mech, num_direct, num_components, max_chain;
    uint32_t col_stride;  // smem words per warp (>= f_width rounded to 32 + max_chain)
    // error model
    const uint32_t *mech_entry_begin;  // [num_mech+1]
    const uint32_t *mech_stream;       // [num_mech] Philox stream (reference index m)
    const uint64_t *entry_lim;         // fire iff (r01 <= lim)
    const uint32_t *entry_flip;        // flip set id or kNoFlip
    const uint64_t *flip_mask;         // [num_flipsets * fw]
    const uint64_t *base_offset;       // [fw]
    // direct outputs
    const uint32_t *direct_out;        // [num_direct] output | (flip_const << 31)
    const uint32_t *direct_bit_begin;  // [num_direct+1]
    const uint32_t *direct_bits;
    // components
    const uint32_t *comp_out_begin;    // [num_components+1]
    const uint32_t *comp_outputs;
    const uint32_t *comp_tensor_begin; // [num_components+1]
    // tensors
    const uint32_t *tensor_term_begin; // [num_tensors+1]
    const double2 *term_c;
    const uint32_t *term_factor_begin; // [num_terms+1]
    const Factor *factors;
    const uint16_t *selectors;
    const double2 *h_table;            // [4 * num_tables]
    const uint8_t *comp_heavy;         // [num_components] 1: chain runs in heavy_kernel
};

}  // namespace zxs_dev
