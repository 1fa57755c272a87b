// zxs_sparse.cuh — the reference's sparse geometric sampler on the device.
//
// For pure-Clifford deterministic models whose mechanisms are all singles
// with p < 1 and few expected flips per shot, the reference does not draw
// every mechanism per shot: it draws, per mechanism m, the gaps between
// firing shots from RngStream(seed, m) (sampler.cpp:214-255):
//   gap_k = floor(log(u_k) / log1p(-p)),  u_k = Philox(seed, m).uniform_at(k)
//   event_k = sum_{j<k} (gap_j + 1) + gap_k,  while event_k < shots
// and XORs each event into the outputs mechanism m flips (cs.flips,
// compile.cpp:285-303). The gaps are independent given k, so one CTA per
// mechanism computes 256 of them at a time, prefix-sums (gap + 1) across the
// block to place the events, and XORs them into the record with 64-bit
// atomics. log1p(-p) comes from the host (the reference's libm value); log(u)
// is CUDA's double log (<= 1 ulp): a floor can only differ when log(u)/log1p
// lands within an ulp of an integer.
#pragma once

#include "zxs_kernels.cuh"

namespace zxs_dev {

constexpr int kSparseThreads = 256;

struct SparseArgs {
    uint64_t seed, shots, words;
    uint32_t num_mech;
    const double *log1mp;        // [num_mech] log1p(-p); +0.0 for p <= 0 (no events)
    const uint32_t *flip_begin;  // [num_mech + 1] CSR of flipped outputs
    const uint32_t *flip_out;
    unsigned long long *cols;    // [num_outputs][words]
};

__global__ void __launch_bounds__(kSparseThreads) sparse_kernel(const __grid_constant__ SparseArgs a) {
    __shared__ unsigned long long warp_tot[kSparseThreads / 32];
    __shared__ unsigned long long carry;
    const uint32_t m = blockIdx.x;
    if (m >= a.num_mech) return;
    const double l1mp = a.log1mp[m];
    const uint32_t f0 = a.flip_begin[m], f1 = a.flip_begin[m + 1];
    if (!(l1mp < 0.0) || f0 == f1) return;  // p <= 0: no events (sampler.cpp:222-224); nothing flipped
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t k0s = uint32_t(a.seed), k1s = uint32_t(a.seed >> 32) ^ m;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (uint64_t k = tid;; k += kSparseThreads) {
        double u = philox_uniform(philox_r01(k0s, k1s, uint32_t(k), uint32_t(k >> 32)));
        if (u <= 0.0) u = 2.2250738585072014e-308;  // numeric_limits<double>::min() (sampler.cpp:230-232)
        const double g = floor(log(u) / l1mp);
        // gap + 1 as an integer, clamped at 2^40 (> any shot count the host admits)
        const unsigned long long step = (g >= 1099511627776.0 ? 1099511627776ull : (unsigned long long)g) + 1ull;
        // inclusive block scan of step
        unsigned long long x = step;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(kFull, x, o);
            if (lane >= uint32_t(o)) x += y;
        }
        if (lane == 31) warp_tot[warp] = x;
        __syncthreads();
        unsigned long long before = carry;
        for (uint32_t w = 0; w < warp; w++) before += warp_tot[w];
        const unsigned long long incl = before + x;  // = event + 1
        const unsigned long long event = incl - 1;
        if (event < a.shots) {
            for (uint32_t i = f0; i < f1; i++) {
                atomicXor(&a.cols[uint64_t(a.flip_out[i]) * a.words + (event >> 6)], 1ull << (event & 63));
            }
        }
        __syncthreads();
        if (tid == kSparseThreads - 1) carry = incl;
        __syncthreads();
        if (carry >= a.shots) break;  // every later event lies beyond the record
        __syncthreads();
    }
}

}  // namespace zxs_dev
