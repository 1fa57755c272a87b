// zxs_dedup.cuh — large-chi components evaluated once per distinct parameter
// vector of a batch.
//
// A chain tensor's value is a pure function of the shot's raw parameters
// (phase_terms.cpp:90-144: the f bits and the outputs sampled so far). At
// the noise rates of every BASELINE circuit those vectors repeat massively:
// on the d=3 cultivation proxy 97.8 % of shots have f = 0 and 2^20 shots carry
// 338 distinct f vectors. Per chain position the path therefore
//   1. hashes each shot's key (its raw parameter bits restricted to the ones
//      the component's tensors read) into an open-addressing table, giving
//      the batch's U distinct keys (dedup_init_kernel / dedup_ar_kernel);
//   2. contracts the tensor for those U keys only, term-parallel: the
//      tensor's terms are cut into G fixed summation segments (host,
//      encode_mono), a warp walks one segment for 1024 keys (mono_walk,
//      the same record code as mono_kernel) and writes the segment sums
//      (dedup_eval_kernel);
//   3. folds the segment sums in order, ((0 + S_0) + S_1) + ... + S_{G-1}
//      (dedup_reduce_kernel) -- the same canonical order mono_kernel uses
//      per shot, so both paths give bit-identical values and a shot's value
//      does not depend on which other shots share its batch;
//   4. runs the autoregressive draw per shot (sampler.cpp:84-99) with the
//      value looked up by key, and inserts the extended key (plus the new
//      bit) for the next tensor (dedup_ar_kernel).
// Every step is recomputed per batch (nothing is cached across calls).
#pragma once

#include "zxs_mono.cuh"

namespace zxs_dev {

constexpr unsigned long long kDedupEmpty = ~0ull;  // keys use at most 63 raw parameter bits
constexpr int kDedupWarps = 16;                    // dedup_eval_kernel: warps per CTA (one segment each)
constexpr uint32_t kDedupKeysPerWarp = 1024;       // 32 keys per lane (NW = 1)

struct DedupTable {
    unsigned long long *keys;  // [mask + 1], kDedupEmpty when free
    uint32_t *ids;             // [mask + 1] dense id of the key in the slot
    uint32_t mask;
    uint32_t max_ids;          // ukeys / uslot capacity; more keys = overflow (host falls back)
    uint32_t *count;           // distinct keys inserted
    unsigned long long *ukeys; // [id] key
    uint32_t *uslot;           // [id] slot (for clearing)
};

__device__ __forceinline__ uint32_t dedup_hash(unsigned long long k, uint32_t mask) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return uint32_t(k) & mask;
}

// Insert (or find) `key`; returns its slot. Plain loads first: the hot keys
// are found without atomics.
__device__ __forceinline__ uint32_t dedup_insert(const DedupTable &t, unsigned long long key) {
    uint32_t slot = dedup_hash(key, t.mask);
    while (true) {
        if (*reinterpret_cast<volatile uint32_t *>(t.count) >= t.max_ids) return 0;  // overflow: batch falls back
        const unsigned long long k = *reinterpret_cast<volatile unsigned long long *>(&t.keys[slot]);
        if (k == key) return slot;
        if (k == kDedupEmpty) {
            const unsigned long long old = atomicCAS(&t.keys[slot], kDedupEmpty, key);
            if (old == kDedupEmpty) {
                const uint32_t id = atomicAdd(t.count, 1u);
                if (id < t.max_ids) {
                    t.ids[slot] = id;
                    t.ukeys[id] = key;
                    t.uslot[id] = slot;
                }
                return slot;
            }
            if (old == key) return slot;
        }
        slot = (slot + 1) & t.mask;
    }
}

// Per-warp cache of recent (key, slot) pairs, one pair per lane (lanes 0..7
// used): the key distribution is extremely skewed (most shots carry the
// all-zero key), so most shots resolve here instead of hammering one table
// line in L2.
struct DedupWarpCache {
    unsigned long long key = kDedupEmpty;
    uint32_t slot = 0;
    uint32_t next = 0;  // round-robin victim (warp-uniform)
};
constexpr uint32_t kDedupCacheWays = 8;

// Warp-cooperative insert: cache lookup, then one table insert per distinct
// missing key of the warp.
__device__ __forceinline__ uint32_t dedup_insert_warp(const DedupTable &t, unsigned long long key, bool valid,
                                                      uint32_t lane, DedupWarpCache &c) {
    const unsigned long long k = valid ? key : kDedupEmpty;
    uint32_t slot = 0;
    bool hit = !valid;
#pragma unroll
    for (uint32_t i = 0; i < kDedupCacheWays; i++) {
        const unsigned long long ck = __shfl_sync(kFull, c.key, i);
        const uint32_t cs = __shfl_sync(kFull, c.slot, i);
        if (!hit && ck == k) {
            hit = true;
            slot = cs;
        }
    }
    const uint32_t miss = __ballot_sync(kFull, !hit);
    if (miss) {
        const uint32_t peers = __match_any_sync(kFull, hit ? kDedupEmpty : k);
        const uint32_t leader = __ffs(peers) - 1;
        uint32_t ns = 0;
        if (!hit && lane == leader) ns = dedup_insert(t, k);
        ns = __shfl_sync(kFull, ns, leader);
        if (!hit) slot = ns;
        // the first missing key enters the cache
        const uint32_t first = __ffs(miss) - 1;
        const unsigned long long fk = __shfl_sync(kFull, k, first);
        const uint32_t fs = __shfl_sync(kFull, slot, first);
        if (lane == c.next) {
            c.key = fk;
            c.slot = fs;
        }
        c.next = (c.next + 1) % kDedupCacheWays;
    }
    return slot;
}

struct DedupInitArgs {
    uint64_t shots;
    const uint32_t *fcols;  // [f_width][fcols_ld32]
    uint64_t fcols_ld32;
    uint32_t n_bits;          // f columns the component's tensors read
    uint8_t bits[64];
    unsigned long long *key;  // [shots]
    uint32_t *slot;           // [shots]
    DedupTable table;
};

// Keys of the chain's first tensors (no sampled bits yet): thread = shot,
// the warp's 32 shots share every f-column word (broadcast loads).
__global__ void __launch_bounds__(256) dedup_init_kernel(const __grid_constant__ DedupInitArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    DedupWarpCache cache;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t s0 = uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); s0 < a.shots; s0 += stride) {
        const uint64_t s = s0 + lane, wd = s0 >> 5;
        const bool valid = s < a.shots;
        unsigned long long key = 0;
        for (uint32_t i0 = 0; i0 < a.n_bits; i0 += 16) {  // 16 column loads in flight
            uint32_t wv[16];
#pragma unroll
            for (uint32_t i = 0; i < 16; i++) {
                wv[i] = i0 + i < a.n_bits ? __ldg(a.fcols + a.bits[i0 + i] * a.fcols_ld32 + wd) : 0u;
            }
#pragma unroll
            for (uint32_t i = 0; i < 16; i++) {
                if (i0 + i < a.n_bits) key |= (unsigned long long)((wv[i] >> lane) & 1u) << a.bits[i0 + i];
            }
        }
        const uint32_t slot = dedup_insert_warp(a.table, key, valid, lane, cache);
        if (valid) {
            a.key[s] = key;
            a.slot[s] = slot;
        }
    }
}

struct DedupEvalArgs {
    const uint32_t *words;  // segment streams
    const uint4 *segs;      // this tensor's segments {word_begin, n_words, n_nodes, 0}
    uint32_t n_segs;
    const uint4 *dict;      // this tensor's dictionary
    uint32_t n_dict;
    const unsigned long long *basis;  // this tensor's W basis vectors (masks over raw params)
    uint32_t width;                   // W
    uint32_t all_plane, n_planes;     // plane indices the dictionary uses: [0, W), ALL, ZERO = ALL + 1
    uint32_t stack_depth;
    const unsigned long long *keys;   // the round's keys
    uint32_t n_keys;
    double *partial;                  // [n_segs][n_keys]
    uint32_t seg_buf_words;           // per-warp shared-memory copy of its segment (0: walk from global)
};

// Items = (key group of 1024, block of kDedupWarps segments); a CTA builds the
// key group's parameter planes once in shared memory (shared by its warps),
// every warp walks one segment for all 1024 keys.
__global__ void __launch_bounds__(kDedupWarps * 32, 1) dedup_eval_kernel(const __grid_constant__ DedupEvalArgs h) {
    extern __shared__ __align__(128) uint8_t dsm[];
    uint4 *sd = reinterpret_cast<uint4 *>(dsm);
    uint32_t *planes = reinterpret_cast<uint32_t *>(sd + h.n_dict);  // [p][lane]
    uint32_t *stack_all = planes + h.n_planes * 32;                  // per warp [depth][3][lane]
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    BW<1> *stk = reinterpret_cast<BW<1> *>(stack_all + warp * h.stack_depth * 96) + lane;
    uint32_t *segbuf = stack_all + kDedupWarps * h.stack_depth * 96 + warp * h.seg_buf_words;
    uint32_t have_seg = 0xffffffffu;  // segment currently in segbuf
    const char *pl = reinterpret_cast<const char *>(planes + lane);

    for (uint32_t i = threadIdx.x; i < h.n_dict; i += blockDim.x) sd[i] = __ldg(h.dict + i);
    const uint32_t n_kg = (h.n_keys + kDedupKeysPerWarp - 1) / kDedupKeysPerWarp;
    const uint32_t n_blk = (h.n_segs + kDedupWarps - 1) / kDedupWarps;
    const uint64_t n_items = uint64_t(n_kg) * n_blk;
    uint32_t cur_kg = 0xffffffffu;
    for (uint64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const uint32_t kg = uint32_t(it / n_blk), blk = uint32_t(it % n_blk);
        if (kg != cur_kg) {
            __syncthreads();  // every warp is done with the previous planes
            // plane b, lane l, bit s = parity(basis_b & key[kg * 1024 + 32 l + s])
            for (uint32_t l = warp; l < 32; l += kDedupWarps) {
                const uint32_t ki = kg * kDedupKeysPerWarp + l * 32 + lane;
                const unsigned long long key = ki < h.n_keys ? __ldg(h.keys + ki) : 0ull;
                uint32_t all = 0;
                for (uint32_t b = 0; b < h.width; b++) {
                    const uint32_t v = __ballot_sync(kFull, __popcll(key & __ldg(h.basis + b)) & 1);
                    all ^= v;
                    if (lane == 0) planes[b * 32 + l] = v;
                }
                if (lane == 0) {
                    planes[h.all_plane * 32 + l] = all;
                    planes[(h.all_plane + 1) * 32 + l] = 0u;
                }
            }
            __syncthreads();
            cur_kg = kg;
        }
        const uint32_t seg = blk * kDedupWarps + warp;
        if (seg >= h.n_segs) continue;
        const uint4 sgd = __ldg(h.segs + seg);
        // the warp's segment into shared memory once (the walk's record loads are
        // warp-uniform and serial: broadcast LDS instead of L1/L2 round trips); a CTA
        // keeps its segment block across key groups
        const uint32_t *w = h.words + sgd.x;
        if (sgd.y <= h.seg_buf_words) {
            if (have_seg != seg) {
                const uint32_t *src = h.words + sgd.x;
#pragma unroll 4
                for (uint32_t i = lane; i < sgd.y; i += 32) segbuf[i] = __ldg(src + i);
                __syncwarp();
                have_seg = seg;
            }
            w = segbuf;
        }
        double acc[32];
#pragma unroll
        for (int s = 0; s < 32; s++) acc[s] = 0.0;
        mono_walk<1, false>(w, sgd.z, sd, pl, stk, acc, nullptr);
        const uint32_t k0 = kg * kDedupKeysPerWarp + lane * 32;
        double *out = h.partial + uint64_t(seg) * h.n_keys + k0;
#pragma unroll
        for (int s = 0; s < 32; s++) {
            if (k0 + s < h.n_keys) out[s] = acc[s];
        }
    }
}

// value[k] = ((0 + S_0[k]) + S_1[k]) + ... in segment order.
__global__ void dedup_reduce_kernel(const double *__restrict__ partial, uint32_t n_segs, uint32_t n_keys,
                                    double *__restrict__ value) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n_keys; k += gridDim.x * blockDim.x) {
        double v = 0.0;
        uint32_t g = 0;
        for (; g + 16 <= n_segs; g += 16) {  // 16 independent loads in flight, adds in order
            double x[16];
#pragma unroll
            for (int i = 0; i < 16; i++) x[i] = __ldg(partial + uint64_t(g + i) * n_keys + k);
#pragma unroll
            for (int i = 0; i < 16; i++) v = __dadd_rn(v, x[i]);
        }
        for (; g < n_segs; g++) v = __dadd_rn(v, __ldg(partial + uint64_t(g) * n_keys + k));
        value[k] = v;
    }
}

__global__ void dedup_add_counts_kernel(const unsigned long long *__restrict__ src, unsigned long long *dst, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && src[i]) dst[i] += src[i];
}

// Frees the slots of the table's keys and resets its count (the next
// insertion round starts empty).
__global__ void dedup_clear_kernel(DedupTable t, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        t.keys[t.uslot[i]] = kDedupEmpty;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *t.count = 0;
}

struct DedupArArgs {
    uint64_t seed, first_shot, shots;
    uint32_t k0_round[10];
    uint32_t ci, j;             // component, output index within the chain (tensor pos = j + 1)
    uint32_t out;               // model output index
    uint32_t f_width;
    unsigned long long key_mask;
    unsigned long long *key;    // [shots]
    uint32_t *slot;             // [shots] slot in `cur`; replaced by the slot in `next`
    double *prev;               // [shots]
    const double *value0;       // j == 0: the normalization's values (same keys)
    const double *value;        // this tensor's values by id
    DedupTable cur;
    DedupTable next;            // insertion table for the next tensor (unused when last)
    bool insert_next;
    uint32_t *out32;            // [num_outputs][out_ld32] (nullable)
    uint64_t out_ld32;
    unsigned long long *counts; // (nullable)
    const double *uniforms;     // injected AR uniforms (nullable): [upos][uniforms_ld]
    uint64_t uniforms_ld, upos;
    unsigned long long *err;
};

// One autoregressive step (sampler.cpp:84-99) for every shot: thread = shot.
__global__ void __launch_bounds__(256) dedup_ar_kernel(const __grid_constant__ DedupArArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t seed_hi = uint32_t(a.seed >> 32);
    const uint32_t k2c = uint32_t(kP1c) ^ a.k0_round[1];
    const uint32_t stream = 0x80000000u ^ (a.ci << 12) ^ a.j;  // sampler.cpp:37-39
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    unsigned long long ones = 0;
    DedupWarpCache cache;
    // up to the 64-shot boundary: the record's last 64-bit word gets zero tail bits
    const uint64_t shots64 = (a.shots + 63) & ~uint64_t(63);
    for (uint64_t s0 = uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); s0 < shots64; s0 += stride) {
        const uint64_t s = s0 + lane;
        const bool valid = s < a.shots;
        bool bit = false;
        unsigned long long key = 0;
        if (valid) {
            const uint32_t id = a.cur.ids[a.slot[s]];
            const double cur = a.value[id];
            const double pv = a.j == 0 ? a.value0[id] : a.prev[s];
            const double ratio = __ddiv_rn(cur, pv);
            if (!(ratio > -1e-6 && ratio < 1.0 + 1e-6)) report_ratio_error(a.err, a.first_shot + s);
            double cl = (0.0 < ratio) ? ratio : 0.0;
            cl = (cl < 1.0) ? cl : 1.0;
            double u;
            if (a.uniforms) {
                u = a.uniforms[a.upos * a.uniforms_ld + s];
            } else {
                const uint64_t shot = a.first_shot + s;
                PhiloxPre pre[1] = {philox_pre(uint32_t(shot), uint32_t(shot >> 32), a.k0_round[0])};
                uint32_t rhi[1], rlo[1];
                philox_tail<1>(pre, seed_hi ^ stream, a.k0_round, k2c, a.k0_round[9], rhi, rlo);
                u = philox_uniform((uint64_t(rhi[0]) << 32) | rlo[0]);
            }
            bit = !(u < cl);
            a.prev[s] = bit ? __dsub_rn(pv, cur) : cur;
            key = a.key[s];
            const uint32_t p = a.f_width + a.j;
            if (bit && p < 63 && ((a.key_mask >> p) & 1ull)) key |= 1ull << p;
        }
        const uint32_t word = __ballot_sync(kFull, bit);
        if (lane == 0) {
            if (a.out32 && (s0 >> 5) < a.out_ld32) a.out32[a.out * a.out_ld32 + (s0 >> 5)] = word;
            ones += __popc(word);
        }
        if (a.insert_next) {
            const uint32_t ns = dedup_insert_warp(a.next, key, valid, lane, cache);
            if (valid) {
                a.key[s] = key;
                a.slot[s] = ns;
            }
        }
    }
    if (a.counts && lane == 0 && ones) atomicAdd(&a.counts[a.out], ones);
}

}  // namespace zxs_dev
