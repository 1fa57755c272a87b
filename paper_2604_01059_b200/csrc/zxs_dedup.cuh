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
//      the batch's U distinct keys (dedup_init_raw_kernel from the f words
//      shot_kernel stores, dedup_init_kernel from f columns, dedup_ar_kernel
//      for keys extended by a sampled bit);
//   2. contracts the tensor for those U keys only, term-parallel: the
//      tensor's terms are cut into G fixed summation segments (host,
//      encode_mono), a warp walks one segment for 1024 keys (mono_walk_fv
//      over block form tables, or mono_walk -- the record code of
//      mono_kernel) and writes the segment sums (dedup_eval_kernel);
//   3. folds the segment sums in order, ((0 + S_0) + S_1) + ... + S_{G-1}
//      (dedup_reduce_kernel) -- the same canonical order mono_kernel uses
//      per shot, so both paths give bit-identical values and a shot's value
//      does not depend on which other shots share its batch;
//   4. runs the autoregressive draws per shot (sampler.cpp:84-99) with the
//      values looked up by key: for short chains every position's keys are
//      expanded over the sampled-bit patterns up front and one kernel runs
//      the whole chain (dedup_expand_kernel, dedup_fused_ar_kernel);
//      otherwise the chain runs as node levels (a shot's state before
//      position j is a node: key + prev marginal; per level the distinct
//      node keys are contracted, one decision record per node, one pass per
//      shot: dedup_node_*_kernel; dedup_ar_kernel is the synchronous path).
// A level's keys are restricted to the parameters its tensor reads and
// reduced modulo the null space of its parity forms (dedup_null_reduce):
// one contraction per coset. Shots whose key is 0 and whose draws stay on
// the all-zero key's likelier-bit chain (the main lineage, contracted once
// per sampler) are finished by dedup_init_spec_kernel; only the others go
// through the node passes.
// Key counts stay on the device; the host checks once per batch and redoes
// an overflowing batch as two halves. Every step except the main lineage is
// recomputed per batch.
#pragma once

#include "zxs_mono.cuh"

namespace zxs_dev {

constexpr unsigned long long kDedupEmpty = ~0ull;  // keys use at most 63 raw parameter bits
constexpr int kDedupWarps = 16;                    // dedup_eval_kernel: warps per CTA (one segment each)
constexpr uint32_t kDedupKeysPerWarp = 1024;       // 32 keys per lane (NW = 1)
#ifndef ZXS_WALK_ILP
#define ZXS_WALK_ILP 0  // 1: two record chains per kind in mono_walk_fv (measured slower: 197 vs 183 ms per 2^28 config-3 batch)
#endif
constexpr uint32_t kDedupMaxBlockForms = 1024;     // form values per block table at least (128 B each in shared memory)

struct DedupTable {
    unsigned long long *keys;  // [mask + 1], kDedupEmpty when free
    uint32_t *ids;             // [mask + 1] dense id of the key in the slot
    uint32_t mask;
    uint32_t max_ids;          // ukeys / uslot capacity; more keys = overflow (host falls back)
    uint32_t *count;           // distinct keys inserted
    unsigned long long *ukeys; // [id] key
    uint32_t *uslot;           // [id] slot (for clearing)
};

constexpr uint32_t kDedupMaxProbes = 256;

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
    for (uint32_t probe = 0;; probe++) {
        if (probe == kDedupMaxProbes) {  // congested (more keys than the table is sized for): fall back
            atomicMax(t.count, t.max_ids + 1);
            return 0;  // any in-range slot: ids[] always holds an in-range id (dedup_reserve)
        }
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
                } else {
                    t.ids[slot] = 0;  // overflowed key: an in-range id until the host redoes the batch
                }
                return slot;
            }
            if (old == key) return slot;
        }
        slot = (slot + 1) & t.mask;
    }
}

// Per-warp cache of recent (key, slot) pairs (default one: the most recent miss; measured
// 1 < 2 < 4 < 8 ways in time), replicated in every lane (warp-
// uniform registers): the key distribution is extremely skewed (most shots
// carry the all-zero key), so most shots resolve here instead of hammering one
// table line in L2.
#ifndef ZXS_DEDUP_CACHE_WAYS
#define ZXS_DEDUP_CACHE_WAYS 1
#endif
constexpr uint32_t kDedupCacheWays = ZXS_DEDUP_CACHE_WAYS;
struct DedupWarpCache {
    unsigned long long key[kDedupCacheWays];
    uint32_t slot[kDedupCacheWays];
    uint32_t next;  // round-robin victim
    __device__ DedupWarpCache() : next(0) {
#pragma unroll
        for (uint32_t i = 0; i < kDedupCacheWays; i++) {
            key[i] = kDedupEmpty;
            slot[i] = 0;
        }
    }
};

// Warp-cooperative insert: cache lookup; lanes whose key missed insert into
// the table themselves (duplicates of a warp resolve to the same slot); the
// first missing key enters the cache.
__device__ __forceinline__ uint32_t dedup_insert_warp(const DedupTable &t, unsigned long long key, bool valid,
                                                      uint32_t lane, DedupWarpCache &c) {
    uint32_t slot = 0;
    bool hit = !valid;
#pragma unroll
    for (uint32_t i = 0; i < kDedupCacheWays; i++) {
        const bool m = key == c.key[i];
        slot = (m && !hit) ? c.slot[i] : slot;
        hit = hit || m;
    }
    const uint32_t miss = __ballot_sync(kFull, !hit);
    if (miss) {
        if (!hit) slot = dedup_insert(t, key);
        const uint32_t first = __ffs(miss) - 1;
        const unsigned long long fk = __shfl_sync(kFull, key, first);
        const uint32_t fs = __shfl_sync(kFull, slot, first);
#pragma unroll
        for (uint32_t i = 0; i < kDedupCacheWays; i++) {
            if (i == c.next) {
                c.key[i] = fk;
                c.slot[i] = fs;
            }
        }
        c.next = (c.next + 1) % kDedupCacheWays;
    }
    return slot;
}

struct DedupInitArgs {
    uint64_t shots;
    const uint32_t *fcols;  // [f_width][fcols_ld32]
    uint64_t fcols_ld32;
    uint32_t n_cols;            // f columns the component's tensors read (< 63)
    uint16_t cols[63];          // raw f column
    uint8_t bits[63];           // its key bit (local parameter index)
    unsigned long long *key;  // [shots] (nullable)
    uint32_t *slot;           // [shots]
    DedupTable table;
};

// Keys of the chain's first tensors (no sampled bits yet). A warp takes 1024
// shots: lane l loads its own 32-shot word of every f column the component
// reads (coalesced), scatters the few set bits into per-shot keys in shared
// memory, then the warp resolves the keys 32 shots at a time (lane = shot):
// the all-zero key (most shots) by a compare, the rest through the warp cache
// and the table.
constexpr uint32_t kDedupInitWarps = 4;
__global__ void __launch_bounds__(kDedupInitWarps * 32) dedup_init_kernel(const __grid_constant__ DedupInitArgs a) {
    __shared__ unsigned long long skeys[kDedupInitWarps][32 * 33];  // [shot bit][lane], padded
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    unsigned long long *kw = skeys[warp];
    DedupWarpCache cache;
    // slot of the all-zero key (inserted once per warp; harmless if no shot has it)
    uint32_t slot0 = 0;
    if (lane == 0) slot0 = dedup_insert(a.table, 0ull);
    slot0 = __shfl_sync(kFull, slot0, 0);
    const uint64_t n_words = (a.shots + 31) / 32;
    const uint64_t wstride = uint64_t(gridDim.x) * kDedupInitWarps * 32;
    for (uint64_t w0 = (uint64_t(blockIdx.x) * kDedupInitWarps + warp) * 32; w0 < n_words; w0 += wstride) {
        const uint64_t wd = w0 + lane;  // this lane's 32-shot word
#pragma unroll
        for (int s = 0; s < 32; s++) kw[s * 33 + lane] = 0ull;
        if (wd < n_words) {
            for (uint32_t i = 0; i < a.n_cols; i++) {
                const uint32_t p = a.cols[i];
                const unsigned long long kb = 1ull << a.bits[i];
                uint32_t w = __ldg(a.fcols + uint64_t(p) * a.fcols_ld32 + wd);
                while (w) {
                    const uint32_t sb = __ffs(w) - 1;
                    w &= w - 1;
                    kw[sb * 33 + lane] |= kb;
                }
            }
        }
        __syncwarp();
        for (uint32_t r = 0; r < 32; r++) {
            const uint64_t sh = (w0 + r) * 32 + lane;  // shot: word w0 + r, bit lane
            const bool valid = sh < a.shots;
            const unsigned long long key = kw[lane * 33 + r];
            const uint32_t nz = __ballot_sync(kFull, valid && key != 0ull);
            uint32_t slot = slot0;
            if (nz) {
                const uint32_t sl = dedup_insert_warp(a.table, key, valid && key != 0ull, lane, cache);
                if (key != 0ull) slot = sl;
            }
            if (valid) {
                if (a.key) a.key[sh] = key;  // null: the fused chain never extends keys
                a.slot[sh] = slot;
            }
        }
        __syncwarp();
    }
}

// Keys from the per-shot f words shot_kernel stored (f_width <= 64): key =
// f & mask; thread = shot, the all-zero key by a compare, the rest through the
// warp cache and the table.
template <typename FW>  // uint32_t (f_width <= 32) or unsigned long long
__global__ void __launch_bounds__(256) dedup_init_raw_kernel(const FW *__restrict__ fraw,
                                                             unsigned long long f_mask, uint64_t shots,
                                                             unsigned long long *key, uint32_t *slot_out,
                                                             DedupTable table) {
    const uint32_t lane = threadIdx.x & 31u;
    DedupWarpCache cache;
    uint32_t slot0 = 0;
    if (lane == 0) slot0 = dedup_insert(table, 0ull);
    slot0 = __shfl_sync(kFull, slot0, 0);
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t s0 = uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); s0 < shots; s0 += stride) {
        const uint64_t s = s0 + lane;
        const bool valid = s < shots;
        const unsigned long long k = valid ? ((unsigned long long)__ldg(fraw + s) & f_mask) : 0ull;
        uint32_t sl = slot0;
        if (__ballot_sync(kFull, k != 0ull)) {
            const uint32_t g = dedup_insert_warp(table, k, k != 0ull, lane, cache);
            if (k != 0ull) sl = g;
        }
        if (valid) {
            if (key) key[s] = k;
            slot_out[s] = sl;
        }
    }
}

// ---- main-lineage speculation (node levels, raw f words). The main lineage is
// the chain of nodes of the all-zero key that always takes the likelier bit;
// its decision records are the same node_rec a node pass would read (computed
// once per sampler, launch_dedup). A shot whose key is 0 draws its chain
// uniforms here (the same Philox draws as the node passes, sampler.cpp:37-39,
// 84-99) and compares them with the lineage's thresholds; while every bit is
// the lineage's the shot is done: its bits are the lineage's, already in the
// record words this kernel writes for every shot. The other shots -- a nonzero
// key, or a draw off the lineage -- go to the active list and through the
// node passes (ACT), which flip their bits where they differ.
constexpr uint32_t kSpecMaxChain = 32;
struct DedupSpecArgs {
    uint64_t seed, first_shot, shots;
    uint32_t k0_round[10];
    uint32_t ci, n_out;
    uint32_t main_bits;                      // bit j: the lineage's bit at position j
    unsigned long long T[kSpecMaxChain];     // bit = (k >= T), node_rec
    unsigned long long tie_lo[kSpecMaxChain];
    uint32_t tie_w[kSpecMaxChain];
    uint32_t out[kSpecMaxChain];             // record row of position j
    uint32_t *out32;
    uint64_t out_ld32;
    unsigned long long *err;                 // err[2]: near-tie draws
    uint32_t *active;                        // [shots] active shots (compacted)
    uint32_t *n_active;
};

#ifndef ZXS_SPEC_G
#define ZXS_SPEC_G 4
#endif
constexpr int kSpecG = ZXS_SPEC_G;
#ifndef ZXS_SPEC_PREFETCH
#define ZXS_SPEC_PREFETCH 0
#endif  // 32-shot groups per warp iteration (independent Philox chains per lane)
template <typename FW>
__global__ void __launch_bounds__(256) dedup_init_spec_kernel(const FW *__restrict__ fraw, unsigned long long f_mask,
                                                              uint32_t *slot_out, DedupTable table,
                                                              const __grid_constant__ DedupSpecArgs a) {
    constexpr int G = kSpecG;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t seed_hi = uint32_t(a.seed >> 32);
    const uint32_t k2c = uint32_t(kP1c) ^ a.k0_round[1];
    DedupWarpCache cache;
    const uint64_t shots64 = (a.shots + 63) & ~uint64_t(63);
    const uint64_t out_words = min(a.out_ld32, shots64 / 32);
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * G;
    const uint64_t sbeg = (uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u)) * G;
#if ZXS_SPEC_PREFETCH
    FW fnext[G];  // the next iteration's f words, loaded before this iteration's draws
#pragma unroll
    for (int g = 0; g < G; g++) fnext[g] = sbeg + 32 * g + lane < a.shots ? __ldg(fraw + sbeg + 32 * g + lane) : FW(0);
#endif
    for (uint64_t s0 = sbeg; s0 < shots64; s0 += stride) {
        uint64_t s[G];
        bool valid[G], on[G];  // on: on the main lineage so far
        unsigned long long k[G];
        uint32_t ties[G];      // counted once the shot is done (an active shot's passes count its own)
        PhiloxPre pre[G];
        bool any_on = false;
#pragma unroll
        for (int g = 0; g < G; g++) {
            s[g] = s0 + 32 * g + lane;
            valid[g] = s[g] < a.shots;
#if ZXS_SPEC_PREFETCH
            k[g] = valid[g] ? ((unsigned long long)fnext[g] & f_mask) : 0ull;
            const uint64_t sn = s[g] + stride;
            fnext[g] = sn < a.shots ? __ldg(fraw + sn) : FW(0);
#else
            k[g] = valid[g] ? ((unsigned long long)__ldg(fraw + s[g]) & f_mask) : 0ull;
#endif
            on[g] = valid[g] && k[g] == 0ull;
            any_on |= on[g];
            ties[g] = 0;
            const uint64_t shot = a.first_shot + s[g];
            pre[g] = philox_pre(uint32_t(shot), uint32_t(shot >> 32), a.k0_round[0]);
        }
        for (uint32_t j = 0; j < a.n_out; j++) {
            if (!__any_sync(kFull, any_on)) break;
            // a certain lineage bit (T = 0: k >= 0; T = 2^53: k < 2^53) needs no draw, has no near ties
            if (a.T[j] == 0ull || a.T[j] == (1ull << 53)) continue;
            const uint32_t stream = 0x80000000u ^ (a.ci << 12) ^ j;  // sampler.cpp:37-39
            uint32_t rhi[G], rlo[G];
            philox_tail<G>(pre, seed_hi ^ stream, a.k0_round, k2c, a.k0_round[9], rhi, rlo);
            any_on = false;
#pragma unroll
            for (int g = 0; g < G; g++) {
                const unsigned long long kk = ((uint64_t(rhi[g]) << 32) | rlo[g]) >> 11;  // uniform_at = kk 2^-53
                if (on[g]) {
                    ties[g] += kk - a.tie_lo[j] <= a.tie_w[j] ? 1u : 0u;
                    on[g] = uint32_t(kk >= a.T[j]) == ((a.main_bits >> j) & 1u);
                }
                any_on |= on[g];
            }
        }
#pragma unroll
        for (int g = 0; g < G; g++) {
            if (on[g] && ties[g]) atomicAdd(&a.err[2], (unsigned long long)ties[g]);
            // every shot's record words start with the lineage's bits (zero tails)
            const uint32_t vm = __ballot_sync(kFull, valid[g]);
            const uint64_t w = (s0 >> 5) + g;
            if (a.out32 && lane < a.n_out && w < out_words) {
                a.out32[a.out[lane] * a.out_ld32 + w] = ((a.main_bits >> lane) & 1u) ? vm : 0u;
            }
            const bool act = valid[g] && !on[g];
            const uint32_t am = __ballot_sync(kFull, act);
            if (am) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(a.n_active, uint32_t(__popc(am)));
                base = __shfl_sync(kFull, base, 0);
                const uint32_t i = base + __popc(am & ((1u << lane) - 1u));
                const uint32_t sl = dedup_insert_warp(table, k[g], act, lane, cache);
                if (act) {
                    a.active[i] = uint32_t(s[g]);
                    slot_out[i] = sl;
                }
            }
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
    uint32_t stack_words;             // stack area (>= kDedupWarps x (depth x 96 + 32), >= 64 x 33 raw planes)
    const unsigned long long *keys;   // the round's keys
    uint32_t n_keys;                  // keys (n_dev: at most this many, the rest read from n_dev)
    const uint32_t *n_dev;            // device-side key count (the table's), or null
    uint32_t n_mult;                  // keys = *n_dev x n_mult (expanded keys: base key x sampled-bit pattern)
    uint32_t key_base;                // first key of this round (keys / partials are relative to it)
    unsigned long long *stats;        // device counters {keys, plane-load bytes} (nullable)
    unsigned long long tensor_loads;  // plane loads per 32-key word of this tensor
    double *partial;                  // [n_segs][keys of the round, even stride]
    uint32_t seg_buf_words;           // per-warp shared-memory copy of its segment (0: walk from global)
    // block form tables (null: records carry tensor dictionary ids): the forms block
    // `first_block + blk` of kDedupWarps segments uses, as tensor dictionary entries
    const uint32_t *block_forms;
    const uint32_t *block_form_begin;
    uint32_t first_block;
    uint32_t table_bytes;  // shared memory before the planes: dictionary or form values
    uint32_t segs_per_warp;  // block = kDedupWarps x segs_per_warp consecutive segments (block form tables)
    uint32_t stage_entries;  // block tables: stage the forms' first dictionary entries in shared memory
};

#ifndef ZXS_REC_UNROLL
#define ZXS_REC_UNROLL 0
#endif
#ifndef ZXS_LEAF_LDS
#define ZXS_LEAF_LDS 1
#endif
// mono_leaf for one 32-key word per lane through a per-warp table of the leaf's
// five possible contributions, indexed by the key's (J mod 4, Z) code:
// {re, -im, -re, im, +0, +0, +0, +0}. A zero-flagged key adds +0.0 instead of
// skipping the add -- the same double (the accumulators start at +0.0 and
// round to nearest, so they are never -0.0) -- so the sums equal mono_leaf's
// bit for bit. Per key: one byte extract, one LDS.64 (five distinct addresses:
// broadcast) and the DADD, instead of mono_leaf's selects on the ALU pipe;
// the codes of four keys are built together (nibble x spread constant).
// Two tables per warp alternate, so one __syncwarp per leaf orders the writes
// after the previous leaf's reads.
__device__ __forceinline__ void dedup_leaf_lds(double (&acc)[32], uint32_t z, uint32_t j0, uint32_t j1, double re,
                                               double im, double *ltab, uint32_t lane, uint32_t &lbuf) {
    double *tab = ltab + lbuf * 8;
    if (lane < 8) {
        const double v = (lane & 1u) ? im : re;          // J odd: the imaginary part
        const double sv = ((lane + 1u) & 2u) ? -v : v;   // J = 1, 2: negated
        tab[lane] = lane < 4 ? sv : 0.0;
    }
    __syncwarp();
    lbuf ^= 1u;
    const char *tb = reinterpret_cast<const char *>(tab);
#pragma unroll
    for (int r = 0; r < 8; r++) {
        // byte k of c = 8 x (j0 | j1 << 1 | z << 2) of key 4r + k: bit k of a nibble times
        // sum_m 2^(7m + sh) lands on bit 8k + sh (no two terms share a position: no carries)
        const uint32_t n0 = (j0 >> (4 * r)) & 0xfu, n1 = (j1 >> (4 * r)) & 0xfu, nz = (z >> (4 * r)) & 0xfu;
        const uint32_t c = ((n0 * 0x01020408u) & 0x08080808u) | ((n1 * 0x02040810u) & 0x10101010u) |
                           ((nz * 0x04081020u) & 0x20202020u);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const uint32_t off = __byte_perm(c, 0u, 0x4440u | uint32_t(k));
            acc[4 * r + k] = __dadd_rn(acc[4 * r + k], *reinterpret_cast<const double *>(tb + off));
        }
    }
}

// mono_walk for one 32-key word per lane when every form value of the block
// is precomputed in shared memory (fv[local form * 32 + lane]): a form costs
// one conflict-free LDS instead of its dictionary entry and selector loads.
__device__ __forceinline__ void mono_walk_fv(const uint32_t *w, uint32_t nnodes, const uint32_t *fv, BW<1> *stk,
                                             double (&acc)[32], double *ltab, uint32_t lane) {
    constexpr int NW = 1;
    uint32_t q = 0;
    uint32_t lbuf = 0;
    for (uint32_t nn = 0; nn < nnodes; nn++) {
        const uint32_t h0 = w[q], h1 = w[q + 1], h2 = w[q + 2];
        const uint32_t depth = (h0 >> 24) & 0x3fu;
        const bool leaf = (h0 >> 31) != 0;
        q += 3;
        double re = 0.0, im = 0.0;
        if (leaf) {
            re = __hiloint2double(int(w[q + 1]), int(w[q]));
            im = __hiloint2double(int(w[q + 3]), int(w[q + 2]));
            q += 4;
        }
        BW<1> z = bw_zero<1>(), j0 = bw_zero<1>(), j1 = bw_zero<1>();
        if (depth) {
            const BW<1> *ps = stk + (depth - 1) * 96;
            z = ps[0];
            j0 = ps[32];
            j1 = ps[64];
        }
        // one-form records grouped by kind (host: encode_mono block tables): one fixed op per loop
        {
            uint32_t zz = z.w[0], a0 = j0.w[0], a1 = j1.w[0];
            const uint32_t n_add = h1 & 0xffu, n_sub = (h1 >> 8) & 0xffu, n_add2 = (h1 >> 16) & 0xffu;
            const uint32_t n_z = h1 >> 24, n_zn = h2 & 0xffu;
            // one-form record word = the form value's byte offset in the block table (host: encode_mono)
            auto fvr = [&](uint32_t i) { return *reinterpret_cast<const uint32_t *>(reinterpret_cast<const char *>(fv) + w[i]); };
#if ZXS_WALK_ILP
            // J (mod 4) and Z are order-free sums / ORs: two independent chains per kind (the
            // form loads of consecutive records overlap), merged at the node's end
            uint32_t e = q + n_add;
            uint32_t b0 = 0, b1 = 0;  // J += a, second chain
            for (; q + 1 < e; q += 2) {
                const uint32_t x = fvr(q), y = fvr(q + 1);
                a1 ^= a0 & x;
                a0 ^= x;
                b1 ^= b0 & y;
                b0 ^= y;
            }
            if (q < e) {
                const uint32_t x = fvr(q++);
                a1 ^= a0 & x;
                a0 ^= x;
            }
            uint32_t c0 = 0, c1 = 0, d0 = 0, d1 = 0;  // J -= a: the subtrahends summed in two chains
            for (e += n_sub; q + 1 < e; q += 2) {
                const uint32_t x = fvr(q), y = fvr(q + 1);
                c1 ^= c0 & x;
                c0 ^= x;
                d1 ^= d0 & y;
                d0 ^= y;
            }
            if (q < e) {
                const uint32_t x = fvr(q++);
                c1 ^= c0 & x;
                c0 ^= x;
            }
            uint32_t t1 = 0;  // J += 2a
            for (e += n_add2; q + 1 < e; q += 2) {
                a1 ^= fvr(q);
                t1 ^= fvr(q + 1);
            }
            if (q < e) a1 ^= fvr(q++);
            uint32_t z2 = 0;  // Z |= a, Z |= ~a
            for (e += n_z; q + 1 < e; q += 2) {
                zz |= fvr(q);
                z2 |= fvr(q + 1);
            }
            if (q < e) zz |= fvr(q++);
            for (e += n_zn; q + 1 < e; q += 2) {
                zz |= ~fvr(q);
                z2 |= ~fvr(q + 1);
            }
            if (q < e) zz |= ~fvr(q++);
            {  // (a) += (b), (c) += (d), (a) -= (c), mod 4 on two bit planes
                const uint32_t cy = a0 & b0;
                a0 ^= b0;
                a1 ^= b1 ^ cy ^ t1;
                const uint32_t cd = c0 & d0;
                c0 ^= d0;
                c1 ^= d1 ^ cd;
                const uint32_t br = ~a0 & c0;
                a0 ^= c0;
                a1 ^= c1 ^ br;
            }
            z.w[0] = zz | z2;
#else
            // ZXS_REC_UNROLL > 0: the kind loops unrolled by hand with a rolled tail (the
            // compiler's own unroll by 8 adds remainder blocks of 4, 2 and 1 per loop)
#if ZXS_REC_UNROLL > 0
#define ZXS_REC_LOOP(END, BODY)                                                     \
    for (; q + ZXS_REC_UNROLL <= (END); q += ZXS_REC_UNROLL) {                      \
        _Pragma("unroll") for (int u_ = 0; u_ < ZXS_REC_UNROLL; u_++) {             \
            const uint32_t x = fvr(q + u_);                                         \
            BODY                                                                    \
        }                                                                           \
    }                                                                               \
    _Pragma("unroll 1") for (; q < (END); q++) {                                    \
        const uint32_t x = fvr(q);                                                  \
        BODY                                                                        \
    }
#else
#define ZXS_REC_LOOP(END, BODY) \
    for (; q < (END); q++) {    \
        const uint32_t x = fvr(q); \
        BODY                    \
    }
#endif
            uint32_t e = q + n_add;
            ZXS_REC_LOOP(e, a1 ^= a0 & x; a0 ^= x;)  // J += a
            e += n_sub;
            ZXS_REC_LOOP(e, a1 ^= ~a0 & x; a0 ^= x;)  // J -= a
            e += n_add2;
            ZXS_REC_LOOP(e, a1 ^= x;)  // J += 2a
            e += n_z;
            ZXS_REC_LOOP(e, zz |= x;)  // Z |= a
            e += n_zn;
            ZXS_REC_LOOP(e, zz |= ~x;)  // Z |= ~a
#undef ZXS_REC_LOOP
            z.w[0] = zz;
#endif
            j0.w[0] = a0;
            j1.w[0] = a1;
        }
        for (uint32_t g = 0; g < (h0 & 0xffu); g++) {  // two-form records
            const uint32_t r = w[q], gw = w[q + 1];
            q += 2;
            const uint32_t fa = r & kFormMask, fb = (r >> kFormShiftB) & kFormMask;
            BW<1> a, bb;
            a.w[0] = fa == kMonoNoForm ? 0u : fv[fa * 32];
            bb.w[0] = fb == kMonoNoForm ? 0u : fv[fb * 32];
            const uint32_t zl = gw >> 6;
            z.w[0] |= ((zl & 1u) ? (~a.w[0] & ~bb.w[0]) : 0u) | ((zl & 2u) ? (~a.w[0] & bb.w[0]) : 0u) |
                      ((zl & 4u) ? (a.w[0] & ~bb.w[0]) : 0u) | ((zl & 8u) ? (a.w[0] & bb.w[0]) : 0u);
            j_add<1>(j0, j1, a, gw & 3u);
            j_add<1>(j0, j1, bb, (gw >> 2) & 3u);
            j_add<1>(j0, j1, bw_and<1>(a, bb), (gw >> 4) & 3u);
        }
        if (!leaf) {
            BW<1> *nsp = stk + depth * 96;
            nsp[0] = z;
            nsp[32] = j0;
            nsp[64] = j1;
            continue;
        }
#if ZXS_LEAF_LDS
        dedup_leaf_lds(acc, z.w[0], j0.w[0], j1.w[0], re, im, ltab, lane, lbuf);
#else
        mono_leaf<1>(acc, z, j0, j1, re, im);
#endif
    }
}

// Items = (key group of 1024, block of kDedupWarps segments); a CTA builds the
// key group's parameter planes once in shared memory (shared by its warps),
// every warp walks one segment for all 1024 keys.
__global__ void __launch_bounds__(kDedupWarps * 32, 1) dedup_eval_kernel(const __grid_constant__ DedupEvalArgs h) {
    extern __shared__ __align__(128) uint8_t dsm[];
    const bool fvm = h.block_forms != nullptr;
    uint4 *sd = reinterpret_cast<uint4 *>(dsm);  // dictionary (fvm: form values [f][lane])
    uint32_t *fv = reinterpret_cast<uint32_t *>(dsm);
    uint32_t *planes = reinterpret_cast<uint32_t *>(dsm + h.table_bytes);  // [p][lane]
    uint32_t *stack_all = planes + h.n_planes * 32;                  // per warp [depth][3][lane]
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    BW<1> *stk = reinterpret_cast<BW<1> *>(stack_all + warp * h.stack_depth * 96) + lane;
    // the warp's two leaf tables (dedup_leaf_lds) after every warp's stack
    double *ltab = reinterpret_cast<double *>(stack_all + kDedupWarps * h.stack_depth * 96) + warp * 16;
    uint32_t *segbuf = stack_all + h.stack_words + warp * h.seg_buf_words;
    uint4 *sent = reinterpret_cast<uint4 *>(stack_all + h.stack_words + kDedupWarps * h.seg_buf_words);
    uint32_t have_seg = 0xffffffffu;  // segment currently in segbuf
    const char *pl = reinterpret_cast<const char *>(planes + lane);

    if (!fvm) {
        for (uint32_t i = threadIdx.x; i < h.n_dict; i += blockDim.x) sd[i] = __ldg(h.dict + i);
    }
    uint32_t cur_blk = 0xffffffffu;
    // keys of this round: the device count (minus the earlier rounds' keys), at most n_keys
    const uint64_t dev_keys = h.n_dev ? uint64_t(*h.n_dev) * max(h.n_mult, 1u) : 0;
    const uint32_t n_keys = h.n_dev ? uint32_t(min(dev_keys > h.key_base ? dev_keys - h.key_base : uint64_t(0), uint64_t(h.n_keys)))
                                    : h.n_keys;
    if (n_keys == 0) return;  // a round past the batch's key count
    if (h.stats && blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd(&h.stats[0], (unsigned long long)n_keys);
        atomicAdd(&h.stats[1], h.tensor_loads * ((n_keys + 31) / 32) * 4);
    }
    const uint32_t n_kg = (n_keys + kDedupKeysPerWarp - 1) / kDedupKeysPerWarp;
    const uint32_t spw = max(h.segs_per_warp, 1u);  // segments each warp walks per item
    const uint32_t bsegs = kDedupWarps * spw;       // segments per block (one form table)
    const uint32_t n_blk = (h.n_segs + bsegs - 1) / bsegs;
    const uint64_t n_items = uint64_t(n_kg) * n_blk;
    uint32_t cur_kg = 0xffffffffu;
    for (uint64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const uint32_t kg = uint32_t(it / n_blk), blk = uint32_t(it % n_blk);
        if (kg != cur_kg) {
            __syncthreads();  // every warp is done with the previous planes (and its stack)
            // plane b, lane l, bit s = parity(basis_b & key[kg * 1024 + 32 l + s]): the key group's
            // raw parameter planes by warp transposes (row l of 32 keys: lane p gets parameter p's
            // word), staged in the stack area, then each basis plane as the XOR of its parameters'
            uint32_t *raw = stack_all;  // [64 parameters][33] (padded: conflict-free)
            for (uint32_t l = warp; l < 32; l += kDedupWarps) {
                const uint32_t ki = kg * kDedupKeysPerWarp + l * 32 + lane;
                const unsigned long long key = ki < n_keys ? __ldg(h.keys + ki) : 0ull;
                raw[lane * 33 + l] = warp_transpose32(uint32_t(key), lane);
                raw[(32 + lane) * 33 + l] = warp_transpose32(uint32_t(key >> 32), lane);
            }
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < h.width * 32; i += blockDim.x) {
                const uint32_t b = i >> 5, l = i & 31u;
                uint32_t v = 0;
                for (unsigned long long m = __ldg(h.basis + b); m; m &= m - 1) v ^= raw[(__ffsll((long long)m) - 1) * 33 + l];
                planes[b * 32 + l] = v;
            }
            __syncthreads();
            if (threadIdx.x < 32) {
                uint32_t all = 0;
                for (uint32_t b = 0; b < h.width; b++) all ^= planes[b * 32 + threadIdx.x];
                planes[h.all_plane * 32 + threadIdx.x] = all;
                planes[(h.all_plane + 1) * 32 + threadIdx.x] = 0u;
            }
            __syncthreads();
            cur_kg = kg;
            cur_blk = 0xffffffffu;
        }
        if (fvm && blk != cur_blk) {
            // the block's form values for this key group: warp w computes forms w, w + 16, ...
            const uint32_t f0 = __ldg(h.block_form_begin + h.first_block + blk);
            const uint32_t nf = __ldg(h.block_form_begin + h.first_block + blk + 1) - f0;
            __syncthreads();  // every warp is done with the previous block's values
#ifndef ZXS_FV_REG_ONLY
#define ZXS_FV_REG_ONLY 0
#endif
            if (h.stage_entries && !ZXS_FV_REG_ONLY) {
                // first dictionary entry of every form, gathered once (L2 -> shared)
                for (uint32_t i = threadIdx.x; i < nf; i += blockDim.x) sent[i] = __ldg(h.dict + __ldg(h.block_forms + f0 + i));
                __syncthreads();
                for (uint32_t f = warp; f < nf; f += kDedupWarps) {
                    uint4 e = sent[f];
                    BW<1> v = mono_entry<1>(e, pl);
                    if (e.x & 0x80u) {  // continuation entries (forms of more than 15 selectors)
                        uint32_t gi = __ldg(h.block_forms + f0 + f);
                        do {
                            e = __ldg(h.dict + ++gi);
                            v = bw_xor<1>(v, mono_entry<1>(e, pl));
                        } while (e.x & 0x80u);
                    }
                    fv[f * 32 + lane] = v.w[0];
                }
            } else {
                // no room to stage them in shared memory: staged in registers instead -- lane i
                // fetches the first entry of the warp's form w + 16 i (32 dependent L2 round trips
                // in flight instead of one), each broadcast by shuffle when its form is computed
                for (uint32_t fb = warp; fb < nf; fb += kDedupWarps * 32) {
                    const uint32_t mf = fb + kDedupWarps * lane;
                    const uint32_t mgi = mf < nf ? __ldg(h.block_forms + f0 + mf) : 0u;
                    const uint4 me = mf < nf ? __ldg(h.dict + mgi) : make_uint4(0, 0, 0, 0);
                    const uint32_t nk = min(32u, (nf - fb + kDedupWarps - 1) / kDedupWarps);
                    for (uint32_t k = 0; k < nk; k++) {
                        uint4 e;
                        e.x = __shfl_sync(kFull, me.x, k);
                        e.y = __shfl_sync(kFull, me.y, k);
                        e.z = __shfl_sync(kFull, me.z, k);
                        e.w = __shfl_sync(kFull, me.w, k);
                        BW<1> v = mono_entry<1>(e, pl);
                        if (e.x & 0x80u) {  // continuation entries (forms of more than 15 selectors)
                            uint32_t gi = __shfl_sync(kFull, mgi, k);
                            do {
                                e = __ldg(h.dict + ++gi);
                                v = bw_xor<1>(v, mono_entry<1>(e, pl));
                            } while (e.x & 0x80u);
                        }
                        fv[(fb + kDedupWarps * k) * 32 + lane] = v.w[0];
                    }
                }
            }
            __syncthreads();
            cur_blk = blk;
        }
        // the warp's summation group: spw consecutive segments accumulated without a reset
        // (the per-shot stream folds only at a group's first segment, encode_mono)
        const uint32_t group = blk * kDedupWarps + warp;
        if (group * spw >= h.n_segs) continue;
        double acc[32];
#pragma unroll
        for (int s = 0; s < 32; s++) acc[s] = 0.0;
        for (uint32_t si = 0; si < spw; si++) {
            const uint32_t seg = group * spw + si;
            if (seg >= h.n_segs) break;
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
            if (fvm && w == segbuf) {  // record words in shared memory: LDS (a separate instantiation)
                mono_walk_fv(segbuf, sgd.z, fv + lane, stk, acc, ltab, lane);
            } else if (fvm) {
                mono_walk_fv(h.words + sgd.x, sgd.z, fv + lane, stk, acc, ltab, lane);
            } else {
                mono_walk<1, false>(w, sgd.z, sd, pl, stk, acc, nullptr);
            }
        }
        // partial sums [group][key] (key stride = the round's capacity, even): a lane's 32 keys are
        // consecutive, so the warp's stores are contiguous
        const uint32_t k0 = kg * kDedupKeysPerWarp + lane * 32;
        const uint64_t stride = (uint64_t(h.n_keys) + 1) & ~uint64_t(1);
        double *out = h.partial + uint64_t(group) * stride + k0;
        if (k0 + 32 <= n_keys) {
            double2 *o2 = reinterpret_cast<double2 *>(out);
#pragma unroll
            for (int s = 0; s < 16; s++) o2[s] = make_double2(acc[2 * s], acc[2 * s + 1]);
        } else {
#pragma unroll
            for (int s = 0; s < 32; s++) {
                if (k0 + s < n_keys) out[s] = acc[s];
            }
        }
    }
}

// value[slot of key k] = ((0 + S_0[k]) + S_1[k]) + ... in segment order (values
// are stored by table slot, or densely for expanded keys). Thread = key: it
// reads its segment sums down a [segment][key] column (a warp's loads are
// contiguous, eight in flight) and adds them in order.
__global__ void dedup_reduce_kernel(const double *__restrict__ partial, uint32_t n_segs, uint32_t max_keys,
                                    const uint32_t *n_dev, uint32_t n_mult, uint32_t key_base,
                                    const uint32_t *__restrict__ uslot, double *__restrict__ value) {
    const uint64_t dev_keys = n_dev ? uint64_t(*n_dev) * max(n_mult, 1u) : 0;
    const uint32_t n_keys = n_dev ? uint32_t(min(dev_keys > key_base ? dev_keys - key_base : uint64_t(0), uint64_t(max_keys)))
                                  : max_keys;
    const uint64_t stride = (uint64_t(max_keys) + 1) & ~uint64_t(1);  // partials [segment][key]
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n_keys; k += gridDim.x * blockDim.x) {
        const double *col = partial + k;  // consecutive threads read consecutive keys
        double v = 0.0;
        uint32_t g = 0;
        for (; g + 8 <= n_segs; g += 8) {
            double x[8];
#pragma unroll
            for (int i = 0; i < 8; i++) x[i] = __ldg(col + uint64_t(g + i) * stride);
#pragma unroll
            for (int i = 0; i < 8; i++) v = __dadd_rn(v, x[i]);
        }
        for (; g < n_segs; g++) v = __dadd_rn(v, __ldg(col + uint64_t(g) * stride));
        value[uslot ? uslot[k] : k] = v;
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

// The same with the key count read on the device (no host round trip); the
// largest count seen goes to *max_count (the host checks it once per batch).
// The count itself is reset by dedup_reset_kernel after this kernel.
__global__ void dedup_clear_dev_kernel(DedupTable t, unsigned int *max_count, uint32_t mult = 1) {
    const uint32_t n = min(*t.count, t.max_ids);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned long long v = (unsigned long long)(*t.count) * mult;
        atomicMax(max_count, *t.count > t.max_ids || v > 0xffffffffull ? 0xffffffffu : uint32_t(v));
    }
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        t.keys[t.uslot[i]] = kDedupEmpty;
    }
}
__global__ void dedup_reset_kernel(uint32_t *count) { *count = 0; }

// Ratio-breakdown reports of the sync-free chain are staged (a batch that is
// redone must not report the garbage of its first attempt) and merged into
// the sampler's error state when the batch is accepted.
__global__ void dedup_err_init_kernel(unsigned long long *e) {
    e[0] = 0ull;
    e[1] = ~0ull;
    e[2] = 0ull;
}
__global__ void dedup_err_merge_kernel(const unsigned long long *e, unsigned long long *err) {
    if (e[0]) report_ratio_error(err, e[1]);
    if (e[2]) err[2] += e[2];
}

// One autoregressive decision, exactly the reference's (sampler.cpp:84-99):
// ratio = cur / prev (IEEE), error outside (-1e-6, 1 + 1e-6), clamp to [0, 1],
// bit = !(u < ratio). The IEEE quotient only matters when u (or an error
// bound) lies within the float estimate's error of it: a float quotient with
// a 4e-7 relative margin (conversion + division error <= 2.4e-7) decides every
// other case with the same result, the rest take __ddiv_rn.
__device__ __forceinline__ bool ar_decide(double cur, double prev, double u, unsigned long long *err, uint64_t shot) {
    const double ac = fabs(cur), ap = fabs(prev);
    if (ap > 1e-30 && ap < 1e30 && (ac == 0.0 || (ac > 1e-30 && ac < 1e30))) {
        const float qf = __fdividef(float(cur), float(prev));
        const double q = double(qf), d = 4e-7 * fabs(q) + 1e-37;
        if (q - d > -1e-6 && q + d < 1.0 + 1e-6) {  // certainly no ratio error
            if (u < q - d) return false;            // u < ratio <= 1 (or ratio clamped to 1)
            if (u > q + d) return true;             // u > max(ratio, 0) >= clamp(ratio)
        }
    }
    const double ratio = __ddiv_rn(cur, prev);
    if (!(ratio > -1e-6 && ratio < 1.0 + 1e-6)) report_ratio_error(err, shot);
    double cl = (0.0 < ratio) ? ratio : 0.0;
    cl = (cl < 1.0) ? cl : 1.0;
    count_near_tie(err, u, cl);
    return !(u < cl);
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
    const double *value0;       // j == 0: the normalization's values by slot (same table)
    const double *value;        // this tensor's values by slot of `cur`
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

// One autoregressive step (sampler.cpp:84-99) for every shot. A warp takes 64
// consecutive shots per iteration, lane = shots s and s + 32: both groups'
// loads, divisions and Philox draws are independent (two chains in flight).
#ifndef ZXS_AR_G
#define ZXS_AR_G 2
#endif
constexpr int kDedupArGroups = ZXS_AR_G;
__global__ void __launch_bounds__(256) dedup_ar_kernel(const __grid_constant__ DedupArArgs a) {
    constexpr int G = kDedupArGroups;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t seed_hi = uint32_t(a.seed >> 32);
    const uint32_t k2c = uint32_t(kP1c) ^ a.k0_round[1];
    const uint32_t stream = 0x80000000u ^ (a.ci << 12) ^ a.j;  // sampler.cpp:37-39
    const uint32_t p = a.f_width + a.j;
    const bool key_bit = p < 63 && ((a.key_mask >> p) & 1ull);  // later tensors read sampled bit j
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * G;
    unsigned long long ones = 0;
    DedupWarpCache cache;
    // up to the 64-shot boundary: the record's last 64-bit word gets zero tail bits
    const uint64_t shots64 = (a.shots + 63) & ~uint64_t(63);
    // this batch's record words (a split batch's rows continue past them: out_ld32 is only the stride)
    const uint64_t out_words = min(a.out_ld32, shots64 / 32);
    for (uint64_t s0 = (uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u)) * G; s0 < shots64; s0 += stride) {
        uint64_t s[G];
        bool valid[G], bit[G];
        uint32_t sl[G];
        double cur[G], pv[G];
#pragma unroll
        for (int g = 0; g < G; g++) {
            s[g] = s0 + 32 * g + lane;
            valid[g] = s[g] < a.shots;
            sl[g] = valid[g] ? a.slot[s[g]] : 0u;
            if (a.j != 0 && valid[g]) pv[g] = a.prev[s[g]];
        }
#pragma unroll
        for (int g = 0; g < G; g++) {
            cur[g] = a.value[sl[g]];
            if (a.j == 0) pv[g] = a.value0[sl[g]];
        }
        double u[G];
        if (a.uniforms) {
#pragma unroll
            for (int g = 0; g < G; g++) u[g] = valid[g] ? a.uniforms[a.upos * a.uniforms_ld + s[g]] : 0.0;
        } else {
            PhiloxPre pre[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                const uint64_t shot = a.first_shot + s[g];
                pre[g] = philox_pre(uint32_t(shot), uint32_t(shot >> 32), a.k0_round[0]);
            }
            uint32_t rhi[G], rlo[G];
            philox_tail<G>(pre, seed_hi ^ stream, a.k0_round, k2c, a.k0_round[9], rhi, rlo);
#pragma unroll
            for (int g = 0; g < G; g++) u[g] = philox_uniform((uint64_t(rhi[g]) << 32) | rlo[g]);
        }
#pragma unroll
        for (int g = 0; g < G; g++) {
            bit[g] = false;
            if (valid[g]) {
                bit[g] = ar_decide(cur[g], pv[g], u[g], a.err, a.first_shot + s[g]);
                a.prev[s[g]] = bit[g] ? __dsub_rn(pv[g], cur[g]) : cur[g];
            }
            const uint32_t word = __ballot_sync(kFull, bit[g]);
            if (lane == 0) {
                const uint64_t wi = (s0 >> 5) + g;
                if (a.out32 && wi < out_words) a.out32[a.out * a.out_ld32 + wi] = word;
                ones += __popc(word);
            }
        }
        if (a.insert_next) {
#pragma unroll
            for (int g = 0; g < G; g++) {
                unsigned long long key = valid[g] ? a.key[s[g]] : 0ull;
                const bool grows = key_bit && bit[g];  // the key gains bit j
                if (grows) key |= 1ull << p;
                const uint32_t ns = dedup_insert_warp(a.next, key, valid[g], lane, cache);
                if (valid[g]) {
                    if (grows) a.key[s[g]] = key;
                    a.slot[s[g]] = ns;
                }
            }
        }
    }
    if (a.counts && lane == 0 && ones) atomicAdd(&a.counts[a.out], ones);
}

// ---- node levels (longer chains, the default when a chain is not fused).
// A shot's state before position j is a NODE: its key (base key plus the
// sampled bits the later tensors read) and its prev marginal; both are
// functions of (base key, bits sampled so far), so they live per node, not
// per shot. Per level: distinct node keys are contracted (dedup_eval), each
// node's decision record is derived once (dedup_node_decide_kernel: the
// IEEE ratio, its clamp, the reference's error test, and the integer draw
// threshold T = ceil(cl 2^53): u = k 2^-53 < cl  <=>  k < T), and one
// per-shot pass (dedup_node_pass_kernel) reads the shot's node slot, draws,
// compares k >= T, and inserts the child node (parent slot << 1 | bit) for
// the next level: 4 B read + 4 B written per shot per position (the
// step-by-step dedup_ar_kernel moves slot, key and prev per shot).
struct __align__(16) DedupNodeRec {
    unsigned long long T;       // bit = (k >= T); bit 63: ratio outside (-1e-6, 1 + 1e-6)
    unsigned long long tie_lo;  // near-tie draws: k - tie_lo <= tie_w (2^62: none)
    double cl;                  // clamped ratio (injected-uniform mode)
    uint32_t tie_w;
    // certain bit (T = 0 or 2^53, no error): the slot of the only child in the next
    // level's table, inserted by the decide kernel (kNodeNoChild on the last level);
    // kNodeDraw otherwise (the pass draws and inserts the child)
    uint32_t child;
};
constexpr unsigned long long kNodeErr = 1ull << 63;
constexpr uint32_t kNodeDraw = 0xffffffffu, kNodeNoChild = 0xfffffffeu;

struct DedupNodeArrays {
    // indexed by the node's slot in its level's node table
    unsigned long long *key;  // key (local parameter bits)
    double *prev;             // prev marginal
    double *cur;              // this level's marginal
    uint32_t *kslot;          // slot of the key in the level's key table
    DedupNodeRec *rec;
};

__device__ __forceinline__ DedupNodeRec node_rec(double cur, double pv, uint32_t sl, const DedupTable &next,
                                                 bool insert_next) {
    // sampler.cpp:84-99, per node: the same division, test and clamp as per shot
    const double ratio = __ddiv_rn(cur, pv);
    const bool err = !(ratio > -1e-6 && ratio < 1.0 + 1e-6);
    double cl = (0.0 < ratio) ? ratio : 0.0;
    cl = (cl < 1.0) ? cl : 1.0;
    DedupNodeRec r;
    r.cl = cl;
    const unsigned long long T = (unsigned long long)ceil(cl * 0x1.0p53);  // cl 2^53 is exact
    r.T = T | (err ? kNodeErr : 0ull);
    const double w = 1e-9 * fmax(cl, 1e-300);
    const double lo = fmax(cl - w, 0.0) * 0x1.0p53, hi = fmin(cl + w, 1.0) * 0x1.0p53;
    const unsigned long long tlo = (unsigned long long)ceil(lo), thi = (unsigned long long)floor(hi);
    const bool certain = T == 0ull || T == (1ull << 53);
    // the window's width is below 2^32 (1e-9 2^53); an empty window or a certain bit never counts
    r.tie_lo = (certain || thi < tlo) ? (1ull << 62) : tlo;
    r.tie_w = (certain || thi < tlo) ? 0u : uint32_t(thi - tlo);
    r.child = kNodeDraw;
    if (certain && !err) {
        // every shot at this node takes the same bit (k < 2^53 <= T, or k >= 0 = T)
        r.child = insert_next ? dedup_insert(next, (unsigned long long)sl << 1 | (T == 0ull ? 1ull : 0ull)) : kNodeNoChild;
    }
    return r;
}

// One node record from (cur, pv) = v[0], v[1] (main-lineage speculation, launch_dedup).
__global__ void dedup_main_rec_kernel(const double *v, DedupNodeRec *out) {
    DedupTable none{};
    *out = node_rec(v[0], v[1], 0u, none, false);
}

// Level 0: the nodes are the base keys (table ids), already contracted for the
// normalization (value0, by node slot) and the first marginal (value, by the
// slot kslot[node slot] of the node's reduced key; kslot null: by node slot).
__global__ void dedup_node_level0_kernel(DedupTable t, const double *__restrict__ value0, const double *__restrict__ value,
                                         const uint32_t *__restrict__ kslot, DedupNodeArrays na, DedupTable next,
                                         bool insert_next) {
    const uint32_t n = min(*t.count, t.max_ids);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t sl = t.uslot[i];  // node arrays are indexed by table slot
        const double pv = value0[sl], cur = value[kslot ? kslot[sl] : sl];
        na.key[sl] = t.ukeys[i];
        na.prev[sl] = pv;
        na.cur[sl] = cur;
        na.kslot[sl] = sl;
        na.rec[sl] = node_rec(cur, pv, sl, next, insert_next);
    }
}

// A key reduced modulo the null space of a tensor's forms (null[2i] = 1 << q_i,
// null[2i + 1] = the null vector with free bit q_i; encode_mono): keys of one
// coset give every form -- so every record and the tensor -- the same value,
// and the representative with no free bit set is evaluated once for all of them.
__device__ __forceinline__ unsigned long long dedup_null_reduce(unsigned long long k,
                                                                const unsigned long long *__restrict__ null,
                                                                uint32_t n_null) {
    for (uint32_t i = 0; i < n_null; i++) {
        if (k & __ldg(null + 2 * i)) k ^= __ldg(null + 2 * i + 1);
    }
    return k;
}

// Level 0's key tables: the base keys restricted to what tensor 0 (or 1) reads
// and reduced modulo its null space; kslot[node slot] = the reduced key's slot.
__global__ void dedup_key_restrict_kernel(DedupTable nodes, unsigned long long read_mask,
                                          const unsigned long long *__restrict__ null, uint32_t n_null, DedupTable keys,
                                          uint32_t *__restrict__ kslot) {
    const uint32_t n = min(*nodes.count, nodes.max_ids);
    const uint32_t lane = threadIdx.x & 31u;
    DedupWarpCache cache;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); i0 < n; i0 += stride) {
        const uint32_t i = i0 + lane;
        const bool valid = i < n;
        const unsigned long long key = valid ? dedup_null_reduce(nodes.ukeys[i] & read_mask, null, n_null) : 0ull;
        const uint32_t ks = dedup_insert_warp(keys, key, valid, lane, cache);
        if (valid) kslot[nodes.uslot[i]] = ks;
    }
}

// dst[node slot] = src[kslot[node slot]] for every node of the table.
__global__ void dedup_gather_kernel(DedupTable nodes, const double *__restrict__ src, const uint32_t *__restrict__ kslot,
                                    double *__restrict__ dst) {
    const uint32_t n = min(*nodes.count, nodes.max_ids);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t sl = nodes.uslot[i];
        dst[sl] = src[kslot[sl]];
    }
}

// Level j + 1's nodes (table entries parent << 1 | bit): key and prev from the
// parent (prev = bit ? prev - cur : cur, sampler.cpp:95-98), the key extended
// by the bit when a later tensor reads it (bit_pos < 64); the key restricted to
// the parameters the level's tensor reads and reduced modulo its null space
// goes into the level's key table.
__global__ void dedup_node_prep_kernel(DedupTable nodes, DedupNodeArrays parent, DedupNodeArrays na, uint32_t bit_pos,
                                       unsigned long long read_mask, const unsigned long long *__restrict__ null,
                                       uint32_t n_null, DedupTable keys) {
    const uint32_t n = min(*nodes.count, nodes.max_ids);
    const uint32_t lane = threadIdx.x & 31u;
    DedupWarpCache cache;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); i0 < n; i0 += stride) {
        const uint32_t i = i0 + lane;
        const bool valid = i < n;
        unsigned long long key = 0;
        uint32_t sl = 0;
        if (valid) {
            const unsigned long long e = nodes.ukeys[i];  // parent slot << 1 | bit
            const uint32_t p = uint32_t(e >> 1), bit = uint32_t(e & 1);
            const double pv = parent.prev[p], cur = parent.cur[p];
            key = parent.key[p] | ((bit && bit_pos < 64) ? (1ull << bit_pos) : 0ull);
            sl = nodes.uslot[i];
            na.key[sl] = key;
            na.prev[sl] = bit ? __dsub_rn(pv, cur) : cur;
        }
        // the value depends only on the parameters the tensor reads: fewer distinct keys to contract
        const uint32_t ks = dedup_insert_warp(keys, dedup_null_reduce(key & read_mask, null, n_null), valid, lane, cache);
        if (valid) na.kslot[sl] = ks;
    }
}

// Decision records once the level's keys are contracted (values by key slot).
__global__ void dedup_node_decide_kernel(DedupTable nodes, const double *__restrict__ value, DedupNodeArrays na,
                                         DedupTable next, bool insert_next) {
    const uint32_t n = min(*nodes.count, nodes.max_ids);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t sl = nodes.uslot[i];
        const double cur = value[na.kslot[sl]];
        na.cur[sl] = cur;
        na.rec[sl] = node_rec(cur, na.prev[sl], sl, next, insert_next);
    }
}

struct DedupNodePassArgs {
    uint64_t seed, first_shot, shots;
    uint32_t k0_round[10];
    uint32_t ci, j, out;
    uint32_t *slot;             // [shots] slot in `cur` (replaced by the slot in `next`)
    DedupTable cur, next;
    bool insert_next;
    const DedupNodeRec *rec;
    uint32_t *out32;
    uint64_t out_ld32;
    unsigned long long *counts;
    const double *uniforms;
    uint64_t uniforms_ld, upos;
    unsigned long long *err;
    // main-lineage speculation (dedup_init_spec_kernel): the pass visits only the active
    // shots (active[i], slot[i] for i < *n_active); every record word already holds the
    // main lineage's bit main_bit, an active shot whose bit differs flips its own bit
    const uint32_t *active;
    const uint32_t *n_active;
    uint32_t main_bit;
};

// One position for every shot: lane = shots s + 32 g (G groups per warp
// iteration, packed into 64/128-bit output stores by lane 0).
#ifndef ZXS_NODE_G
#define ZXS_NODE_G 4
#endif
constexpr int kNodePassG = ZXS_NODE_G;  // 4 or 8
static_assert(kNodePassG % 4 == 0, "node pass stores 128-bit groups of four 32-shot words");
#ifndef ZXS_NODE_ACT_MINB
#define ZXS_NODE_ACT_MINB 3  // measured: 3 (80 registers) beats 1 (108): node passes + init 23.1 -> 20.4 ms per 2^28 config-3 shots
#endif
template <bool ACT>
__global__ void __launch_bounds__(256, ACT ? ZXS_NODE_ACT_MINB : 1) dedup_node_pass_kernel(const __grid_constant__ DedupNodePassArgs a) {
    constexpr int G = kNodePassG;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t seed_hi = uint32_t(a.seed >> 32);
    const uint32_t k2c = uint32_t(kP1c) ^ a.k0_round[1];
    const uint32_t stream = 0x80000000u ^ (a.ci << 12) ^ a.j;  // sampler.cpp:37-39
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * G;
    unsigned long long ones = 0;
    DedupWarpCache cache;
    const uint64_t shots64 = (a.shots + 63) & ~uint64_t(63);
    // this batch's record words (a split batch's rows continue past them: out_ld32 is only the stride)
    const uint64_t out_words = min(a.out_ld32, shots64 / 32);
    const uint64_t n_items = ACT ? uint64_t(*a.n_active) : shots64;
    int delta = 0;  // ACT: ones minus the main lineage's, this lane's shots
    for (uint64_t s0 = (uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u)) * G; s0 < n_items; s0 += stride) {
        uint64_t s[G], idx[G];
        bool valid[G], bit[G];
        uint32_t node[G];
#pragma unroll
        for (int g = 0; g < G; g++) {
            idx[g] = s0 + 32 * g + lane;
            if (ACT) {
                valid[g] = idx[g] < n_items;
                s[g] = valid[g] ? __ldg(a.active + idx[g]) : 0ull;
            } else {
                s[g] = idx[g];
                valid[g] = s[g] < a.shots;
            }
            // node arrays are indexed by table slot (measured: prefetching the next iteration's slots,
            // or 8 shots per lane, is slower)
            node[g] = valid[g] ? __ldg(a.slot + idx[g]) : 0u;
        }
        DedupNodeRec r[G];
        bool need = false;  // a draw is needed unless every node's bit is certain (T = 0 or 2^53, no error)
#pragma unroll
        for (int g = 0; g < G; g++) {
            r[g] = a.rec[node[g]];
            need |= valid[g] && r[g].child == kNodeDraw;
        }
        unsigned long long k[G];
        if (a.uniforms) {
#pragma unroll
            for (int g = 0; g < G; g++) k[g] = 0;
        } else if (__any_sync(kFull, need)) {
            PhiloxPre pre[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                const uint64_t shot = a.first_shot + s[g];
                pre[g] = philox_pre(uint32_t(shot), uint32_t(shot >> 32), a.k0_round[0]);
            }
            uint32_t rhi[G], rlo[G];
            philox_tail<G>(pre, seed_hi ^ stream, a.k0_round, k2c, a.k0_round[9], rhi, rlo);
#pragma unroll
            for (int g = 0; g < G; g++) k[g] = ((uint64_t(rhi[g]) << 32) | rlo[g]) >> 11;  // uniform_at = k 2^-53
        } else {
#pragma unroll
            for (int g = 0; g < G; g++) k[g] = 0;  // unused: every T is 0 or 2^53
        }
        uint32_t word[G];
#pragma unroll
        for (int g = 0; g < G; g++) {
            bit[g] = false;
            if (valid[g]) {
                const unsigned long long T = r[g].T & ~kNodeErr;
                if (a.uniforms) {
                    const double u = a.uniforms[a.upos * a.uniforms_ld + s[g]];
                    bit[g] = !(u < r[g].cl);
                    if (fabs(u - r[g].cl) <= 1e-9 * fmax(r[g].cl, 1e-300)) atomicAdd(&a.err[2], 1ull);
                } else {
                    bit[g] = k[g] >= T;
                    if (k[g] - r[g].tie_lo <= r[g].tie_w) atomicAdd(&a.err[2], 1ull);
                }
                if (r[g].T & kNodeErr) report_ratio_error(a.err, a.first_shot + s[g]);
            }
            if (!ACT) word[g] = __ballot_sync(kFull, bit[g]);
        }
        if (ACT) {
#pragma unroll
            for (int g = 0; g < G; g++) {
                if (valid[g] && uint32_t(bit[g]) != a.main_bit) {
                    delta += bit[g] ? 1 : -1;
                    if (a.out32 && (s[g] >> 5) < out_words) {
                        atomicXor(a.out32 + a.out * a.out_ld32 + (s[g] >> 5), 1u << (s[g] & 31));
                    }
                }
            }
        } else if (lane == 0) {
            const uint64_t w0 = s0 >> 5;
            if (a.out32) {
                uint32_t *row = a.out32 + a.out * a.out_ld32;
                if (w0 + G <= out_words && (reinterpret_cast<uintptr_t>(row + w0) & 15) == 0) {
#pragma unroll
                    for (int g = 0; g < G; g += 4) {
                        *reinterpret_cast<uint4 *>(row + w0 + g) = make_uint4(word[g], word[g + 1], word[g + 2], word[g + 3]);
                    }
                } else {
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        if (w0 + g < out_words) row[w0 + g] = word[g];
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < G; g++) ones += __popc(word[g]);
        }
        if (a.insert_next) {
#pragma unroll
            for (int g = 0; g < G; g++) {
                const unsigned long long e = (unsigned long long)node[g] << 1 | (bit[g] ? 1ull : 0ull);
                // a certain bit's child was inserted by the decide kernel (an injected uniform
                // outside [0, 1) can still take the other bit)
                const bool known = r[g].child < kNodeNoChild && bit[g] == ((r[g].T & ~kNodeErr) == 0ull);
                const uint32_t ns = dedup_insert_warp(a.next, e, valid[g] && !known, lane, cache);
                if (valid[g]) a.slot[idx[g]] = known ? r[g].child : ns;
            }
        }
    }
    if (ACT) {
        // every shot's word was written with the main lineage's bit: shots x main_bit, then the deltas
        if (a.counts && blockIdx.x == 0 && threadIdx.x == 0 && a.main_bit) atomicAdd(&a.counts[a.out], a.shots);
        const int d = __reduce_add_sync(kFull, delta);
        if (a.counts && lane == 0 && d) atomicAdd(&a.counts[a.out], (unsigned long long)(long long)d);
    } else if (a.counts && lane == 0 && ones) {
        atomicAdd(&a.counts[a.out], ones);
    }
}

// ---- fused chain (short chains): every position's keys are the base keys
// (f bits) times the patterns of the sampled bits the tensor reads, so all
// tensors are contracted before any draw and one per-shot kernel runs the
// whole autoregressive chain with its state in registers.
constexpr uint32_t kDedupMaxFused = 6;  // outputs per fused chain

// keys_out[id * P + pat] = base key id | pattern bits at their raw parameter positions.
__global__ void dedup_expand_kernel(const unsigned long long *__restrict__ ukeys0, const uint32_t *n0, uint32_t nbits,
                                    uint64_t relpos, uint32_t cap, unsigned long long *__restrict__ keys_out) {
    const uint32_t P = 1u << nbits;
    const uint32_t n = uint32_t(min(uint64_t(*n0) * P, uint64_t(cap)));
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        unsigned long long key = __ldg(ukeys0 + (k >> nbits));
        for (uint32_t b = 0; b < nbits; b++) {
            if ((k >> b) & 1u) key |= 1ull << ((relpos >> (8 * b)) & 0xffu);
        }
        keys_out[k] = key;
    }
}

struct DedupFusedArgs {
    uint64_t seed, first_shot, shots;
    uint32_t k0_round[10];
    uint32_t ci, n_out;
    uint32_t out[kDedupMaxFused];
    uint32_t relevant;           // bit j: a later tensor reads sampled bit j
    const uint32_t *slot;        // [shots] slot in the base table
    const uint32_t *ids;         // base table: slot -> id
    const double *value[kDedupMaxFused + 1];  // tensor pos: [id << nb + pattern]
    uint32_t value_cap;                       // entries per value array
    uint32_t *out32;
    uint64_t out_ld32;
    unsigned long long *counts;
    const double *uniforms;
    uint64_t uniforms_ld, upos_base;
    unsigned long long *err;
};

// The whole chain (sampler.cpp:84-99) per shot: lane = shots s, s + 32.
// (Drawing every position's uniform first and loading both candidates of the
// next position while deciding this one measured slower: 102 registers.)
#ifndef ZXS_FUSED_G
#define ZXS_FUSED_G 1  // measured: 1 < 2 < 4 shots per lane in time (register pressure)
#endif
__global__ void __launch_bounds__(256) dedup_fused_ar_kernel(const __grid_constant__ DedupFusedArgs a) {
    constexpr int G = ZXS_FUSED_G;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t seed_hi = uint32_t(a.seed >> 32);
    const uint32_t k2c = uint32_t(kP1c) ^ a.k0_round[1];
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * G;
    unsigned long long ones[kDedupMaxFused] = {};
    const uint64_t shots64 = (a.shots + 63) & ~uint64_t(63);
    // this batch's record words (a split batch's rows continue past them: out_ld32 is only the stride)
    const uint64_t out_words = min(a.out_ld32, shots64 / 32);
    for (uint64_t s0 = (uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u)) * G; s0 < shots64; s0 += stride) {
        uint64_t s[G];
        bool valid[G];
        uint32_t id[G], pat[G];
        double prev[G];
#pragma unroll
        for (int g = 0; g < G; g++) {
            s[g] = s0 + 32 * g + lane;
            valid[g] = s[g] < a.shots;
            id[g] = valid[g] ? a.ids[a.slot[s[g]]] : 0u;
            prev[g] = a.value[0][min(id[g], a.value_cap - 1)];
            pat[g] = 0;
        }
        uint32_t nb = 0;
#pragma unroll 1
        for (uint32_t j = 0; j < a.n_out; j++) {
            const uint32_t stream = 0x80000000u ^ (a.ci << 12) ^ j;  // sampler.cpp:37-39
            double u[G];
            if (a.uniforms) {
#pragma unroll
                for (int g = 0; g < G; g++) u[g] = valid[g] ? a.uniforms[(a.upos_base + j) * a.uniforms_ld + s[g]] : 0.0;
            } else {
                PhiloxPre pre[G];
#pragma unroll
                for (int g = 0; g < G; g++) {
                    const uint64_t shot = a.first_shot + s[g];
                    pre[g] = philox_pre(uint32_t(shot), uint32_t(shot >> 32), a.k0_round[0]);
                }
                uint32_t rhi[G], rlo[G];
                philox_tail<G>(pre, seed_hi ^ stream, a.k0_round, k2c, a.k0_round[9], rhi, rlo);
#pragma unroll
                for (int g = 0; g < G; g++) u[g] = philox_uniform((uint64_t(rhi[g]) << 32) | rlo[g]);
            }
            const double *vj = a.value[j + 1];
            bool bit[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                bit[g] = false;
                if (valid[g]) {
                    // clamped: after a table overflow (the host redoes the batch) ids can exceed the
                    // values the round computed; the garbage pass must stay in bounds
                    const double cur = vj[min((id[g] << nb) | pat[g], a.value_cap - 1)];
                    bit[g] = ar_decide(cur, prev[g], u[g], a.err, a.first_shot + s[g]);
                    prev[g] = bit[g] ? __dsub_rn(prev[g], cur) : cur;
                }
                const uint32_t word = __ballot_sync(kFull, bit[g]);
                if (lane == 0) {
                    const uint64_t wi = (s0 >> 5) + g;
                    if (a.out32 && wi < out_words) a.out32[a.out[j] * a.out_ld32 + wi] = word;
#pragma unroll
                    for (uint32_t q = 0; q < kDedupMaxFused; q++) {
                        if (q == j) ones[q] += __popc(word);
                    }
                }
            }
            if ((a.relevant >> j) & 1u) {
#pragma unroll
                for (int g = 0; g < G; g++) pat[g] |= uint32_t(bit[g]) << nb;
                nb++;
            }
        }
    }
    if (a.counts && lane == 0) {
#pragma unroll
        for (uint32_t q = 0; q < kDedupMaxFused; q++) {
            if (q < a.n_out && ones[q]) atomicAdd(&a.counts[a.out[q]], ones[q]);
        }
    }
}

}  // namespace zxs_dev
