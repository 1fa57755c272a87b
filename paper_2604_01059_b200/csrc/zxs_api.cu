// zxs_api.cu — C-ABI implementation (include/zxs_b200.h): model upload and
// kernel launches. Host-side preprocessing turns the reference's
// floating-point draw rules into exact integer thresholds:
//
//   single mechanism  fire iff u < p              (sampler.cpp:272)
//   joint mechanism   first o with u < sum_{j<=o} table[j], else 0
//                                                  (sampler.cpp:283-293)
//
// with u = k * 2^-53 and k = r01 >> 11 (rng.hpp:35-37). Since scaling by a
// power of two is exact, u < x  <=>  k < ceil(x * 2^53) =: T(x), and
// k < T  <=>  r01 <= T * 2^11 - 1 =: lim. The cumulative sums are formed
// with the same sequential double additions as the reference, so the integer
// compare on the device reproduces every draw bit for bit. Outcomes that can
// never be first (T not above the running maximum) are dropped, as are
// mechanisms that cannot change f; their Philox streams are keyed by the
// reference's mechanism index, so dropping them changes no other draw.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <chrono>
#include <limits>
#include <unordered_map>
#include <iterator>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "zxs_b200.h"
#include "zxs_heavy.cuh"
#include "zxs_mono.cuh"
#include "zxs_dedup.cuh"
#include "zxs_encode.cuh"
#include "zxs_sparse.cuh"

using zxs_dev::DevModel;
using zxs_dev::Factor;

namespace {

thread_local std::string g_last_error;

struct ZxsError {
    zxs_status status;
    std::string msg;
};

[[noreturn]] void fail(zxs_status st, const std::string &msg) { throw ZxsError{st, msg}; }

void cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        zxs_status st = e == cudaErrorMemoryAllocation ? ZXS_OUT_OF_MEMORY : ZXS_CUDA_ERROR;
        fail(st, std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define CK(x) cuda_check((x), #x)

template <typename F>
zxs_status guarded(F &&f) {
    try {
        f();
        return ZXS_OK;
    } catch (const ZxsError &e) {
        g_last_error = e.msg;
        return e.status;
    } catch (const std::bad_alloc &) {
        g_last_error = "host allocation failed";
        return ZXS_OUT_OF_MEMORY;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return ZXS_RUNTIME_ERROR;
    }
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        CK(cudaGetDevice(&prev));
        if (prev != dev) CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

uint64_t threshold_of(double x) {
    if (!(x > 0.0)) return 0;                      // u < x never holds (also NaN)
    if (x >= 1.0) return uint64_t(1) << 53;        // u < x always holds
    return static_cast<uint64_t>(std::ceil(std::ldexp(x, 53)));
}

uint64_t lim_of(uint64_t T) {  // T in [1, 2^53]
    return (T << 11) - 1;      // T = 2^53 wraps to 2^64 - 1: always fires
}

struct Arena {
    std::vector<char> host;
    template <typename T>
    size_t add(const T *data, size_t n) {
        size_t off = (host.size() + 255) & ~size_t(255);
        host.resize(off + n * sizeof(T));
        if (n) std::memcpy(host.data() + off, data, n * sizeof(T));
        return off;
    }
    template <typename T>
    size_t add(const std::vector<T> &v) {
        return add(v.data(), v.size());
    }
};

}  // namespace

struct zxs_sampler {
    int device = 0;
    uint32_t mode = 0;
    int fw_template = 1;
    int shots_per_lane = 2;  // shot_kernel S (ZXS_SHOTS_PER_LANE)
    DevModel m{};
    zxs_sampler_info info{};
    bool all_outputs_covered = true;
    uint32_t num_tensors = 0;
    std::vector<uint32_t> tensor_width;
    std::vector<uint32_t> comp_out_begin, comp_tensor_begin, comp_outputs;
    std::vector<uint32_t> direct_out;
    char *dev_model = nullptr;
    size_t dev_model_bytes = 0;
    bool param_mechs = true;
    std::unique_ptr<zxs_dev::MechTable<zxs_dev::kParamMechs>> mech_table;
    std::unique_ptr<zxs_dev::MechTable<1>> mech_table1;  // parameter block of the global-mechanism variant
    uint32_t light_tables = 0;                          // h tables staged in smem (LightProg valid)
    double *dev_tab = nullptr;                          // tabulated chains (LightProg.tab)
    const zxs_dev::MechRec *mech_global = nullptr;
    const zxs_dev::MechFast *fast_global = nullptr;
    const uint32_t *ext_begin = nullptr;
    const ulonglong2 *ext = nullptr;
    uint32_t dead_mechanisms = 0;
    unsigned long long *dev_err = nullptr;  // [3]: ratio breakdown flag, first shot, near-tie draws
    cudaStream_t stream = nullptr, copy_stream = nullptr;
    cudaEvent_t ev_done[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
    char *scratch = nullptr;
    size_t scratch_bytes = 0;
    int sm_count = 148;
    int blocks_per_sm = 1;
    std::mutex mu;
    // heavy (large-chi) components, see zxs_heavy.cuh
    bool has_heavy = false;
    zxs_dev::HeavyArgs heavy{};
    size_t heavy_smem = 0;
    int heavy_blocks_per_sm = 0;
    uint64_t heavy_words = 0;
    char *heavy_scratch = nullptr;
    size_t heavy_scratch_bytes = 0;

    // large-chi components on the integer monomial path, see zxs_mono.cuh
    bool has_mono = false;
    int mono_nw = 2;  // 32-shot words per lane in mono_kernel (ZXS_MONO_WORDS)
    zxs_dev::MonoArgs mono{};
    size_t mono_smem = 0;
    int mono_blocks_per_sm = 0;
    std::map<uint32_t, uint32_t> mono_tensor;  // model tensor -> mono tensor index
    char *mono_scratch = nullptr;
    size_t mono_scratch_bytes = 0;

    // deduplicated large-chi path (zxs_dedup.cuh; ZXS_DEDUP, default on)
    bool dedup = false;
    const uint32_t *dd_words = nullptr;  // segment streams (device)
    const uint4 *dd_segs = nullptr;
    std::vector<uint32_t> dd_tsb, dd_tdb, dd_tw, dd_tbb;  // host copies per mono tensor
    std::vector<unsigned long long> dd_key_mask;          // per mono component (local parameters)
    std::vector<uint16_t> dd_param_map;                   // MonoHost::param_map
    std::vector<unsigned long long> dd_tread;             // per mono tensor: local parameters it reads
    const unsigned long long *dd_null = nullptr;          // device: null pairs of every mono tensor
    std::vector<uint32_t> dd_null_begin;                  // per mono tensor: first pair (2 words each), then the end
    // main-lineage speculation (dedup_init_spec_kernel): per mono component, the node
    // records of the all-zero key's likelier-bit chain, computed on first use
    struct Lineage {
        bool done = false, ok = false;
        uint32_t bits = 0;
        unsigned long long T[zxs_dev::kSpecMaxChain], tie_lo[zxs_dev::kSpecMaxChain];
        uint32_t tie_w[zxs_dev::kSpecMaxChain];
    };
    std::vector<Lineage> dd_lineage;
    bool dd_spec = true;                                  // ZXS_DEDUP_SPEC=0: every shot through the node passes
    char *dd_spec_dev = nullptr;                          // 64 B: one key, one value, one node record
    std::vector<uint32_t> dd_tspw;                        // per mono tensor: segments per warp per eval item
    uint32_t dd_stack_words = 0;                          // dedup_eval_kernel stack area (words)
    std::vector<uint4> dd_t_layout;                       // per mono tensor: {table bytes, segbuf words, stage, smem}
    bool dd_identity_map = true;                          // every mono component's local params = raw
    size_t dd_smem = 0;
    const uint32_t *dd_block_forms = nullptr, *dd_block_form_begin = nullptr;
    std::vector<uint32_t> dd_tfb;    // per mono tensor: first block form table (~0: dictionary ids)
    int dd_init_occ = 1, dd_ar_occ = 1, dd_fused_occ = 1, dd_raw_occ = 1, dd_node_occ = 1, dd_node_act_occ = 1, dd_spec_occ = 1;  // resident blocks per SM (per-shot dedup kernels)
    bool dd_async = true;                 // key counts stay on the device (ZXS_DEDUP_SYNC=1: host round trips)
    bool dd_fused = true;                 // short chains in one per-shot kernel (ZXS_DEDUP_FUSED=0: step by step)
    unsigned long long *dd_dev_stats = nullptr;  // {keys, plane-load bytes} accumulated by dedup_eval_kernel
    char *dd_buf = nullptr;  // keys, slots, prev, values, partials, two tables
    size_t dd_buf_bytes = 0;
    uint64_t dd_cap_shots = 0;
    uint32_t dd_table_slots = 0;
    bool dd_dirty = true;  // tables need a full reset
    uint32_t *dd_pinned = nullptr;
    std::vector<uint64_t> dd_tloads;  // per mono tensor: plane loads per 32-key word
    uint64_t dd_stats[5] = {};        // batches, fallbacks, evaluated keys, plane-load bytes, eval launches

    // error model kept on the host for probability_of's enumeration
    // (sampler.cpp:370-429): per mechanism the f_vectors as FW-word masks and
    // either the probability (single) or the outcome table (joint).
    struct HostMech {
        bool joint = false;
        double p = 0.0;
        std::vector<double> table;
        std::vector<std::vector<uint64_t>> vecs;
    };
    std::vector<HostMech> host_mechs;
    std::vector<uint64_t> host_base;

    // sparse geometric path (sampler.cpp:104-147, 214-255)
    uint32_t model_flags = 0;
    bool sparse_structural = false;     // pure-Clifford deterministic, all singles with p < 1
    double sparse_expected_flips = 0;   // sum_m p_m |flips(m)|  (sampler.cpp:112-114)
    std::vector<uint32_t> const_one_outputs;  // direct outputs whose constant part is 1
    double *dev_log1mp = nullptr;
    uint32_t *dev_flip_begin = nullptr, *dev_flip_out = nullptr;

    // per-kernel CUDA-event timing (zxs_kernel_timing / zxs_kernel_times)
    bool timing = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> timed;
    void time_begin(int which, cudaStream_t st, cudaEvent_t &e0) {
        if (!timing) return;
        CK(cudaEventCreate(&e0));
        CK(cudaEventRecord(e0, st));
        (void)which;
    }
    void time_end(int which, cudaStream_t st, cudaEvent_t e0) {
        if (!timing) return;
        cudaEvent_t e1;
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e1, st));
        timed.push_back({which, {e0, e1}});
    }

    double *mono_scratch_get(size_t bytes) {
        if (bytes > mono_scratch_bytes) {
            if (mono_scratch) CK(cudaFree(mono_scratch));
            mono_scratch = nullptr;
            mono_scratch_bytes = 0;
            CK(cudaMalloc(&mono_scratch, bytes));
            mono_scratch_bytes = bytes;
        }
        return reinterpret_cast<double *>(mono_scratch);
    }

    uint32_t *heavy_fcols_get(size_t bytes) {
        if (bytes > heavy_scratch_bytes) {
            if (heavy_scratch) CK(cudaFree(heavy_scratch));
            heavy_scratch = nullptr;
            heavy_scratch_bytes = 0;
            CK(cudaMalloc(&heavy_scratch, bytes));
            heavy_scratch_bytes = bytes;
        }
        return reinterpret_cast<uint32_t *>(heavy_scratch);
    }

    char *scratch_get(size_t bytes) {
        if (bytes > scratch_bytes) {
            if (scratch) CK(cudaFree(scratch));
            scratch = nullptr;
            scratch_bytes = 0;
            CK(cudaMalloc(&scratch, bytes));
            scratch_bytes = bytes;
        }
        return scratch;
    }
};

namespace {

template <int FW, int S>
const void *kernel_ptr(bool param_mechs) {
    return param_mechs ? reinterpret_cast<const void *>(&zxs_dev::shot_kernel<FW, true, S>)
                       : reinterpret_cast<const void *>(&zxs_dev::shot_kernel<FW, false, S>);
}

// S = shots per lane: 4 for narrow f (FW <= 2: the f register file stays small),
// else 2.
const void *shot_kernel_for(int fw, bool param_mechs, int S) {
    if (S == 4) {
        if (fw == 1) return kernel_ptr<1, 4>(param_mechs);
        if (fw == 2) return kernel_ptr<2, 4>(param_mechs);
    }
    switch (fw) {
        case 1: return kernel_ptr<1, 2>(param_mechs);
        case 2: return kernel_ptr<2, 2>(param_mechs);
        case 4: return kernel_ptr<4, 2>(param_mechs);
        case 8: return kernel_ptr<8, 2>(param_mechs);
        case 16: return kernel_ptr<16, 2>(param_mechs);
    }
    fail(ZXS_UNSUPPORTED, "f_width above 1024 is not supported");
}

constexpr int kThreads = 256;

size_t shot_smem_bytes(const zxs_sampler *s) {  // one warp per CTA
    const size_t sh_off = (2 * size_t(s->m.num_outputs) + 3) & ~size_t(3);
    return (sh_off + 16 * size_t(s->light_tables)) * 4 + size_t(s->shots_per_lane) * s->m.col_stride * 4;
}

void validate_csr(const char *name, const uint32_t *b, size_t n, size_t total) {
    if (!b) fail(ZXS_INVALID_ARGUMENT, std::string(name) + " is null");
    if (b[0] != 0) fail(ZXS_INVALID_ARGUMENT, std::string(name) + "[0] != 0");
    for (size_t i = 0; i < n; i++) {
        if (b[i + 1] < b[i]) fail(ZXS_INVALID_ARGUMENT, std::string(name) + " not monotone");
    }
    if (total != SIZE_MAX && b[n] != total) fail(ZXS_INVALID_ARGUMENT, std::string(name) + " total mismatch");
}
void validate_csr64(const char *name, const uint64_t *b, size_t n) {
    if (!b) fail(ZXS_INVALID_ARGUMENT, std::string(name) + " is null");
    if (b[0] != 0) fail(ZXS_INVALID_ARGUMENT, std::string(name) + "[0] != 0");
    for (size_t i = 0; i < n; i++) {
        if (b[i + 1] < b[i]) fail(ZXS_INVALID_ARGUMENT, std::string(name) + " not monotone");
    }
}

// Host encoding of the heavy (large-chi) components for heavy_kernel: one
// compact word stream per chain tensor, cut into chunks on term boundaries
// (see zxs_heavy.cuh for the record layout). Components with fewer than
// `heavy_min` factors, or that do not fit the envelope (<= 256 plane rows,
// <= 256 h tables, terms smaller than a chunk), stay on the shot kernel.
struct HeavyHost {
    std::vector<uint8_t> comp_heavy;
    std::vector<uint32_t> words;
    std::vector<uint4> chunks;
    std::vector<uint32_t> tensor_chunk_begin{0};
    std::vector<zxs_dev::HeavyComp> comps;
    uint32_t max_chain = 0, zero_row = 0;
};

HeavyHost encode_heavy(const zxs_model_desc *d, uint32_t max_chain, uint64_t heavy_min,
                       const std::vector<uint8_t> *skip = nullptr) {
    HeavyHost H;
    std::vector<uint8_t> &comp_heavy = H.comp_heavy;
    std::vector<uint32_t> &hw = H.words;
    std::vector<uint4> &hchunks = H.chunks;
    std::vector<uint32_t> &htcb = H.tensor_chunk_begin;
    std::vector<zxs_dev::HeavyComp> &hcomps = H.comps;
    uint32_t &heavy_max_chain = H.max_chain;
    const uint32_t fwid = d->f_width;
    comp_heavy.assign(std::max<uint32_t>(1, d->num_components), 0);
    // plane rows: f columns, sampled-bit columns of the longest chain, one all-zero row
    const uint32_t heavy_zero_row = fwid + max_chain;
    H.zero_row = heavy_zero_row;
    {
        uint32_t upos = 0;
        for (uint32_t c = 0; c < d->num_components; c++) {
            const uint32_t n = d->comp_out_begin[c + 1] - d->comp_out_begin[c];
            const uint32_t t0 = d->comp_tensor_begin[c], t1 = d->comp_tensor_begin[c + 1];
            uint64_t nf = d->term_factor_begin[d->tensor_term_begin[t1]] - d->term_factor_begin[d->tensor_term_begin[t0]];
            bool ok = nf >= heavy_min && d->num_h_tables <= 256 && hcomps.size() < size_t(zxs_dev::kMaxHeavyComps) &&
                      heavy_zero_row < 256 && !(skip && (*skip)[c]);
            // encode every tensor of the chain; abandon (light path) on any misfit
            std::vector<uint32_t> w;
            std::vector<uint4> ch;
            std::vector<uint32_t> tcb;
            for (uint32_t t = t0; ok && t < t1; t++) {
                uint32_t cur_begin = uint32_t(hw.size() + w.size()), cur_terms = 0;
                auto close_chunk = [&]() {
                    if (hw.size() + w.size() == cur_begin) w.insert(w.end(), 4, 0u);  // no 0-byte bulk copies
                    while ((hw.size() + w.size()) % 4) w.push_back(0);
                    uint32_t end = uint32_t(hw.size() + w.size());
                    ch.push_back(make_uint4(cur_begin, end - cur_begin, cur_terms, 0));
                    cur_begin = end;
                    cur_terms = 0;
                };
                tcb.push_back(uint32_t(hchunks.size() + ch.size()));
                for (uint64_t term = d->tensor_term_begin[t]; ok && term < d->tensor_term_begin[t + 1]; term++) {
                    std::vector<uint32_t> tw;
                    const uint64_t f0 = d->term_factor_begin[term], f1 = d->term_factor_begin[term + 1];
                    uint64_t re, im;
                    std::memcpy(&re, &d->term_c[2 * term], 8);
                    std::memcpy(&im, &d->term_c[2 * term + 1], 8);
                    // term: {nfac, re.lo, re.hi, im.lo}, {im.hi, 0, 0, 0}
                    tw.insert(tw.end(), {uint32_t(f1 - f0), uint32_t(re), uint32_t(re >> 32), uint32_t(im),
                                         uint32_t(im >> 32), 0u, 0u, 0u});
                    for (uint64_t k = f0; ok && k < f1; k++) {
                        const uint64_t u0 = d->factor_u_begin[k], u1 = d->factor_u_begin[k + 1];
                        const uint64_t v0 = d->factor_v_begin[k], v1 = d->factor_v_begin[k + 1];
                        const uint32_t gu = uint32_t((u1 - u0 + 3) / 4), gv = uint32_t((v1 - v0 + 3) / 4);
                        if (gu > 255 || gv > 255) {
                            ok = false;
                            break;
                        }
                        // factor: {table | u groups << 8 | v groups << 16, 0, 0, 0}, then groups of
                        // four byte offsets (param * 64) into the 16-bit parameter planes; padding
                        // entries point at the all-zero row `heavy_zero_row`.
                        tw.insert(tw.end(), {d->factor_table[k] | gu << 8 | gv << 16, 0u, 0u, 0u});
                        auto put_group = [&](const uint32_t *bits, uint64_t n) {
                            for (uint64_t i = 0; i < 4 * ((n + 3) / 4); i++) {
                                tw.push_back(64u * (i < n ? bits[i] : heavy_zero_row));
                            }
                        };
                        put_group(d->factor_u_bits + u0, u1 - u0);
                        put_group(d->factor_v_bits + v0, v1 - v0);
                    }
                    if (!ok) break;
                    if (tw.size() + 4 > zxs_dev::kChunkWords) {
                        ok = false;  // a single term larger than a chunk buffer
                        break;
                    }
                    if (hw.size() + w.size() + tw.size() - cur_begin > zxs_dev::kChunkWords) close_chunk();
                    w.insert(w.end(), tw.begin(), tw.end());
                    cur_terms++;
                }
                if (ok && (cur_terms || hw.size() + w.size() == cur_begin)) close_chunk();
            }
            if (ok) {
                zxs_dev::HeavyComp hc;
                hc.ci = c;
                hc.n_out = n;
                hc.upos_base = upos;
                hc.out_begin = d->comp_out_begin[c];
                hc.first_tensor = uint32_t(htcb.size() - 1);
                hw.insert(hw.end(), w.begin(), w.end());
                hchunks.insert(hchunks.end(), ch.begin(), ch.end());
                for (size_t i = 1; i < tcb.size(); i++) htcb.push_back(tcb[i]);
                htcb.push_back(uint32_t(hchunks.size()));
                hcomps.push_back(hc);
                comp_heavy[c] = 1;
                heavy_max_chain = std::max(heavy_max_chain, n);
            }
            upos += n;
        }
    }
    if (hw.empty()) hw.assign(4, 0);
    if (hchunks.empty()) hchunks.push_back(make_uint4(0, 0, 0, 0));
    return H;
}

// ---------------------------------------------------------------- monomial path
// Exact value of h(a,b) for a table with alpha = pa*pi/2, beta = pb*pi/2
// (scalar.cpp:81-85): h = 1 + x + y - xy = 2 - (1-x)(1-y), x = i^(pa+2a),
// y = i^(pb+2b), as a Gaussian integer; then 0 or 2^(m/2) w^k.
struct MonoEntry {
    bool zero;
    int m, k;  // h = 2^(m/2) w^k
    int re, im;
};

MonoEntry mono_entry(int pa, int pb, int a, int b) {
    static const int ire[4] = {1, 0, -1, 0}, iim[4] = {0, 1, 0, -1};
    const int jx = (pa + 2 * a) & 3, jy = (pb + 2 * b) & 3;
    const int x1 = 1 - ire[jx], y1 = -iim[jx], x2 = 1 - ire[jy], y2 = -iim[jy];
    const int pr = x1 * x2 - y1 * y2, pi = x1 * y2 + y1 * x2;
    MonoEntry e{false, 0, 0, 2 - pr, -pi};
    if (e.re == 0 && e.im == 0) {
        e.zero = true;
        return e;
    }
    const int n2 = e.re * e.re + e.im * e.im;
    e.m = n2 == 4 ? 2 : (n2 == 8 ? 3 : -1);
    static const int kr[8] = {2, 2, 0, -2, -2, -2, 0, 2}, ki[8] = {0, 2, 2, 2, 0, -2, -2, -2};
    e.k = -1;
    for (int k = 0; k < 8; k++) {
        if (kr[k] == e.re && ki[k] == e.im) e.k = k;
    }
    return e;
}

// mono_kernel configurations: 2 = two 32-shot words per lane, 12 warps; 1 = one word, 16 warps;
// 3 = one word, 4 warps (narrow: large dictionaries / many parameter planes)
int mono_words(int cfg) { return cfg == 2 ? 2 : 1; }
int mono_warps(int cfg) {
    return cfg == 2 ? zxs_dev::MonoCfg<2>::kWarps : cfg == 1 ? zxs_dev::MonoCfg<1>::kWarps : 4;
}

size_t mono_smem_bytes(uint32_t n_planes, uint32_t max_dict, int cfg, uint32_t depth) {
    return 128 + 2 * size_t(zxs_dev::kMonoChunkWords) * 4 + size_t(max_dict) * 16 +
           size_t(mono_warps(cfg)) * mono_words(cfg) * (size_t(depth) * 3 * 128 + size_t(n_planes) * 128);
}

const void *mono_kernel_ptr(int cfg) {
    return cfg == 2 ? reinterpret_cast<const void *>(&zxs_dev::mono_kernel<2>)
           : cfg == 1 ? reinterpret_cast<const void *>(&zxs_dev::mono_kernel<1>)
                      : reinterpret_cast<const void *>(&zxs_dev::mono_kernel<1, 4>);
}

struct MonoHost {
    std::vector<uint8_t> comp_mono;
    std::vector<uint32_t> words;
    std::vector<uint4> chunks;
    std::vector<uint32_t> tensor_chunk_begin{0};
    std::vector<uint4> dict;
    std::vector<zxs_dev::HeavyComp> comps;
    std::map<uint32_t, uint32_t> tensor_index;  // model tensor -> index into tensor_chunk_begin
    uint32_t max_chain = 0;
    uint64_t records = 0, dead_terms = 0, selectors = 0;
    uint64_t negligible_terms = 0;  // terms with |c'| < 2^-40 of their tensor's largest (dropped)
    uint64_t loads = 0;  // plane loads per 32-shot word for one pass over every mono chain tensor
    uint64_t nodes = 0;
    std::vector<uint32_t> tensor_dict_begin;  // first dictionary entry per mono tensor, then the total
    std::vector<uint32_t> tensor_width;       // param width per mono tensor
    std::vector<uint32_t> tensor_basis_begin; // first basis vector per mono tensor (W_t of them)
    std::vector<unsigned long long> basis;    // basis vectors: masks over the tensor's raw params
    uint32_t all_plane = 0;                    // plane index of the per-tensor ALL plane
    uint32_t max_dict = 1;
    uint32_t max_depth = 1;  // deepest tree node + 1
    // summation segments (zxs_dedup.cuh): per mono tensor, up to kDedupSegs
    // self-contained node streams (each replays its first node's ancestors)
    std::vector<uint32_t> seg_words;
    std::vector<uint4> segs;                   // {word_begin, n_words, n_nodes, 0}
    std::vector<uint32_t> tensor_seg_begin{0};
    std::vector<unsigned long long> comp_key_mask;  // per mono component: local params any tensor reads
    // component-local parameters: local p < nf -> raw f column param_map[pmap_begin + p];
    // local nf + j -> sampled bit j (param_map holds f_width + j). Identity when
    // f_width + chain <= 63, else the f columns the component's tensors read.
    std::vector<uint16_t> param_map;
    std::vector<uint64_t> tensor_loads;             // per mono tensor: plane loads per 32-shot word
    std::vector<unsigned long long> tensor_read_mask;  // per mono tensor: local parameters its forms read
    // per mono tensor: the null space of its forms inside the read mask, as pairs {1 << q, n_q}
    // (q a free parameter, n_q the null vector with bit q and otherwise pivot bits only); keys
    // that differ by a null vector give every form the same value, hence the same tensor value
    std::vector<uint32_t> tensor_null_begin{0};
    std::vector<unsigned long long> tensor_null;
    std::vector<uint32_t> tensor_spw;                  // per mono tensor: segments per warp per eval item
    // block form tables (dedup_eval_kernel): per block of kDedupWarps segments the
    // tensor dictionary entries its records use; segment streams carry block-local ids
    std::vector<uint32_t> block_forms;
    std::vector<uint32_t> block_form_begin{0};
    std::vector<uint32_t> tensor_first_block;  // per mono tensor
    uint32_t max_block_forms = 0;
};

// One term after lowering: its records as sorted tokens (record word, plus
// GEN aux word + 1 in the high half) and c' = c 2^(M/2) w^K0.
struct MonoTerm {
    std::vector<uint64_t> recs;
    double re = 0, im = 0;
};

struct MonoNode {
    uint32_t depth = 0;
    bool leaf = false;
    std::vector<uint64_t> recs;  // records applied on top of the parent's state
    double re = 0, im = 0;       // leaves: the term's c'
};

std::vector<uint64_t> ms_inter(const std::vector<uint64_t> &a, const std::vector<uint64_t> &b) {
    std::vector<uint64_t> r;
    std::set_intersection(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(r));
    return r;
}
std::vector<uint64_t> ms_diff(const std::vector<uint64_t> &a, const std::vector<uint64_t> &b) {
    std::vector<uint64_t> r;
    std::set_difference(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(r));
    return r;
}

// Shared-prefix tree over consecutive terms: a node covers a contiguous term
// range and carries the records common to all of them (multiset
// intersection) minus its parent's; leaves are the terms, in order, so a DFS
// in preorder visits the terms in the reference's summation order
// (phase_terms.cpp:129-131). J (mod 4) and Z are sums / ORs of independent
// record contributions, so a term's state = the union of the records on its
// root-to-leaf path. Children split the range into `fan` equal parts; the
// fan (or no tree at all) is chosen per tensor to minimise emitted words.
void mono_tree_rec(const std::vector<MonoTerm> &T, size_t lo, size_t hi, const std::vector<uint64_t> &parent,
                   uint32_t depth, uint32_t fan, std::vector<MonoNode> &out, uint64_t &cost) {
    MonoNode nd;
    nd.depth = depth;
    if (hi - lo == 1) {
        nd.leaf = true;
        nd.recs = ms_diff(T[lo].recs, parent);
        nd.re = T[lo].re;
        nd.im = T[lo].im;
        cost += 5 + nd.recs.size();
        out.push_back(std::move(nd));
        return;
    }
    std::vector<uint64_t> inter = T[lo].recs;
    for (size_t i = lo + 1; i < hi && !inter.empty(); i++) inter = ms_inter(inter, T[i].recs);
    nd.recs = ms_diff(inter, parent);
    cost += 1 + nd.recs.size();
    out.push_back(std::move(nd));
    const size_t n = hi - lo, parts = std::min<size_t>(fan, n);
    for (size_t p = 0; p < parts; p++) {
        const size_t a = lo + n * p / parts, b = lo + n * (p + 1) / parts;
        if (b > a) mono_tree_rec(T, a, b, inter, depth + 1, fan, out, cost);
    }
}

std::vector<MonoNode> mono_tree(const std::vector<MonoTerm> &T) {
    // flat: every term a leaf at depth 0
    std::vector<MonoNode> best;
    uint64_t best_cost = 0;
    for (const MonoTerm &t : T) {
        MonoNode nd;
        nd.leaf = true;
        nd.recs = t.recs;
        nd.re = t.re;
        nd.im = t.im;
        best_cost += 5 + nd.recs.size();
        best.push_back(std::move(nd));
    }
    if (T.size() < 4) return best;
    for (uint32_t fan : {2u, 3u, 4u, 6u, 8u, 16u}) {
        // depth bound: ceil(log_fan(N)) + 1 levels
        uint32_t depth = 1;
        for (size_t x = 1; x < T.size(); x *= fan) depth++;
        if (depth >= zxs_dev::kMonoMaxDepth) continue;
        std::vector<MonoNode> nodes;
        uint64_t cost = 0;
        mono_tree_rec(T, 0, T.size(), {}, 0, fan, nodes, cost);
        if (cost < best_cost) {
            best_cost = cost;
            best = std::move(nodes);
        }
    }
    return best;
}

// Lowers every eligible large component to the record streams of
// zxs_mono.cuh. A component is eligible when every h table it uses is the
// exact Clifford form above (alpha, beta multiples of pi/2; table values equal
// to the exact ones within 1e-9), each table's non-zero entries share m and
// k mod 2, and its parameters fit the byte selectors.
MonoHost encode_mono(const zxs_model_desc *d, uint32_t max_chain, uint64_t heavy_min) {
    MonoHost H;
    H.comp_mono.assign(std::max<uint32_t>(1, d->num_components), 0);
    const uint32_t fwid = d->f_width;
    // table classes
    std::vector<int> tpa(d->num_h_tables, -1), tpb(d->num_h_tables, -1);
    for (uint32_t t = 0; t < d->num_h_tables; t++) {
        const double qa = d->h_alpha[t] / (M_PI / 2), qb = d->h_beta[t] / (M_PI / 2);
        if (std::fabs(qa - std::round(qa)) > 1e-9 || std::fabs(qb - std::round(qb)) > 1e-9) continue;
        const int pa = int(((long long)std::llround(qa) % 4 + 4) % 4), pb = int(((long long)std::llround(qb) % 4 + 4) % 4);
        bool ok = true;
        for (int ab = 0; ab < 4 && ok; ab++) {
            const MonoEntry e = mono_entry(pa, pb, ab >> 1, ab & 1);
            if (!e.zero && (e.m < 0 || e.k < 0)) ok = false;
            const double re = d->h_table[8 * t + 2 * ab], im = d->h_table[8 * t + 2 * ab + 1];
            if (std::fabs(re - e.re) > 1e-9 || std::fabs(im - e.im) > 1e-9) ok = false;
        }
        if (ok) {
            tpa[t] = pa;
            tpb[t] = pb;
        }
    }
    // One dictionary per chain tensor (staged in shared memory while that
    // tensor is evaluated). Lowering first collects the tensor's distinct
    // parity forms as 64-bit masks over its W raw parameters; once the
    // tensor's record stream is known, a basis of W parity forms is chosen
    // (greedy: the forms carrying the most selector loads, kept while linearly
    // independent, completed with unit vectors) and every form is rewritten in
    // that basis -- the device forms the W basis planes once per tensor and
    // tile -- and, when longer than W/2, as its complement plus the ALL plane
    // (XOR of the W basis planes).
    // Component-local parameter spaces (the 64-bit form masks and dedup keys
    // index parameters): a component whose raw width f_width + chain exceeds 63
    // reads its tensors through the f columns they actually use, in column order.
    std::vector<std::vector<uint32_t>> comp_local(d->num_components);  // local f param -> raw f column
    uint32_t lf_max = 0;
    for (uint32_t c = 0; c < d->num_components; c++) {
        const uint32_t n = d->comp_out_begin[c + 1] - d->comp_out_begin[c];
        std::vector<uint32_t> &loc = comp_local[c];
        if (fwid + n <= 63) {
            for (uint32_t p = 0; p < fwid; p++) loc.push_back(p);
        } else {
            std::vector<uint8_t> used(fwid, 0);
            const uint32_t t0 = d->comp_tensor_begin[c], t1 = d->comp_tensor_begin[c + 1];
            const uint64_t k0 = d->term_factor_begin[d->tensor_term_begin[t0]];
            const uint64_t k1 = d->term_factor_begin[d->tensor_term_begin[t1]];
            for (uint64_t x = d->factor_u_begin[k0]; x < d->factor_u_begin[k1]; x++) {
                if (d->factor_u_bits[x] < fwid) used[d->factor_u_bits[x]] = 1;
            }
            for (uint64_t x = d->factor_v_begin[k0]; x < d->factor_v_begin[k1]; x++) {
                if (d->factor_v_bits[x] < fwid) used[d->factor_v_bits[x]] = 1;
            }
            for (uint32_t p = 0; p < fwid; p++) {
                if (used[p]) loc.push_back(p);
            }
        }
        const uint64_t nfac = d->term_factor_begin[d->tensor_term_begin[d->comp_tensor_begin[c + 1]]] -
                              d->term_factor_begin[d->tensor_term_begin[d->comp_tensor_begin[c]]];
        if (nfac >= heavy_min && loc.size() + n <= 63) lf_max = std::max(lf_max, uint32_t(loc.size()));
    }
    std::unordered_map<uint64_t, uint32_t> form_id;  // local mask -> form id (per tensor)
    form_id.reserve(1 << 14);
    std::vector<uint64_t> form_mask;        // form id -> raw mask
    std::map<uint32_t, uint32_t> form_size; // dictionary entry index -> plane loads
    size_t dict_base = 0;
    // ALL plane (>= every mono tensor's local width); all_plane + 1: ZERO; + 2 + j: raw sampled bit j
    const uint32_t all_plane = lf_max + max_chain;
    // Block form tables (dedup_eval_kernel): 128 B of shared memory per form value; the capacity is
    // what the kernel's 227 KB leave after its parameter planes and the deepest (Z, J0, J1) stacks
    // (at least kDedupMaxBlockForms)
    // summation segments per tensor at most (the canonical order's granularity; ZXS_DEDUP_SEGS)
    uint32_t max_segs = zxs_dev::kDedupSegs;
    if (const char *e = std::getenv("ZXS_DEDUP_SEGS")) {
        max_segs = uint32_t(std::min<long>(zxs_dev::kDedupSegs, std::max(16L, std::atol(e))));
    }
    const uint32_t block_form_cap = std::max<uint32_t>(
        zxs_dev::kDedupMaxBlockForms,
        uint32_t((227u * 1024u - 1024u - (all_plane + 2) * 128u -
                  uint32_t(zxs_dev::kDedupWarps) * zxs_dev::kMonoMaxDepth * 384u) / 128u));
    uint32_t cur_width = 0;                        // param width of the tensor being encoded
    auto dict_form = [&](uint64_t m) -> uint32_t {
        auto it = form_id.find(m);
        if (it != form_id.end()) return it->second;
        const uint32_t id = uint32_t(form_mask.size());
        form_mask.push_back(m);
        form_id.emplace(m, id);
        return id;
    };
    auto weight = [](uint64_t x) { return uint32_t(__builtin_popcountll(x)); };
    // Chooses the tensor's basis, writes its dictionary, returns form id -> entry index.
    auto finish_dictionary = [&](const std::vector<uint64_t> &usage, std::vector<uint64_t> &basis) {
        const uint32_t W = cur_width;
        auto cost = [&](uint64_t x) { const uint32_t k = weight(x); return std::min(k, W - k + 1); };
        // echelon form of a candidate basis: rows (pivot bit, vector) and the basis
        // vectors each row combines; false if the vectors are dependent
        std::vector<std::pair<int, uint64_t>> rows;
        std::vector<uint64_t> comb;
        auto echelon = [&](const std::vector<uint64_t> &B) {
            rows.clear();
            comb.clear();
            for (size_t i = 0; i < B.size(); i++) {
                uint64_t v = B[i], c = 1ull << i;
                for (size_t r = 0; r < rows.size(); r++) {
                    if ((v >> rows[r].first) & 1) {
                        v ^= rows[r].second;
                        c ^= comb[r];
                    }
                }
                if (!v) return false;
                rows.push_back({63 - __builtin_clzll(v), v});
                comb.push_back(c);
            }
            return true;
        };
        auto coords = [&](uint64_t m) {  // after echelon(): basis coordinates of m
            uint64_t c = 0;
            for (size_t r = 0; r < rows.size(); r++) {
                if ((m >> rows[r].first) & 1) {
                    m ^= rows[r].second;
                    c ^= comb[r];
                }
            }
            return c;
        };
        auto total = [&](const std::vector<uint64_t> &B) -> uint64_t {  // selector loads of the stream
            if (!echelon(B)) return ~0ull;
            uint64_t sum = 0;
            for (size_t f = 0; f < form_mask.size(); f++) {
                if (usage[f]) sum += usage[f] * cost(coords(form_mask[f]));
            }
            return sum;
        };
        // start: the better of the identity and a greedy independent set of the
        // forms carrying the most loads; then first-improvement swaps against the
        // most loaded forms until no swap helps (bounded rounds)
        std::vector<uint32_t> order(form_mask.size());
        for (uint32_t i = 0; i < order.size(); i++) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
            return usage[a] * cost(form_mask[a]) > usage[b] * cost(form_mask[b]);
        });
        std::vector<uint64_t> ident, greedy;
        for (uint32_t p = 0; p < W; p++) ident.push_back(1ull << p);
        for (uint32_t i : order) {
            if (greedy.size() == W) break;
            greedy.push_back(form_mask[i]);
            if (!form_mask[i] || !echelon(greedy)) greedy.pop_back();
        }
        for (uint32_t p = 0; p < W && greedy.size() < W; p++) {
            greedy.push_back(1ull << p);
            if (!echelon(greedy)) greedy.pop_back();
        }
        basis = ident;
        uint64_t best = total(ident);
        const uint64_t tg = total(greedy);
        if (tg < best) {
            best = tg;
            basis = greedy;
        }
        std::vector<uint64_t> cand;
        for (uint32_t i : order) {
            if (cand.size() >= 160) break;
            if (form_mask[i]) cand.push_back(form_mask[i]);
        }
        for (int round = 0; round < 12; round++) {
            bool improved = false;
            for (uint32_t slot = 0; slot < W; slot++) {
                for (uint64_t cv : cand) {
                    if (std::find(basis.begin(), basis.end(), cv) != basis.end()) continue;
                    std::vector<uint64_t> nb = basis;
                    nb[slot] = cv;
                    const uint64_t tc = total(nb);
                    if (tc < best) {
                        best = tc;
                        basis = nb;
                        improved = true;
                    }
                }
            }
            if (!improved) break;
        }
        echelon(basis);
        std::vector<uint32_t> entry_of(form_mask.size());
        for (uint32_t f = 0; f < form_mask.size(); f++) {
            const uint64_t x = coords(form_mask[f]);
            std::vector<uint32_t> sel;
            if (W >= 2 && weight(x) > (W + 1) / 2) {
                for (uint32_t b = 0; b < W; b++) {
                    if (!((x >> b) & 1)) sel.push_back(b);
                }
                sel.push_back(all_plane);
            } else {
                for (uint32_t b = 0; b < W; b++) {
                    if ((x >> b) & 1) sel.push_back(b);
                }
            }
            const uint32_t id = uint32_t(H.dict.size() - dict_base);
            entry_of[f] = id;
            uint32_t slots = 0;
            for (size_t i = 0; i < sel.size() || i == 0; i += 15) {
                const size_t n = std::min<size_t>(15, sel.size() - i);
                uint8_t e[16];
                std::memset(e, int(all_plane + 1), 16);  // unused slots read the all-zero plane
                const uint8_t cls = n >= 15 ? 7 : uint8_t((std::max<size_t>(n, 1) - 1) / 2);  // 2c + 2 slots
                e[0] = uint8_t(cls | (i + 15 < sel.size() ? 0x80 : 0));
                for (size_t k = 0; k < n; k++) e[1 + k] = uint8_t(sel[i + k]);
                uint4 wv;
                std::memcpy(&wv, e, 16);
                H.dict.push_back(wv);
                slots += n >= 15 ? 15 : uint32_t(2 * ((std::max<size_t>(n, 1) - 1) / 2) + 2);
            }
            form_size[id] = slots;
        }
        return entry_of;
    };

    // Per (h table, u form present, v form present): the factor's exact entries on its domain,
    // the common m and k mod 2 of its non-zero entries, the cheapest J polynomial
    // d00 + al a + be b + ga ab (mod 4) matching (k - o)/2 there, and its zero pattern.
    struct FactorRule {
        int status = -1;  // -1 unset, 0 record, 1 identically zero, 2 m / k mod 2 differ, 3 no J polynomial
        int mset = 0, oset = 0, best = 0;
        uint32_t zl = 0, dm = 0;
    };
    std::vector<FactorRule> rules(size_t(std::max<uint32_t>(1, d->num_h_tables)) * 4);
    auto factor_rule = [&](uint32_t tb, bool ua, bool vb) -> const FactorRule & {
        FactorRule &r = rules[size_t(tb) * 4 + (ua ? 2 : 0) + (vb ? 1 : 0)];
        if (r.status >= 0) return r;
        MonoEntry en[4];
        int mset = -1, oset = -1, nnz = 0;
        bool indomain[4], zero[4];
        r.status = 0;
        for (int ab = 0; ab < 4; ab++) {
            const int a = ab >> 1, b = ab & 1;
            en[ab] = mono_entry(tpa[tb], tpb[tb], a, b);
            indomain[ab] = (a == 0 || ua) && (b == 0 || vb);
            zero[ab] = en[ab].zero;
            if (!indomain[ab] || zero[ab]) continue;
            nnz++;
            if (mset < 0) mset = en[ab].m;
            if (oset < 0) oset = en[ab].k & 1;
            if (mset != en[ab].m || oset != (en[ab].k & 1)) r.status = 2;
        }
        if (r.status) return r;
        if (nnz == 0) {
            r.status = 1;
            return r;
        }
        int best = -1, bc = 1 << 30;
        for (int code = 0; code < 256; code++) {
            const int d00 = code & 3, al = (code >> 2) & 3, be = (code >> 4) & 3, ga = (code >> 6) & 3;
            if ((!ua && (al || ga)) || (!vb && (be || ga))) continue;
            bool fits = true;
            for (int ab = 0; ab < 4 && fits; ab++) {
                if (!indomain[ab] || zero[ab]) continue;
                const int a = ab >> 1, b = ab & 1;
                fits = ((d00 + al * a + be * b + ga * a * b) & 3) == (((en[ab].k - oset) / 2) & 3);
            }
            if (!fits) continue;
            const int cost = (al != 0) + 4 * (be != 0) + 8 * (ga != 0);
            if (cost < bc) {
                bc = cost;
                best = code;
            }
        }
        if (best < 0) {
            r.status = 3;
            return r;
        }
        r.mset = mset;
        r.oset = oset;
        r.best = best;
        for (int ab = 0; ab < 4; ab++) {
            if (indomain[ab] && zero[ab]) r.zl |= 1u << ab;  // zero on the domain (outside: don't-care)
            r.dm |= indomain[ab] ? 1u << ab : 0u;
        }
        return r;
    };

    uint32_t upos = 0;
    for (uint32_t c = 0; c < d->num_components; c++) {
        const uint32_t n = d->comp_out_begin[c + 1] - d->comp_out_begin[c];
        const uint32_t t0 = d->comp_tensor_begin[c], t1 = d->comp_tensor_begin[c + 1];
        const uint64_t nf = d->term_factor_begin[d->tensor_term_begin[t1]] - d->term_factor_begin[d->tensor_term_begin[t0]];
        const std::vector<uint32_t> &loc = comp_local[c];
        const uint32_t nloc = uint32_t(loc.size());
        bool ok = nf >= heavy_min && H.comps.size() < size_t(zxs_dev::kMaxMonoComps) && nloc + n <= 63 &&
                  all_plane + 2 <= 255;
        const char *why = ok ? nullptr : (nf < heavy_min ? "small" : "parameters / planes / component count");
        std::vector<uint32_t> to_local(fwid + n, ~0u);  // raw param -> local param
        for (uint32_t i = 0; i < nloc; i++) to_local[loc[i]] = i;
        for (uint32_t j = 0; j < n; j++) to_local[fwid + j] = nloc + j;
        const size_t dict_mark = H.dict.size();
        std::vector<uint32_t> tdb;  // per tensor: first dictionary entry
        std::vector<uint32_t> twid;  // per tensor: param width (the ALL plane spans planes 0..W-1)
        std::vector<uint32_t> tbb;   // per tensor: first basis vector
        std::vector<uint64_t> cb;    // basis vectors (raw masks)
        uint32_t comp_max_dict = 1, comp_depth = 1;
        std::vector<uint32_t> w;
        std::vector<uint4> ch;
        std::vector<uint32_t> tcb;
        std::vector<uint32_t> sw;   // segment streams of this component
        std::vector<uint4> sg;      // segments (word_begin relative to sw)
        std::vector<uint32_t> tsb;  // per tensor: first segment (relative to sg)
        std::vector<uint64_t> tl;   // per tensor: plane loads per 32-shot word
        std::vector<unsigned long long> trm;  // per tensor: local parameters read
        std::vector<uint32_t> tnb;            // per tensor: null pairs (end, relative to tn)
        std::vector<unsigned long long> tn;   // null pairs of this component's tensors
        std::vector<uint32_t> tspw;           // per tensor: segments per warp in a dedup_eval_kernel item
        std::vector<uint32_t> bf, bfb, tfb;  // block forms, block ends (relative), per tensor first block
        uint32_t max_bf = 0;
        uint64_t recs = 0, dead = 0, nsel = 0, loads = 0, nodes_total = 0, negligible = 0;
        for (uint32_t t = t0; ok && t < t1; t++) {
            form_id.clear();
            form_mask.clear();
            form_size.clear();
            dict_base = H.dict.size();
            tdb.push_back(uint32_t(dict_base));
            cur_width = nloc + n;  // the local width (reference width f_width + n, compile.cpp:256)
            twid.push_back(cur_width);
            if (d->tensor_param_width[t] > fwid + n || cur_width > 63) { ok = false; if (!why) why = "width"; }  // local forms as 64-bit masks
            // ---- lower every term of tensor t to record tokens (order-free: J and Z commute)
            std::vector<MonoTerm> terms;
            terms.reserve(size_t(d->tensor_term_begin[t + 1] - d->tensor_term_begin[t]));
            for (uint64_t term = d->tensor_term_begin[t]; ok && term < d->tensor_term_begin[t + 1]; term++) {
                std::vector<uint64_t> tw;
                int M = 0, K = 0;
                bool term_dead = false;
                for (uint64_t k = d->term_factor_begin[term]; k < d->term_factor_begin[term + 1]; k++) {
                    const uint32_t tb = d->factor_table[k];
                    if (tb >= d->num_h_tables || tpa[tb] < 0) {
                        { ok = false; if (!why) why = "table class"; }
                        break;
                    }
                    // the factor's parity forms as masks over local parameters (XOR: repeated
                    // selectors cancel, phase_terms.cpp:108-121)
                    uint64_t us = 0, vs = 0;
                    for (uint64_t x = d->factor_u_begin[k]; ok && x < d->factor_u_begin[k + 1]; x++) {
                        const uint32_t p = d->factor_u_bits[x];
                        ok = p < fwid + n && to_local[p] != ~0u;
                        if (ok) us ^= 1ull << to_local[p];
                    }
                    for (uint64_t x = d->factor_v_begin[k]; ok && x < d->factor_v_begin[k + 1]; x++) {
                        const uint32_t p = d->factor_v_bits[x];
                        ok = p < fwid + n && to_local[p] != ~0u;
                        if (ok) vs ^= 1ull << to_local[p];
                    }
                    if (!ok) {
                        if (!why) why = "selector range";
                        break;
                    }
                    const bool ua = us != 0, vb = vs != 0;
                    // the factor's record depends on the (table, ua, vb) triple only: memoised rule
                    const FactorRule &fr = factor_rule(tb, ua, vb);
                    if (fr.status == 2) { ok = false; if (!why) why = "table m/k mismatch"; }
                    if (fr.status == 3) { ok = false; if (!why) why = "J polynomial"; }
                    if (!ok) break;
                    if (fr.status == 1) {
                        term_dead = true;  // identically zero factor: the term is exactly 0
                        continue;
                    }
                    M += fr.mset;
                    K += fr.oset;
                    const int best = fr.best;
                    const int d00 = best & 3, al = (best >> 2) & 3, be = (best >> 4) & 3, ga = (best >> 6) & 3;
                    K += 2 * d00;
                    const uint32_t zl = fr.zl, dm = fr.dm;
                    const uint32_t fa = ua ? dict_form(us) : zxs_dev::kFormMask, fbv = vb ? dict_form(vs) : zxs_dev::kFormMask;
                    nsel += uint64_t(__builtin_popcountll(us) + __builtin_popcountll(vs));
                    // token: record word | (GEN aux word + 1) << 32
                    auto rec = [&](uint32_t kind, uint32_t a_form, uint32_t b_form, uint64_t aux = 0) {
                        tw.push_back(uint64_t(kind << 28 | (b_form & zxs_dev::kFormMask) << zxs_dev::kFormShiftB | (a_form & zxs_dev::kFormMask)) | aux << 32);
                    };
                    const bool jnone = !al && !be && !ga;
                    // Z patterns over the domain points present (bit index a*2+b)
                    const uint32_t zA = ua ? 0xCu : 0u;          // a == 1
                    const uint32_t zAn = 0x3u;                   // a == 0
                    const uint32_t zB = vb ? 0xAu : 0u;          // b == 1
                    const uint32_t zBn = 0x5u;                   // b == 0
                    auto zis = [&](uint32_t pat) { return (pat & dm) == zl; };
                    if (zl == 0) {
                        if (jnone) continue;  // constant factor
                        if (!be && !ga) {
                            rec(al == 1 ? zxs_dev::kRecAdd : al == 3 ? zxs_dev::kRecSub : zxs_dev::kRecAdd2, fa, zxs_dev::kFormMask);
                        } else if (!al && !ga) {
                            rec(be == 1 ? zxs_dev::kRecAdd : be == 3 ? zxs_dev::kRecSub : zxs_dev::kRecAdd2,
                                dict_form(vs), zxs_dev::kFormMask);
                        } else {
                            rec(zxs_dev::kRecGen, fa, fbv, uint64_t(al | be << 2 | ga << 4) + 1);
                        }
                    } else if (jnone && ua && zis(zA)) {
                        rec(zxs_dev::kRecZ, fa, zxs_dev::kFormMask);
                    } else if (jnone && ua && zis(zAn)) {
                        rec(zxs_dev::kRecZn, fa, zxs_dev::kFormMask);
                    } else if (jnone && vb && zis(zB)) {
                        rec(zxs_dev::kRecZ, dict_form(vs), zxs_dev::kFormMask);
                    } else if (jnone && vb && zis(zBn)) {
                        rec(zxs_dev::kRecZn, dict_form(vs), zxs_dev::kFormMask);
                    } else {
                        rec(zxs_dev::kRecGen, fa, fbv, (uint64_t(al | be << 2 | ga << 4) | uint64_t(zl) << 6) + 1);
                    }
                }
                if (!ok) break;
                if (term_dead) {
                    dead++;
                    continue;
                }
                // c' = c * 2^(M/2) * w^K
                static const long double s2 = 0.70710678118654752440084436210484903928L;
                static const long double wr[8] = {1, s2, 0, -s2, -1, -s2, 0, s2}, wi[8] = {0, s2, 1, s2, 0, -s2, -1, -s2};
                const int k8 = K & 7;
                long double mag = std::ldexp(1.0L, M / 2);
                if (M & 1) mag *= 1.41421356237309504880168872420969807857L;
                const long double cr = d->term_c[2 * term], ci = d->term_c[2 * term + 1];
                MonoTerm mt;
                mt.re = double((cr * wr[k8] - ci * wi[k8]) * mag);
                mt.im = double((cr * wi[k8] + ci * wr[k8]) * mag);
                std::sort(tw.begin(), tw.end());
                mt.recs = std::move(tw);
                terms.push_back(std::move(mt));
            }
            if (!ok) break;
            // ---- numerically zero terms: a coefficient below 2^-40 of the tensor's largest is the
            // rounding residue of an exact cancellation in the reference's decomposition weights
            // (e.g. 1 + e^{i pi} = 1.2e-16 i; cultivation: a third of the terms, 40+ binades below
            // the rest). They are dropped; the value moves by < 1e-16 relative, the order of the
            // reference's own rounding (the h entries are already exact here)
            {
                double mx = 0.0;
                for (const MonoTerm &mt : terms) mx = std::max(mx, std::hypot(mt.re, mt.im));
                const double floor_c = std::ldexp(mx, -40);
                size_t keep = 0;
                for (size_t i = 0; i < terms.size(); i++) {
                    if (std::hypot(terms[i].re, terms[i].im) >= floor_c) {
                        if (keep != i) terms[keep] = std::move(terms[i]);
                        keep++;
                    }
                }
                negligible += terms.size() - keep;
                terms.resize(keep);
            }
            // ---- shared-prefix tree over the terms in order, emitted in DFS preorder
            const auto tm0 = std::chrono::steady_clock::now();
            std::vector<MonoNode> nodes = mono_tree(terms);
            const auto tm1 = std::chrono::steady_clock::now();
            for (const MonoNode &nd : nodes) comp_depth = std::max(comp_depth, nd.depth + 1);
            // basis and dictionary, weighted by the records actually emitted
            std::vector<uint64_t> usage(form_mask.size(), 0);
            for (const MonoNode &nd : nodes) {
                for (uint64_t tok : nd.recs) {
                    const uint32_t r = uint32_t(tok), fa = r & zxs_dev::kFormMask, fbv = (r >> zxs_dev::kFormShiftB) & zxs_dev::kFormMask;
                    if (fa != zxs_dev::kFormMask && fa < usage.size()) usage[fa]++;
                    if ((r >> 28) == zxs_dev::kRecGen && fbv != zxs_dev::kFormMask && fbv < usage.size()) usage[fbv]++;
                }
            }
            if (form_mask.size() >= zxs_dev::kFormMask) { ok = false; if (!why) why = "forms > 16382"; }
            if (!ok) break;
            std::vector<uint64_t> basis;
            const std::vector<uint32_t> entry_of = finish_dictionary(usage, basis);
            const auto tm2 = std::chrono::steady_clock::now();
            tbb.push_back(uint32_t(H.basis.size() + cb.size()));
            cb.insert(cb.end(), basis.begin(), basis.end());
            auto remap = [&](uint32_t r) {
                const uint32_t fa = r & zxs_dev::kFormMask, fbv = (r >> zxs_dev::kFormShiftB) & zxs_dev::kFormMask;
                const uint32_t na = fa == zxs_dev::kFormMask ? zxs_dev::kFormMask : entry_of[fa];
                const uint32_t nb = fbv == zxs_dev::kFormMask ? zxs_dev::kFormMask : entry_of[fbv];
                return (r & 0xf0000000u) | (nb << zxs_dev::kFormShiftB) | na;
            };
            uint32_t cur_begin = uint32_t(H.words.size() + w.size()), cur_nodes = 0;
            auto close_chunk = [&]() {
                if (H.words.size() + w.size() == cur_begin) w.insert(w.end(), 4, 0u);  // no 0-byte bulk copies
                while ((H.words.size() + w.size()) % 4) w.push_back(0);
                const uint32_t end = uint32_t(H.words.size() + w.size());
                ch.push_back(make_uint4(cur_begin, end - cur_begin, cur_nodes, 0));
                cur_begin = end;
                cur_nodes = 0;
            };
            tcb.push_back(uint32_t(H.chunks.size() + ch.size()));
            if (H.dict.size() - dict_base >= zxs_dev::kFormMask) { ok = false; if (!why) why = "dictionary > 16382"; }  // 14-bit form ids
            comp_max_dict = std::max<uint32_t>(comp_max_dict, uint32_t(H.dict.size() - dict_base));
            // summation segments: contiguous node ranges of about equal cost, the tensor value
            // being the ordered sum of the segment sums. Cost in issued instructions per 32-key
            // word of the walk (mono_walk_fv SASS): a node's header and stack ~30, a one-form
            // record ~4, a two-form record ~25, a leaf's epilogue ~140 (32 keys); the warps of a
            // dedup_eval_kernel item wait for the slowest at the next barrier
            std::vector<uint8_t> seg_start(nodes.size(), 0);
            {
                const uint32_t G = std::max<uint32_t>(
                    1, std::min<uint32_t>(max_segs, uint32_t(nodes.size() / 8)));
                auto cost = [](const MonoNode &nd) {
                    uint64_t c = 30 + (nd.leaf ? 140 : 0);
                    for (uint64_t tok : nd.recs) c += (uint32_t(tok) >> 28) == zxs_dev::kRecGen ? 25 : 4;
                    return c;
                };
                uint64_t total = 0;
                for (const MonoNode &nd : nodes) total += cost(nd);
                uint64_t cum = 0, k = 1;
                for (size_t i = 0; i < nodes.size(); i++) {
                    if (i == 0) seg_start[i] = 1;
                    else if (k < G && cum * G >= total * k) {
                        seg_start[i] = 1;
                        while (k < G && cum * G >= total * k) k++;
                    }
                    cum += cost(nodes[i]);
                }
            }
            const uint64_t loads_before = loads;
            std::vector<uint32_t> node_off(nodes.size()), node_len(nodes.size());
            std::vector<uint32_t> nw;
            size_t node_i = 0;
            for (const MonoNode &nd : nodes) {
                if (!ok) break;
                // node: {leaf << 31 | depth << 24 | n_gen, n_add | n_sub << 8 | n_add2 << 16 | n_z << 24, n_zn}
                // [+ re, im for leaves], then the one-form records grouped by kind, then GEN pairs
                uint32_t cnt[16] = {};
                for (uint64_t tok : nd.recs) cnt[uint32_t(tok) >> 28]++;
                for (int k = 0; k < 16; k++) ok &= cnt[k] < 256; if (!ok && !why) why = "records per node kind >= 256";
                if (!ok) break;
                nw.clear();
                nw.push_back((nd.leaf ? 0x80000000u : 0u) | (seg_start[node_i] ? zxs_dev::kMonoSegStart : 0u) |
                             uint32_t(nd.depth) << 24 | cnt[zxs_dev::kRecGen]);
                nw.push_back(cnt[zxs_dev::kRecAdd] | cnt[zxs_dev::kRecSub] << 8 | cnt[zxs_dev::kRecAdd2] << 16 |
                             cnt[zxs_dev::kRecZ] << 24);
                nw.push_back(cnt[zxs_dev::kRecZn]);
                if (nd.leaf) {
                    uint64_t rb, ib;
                    std::memcpy(&rb, &nd.re, 8);
                    std::memcpy(&ib, &nd.im, 8);
                    nw.insert(nw.end(), {uint32_t(rb), uint32_t(rb >> 32), uint32_t(ib), uint32_t(ib >> 32)});
                }
                // records of a kind ordered by their form's first dictionary entry size class, so
                // consecutive pairs mostly share a class (mono_kernel's paired straight-line loads)
                std::vector<uint64_t> recs_sorted(nd.recs.begin(), nd.recs.end());
                auto cls_of = [&](uint64_t tok) {
                    const uint32_t r = remap(uint32_t(tok)), fa = r & zxs_dev::kFormMask;
                    return fa == zxs_dev::kFormMask ? 0u : uint32_t(H.dict[dict_base + fa].x & 0x87u);
                };
                std::stable_sort(recs_sorted.begin(), recs_sorted.end(),
                                 [&](uint64_t x, uint64_t y) { return cls_of(x) > cls_of(y); });
                // one-form records of every kind (sorted by class: mono_kernel pairs them), then GEN
                for (int gen_pass = 0; gen_pass < 2; gen_pass++) {
                    for (uint64_t tok : recs_sorted) {
                        const uint32_t r = remap(uint32_t(tok));
                        const uint32_t kind = r >> 28;
                        if ((kind == zxs_dev::kRecGen) != (gen_pass == 1)) continue;
                        nw.push_back(r);
                        if (tok >> 32) nw.push_back(uint32_t((tok >> 32) - 1));
                        recs++;
                        const uint32_t fa = r & zxs_dev::kFormMask, fbv = (r >> zxs_dev::kFormShiftB) & zxs_dev::kFormMask;
                        if (fa != zxs_dev::kFormMask) loads += form_size[fa];
                        if (kind == zxs_dev::kRecGen && fbv != zxs_dev::kFormMask) loads += form_size[fbv];
                    }
                }
                if (nw.size() + 4 > zxs_dev::kMonoChunkWords || nd.depth >= zxs_dev::kMonoMaxDepth) {
                    { ok = false; if (!why) why = "node too large or tree too deep"; }
                    break;
                }
                if (H.words.size() + w.size() + nw.size() - cur_begin > zxs_dev::kMonoChunkWords) close_chunk();
                node_off[node_i] = uint32_t(w.size());
                node_len[node_i] = uint32_t(nw.size());
                node_i++;
                w.insert(w.end(), nw.begin(), nw.end());
                cur_nodes++;
            }
            if (ok) close_chunk();
            tl.push_back(loads - loads_before);
            {
                unsigned long long rm = 0;  // local parameters any of the tensor's forms reads
                for (uint64_t fm : form_mask) rm |= fm;
                trm.push_back(rm);
                // reduced row echelon form of the forms (pivot = highest bit), then one null
                // vector per free parameter q of rm: e_q + the pivots of the rows holding q
                std::vector<uint64_t> rows;
                std::vector<int> piv;
                for (uint64_t fm : form_mask) {
                    uint64_t v = fm;
                    for (size_t r = 0; r < rows.size(); r++) {
                        if ((v >> piv[r]) & 1) v ^= rows[r];
                    }
                    if (!v) continue;
                    const int pb = 63 - __builtin_clzll(v);
                    for (uint64_t &row : rows) {
                        if ((row >> pb) & 1) row ^= v;
                    }
                    rows.push_back(v);
                    piv.push_back(pb);
                }
                uint64_t pivm = 0;
                for (int pb : piv) pivm |= 1ull << pb;
                for (uint64_t fr = rm & ~pivm; fr; fr &= fr - 1) {
                    const int q = __builtin_ctzll(fr);
                    uint64_t nv = 1ull << q;
                    for (size_t r = 0; r < rows.size(); r++) {
                        if ((rows[r] >> q) & 1) nv |= 1ull << piv[r];
                    }
                    tn.push_back(1ull << q);
                    tn.push_back(nv);
                }
                tnb.push_back(uint32_t(tn.size()));
            }
            // segment streams: each starts with its first node's ancestors (internal nodes,
            // replayed to rebuild the stack), then the segment's own nodes; flags cleared
            tsb.push_back(uint32_t(sg.size()));
            if (ok) {
                std::vector<size_t> anc(zxs_dev::kMonoMaxDepth, 0);
                for (size_t i = 0; i < nodes.size();) {
                    size_t j = i + 1;
                    while (j < nodes.size() && !seg_start[j]) j++;
                    const uint32_t b = uint32_t(sw.size());
                    uint32_t nn = 0;
                    auto copy_node = [&](size_t x) {
                        const size_t o = sw.size();
                        sw.insert(sw.end(), w.begin() + node_off[x], w.begin() + node_off[x] + node_len[x]);
                        sw[o] &= ~zxs_dev::kMonoSegStart;
                        nn++;
                    };
                    for (uint32_t dd = 0; dd < nodes[i].depth; dd++) copy_node(anc[dd]);
                    for (size_t x = i; x < j; x++) {
                        copy_node(x);
                        anc[nodes[x].depth] = x;
                    }
                    sg.push_back(make_uint4(b, uint32_t(sw.size()) - b, nn, 0));
                    i = j;
                }
                // block form tables: the dictionary entries each block of kDedupWarps x spw segments
                // uses (one dedup_eval_kernel item: every warp walks spw consecutive segments); its
                // records are rewritten to block-local ids (kept global when a block needs more
                // than the table holds: tensor_first_block = ~0). spw is the largest of 8, 4, 2, 1
                // whose blocks all fit and leave at least 32 blocks (work items per key group):
                // the per-item costs (parameter planes, form values, barriers) amortise over
                // longer walks
                const uint32_t s0 = tsb.back(), s1 = uint32_t(sg.size());
                uint32_t bsegs = zxs_dev::kDedupWarps;
                auto for_forms = [&](uint32_t b0, const std::function<uint32_t(uint32_t)> &fn) {
                    for (uint32_t g = b0; g < std::min(s1, b0 + bsegs); g++) {
                        uint32_t q = sg[g].x;
                        for (uint32_t nn2 = 0; nn2 < sg[g].z; nn2++) {
                            const uint32_t h0 = sw[q], h1 = sw[q + 1], h2 = sw[q + 2];
                            q += 3 + ((h0 >> 31) ? 4 : 0);
                            const uint32_t ns = (h1 & 0xffu) + ((h1 >> 8) & 0xffu) + ((h1 >> 16) & 0xffu) + (h1 >> 24) +
                                                (h2 & 0xffu);
                            for (uint32_t r = 0; r < ns; r++, q++) sw[q] = (sw[q] & ~zxs_dev::kFormMask) | fn(sw[q] & zxs_dev::kFormMask);
                            for (uint32_t gg = 0; gg < (h0 & 0xffu); gg++, q += 2) {
                                const uint32_t r = sw[q];
                                sw[q] = (r & 0xf0000000u) | (fn((r >> zxs_dev::kFormShiftB) & zxs_dev::kFormMask) << zxs_dev::kFormShiftB) | fn(r & zxs_dev::kFormMask);
                            }
                        }
                    }
                };
                std::vector<std::vector<uint32_t>> lists;
                bool fits = false;
                uint32_t spw = 8;
                for (;; spw /= 2) {
                    bsegs = zxs_dev::kDedupWarps * spw;
                    lists.clear();
                    fits = true;
                    for (uint32_t b0 = s0; b0 < s1; b0 += bsegs) {
                        std::unordered_map<uint32_t, uint32_t> local;
                        std::vector<uint32_t> list;
                        for_forms(b0, [&](uint32_t f) {  // identity pass: collect
                            if (f != zxs_dev::kMonoNoForm && local.emplace(f, uint32_t(list.size())).second) list.push_back(f);
                            return f;
                        });
                        fits = fits && list.size() <= block_form_cap;
                        lists.push_back(std::move(list));
                    }
                    if (spw == 1 || (fits && lists.size() >= 32)) break;
                }
                if (std::getenv("ZXS_DEBUG_MONO")) {
                    size_t mx = 0, over = 0;
                    for (const auto &l : lists) {
                        mx = std::max(mx, l.size());
                        over += l.size() > block_form_cap;
                    }
                    std::fprintf(stderr, "encode_mono: tensor %u: %u segments per warp, %zu blocks, max %zu forms per block, %zu over %u\n",
                                 t, spw, lists.size(), mx, over, block_form_cap);
                }
                tspw.push_back(spw);
                // the canonical summation groups are runs of spw consecutive segments (one warp's
                // walk in dedup_eval_kernel, accumulated without a reset): only a group's first
                // segment folds in the per-shot stream
                if (spw > 1) {
                    uint32_t si = 0;
                    for (size_t x = 0; x < nodes.size(); x++) {
                        if (!seg_start[x]) continue;
                        if (si++ % spw != 0) w[node_off[x]] &= ~zxs_dev::kMonoSegStart;
                    }
                }
                if (!fits) {
                    tfb.push_back(0xffffffffu);
                } else {
                    tfb.push_back(uint32_t(bfb.size()));
                    size_t k = 0;
                    for (uint32_t b0 = s0; b0 < s1; b0 += bsegs, k++) {
                        std::unordered_map<uint32_t, uint32_t> local;
                        for (uint32_t i = 0; i < lists[k].size(); i++) local.emplace(lists[k][i], i);
                        for_forms(b0, [&](uint32_t f) { return f == zxs_dev::kMonoNoForm ? f : local.at(f); });
                        // one-form records grouped by kind (ADD, SUB, ADD2, Z, ZN: the header's counts),
                        // so mono_walk_fv runs one fixed operation per loop
                        for (uint32_t g = b0; g < std::min(s1, b0 + bsegs); g++) {
                            uint32_t q = sg[g].x;
                            for (uint32_t nn2 = 0; nn2 < sg[g].z; nn2++) {
                                const uint32_t h0 = sw[q], h1 = sw[q + 1], h2 = sw[q + 2];
                                q += 3 + ((h0 >> 31) ? 4 : 0);
                                const uint32_t ns = (h1 & 0xffu) + ((h1 >> 8) & 0xffu) + ((h1 >> 16) & 0xffu) +
                                                    (h1 >> 24) + (h2 & 0xffu);
                                std::stable_sort(sw.begin() + q, sw.begin() + q + ns,
                                                 [](uint32_t x, uint32_t y) { return (x >> 28) < (y >> 28); });
                                // the kind is implied by the position; the word becomes the form value's
                                // byte offset in the block table (fv[form][lane]: 128 B per form)
                                for (uint32_t r = q; r < q + ns; r++) {
                                    const uint32_t f = sw[r] & zxs_dev::kFormMask;
                                    if (f == zxs_dev::kMonoNoForm) { ok = false; if (!why) why = "one-form record without a form"; }
                                    sw[r] = f * zxs_dev::kFvFormBytes;
                                }
                                q += ns + 2 * (h0 & 0xffu);
                            }
                        }
                        max_bf = std::max(max_bf, uint32_t(lists[k].size()));
                        bf.insert(bf.end(), lists[k].begin(), lists[k].end());
                        bfb.push_back(uint32_t(bf.size()));
                    }
                }
            } else {
                tspw.push_back(1);
            }
            nodes_total += nodes.size();
            if (std::getenv("ZXS_DEBUG_MONO")) {
                const auto tm3 = std::chrono::steady_clock::now();
                auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
                std::fprintf(stderr, "encode_mono: tensor %u: %zu terms %zu forms, tree %.2fs dictionary %.2fs streams %.2fs\n",
                             t, terms.size(), form_mask.size(), sec(tm0, tm1), sec(tm1, tm2), sec(tm2, tm3));
            }
        }
        // the narrow mono_kernel must fit (the per-shot path is every large component's fallback
        // and its verification seam); the deduplicated path sizes its own shared memory
        if (ok && mono_smem_bytes(all_plane + max_chain + 2, std::max(comp_max_dict, H.max_dict), 3,
                                  std::max(comp_depth, H.max_depth)) > 227 * 1024) {
            { ok = false; if (!why) why = "shared memory"; }
        }
        if (std::getenv("ZXS_DEBUG_MONO") && nf >= heavy_min) {
            std::fprintf(stderr, "encode_mono: component %u (%llu factors): %s\n", c, (unsigned long long)nf,
                         ok ? "monomial path" : (why ? why : "?"));
        }
        if (ok) {
            zxs_dev::HeavyComp hc;
            hc.ci = c;
            hc.n_out = n;
            hc.upos_base = upos;
            hc.out_begin = d->comp_out_begin[c];
            hc.first_tensor = uint32_t(H.tensor_chunk_begin.size() - 1);
            hc.nf = nloc;
            hc.pmap_begin = uint32_t(H.param_map.size());
            for (uint32_t p : loc) H.param_map.push_back(uint16_t(p));
            for (uint32_t j = 0; j < n; j++) H.param_map.push_back(uint16_t(fwid + j));
            for (uint32_t t = t0; t < t1; t++) H.tensor_index[t] = hc.first_tensor + (t - t0);
            H.words.insert(H.words.end(), w.begin(), w.end());
            H.chunks.insert(H.chunks.end(), ch.begin(), ch.end());
            {
                const uint32_t wb = uint32_t(H.seg_words.size()), sb = uint32_t(H.segs.size());
                H.seg_words.insert(H.seg_words.end(), sw.begin(), sw.end());
                for (uint4 x : sg) H.segs.push_back(make_uint4(x.x + wb, x.y, x.z, 0));
                for (size_t i = 1; i < tsb.size(); i++) H.tensor_seg_begin.push_back(tsb[i] + sb);
                H.tensor_seg_begin.push_back(uint32_t(H.segs.size()));
                unsigned long long km = 0;
                for (uint64_t v : cb) km |= v;
                H.comp_key_mask.push_back(km);
                H.tensor_loads.insert(H.tensor_loads.end(), tl.begin(), tl.end());
                H.tensor_read_mask.insert(H.tensor_read_mask.end(), trm.begin(), trm.end());
                const uint32_t nb0 = uint32_t(H.tensor_null.size());
                H.tensor_null.insert(H.tensor_null.end(), tn.begin(), tn.end());
                for (uint32_t x : tnb) H.tensor_null_begin.push_back(x + nb0);
                H.tensor_spw.insert(H.tensor_spw.end(), tspw.begin(), tspw.end());
                const uint32_t fb0 = uint32_t(H.block_forms.size()), blk0 = uint32_t(H.block_form_begin.size() - 1);
                H.block_forms.insert(H.block_forms.end(), bf.begin(), bf.end());
                for (uint32_t x : bfb) H.block_form_begin.push_back(x + fb0);
                for (uint32_t x : tfb) H.tensor_first_block.push_back(x == 0xffffffffu ? x : x + blk0);
                H.max_block_forms = std::max(H.max_block_forms, max_bf);
            }
            for (size_t i = 1; i < tcb.size(); i++) H.tensor_chunk_begin.push_back(tcb[i]);
            H.tensor_chunk_begin.push_back(uint32_t(H.chunks.size()));
            H.tensor_dict_begin.insert(H.tensor_dict_begin.end(), tdb.begin(), tdb.end());
            H.tensor_width.insert(H.tensor_width.end(), twid.begin(), twid.end());
            const uint32_t bb0 = uint32_t(H.basis.size());
            for (uint32_t x : tbb) H.tensor_basis_begin.push_back(x);
            (void)bb0;
            H.basis.insert(H.basis.end(), cb.begin(), cb.end());
            H.comps.push_back(hc);
            H.comp_mono[c] = 1;
            H.max_dict = std::max(H.max_dict, comp_max_dict);
            H.max_depth = std::max(H.max_depth, comp_depth);
            H.max_chain = std::max(H.max_chain, n);
            H.records += recs;
            H.dead_terms += dead;
            H.negligible_terms += negligible;
            H.selectors += nsel;
            H.loads += loads;
            H.nodes += nodes_total;
        } else {
            H.dict.resize(dict_mark);
        }
        upos += n;
    }
    if (H.words.empty()) H.words.assign(4, 0);
    if (H.chunks.empty()) H.chunks.push_back(make_uint4(0, 0, 0, 0));
    if (H.dict.empty()) H.dict.push_back(make_uint4(0, 0, 0, 0));
    H.tensor_dict_begin.push_back(uint32_t(H.dict.size()));
    if (H.tensor_width.empty()) H.tensor_width.push_back(0);
    if (H.tensor_basis_begin.empty()) H.tensor_basis_begin.push_back(0);
    if (H.basis.empty()) H.basis.push_back(0);
    if (H.param_map.empty()) H.param_map.push_back(0);
    H.all_plane = all_plane;
    return H;
}

void build(zxs_sampler *s, const zxs_model_desc *d) {
    if (!d) fail(ZXS_INVALID_ARGUMENT, "null model");
    if (d->abi_version != ZXS_ABI_VERSION) fail(ZXS_INVALID_ARGUMENT, "model ABI version mismatch");
    if (d->mode > 1) fail(ZXS_INVALID_ARGUMENT, "bad mode");
    const uint32_t fwid = d->f_width;
    if (fwid > 1024) fail(ZXS_UNSUPPORTED, "f_width above 1024 is not supported");
    const int fw_need = std::max(1, int((fwid + 63) / 64));
    int FW = 1;
    while (FW < fw_need) FW *= 2;
    s->fw_template = FW;
    s->mode = d->mode;

    // ---- error model -> scan entries
    validate_csr("mech_vec_begin", d->mech_vec_begin, d->num_mechanisms, d->num_vectors);
    validate_csr("vec_bit_begin", d->vec_bit_begin, d->num_vectors, SIZE_MAX);
    validate_csr("mech_table_begin", d->mech_table_begin, d->num_mechanisms, SIZE_MAX);
    auto vec_mask = [&](uint32_t v, std::vector<uint64_t> &mask) {
        for (uint32_t i = d->vec_bit_begin[v]; i < d->vec_bit_begin[v + 1]; i++) {
            uint32_t b = d->vec_bits[i];
            if (b >= fwid) fail(ZXS_INVALID_ARGUMENT, "f_vector bit out of range");
            mask[b >> 6] ^= uint64_t(1) << (b & 63);
        }
    };
    std::map<std::vector<uint64_t>, uint32_t> flipsets;
    std::vector<uint64_t> flip_masks;
    auto flip_id = [&](const std::vector<uint64_t> &mask) -> uint32_t {
        bool any = false;
        for (uint64_t w : mask) any |= w != 0;
        if (!any) return zxs_dev::kNoFlip;
        auto it = flipsets.find(mask);
        if (it != flipsets.end()) return it->second;
        uint32_t id = static_cast<uint32_t>(flipsets.size());
        flipsets.emplace(mask, id);
        flip_masks.insert(flip_masks.end(), mask.begin(), mask.end());
        return id;
    };
    std::vector<zxs_dev::MechRec> recs;
    std::vector<uint32_t> ext_begin;
    std::vector<ulonglong2> ext;
    uint32_t dead = 0;
    for (uint32_t mi = 0; mi < d->num_mechanisms; mi++) {
        uint32_t v0 = d->mech_vec_begin[mi], nv = d->mech_vec_begin[mi + 1] - v0;
        std::vector<std::pair<uint64_t, uint32_t>> scan;  // (lim, flip)
        if (nv == 1) {
            // single: fire iff u < probability (sampler.cpp:269-280)
            uint64_t T = threshold_of(d->mech_probability[mi]);
            std::vector<uint64_t> mask(FW, 0);
            vec_mask(v0, mask);
            uint32_t fid = flip_id(mask);
            if (T > 0 && fid != zxs_dev::kNoFlip) scan.push_back({lim_of(T), fid});
        } else if (nv > 1) {
            // joint: inverse CDF over the table (sampler.cpp:281-302)
            uint32_t t0 = d->mech_table_begin[mi], t1 = d->mech_table_begin[mi + 1];
            if (nv > 31) fail(ZXS_UNSUPPORTED, "joint mechanism with more than 31 vectors");
            double acc = 0.0;
            uint64_t best = 0;
            bool effect = false;
            for (uint32_t o = 0; o < t1 - t0; o++) {
                acc += d->table[t0 + o];
                uint64_t T = threshold_of(acc);
                if (T <= best) continue;  // can never be the first hit
                best = T;
                std::vector<uint64_t> mask(FW, 0);
                for (uint32_t b = 0; b < nv; b++) {
                    if ((uint64_t(o) >> b) & 1) vec_mask(v0 + b, mask);
                }
                uint32_t fid = flip_id(mask);
                effect |= fid != zxs_dev::kNoFlip;
                scan.push_back({lim_of(T), fid});
                if (T == (uint64_t(1) << 53)) break;  // every later entry is unreachable
            }
            // Trailing no-flip entries behave like the no-hit fallback (outcome 0).
            while (!scan.empty() && scan.back().second == zxs_dev::kNoFlip) scan.pop_back();
            if (!effect) scan.clear();
        }
        // Record index = Philox stream = reference mechanism index (sampler.cpp:268).
        zxs_dev::MechRec rec;
        ext_begin.push_back(static_cast<uint32_t>(ext.size()));
        if (scan.empty()) {
            rec.lim0 = ~0ull;  // always "hits" the no-flip entry
            rec.flip0 = zxs_dev::kNoFlip;
            rec.n_extra = 0;
            dead++;
        } else {
            rec.lim0 = scan[0].first;
            rec.flip0 = scan[0].second;
            rec.n_extra = static_cast<uint32_t>(scan.size() - 1);
            for (size_t e = 1; e < scan.size(); e++) ext.push_back(make_ulonglong2(scan[e].first, scan[e].second));
        }
        recs.push_back(rec);
    }
    if (flip_masks.empty()) flip_masks.assign(FW, 0);
    std::vector<uint64_t> base(FW, 0);
    for (uint32_t i = 0; i < d->num_base_offset; i++) {
        uint32_t b = d->base_offset[i];
        if (b >= fwid) fail(ZXS_INVALID_ARGUMENT, "base_offset bit out of range");
        base[b >> 6] |= uint64_t(1) << (b & 63);
    }
    s->host_base = base;
    s->host_mechs.resize(d->num_mechanisms);
    for (uint32_t mi = 0; mi < d->num_mechanisms; mi++) {
        zxs_sampler::HostMech &hm = s->host_mechs[mi];
        const uint32_t v0 = d->mech_vec_begin[mi], nv = d->mech_vec_begin[mi + 1] - v0;
        hm.joint = nv > 1;
        for (uint32_t b = 0; b < nv; b++) {
            std::vector<uint64_t> mask(FW, 0);
            vec_mask(v0 + b, mask);
            hm.vecs.push_back(mask);
        }
        if (hm.joint) {
            hm.table.assign(d->table + d->mech_table_begin[mi], d->table + d->mech_table_begin[mi + 1]);
        } else {
            hm.p = d->mech_probability[mi];
        }
    }

    // ---- direct outputs
    validate_csr("direct_bit_begin", d->direct_bit_begin, d->num_direct, SIZE_MAX);
    std::vector<uint8_t> covered(d->num_outputs, 0);
    std::vector<uint32_t> direct_out(d->num_direct), direct_bits;
    for (uint32_t i = 0; i < d->num_direct; i++) {
        uint32_t o = d->direct_output[i];
        if (o >= d->num_outputs || covered[o]) fail(ZXS_INVALID_ARGUMENT, "bad direct output index");
        covered[o] = 1;
        direct_out[i] = o | (d->direct_flip_const[i] ? 0x80000000u : 0u);
        for (uint32_t b = d->direct_bit_begin[i]; b < d->direct_bit_begin[i + 1]; b++) {
            if (d->direct_bits[b] >= fwid) fail(ZXS_INVALID_ARGUMENT, "direct f bit out of range");
            direct_bits.push_back(d->direct_bits[b]);
        }
    }
    std::vector<uint32_t> direct_bit_begin(d->direct_bit_begin, d->direct_bit_begin + d->num_direct + 1);

    // ---- sparse geometric path data (compile.cpp:285-303 flip matrix, sampler.cpp:104-117)
    s->model_flags = d->flags;
    {
        bool structural = (d->flags & ZXS_MODEL_PURE_CLIFFORD_DETERMINISTIC) != 0;
        std::vector<double> l1mp(std::max<uint32_t>(1, d->num_mechanisms), 0.0);
        std::vector<uint32_t> fb{0}, fo;
        double expected = 0;
        for (uint32_t mi = 0; mi < d->num_mechanisms; mi++) {
            const auto &hm = s->host_mechs[mi];
            if (hm.joint || hm.vecs.size() != 1 || hm.p >= 1.0) structural = false;
            if (!hm.joint && hm.vecs.size() == 1) {
                for (uint32_t i = 0; i < d->num_direct; i++) {
                    bool acc = false;
                    for (uint32_t b = d->direct_bit_begin[i]; b < d->direct_bit_begin[i + 1]; b++) {
                        const uint32_t f = d->direct_bits[b];
                        acc ^= ((hm.vecs[0][f >> 6] >> (f & 63)) & 1) != 0;
                    }
                    if (acc) fo.push_back(d->direct_output[i]);
                }
                if (hm.p > 0.0 && hm.p < 1.0) l1mp[mi] = std::log1p(-hm.p);  // sampler.cpp:226
                expected += hm.p * double(fo.size() - fb.back());
            }
            fb.push_back(uint32_t(fo.size()));
        }
        s->sparse_structural = structural;
        s->sparse_expected_flips = expected;
        for (uint32_t i = 0; i < d->num_direct; i++) {  // sampler.cpp:131-140
            bool base_bit = d->direct_flip_const[i] != 0;
            for (uint32_t b = d->direct_bit_begin[i]; b < d->direct_bit_begin[i + 1]; b++) {
                const uint32_t f = d->direct_bits[b];
                base_bit ^= ((base[f >> 6] >> (f & 63)) & 1) != 0;
            }
            if (base_bit) s->const_one_outputs.push_back(d->direct_output[i]);
        }
        if (structural) {
            if (fo.empty()) fo.push_back(0);
            CK(cudaMalloc(&s->dev_log1mp, l1mp.size() * 8));
            CK(cudaMalloc(&s->dev_flip_begin, fb.size() * 4));
            CK(cudaMalloc(&s->dev_flip_out, fo.size() * 4));
            CK(cudaMemcpy(s->dev_log1mp, l1mp.data(), l1mp.size() * 8, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(s->dev_flip_begin, fb.data(), fb.size() * 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(s->dev_flip_out, fo.data(), fo.size() * 4, cudaMemcpyHostToDevice));
        }
    }

    // ---- components and chain tensors
    validate_csr("comp_out_begin", d->comp_out_begin, d->num_components, SIZE_MAX);
    validate_csr("comp_tensor_begin", d->comp_tensor_begin, d->num_components, d->num_tensors);
    validate_csr64("tensor_term_begin", d->tensor_term_begin, d->num_tensors);
    validate_csr64("term_factor_begin", d->term_factor_begin, d->num_terms);
    validate_csr64("factor_u_begin", d->factor_u_begin, d->num_factors);
    validate_csr64("factor_v_begin", d->factor_v_begin, d->num_factors);
    if (d->tensor_term_begin[d->num_tensors] != d->num_terms ||
        d->term_factor_begin[d->num_terms] != d->num_factors) {
        fail(ZXS_INVALID_ARGUMENT, "tensor/term totals mismatch");
    }
    if (d->num_terms >= (uint64_t(1) << 32) || d->num_factors >= (uint64_t(1) << 32)) {
        fail(ZXS_UNSUPPORTED, "more than 2^32 terms or factors");
    }
    uint32_t max_chain = 0;
    std::vector<uint32_t> comp_outputs;
    for (uint32_t c = 0; c < d->num_components; c++) {
        uint32_t n = d->comp_out_begin[c + 1] - d->comp_out_begin[c];
        if (d->comp_tensor_begin[c + 1] - d->comp_tensor_begin[c] != n + 1) {
            fail(ZXS_INVALID_ARGUMENT, "component needs normalization + one marginal per output");
        }
        if (n >= 4096) fail(ZXS_UNSUPPORTED, "component chain longer than 4095");
        max_chain = std::max(max_chain, n);
        for (uint32_t i = d->comp_out_begin[c]; i < d->comp_out_begin[c + 1]; i++) {
            uint32_t o = d->comp_outputs[i];
            if (o >= d->num_outputs || covered[o]) fail(ZXS_INVALID_ARGUMENT, "bad component output index");
            covered[o] = 1;
            comp_outputs.push_back(o);
        }
        for (uint32_t t = d->comp_tensor_begin[c]; t < d->comp_tensor_begin[c + 1]; t++) {
            if (d->tensor_param_width[t] > fwid + n) {
                fail(ZXS_INVALID_ARGUMENT, "eval_batch: parameter width mismatch");
            }
        }
    }
    s->all_outputs_covered = std::all_of(covered.begin(), covered.end(), [](uint8_t c) { return c != 0; });
    std::vector<uint32_t> tensor_term_begin(d->num_tensors + 1), term_factor_begin(d->num_terms + 1);
    for (uint32_t t = 0; t <= d->num_tensors; t++) tensor_term_begin[t] = uint32_t(d->tensor_term_begin[t]);
    for (uint64_t t = 0; t <= d->num_terms; t++) term_factor_begin[t] = uint32_t(d->term_factor_begin[t]);
    std::vector<double2> term_c(d->num_terms);
    for (uint64_t t = 0; t < d->num_terms; t++) term_c[t] = make_double2(d->term_c[2 * t], d->term_c[2 * t + 1]);
    std::vector<Factor> factors(d->num_factors);
    std::vector<uint16_t> selectors;
    selectors.reserve(d->factor_u_begin[d->num_factors] + d->factor_v_begin[d->num_factors]);
    std::vector<uint32_t> factor_width(d->num_factors, 0);
    for (uint32_t t = 0; t < d->num_tensors; t++) {
        for (uint64_t term = d->tensor_term_begin[t]; term < d->tensor_term_begin[t + 1]; term++) {
            for (uint64_t k = d->term_factor_begin[term]; k < d->term_factor_begin[term + 1]; k++) {
                factor_width[k] = d->tensor_param_width[t];
            }
        }
    }
    uint64_t nsel = 0;
    for (uint64_t k = 0; k < d->num_factors; k++) {
        Factor fr;
        fr.sel = static_cast<uint32_t>(selectors.size());
        uint64_t u0 = d->factor_u_begin[k], u1 = d->factor_u_begin[k + 1];
        uint64_t v0 = d->factor_v_begin[k], v1 = d->factor_v_begin[k + 1];
        if (u1 - u0 > 65535 || v1 - v0 > 65535) fail(ZXS_UNSUPPORTED, "selector too long");
        fr.nu = uint16_t(u1 - u0);
        fr.nv = uint16_t(v1 - v0);
        for (uint64_t i = u0; i < u1; i++) {
            if (d->factor_u_bits[i] >= factor_width[k]) fail(ZXS_INVALID_ARGUMENT, "eval_batch: parameter width mismatch");
            selectors.push_back(uint16_t(d->factor_u_bits[i]));
        }
        for (uint64_t i = v0; i < v1; i++) {
            if (d->factor_v_bits[i] >= factor_width[k]) fail(ZXS_INVALID_ARGUMENT, "eval_batch: parameter width mismatch");
            selectors.push_back(uint16_t(d->factor_v_bits[i]));
        }
        nsel += (u1 - u0) + (v1 - v0);
        if (d->factor_table[k] >= d->num_h_tables) fail(ZXS_INVALID_ARGUMENT, "h table index out of range");
        fr.table = d->factor_table[k];
        fr.pad = 0;
        factors[k] = fr;
    }
    if (selectors.empty()) selectors.push_back(0);
    std::vector<double2> h(4 * std::max<uint32_t>(1, d->num_h_tables), make_double2(0, 0));
    bool monomial = true;
    for (uint32_t t = 0; t < d->num_h_tables; t++) {
        for (int ab = 0; ab < 4; ab++) {
            double re = d->h_table[8 * t + 2 * ab], im = d->h_table[8 * t + 2 * ab + 1];
            h[4 * t + ab] = make_double2(re, im);
            // Clifford monomial check: 0 or 2^(m/2) w^k within 1e-9
            double mag = std::hypot(re, im);
            if (mag > 1e-9) {
                double lm = std::log2(mag) * 2.0;
                double ang = std::atan2(im, re) / (M_PI / 4);
                if (std::fabs(lm - std::round(lm)) > 1e-9 || std::fabs(ang - std::round(ang)) > 1e-9) monomial = false;
            }
        }
    }

    // ---- light program (zxs_kernels.cuh LightProg), filled after the heavy/mono split below
    auto build_light = [&](const std::vector<uint8_t> &comp_heavy, zxs_dev::LightProg &pg) -> bool {
        std::memset(&pg, 0, sizeof(pg));
        if (d->num_tensors > zxs_dev::kLightTensors || d->num_h_tables > zxs_dev::kLightTables) return false;
        uint32_t chain = 0;
        for (uint32_t c = 0; c < d->num_components; c++) {
            if (!comp_heavy[c]) chain = std::max(chain, d->comp_out_begin[c + 1] - d->comp_out_begin[c]);
        }
        if (fwid + chain > 64) return false;
        uint32_t nterm = 0, nfac = 0;
        std::vector<uint8_t> tensor_light(d->num_tensors, 0);
        for (uint32_t c = 0; c < d->num_components; c++) {
            if (comp_heavy[c]) continue;
            for (uint32_t t = d->comp_tensor_begin[c]; t < d->comp_tensor_begin[c + 1]; t++) tensor_light[t] = 1;
        }
        for (uint32_t t = 0; t < d->num_tensors; t++) {
            pg.tensor_term[t] = nterm;
            if (!tensor_light[t]) continue;
            for (uint64_t term = d->tensor_term_begin[t]; term < d->tensor_term_begin[t + 1]; term++) {
                if (nterm >= zxs_dev::kLightTerms) return false;
                pg.term_c[nterm] = make_double2(d->term_c[2 * term], d->term_c[2 * term + 1]);
                pg.term_factor[nterm] = nfac;
                for (uint64_t k = d->term_factor_begin[term]; k < d->term_factor_begin[term + 1]; k++) {
                    if (nfac >= zxs_dev::kLightFactors) return false;
                    unsigned long long u = 0, v = 0;
                    for (uint64_t i = d->factor_u_begin[k]; i < d->factor_u_begin[k + 1]; i++) u ^= 1ull << d->factor_u_bits[i];
                    for (uint64_t i = d->factor_v_begin[k]; i < d->factor_v_begin[k + 1]; i++) v ^= 1ull << d->factor_v_bits[i];
                    pg.fu[nfac] = u;
                    pg.fv[nfac] = v;
                    pg.ftable[nfac] = uint8_t(d->factor_table[k]);
                    nfac++;
                }
                nterm++;
            }
        }
        pg.tensor_term[d->num_tensors] = nterm;
        pg.term_factor[nterm] = nfac;
        pg.n_tables = std::max<uint32_t>(1, d->num_h_tables);
        pg.valid = 1;
        return true;
    };

    // ---- tabulated chains (zxs_kernels.cuh TabProg): each eligible light component's
    // autoregressive chain evaluated on the host for every assignment of its f-form
    // parities and sampled bits, in the reference's arithmetic (eval_batch order, no
    // FMA contraction, IEEE ratio; sampler.cpp:72-101)
    auto build_tab = [&](const std::vector<uint8_t> &comp_heavy, zxs_dev::LightProg &pg, std::vector<double> &tab) {
        pg.tab_valid = 0;
        std::memset(&pg.tab, 0, sizeof(pg.tab));
        tab.clear();
        uint32_t nforms = 0, nsel = 0;
        pg.tab.form_sel_begin[0] = 0;
        for (uint32_t c = 0; c < d->num_components && c < zxs_dev::kTabComps; c++) {
            if (comp_heavy[c]) continue;
            const uint32_t n = d->comp_out_begin[c + 1] - d->comp_out_begin[c];
            if (n == 0 || n > 10) continue;
            const uint32_t t0 = d->comp_tensor_begin[c];
            // distinct f-forms and per-factor (form id, sampled-bit mask) for u and v
            std::map<std::vector<uint32_t>, int> fid;
            std::vector<std::vector<uint32_t>> forms;
            struct FacT { int fu, fv; uint32_t su, sv, table; };
            std::vector<std::vector<std::pair<double2, std::vector<FacT>>>> tens(n + 1);
            bool ok = true;
            auto split = [&](const uint32_t *bits, uint64_t cnt, int &form, uint32_t &smask) {
                std::vector<uint32_t> fsel;
                smask = 0;
                for (uint64_t i = 0; i < cnt; i++) {
                    const uint32_t p = bits[i];
                    if (p < fwid) {
                        auto it = std::find(fsel.begin(), fsel.end(), p);
                        if (it != fsel.end()) fsel.erase(it); else fsel.push_back(p);
                    } else if (p - fwid < n) {
                        smask ^= 1u << (p - fwid);
                    } else {
                        ok = false;
                    }
                }
                std::sort(fsel.begin(), fsel.end());
                if (fsel.empty()) {
                    form = -1;
                    return;
                }
                auto it = fid.find(fsel);
                if (it != fid.end()) {
                    form = it->second;
                    return;
                }
                form = int(forms.size());
                fid.emplace(fsel, form);
                forms.push_back(fsel);
            };
            for (uint32_t j = 0; j <= n && ok; j++) {
                const uint32_t t = t0 + j;
                for (uint64_t term = d->tensor_term_begin[t]; term < d->tensor_term_begin[t + 1] && ok; term++) {
                    std::vector<FacT> fs;
                    for (uint64_t k = d->term_factor_begin[term]; k < d->term_factor_begin[term + 1]; k++) {
                        FacT f{};
                        split(d->factor_u_bits + d->factor_u_begin[k], d->factor_u_begin[k + 1] - d->factor_u_begin[k], f.fu, f.su);
                        split(d->factor_v_bits + d->factor_v_begin[k], d->factor_v_begin[k + 1] - d->factor_v_begin[k], f.fv, f.sv);
                        f.table = d->factor_table[k];
                        fs.push_back(f);
                    }
                    tens[j].push_back({make_double2(d->term_c[2 * term], d->term_c[2 * term + 1]), fs});
                }
            }
            const uint32_t mf = uint32_t(forms.size());
            if (!ok || mf + n - 1 > 12) continue;
            uint32_t fsel_count = 0;
            for (auto &f : forms) fsel_count += uint32_t(f.size());
            if (nforms + mf > zxs_dev::kTabForms || nsel + fsel_count > zxs_dev::kTabSel) continue;
            const size_t entries = (size_t(1) << mf) * ((size_t(1) << n) - 1);
            if (tab.size() + entries > (size_t(1) << 20)) continue;
            // exact host evaluation of tensor j at (f-form bits fa, sampled prefix)
            auto eval = [&](uint32_t j, uint32_t fa, uint32_t prefix) {
                volatile double acc_re = 0.0, acc_im = 0.0;
                for (const auto &tm : tens[j]) {
                    double pr = tm.first.x, pi = tm.first.y;
                    for (const FacT &f : tm.second) {
                        const uint32_t av = (f.fu >= 0 ? (fa >> f.fu) & 1u : 0u) ^ (__builtin_popcount(prefix & f.su) & 1u);
                        const uint32_t bv = (f.fv >= 0 ? (fa >> f.fv) & 1u : 0u) ^ (__builtin_popcount(prefix & f.sv) & 1u);
                        const double hr = d->h_table[8 * f.table + 2 * ((av << 1) | bv)];
                        const double hi = d->h_table[8 * f.table + 2 * ((av << 1) | bv) + 1];
                        volatile double t1 = pr * hr, t2 = pi * hi, t3 = pr * hi, t4 = pi * hr;
                        const double nr = t1 - t2, ni = t3 + t4;
                        pr = nr;
                        pi = ni;
                    }
                    acc_re = acc_re + pr;
                    acc_im = acc_im + pi;
                }
                return double(acc_re);
            };
            const size_t base = tab.size();
            tab.resize(base + entries);
            for (uint32_t fa = 0; fa < (1u << mf); fa++) {
                const double norm = eval(0, fa, 0);
                std::function<void(uint32_t, uint32_t, double)> dfs = [&](uint32_t j, uint32_t prefix, double prev) {
                    const double cur = eval(1 + j, fa, prefix);
                    const double ratio = cur / prev;
                    double cl;
                    if (!(ratio > -1e-6 && ratio < 1.0 + 1e-6)) {
                        cl = std::numeric_limits<double>::quiet_NaN();
                    } else {
                        cl = std::min(1.0, std::max(0.0, ratio));
                    }
                    tab[base + ((size_t((1u << j) - 1u)) << mf) + (size_t(prefix) << mf) + fa] = cl;
                    if (j + 1 < n) {
                        dfs(j + 1, prefix, cur);                     // bit j = 0: prev = cur
                        dfs(j + 1, prefix | (1u << j), prev - cur);  // bit j = 1: prev -= cur
                    }
                };
                dfs(0, 0, norm);
            }
            pg.tab.comp[c] = 0x80000000u | mf << 24 | nforms;
            pg.tab.base[c] = uint32_t(base);
            for (auto &f : forms) {
                for (uint32_t p : f) pg.tab.form_sel[nsel++] = uint16_t(p);
                pg.tab.form_sel_begin[++nforms] = uint16_t(nsel);
            }
            pg.tab_valid = 1;
        }
        if (tab.empty()) tab.push_back(0.0);
    };

    // ---- heavy components: compact chunked streams (zxs_heavy.cuh)
    // Components with >= mono_min factors run in mono_kernel (measured faster
    // than the per-warp shot-kernel chain from ~2k factors: config 4's chi=64
    // component, 2316 factors, 5.5e8 vs 4.1e8 shots/s); with ZXS_MONO=0, those
    // with >= heavy_min run in the exact heavy_kernel.
    uint64_t heavy_min = 20000, mono_min = 2000;
    if (const char *e = std::getenv("ZXS_HEAVY_MIN_FACTORS")) heavy_min = mono_min = std::strtoull(e, nullptr, 10);
    if (const char *e = std::getenv("ZXS_MONO_MIN_FACTORS")) mono_min = std::strtoull(e, nullptr, 10);
    bool use_mono = true;
    if (const char *e = std::getenv("ZXS_MONO")) use_mono = std::strcmp(e, "0") != 0;
    MonoHost MH = use_mono ? encode_mono(d, max_chain, mono_min) : MonoHost{};
    if (!use_mono) {
        MH.comp_mono.assign(std::max<uint32_t>(1, d->num_components), 0);
        MH.words.assign(4, 0);
        MH.chunks.push_back(make_uint4(0, 0, 0, 0));
        MH.dict.push_back(make_uint4(0, 0, 0, 0));
    }
    HeavyHost H = encode_heavy(d, max_chain, heavy_min, &MH.comp_mono);
    std::vector<uint8_t> &comp_heavy = H.comp_heavy;
    for (size_t c = 0; c < comp_heavy.size(); c++) comp_heavy[c] |= MH.comp_mono[c] ? 2 : 0;
    std::vector<uint32_t> &hw = H.words;
    std::vector<uint4> &hchunks = H.chunks;
    std::vector<uint32_t> &htcb = H.tensor_chunk_begin;
    std::vector<zxs_dev::HeavyComp> &hcomps = H.comps;
    const uint32_t heavy_zero_row = H.zero_row;

    // ---- device upload
    Arena ar;
    std::vector<zxs_dev::MechRec> recs_pad = recs.empty() ? std::vector<zxs_dev::MechRec>(1) : recs;
    size_t o_recs = ar.add(recs_pad);
    // fast filters (see zxs_dev::MechFast)
    std::vector<zxs_dev::MechFast> fast(recs.size());
    for (size_t i = 0; i < recs.size(); i++) {
        const zxs_dev::MechRec &r = recs[i];
        const uint32_t hi = uint32_t(r.lim0 >> 32);
        if (r.flip0 == zxs_dev::kNoFlip) {
            fast[i] = {hi, 0u};                 // hit at entry 0 = no error
        } else if (r.n_extra == 0) {
            fast[i] = {~hi, 0xffffffffu};       // miss = no error
        } else {
            fast[i] = {0u, 0u};                 // always resolve exactly
        }
    }
    std::vector<zxs_dev::MechFast> fast_pad = fast.empty() ? std::vector<zxs_dev::MechFast>(1, {0u, 0u}) : fast;
    size_t o_fast = ar.add(fast_pad);
    std::vector<uint32_t> ext_begin_pad = ext_begin.empty() ? std::vector<uint32_t>(1, 0) : ext_begin;
    size_t o_extb = ar.add(ext_begin_pad);
    size_t o_ext = ar.add(ext.empty() ? std::vector<ulonglong2>(1, make_ulonglong2(0, 0)) : ext);
    size_t o_flip = ar.add(flip_masks);
    size_t o_base = ar.add(base);
    std::vector<uint32_t> direct_out_pad = direct_out.empty() ? std::vector<uint32_t>(1, 0) : direct_out;
    size_t o_dout = ar.add(direct_out_pad);
    size_t o_dbb = ar.add(direct_bit_begin);
    std::vector<uint32_t> direct_bits_pad = direct_bits.empty() ? std::vector<uint32_t>(1, 0) : direct_bits;
    size_t o_dbits = ar.add(direct_bits_pad);
    std::vector<uint32_t> cob(d->comp_out_begin, d->comp_out_begin + d->num_components + 1);
    std::vector<uint32_t> ctb(d->comp_tensor_begin, d->comp_tensor_begin + d->num_components + 1);
    size_t o_cob = ar.add(cob);
    std::vector<uint32_t> comp_outputs_pad = comp_outputs.empty() ? std::vector<uint32_t>(1, 0) : comp_outputs;
    size_t o_co = ar.add(comp_outputs_pad);
    size_t o_ctb = ar.add(ctb);
    size_t o_ttb = ar.add(tensor_term_begin);
    std::vector<double2> term_c_pad = term_c.empty() ? std::vector<double2>(1, make_double2(0, 0)) : term_c;
    size_t o_tc = ar.add(term_c_pad);
    size_t o_tfb = ar.add(term_factor_begin);
    std::vector<Factor> factors_pad = factors.empty() ? std::vector<Factor>(1, Factor{}) : factors;
    size_t o_fac = ar.add(factors_pad);
    size_t o_sel = ar.add(selectors);
    size_t o_h = ar.add(h);
    size_t o_cheavy = ar.add(comp_heavy);
    size_t o_hchunks = ar.add(hchunks);
    size_t o_htcb = ar.add(htcb);
    size_t o_hw = ar.add(hw);
    size_t o_mw = ar.add(MH.words);
    size_t o_mch = ar.add(MH.chunks);
    size_t o_mtcb = ar.add(MH.tensor_chunk_begin);
    size_t o_mdict = ar.add(MH.dict);
    size_t o_mtdb = ar.add(MH.tensor_dict_begin);
    size_t o_mtw = ar.add(MH.tensor_width);
    size_t o_mtbb = ar.add(MH.tensor_basis_begin);
    size_t o_mbasis = ar.add(MH.basis);
    size_t o_mpmap = ar.add(MH.param_map);
    if (MH.block_forms.empty()) MH.block_forms.push_back(0);
    size_t o_bf = ar.add(MH.block_forms);
    size_t o_bfb = ar.add(MH.block_form_begin);
    if (MH.seg_words.empty()) MH.seg_words.assign(4, 0);
    if (MH.segs.empty()) MH.segs.push_back(make_uint4(0, 0, 0, 0));
    size_t o_sw = ar.add(MH.seg_words);
    size_t o_sg = ar.add(MH.segs);
    if (MH.tensor_null.empty()) MH.tensor_null.assign(2, 0ull);
    size_t o_null = ar.add(MH.tensor_null);

    CK(cudaMalloc(&s->dev_model, ar.host.size()));
    s->dev_model_bytes = ar.host.size();
    CK(cudaMemcpy(s->dev_model, ar.host.data(), ar.host.size(), cudaMemcpyHostToDevice));
    char *b = s->dev_model;
    DevModel &m = s->m;
    m.f_width = fwid;
    m.fw = FW;
    m.num_outputs = d->num_outputs;
    m.num_mech = d->num_mechanisms;
    m.num_direct = d->num_direct;
    m.num_components = d->num_components;
    m.max_chain = max_chain;
    uint32_t cs = std::max((fwid + 31) & ~31u, fwid + max_chain);
    m.col_stride = (cs + 3) & ~3u;
    if (m.col_stride == 0) m.col_stride = 4;
    s->mech_global = reinterpret_cast<const zxs_dev::MechRec *>(b + o_recs);
    s->ext_begin = reinterpret_cast<const uint32_t *>(b + o_extb);
    s->ext = reinterpret_cast<const ulonglong2 *>(b + o_ext);
    s->param_mechs = d->num_mechanisms <= zxs_dev::kParamMechs;
    s->mech_table.reset(new zxs_dev::MechTable<zxs_dev::kParamMechs>());
    s->mech_table1.reset(new zxs_dev::MechTable<1>());
    if (s->param_mechs) std::copy(fast.begin(), fast.end(), s->mech_table->fast);
    {
        bool use_light = true;
        if (const char *e = std::getenv("ZXS_LIGHT_PROG")) use_light = std::strcmp(e, "0") != 0;
        zxs_dev::LightProg &pg = s->mech_table->prog;
        if (use_light && build_light(comp_heavy, pg)) {
            s->light_tables = pg.n_tables;
        } else {
            pg.valid = 0;
            s->light_tables = 0;
        }
        bool use_tab = true;
        if (const char *e = std::getenv("ZXS_TAB")) use_tab = std::strcmp(e, "0") != 0;
        std::vector<double> tab;
        if (use_tab) build_tab(comp_heavy, pg, tab);
        if (!pg.tab_valid) tab.assign(1, 0.0);
        CK(cudaMalloc(&s->dev_tab, tab.size() * 8));
        CK(cudaMemcpy(s->dev_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
        s->info.num_tab_entries = pg.tab_valid ? tab.size() : 0;
        s->mech_table1->prog = pg;
    }
    s->fast_global = reinterpret_cast<const zxs_dev::MechFast *>(b + o_fast);
    s->dead_mechanisms = dead;
    m.flip_mask = reinterpret_cast<const uint64_t *>(b + o_flip);
    m.base_offset = reinterpret_cast<const uint64_t *>(b + o_base);
    m.direct_out = reinterpret_cast<const uint32_t *>(b + o_dout);
    m.direct_bit_begin = reinterpret_cast<const uint32_t *>(b + o_dbb);
    m.direct_bits = reinterpret_cast<const uint32_t *>(b + o_dbits);
    m.comp_out_begin = reinterpret_cast<const uint32_t *>(b + o_cob);
    m.comp_outputs = reinterpret_cast<const uint32_t *>(b + o_co);
    m.comp_tensor_begin = reinterpret_cast<const uint32_t *>(b + o_ctb);
    m.tensor_term_begin = reinterpret_cast<const uint32_t *>(b + o_ttb);
    m.term_c = reinterpret_cast<const double2 *>(b + o_tc);
    m.term_factor_begin = reinterpret_cast<const uint32_t *>(b + o_tfb);
    m.factors = reinterpret_cast<const Factor *>(b + o_fac);
    m.selectors = reinterpret_cast<const uint16_t *>(b + o_sel);
    m.h_table = reinterpret_cast<const double2 *>(b + o_h);
    m.comp_heavy = reinterpret_cast<const uint8_t *>(b + o_cheavy);
    s->has_heavy = !hcomps.empty();
    if (s->has_heavy) {
        zxs_dev::HeavyArgs &ha = s->heavy;
        ha.f_width = fwid;
        ha.col_words = heavy_zero_row + 1;  // rows incl. the all-zero padding row
        (void)H.max_chain;
        ha.words = reinterpret_cast<const uint32_t *>(b + o_hw);
        ha.chunks = reinterpret_cast<const uint4 *>(b + o_hchunks);
        ha.tensor_chunk_begin = reinterpret_cast<const uint32_t *>(b + o_htcb);
        ha.total_chunks = static_cast<uint32_t>(hchunks.size());
        ha.comp_outputs = m.comp_outputs;
        ha.htab = m.h_table;
        ha.n_tables = std::max<uint32_t>(1, d->num_h_tables);
        ha.n_comps = static_cast<uint32_t>(hcomps.size());
        for (size_t i = 0; i < hcomps.size(); i++) ha.comps[i] = hcomps[i];
        s->heavy_words = hw.size();
        s->heavy_smem = 128 + 2 * size_t(zxs_dev::kChunkWords) * 4 + size_t(ha.n_tables) * 64 +
                        size_t(zxs_dev::kHeavyWarps) * ha.col_words * 64;  // 16-bit planes
    }
    s->has_mono = !MH.comps.empty();
    if (s->has_mono) {
        zxs_dev::MonoArgs &ma = s->mono;
        ma.f_width = fwid;
        ma.n_planes = MH.all_plane + 2 + MH.max_chain;  // basis planes, ALL, ZERO, raw sampled bits
        ma.all_plane = MH.all_plane;
        ma.tensor_width = reinterpret_cast<const uint32_t *>(b + o_mtw);
        ma.tensor_basis_begin = reinterpret_cast<const uint32_t *>(b + o_mtbb);
        ma.basis = reinterpret_cast<const unsigned long long *>(b + o_mbasis);
        ma.param_map = reinterpret_cast<const uint16_t *>(b + o_mpmap);
        ma.words = reinterpret_cast<const uint32_t *>(b + o_mw);
        ma.chunks = reinterpret_cast<const uint4 *>(b + o_mch);
        ma.tensor_chunk_begin = reinterpret_cast<const uint32_t *>(b + o_mtcb);
        ma.total_chunks = static_cast<uint32_t>(MH.chunks.size());
        ma.dict = reinterpret_cast<const uint4 *>(b + o_mdict);
        ma.tensor_dict_begin = reinterpret_cast<const uint32_t *>(b + o_mtdb);
        ma.max_dict = std::max<uint32_t>(1, MH.max_dict);
        ma.stack_depth = std::max<uint32_t>(1, MH.max_depth);
        ma.comp_outputs = m.comp_outputs;
        ma.eval_tensor = -1;
        ma.n_comps = static_cast<uint32_t>(MH.comps.size());
        for (size_t i = 0; i < MH.comps.size(); i++) ma.comps[i] = MH.comps[i];
        s->mono_tensor = MH.tensor_index;
        if (const char *e = std::getenv("ZXS_MONO_WORDS")) s->mono_nw = std::atoi(e) == 1 ? 1 : 2;
        if (mono_smem_bytes(ma.n_planes, ma.max_dict, s->mono_nw, ma.stack_depth) > 227 * 1024) s->mono_nw = 1;
        if (mono_smem_bytes(ma.n_planes, ma.max_dict, s->mono_nw, ma.stack_depth) > 227 * 1024) s->mono_nw = 3;
        s->mono_smem = mono_smem_bytes(ma.n_planes, ma.max_dict, s->mono_nw, ma.stack_depth);
        s->dd_words = reinterpret_cast<const uint32_t *>(b + o_sw);
        s->dd_segs = reinterpret_cast<const uint4 *>(b + o_sg);
        s->dd_tsb = MH.tensor_seg_begin;
        s->dd_tdb = MH.tensor_dict_begin;
        s->dd_tw = MH.tensor_width;
        s->dd_tbb = MH.tensor_basis_begin;
        s->dd_key_mask = MH.comp_key_mask;
        s->dd_param_map = MH.param_map;
        s->dd_identity_map = true;  // every component reads its f columns at their raw positions
        for (uint32_t hc = 0; hc < MH.comps.size(); hc++) {
            s->dd_identity_map = s->dd_identity_map && MH.comps[hc].nf == fwid;
        }
        s->dd_tloads = MH.tensor_loads;
        s->dd_tread = MH.tensor_read_mask;
        s->dd_null = reinterpret_cast<const unsigned long long *>(b + o_null);
        s->dd_null_begin = MH.tensor_null_begin;
        if (const char *e = std::getenv("ZXS_DEDUP_NULL")) {
            if (std::atoi(e) == 0) s->dd_null_begin.assign(s->dd_null_begin.size(), 0u);
        }
        s->dd_tspw = MH.tensor_spw;
        s->dd_block_forms = reinterpret_cast<const uint32_t *>(b + o_bf);
        s->dd_block_form_begin = reinterpret_cast<const uint32_t *>(b + o_bfb);
        s->dd_tfb = MH.tensor_first_block;
        // stacks: kDedupWarps x depth x (Z, J0, J1) words per lane, then two 8-double leaf tables
        // per warp; between items the same area holds the key group's 64 raw parameter planes
        // (64 x 33 words)
        s->dd_stack_words = std::max<uint32_t>(zxs_dev::kDedupWarps * (ma.stack_depth * 96 + 32), 64 * 33);
        // dedup_eval_kernel's shared memory, per tensor: its form table (the block form values, or
        // the whole dictionary when a block does not fit), planes, stacks, then -- when they fit --
        // a copy of each warp's segment (record words read by LDS instead of L1/L2) and the staged
        // first dictionary entries of the block's forms
        const size_t fixed = size_t(MH.all_plane + 2) * 32 * 4 + size_t(s->dd_stack_words) * 4;
        const size_t nmt = MH.tensor_width.size();
        s->dd_t_layout.assign(nmt, uint4{0, 0, 0, 0});
        // ZXS_DEDUP_STAGE=0: block form values from register-staged entries only (tests)
        const char *stage_env = std::getenv("ZXS_DEDUP_STAGE");
        const bool stage_ok = !stage_env || std::atoi(stage_env) != 0;
        s->dd_smem = 0;
        for (size_t t = 0; t < nmt; t++) {
            uint32_t bforms = 0;
            const bool blocks = t < MH.tensor_first_block.size() && MH.tensor_first_block[t] != 0xffffffffu;
            if (blocks) {
                const uint32_t b0 = MH.tensor_first_block[t];
                const uint32_t nsg = MH.tensor_seg_begin[t + 1] - MH.tensor_seg_begin[t];
                const uint32_t bsegs = zxs_dev::kDedupWarps * std::max<uint32_t>(1, MH.tensor_spw[t]);
                for (uint32_t b = b0; b < b0 + (nsg + bsegs - 1) / bsegs; b++) {
                    bforms = std::max(bforms, MH.block_form_begin[b + 1] - MH.block_form_begin[b]);
                }
            }
            const uint32_t table = uint32_t(blocks ? std::max<size_t>(16, size_t(bforms) * 128)
                                                   : size_t(MH.tensor_dict_begin[t + 1] - MH.tensor_dict_begin[t]) * 16);
            uint32_t max_seg = 0;
            for (uint32_t g = MH.tensor_seg_begin[t]; g < MH.tensor_seg_begin[t + 1]; g++) max_seg = std::max(max_seg, MH.segs[g].y);
            size_t smem = table + fixed;
            uint32_t segbuf = (max_seg + 3) & ~3u;
            if (smem + size_t(zxs_dev::kDedupWarps) * segbuf * 4 > 227 * 1024) segbuf = 0;
            smem += size_t(zxs_dev::kDedupWarps) * segbuf * 4;
            const bool stage = blocks && bforms > 0 && smem + size_t(bforms) * 16 <= 227 * 1024 && stage_ok;
            if (stage) smem += size_t(bforms) * 16;
            s->dd_t_layout[t] = make_uint4(table, segbuf, stage ? 1u : 0u, uint32_t(smem));
            s->dd_smem = std::max(s->dd_smem, smem);
        }
        s->dedup = s->dd_smem <= 227 * 1024 && s->dd_key_mask.size() == MH.comps.size();
        if (const char *e = std::getenv("ZXS_DEDUP")) s->dedup = s->dedup && std::atoi(e) != 0;
    }
    s->info.num_mono_components = uint32_t(MH.comps.size());
    s->info.num_mono_records = MH.records;
    s->info.num_mono_dead_terms = MH.dead_terms;
    s->info.num_mono_negligible_terms = MH.negligible_terms;
    s->info.num_mono_forms = uint32_t(MH.dict.size());
    s->info.num_mono_loads = MH.loads;
    m.mech_entry_begin = nullptr;
    m.mech_stream = nullptr;
    m.entry_lim = nullptr;
    m.entry_flip = nullptr;

    s->num_tensors = d->num_tensors;
    s->tensor_width.assign(d->tensor_param_width, d->tensor_param_width + d->num_tensors);
    s->comp_out_begin = cob;
    s->comp_tensor_begin = ctb;
    s->comp_outputs = comp_outputs;
    s->direct_out = direct_out;

    zxs_sampler_info &in = s->info;
    in.mode = d->mode;
    in.num_outputs = d->num_outputs;
    in.num_detectors = d->num_detectors;
    in.num_observables = d->num_observables;
    in.f_width = fwid;
    in.num_mechanisms = d->num_mechanisms;
    in.num_direct = d->num_direct;
    in.num_components = d->num_components;
    in.max_chain = max_chain;
    in.fwords = FW;
    in.num_terms = d->num_terms;
    in.num_factors = d->num_factors;
    in.num_selector_bits = nsel;
    uint64_t chain_total = comp_outputs.size();
    in.philox_blocks_per_shot = d->num_mechanisms + chain_total;
    in.device_bytes = ar.host.size();
    in.device = s->device;
    in.monomial = monomial ? 1 : 0;

    CK(cudaMalloc(&s->dev_err, 3 * sizeof(unsigned long long)));
    unsigned long long init[3] = {0, ~0ull, 0};
    CK(cudaMemcpy(s->dev_err, init, sizeof(init), cudaMemcpyHostToDevice));
    CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; i++) {
        CK(cudaEventCreateWithFlags(&s->ev_done[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&s->ev_copied[i], cudaEventDisableTiming));
    }
    CK(cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, s->device));
    s->shots_per_lane = FW <= 2 ? 4 : 2;
    if (const char *e = std::getenv("ZXS_SHOTS_PER_LANE")) s->shots_per_lane = (std::atoi(e) == 4 && FW <= 2) ? 4 : 2;
    const void *kern = shot_kernel_for(FW, s->param_mechs, s->shots_per_lane);
    size_t smem = shot_smem_bytes(s);
    if (smem > 48 * 1024) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    }
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s->blocks_per_sm, kern, 32, smem));
    if (s->blocks_per_sm < 1) fail(ZXS_UNSUPPORTED, "shot kernel does not fit on an SM");
    if (s->has_heavy) {
        const void *hk = reinterpret_cast<const void *>(&zxs_dev::heavy_kernel);
        CK(cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s->heavy_smem)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s->heavy_blocks_per_sm, hk, zxs_dev::kHeavyWarps * 32,
                                                         s->heavy_smem));
        if (s->heavy_blocks_per_sm < 1) fail(ZXS_UNSUPPORTED, "heavy kernel does not fit on an SM");
    }
    if (s->has_mono) {
        const void *mk = mono_kernel_ptr(s->mono_nw);
        CK(cudaFuncSetAttribute(mk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s->mono_smem)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s->mono_blocks_per_sm, mk, mono_warps(s->mono_nw) * 32,
                                                         s->mono_smem));
        if (s->mono_blocks_per_sm < 1) fail(ZXS_UNSUPPORTED, "mono kernel does not fit on an SM");
        if (s->dedup) {
            CK(cudaFuncSetAttribute(reinterpret_cast<const void *>(&zxs_dev::dedup_eval_kernel),
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, int(s->dd_smem)));
            CK(cudaMallocHost(&s->dd_pinned, 64));
            CK(cudaMalloc(&s->dd_dev_stats, 16));
            CK(cudaMemset(s->dd_dev_stats, 0, 16));
            if (const char *e = std::getenv("ZXS_DEDUP_SYNC")) s->dd_async = std::atoi(e) == 0;
            if (const char *e = std::getenv("ZXS_DEDUP_FUSED")) s->dd_fused = std::atoi(e) != 0;
            // per-shot kernels: one full wave of resident blocks (grid-stride loops, no tail wave)
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &s->dd_init_occ, reinterpret_cast<const void *>(&zxs_dev::dedup_init_kernel), zxs_dev::kDedupInitWarps * 32, 0));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &s->dd_ar_occ, reinterpret_cast<const void *>(&zxs_dev::dedup_ar_kernel), 256, 0));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &s->dd_node_occ, reinterpret_cast<const void *>(&zxs_dev::dedup_node_pass_kernel<false>), 256, 0));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &s->dd_node_act_occ, reinterpret_cast<const void *>(&zxs_dev::dedup_node_pass_kernel<true>), 256, 0));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &s->dd_spec_occ, reinterpret_cast<const void *>(&zxs_dev::dedup_init_spec_kernel<unsigned long long>), 256, 0));
            if (const char *e = std::getenv("ZXS_DEDUP_SPEC")) s->dd_spec = std::atoi(e) != 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &s->dd_fused_occ, reinterpret_cast<const void *>(&zxs_dev::dedup_fused_ar_kernel), 256, 0));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &s->dd_raw_occ, reinterpret_cast<const void *>(&zxs_dev::dedup_init_raw_kernel<unsigned long long>), 256, 0));
        }
    }
}

// Launches mono_kernel for shots [first_shot, first_shot + shots): the
// large-chi components on the integer path, after shot_kernel left their
// f-columns in `fcols` ([f_width][fcols_ld32] 32-bit words).
void launch_mono(zxs_sampler *s, const zxs_dev::LaunchArgs &a, const uint32_t *fcols, uint64_t fcols_ld32,
                 int eval_tensor, double *eval_out, uint32_t f_width, cudaStream_t st) {
    zxs_dev::MonoArgs h = s->mono;
    h.seed = a.seed;
    h.first_shot = a.first_shot;
    h.shots = a.shots;
    for (int i = 0; i < 10; i++) h.k0_round[i] = a.k0_round[i];
    h.fcols = fcols;
    h.fcols_ld32 = fcols_ld32;
    h.out32 = a.out32;
    h.out_ld32 = a.ld32;
    h.counts = a.counts;
    h.uniforms = a.uniforms;
    h.uniforms_ld = a.uniforms_ld;
    h.err = s->dev_err;
    h.eval_tensor = eval_tensor;
    h.eval_out = eval_out;
    if (eval_tensor >= 0) {  // injected params: every raw parameter (f bits and sampled bits) is a column
        h.f_width = f_width;
        for (uint32_t hc = 0; hc < h.n_comps; hc++) {
            if (uint32_t(eval_tensor) >= h.comps[hc].first_tensor &&
                uint32_t(eval_tensor) <= h.comps[hc].first_tensor + h.comps[hc].n_out) {
                h.eval_comp = hc;
            }
        }
    }
    const int nw = s->mono_nw;  // configuration (mono_kernel_ptr)
    const uint64_t per_cta = uint64_t(mono_warps(nw)) * 1024 * mono_words(nw);
    h.n_cta_tiles = (a.shots + per_cta - 1) / per_cta;
    if (h.n_cta_tiles == 0) return;
    h.scratch = s->mono_scratch_get(size_t(3) * h.n_cta_tiles * per_cta * 8);
    const size_t smem = mono_smem_bytes(h.n_planes, h.max_dict, nw, h.stack_depth);
    if (smem > s->mono_smem) {
        CK(cudaFuncSetAttribute(mono_kernel_ptr(nw), cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    }
    const unsigned grid = unsigned(std::min<uint64_t>(h.n_cta_tiles, uint64_t(s->sm_count) * std::max(1, s->mono_blocks_per_sm)));
    void *args[] = {&h};
    CK(cudaLaunchKernel(mono_kernel_ptr(nw), dim3(grid), dim3(mono_warps(nw) * 32), args, smem, st));
}

// ---- deduplicated large-chi path (zxs_dedup.cuh)
constexpr uint32_t kDedupRoundKeys = 65536;  // fused chains: expanded keys per position (one round)
// Group partial sums of one evaluation round live in one buffer of at most this many bytes (4 GB
// of the 180 GB: config 3 then needs 38 evaluation rounds per 2^28 shots instead of 91 at 1 GB);
// a tensor of G summation groups is evaluated in rounds of about budget / (8 G) keys, each round
// reading the device key count (rounds past it exit at once), so no host round trip decides how
// many run.
size_t dedup_partial_budget() {
    size_t mb = 4096;
    if (const char *e = std::getenv("ZXS_DEDUP_PARTIAL_MB")) mb = size_t(std::max(64L, std::atol(e)));
    return mb << 20;
}

struct DedupBufs {
    unsigned long long *key;
    uint32_t *active;    // main-lineage speculation: active shots (aliases key, unused on that path)
    uint32_t *n_active;
    uint32_t *slot;
    double *prev, *value0, *value, *partial;
    size_t partial_bytes;
    unsigned long long *counts;  // per output, added to the caller's counts when the chain completes
    unsigned int *max_count;     // sync-free path: [0] largest key count of a position, [1] largest
                                 // expanded key count of a fused chain
    unsigned long long *err;     // staged ratio-breakdown report of the sync-free path
    unsigned long long *xkeys;   // expanded keys of one chain position (fused chains)
    double *fvals[zxs_dev::kDedupMaxFused + 1];  // dense values per chain position (fused chains)
    // [0] base keys (= level-0 nodes), [1], [2] node tables of the later levels (alternating),
    // [3] the level's node keys (node levels); the step-by-step sync path uses [0], [1]
    zxs_dev::DedupTable table[4];
    zxs_dev::DedupNodeArrays nodes[2];  // node levels: per node key, prev, cur, key slot, decision
};

// Distinct keys per chain position the tables hold (ZXS_DEDUP_MAX_KEYS, default
// 2^20); a batch with more falls back to mono_kernel (bit-identical values).
uint32_t dedup_max_keys() {
    uint32_t m = 1u << 20;
    if (const char *e = std::getenv("ZXS_DEDUP_MAX_KEYS")) m = uint32_t(std::max(16L, std::atol(e)));
    return m;
}

DedupBufs dedup_reserve(zxs_sampler *s, uint64_t shots) {
    uint64_t cap = std::max<uint64_t>(s->dd_cap_shots, 1024);
    while (cap < shots) cap *= 2;
    const uint32_t max_ids = uint32_t(std::min<uint64_t>(cap, dedup_max_keys()));
    uint32_t slots = 4096;  // >= 2 max_ids + room for the inserts in flight when the limit is hit
    while (slots < 2 * max_ids + 65536u) slots *= 2;
    uint32_t max_segs = 1;
    for (size_t t = 0; t + 1 < s->dd_tsb.size(); t++) max_segs = std::max(max_segs, s->dd_tsb[t + 1] - s->dd_tsb[t]);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t nout = std::max<uint32_t>(1, s->m.num_outputs);
    const size_t per_table = al(size_t(slots) * 8) + al(size_t(slots) * 4) + al(4) + al(size_t(max_ids) * 8) +
                             al(size_t(max_ids) * 4);
    // partials: one round of the fused chain's expanded keys at least, else the budget (or all keys)
    const size_t partial_bytes = std::max(size_t(max_segs) * kDedupRoundKeys * 8,
                                          std::min(dedup_partial_budget(), size_t(max_segs) * max_ids * 8));
    const size_t bytes = al(cap * 8) + al(cap * 4) + al(cap * 8) + 2 * al(size_t(slots) * 8) +
                         al(partial_bytes) + al(nout * 8) + al(4) + al(8) + al(24) + al(size_t(kDedupRoundKeys) * 8) +
                         (zxs_dev::kDedupMaxFused + 1) * al(size_t(kDedupRoundKeys) * 8) + 4 * per_table +
                         2 * (3 * al(size_t(slots) * 8) + al(size_t(slots) * 4) +
                              al(size_t(slots) * sizeof(zxs_dev::DedupNodeRec)));
    if (bytes > s->dd_buf_bytes || slots != s->dd_table_slots) {
        if (s->dd_buf) CK(cudaFree(s->dd_buf));
        s->dd_buf = nullptr;
        s->dd_buf_bytes = 0;
        CK(cudaMalloc(&s->dd_buf, bytes));
        s->dd_buf_bytes = bytes;
        s->dd_dirty = true;
    }
    s->dd_cap_shots = cap;
    DedupBufs d;
    char *p = s->dd_buf;
    auto take = [&](size_t n) { char *r = p; p += al(n); return r; };
    d.key = reinterpret_cast<unsigned long long *>(take(cap * 8));
    d.slot = reinterpret_cast<uint32_t *>(take(cap * 4));
    d.prev = reinterpret_cast<double *>(take(cap * 8));
    d.value0 = reinterpret_cast<double *>(take(size_t(slots) * 8));
    d.value = reinterpret_cast<double *>(take(size_t(slots) * 8));
    d.partial = reinterpret_cast<double *>(take(partial_bytes));
    d.partial_bytes = partial_bytes;
    d.counts = reinterpret_cast<unsigned long long *>(take(nout * 8));
    d.max_count = reinterpret_cast<unsigned int *>(take(8));
    d.active = reinterpret_cast<uint32_t *>(d.key);
    d.n_active = reinterpret_cast<uint32_t *>(take(8));
    d.err = reinterpret_cast<unsigned long long *>(take(24));
    d.xkeys = reinterpret_cast<unsigned long long *>(take(size_t(kDedupRoundKeys) * 8));
    for (uint32_t i = 0; i <= zxs_dev::kDedupMaxFused; i++) d.fvals[i] = reinterpret_cast<double *>(take(size_t(kDedupRoundKeys) * 8));
    for (int i = 0; i < 4; i++) {
        zxs_dev::DedupTable &t = d.table[i];
        t.keys = reinterpret_cast<unsigned long long *>(take(size_t(slots) * 8));
        t.ids = reinterpret_cast<uint32_t *>(take(size_t(slots) * 4));
        t.mask = slots - 1;
        t.max_ids = max_ids;
        t.count = reinterpret_cast<uint32_t *>(take(4));
        t.ukeys = reinterpret_cast<unsigned long long *>(take(size_t(max_ids) * 8));
        t.uslot = reinterpret_cast<uint32_t *>(take(size_t(max_ids) * 4));
    }
    for (int i = 0; i < 2; i++) {
        zxs_dev::DedupNodeArrays &na = d.nodes[i];
        na.key = reinterpret_cast<unsigned long long *>(take(size_t(slots) * 8));
        na.prev = reinterpret_cast<double *>(take(size_t(slots) * 8));
        na.cur = reinterpret_cast<double *>(take(size_t(slots) * 8));
        na.kslot = reinterpret_cast<uint32_t *>(take(size_t(slots) * 4));
        na.rec = reinterpret_cast<zxs_dev::DedupNodeRec *>(take(size_t(slots) * sizeof(zxs_dev::DedupNodeRec)));
    }
    if (s->dd_dirty) {
        for (int i = 0; i < 4; i++) {
            CK(cudaMemset(d.table[i].keys, 0xff, size_t(slots) * 8));
            CK(cudaMemset(d.table[i].ids, 0, size_t(slots) * 4));  // ids stay in range (dedup_insert)
            CK(cudaMemset(d.table[i].count, 0, 4));
        }
        CK(cudaDeviceSynchronize());
        s->dd_table_slots = slots;
        s->dd_dirty = false;
    }
    return d;
}

uint32_t dedup_count(zxs_sampler *s, const zxs_dev::DedupTable &t, cudaStream_t st) {
    CK(cudaMemcpyAsync(s->dd_pinned, t.count, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return s->dd_pinned[0];
}

// Values of mono tensor `mt` for the table's n distinct keys, in id order.
// n_dev: the key count is read on the device (one round of at most n = kDedupRoundKeys keys).
// keys/uslot: the keys to contract and where their values go (value[uslot[k]], or value[k] when
// uslot is null); n_dev/n_mult: n = min(*n_dev x n_mult, n) read on the device.
void dedup_eval(zxs_sampler *s, uint32_t mt, const unsigned long long *keys, const uint32_t *uslot, uint32_t n,
                double *value, double *partial, size_t partial_bytes, cudaStream_t st, const uint32_t *n_dev = nullptr,
                uint32_t n_mult = 1, size_t value_slots = 0) {
    const uint32_t g0 = s->dd_tsb[mt], ng = s->dd_tsb[mt + 1] - g0;
    if (n == 0) return;
    if (ng == 0) {  // every term dead: the value is exactly 0 (for every slot)
        CK(cudaMemsetAsync(value, 0, value_slots * 8, st));
        return;
    }
    const zxs_dev::MonoArgs &m = s->mono;
    // partial sums: one per summation group (spw consecutive segments, walked by one warp)
    const uint32_t spw = std::max<uint32_t>(1, mt < s->dd_tspw.size() ? s->dd_tspw[mt] : 1);
    const uint32_t ngroups = (ng + spw - 1) / spw;
    // keys per round: as many as the partial buffer holds for this tensor's groups (whole key groups)
    const uint64_t fit = partial_bytes / (uint64_t(ngroups) * 8);
    uint64_t cap = fit;
    if (const char *e = std::getenv("ZXS_DEDUP_ROUND_KEYS")) cap = std::min<uint64_t>(cap, uint64_t(std::max(1L, std::atol(e))));
    const uint32_t round = uint32_t(std::max<uint64_t>(zxs_dev::kDedupKeysPerWarp,
                                                       std::min<uint64_t>(n, cap) / zxs_dev::kDedupKeysPerWarp *
                                                           zxs_dev::kDedupKeysPerWarp));
    for (uint32_t r0 = 0; r0 < n; r0 += round) {
        zxs_dev::DedupEvalArgs e{};
        e.words = s->dd_words;
        e.segs = s->dd_segs + g0;
        e.n_segs = ng;
        e.dict = m.dict + s->dd_tdb[mt];
        e.n_dict = s->dd_tdb[mt + 1] - s->dd_tdb[mt];
        e.basis = m.basis + s->dd_tbb[mt];
        e.width = std::min(s->dd_tw[mt], m.all_plane);
        e.all_plane = m.all_plane;
        e.n_planes = m.all_plane + 2;
        e.stack_depth = m.stack_depth;
        e.stack_words = s->dd_stack_words;
        e.keys = keys + r0;
        e.n_keys = std::min(round, n - r0);
        e.key_base = r0;
        e.partial = partial;
        const uint4 lay = s->dd_t_layout[mt];  // {table bytes, segment buffer words, stage entries, smem}
        e.seg_buf_words = lay.y;
        e.table_bytes = lay.x;
        if (mt < s->dd_tfb.size() && s->dd_tfb[mt] != 0xffffffffu) {
            e.block_forms = s->dd_block_forms;
            e.block_form_begin = s->dd_block_form_begin;
            e.first_block = s->dd_tfb[mt];
            e.stage_entries = lay.z;
        }
        e.segs_per_warp = spw;
        e.n_dev = n_dev;
        e.n_mult = n_mult;
        e.stats = s->dd_dev_stats;
        e.tensor_loads = mt < s->dd_tloads.size() ? s->dd_tloads[mt] : 0;
        s->dd_stats[4] += 1;
        const uint32_t bsegs = zxs_dev::kDedupWarps * std::max(e.segs_per_warp, 1u);
        const uint64_t items = uint64_t((e.n_keys + zxs_dev::kDedupKeysPerWarp - 1) / zxs_dev::kDedupKeysPerWarp) *
                               ((ng + bsegs - 1) / bsegs);
        const unsigned grid = unsigned(std::min<uint64_t>(items, uint64_t(s->sm_count)));
        cudaEvent_t t0 = nullptr;
        s->time_begin(3, st, t0);
        void *args[] = {&e};
        CK(cudaLaunchKernel(reinterpret_cast<const void *>(&zxs_dev::dedup_eval_kernel), dim3(grid),
                            dim3(zxs_dev::kDedupWarps * 32), args, lay.w, st));
        s->time_end(3, st, t0);
        s->time_begin(4, st, t0);
        zxs_dev::dedup_reduce_kernel<<<std::min((e.n_keys + 127) / 128, uint32_t(s->sm_count) * 8), 128, 0, st>>>(
            partial, ngroups, e.n_keys, n_dev, n_mult, r0, uslot ? uslot + r0 : nullptr, uslot ? value : value + r0);
        CK(cudaGetLastError());
        s->time_end(4, st, t0);
    }
}

// The large-chi components of shots [first_shot, first_shot + shots) on the
// deduplicated path, after shot_kernel left their f-columns in `fcols`. A
// chain position with more distinct keys than the tables hold sends the
// whole batch to mono_kernel instead (same canonical values, so the same bits).
void launch_dedup_sync(zxs_sampler *s, const zxs_dev::LaunchArgs &a, const uint32_t *fcols, uint64_t fcols_ld32,
                       cudaStream_t st) {
    if (a.shots == 0) return;
    DedupBufs d = dedup_reserve(s, a.shots);
    const zxs_dev::MonoArgs &m = s->mono;
    const unsigned pgrid = unsigned(std::min<uint64_t>((a.shots + 255) / 256, uint64_t(s->sm_count) * 8));
    const uint32_t nout = s->m.num_outputs;
    s->dd_dirty = true;  // until the chain completes
    if (a.counts) CK(cudaMemsetAsync(d.counts, 0, size_t(std::max<uint32_t>(nout, 1)) * 8, st));
    cudaEvent_t t0 = nullptr;
    auto clear = [&](const zxs_dev::DedupTable &t, uint32_t n) {
        s->time_begin(4, st, t0);
        zxs_dev::dedup_clear_kernel<<<std::max(1u, std::min((n + 255) / 256, 1024u)), 256, 0, st>>>(t, n);
        CK(cudaGetLastError());
        s->time_end(4, st, t0);
    };
    s->dd_stats[0] += 1;
    auto fallback = [&]() {  // tables left dirty: reset on the next call
        s->dd_stats[1] += 1;
        s->time_begin(2, st, t0);
        launch_mono(s, a, fcols, fcols_ld32, -1, nullptr, 0, st);
        s->time_end(2, st, t0);
    };
    for (uint32_t hc = 0; hc < m.n_comps; hc++) {
        const zxs_dev::HeavyComp cd = m.comps[hc];
        zxs_dev::DedupInitArgs ia{};
        ia.shots = a.shots;
        ia.fcols = fcols;
        ia.fcols_ld32 = fcols_ld32;
        for (uint32_t p = 0; p < cd.nf; p++) {  // key bit p = local f parameter p
            if ((s->dd_key_mask[hc] >> p) & 1ull) {
                ia.cols[ia.n_cols] = s->dd_param_map[cd.pmap_begin + p];
                ia.bits[ia.n_cols++] = uint8_t(p);
            }
        }
        ia.key = d.key;
        ia.slot = d.slot;
        ia.table = d.table[0];
        s->time_begin(4, st, t0);
        void *iargs[] = {&ia};
        const uint64_t iwarps = (a.shots + 1023) / 1024;
        const unsigned igrid = unsigned(std::min<uint64_t>((iwarps + zxs_dev::kDedupInitWarps - 1) / zxs_dev::kDedupInitWarps,
                                                           uint64_t(s->sm_count) * std::max(1, s->dd_init_occ)));
        CK(cudaLaunchKernel(reinterpret_cast<const void *>(&zxs_dev::dedup_init_kernel), dim3(igrid),
                            dim3(zxs_dev::kDedupInitWarps * 32), iargs, 0, st));
        s->time_end(4, st, t0);
        uint32_t n = dedup_count(s, d.table[0], st);
        if (n > d.table[0].max_ids) return fallback();
        dedup_eval(s, cd.first_tensor, d.table[0].ukeys, d.table[0].uslot, n, d.value0, d.partial, d.partial_bytes, st, nullptr, 1,
                   d.table[0].mask + 1);
        for (uint32_t j = 0; j < cd.n_out; j++) {
            const zxs_dev::DedupTable &cur = d.table[j & 1], &nxt = d.table[(j + 1) & 1];
            dedup_eval(s, cd.first_tensor + 1 + j, cur.ukeys, cur.uslot, n, d.value, d.partial, d.partial_bytes, st, nullptr, 1,
                       cur.mask + 1);
            zxs_dev::DedupArArgs ra{};
            ra.seed = a.seed;
            ra.first_shot = a.first_shot;
            ra.shots = a.shots;
            for (int i = 0; i < 10; i++) ra.k0_round[i] = a.k0_round[i];
            ra.ci = cd.ci;
            ra.j = j;
            ra.out = s->comp_outputs[cd.out_begin + j];
            ra.f_width = cd.nf;  // the key's sampled bits follow the local f parameters
            ra.key_mask = s->dd_key_mask[hc];
            ra.key = d.key;
            ra.slot = d.slot;
            ra.prev = d.prev;
            ra.value0 = d.value0;
            ra.value = d.value;
            ra.cur = cur;
            ra.next = nxt;
            ra.insert_next = j + 1 < cd.n_out;
            ra.out32 = a.out32;
            ra.out_ld32 = a.ld32;
            ra.counts = a.counts ? d.counts : nullptr;
            ra.uniforms = a.uniforms;
            ra.uniforms_ld = a.uniforms_ld;
            ra.upos = cd.upos_base + j;
            ra.err = s->dev_err;
            s->time_begin(4, st, t0);
            void *rargs[] = {&ra};
            const unsigned agrid =
                unsigned(std::min<uint64_t>((a.shots + 256 * zxs_dev::kDedupArGroups - 1) / (256 * zxs_dev::kDedupArGroups), uint64_t(s->sm_count) * std::max(1, s->dd_ar_occ)));
            CK(cudaLaunchKernel(reinterpret_cast<const void *>(&zxs_dev::dedup_ar_kernel), dim3(agrid), dim3(256), rargs,
                                0, st));
            s->time_end(4, st, t0);
            clear(cur, n);
            if (ra.insert_next) {
                n = dedup_count(s, nxt, st);
                if (n > nxt.max_ids) return fallback();
            }
        }
        if (cd.n_out == 0) clear(d.table[0], n);  // no autoregressive step cleared it
    }
    if (a.counts) {
        s->time_begin(4, st, t0);
        zxs_dev::dedup_add_counts_kernel<<<(nout + 255) / 256, 256, 0, st>>>(d.counts, a.counts, nout);
        CK(cudaGetLastError());
        s->time_end(4, st, t0);
    }
    s->dd_dirty = false;
}

void launch_shots(zxs_sampler *s, zxs_dev::LaunchArgs &a, cudaStream_t st);

// The f columns of a batch whose shot_kernel pass stored only per-shot f words
// (raw keys): shot_kernel again in error-batch mode (no outputs), into the spare
// buffer. Only a batch the deduplicated path must redo needs them.
const uint32_t *regen_fcols(zxs_sampler *s, const zxs_dev::LaunchArgs &a, cudaStream_t st) {
    zxs_dev::LaunchArgs b = a;
    b.fcols_out = a.fcols_spare;
    b.fcols_ld32 = a.heavy_ld32;
    b.out32 = nullptr;
    b.counts = nullptr;
    b.heavy_fcols = nullptr;
    b.heavy_fraw = nullptr;
    launch_shots(s, b, st);
    CK(cudaGetLastError());
    return a.fcols_spare;
}

// The same chain without host round trips: key counts stay on the device (one
// evaluation round of at most kDedupRoundKeys keys per position), the largest
// count is checked once at the end; a batch that needed more rounds (or
// overflowed the tables) is redone on the synchronous path, which overwrites
// every output it wrote (counts are staged, so nothing is added twice).
//
// dedup_lineage: the main lineage of component hc for dedup_init_spec_kernel --
// the all-zero key's node at each level, contracted one key at a time with the
// same dedup_eval, its record from the same node_rec (dedup_main_rec_kernel),
// the likelier bit taken (P(bit = 1) = 1 - T 2^-53). Computed once per sampler
// (the values depend only on the model); ok = false (no speculation) when a
// level's ratio is out of range, which the node passes must report per shot.
const zxs_sampler::Lineage *dedup_lineage(zxs_sampler *s, uint32_t hc, const DedupBufs &d, cudaStream_t st) {
    if (s->dd_lineage.size() < s->mono.n_comps) s->dd_lineage.resize(s->mono.n_comps);
    zxs_sampler::Lineage &L = s->dd_lineage[hc];
    if (L.done) return &L;
    L.done = true;
    const zxs_dev::HeavyComp cd = s->mono.comps[hc];
    if (!s->dd_spec_dev) CK(cudaMalloc(&s->dd_spec_dev, 64));
    auto *kdev = reinterpret_cast<unsigned long long *>(s->dd_spec_dev);
    auto *vdev = reinterpret_cast<double *>(s->dd_spec_dev + 8);               // cur, pv
    auto *rdev = reinterpret_cast<zxs_dev::DedupNodeRec *>(s->dd_spec_dev + 32);
    auto value = [&](uint32_t tj, unsigned long long key) {
        key &= s->dd_tread[tj];
        CK(cudaMemcpyAsync(kdev, &key, 8, cudaMemcpyHostToDevice, st));
        dedup_eval(s, tj, kdev, nullptr, 1, vdev, d.partial, d.partial_bytes, st, nullptr, 1, 1);
        double v = 0;
        CK(cudaMemcpyAsync(&v, vdev, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return v;
    };
    double pv = value(cd.first_tensor, 0ull);
    unsigned long long key = 0;
    for (uint32_t j = 0; j < cd.n_out; j++) {
        const double cur = value(cd.first_tensor + 1 + j, key);
        const double in[2] = {cur, pv};
        CK(cudaMemcpyAsync(vdev, in, 16, cudaMemcpyHostToDevice, st));
        zxs_dev::dedup_main_rec_kernel<<<1, 1, 0, st>>>(vdev, rdev);
        CK(cudaGetLastError());
        zxs_dev::DedupNodeRec r;
        CK(cudaMemcpyAsync(&r, rdev, sizeof r, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (r.T & zxs_dev::kNodeErr) return &L;
        const uint32_t b = r.T < (1ull << 52) ? 1u : 0u;
        L.T[j] = r.T;
        L.tie_lo[j] = r.tie_lo;
        L.tie_w[j] = r.tie_w;
        L.bits |= b << j;
        pv = b ? pv - cur : cur;  // sampler.cpp:95-98 (dedup_node_prep_kernel's __dsub_rn)
        const uint32_t p = cd.nf + j;
        if (b && p < 63 && ((s->dd_key_mask[hc] >> p) & 1ull)) key |= 1ull << p;
    }
    L.ok = true;
    return &L;
}

void launch_dedup(zxs_sampler *s, const zxs_dev::LaunchArgs &a, const uint32_t *fcols, uint64_t fcols_ld32,
                  cudaStream_t st) {
    if (a.shots == 0) return;
    if (!s->dd_async) return launch_dedup_sync(s, a, fcols, fcols_ld32, st);
    DedupBufs d = dedup_reserve(s, a.shots);
    const zxs_dev::MonoArgs &m = s->mono;
    const uint32_t nout = s->m.num_outputs;
    const uint32_t limit = d.table[0].max_ids;                               // keys per position (rounds)
    const uint32_t flimit = std::min(kDedupRoundKeys, d.table[0].max_ids);   // fused chains: expanded keys
    s->dd_dirty = true;  // until the chain completes
    CK(cudaMemsetAsync(d.max_count, 0, 8, st));
    if (a.counts) CK(cudaMemsetAsync(d.counts, 0, size_t(std::max<uint32_t>(nout, 1)) * 8, st));
    zxs_dev::dedup_err_init_kernel<<<1, 1, 0, st>>>(d.err);
    CK(cudaGetLastError());
    cudaEvent_t t0 = nullptr;
    const unsigned cgrid = unsigned(s->sm_count) * 2;
    auto clear = [&](const zxs_dev::DedupTable &t, uint32_t mult = 1, unsigned int *maxc = nullptr) {
        s->time_begin(4, st, t0);
        zxs_dev::dedup_clear_dev_kernel<<<cgrid, 256, 0, st>>>(t, maxc ? maxc : d.max_count, mult);
        CK(cudaGetLastError());
        s->time_end(4, st, t0);
        s->time_begin(4, st, t0);
        zxs_dev::dedup_reset_kernel<<<1, 1, 0, st>>>(t.count);
        CK(cudaGetLastError());
        s->time_end(4, st, t0);
    };
    s->dd_stats[0] += 1;
    for (uint32_t hc = 0; hc < m.n_comps; hc++) {
        const zxs_dev::HeavyComp cd = m.comps[hc];
        // fused chain: every position's keys = base keys x patterns of the sampled bits it reads
        uint32_t relevant = 0, nrel = 0;
        uint64_t relpos = 0;
        for (uint32_t j = 0; j + 1 < cd.n_out; j++) {
            const uint32_t p = cd.nf + j;
            if (p < 63 && ((s->dd_key_mask[hc] >> p) & 1ull)) {
                relevant |= 1u << j;
                if (nrel < 8) relpos |= uint64_t(p) << (8 * nrel);
                nrel++;
            }
        }
        auto nb_of = [&](uint32_t pos) { return pos < 2 ? 0u : uint32_t(__builtin_popcount(relevant & ((1u << (pos - 1)) - 1))); };
        uint32_t sum_p = 0;
        for (uint32_t pos = 0; pos <= cd.n_out; pos++) sum_p += 1u << nb_of(pos);
        const bool fused = s->dd_fused && cd.n_out >= 1 && cd.n_out <= zxs_dev::kDedupMaxFused && sum_p <= 16;
        zxs_dev::DedupInitArgs ia{};
        ia.shots = a.shots;
        ia.fcols = fcols;
        ia.fcols_ld32 = fcols_ld32;
        for (uint32_t p = 0; p < cd.nf; p++) {  // key bit p = local f parameter p
            if ((s->dd_key_mask[hc] >> p) & 1ull) {
                ia.cols[ia.n_cols] = s->dd_param_map[cd.pmap_begin + p];
                ia.bits[ia.n_cols++] = uint8_t(p);
            }
        }
        ia.key = fused ? nullptr : d.key;
        ia.slot = d.slot;
        ia.table = d.table[0];
        const uint64_t iwarps = (a.shots + 1023) / 1024;
        const unsigned igrid = unsigned(std::min<uint64_t>((iwarps + zxs_dev::kDedupInitWarps - 1) / zxs_dev::kDedupInitWarps,
                                                           uint64_t(s->sm_count) * std::max(1, s->dd_init_occ)));
        // main-lineage speculation: zero-key shots that stay on the lineage skip the node passes
        const bool spec_ok = s->dd_spec && !fused && a.heavy_fraw && !a.uniforms && cd.n_out >= 1 &&
                             cd.n_out <= zxs_dev::kSpecMaxChain && s->dd_identity_map;
        const zxs_sampler::Lineage *lin = spec_ok ? dedup_lineage(s, hc, d, st) : nullptr;
        const bool spec = lin && lin->ok;
        s->time_begin(4, st, t0);
        if (spec) {
            const unsigned long long fm = s->dd_key_mask[hc] & (cd.nf >= 63 ? (1ull << 63) - 1 : (1ull << cd.nf) - 1);
            zxs_dev::DedupSpecArgs sa{};
            sa.seed = a.seed;
            sa.first_shot = a.first_shot;
            sa.shots = a.shots;
            for (int i = 0; i < 10; i++) sa.k0_round[i] = a.k0_round[i];
            sa.ci = cd.ci;
            sa.n_out = cd.n_out;
            sa.main_bits = lin->bits;
            for (uint32_t j = 0; j < cd.n_out; j++) {
                sa.T[j] = lin->T[j];
                sa.tie_lo[j] = lin->tie_lo[j];
                sa.tie_w[j] = lin->tie_w[j];
                sa.out[j] = s->comp_outputs[cd.out_begin + j];
            }
            sa.out32 = a.out32;
            sa.out_ld32 = a.ld32;
            sa.err = d.err;
            sa.active = d.active;
            sa.n_active = d.n_active;
            CK(cudaMemsetAsync(d.n_active, 0, 4, st));
            const unsigned rgrid = unsigned(std::min<uint64_t>((a.shots + 256 * zxs_dev::kSpecG - 1) / (256 * zxs_dev::kSpecG),
                                                               uint64_t(s->sm_count) * std::max(1, s->dd_spec_occ)));
            if (a.fraw_bytes == 4) {
                zxs_dev::dedup_init_spec_kernel<uint32_t><<<rgrid, 256, 0, st>>>(
                    static_cast<const uint32_t *>(a.heavy_fraw), fm, d.slot, d.table[0], sa);
            } else {
                zxs_dev::dedup_init_spec_kernel<unsigned long long><<<rgrid, 256, 0, st>>>(
                    static_cast<const unsigned long long *>(a.heavy_fraw), fm, d.slot, d.table[0], sa);
            }
            CK(cudaGetLastError());
        } else if (a.heavy_fraw) {  // per-shot f words from shot_kernel (identity parameter maps only)
            const unsigned long long fm = s->dd_key_mask[hc] & (cd.nf >= 63 ? (1ull << 63) - 1 : (1ull << cd.nf) - 1);
            const unsigned rgrid =
                unsigned(std::min<uint64_t>((a.shots + 255) / 256, uint64_t(s->sm_count) * std::max(1, s->dd_raw_occ)));
            if (a.fraw_bytes == 4) {
                zxs_dev::dedup_init_raw_kernel<uint32_t><<<rgrid, 256, 0, st>>>(
                    static_cast<const uint32_t *>(a.heavy_fraw), fm, a.shots, ia.key, d.slot, d.table[0]);
            } else {
                zxs_dev::dedup_init_raw_kernel<unsigned long long><<<rgrid, 256, 0, st>>>(
                    static_cast<const unsigned long long *>(a.heavy_fraw), fm, a.shots, ia.key, d.slot, d.table[0]);
            }
            CK(cudaGetLastError());
        } else {
            void *iargs[] = {&ia};
            CK(cudaLaunchKernel(reinterpret_cast<const void *>(&zxs_dev::dedup_init_kernel), dim3(igrid),
                                dim3(zxs_dev::kDedupInitWarps * 32), iargs, 0, st));
        }
        s->time_end(4, st, t0);
        if (fused) {
            for (uint32_t pos = 0; pos <= cd.n_out; pos++) {
                const uint32_t nb = nb_of(pos);
                const unsigned long long *keys = d.table[0].ukeys;
                if (nb) {
                    s->time_begin(4, st, t0);
                    zxs_dev::dedup_expand_kernel<<<unsigned(s->sm_count) * 4, 256, 0, st>>>(
                        d.table[0].ukeys, d.table[0].count, nb, relpos, flimit, d.xkeys);
                    CK(cudaGetLastError());
                    s->time_end(4, st, t0);
                    keys = d.xkeys;
                }
                dedup_eval(s, cd.first_tensor + pos, keys, nullptr, flimit, d.fvals[pos], d.partial, d.partial_bytes, st,
                           d.table[0].count, 1u << nb, flimit);
            }
            zxs_dev::DedupFusedArgs fa{};
            fa.seed = a.seed;
            fa.first_shot = a.first_shot;
            fa.shots = a.shots;
            for (int i = 0; i < 10; i++) fa.k0_round[i] = a.k0_round[i];
            fa.ci = cd.ci;
            fa.n_out = cd.n_out;
            for (uint32_t j = 0; j < cd.n_out; j++) fa.out[j] = s->comp_outputs[cd.out_begin + j];
            fa.relevant = relevant;
            fa.slot = d.slot;
            fa.ids = d.table[0].ids;
            for (uint32_t pos = 0; pos <= cd.n_out; pos++) fa.value[pos] = d.fvals[pos];
            fa.value_cap = flimit;
            fa.out32 = a.out32;
            fa.out_ld32 = a.ld32;
            fa.counts = a.counts ? d.counts : nullptr;
            fa.uniforms = a.uniforms;
            fa.uniforms_ld = a.uniforms_ld;
            fa.upos_base = cd.upos_base;
            fa.err = d.err;
            const unsigned fgrid =
                unsigned(std::min<uint64_t>((a.shots + 256 * ZXS_FUSED_G - 1) / (256 * ZXS_FUSED_G),
                                            uint64_t(s->sm_count) * std::max(1, s->dd_fused_occ)));
            s->time_begin(4, st, t0);
            void *fargs[] = {&fa};
            CK(cudaLaunchKernel(reinterpret_cast<const void *>(&zxs_dev::dedup_fused_ar_kernel), dim3(fgrid), dim3(256),
                                fargs, 0, st));
            s->time_end(4, st, t0);
            clear(d.table[0], 1u << nb_of(cd.n_out), d.max_count + 1);
            continue;
        }
        // ---- node levels (zxs_dedup.cuh): level 0's nodes are the base keys
        const unsigned ngrid = unsigned(s->sm_count) * 4;
        if (cd.n_out == 0) {
            dedup_eval(s, cd.first_tensor, d.table[0].ukeys, d.table[0].uslot, limit, d.value0, d.partial, d.partial_bytes,
                       st, d.table[0].count, 1, d.table[0].mask + 1);
            clear(d.table[0]);
            continue;
        }
        // tensors 0 and 1 on the base keys restricted to what each reads and reduced modulo its
        // null space (dedup_key_restrict_kernel; table 3, kslot in the level-1 node arrays)
        uint32_t *kslot0 = d.nodes[1].kslot;
        for (uint32_t pos = 0; pos < 2; pos++) {
            const uint32_t tj = cd.first_tensor + pos;
            const uint32_t nb = s->dd_null_begin[tj], ne = s->dd_null_begin[tj + 1];
            s->time_begin(4, st, t0);
            zxs_dev::dedup_key_restrict_kernel<<<ngrid, 256, 0, st>>>(d.table[0], s->dd_tread[tj], s->dd_null + nb,
                                                                     (ne - nb) / 2, d.table[3], kslot0);
            CK(cudaGetLastError());
            s->time_end(4, st, t0);
            dedup_eval(s, tj, d.table[3].ukeys, d.table[3].uslot, limit, d.value, d.partial, d.partial_bytes, st,
                       d.table[3].count, 1, d.table[3].mask + 1);
            if (pos == 0) {
                s->time_begin(4, st, t0);
                zxs_dev::dedup_gather_kernel<<<ngrid, 256, 0, st>>>(d.table[0], d.value, kslot0, d.value0);
                CK(cudaGetLastError());
                s->time_end(4, st, t0);
                clear(d.table[3]);
            }
        }
        s->time_begin(4, st, t0);
        auto node_table = [&](uint32_t j) -> const zxs_dev::DedupTable & { return j == 0 ? d.table[0] : d.table[1 + ((j - 1) & 1)]; };
        // a node whose bit is certain gets its only child in the next level's (clear) table here
        zxs_dev::dedup_node_level0_kernel<<<ngrid, 256, 0, st>>>(d.table[0], d.value0, d.value, kslot0, d.nodes[0],
                                                                 node_table(1), cd.n_out > 1);
        CK(cudaGetLastError());
        s->time_end(4, st, t0);
        clear(d.table[3]);
        for (uint32_t j = 0; j < cd.n_out; j++) {
            const zxs_dev::DedupTable &cur = node_table(j);
            const zxs_dev::DedupNodeArrays &na = d.nodes[j & 1];
            if (j > 0) {
                // the bit sampled at position j - 1 enters the key when a later tensor reads it
                const uint32_t p = cd.nf + j - 1;
                const uint32_t bit_pos = (p < 63 && ((s->dd_key_mask[hc] >> p) & 1ull)) ? p : 64u;
                s->time_begin(4, st, t0);
                // the level's key table holds the node keys restricted to what tensor j + 1 reads
                // and reduced to one representative per coset of the forms' null space
                const uint32_t tj = cd.first_tensor + 1 + j;
                const unsigned long long tmask = s->dd_tread[tj];
                const uint32_t nb = s->dd_null_begin[tj], ne = s->dd_null_begin[tj + 1];
                zxs_dev::dedup_node_prep_kernel<<<ngrid, 256, 0, st>>>(cur, d.nodes[(j - 1) & 1], na, bit_pos, tmask,
                                                                      s->dd_null + nb, (ne - nb) / 2, d.table[3]);
                CK(cudaGetLastError());
                s->time_end(4, st, t0);
                dedup_eval(s, cd.first_tensor + 1 + j, d.table[3].ukeys, d.table[3].uslot, limit, d.value, d.partial,
                           d.partial_bytes, st, d.table[3].count, 1, d.table[3].mask + 1);
                s->time_begin(4, st, t0);
                zxs_dev::dedup_node_decide_kernel<<<ngrid, 256, 0, st>>>(cur, d.value, na, node_table(j + 1),
                                                                        j + 1 < cd.n_out);
                CK(cudaGetLastError());
                s->time_end(4, st, t0);
                clear(d.table[3]);
            }
            zxs_dev::DedupNodePassArgs ra{};
            ra.seed = a.seed;
            ra.first_shot = a.first_shot;
            ra.shots = a.shots;
            for (int i = 0; i < 10; i++) ra.k0_round[i] = a.k0_round[i];
            ra.ci = cd.ci;
            ra.j = j;
            ra.out = s->comp_outputs[cd.out_begin + j];
            ra.slot = d.slot;
            ra.cur = cur;
            ra.next = node_table(j + 1);
            ra.insert_next = j + 1 < cd.n_out;
            ra.rec = na.rec;
            ra.out32 = a.out32;
            ra.out_ld32 = a.ld32;
            ra.counts = a.counts ? d.counts : nullptr;
            ra.uniforms = a.uniforms;
            ra.uniforms_ld = a.uniforms_ld;
            ra.upos = cd.upos_base + j;
            ra.err = d.err;
            s->time_begin(4, st, t0);
            void *rargs[] = {&ra};
            const unsigned agrid = unsigned(std::min<uint64_t>(
                (a.shots + 256 * zxs_dev::kNodePassG - 1) / (256 * zxs_dev::kNodePassG),
                uint64_t(s->sm_count) * std::max(1, spec ? s->dd_node_act_occ : s->dd_node_occ)));
            ra.active = spec ? d.active : nullptr;
            ra.n_active = d.n_active;
            ra.main_bit = spec ? (lin->bits >> j) & 1u : 0u;
            const void *pk = spec ? reinterpret_cast<const void *>(&zxs_dev::dedup_node_pass_kernel<true>)
                                  : reinterpret_cast<const void *>(&zxs_dev::dedup_node_pass_kernel<false>);
            CK(cudaLaunchKernel(pk, dim3(agrid), dim3(256),
                                rargs, 0, st));
            s->time_end(4, st, t0);
            clear(cur);
        }
    }
    CK(cudaMemcpyAsync(s->dd_pinned, d.max_count, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (s->dd_pinned[0] > limit || s->dd_pinned[1] > flimit) {
        // more distinct keys at some position than the tables hold: distinct keys grow sublinearly
        // with the batch, so redo the batch as two halves on this path (down to 2^20 shots), and
        // only then synchronously (whose own fallback is the per-shot mono_kernel)
        s->dd_dirty = true;
        s->dd_stats[0] -= 1;
        constexpr uint64_t kMinSplit = uint64_t(1) << 20;
        if (a.shots >= 2 * kMinSplit) {
            const uint64_t h = (a.shots / 2 + 63) & ~uint64_t(63);  // whole 64-shot record words
            zxs_dev::LaunchArgs lo = a, hi = a;
            lo.shots = h;
            hi.first_shot = a.first_shot + h;
            hi.shots = a.shots - h;
            if (hi.out32) hi.out32 = a.out32 + h / 32;
            if (a.uniforms) hi.uniforms = a.uniforms + h;  // [position][uniforms_ld]: same row stride
            if (a.heavy_fraw) hi.heavy_fraw = static_cast<char *>(a.heavy_fraw) + h * a.fraw_bytes;
            hi.heavy_ld32 = a.heavy_ld32;
            if (a.fcols_spare) hi.fcols_spare = a.fcols_spare + h / 32;
            s->dd_stats[1] += 1;
            launch_dedup(s, lo, fcols, fcols_ld32, st);
            launch_dedup(s, hi, fcols ? fcols + h / 32 : nullptr, fcols_ld32, st);
            return;
        }
        if (!fcols) fcols = regen_fcols(s, a, st);
        return launch_dedup_sync(s, a, fcols, fcols_ld32, st);
    }
    zxs_dev::dedup_err_merge_kernel<<<1, 1, 0, st>>>(d.err, s->dev_err);
    CK(cudaGetLastError());
    if (a.counts) {
        s->time_begin(4, st, t0);
        zxs_dev::dedup_add_counts_kernel<<<(nout + 255) / 256, 256, 0, st>>>(d.counts, a.counts, nout);
        CK(cudaGetLastError());
        s->time_end(4, st, t0);
    }
    s->dd_dirty = false;
}

void launch_shots(zxs_sampler *s, zxs_dev::LaunchArgs &a, cudaStream_t st) {
    a.m = s->m;
    a.num_mech = s->info.num_mechanisms;
    a.debug_ar_components = 0xffffffffu;
    a.tab = s->dev_tab;
    if (const char *e = std::getenv("ZXS_DEBUG_AR_COMPONENTS")) a.debug_ar_components = uint32_t(std::atoi(e));
    a.mech_global = s->mech_global;
    a.fast_global = s->fast_global;
    a.ext_begin = s->ext_begin;
    a.ext = s->ext;
    a.err = s->dev_err;
    for (int i = 0; i < 10; i++) a.k0_round[i] = uint32_t(a.seed) + uint32_t(i) * 0x9E3779B9u;
    // One warp tile = 32 * S shots (S/2 u64 output words per output).
    const uint64_t tile_shots = 32ull * s->shots_per_lane;
    a.n_tiles = (a.shots + tile_shots - 1) / tile_shots;
    if (a.n_tiles == 0) return;
    uint64_t cap = uint64_t(s->sm_count) * s->blocks_per_sm;
    unsigned grid = unsigned(std::min(a.n_tiles, cap));
    size_t smem = shot_smem_bytes(s);
    const bool heavy = (s->has_heavy || s->has_mono) && !a.fcols_out && !a.forced;
    if (heavy) {
        a.heavy_ld32 = 2 * ((a.shots + 63) / 64);
        const size_t fc_bytes = (std::max<size_t>(16, size_t(s->m.f_width) * a.heavy_ld32 * 4) + 255) & ~size_t(255);
        const bool raw = s->has_mono && s->dedup && s->dd_async && s->fw_template == 1 && !a.fcols_in && s->dd_identity_map;
        // raw keys: 4 B per shot when f fits 32 bits; the f columns are then not stored at all
        // (no heavy_kernel component reads them; a batch the deduplicated path must redo
        // regenerates them, launch_dedup)
        a.fraw_bytes = s->m.f_width <= 32 ? 4 : 8;
        char *hb = reinterpret_cast<char *>(s->heavy_fcols_get(fc_bytes + (raw ? size_t(a.shots) * a.fraw_bytes : 0)));
        a.heavy_fcols = (raw && !s->has_heavy) ? nullptr : reinterpret_cast<uint32_t *>(hb);
        a.heavy_fraw = raw ? static_cast<void *>(hb + fc_bytes) : nullptr;
        a.fcols_spare = reinterpret_cast<uint32_t *>(hb);
    }
    void *args[] = {&a, s->param_mechs ? static_cast<void *>(s->mech_table.get()) : static_cast<void *>(s->mech_table1.get())};
    cudaEvent_t t0 = nullptr;
    s->time_begin(0, st, t0);
    CK(cudaLaunchKernel(shot_kernel_for(s->fw_template, s->param_mechs, s->shots_per_lane), dim3(grid), dim3(32), args,
                        smem, st));
    s->time_end(0, st, t0);
    if (heavy && s->has_mono && s->dedup) {
        launch_dedup(s, a, a.heavy_fcols, a.heavy_ld32, st);
    } else if (heavy && s->has_mono) {
        s->time_begin(2, st, t0);
        launch_mono(s, a, a.heavy_fcols, a.heavy_ld32, -1, nullptr, 0, st);
        s->time_end(2, st, t0);
    }
    if (heavy && s->has_heavy) {
        s->time_begin(1, st, t0);
        zxs_dev::HeavyArgs h = s->heavy;
        h.seed = a.seed;
        h.first_shot = a.first_shot;
        h.shots = a.shots;
        for (int i = 0; i < 10; i++) h.k0_round[i] = a.k0_round[i];
        h.fcols = a.heavy_fcols;
        h.fcols_ld32 = a.heavy_ld32;
        h.out32 = a.out32;
        h.out_ld32 = a.ld32;
        h.counts = a.counts;
        h.uniforms = a.uniforms;
        h.uniforms_ld = a.uniforms_ld;
        h.err = a.err;
        const uint64_t per_cta = uint64_t(zxs_dev::kHeavyWarps) * 32 * zxs_dev::kHS;
        h.n_cta_tiles = (a.shots + per_cta - 1) / per_cta;
        const unsigned hgrid = unsigned(std::min<uint64_t>(h.n_cta_tiles, uint64_t(s->sm_count) * s->heavy_blocks_per_sm));
        void *hargs[] = {&h};
        CK(cudaLaunchKernel(reinterpret_cast<const void *>(&zxs_dev::heavy_kernel), dim3(hgrid),
                            dim3(zxs_dev::kHeavyWarps * 32), hargs, s->heavy_smem, st));
        s->time_end(1, st, t0);
    }
}

void check_ratio_error(zxs_sampler *s, cudaStream_t st) {
    unsigned long long h[2];
    CK(cudaMemcpyAsync(h, s->dev_err, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h[0]) {
        unsigned long long init[2] = {0, ~0ull};
        CK(cudaMemcpy(s->dev_err, init, sizeof(init), cudaMemcpyHostToDevice));
        // sampler.cpp:86-89
        fail(ZXS_RUNTIME_ERROR, "autoregressive ratio outside [0, 1]: numeric breakdown");
    }
}

void check_mode(const zxs_sampler *s, uint32_t expected) {
    if (expected != s->mode) {  // sampler.cpp:308-309, 316-317
        fail(ZXS_INVALID_ARGUMENT, s->mode == ZXS_MODE_MEASUREMENTS ? "sampler was compiled in measurement mode"
                                                                     : "sampler was compiled in detector mode");
    }
}

// Device-side entry points take the caller's stream as is (NULL is the
// legacy default stream, as everywhere in CUDA); synchronous host entry
// points use the sampler's own stream when given NULL.
cudaStream_t device_stream(void *stream) { return reinterpret_cast<cudaStream_t>(stream); }
cudaStream_t host_stream(zxs_sampler *s, void *stream) {
    return stream ? reinterpret_cast<cudaStream_t>(stream) : s->stream;
}

bool sparse_eligible(const zxs_sampler *s, const zxs_sample_options *opts) {
    const bool force_dense = opts ? opts->force_dense != 0 : false;
    const double threshold = opts ? opts->sparse_threshold : 8.0;
    return !force_dense && s->sparse_structural && s->sparse_expected_flips < threshold;  // sampler.cpp:104-117
}

// The sparse geometric record of shots [0, shots) into device columns
// [num_outputs][words] (sampler.cpp:130-147, 214-255).
void sparse_record_device(zxs_sampler *s, uint64_t seed, uint64_t shots, unsigned long long *cols, cudaStream_t st) {
    if (shots >= (uint64_t(1) << 40)) fail(ZXS_UNSUPPORTED, "sparse path limited to 2^40 shots");
    const uint64_t words = (shots + 63) / 64;
    const uint32_t nout = s->m.num_outputs;
    CK(cudaMemsetAsync(cols, 0, size_t(words) * nout * 8, st));
    // constant part: all-ones words, tail bits included (the sparse branch
    // returns before sample_outputs zeroes tails, sampler.cpp:131-146)
    for (uint32_t o : s->const_one_outputs) CK(cudaMemsetAsync(cols + size_t(o) * words, 0xff, words * 8, st));
    zxs_dev::SparseArgs a;
    a.seed = seed;
    a.shots = shots;
    a.words = words;
    a.num_mech = s->info.num_mechanisms;
    a.log1mp = s->dev_log1mp;
    a.flip_begin = s->dev_flip_begin;
    a.flip_out = s->dev_flip_out;
    a.cols = cols;
    if (a.num_mech) {
        zxs_dev::sparse_kernel<<<a.num_mech, zxs_dev::kSparseThreads, 0, st>>>(a);
        CK(cudaGetLastError());
    }
}


}  // namespace

extern "C" {

const char *zxs_last_error(void) { return g_last_error.c_str(); }
uint32_t zxs_abi_version(void) { return ZXS_ABI_VERSION; }

zxs_status zxs_sampler_create(const zxs_model_desc *desc, int device, zxs_sampler **out) {
    return guarded([&] {
        if (!out) fail(ZXS_INVALID_ARGUMENT, "null output handle");
        *out = nullptr;
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0) fail(ZXS_CUDA_ERROR, "no CUDA device available (the sampler has no CPU fallback)");
        if (device < 0 || device >= n) fail(ZXS_INVALID_ARGUMENT, "device ordinal out of range");
        DeviceGuard g(device);
        auto *s = new zxs_sampler;
        s->device = device;
        try {
            build(s, desc);
        } catch (...) {
            zxs_sampler_destroy(s);
            throw;
        }
        *out = s;
    });
}

void zxs_sampler_destroy(zxs_sampler *s) {
    if (!s) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->copy_stream) cudaStreamSynchronize(s->copy_stream);
    for (int i = 0; i < 2; i++) {
        if (s->ev_done[i]) cudaEventDestroy(s->ev_done[i]);
        if (s->ev_copied[i]) cudaEventDestroy(s->ev_copied[i]);
    }
    if (s->stream) cudaStreamDestroy(s->stream);
    if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
    if (s->dev_model) cudaFree(s->dev_model);
    if (s->dev_err) cudaFree(s->dev_err);
    if (s->scratch) cudaFree(s->scratch);
    if (s->heavy_scratch) cudaFree(s->heavy_scratch);
    if (s->dev_log1mp) cudaFree(s->dev_log1mp);
    if (s->dev_tab) cudaFree(s->dev_tab);
    if (s->dev_flip_begin) cudaFree(s->dev_flip_begin);
    if (s->dev_flip_out) cudaFree(s->dev_flip_out);
    if (s->mono_scratch) cudaFree(s->mono_scratch);
    if (s->dd_buf) cudaFree(s->dd_buf);
    if (s->dd_spec_dev) cudaFree(s->dd_spec_dev);
    if (s->dd_pinned) cudaFreeHost(s->dd_pinned);
    if (s->dd_dev_stats) cudaFree(s->dd_dev_stats);
    for (auto &t : s->timed) {
        cudaEventDestroy(t.second.first);
        cudaEventDestroy(t.second.second);
    }
    if (prev >= 0) cudaSetDevice(prev);
    delete s;
}

zxs_status zxs_sampler_get_info(const zxs_sampler *s, zxs_sampler_info *info) {
    return guarded([&] {
        if (!s || !info) fail(ZXS_INVALID_ARGUMENT, "null argument");
        *info = s->info;
    });
}

// Shots per launch_shots batch on the device-buffer and count entry points:
// per-shot scratch (f columns, f words, dedup keys/slots/marginals) is sized
// by the batch, so a 1e10-shot sweep runs as 2^28-shot batches (a multiple of
// 64: every batch starts on a record word).
constexpr uint64_t kMaxBatchShots = uint64_t(1) << 28;

void launch_shots_chunked(zxs_sampler *s, const zxs_dev::LaunchArgs &tmpl, cudaStream_t st) {
    for (uint64_t done = 0; done < tmpl.shots; done += kMaxBatchShots) {
        zxs_dev::LaunchArgs a = tmpl;
        a.first_shot = tmpl.first_shot + done;
        a.shots = std::min(kMaxBatchShots, tmpl.shots - done);
        if (a.out32) a.out32 = tmpl.out32 + done / 32;  // done is a multiple of 64
        launch_shots(s, a, st);
        CK(cudaGetLastError());
    }
}

zxs_status zxs_sample_device(zxs_sampler *s, uint64_t seed, uint64_t first_shot, uint64_t shots,
                             uint64_t *dev_columns, uint64_t ld_words, uint64_t *dev_counts, void *stream) {
    return guarded([&] {
        if (!s) fail(ZXS_INVALID_ARGUMENT, "null sampler");
        if (dev_columns && ld_words < (shots + 63) / 64) fail(ZXS_INVALID_ARGUMENT, "ld_words < ceil(shots/64)");
        // the sampler's per-shot scratch is shared by every entry point: calls are serialised
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        cudaStream_t st = device_stream(stream);
        if (dev_columns && !s->all_outputs_covered) {
            CK(cudaMemsetAsync(dev_columns, 0, size_t(s->m.num_outputs) * ld_words * 8, st));
        }
        zxs_dev::LaunchArgs a{};
        a.seed = seed;
        a.first_shot = first_shot;
        a.shots = shots;
        a.out32 = reinterpret_cast<uint32_t *>(dev_columns);
        a.ld32 = 2 * ld_words;
        a.counts = reinterpret_cast<unsigned long long *>(dev_counts);
        launch_shots_chunked(s, a, st);
    });
}

zxs_status zxs_count_device(zxs_sampler *s, uint64_t seed, uint64_t first_shot, uint64_t shots,
                            uint64_t *dev_counts, void *stream) {
    if (!dev_counts) {
        g_last_error = "null counts";
        return ZXS_INVALID_ARGUMENT;
    }
    return zxs_sample_device(s, seed, first_shot, shots, nullptr, 0, dev_counts, stream);
}

zxs_status zxs_kernel_timing(zxs_sampler *s, int enable) {
    return guarded([&] {
        if (!s) fail(ZXS_INVALID_ARGUMENT, "null sampler");
        DeviceGuard g(s->device);
        for (auto &t : s->timed) {
            cudaEventDestroy(t.second.first);
            cudaEventDestroy(t.second.second);
        }
        s->timed.clear();
        s->timing = enable != 0;
    });
}

zxs_status zxs_kernel_times(zxs_sampler *s, double *ms, uint64_t *launches) {
    return zxs_kernel_times_n(s, ms, launches, 3);
}

zxs_status zxs_kernel_times_n(zxs_sampler *s, double *ms, uint64_t *launches, uint32_t n) {
    return guarded([&] {
        if (!s || (n && (!ms || !launches))) fail(ZXS_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(s->device);
        for (uint32_t i = 0; i < n; i++) {
            ms[i] = 0.0;
            launches[i] = 0;
        }
        for (auto &t : s->timed) {
            if (uint32_t(t.first) >= n) continue;
            CK(cudaEventSynchronize(t.second.second));
            float e = 0.f;
            CK(cudaEventElapsedTime(&e, t.second.first, t.second.second));
            ms[t.first] += e;
            launches[t.first]++;
        }
    });
}

zxs_status zxs_dedup_stats(zxs_sampler *s, int reset, uint64_t *out) {
    return guarded([&] {
        if (!s || !out) fail(ZXS_INVALID_ARGUMENT, "null argument");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        unsigned long long dev[2] = {0, 0};
        if (s->dd_dev_stats) {
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(dev, s->dd_dev_stats, 16, cudaMemcpyDeviceToHost));
        }
        for (int i = 0; i < 5; i++) out[i] = s->dd_stats[i];
        out[2] += dev[0];
        out[3] += dev[1];
        out[5] = s->dedup ? 1 : 0;
        if (reset) {
            std::memset(s->dd_stats, 0, sizeof(s->dd_stats));
            if (s->dd_dev_stats) CK(cudaMemset(s->dd_dev_stats, 0, 16));
        }
    });
}

zxs_status zxs_tie_count(zxs_sampler *s, int reset, uint64_t *out) {
    return guarded([&] {
        if (!s || !out) fail(ZXS_INVALID_ARGUMENT, "null argument");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        CK(cudaDeviceSynchronize());
        unsigned long long t = 0;
        CK(cudaMemcpy(&t, s->dev_err + 2, 8, cudaMemcpyDeviceToHost));
        *out = t;
        if (reset) CK(cudaMemset(s->dev_err + 2, 0, 8));
    });
}

zxs_status zxs_sparse_eligible(const zxs_sampler *s, const zxs_sample_options *opts, int *eligible) {
    return guarded([&] {
        if (!s || !eligible) fail(ZXS_INVALID_ARGUMENT, "null argument");
        *eligible = sparse_eligible(s, opts) ? 1 : 0;
    });
}

zxs_status zxs_sample_opts(zxs_sampler *s, uint32_t expected_mode, uint64_t seed, uint64_t shots,
                           const zxs_sample_options *opts, uint64_t *host_columns, void *stream) {
    if (!s || !sparse_eligible(s, opts)) return zxs_sample(s, expected_mode, seed, 0, shots, host_columns, stream);
    return guarded([&] {
        check_mode(s, expected_mode);
        if (shots == 0) return;
        if (!host_columns) fail(ZXS_INVALID_ARGUMENT, "null output");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        cudaStream_t st = host_stream(s, stream);
        const uint64_t words = (shots + 63) / 64;
        const uint32_t nout = s->m.num_outputs;
        auto *cols = reinterpret_cast<unsigned long long *>(
            s->scratch_get(size_t(words) * std::max<uint32_t>(nout, 1) * 8));
        sparse_record_device(s, seed, shots, cols, st);
        CK(cudaMemcpyAsync(host_columns, cols, size_t(words) * nout * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

zxs_status zxs_check_errors(zxs_sampler *s, void *stream) {
    return guarded([&] {
        if (!s) fail(ZXS_INVALID_ARGUMENT, "null sampler");
        DeviceGuard g(s->device);
        check_ratio_error(s, device_stream(stream));
    });
}

zxs_status zxs_count(zxs_sampler *s, uint64_t seed, uint64_t first_shot, uint64_t shots, uint64_t *host_counts,
                     void *stream) {
    return guarded([&] {
        if (!s || !host_counts) fail(ZXS_INVALID_ARGUMENT, "null argument");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        cudaStream_t st = host_stream(s, stream);
        size_t bytes = size_t(s->m.num_outputs) * 8;
        auto *dc = reinterpret_cast<unsigned long long *>(s->scratch_get(std::max<size_t>(bytes, 8)));
        CK(cudaMemsetAsync(dc, 0, bytes, st));
        zxs_dev::LaunchArgs a{};
        a.seed = seed;
        a.first_shot = first_shot;
        a.shots = shots;
        a.counts = dc;
        launch_shots_chunked(s, a, st);
        CK(cudaMemcpyAsync(host_counts, dc, bytes, cudaMemcpyDeviceToHost, st));
        check_ratio_error(s, st);
    });
}

// Host-buffer sampling: chunks of shots are sampled into two device buffers
// in turn; each chunk's columns are copied into the caller's column-major
// record on a second stream while the next chunk is sampled.
zxs_status zxs_sample(zxs_sampler *s, uint32_t expected_mode, uint64_t seed, uint64_t first_shot, uint64_t shots,
                      uint64_t *host_columns, void *stream) {
    return guarded([&] {
        if (!s) fail(ZXS_INVALID_ARGUMENT, "null sampler");
        check_mode(s, expected_mode);
        if (shots == 0) return;
        if (!host_columns) fail(ZXS_INVALID_ARGUMENT, "null output");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        cudaStream_t st = host_stream(s, stream);
        const uint64_t words = (shots + 63) / 64;
        const uint32_t nout = s->m.num_outputs;
        if (nout == 0) {
            check_ratio_error(s, st);
            return;
        }
        // chunk: multiple of 64 shots, ~64 MiB of output per buffer (copies overlap the next chunk);
        // on the deduplicated path, whose per-batch contraction amortises, up to 2^28 shots while
        // a buffer stays within 1 GiB
        uint64_t chunk_words = std::max<uint64_t>(1, (uint64_t(64) << 20) / (8ull * nout));
        if (s->has_mono && s->dedup) {
            chunk_words = std::max<uint64_t>(chunk_words, std::min<uint64_t>(kMaxBatchShots / 64, (uint64_t(1024) << 20) / (8ull * nout)));
        }
        chunk_words = std::min(chunk_words, words);
        const size_t buf_bytes = size_t(chunk_words) * nout * 8;
        char *scratch = s->scratch_get(2 * buf_bytes);
        uint64_t nchunks = (words + chunk_words - 1) / chunk_words;
        for (uint64_t c = 0; c < nchunks; c++) {
            int bi = int(c & 1);
            uint64_t w0 = c * chunk_words;
            uint64_t cw = std::min(chunk_words, words - w0);
            uint64_t cshots = std::min<uint64_t>(cw * 64, shots - w0 * 64);
            auto *buf = reinterpret_cast<uint64_t *>(scratch + bi * buf_bytes);
            if (c >= 2) CK(cudaStreamWaitEvent(st, s->ev_copied[bi], 0));
            if (!s->all_outputs_covered) CK(cudaMemsetAsync(buf, 0, size_t(cw) * nout * 8, st));
            zxs_dev::LaunchArgs a{};
            a.seed = seed;
            a.first_shot = first_shot + w0 * 64;
            a.shots = cshots;
            a.out32 = reinterpret_cast<uint32_t *>(buf);
            a.ld32 = 2 * cw;
            launch_shots(s, a, st);
            CK(cudaGetLastError());
            CK(cudaEventRecord(s->ev_done[bi], st));
            CK(cudaStreamWaitEvent(s->copy_stream, s->ev_done[bi], 0));
            CK(cudaMemcpy2DAsync(host_columns + w0, words * 8, buf, cw * 8, cw * 8, nout, cudaMemcpyDeviceToHost,
                                 s->copy_stream));
            CK(cudaEventRecord(s->ev_copied[bi], s->copy_stream));
        }
        CK(cudaStreamSynchronize(s->copy_stream));
        check_ratio_error(s, st);
    });
}

// ---------------------------------------------------------------- encode_shots
namespace {
// encode.cpp:23-25: the encoded output range, clamped to the record width
uint32_t encode_width(uint32_t num_outputs, uint32_t first_output, uint32_t output_count) {
    if (first_output > num_outputs) fail(ZXS_INVALID_ARGUMENT, "first_output beyond the record width");
    const uint32_t last = std::min(num_outputs, first_output + std::min(output_count, num_outputs - first_output));
    return last - first_output;
}

uint64_t encoded_row_bytes(uint32_t width, uint32_t format) {
    if (format > 1) fail(ZXS_INVALID_ARGUMENT, "unknown shot format");
    return format == ZXS_FORMAT_B8 ? (width + 7) / 8 : uint64_t(width) + 1;
}

void launch_encode(const uint32_t *cols, uint64_t ld32, uint32_t first_output, uint32_t width, uint64_t shots,
                   uint32_t format, uint8_t *dev_out, cudaStream_t st) {
    if (shots == 0) return;
    zxs_dev::EncodeArgs e;
    e.cols = cols;
    e.ld32 = ld32;
    e.first_output = first_output;
    e.width = width;
    e.format = format;
    e.shots = shots;
    e.out = dev_out;
    e.row_bytes = uint32_t(encoded_row_bytes(width, format));
    if (e.row_bytes == 0) return;
    e.smem_per_warp = (32 * e.row_bytes + 15) & ~15u;
    const size_t smem = size_t(zxs_dev::kEncWarps) * e.smem_per_warp;
    if (smem > 200 * 1024) fail(ZXS_UNSUPPORTED, "record too wide for the device encoder");
    if (smem > 48 * 1024) {
        CK(cudaFuncSetAttribute(reinterpret_cast<const void *>(&zxs_dev::encode_kernel),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    }
    int dev = 0, sms = 148;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const uint64_t nwords = (shots + 31) / 32;
    const unsigned grid = unsigned(std::min<uint64_t>((nwords + zxs_dev::kEncWarps - 1) / zxs_dev::kEncWarps,
                                                      uint64_t(sms) * 16));
    zxs_dev::encode_kernel<<<grid, zxs_dev::kEncWarps * 32, smem, st>>>(e);
    CK(cudaGetLastError());
}
}  // namespace

uint64_t zxs_encoded_bytes(uint32_t num_outputs, uint64_t shots, uint32_t first_output, uint32_t output_count,
                           uint32_t format) {
    if (first_output > num_outputs || format > 1) return 0;
    const uint32_t last = std::min(num_outputs, first_output + std::min(output_count, num_outputs - first_output));
    const uint32_t width = last - first_output;
    return shots * (format == ZXS_FORMAT_B8 ? (uint64_t(width) + 7) / 8 : uint64_t(width) + 1);
}

zxs_status zxs_encode_shots_device(const uint64_t *dev_columns, uint64_t ld_words, uint32_t num_outputs,
                                   uint64_t shots, uint32_t first_output, uint32_t output_count, uint32_t format,
                                   uint8_t *dev_out, void *stream) {
    return guarded([&] {
        const uint32_t width = encode_width(num_outputs, first_output, output_count);
        encoded_row_bytes(width, format);
        if (shots == 0 || width == 0 && format == ZXS_FORMAT_B8) return;
        if (!dev_columns || !dev_out) fail(ZXS_INVALID_ARGUMENT, "null argument");
        if (ld_words < (shots + 63) / 64) fail(ZXS_INVALID_ARGUMENT, "ld_words < ceil(shots/64)");
        launch_encode(reinterpret_cast<const uint32_t *>(dev_columns), 2 * ld_words, first_output, width, shots,
                      format, dev_out, device_stream(stream));
    });
}

// sample_detectors / sample_measurements followed by encode_shots, fused:
// chunks are sampled into device columns, encoded on the device, and the
// encoded bytes copied to the host on a second stream while the next chunk
// is sampled. (zxsim.cpp:142-163: write_output(encode_shots(sample_*(...))).)
zxs_status zxs_sample_encoded(zxs_sampler *s, uint32_t expected_mode, uint64_t seed, uint64_t first_shot,
                              uint64_t shots, const zxs_sample_options *opts, uint32_t format, uint32_t first_output,
                              uint32_t output_count, uint8_t *host_out, void *stream) {
    return guarded([&] {
        if (!s) fail(ZXS_INVALID_ARGUMENT, "null sampler");
        check_mode(s, expected_mode);
        const uint32_t nout = s->m.num_outputs;
        const uint32_t width = encode_width(nout, first_output, output_count);
        const uint64_t rb = encoded_row_bytes(width, format);
        if (shots == 0 || rb == 0) return;
        if (!host_out) fail(ZXS_INVALID_ARGUMENT, "null output");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        cudaStream_t st = host_stream(s, stream);
        if (first_shot == 0 && sparse_eligible(s, opts)) {  // the reference's sparse record, encoded on device
            const uint64_t words = (shots + 63) / 64;
            auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
            const size_t cbytes = al(size_t(words) * std::max<uint32_t>(nout, 1) * 8);
            char *base = s->scratch_get(cbytes + al(size_t(shots * rb)));
            auto *cols = reinterpret_cast<unsigned long long *>(base);
            sparse_record_device(s, seed, shots, cols, st);
            launch_encode(reinterpret_cast<const uint32_t *>(cols), 2 * words, first_output, width, shots, format,
                          reinterpret_cast<uint8_t *>(base + cbytes), st);
            CK(cudaMemcpyAsync(host_out, base + cbytes, size_t(shots * rb), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            return;
        }
        // chunk: multiple of 64 shots, ~64 MiB of encoded output per buffer
        uint64_t chunk = std::max<uint64_t>(64, ((uint64_t(64) << 20) / rb) & ~uint64_t(63));
        chunk = std::min<uint64_t>(chunk, (shots + 63) & ~uint64_t(63));
        const uint64_t cw = chunk / 64;
        auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
        const size_t col_bytes = al(size_t(cw) * std::max<uint32_t>(nout, 1) * 8), enc_bytes = al(size_t(chunk * rb));
        char *scratch = s->scratch_get(2 * (col_bytes + enc_bytes));
        const uint64_t nchunks = (shots + chunk - 1) / chunk;
        for (uint64_t c = 0; c < nchunks; c++) {
            const int bi = int(c & 1);
            const uint64_t s0 = c * chunk, cs = std::min(chunk, shots - s0);
            auto *cols = reinterpret_cast<uint64_t *>(scratch + bi * (col_bytes + enc_bytes));
            auto *enc = reinterpret_cast<uint8_t *>(scratch + bi * (col_bytes + enc_bytes) + col_bytes);
            if (c >= 2) CK(cudaStreamWaitEvent(st, s->ev_copied[bi], 0));
            if (!s->all_outputs_covered) CK(cudaMemsetAsync(cols, 0, size_t(cw) * nout * 8, st));
            zxs_dev::LaunchArgs a{};
            a.seed = seed;
            a.first_shot = first_shot + s0;
            a.shots = cs;
            a.out32 = reinterpret_cast<uint32_t *>(cols);
            a.ld32 = 2 * cw;
            launch_shots(s, a, st);
            CK(cudaGetLastError());
            launch_encode(reinterpret_cast<const uint32_t *>(cols), 2 * cw, first_output, width, cs, format, enc, st);
            CK(cudaEventRecord(s->ev_done[bi], st));
            CK(cudaStreamWaitEvent(s->copy_stream, s->ev_done[bi], 0));
            CK(cudaMemcpyAsync(host_out + s0 * rb, enc, size_t(cs * rb), cudaMemcpyDeviceToHost, s->copy_stream));
            CK(cudaEventRecord(s->ev_copied[bi], s->copy_stream));
        }
        CK(cudaStreamSynchronize(s->copy_stream));
        check_ratio_error(s, st);
    });
}

zxs_status zxs_sample_error_batch(zxs_sampler *s, uint64_t seed, uint64_t first_shot, uint64_t shots,
                                  uint64_t *host_fcols) {
    return guarded([&] {
        if (!s) fail(ZXS_INVALID_ARGUMENT, "null sampler");
        if (shots == 0 || s->m.f_width == 0) return;
        if (!host_fcols) fail(ZXS_INVALID_ARGUMENT, "null output");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        cudaStream_t st = s->stream;
        const uint64_t words = (shots + 63) / 64;
        size_t bytes = size_t(words) * s->m.f_width * 8;
        auto *buf = reinterpret_cast<uint32_t *>(s->scratch_get(bytes));
        zxs_dev::LaunchArgs a{};
        a.seed = seed;
        a.first_shot = first_shot;
        a.shots = shots;
        a.fcols_out = buf;
        a.fcols_ld32 = 2 * words;
        launch_shots(s, a, st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(host_fcols, buf, bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

zxs_status zxs_sample_given_f(zxs_sampler *s, uint64_t seed, uint64_t first_shot, uint64_t shots,
                              const uint64_t *host_fcols, const double *host_uniforms, uint64_t *host_columns) {
    return guarded([&] {
        if (!s) fail(ZXS_INVALID_ARGUMENT, "null sampler");
        if (shots == 0) return;
        if (!host_columns || (!host_fcols && s->m.f_width)) fail(ZXS_INVALID_ARGUMENT, "null argument");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        cudaStream_t st = s->stream;
        const uint64_t words = (shots + 63) / 64;
        const uint32_t nout = s->m.num_outputs;
        size_t fbytes = size_t(words) * s->m.f_width * 8;
        size_t obytes = size_t(words) * nout * 8;
        size_t npos = s->comp_outputs.size();
        size_t ubytes = host_uniforms ? npos * shots * 8 : 0;
        auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
        char *base = s->scratch_get(al(fbytes) + al(obytes) + al(ubytes) + 256);
        auto *df = reinterpret_cast<uint32_t *>(base);
        auto *dout = reinterpret_cast<uint32_t *>(base + al(fbytes));
        auto *du = reinterpret_cast<double *>(base + al(fbytes) + al(obytes));
        if (fbytes) CK(cudaMemcpyAsync(df, host_fcols, fbytes, cudaMemcpyHostToDevice, st));
        if (ubytes) CK(cudaMemcpyAsync(du, host_uniforms, ubytes, cudaMemcpyHostToDevice, st));
        if (obytes) CK(cudaMemsetAsync(dout, 0, obytes, st));
        zxs_dev::LaunchArgs a{};
        a.seed = seed;
        a.first_shot = first_shot;
        a.shots = shots;
        a.fcols_in = df;
        a.fcols_ld32 = 2 * words;
        a.uniforms = host_uniforms ? du : nullptr;
        a.uniforms_ld = shots;
        a.out32 = dout;
        a.ld32 = 2 * words;
        launch_shots(s, a, st);
        CK(cudaGetLastError());
        if (obytes) CK(cudaMemcpyAsync(host_columns, dout, obytes, cudaMemcpyDeviceToHost, st));
        check_ratio_error(s, st);
    });
}

namespace {
void eval_on_device(zxs_sampler *s, uint32_t tensor, const uint64_t *host_params, uint32_t param_cols,
                    uint64_t shots, double *host_values, double *max_imag, double *host_imag = nullptr) {
    const uint64_t words = (shots + 63) / 64;
    cudaStream_t st = s->stream;
    size_t pbytes = size_t(words) * param_cols * 8;
    size_t vbytes = size_t(shots) * 8;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    char *base = s->scratch_get(al(pbytes) + 2 * al(vbytes) + 256);
    auto *dp = reinterpret_cast<uint32_t *>(base);
    auto *dv = reinterpret_cast<double *>(base + al(pbytes));
    auto *dmi = reinterpret_cast<unsigned long long *>(base + al(pbytes) + al(vbytes));
    auto *dimag = reinterpret_cast<double *>(base + al(pbytes) + al(vbytes) + 256);
    if (pbytes) CK(cudaMemcpyAsync(dp, host_params, pbytes, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(dmi, 0, 8, st));
    uint32_t col_stride = std::max<uint32_t>(4, (param_cols + 3) & ~3u);
    uint64_t n_tiles = words;
    unsigned grid = unsigned(std::min<uint64_t>((n_tiles + 7) / 8, uint64_t(s->sm_count) * 8));
    size_t smem = size_t(8) * zxs_dev::kS * col_stride * 4;
    if (smem > 48 * 1024) {
        CK(cudaFuncSetAttribute(reinterpret_cast<const void *>(&zxs_dev::eval_kernel),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    }
    zxs_dev::eval_kernel<<<grid, kThreads, smem, st>>>(s->m, tensor, dp, 2 * words, param_cols, col_stride, shots,
                                                       n_tiles, dv, dmi, host_imag ? dimag : nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(host_values, dv, vbytes, cudaMemcpyDeviceToHost, st));
    if (host_imag) CK(cudaMemcpyAsync(host_imag, dimag, vbytes, cudaMemcpyDeviceToHost, st));
    unsigned long long mib = 0;
    CK(cudaMemcpyAsync(&mib, dmi, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (max_imag) std::memcpy(max_imag, &mib, 8);
}
}  // namespace

zxs_status zxs_eval_batch(zxs_sampler *s, uint32_t component, uint32_t chain_pos, const uint64_t *host_params,
                          uint32_t param_cols, uint64_t shots, double *host_values, double *max_imag_ratio) {
    return guarded([&] {
        if (!s) fail(ZXS_INVALID_ARGUMENT, "null sampler");
        if (component >= s->comp_out_begin.size() - 1) fail(ZXS_INVALID_ARGUMENT, "component out of range");
        uint32_t n = s->comp_out_begin[component + 1] - s->comp_out_begin[component];
        if (chain_pos > n) fail(ZXS_INVALID_ARGUMENT, "chain position out of range");
        uint32_t t = s->comp_tensor_begin[component] + chain_pos;
        if (param_cols < s->tensor_width[t]) fail(ZXS_INVALID_ARGUMENT, "eval_batch: parameter width mismatch");
        if (max_imag_ratio) *max_imag_ratio = 0.0;
        if (shots == 0) return;
        if (!host_params || !host_values) fail(ZXS_INVALID_ARGUMENT, "null argument");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        eval_on_device(s, t, host_params, param_cols, shots, host_values, max_imag_ratio);
    });
}

zxs_status zxs_eval_batch_mono(zxs_sampler *s, uint32_t component, uint32_t chain_pos, const uint64_t *host_params,
                               uint32_t param_cols, uint64_t shots, double *host_values) {
    return guarded([&] {
        if (!s) fail(ZXS_INVALID_ARGUMENT, "null sampler");
        if (component >= s->comp_out_begin.size() - 1) fail(ZXS_INVALID_ARGUMENT, "component out of range");
        uint32_t n = s->comp_out_begin[component + 1] - s->comp_out_begin[component];
        if (chain_pos > n) fail(ZXS_INVALID_ARGUMENT, "chain position out of range");
        uint32_t t = s->comp_tensor_begin[component] + chain_pos;
        if (param_cols < s->tensor_width[t]) fail(ZXS_INVALID_ARGUMENT, "eval_batch: parameter width mismatch");
        auto it = s->mono_tensor.find(t);
        if (it == s->mono_tensor.end()) fail(ZXS_UNSUPPORTED, "component is not on the monomial path");
        if (param_cols > 255) fail(ZXS_UNSUPPORTED, "too many parameter columns for the monomial path");
        if (shots == 0) return;
        if (!host_params || !host_values) fail(ZXS_INVALID_ARGUMENT, "null argument");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        cudaStream_t st = s->stream;
        const uint64_t words = (shots + 63) / 64;
        size_t pbytes = size_t(words) * param_cols * 8;
        size_t vbytes = size_t(shots) * 8;
        auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
        char *base = s->scratch_get(al(pbytes) + al(vbytes) + 256);
        auto *dp = reinterpret_cast<uint32_t *>(base);
        auto *dv = reinterpret_cast<double *>(base + al(pbytes));
        CK(cudaMemcpyAsync(dp, host_params, pbytes, cudaMemcpyHostToDevice, st));
        zxs_dev::LaunchArgs a{};
        a.shots = shots;
        launch_mono(s, a, dp, 2 * words, int(it->second), dv, param_cols, st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(host_values, dv, vbytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

// Compile-time health check (SURVEY finding 3): the reference records
// max |Im P| / |P| per shot (phase_terms.cpp:134-141) but never checks it.
// Here every chain tensor of every component is evaluated with the exact
// kernel on `samples` uniformly random parameter vectors; out[c] = the
// component's largest max|Im P| / max|Re P| over its tensors (relative to the
// tensor's scale, so rounding noise on vanishing P does not register).
zxs_status zxs_imag_health(zxs_sampler *s, uint64_t samples, uint64_t seed, double *out) {
    return guarded([&] {
        if (!s || !out) fail(ZXS_INVALID_ARGUMENT, "null argument");
        if (samples == 0) fail(ZXS_INVALID_ARGUMENT, "samples must be positive");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        uint64_t x = seed ^ 0x9E3779B97F4A7C15ull;
        auto next = [&]() {  // splitmix64
            uint64_t z = (x += 0x9E3779B97F4A7C15ull);
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            return z ^ (z >> 31);
        };
        const uint64_t words = (samples + 63) / 64;
        std::vector<double> vals(samples);
        for (size_t c = 0; c + 1 < s->comp_out_begin.size(); c++) {
            double worst = 0.0;
            for (uint32_t t = s->comp_tensor_begin[c]; t < s->comp_tensor_begin[c + 1]; t++) {
                const uint32_t W = std::max<uint32_t>(1, s->tensor_width[t]);
                std::vector<uint64_t> params(size_t(W) * words);
                for (auto &w : params) w = next();
                if (samples & 63) {
                    for (uint32_t p = 0; p < W; p++) params[p * words + words - 1] &= (uint64_t(1) << (samples & 63)) - 1;
                }
                std::vector<double> ims(samples);
                eval_on_device(s, t, params.data(), W, samples, vals.data(), nullptr, ims.data());
                double pmax = 0.0, imax = 0.0;
                for (uint64_t i = 0; i < samples; i++) {
                    pmax = std::max(pmax, std::fabs(vals[i]));
                    imax = std::max(imax, std::fabs(ims[i]));
                }
                if (pmax > 0) worst = std::max(worst, imax / pmax);
            }
            out[c] = worst;
        }
    });
}

// probability_of_at (sampler.cpp:360-368) -> outcome_probability_given
// (sampler.cpp:324-356), every eval on the device.
zxs_status zxs_probability_of_at(zxs_sampler *s, const uint8_t *outcome, uint32_t n_outcome,
                                 const uint8_t *f_assignment, uint32_t n_f, double *out) {
    return guarded([&] {
        if (!s || !out || (!outcome && n_outcome) || (!f_assignment && n_f)) fail(ZXS_INVALID_ARGUMENT, "null argument");
        if (n_outcome != s->m.num_outputs) fail(ZXS_INVALID_ARGUMENT, "outcome length must match the output count");
        if (n_f != s->m.f_width) fail(ZXS_INVALID_ARGUMENT, "f assignment length must match f_width");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        // f = f_assignment ^ base_offset
        std::vector<uint64_t> base(s->fw_template);
        CK(cudaMemcpy(base.data(), s->m.base_offset, base.size() * 8, cudaMemcpyDeviceToHost));
        std::vector<uint8_t> f(n_f);
        for (uint32_t i = 0; i < n_f; i++) f[i] = (f_assignment[i] ^ uint8_t((base[i >> 6] >> (i & 63)) & 1)) & 1;
        // direct outputs
        std::vector<uint32_t> dbb(s->m.num_direct + 1), dbits;
        CK(cudaMemcpy(dbb.data(), s->m.direct_bit_begin, dbb.size() * 4, cudaMemcpyDeviceToHost));
        dbits.resize(std::max<uint32_t>(1, dbb.back()));
        CK(cudaMemcpy(dbits.data(), s->m.direct_bits, dbits.size() * 4, cudaMemcpyDeviceToHost));
        for (uint32_t d = 0; d < s->m.num_direct; d++) {
            uint32_t od = s->direct_out[d];
            bool bit = (od >> 31) != 0;
            for (uint32_t b = dbb[d]; b < dbb[d + 1]; b++) bit ^= f[dbits[b]] != 0;
            if (bit != (outcome[od & 0x7fffffffu] != 0)) {
                *out = 0.0;
                return;
            }
        }
        double p = 1.0;
        for (size_t c = 0; c + 1 < s->comp_out_begin.size(); c++) {
            uint32_t n = s->comp_out_begin[c + 1] - s->comp_out_begin[c];
            uint32_t cols = s->m.f_width + n;
            std::vector<uint64_t> params(std::max<uint32_t>(cols, 1), 0);
            for (uint32_t i = 0; i < s->m.f_width; i++) params[i] = f[i];
            double norm = 0.0;
            eval_on_device(s, s->comp_tensor_begin[c], params.data(), cols, 1, &norm, nullptr);
            if (!(norm > 0.0)) fail(ZXS_RUNTIME_ERROR, "component normalization is not positive");
            double prev = norm;
            for (uint32_t pos = 0; pos < n; pos++) {
                double p0 = 0.0;
                eval_on_device(s, s->comp_tensor_begin[c] + 1 + pos, params.data(), cols, 1, &p0, nullptr);
                bool bit = outcome[s->comp_outputs[s->comp_out_begin[c] + pos]] != 0;
                prev = bit ? prev - p0 : p0;
                params[s->m.f_width + pos] = bit ? 1 : 0;
            }
            p *= prev / norm;
        }
        *out = p;
    });
}

// probability_of (sampler.cpp:370-429): the enumeration over mechanism
// outcomes runs on the host in the reference's DFS order (weights formed by
// the same left-to-right products, zero-weight subtrees pruned), every leaf's
// outcome_probability_given is evaluated on the device as one "shot" with its
// f injected and the outcome bits forced (shot_kernel probability mode), and
// the leaves are Kahan-summed in DFS order like the reference.
zxs_status zxs_probability_of(zxs_sampler *s, const uint8_t *outcome, uint32_t n_outcome, double *out) {
    return guarded([&] {
        if (!s || !out || (!outcome && n_outcome)) fail(ZXS_INVALID_ARGUMENT, "null argument");
        if (n_outcome != s->m.num_outputs) fail(ZXS_INVALID_ARGUMENT, "outcome length must match the output count");
        double entropy_bits = 0;
        for (const auto &m : s->host_mechs) entropy_bits += m.joint ? std::log2(double(m.table.size())) : 1.0;
        if (entropy_bits > 20.0) fail(ZXS_INVALID_ARGUMENT, "noise entropy guard exceeded for exact marginalization");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard g(s->device);
        const size_t FW = s->host_base.size();
        // ---- leaves in DFS order
        std::vector<double> weights;
        std::vector<uint64_t> fs;  // [leaf][FW]
        std::vector<uint64_t> f = s->host_base;
        const size_t M = s->host_mechs.size();
        std::function<void(size_t, double)> walk = [&](size_t idx, double weight) {
            if (weight == 0.0) return;
            if (idx == M) {
                weights.push_back(weight);
                fs.insert(fs.end(), f.begin(), f.end());
                return;
            }
            const auto &m = s->host_mechs[idx];
            auto flip = [&](const std::vector<uint64_t> &v) {
                for (size_t w = 0; w < FW; w++) f[w] ^= v[w];
            };
            if (!m.joint) {
                walk(idx + 1, weight * (1.0 - m.p));
                flip(m.vecs[0]);
                walk(idx + 1, weight * m.p);
                flip(m.vecs[0]);
                return;
            }
            for (size_t o = 0; o < m.table.size(); o++) {
                if (m.table[o] == 0.0) continue;
                for (size_t b = 0; b < m.vecs.size(); b++) {
                    if ((o >> b) & 1) flip(m.vecs[b]);
                }
                walk(idx + 1, weight * m.table[o]);
                for (size_t b = 0; b < m.vecs.size(); b++) {
                    if ((o >> b) & 1) flip(m.vecs[b]);
                }
            }
        };
        walk(0, 1.0);
        const uint64_t n = weights.size();
        if (n == 0) {
            *out = 0.0;
            return;
        }
        // ---- f-columns of the leaves: [f_width][ceil(n/64)] u64
        const uint64_t words = (n + 63) / 64;
        const uint32_t fwid = s->m.f_width;
        std::vector<uint64_t> cols(std::max<size_t>(1, size_t(fwid) * words), 0);
        for (uint64_t l = 0; l < n; l++) {
            for (uint32_t b = 0; b < fwid; b++) {
                if ((fs[l * FW + (b >> 6)] >> (b & 63)) & 1) cols[b * words + (l >> 6)] |= uint64_t(1) << (l & 63);
            }
        }
        cudaStream_t st = s->stream;
        auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
        const size_t fbytes = size_t(fwid) * words * 8, pbytes = size_t(n) * 8, obytes = std::max<size_t>(n_outcome, 1);
        char *base = s->scratch_get(al(fbytes) + al(pbytes) + al(obytes) + 256);
        auto *df = reinterpret_cast<uint32_t *>(base);
        auto *dp = reinterpret_cast<double *>(base + al(fbytes));
        auto *dout = reinterpret_cast<uint8_t *>(base + al(fbytes) + al(pbytes));
        if (fbytes) CK(cudaMemcpyAsync(df, cols.data(), fbytes, cudaMemcpyHostToDevice, st));
        std::vector<uint8_t> oc(obytes, 0);
        for (uint32_t i = 0; i < n_outcome; i++) oc[i] = outcome[i] ? 1 : 0;
        CK(cudaMemcpyAsync(dout, oc.data(), obytes, cudaMemcpyHostToDevice, st));
        zxs_dev::LaunchArgs a{};
        a.shots = n;
        a.fcols_in = df;
        a.fcols_ld32 = 2 * words;
        a.forced = dout;
        a.prob = dp;
        launch_shots(s, a, st);
        CK(cudaGetLastError());
        std::vector<double> pg(n);
        CK(cudaMemcpyAsync(pg.data(), dp, pbytes, cudaMemcpyDeviceToHost, st));
        unsigned long long h[2];
        CK(cudaMemcpyAsync(h, s->dev_err, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h[0]) {
            unsigned long long init[2] = {0, ~0ull};
            CK(cudaMemcpy(s->dev_err, init, sizeof(init), cudaMemcpyHostToDevice));
            fail(ZXS_RUNTIME_ERROR, "component normalization is not positive");  // sampler.cpp:343-345
        }
        // ---- Kahan-compensated sum in DFS order (sampler.cpp:388-395)
        double sum = 0.0, carry = 0.0;
        for (uint64_t l = 0; l < n; l++) {
            const double term = weights[l] * pg[l];
            const double y = term - carry;
            const double t = sum + y;
            carry = (t - sum) - y;
            sum = t;
        }
        *out = sum;
    });
}

zxs_status zxs_debug_heavy_layout(const zxs_model_desc *desc, uint64_t min_factors, uint32_t *out, uint64_t cap,
                                  uint64_t *needed) {
    return guarded([&] {
        if (!desc || !needed) fail(ZXS_INVALID_ARGUMENT, "null argument");
        uint32_t max_chain = 0;
        for (uint32_t c = 0; c < desc->num_components; c++) {
            max_chain = std::max(max_chain, desc->comp_out_begin[c + 1] - desc->comp_out_begin[c]);
        }
        HeavyHost H = encode_heavy(desc, max_chain, min_factors);
        std::vector<uint32_t> blob = {uint32_t(H.words.size()), uint32_t(H.chunks.size()),
                                      uint32_t(H.tensor_chunk_begin.size()), H.zero_row, uint32_t(H.comps.size()),
                                      uint32_t(H.comp_heavy.size()), 0u, 0u};
        for (const auto &c : H.comps) blob.insert(blob.end(), {c.ci, c.n_out, c.upos_base, c.out_begin, c.first_tensor});
        for (uint8_t f : H.comp_heavy) blob.push_back(f);
        blob.insert(blob.end(), H.tensor_chunk_begin.begin(), H.tensor_chunk_begin.end());
        for (const uint4 &c : H.chunks) blob.insert(blob.end(), {c.x, c.y, c.z, c.w});
        blob.insert(blob.end(), H.words.begin(), H.words.end());
        *needed = blob.size();
        if (out && cap >= blob.size()) std::memcpy(out, blob.data(), blob.size() * 4);
    });
}

zxs_status zxs_debug_mono_layout(const zxs_model_desc *desc, uint64_t min_factors, uint32_t *out, uint64_t cap,
                                 uint64_t *needed) {
    return guarded([&] {
        if (!desc || !needed) fail(ZXS_INVALID_ARGUMENT, "null argument");
        uint32_t max_chain = 0;
        for (uint32_t c = 0; c < desc->num_components; c++) {
            max_chain = std::max(max_chain, desc->comp_out_begin[c + 1] - desc->comp_out_begin[c]);
        }
        MonoHost H = encode_mono(desc, max_chain, min_factors);
        std::vector<uint32_t> blob = {uint32_t(H.words.size()), uint32_t(H.chunks.size()),
                                      uint32_t(H.tensor_chunk_begin.size()), uint32_t(H.dict.size()),
                                      uint32_t(H.comps.size()), uint32_t(H.comp_mono.size()), H.all_plane, 0u};
        for (const auto &c : H.comps) blob.insert(blob.end(), {c.ci, c.n_out, c.upos_base, c.out_begin, c.first_tensor});
        for (uint8_t f : H.comp_mono) blob.push_back(f);
        blob.insert(blob.end(), H.tensor_chunk_begin.begin(), H.tensor_chunk_begin.end());
        for (const uint4 &c : H.chunks) blob.insert(blob.end(), {c.x, c.y, c.z, c.w});
        for (const uint4 &c : H.dict) blob.insert(blob.end(), {c.x, c.y, c.z, c.w});
        blob.insert(blob.end(), H.tensor_dict_begin.begin(), H.tensor_dict_begin.end());
        const size_t nt = H.tensor_chunk_begin.size() - 1;
        blob.insert(blob.end(), H.tensor_width.begin(), H.tensor_width.begin() + nt);
        blob.insert(blob.end(), H.tensor_basis_begin.begin(), H.tensor_basis_begin.begin() + nt);
        blob.push_back(uint32_t(H.basis.size()));
        for (unsigned long long x : H.basis) blob.insert(blob.end(), {uint32_t(x), uint32_t(x >> 32)});
        blob.insert(blob.end(), H.words.begin(), H.words.end());
        // summation segments (zxs_dedup.cuh): counts, tensor_seg_begin, segments, streams, key masks
        blob.insert(blob.end(), {uint32_t(H.tensor_seg_begin.size()), uint32_t(H.segs.size()),
                                 uint32_t(H.seg_words.size()), uint32_t(H.comp_key_mask.size())});
        blob.insert(blob.end(), H.tensor_seg_begin.begin(), H.tensor_seg_begin.end());
        for (const uint4 &c : H.segs) blob.insert(blob.end(), {c.x, c.y, c.z, c.w});
        blob.insert(blob.end(), H.seg_words.begin(), H.seg_words.end());
        for (unsigned long long x : H.comp_key_mask) blob.insert(blob.end(), {uint32_t(x), uint32_t(x >> 32)});
        // block form tables: counts, tensor_first_block, block_form_begin, block_forms
        blob.insert(blob.end(), {uint32_t(H.tensor_first_block.size()), uint32_t(H.block_form_begin.size()),
                                 uint32_t(H.block_forms.size())});
        blob.insert(blob.end(), H.tensor_first_block.begin(), H.tensor_first_block.end());
        blob.insert(blob.end(), H.block_form_begin.begin(), H.block_form_begin.end());
        blob.insert(blob.end(), H.block_forms.begin(), H.block_forms.end());
        // segments per warp per eval item, per mono tensor (a block = 16 x spw segments)
        blob.push_back(uint32_t(H.tensor_spw.size()));
        blob.insert(blob.end(), H.tensor_spw.begin(), H.tensor_spw.end());
        // per mono tensor: read mask and null-space pairs (dedup_node_prep_kernel's key reduction)
        blob.insert(blob.end(), {uint32_t(H.tensor_read_mask.size()), uint32_t(H.tensor_null_begin.size()),
                                 uint32_t(H.tensor_null.size())});
        for (unsigned long long x : H.tensor_read_mask) blob.insert(blob.end(), {uint32_t(x), uint32_t(x >> 32)});
        blob.insert(blob.end(), H.tensor_null_begin.begin(), H.tensor_null_begin.end());
        for (unsigned long long x : H.tensor_null) blob.insert(blob.end(), {uint32_t(x), uint32_t(x >> 32)});
        *needed = blob.size();
        if (out && cap >= blob.size()) std::memcpy(out, blob.data(), blob.size() * 4);
    });
}

zxs_status zxs_measure_philox_peak(int device, double *blocks_per_s) {
    return guarded([&] {
        if (!blocks_per_s) fail(ZXS_INVALID_ARGUMENT, "null output");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) fail(ZXS_CUDA_ERROR, "no CUDA device available");
        DeviceGuard g(device);
        int sms = 0, occ = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, zxs_dev::philox_peak_kernel, 32, 0));
        zxs_dev::LaunchArgs a{};
        a.seed = 0x0123456789abcdefull;
        for (int i = 0; i < 10; i++) a.k0_round[i] = uint32_t(a.seed) + uint32_t(i) * 0x9E3779B9u;
        uint32_t *sink = nullptr;
        CK(cudaMalloc(&sink, 4));
        const uint32_t nmech = 256, tiles = 16;
        const unsigned grid = unsigned(sms * std::max(occ, 1));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        zxs_dev::philox_peak_kernel<<<grid, 32>>>(a, nmech, tiles, sink);  // warm-up
        CK(cudaEventRecord(e0));
        const int reps = 5;
        for (int r = 0; r < reps; r++) zxs_dev::philox_peak_kernel<<<grid, 32>>>(a, nmech, tiles, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(sink);
        *blocks_per_s = double(reps) * grid * tiles * zxs_dev::kTileShots * nmech / (ms * 1e-3);
    });
}

zxs_status zxs_measure_fp64_peak(int device, double *ops_per_s) {
    return guarded([&] {
        if (!ops_per_s) fail(ZXS_INVALID_ARGUMENT, "null output");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) fail(ZXS_CUDA_ERROR, "no CUDA device available");
        DeviceGuard g(device);
        int sms = 0, occ = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, zxs_dev::fp64_peak_kernel, 256, 0));
        double *sink = nullptr;
        CK(cudaMalloc(&sink, 8));
        const uint32_t iters = 4096;
        const unsigned grid = unsigned(sms * std::max(occ, 1));
        const double2 hv = make_double2(0.70710678118654757, 0.70710678118654757);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        zxs_dev::fp64_peak_kernel<<<grid, 256>>>(hv, iters, sink);  // warm-up
        CK(cudaEventRecord(e0));
        const int reps = 3;
        for (int r = 0; r < reps; r++) zxs_dev::fp64_peak_kernel<<<grid, 256>>>(hv, iters, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(sink);
        *ops_per_s = double(reps) * grid * 256.0 * iters * 8 * 8 / (ms * 1e-3);  // 8 chains x (4 DMUL + 4 DADD)
    });
}

zxs_status zxs_measure_smem_peak(int device, double *bytes_per_s) {
    return guarded([&] {
        if (!bytes_per_s) fail(ZXS_INVALID_ARGUMENT, "null output");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) fail(ZXS_CUDA_ERROR, "no CUDA device available");
        DeviceGuard g(device);
        int sms = 0, occ = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, zxs_dev::smem_peak_kernel, 256, 0));
        uint32_t *sink = nullptr;
        CK(cudaMalloc(&sink, 4));
        const uint32_t iters = 8192;
        const unsigned grid = unsigned(sms * std::max(occ, 1));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        zxs_dev::smem_peak_kernel<<<grid, 256>>>(iters, sink);  // warm-up
        CK(cudaEventRecord(e0));
        const int reps = 3;
        for (int r = 0; r < reps; r++) zxs_dev::smem_peak_kernel<<<grid, 256>>>(iters, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(sink);
        // every warp load instruction moves 32 x 4 B
        *bytes_per_s = double(reps) * grid * 256.0 * iters * 16 * 4 / (ms * 1e-3);
    });
}

zxs_status zxs_philox_uniform(int device, uint64_t seed, uint32_t stream, uint64_t first_index, uint64_t n,
                              double *host_out) {
    return guarded([&] {
        if (n == 0) return;
        if (!host_out) fail(ZXS_INVALID_ARGUMENT, "null output");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) fail(ZXS_CUDA_ERROR, "no CUDA device available");
        DeviceGuard g(device);
        double *d = nullptr;
        CK(cudaMalloc(&d, n * 8));
        unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, 4096));
        zxs_dev::philox_kernel<<<grid, 256>>>(seed, stream, first_index, n, d);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpy(host_out, d, n * 8, cudaMemcpyDeviceToHost);
        cudaFree(d);
        CK(e);
    });
}

}  // extern "C"
