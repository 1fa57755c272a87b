// zxs_b200_shim.hpp — reference-side adapter: zxsim::CompiledSampler -> C ABI.
//
// Include this from code that already links the reference front-end
// (proj/include/zxsim/*.hpp). It keeps the reference's signatures so callers
// such as tools/zxsim.cpp:149-163 switch by namespace only:
//
//   zxsim::sample_detectors(cs, shots, opt)      (sampler.hpp:57-58)
//     -> zxsim_b200::sample_detectors(cs, shots, opt)
//
// and re-raises C-ABI status codes as the reference's exception classes
// (std::invalid_argument / std::runtime_error). There is no CPU
// fallback: without a GPU the call throws.
#pragma once

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <tuple>

#include "zxs_b200.h"
#include "zxs_b200_flatten.hpp"
#include "zxs_flat.hpp"
#include "zxsim/compile.hpp"
#include "zxsim/sampler.hpp"

namespace zxsim_b200 {

inline void raise_status(zxs_status st) {
    if (st == ZXS_OK) return;
    std::string msg = zxs_last_error();
    if (st == ZXS_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// RAII handle over one uploaded sampler.
class Sampler {
  public:
    Sampler(const zxsim::CompiledSampler &cs, int device = 0) {
        zxs::FlatModel flat = flatten(cs);
        zxs_model_desc d = flat.desc();
        raise_status(zxs_sampler_create(&d, device, &s_));
    }
    explicit Sampler(const zxs::FlatModel &flat, int device = 0) {
        zxs_model_desc d = flat.desc();
        raise_status(zxs_sampler_create(&d, device, &s_));
    }
    ~Sampler() { zxs_sampler_destroy(s_); }
    Sampler(const Sampler &) = delete;
    Sampler &operator=(const Sampler &) = delete;
    zxs_sampler *get() const { return s_; }

    zxsim::SampleRecord sample(zxs_mode mode, size_t shots, const zxsim::SamplerOptions &opt) const {
        zxs_sample_options o{opt.force_dense ? 1u : 0u, 0u, opt.sparse_threshold};
        return sample(mode, shots, opt.seed, &o);
    }

    zxsim::SampleRecord sample(zxs_mode mode, size_t shots, uint64_t seed,
                               const zxs_sample_options *opts = nullptr) const {
        zxs_sampler_info info;
        raise_status(zxs_sampler_get_info(s_, &info));
        zxsim::SampleRecord rec;
        rec.shots = shots;
        rec.width = info.num_outputs;
        size_t words = (shots + 63) / 64;
        std::vector<uint64_t> flat(static_cast<size_t>(info.num_outputs) * words);
        raise_status(zxs_sample_opts(s_, mode, seed, shots, opts, flat.data(), nullptr));
        rec.columns.assign(info.num_outputs, std::vector<uint64_t>(words));
        for (uint32_t o = 0; o < info.num_outputs; o++) {
            std::memcpy(rec.columns[o].data(), flat.data() + o * words, words * 8);
        }
        return rec;
    }

  private:
    zxs_sampler *s_ = nullptr;
};

// Uploaded samplers are cached per CompiledSampler (the reference's compiled
// sampler is immutable, compile.hpp:57-58), so repeated calls on the same
// object -- a CLI sweep, a decoder loop -- flatten and upload once. The key is
// the object's address plus a fingerprint of its contents (sizes, error-model
// probabilities, first/last term coefficients of every tensor), so a new
// sampler allocated at a recycled address is not mistaken for the old one.
struct CacheKey {
    const void *addr;
    uint64_t fingerprint;
    int device;
    bool operator<(const CacheKey &o) const {
        return std::tie(addr, fingerprint, device) < std::tie(o.addr, o.fingerprint, o.device);
    }
};

inline uint64_t fingerprint(const zxsim::CompiledSampler &cs) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t x) { h = (h ^ x) * 1099511628211ull; };
    auto mixd = [&](double d) { uint64_t x; std::memcpy(&x, &d, 8); mix(x); };
    mix(cs.f_width);
    mix(cs.num_outputs);
    mix(uint64_t(cs.mode));
    mix(cs.error_model.mechanisms.size());
    for (const auto &m : cs.error_model.mechanisms) {
        mixd(m.probability);
        mix(m.table.size());
        if (!m.table.empty()) mixd(m.table.back());
        mix(m.f_vectors.size());
    }
    mix(cs.direct.size());
    for (const auto &d : cs.direct) mix(d.output_index * 2 + d.flip_const + d.f_bits.size() * 1024);
    mix(cs.components.size());
    for (const auto &ac : cs.components) {
        mix(ac.output_indices.size());
        auto tens = [&](const zxsim::PhaseTermTensors &t) {
            mix(t.terms.size());
            if (!t.terms.empty()) {
                mixd(t.terms.front().c.real());
                mixd(t.terms.back().c.imag());
                mix(t.terms.back().num_factors());
            }
        };
        tens(ac.normalization);
        for (const auto &t : ac.marginals) tens(t);
    }
    return h;
}

inline std::shared_ptr<Sampler> cached_sampler(const zxsim::CompiledSampler &cs, int device = 0) {
    static std::mutex mu;
    static std::map<CacheKey, std::shared_ptr<Sampler>> cache;
    const CacheKey key{&cs, fingerprint(cs), device};
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (cache.size() >= 8) cache.erase(cache.begin());  // bounded: samplers hold device memory
    auto s = std::make_shared<Sampler>(cs, device);
    cache.emplace(key, s);
    return s;
}

// Drop-in replacements for sampler.hpp:57-60. `seed`, `sparse_threshold` and
// `force_dense` choose the bits exactly as in the reference (dense path, or
// the sparse geometric path when sparse_eligible, sampler.cpp:104-147);
// `batch_size` and `threads` are accepted and ignored -- the dense path's bits
// are the same for any batch split (sampler.cpp:82, 91, 268-284).
inline zxsim::SampleRecord sample_detectors(const zxsim::CompiledSampler &cs, size_t shots,
                                            const zxsim::SamplerOptions &opt) {
    return cached_sampler(cs)->sample(ZXS_MODE_DETECTORS, shots, opt);
}

inline zxsim::SampleRecord sample_measurements(const zxsim::CompiledSampler &cs, size_t shots,
                                               const zxsim::SamplerOptions &opt) {
    return cached_sampler(cs)->sample(ZXS_MODE_MEASUREMENTS, shots, opt);
}

}  // namespace zxsim_b200
