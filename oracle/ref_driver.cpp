// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (see oracle/README.md).
//
// A thin extern "C" driver over the UNMODIFIED reference library (zxsim,
// compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libzxsim_ref.so). It stands in for the reference's CLI and
// doctest harness, which cannot build here (proj/vendor is absent,
// proj/.gitignore:2). Only tests/, __graft_entry__.smoke() and bench.py's
// reference / cpu_baseline legs load it.
//
// What it exposes:
//  * zr_compile / zr_save / zr_load: the reference front-end and the .zxs
//    round trip (unflatten rebuilds a zxsim::CompiledSampler so the
//    reference can sample a model on a host without /root/reference).
//  * zr_sample: the reference's public sample_detectors / sample_measurements
//    (sampler.cpp:306-320), unmodified.
//  * zr_sample_rb: a restatement of the reference's private run_batch
//    (sampler.cpp:51-102) built from its PUBLIC pieces (sample_error_batch,
//    eval_batch, Philox), with one ParamBatch per component sized to that
//    component's param_width. This sidesteps the width check at
//    phase_terms.cpp:91-97 that makes sample_outputs throw when components
//    differ in output count (SURVEY finding 2) without patching the
//    reference; the arithmetic is identical. Also takes any first_shot.
//  * zr_sample_error_batch, zr_eval_batch, zr_probability_of(_at),
//    zr_uniform_at: the reference's verification seams.
#include <atomic>
#include <complex>
#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "zxs_b200.h"
#include "zxs_flat.hpp"
#include "zxsim/circuit.hpp"
#include "zxsim/compile.hpp"
#include "zxsim/decompose.hpp"
#include "zxsim/lowering.hpp"
#include "zxsim/oracle.hpp"
#include "zxsim/simplify.hpp"
#include "zxsim/encode.hpp"
#include "zxsim/rng.hpp"
#include "zxsim/sampler.hpp"

// flatten() is shared with the product-side shim so the oracle and the
// product agree on the flattening by construction.
#include "zxs_b200_flatten.hpp"

namespace {

thread_local std::string g_error;

struct Handle {
    zxsim::CompiledSampler cs;
};

template <typename F>
int guarded(F &&f) {
    try {
        f();
        g_error.clear();
        return 0;
    } catch (const std::invalid_argument &e) {
        g_error = e.what();
        return 1;
    } catch (const std::exception &e) {
        g_error = e.what();
        return 2;
    }
}

zxsim::BitRow row_of(const uint32_t *bits, size_t n, uint32_t width) {
    zxsim::BitRow r(width);
    for (size_t i = 0; i < n; i++) r.set(bits[i], true);
    return r;
}

// Inverse of zxsim_b200::flatten: rebuilds every field the sampler reads.
zxsim::CompiledSampler unflatten(const zxs::FlatModel &m) {
    zxsim::CompiledSampler cs;
    cs.mode = m.mode == 0 ? zxsim::SampleMode::detectors : zxsim::SampleMode::measurements;
    cs.num_detectors = m.num_detectors;
    cs.num_observables = m.num_observables;
    cs.num_outputs = m.num_outputs;
    cs.f_width = m.f_width;
    cs.error_model.f_width = m.f_width;
    cs.error_model.base_offset = row_of(m.base_offset.data(), m.base_offset.size(), m.f_width);
    size_t nmech = m.mech_vec_begin.size() - 1;
    for (size_t i = 0; i < nmech; i++) {
        zxsim::ErrorMechanism mech;
        for (uint32_t v = m.mech_vec_begin[i]; v < m.mech_vec_begin[i + 1]; v++) {
            mech.f_vectors.push_back(row_of(m.vec_bits.data() + m.vec_bit_begin[v],
                                            m.vec_bit_begin[v + 1] - m.vec_bit_begin[v], m.f_width));
        }
        mech.probability = m.mech_probability[i];
        mech.table.assign(m.table.begin() + m.mech_table_begin[i],
                          m.table.begin() + m.mech_table_begin[i + 1]);
        cs.error_model.mechanisms.push_back(std::move(mech));
    }
    for (size_t i = 0; i < m.direct_output.size(); i++) {
        zxsim::DirectOutput d;
        d.output_index = m.direct_output[i];
        d.flip_const = m.direct_flip_const[i] != 0;
        d.f_bits.assign(m.direct_bits.begin() + m.direct_bit_begin[i],
                        m.direct_bits.begin() + m.direct_bit_begin[i + 1]);
        cs.direct.push_back(std::move(d));
    }
    auto tensor = [&](uint32_t t) {
        zxsim::PhaseTermTensors out;
        out.param_width = m.tensor_param_width[t];
        out.exponent_halves = m.tensor_exponent_halves[t];
        for (uint64_t term = m.tensor_term_begin[t]; term < m.tensor_term_begin[t + 1]; term++) {
            zxsim::PhaseTerm pt;
            pt.c = {m.term_c[2 * term], m.term_c[2 * term + 1]};
            for (uint64_t f = m.term_factor_begin[term]; f < m.term_factor_begin[term + 1]; f++) {
                uint32_t h = m.factor_table[f];
                pt.alpha.push_back(m.h_alpha[h]);
                pt.beta.push_back(m.h_beta[h]);
                pt.u.push_back(row_of(m.factor_u_bits.data() + m.factor_u_begin[f],
                                      m.factor_u_begin[f + 1] - m.factor_u_begin[f], out.param_width));
                pt.v.push_back(row_of(m.factor_v_bits.data() + m.factor_v_begin[f],
                                      m.factor_v_begin[f + 1] - m.factor_v_begin[f], out.param_width));
                std::array<zxsim::cdouble, 4> ht;
                for (int ab = 0; ab < 4; ab++) {
                    ht[ab] = {m.h_table[8 * h + 2 * ab], m.h_table[8 * h + 2 * ab + 1]};
                }
                pt.h_table.push_back(ht);
            }
            out.terms.push_back(std::move(pt));
        }
        return out;
    };
    size_t ncomp = m.comp_out_begin.size() - 1;
    for (size_t c = 0; c < ncomp; c++) {
        zxsim::AutoComponent ac;
        ac.output_indices.assign(m.comp_outputs.begin() + m.comp_out_begin[c],
                                 m.comp_outputs.begin() + m.comp_out_begin[c + 1]);
        ac.num_magic = m.comp_num_magic[c];
        ac.chi = m.comp_chi[c];
        uint32_t t0 = m.comp_tensor_begin[c], t1 = m.comp_tensor_begin[c + 1];
        ac.normalization = tensor(t0);
        for (uint32_t t = t0 + 1; t < t1; t++) ac.marginals.push_back(tensor(t));
        cs.stats.num_magic += ac.num_magic;
        cs.components.push_back(std::move(ac));
    }
    // Flip matrix and the sparse-eligibility flag (compile.cpp:285-325), so a
    // reloaded sampler takes the same dense/sparse branch as the original.
    cs.flips.rows.assign(cs.num_outputs, zxsim::BitRow(static_cast<uint32_t>(nmech)));
    cs.flips.columns.resize(nmech);
    bool any_joint = false;
    for (size_t i = 0; i < nmech; i++) {
        const zxsim::ErrorMechanism &mech = cs.error_model.mechanisms[i];
        if (mech.joint()) {
            any_joint = true;
            continue;
        }
        for (const zxsim::DirectOutput &d : cs.direct) {
            bool acc = false;
            for (uint32_t f : d.f_bits) acc ^= mech.f_vectors[0].get(f);
            if (acc) {
                cs.flips.columns[i].push_back(d.output_index);
                cs.flips.rows[d.output_index].set(static_cast<uint32_t>(i), true);
            }
        }
    }
    cs.stats.num_mechanisms = static_cast<uint32_t>(nmech);
    cs.stats.rank = cs.f_width;
    cs.stats.pure_clifford_deterministic =
        m.flags_known ? (m.flags & ZXS_MODEL_PURE_CLIFFORD_DETERMINISTIC) != 0
                      : (cs.stats.num_magic == 0 && cs.components.empty() && !any_joint);
    return cs;
}

constexpr double kRatioEps = 1e-6;                 // sampler.cpp:32
uint32_t auto_stream(uint32_t component, uint32_t pos) {  // sampler.cpp:37-39
    return 0x80000000u ^ (component << 12) ^ pos;
}

// Restatement of run_batch (sampler.cpp:51-102) over one shot range, writing
// into a [num_outputs][total_words] record at word offset word0. `fcols`
// (nullable) injects the f-columns; `uniforms` (nullable) injects the
// autoregressive draws as [chain position][shots].
void run_range(const zxsim::CompiledSampler &cs, uint64_t seed, size_t first_shot, size_t shots,
               const uint64_t *fcols, size_t fcols_ld, const double *uniforms, size_t uniforms_ld,
               uint64_t *rec, size_t rec_ld, size_t word0) {
    size_t words = (shots + 63) / 64;
    zxsim::ParamBatch fb(cs.f_width, shots);
    if (fcols) {
        for (uint32_t f = 0; f < cs.f_width; f++) {
            std::memcpy(fb.columns[f].data(), fcols + f * fcols_ld, words * 8);
        }
    } else {
        zxsim::sample_error_batch(cs, seed, first_shot, fb);
    }
    for (const zxsim::DirectOutput &d : cs.direct) {
        uint64_t *dst = rec + size_t(d.output_index) * rec_ld + word0;
        for (size_t w = 0; w < words; w++) {
            uint64_t acc = d.flip_const ? ~uint64_t(0) : 0;
            for (uint32_t f : d.f_bits) acc ^= fb.columns[f][w];
            dst[w] = acc;
        }
    }
    size_t upos = 0;
    for (uint32_t ci = 0; ci < cs.components.size(); ci++) {
        const zxsim::AutoComponent &ac = cs.components[ci];
        uint32_t n = static_cast<uint32_t>(ac.output_indices.size());
        zxsim::ParamBatch batch(cs.f_width + n, shots);
        for (uint32_t f = 0; f < cs.f_width; f++) batch.columns[f] = fb.columns[f];
        zxsim::BatchEvalResult prev = zxsim::eval_batch(ac.normalization, batch);
        for (uint32_t pos = 0; pos < n; pos++, upos++) {
            zxsim::BatchEvalResult cur = zxsim::eval_batch(ac.marginals[pos], batch);
            zxsim::Philox rng(seed, auto_stream(ci, pos));
            uint64_t *dst = rec + size_t(ac.output_indices[pos]) * rec_ld + word0;
            for (size_t w = 0; w < words; w++) dst[w] = 0;
            for (size_t s = 0; s < shots; s++) {
                double ratio = cur.values[s] / prev.values[s];
                if (!(ratio > -kRatioEps && ratio < 1.0 + kRatioEps)) {
                    throw std::runtime_error("autoregressive ratio outside [0, 1]: numeric breakdown");
                }
                ratio = std::min(1.0, std::max(0.0, ratio));
                double u = uniforms ? uniforms[upos * uniforms_ld + s] : rng.uniform_at(first_shot + s);
                bool bit = !(u < ratio);
                if (bit) {
                    batch.set(cs.f_width + pos, s, true);
                    dst[s >> 6] |= uint64_t(1) << (s & 63);
                    prev.values[s] -= cur.values[s];
                } else {
                    prev.values[s] = cur.values[s];
                }
            }
        }
    }
}

}  // namespace

extern "C" {

const char *zr_last_error() { return g_error.c_str(); }

int zr_compile(const char *text, int mode, void **out) {
    return guarded([&] {
        zxsim::Circuit c = zxsim::parse_circuit(text);
        auto *h = new Handle;
        h->cs = zxsim::compile_circuit(c, mode == 0 ? zxsim::SampleMode::detectors
                                                    : zxsim::SampleMode::measurements);
        *out = h;
    });
}

int zr_load(const char *path, void **out) {
    return guarded([&] {
        auto *h = new Handle;
        h->cs = unflatten(zxs::FlatModel::load(path));
        *out = h;
    });
}

int zr_save(void *handle, const char *path) {
    return guarded([&] { zxsim_b200::flatten(static_cast<Handle *>(handle)->cs).save(path); });
}

void zr_free(void *handle) { delete static_cast<Handle *>(handle); }

// info[0..15]: mode, num_detectors, num_observables, num_outputs, f_width,
// num_mechanisms, num_direct, num_components, joint mechanisms, max chain,
// total terms, total factors, chi product (clamped), num_magic,
// pure_clifford_deterministic, separation_complete
int zr_info(void *handle, uint64_t *info) {
    return guarded([&] {
        const zxsim::CompiledSampler &cs = static_cast<Handle *>(handle)->cs;
        uint64_t joints = 0, maxchain = 0, terms = 0, factors = 0;
        for (const auto &m : cs.error_model.mechanisms) joints += m.joint();
        for (const auto &ac : cs.components) {
            maxchain = std::max<uint64_t>(maxchain, ac.output_indices.size());
            auto add = [&](const zxsim::PhaseTermTensors &t) {
                terms += t.terms.size();
                for (const auto &pt : t.terms) factors += pt.num_factors();
            };
            add(ac.normalization);
            for (const auto &t : ac.marginals) add(t);
        }
        uint64_t v[16] = {uint64_t(cs.mode == zxsim::SampleMode::detectors ? 0 : 1),
                          cs.num_detectors, cs.num_observables, cs.num_outputs, cs.f_width,
                          cs.error_model.mechanisms.size(), cs.direct.size(), cs.components.size(),
                          joints, maxchain, terms, factors, cs.stats.chi, cs.stats.num_magic,
                          cs.stats.pure_clifford_deterministic, cs.stats.separation_complete};
        std::memcpy(info, v, sizeof(v));
    });
}

int zr_format_stats(void *handle, char *buf, size_t cap) {
    return guarded([&] {
        std::string s = zxsim::format_stats(static_cast<Handle *>(handle)->cs);
        std::snprintf(buf, cap, "%s", s.c_str());
    });
}

// The reference's public sampler, unmodified (sampler.cpp:306-320).
// out: [num_outputs][ceil(shots/64)].
int zr_sample(void *handle, uint64_t shots, uint64_t seed, uint64_t batch_size, uint32_t threads,
              int force_dense, uint64_t *out) {
    return guarded([&] {
        const zxsim::CompiledSampler &cs = static_cast<Handle *>(handle)->cs;
        zxsim::SamplerOptions opt;
        opt.seed = seed;
        opt.batch_size = batch_size;
        opt.threads = threads;
        opt.force_dense = force_dense != 0;
        zxsim::SampleRecord rec = cs.mode == zxsim::SampleMode::detectors
                                      ? zxsim::sample_detectors(cs, shots, opt)
                                      : zxsim::sample_measurements(cs, shots, opt);
        size_t words = (shots + 63) / 64;
        for (uint32_t o = 0; o < rec.width; o++) {
            std::memcpy(out + o * words, rec.columns[o].data(), words * 8);
        }
    });
}

// sample_detectors / sample_measurements with force_dense and sparse_threshold
// (sampler.hpp:32-38) -- the options that select the sparse path.
int zr_sample_opts(void *handle, uint64_t shots, uint64_t seed, int force_dense, double sparse_threshold,
                   uint64_t *out) {
    return guarded([&] {
        const zxsim::CompiledSampler &cs = static_cast<Handle *>(handle)->cs;
        zxsim::SamplerOptions opt;
        opt.seed = seed;
        opt.force_dense = force_dense != 0;
        opt.sparse_threshold = sparse_threshold;
        zxsim::SampleRecord rec = cs.mode == zxsim::SampleMode::detectors
                                      ? zxsim::sample_detectors(cs, shots, opt)
                                      : zxsim::sample_measurements(cs, shots, opt);
        size_t words = (shots + 63) / 64;
        for (uint32_t o = 0; o < rec.width; o++) {
            std::memcpy(out + o * words, rec.columns[o].data(), words * 8);
        }
    });
}

// run_batch restatement with per-component batch widths, over
// [first_shot, first_shot+shots), batches of batch_size claimed by `threads`
// workers like sample_outputs (sampler.cpp:149-199).
int zr_sample_rb(void *handle, uint64_t seed, uint64_t first_shot, uint64_t shots,
                 uint64_t batch_size, uint32_t threads, uint64_t *out) {
    return guarded([&] {
        const zxsim::CompiledSampler &cs = static_cast<Handle *>(handle)->cs;
        size_t words = (shots + 63) / 64;
        std::memset(out, 0, size_t(cs.num_outputs) * words * 8);
        if (shots == 0) return;
        size_t bs = std::max<size_t>(64, (batch_size + 63) & ~size_t(63));
        size_t nb = (shots + bs - 1) / bs;
        uint32_t nt = threads ? threads : std::thread::hardware_concurrency();
        nt = std::max(1u, std::min<uint32_t>(nt, static_cast<uint32_t>(nb)));
        std::atomic<size_t> next{0};
        std::atomic<bool> failed{false};
        std::string msg;
        std::mutex mu;
        auto worker = [&] {
            for (;;) {
                size_t b = next.fetch_add(1);
                if (b >= nb || failed.load()) return;
                size_t first = b * bs;
                size_t count = std::min(bs, size_t(shots) - first);
                try {
                    run_range(cs, seed, first_shot + first, count, nullptr, 0, nullptr, 0, out,
                              words, first / 64);
                } catch (const std::exception &e) {
                    std::lock_guard<std::mutex> lk(mu);
                    failed = true;
                    msg = e.what();
                    return;
                }
            }
        };
        if (nt == 1) {
            worker();
        } else {
            std::vector<std::thread> pool;
            for (uint32_t t = 0; t < nt; t++) pool.emplace_back(worker);
            for (auto &t : pool) t.join();
        }
        if (failed) throw std::runtime_error(msg);
        if (shots & 63) {
            uint64_t mask = (uint64_t(1) << (shots & 63)) - 1;
            for (uint32_t o = 0; o < cs.num_outputs; o++) out[o * words + words - 1] &= mask;
        }
    });
}

int zr_sample_given_f(void *handle, uint64_t seed, uint64_t first_shot, uint64_t shots,
                      const uint64_t *fcols, const double *uniforms, uint64_t *out) {
    return guarded([&] {
        const zxsim::CompiledSampler &cs = static_cast<Handle *>(handle)->cs;
        size_t words = (shots + 63) / 64;
        std::memset(out, 0, size_t(cs.num_outputs) * words * 8);
        if (shots == 0) return;
        run_range(cs, seed, first_shot, shots, fcols, words, uniforms, shots, out, words, 0);
        if (shots & 63) {
            uint64_t mask = (uint64_t(1) << (shots & 63)) - 1;
            for (uint32_t o = 0; o < cs.num_outputs; o++) out[o * words + words - 1] &= mask;
        }
    });
}

// sample_error_batch (sampler.cpp:257-304): fcols [f_width][ceil(shots/64)].
int zr_sample_error_batch(void *handle, uint64_t seed, uint64_t first_shot, uint64_t shots,
                          uint64_t *fcols) {
    return guarded([&] {
        const zxsim::CompiledSampler &cs = static_cast<Handle *>(handle)->cs;
        zxsim::ParamBatch batch(cs.f_width, shots);
        zxsim::sample_error_batch(cs, seed, first_shot, batch);
        size_t words = batch.words();
        for (uint32_t f = 0; f < cs.f_width; f++) {
            std::memcpy(fcols + f * words, batch.columns[f].data(), words * 8);
        }
    });
}

// eval_batch (phase_terms.cpp:90-144) on chain tensor `pos` (0 = normalization).
int zr_eval_batch(void *handle, uint32_t comp, uint32_t pos, const uint64_t *params,
                  uint32_t param_cols, uint64_t shots, double *values, double *max_imag) {
    return guarded([&] {
        const zxsim::CompiledSampler &cs = static_cast<Handle *>(handle)->cs;
        const zxsim::AutoComponent &ac = cs.components.at(comp);
        const zxsim::PhaseTermTensors &t = pos == 0 ? ac.normalization : ac.marginals.at(pos - 1);
        zxsim::ParamBatch batch(t.param_width, shots);
        size_t words = batch.words();
        if (param_cols < t.param_width) throw std::invalid_argument("eval_batch: parameter width mismatch");
        for (uint32_t p = 0; p < t.param_width; p++) {
            std::memcpy(batch.columns[p].data(), params + p * words, words * 8);
        }
        zxsim::BatchEvalResult r = zxsim::eval_batch(t, batch);
        std::memcpy(values, r.values.data(), shots * 8);
        if (max_imag) *max_imag = r.max_imag_ratio;
    });
}

int zr_probability_of_at(void *handle, const uint8_t *outcome, const uint8_t *f, double *out) {
    return guarded([&] {
        const zxsim::CompiledSampler &cs = static_cast<Handle *>(handle)->cs;
        std::vector<bool> o(cs.num_outputs);
        for (uint32_t i = 0; i < cs.num_outputs; i++) o[i] = outcome[i] != 0;
        zxsim::BitRow fr(cs.f_width);
        for (uint32_t i = 0; i < cs.f_width; i++) fr.set(i, f[i] != 0);
        *out = zxsim::probability_of_at(cs, o, fr);
    });
}

int zr_probability_of(void *handle, const uint8_t *outcome, double *out) {
    return guarded([&] {
        const zxsim::CompiledSampler &cs = static_cast<Handle *>(handle)->cs;
        std::vector<bool> o(cs.num_outputs);
        for (uint32_t i = 0; i < cs.num_outputs; i++) o[i] = outcome[i] != 0;
        *out = zxsim::probability_of(cs, o);
    });
}

double zr_uniform_at(uint64_t seed, uint32_t stream, uint64_t index) {
    return zxsim::Philox(seed, stream).uniform_at(index);
}

// encode_shots (encode.cpp:22-48) of a [width][ceil(shots/64)] record.
int zr_encode(const uint64_t *cols, uint32_t width, uint64_t shots, int format, char *out,
              uint64_t cap, uint64_t *written) {
    return guarded([&] {
        zxsim::SampleRecord rec;
        rec.shots = shots;
        rec.width = width;
        size_t words = (shots + 63) / 64;
        rec.columns.assign(width, std::vector<uint64_t>(words));
        for (uint32_t o = 0; o < width; o++) std::memcpy(rec.columns[o].data(), cols + o * words, words * 8);
        std::string s = zxsim::encode_shots(rec, format == 0 ? zxsim::ShotFormat::ascii01 : zxsim::ShotFormat::b8);
        if (s.size() > cap) throw std::invalid_argument("encode buffer too small");
        std::memcpy(out, s.data(), s.size());
        *written = s.size();
    });
}

// Front-end probe without the tensor build (compile.cpp:126-127, 249):
// lower -> undouble -> clifford_simplify -> plan_decomposition over the whole
// reduced diagram. out[0..4] = doubled magic spiders, total terms (chi),
// surviving vertices, error parameters, channel groups. Seconds where the
// full compile of a chi ~ 5e4 circuit takes minutes.
int zr_plan(const char *text, int mode, uint64_t *out) {
    return guarded([&] {
        zxsim::Circuit c = zxsim::parse_circuit(text);
        zxsim::LoweredProgram lp = zxsim::lower(c, mode == 0 ? zxsim::SampleMode::detectors
                                                             : zxsim::SampleMode::measurements);
        auto [reduced, trace] = zxsim::clifford_simplify(zxsim::undouble(lp.diagram));
        zxsim::DecompositionPlan plan = zxsim::plan_decomposition(reduced);
        out[0] = plan.num_magic;
        out[1] = plan.total_terms;
        out[2] = reduced.vertex_count();
        out[3] = lp.e_param_count;
        out[4] = lp.channels.size();
    });
}

// The reference's exact branching statevector oracle (oracle.cpp:494-542;
// <= 12 qubits, <= 16 measurements): outcome keys (bit i = output i) and
// their probabilities.
int zr_oracle_distribution(const char *text, int mode, uint64_t *keys, double *probs, uint64_t cap,
                           uint64_t *n) {
    return guarded([&] {
        zxsim::Circuit c = zxsim::parse_circuit(text);
        zxsim::OutcomeDistribution d = zxsim::oracle_distribution(
            c, mode == 0 ? zxsim::SampleMode::detectors : zxsim::SampleMode::measurements);
        uint64_t i = 0;
        for (const auto &[k, p] : d.probs) {
            if (i < cap) {
                keys[i] = k;
                probs[i] = p;
            }
            i++;
        }
        *n = i;
    });
}

}  // extern "C"
