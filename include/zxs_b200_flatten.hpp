// zxs_b200_flatten.hpp — zxsim::CompiledSampler -> zxs::FlatModel (the C-ABI arrays).
//
// Reference-side code: include it from a translation unit that has the
// reference headers (proj/include) on its include path. Shared by the
// product shim (zxs_b200_shim.hpp) and the oracle driver (oracle/ref_driver.cpp)
// so both flatten identically by construction.
#pragma once

#include <cstring>
#include <map>
#include <vector>

#include "zxs_b200.h"
#include "zxs_flat.hpp"
#include "zxsim/compile.hpp"

namespace zxsim_b200 {

// Flattens a compiled sampler (compile.hpp:59-72) into the C-ABI arrays.
// h tables are deduplicated by exact bit pattern of (alpha, beta, h[4]).
inline zxs::FlatModel flatten(const zxsim::CompiledSampler &cs) {
    zxs::FlatModel m;
    m.mode = cs.mode == zxsim::SampleMode::detectors ? ZXS_MODE_DETECTORS : ZXS_MODE_MEASUREMENTS;
    m.num_detectors = cs.num_detectors;
    m.num_observables = cs.num_observables;
    m.num_outputs = cs.num_outputs;
    m.f_width = cs.f_width;
    m.flags = cs.stats.pure_clifford_deterministic ? ZXS_MODEL_PURE_CLIFFORD_DETERMINISTIC : 0u;
    m.flags_known = true;
    const zxsim::ErrorModel &em = cs.error_model;
    if (em.base_offset.width() != 0) m.base_offset = em.base_offset.set_bits();
    for (const zxsim::ErrorMechanism &mech : em.mechanisms) {
        for (const zxsim::BitRow &v : mech.f_vectors) {
            for (uint32_t b : v.set_bits()) m.vec_bits.push_back(b);
            m.vec_bit_begin.push_back(static_cast<uint32_t>(m.vec_bits.size()));
        }
        m.mech_vec_begin.push_back(static_cast<uint32_t>(m.vec_bit_begin.size() - 1));
        m.mech_probability.push_back(mech.probability);
        for (double t : mech.table) m.table.push_back(t);
        m.mech_table_begin.push_back(static_cast<uint32_t>(m.table.size()));
    }
    for (const zxsim::DirectOutput &d : cs.direct) {
        m.direct_output.push_back(d.output_index);
        m.direct_flip_const.push_back(d.flip_const ? 1 : 0);
        for (uint32_t b : d.f_bits) m.direct_bits.push_back(b);
        m.direct_bit_begin.push_back(static_cast<uint32_t>(m.direct_bits.size()));
    }
    std::map<std::vector<uint64_t>, uint32_t> tables;
    auto bits_of = [](double x) {
        uint64_t u;
        std::memcpy(&u, &x, 8);
        return u;
    };
    auto add_tensor = [&](const zxsim::PhaseTermTensors &t) {
        m.tensor_param_width.push_back(t.param_width);
        m.tensor_exponent_halves.push_back(t.exponent_halves);
        for (const zxsim::PhaseTerm &term : t.terms) {
            m.term_c.push_back(term.c.real());
            m.term_c.push_back(term.c.imag());
            for (size_t k = 0; k < term.num_factors(); k++) {
                std::vector<uint64_t> key = {bits_of(term.alpha[k]), bits_of(term.beta[k])};
                for (const auto &h : term.h_table[k]) {
                    key.push_back(bits_of(h.real()));
                    key.push_back(bits_of(h.imag()));
                }
                auto it = tables.find(key);
                uint32_t id;
                if (it == tables.end()) {
                    id = static_cast<uint32_t>(m.h_alpha.size());
                    tables.emplace(key, id);
                    m.h_alpha.push_back(term.alpha[k]);
                    m.h_beta.push_back(term.beta[k]);
                    for (const auto &h : term.h_table[k]) {
                        m.h_table.push_back(h.real());
                        m.h_table.push_back(h.imag());
                    }
                } else {
                    id = it->second;
                }
                m.factor_table.push_back(id);
                for (uint32_t b : term.u[k].set_bits()) m.factor_u_bits.push_back(b);
                m.factor_u_begin.push_back(m.factor_u_bits.size());
                for (uint32_t b : term.v[k].set_bits()) m.factor_v_bits.push_back(b);
                m.factor_v_begin.push_back(m.factor_v_bits.size());
            }
            m.term_factor_begin.push_back(m.factor_table.size());
        }
        m.tensor_term_begin.push_back(m.term_factor_begin.size() - 1);
    };
    for (const zxsim::AutoComponent &ac : cs.components) {
        for (uint32_t o : ac.output_indices) m.comp_outputs.push_back(o);
        m.comp_out_begin.push_back(static_cast<uint32_t>(m.comp_outputs.size()));
        m.comp_num_magic.push_back(ac.num_magic);
        m.comp_chi.push_back(ac.chi);
        add_tensor(ac.normalization);
        for (const zxsim::PhaseTermTensors &t : ac.marginals) add_tensor(t);
        m.comp_tensor_begin.push_back(static_cast<uint32_t>(m.tensor_param_width.size()));
    }
    return m;
}

}  // namespace zxsim_b200
