// zxs_flat.hpp — owning container for a flattened compiled sampler plus the
// `.zxs` file format (a list of named little-endian arrays).
//
// Header-only, no dependency on the reference: `zxs_b200_shim.hpp` fills a
// FlatModel from a zxsim::CompiledSampler, `desc()` views it as the C-ABI
// struct, and save()/load() move it through a file so a compiled sampler can
// be produced once on a host that has the reference front-end and sampled on
// a GPU host that does not. The Python reader is paper_2604_01059_b200/zxs_format.py.
//
// File layout: "ZXS1\0\0\0\0", u32 n_arrays, then per array
//   u32 name_len, name bytes, u32 dtype (0 u8, 1 u32, 2 i64, 3 f64, 4 u64),
//   u64 count, raw little-endian data, zero padding to 8-byte alignment.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "zxs_b200.h"

namespace zxs {

struct FlatModel {
    uint32_t mode = 0, num_detectors = 0, num_observables = 0, num_outputs = 0, f_width = 0;
    uint32_t flags = 0;        // ZXS_MODEL_* (header element 5; absent in older files)
    bool flags_known = false;  // the file carried the flags element
    std::vector<uint32_t> base_offset;
    std::vector<uint32_t> mech_vec_begin{0}, vec_bit_begin{0}, vec_bits;
    std::vector<double> mech_probability;
    std::vector<uint32_t> mech_table_begin{0};
    std::vector<double> table;
    std::vector<uint32_t> direct_output;
    std::vector<uint8_t> direct_flip_const;
    std::vector<uint32_t> direct_bit_begin{0}, direct_bits;
    std::vector<uint32_t> comp_out_begin{0}, comp_outputs, comp_num_magic;
    std::vector<uint64_t> comp_chi;
    std::vector<uint32_t> comp_tensor_begin{0};
    std::vector<uint32_t> tensor_param_width;
    std::vector<int64_t> tensor_exponent_halves;
    std::vector<uint64_t> tensor_term_begin{0};
    std::vector<double> term_c;
    std::vector<uint64_t> term_factor_begin{0};
    std::vector<uint32_t> factor_table;
    std::vector<uint64_t> factor_u_begin{0};
    std::vector<uint32_t> factor_u_bits;
    std::vector<uint64_t> factor_v_begin{0};
    std::vector<uint32_t> factor_v_bits;
    std::vector<double> h_table, h_alpha, h_beta;

    zxs_model_desc desc() const {
        zxs_model_desc d;
        std::memset(&d, 0, sizeof(d));
        d.abi_version = ZXS_ABI_VERSION;
        d.mode = mode;
        d.num_detectors = num_detectors;
        d.num_observables = num_observables;
        d.num_outputs = num_outputs;
        d.f_width = f_width;
        d.num_base_offset = static_cast<uint32_t>(base_offset.size());
        d.base_offset = base_offset.data();
        d.num_mechanisms = static_cast<uint32_t>(mech_vec_begin.size() - 1);
        d.mech_vec_begin = mech_vec_begin.data();
        d.num_vectors = static_cast<uint32_t>(vec_bit_begin.size() - 1);
        d.vec_bit_begin = vec_bit_begin.data();
        d.vec_bits = vec_bits.data();
        d.mech_probability = mech_probability.data();
        d.mech_table_begin = mech_table_begin.data();
        d.table = table.data();
        d.num_direct = static_cast<uint32_t>(direct_output.size());
        d.direct_output = direct_output.data();
        d.direct_flip_const = direct_flip_const.data();
        d.direct_bit_begin = direct_bit_begin.data();
        d.direct_bits = direct_bits.data();
        d.num_components = static_cast<uint32_t>(comp_out_begin.size() - 1);
        d.comp_out_begin = comp_out_begin.data();
        d.comp_outputs = comp_outputs.data();
        d.comp_num_magic = comp_num_magic.data();
        d.comp_chi = comp_chi.data();
        d.comp_tensor_begin = comp_tensor_begin.data();
        d.num_tensors = static_cast<uint32_t>(tensor_param_width.size());
        d.tensor_param_width = tensor_param_width.data();
        d.tensor_exponent_halves = tensor_exponent_halves.data();
        d.tensor_term_begin = tensor_term_begin.data();
        d.num_terms = term_factor_begin.size() - 1;
        d.term_c = term_c.data();
        d.term_factor_begin = term_factor_begin.data();
        d.num_factors = factor_table.size();
        d.factor_table = factor_table.data();
        d.factor_u_begin = factor_u_begin.data();
        d.factor_u_bits = factor_u_bits.data();
        d.factor_v_begin = factor_v_begin.data();
        d.factor_v_bits = factor_v_bits.data();
        d.num_h_tables = static_cast<uint32_t>(h_alpha.size());
        d.h_table = h_table.data();
        d.h_alpha = h_alpha.data();
        d.h_beta = h_beta.data();
        d.flags = flags;
        return d;
    }

    // ---- .zxs container --------------------------------------------------
    template <typename F>
    void visit(F &&f) {
        std::vector<uint32_t> header = {mode, num_detectors, num_observables, num_outputs, f_width, flags};
        f("header", header);
        mode = header.at(0);
        num_detectors = header.at(1);
        num_observables = header.at(2);
        num_outputs = header.at(3);
        f_width = header.at(4);
        flags_known = header.size() > 5;
        flags = flags_known ? header[5] : 0u;
        f("base_offset", base_offset);
        f("mech_vec_begin", mech_vec_begin);
        f("vec_bit_begin", vec_bit_begin);
        f("vec_bits", vec_bits);
        f("mech_probability", mech_probability);
        f("mech_table_begin", mech_table_begin);
        f("table", table);
        f("direct_output", direct_output);
        f("direct_flip_const", direct_flip_const);
        f("direct_bit_begin", direct_bit_begin);
        f("direct_bits", direct_bits);
        f("comp_out_begin", comp_out_begin);
        f("comp_outputs", comp_outputs);
        f("comp_num_magic", comp_num_magic);
        f("comp_chi", comp_chi);
        f("comp_tensor_begin", comp_tensor_begin);
        f("tensor_param_width", tensor_param_width);
        f("tensor_exponent_halves", tensor_exponent_halves);
        f("tensor_term_begin", tensor_term_begin);
        f("term_c", term_c);
        f("term_factor_begin", term_factor_begin);
        f("factor_table", factor_table);
        f("factor_u_begin", factor_u_begin);
        f("factor_u_bits", factor_u_bits);
        f("factor_v_begin", factor_v_begin);
        f("factor_v_bits", factor_v_bits);
        f("h_table", h_table);
        f("h_alpha", h_alpha);
        f("h_beta", h_beta);
    }

    template <typename T>
    static uint32_t dtype_code() {
        if constexpr (std::is_same_v<T, uint8_t>) return 0;
        if constexpr (std::is_same_v<T, uint32_t>) return 1;
        if constexpr (std::is_same_v<T, int64_t>) return 2;
        if constexpr (std::is_same_v<T, double>) return 3;
        if constexpr (std::is_same_v<T, uint64_t>) return 4;
    }

    void save(const std::string &path) {
        FILE *fp = std::fopen(path.c_str(), "wb");
        if (!fp) throw std::runtime_error("cannot open '" + path + "' for writing");
        std::fwrite("ZXS1\0\0\0\0", 1, 8, fp);
        uint32_t n = 0;
        visit([&](const char *, auto &) { n++; });
        std::fwrite(&n, 4, 1, fp);
        visit([&](const char *name, auto &vec) {
            using T = typename std::decay_t<decltype(vec)>::value_type;
            uint32_t len = static_cast<uint32_t>(std::strlen(name));
            uint32_t code = dtype_code<T>();
            uint64_t count = vec.size();
            std::fwrite(&len, 4, 1, fp);
            std::fwrite(name, 1, len, fp);
            std::fwrite(&code, 4, 1, fp);
            std::fwrite(&count, 8, 1, fp);
            size_t bytes = count * sizeof(T);
            if (bytes) std::fwrite(vec.data(), 1, bytes, fp);
            static const char pad[8] = {0};
            size_t used = 4 + len + 4 + 8 + bytes;
            if (used % 8) std::fwrite(pad, 1, 8 - used % 8, fp);
        });
        if (std::fclose(fp) != 0) throw std::runtime_error("write failed: " + path);
    }

    static FlatModel load(const std::string &path) {
        FILE *fp = std::fopen(path.c_str(), "rb");
        if (!fp) throw std::runtime_error("cannot open '" + path + "'");
        char magic[8];
        uint32_t n = 0;
        if (std::fread(magic, 1, 8, fp) != 8 || std::memcmp(magic, "ZXS1", 4) != 0 ||
            std::fread(&n, 4, 1, fp) != 1) {
            std::fclose(fp);
            throw std::runtime_error("not a .zxs file: " + path);
        }
        struct Raw {
            uint32_t code;
            std::vector<char> bytes;
        };
        std::map<std::string, Raw> arrays;
        for (uint32_t i = 0; i < n; i++) {
            uint32_t len = 0, code = 0;
            uint64_t count = 0;
            std::string name;
            bool ok = std::fread(&len, 4, 1, fp) == 1;
            name.resize(len);
            ok = ok && std::fread(name.data(), 1, len, fp) == len;
            ok = ok && std::fread(&code, 4, 1, fp) == 1 && std::fread(&count, 8, 1, fp) == 1;
            static const size_t sizes[5] = {1, 4, 8, 8, 8};
            if (!ok || code > 4) {
                std::fclose(fp);
                throw std::runtime_error("corrupt .zxs file: " + path);
            }
            size_t bytes = count * sizes[code];
            Raw r{code, std::vector<char>(bytes)};
            if (bytes && std::fread(r.bytes.data(), 1, bytes, fp) != bytes) {
                std::fclose(fp);
                throw std::runtime_error("truncated .zxs file: " + path);
            }
            size_t used = 4 + len + 4 + 8 + bytes;
            if (used % 8) std::fseek(fp, static_cast<long>(8 - used % 8), SEEK_CUR);
            arrays[name] = std::move(r);
        }
        std::fclose(fp);
        FlatModel m;
        m.visit([&](const char *name, auto &vec) {
            using T = typename std::decay_t<decltype(vec)>::value_type;
            auto it = arrays.find(name);
            if (it == arrays.end() || it->second.code != dtype_code<T>()) {
                throw std::runtime_error(std::string(".zxs array missing or mistyped: ") + name);
            }
            vec.resize(it->second.bytes.size() / sizeof(T));
            if (!vec.empty()) std::memcpy(vec.data(), it->second.bytes.data(), it->second.bytes.size());
        });
        return m;
    }
};

}  // namespace zxs
