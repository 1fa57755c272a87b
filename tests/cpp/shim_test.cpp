// tests/cpp/shim_test.cpp -- builds the reference-side drop-in
// (include/zxs_b200_shim.hpp) the way a reference maintainer would: against
// the reference's own headers and library (proj/include, oracle/_ref) plus
// libzxs_b200.so. Run on a GPU box by tests/test_shim.py.
//
// usage: shim_test <circuit.stim> <shots> <seed>
// Compiles the circuit with the reference front-end, samples it with
// zxsim::sample_detectors (the CPU reference, force_dense) and with
// zxsim_b200::sample_detectors twice (the second call must hit the sampler
// cache), and prints "OK <ones> <cached>" when all three records are equal.
#include <cstdio>
#include <fstream>
#include <sstream>

#include "zxs_b200_shim.hpp"
#include "zxsim/circuit.hpp"

int main(int argc, char **argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s circuit.stim shots seed\n", argv[0]);
        return 2;
    }
    std::ifstream in(argv[1]);
    std::stringstream ss;
    ss << in.rdbuf();
    const size_t shots = std::stoull(argv[2]);
    zxsim::SamplerOptions opt;
    opt.seed = std::stoull(argv[3]);
    opt.force_dense = true;
    try {
        zxsim::Circuit c = zxsim::parse_circuit(ss.str());
        zxsim::CompiledSampler cs = zxsim::compile_circuit(c, zxsim::SampleMode::detectors);
        zxsim::SampleRecord want = zxsim::sample_detectors(cs, shots, opt);
        zxsim::SampleRecord a = zxsim_b200::sample_detectors(cs, shots, opt);
        auto s1 = zxsim_b200::cached_sampler(cs);
        zxsim::SampleRecord b = zxsim_b200::sample_detectors(cs, shots, opt);
        auto s2 = zxsim_b200::cached_sampler(cs);
        if (a.columns != want.columns || b.columns != want.columns) {
            std::printf("MISMATCH\n");
            return 1;
        }
        uint64_t ones = 0;
        for (const auto &col : want.columns)
            for (uint64_t w : col) ones += __builtin_popcountll(w);
        std::printf("OK %llu %d\n", (unsigned long long)ones, s1.get() == s2.get() ? 1 : 0);
        // the reference's exception classes come back through the shim
        try {
            zxsim_b200::sample_measurements(cs, 64, opt);
            std::printf("NO-THROW\n");
            return 1;
        } catch (const std::invalid_argument &e) {
            std::printf("invalid_argument: %s\n", e.what());
        }
    } catch (const std::exception &e) {
        std::printf("ERROR %s\n", e.what());
        return 1;
    }
    return 0;
}
