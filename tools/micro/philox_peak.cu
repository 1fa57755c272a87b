// Philox4x32-10 throughput microbenchmark (same-op-mix roofline for the
// sampler's error draw). Variants: S shots per lane sharing one key schedule,
// and the 32x32->64 multiply as mul.wide.u32 (IMAD.WIDE) or mul.hi + mul.lo.
// Prints blocks/s per variant. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <bool WIDE>
__device__ __forceinline__ void mulw(uint32_t a, uint32_t b, uint32_t &lo, uint32_t &hi) {
    if (WIDE) {
        asm("{\n\t.reg .b64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}" : "=r"(lo), "=r"(hi) : "r"(a), "r"(b));
    } else {
        hi = __umulhi(a, b);
        lo = a * b;
    }
}
template <int S, bool WIDE>
__global__ void __launch_bounds__(256) philox_peak(uint32_t nmech, uint64_t seed, unsigned long long lim, uint32_t *out) {
    uint64_t base = (uint64_t(blockIdx.x) * 256 + threadIdx.x) * S;
    uint32_t lo[S], hi[S], acc[S];
#pragma unroll
    for (int s = 0; s < S; s++) { lo[s] = uint32_t(base + s); hi[s] = uint32_t((base + s) >> 32); acc[s] = 0; }
    const uint32_t sl = uint32_t(seed), sh = uint32_t(seed >> 32);
    for (uint32_t m = 0; m < nmech; m++) {
        uint32_t c0[S], c1[S], c2[S], c3[S];
#pragma unroll
        for (int s = 0; s < S; s++) { c0[s] = lo[s]; c1[s] = hi[s]; c2[s] = 0x9e3779b9u; c3[s] = 0; }
        uint32_t k0 = sl, k1 = sh ^ m;
#pragma unroll
        for (int i = 0; i < 10; i++) {
#pragma unroll
            for (int s = 0; s < S; s++) {
                uint32_t h0, l0, h1, l1;
                mulw<WIDE>(c0[s], 0xD2511F53u, l0, h0);
                mulw<WIDE>(c2[s], 0xCD9E8D57u, l1, h1);
                uint32_t n0 = h1 ^ c1[s] ^ k0, n2 = h0 ^ c3[s] ^ k1;
                c0[s] = n0; c1[s] = l1; c2[s] = n2; c3[s] = l0;
            }
            k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
        }
#pragma unroll
        for (int s = 0; s < S; s++) {
            uint64_t r = (uint64_t(c0[s]) << 32) | c1[s];
            if (r <= lim) acc[s] ^= m;
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int s = 0; s < S; s++) x ^= acc[s];
    if (x == 0xdeadbeef) out[0] = x;
}

template <int S, bool WIDE>
void run(const char *name, int sms) {
    uint32_t *out;
    cudaMalloc(&out, 4);
    const uint32_t nmech = 1000;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, philox_peak<S, WIDE>, 256, 0);
    unsigned grid = sms * occ * 8;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    philox_peak<S, WIDE><<<grid, 256>>>(nmech, 1, 1ull << 50, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) philox_peak<S, WIDE><<<grid, 256>>>(nmech, 1 + r, 1ull << 50, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double blocks = 5.0 * grid * 256.0 * S * nmech;
    printf("{\"variant\": \"%s\", \"S\": %d, \"wide\": %d, \"occ\": %d, \"blocks_per_s\": %.4e, \"ms\": %.3f}\n", name, S, WIDE,
           occ, blocks / (ms / 1e3), ms);
    cudaFree(out);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1, true>("S1_wide", sms);
    run<2, true>("S2_wide", sms);
    run<4, true>("S4_wide", sms);
    run<1, false>("S1_hilo", sms);
    run<2, false>("S2_hilo", sms);
    run<4, false>("S4_hilo", sms);
    return 0;
}
