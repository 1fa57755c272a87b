// zxs_encode.cuh — encode_shots (proj/src/encode.cpp:22-48) on the device.
//
// The record is column-major (SampleRecord.columns, sampler.hpp:22-30): bit s
// of output o lives in word s >> 6 of column o. The CLI writes it shot-major:
//   b8     per shot ceil(width/8) bytes, output b at bit b % 8 of byte b / 8
//   01     per shot `width` characters '0'/'1' and a '\n'
// One warp turns one 32-shot word of up to 32 outputs at a time into shot-major
// bits with the in-register 32x32 transpose (lane o loads output o's word,
// lane s ends up with output bits of shot s), builds the 32 shots' bytes in
// shared memory and copies the contiguous block out with 32-bit stores. Every
// byte of the record is read once and every output byte written once: the
// kernel is HBM-bound.
#pragma once

#include "zxs_device.cuh"

namespace zxs_dev {

constexpr int kEncWarps = 4;

struct EncodeArgs {
    const uint32_t *cols;     // [num_outputs][ld32]
    uint64_t ld32;
    uint32_t first_output, width, format;  // format: 0 = 01, 1 = b8
    uint64_t shots;
    uint8_t *out;
    uint32_t row_bytes;       // b8: ceil(width/8); 01: width + 1
    uint32_t smem_per_warp;   // 32 * row_bytes rounded up to 16
};

__global__ void __launch_bounds__(kEncWarps * 32) encode_kernel(const __grid_constant__ EncodeArgs e) {
    extern __shared__ __align__(16) uint8_t esm[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint8_t *blk = esm + warp * e.smem_per_warp;
    const uint64_t nwords = (e.shots + 31) / 32;
    const uint32_t groups = (e.width + 31) / 32;
    const uint32_t rb = e.row_bytes;
    for (uint64_t w = uint64_t(blockIdx.x) * kEncWarps + warp; w < nwords; w += uint64_t(gridDim.x) * kEncWarps) {
        for (uint32_t g = 0; g < groups; g++) {
            const uint32_t o = g * 32 + lane;
            const uint32_t v = o < e.width ? e.cols[uint64_t(e.first_output + o) * e.ld32 + w] : 0u;
            const uint32_t t = warp_transpose32(v, lane);  // bit j = output g*32+j of shot w*32+lane
            uint8_t *row = blk + lane * rb;
            if (e.format == 1) {
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    if (g * 4 + k < rb) row[g * 4 + k] = uint8_t(t >> (8 * k));
                }
            } else {
                const uint32_t n = min(32u, e.width - g * 32);
                for (uint32_t j = 0; j < n; j++) row[g * 32 + j] = uint8_t('0' + ((t >> j) & 1u));
            }
        }
        if (e.format == 0) blk[lane * rb + e.width] = '\n';
        __syncwarp();
        const uint64_t s0 = w * 32;
        const uint32_t nshots = uint32_t(e.shots - s0 < 32 ? e.shots - s0 : 32);
        const uint32_t bytes = nshots * rb;
        uint8_t *dst = e.out + s0 * rb;
        if (nshots == 32) {  // 32 * rb bytes: a multiple of 32, 32-byte aligned in both spaces
            const uint32_t *src4 = reinterpret_cast<const uint32_t *>(blk);
            uint32_t *dst4 = reinterpret_cast<uint32_t *>(dst);
            for (uint32_t i = lane; i < bytes / 4; i += 32) dst4[i] = src4[i];
        } else {
            for (uint32_t i = lane; i < bytes; i += 32) dst[i] = blk[i];
        }
        __syncwarp();
    }
}

}  // namespace zxs_dev
