// qz_bits.cuh — index bit helpers shared by host code, the AOT kernels and
// the runtime-specialised gate passes (qz_jit.cu compiles this header with
// NVRTC, so it includes nothing).
#pragma once

#include "qz_rtc_types.cuh"

namespace qz {

__host__ __device__ __forceinline__ uint64_t insert_zero_bit(uint64_t x, uint32_t bit) {
    uint64_t low = x & ((uint64_t(1) << bit) - 1);
    return ((x >> bit) << (bit + 1)) | low;
}

__host__ __device__ __forceinline__ uint32_t insert_zero_bit32(uint32_t x, uint32_t bit) {
    uint32_t low = x & ((1u << bit) - 1);
    return ((x >> bit) << (bit + 1)) | low;
}

// Scatter the low bits of v into the set bits of mask (ascending), i.e. pdep.
__host__ __device__ __forceinline__ uint64_t deposit_bits(uint64_t v, uint64_t mask) {
    uint64_t out = 0;
    while (mask) {
        uint64_t low = mask & (~mask + 1);
        if (v & 1) out |= low;
        v >>= 1;
        mask &= mask - 1;
    }
    return out;
}

} // namespace qz
