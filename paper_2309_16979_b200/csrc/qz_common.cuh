// qz_common.cuh — shared device/host helpers for the sm_100a engine.
//
// Bit-exactness rules (probe-verified against the reference):
//  * complex products round like libstdc++ std::complex<double> without FMA:
//    re = fl(fl(a*c) - fl(b*d)), im = fl(fl(a*d) + fl(b*c))  (kernels.cpp:31-32)
//  * every fp64 op below is an explicit __d*_rn intrinsic, never contracted;
//    the library is also built with --fmad=false as a second guard.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/qzcuda.h"
#include "qz_bits.cuh"

namespace qz {

// ---------------------------------------------------------------- errors --
struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define QZ_CUDA(expr)                                                            \
    do {                                                                         \
        cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess)                                                   \
            throw ::qz::Failure(QZC_ECUDA, std::string(#expr) + ": " +           \
                                               cudaGetErrorString(_e));          \
    } while (0)

#define QZ_CHECK_LAUNCH() QZ_CUDA(cudaGetLastError())

// Device-side status word: the first failing chunk records (code, index).
struct DevStatus {
    int code;          // 0 ok, else a QZS_* value below
    int pad;
    uint64_t index;    // chunk index (or slot) that failed
};

enum : int {
    QZS_OK = 0,
    QZS_CRC = 1,          // "checksum mismatch on chunk i"   (codec.cpp:188-190)
    QZS_HEADER = 2,       // truncated header / unknown codec / disagreement
    QZS_RLE_TRUNC = 3,    // "truncated RLE stream"           (codec.cpp:70)
    QZS_RLE_RUN = 4,      // "bad RLE run length"             (codec.cpp:73-74)
    QZS_RAW_MISSING = 5,  // "missing raw values"             (codec.cpp:221-222)
    QZS_RAW_UNDER = 6,    // "raw value underflow"            (codec.cpp:235-237)
    QZS_RAW_UNUSED = 7,   // "unused raw values"              (codec.cpp:247-248)
    QZS_ARENA = 8,        // compressed arena capacity exhausted
};

__device__ inline void dev_fail(DevStatus *st, int code, uint64_t index) {
    if (atomicCAS(&st->code, 0, code) == 0) st->index = index;
}

// ------------------------------------------------------- exact fp64 math --
struct cplx {
    double re, im;
};

__device__ __forceinline__ cplx cmul(double mr, double mi, double2 a) {
    cplx r;
    r.re = __dsub_rn(__dmul_rn(mr, a.x), __dmul_rn(mi, a.y));
    r.im = __dadd_rn(__dmul_rn(mr, a.y), __dmul_rn(mi, a.x));
    return r;
}

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

constexpr int kNumSMs = 148;

} // namespace qz
