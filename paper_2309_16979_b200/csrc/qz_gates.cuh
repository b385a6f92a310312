// qz_gates.cuh — gate matrices, fused gate passes and the tile kernel API.
#pragma once

#include <vector>

#include "qz_common.cuh"

namespace qz {

// One gate with its host-computed matrix (gates.cpp:114-182) on buffer bits.
struct DevGate {
    uint32_t nq;       // 1 or 2
    uint32_t b0, b1;   // buffer bits (b0 = first listed = matrix high bit)
    uint32_t cls;      // structure class, see GateClass
    double2 m[16];     // row-major, dim = 2 or 4
};

// Structure classes let the kernel skip exactly-zero coefficients.  A term
// with coefficient exactly 0 contributes ±0, which can only change the SIGN
// of an exactly-zero result; any such result is recomputed with the full
// formula, so every class is bit-identical to the dense formula.
enum GateClass : uint32_t {
    GC_DENSE = 0,   // general matrix
    GC_DIAG = 1,    // 1q: m01 == m10 == 0       (Z S T U1 RZ SDG TDG)
    GC_ANTI = 2,    // 1q: m00 == m11 == 0       (X Y)
    GC_PERM4 = 3,   // 2q: one nonzero per row   (CX CZ SWAP)
};

// A fused pass: gates whose buffer bits all lie in the tile bit set T.
struct PassDesc {
    uint32_t k;            // tile bits (|T|)
    uint32_t lowbits;      // T ⊇ {0..lowbits-1}
    uint32_t first_gate;   // into the pass-local gate array
    uint32_t ngates;
    uint64_t tmask;        // T as a bit mask over buffer bits
};

// Pass-local gate: bits are positions inside the tile.
struct TileGate {
    uint32_t nq, t0, t1, cls;
    double2 m[16];
};

struct GatePlan {
    std::vector<PassDesc> passes;
    std::vector<TileGate> gates;
};

// Host: matrix for a qzc_gate, bit-identical to qzsim::gate_matrix.
void gate_matrix_host(const qzc_gate &g, double2 *m, uint32_t *dim);
uint32_t gate_arity(uint32_t kind);
uint32_t gate_nparams(uint32_t kind);

// Host: greedy in-order fusion of gates (already on buffer bits) into passes
// over a buffer of 2^nbits amplitudes with tiles of at most 2^kmax.
GatePlan build_passes(const std::vector<DevGate> &gates, uint32_t nbits,
                      uint32_t kmax, bool fuse);

DevGate make_dev_gate(const qzc_gate &g);

// Device-resident copy of a GatePlan.
struct DevPlan {
    PassDesc *passes = nullptr;
    TileGate *gates = nullptr;
    size_t npasses = 0, ngates = 0;
    std::vector<PassDesc> host_passes;
};
void upload_plan(const GatePlan &plan, DevPlan &out, cudaStream_t s);
void free_plan(DevPlan &p);

// Launch every pass of `plan` over buf (2^nbits amplitudes).  Returns the
// number of kernel launches.
uint64_t run_passes(const DevPlan &plan, double2 *buf, uint32_t nbits,
                    cudaStream_t s);

} // namespace qz
