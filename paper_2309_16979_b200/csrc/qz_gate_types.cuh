// qz_gate_types.cuh — plan records the fused gate-pass kernel reads (gate,
// group and pass descriptors).  Plain data, no includes beyond fixed-width
// types: also compiled by NVRTC for the runtime-specialised passes.
#pragma once

#include "qz_rtc_types.cuh"

namespace qz {

// Coefficient kinds of a matrix entry; the kernel evaluates each product
// with the cheapest form that is exact for NONZERO results (see qz_gates.cu).
enum CoefKind : uint32_t { CK_ZERO = 0, CK_ONE = 1, CK_NEG = 2, CK_REAL = 3, CK_IMAG = 4, CK_CPLX = 5 };


// Matrix structure for the zero-free register fast path.  CX / CZ / SWAP are
// recognised by value (their ±0 entries only ever matter for zero outputs,
// which the fast path never produces without falling back).
enum GateOp : uint32_t {
    OP_GEN1 = 0, OP_DIAG = 1, OP_CX = 2, OP_CZ = 3, OP_SWAP = 4, OP_GEN2 = 5,
    // fast-path macros (a run of gates on one qubit pair, same operations)
    OP_CP5 = 6,  // U1(a) CX(a,b) U1(b) CX(a,b) U1(b): m[0..2] = the U1s' phase entries
    OP_CXD = 7,  // CX(a,b) D(b) CX(a,b), D diagonal: m[0], m[1] = D's entries
    // diagonal unit (1q diagonal, CZ, CP5 or CXD run) with qubits that are not
    // register bits of its group (outside the pass's tile set, or tile bits
    // held constant across a thread's registers): per thread the unit reduces
    // to a diagonal chain on <= 1 register bit.  Variant v = values of those
    // bits in the thread's amplitude index (ob0 -> bit 0, ob1 -> bit 1); state s of the
    // register bit (s = 0 only when nq == 0: uniform over the block); step
    // j < 2: kinds nibble 4v+2s+j (CK_ZERO = no step), coefficient m[4v+2s+j],
    // srow bit 4v+2s+j = step is +0-safe.
    OP_PDIAG = 8,
};

// A gate inside a register group: r0/r1 are the gate's qubits as bit
// positions of the thread's 16-amplitude register block.
struct TileGate {
    uint32_t nq, r0, r1, t0, t1;  // t0/t1: tile-local bits (tiny-buffer path)
    uint32_t sgn;
    uint64_t kinds;
    uint32_t cls;                 // GateClass
    uint32_t perm;                // TG_PERM: per row 2 bits column + 1 bit negate
    uint32_t zm;                  // bit e: Re m_e == 0; bit 16+e: Im m_e == 0
    uint32_t smask;               // bit e: sign(Re m_e); bit 16+e: sign(Im m_e)
    uint32_t op;                  // GateOp
    uint32_t pad;                 // bit r: row r maps all-(+0) inputs to (+0,+0)
    uint32_t srow;                // bit r: row r is "+0-safe" (see qz_gates.cu)
    uint32_t pad2;                // compile-time specialisation code of the fast path
    uint32_t ob0, ob1;            // OP_PDIAG: outside buffer bits (ob1 = 63 if unused)
    uint32_t run;                 // OP_PDIAG, all steps CPLX and +0-safe: length of the
                                  // run of such ops starting here (0 otherwise)
    uint32_t steps;               // OP_PDIAG: bit 4v+e set = step e of variant v present
    uint32_t cid;                 // fast-path case id (the kernel's jump table)
    uint32_t pad4[3];
    double2 m[16];
};

// Gate structure for the register fast path.
enum GateClass : uint32_t {
    TG_GEN = 0,    // general: per-entry kinds
    TG_PERM = 1,   // each row has one nonzero entry, exactly +1 or -1 (X CX CZ SWAP Z)
    TG_DIAG = 2,   // 1q diagonal (U1 S T SDG TDG RZ)
};

// Register block of the fused pass: each thread applies a group's gates to
// 2^kRegBits amplitudes held in registers.
#ifndef QZ_REG_BITS
#define QZ_REG_BITS 3
#endif
constexpr int kRegBits = QZ_REG_BITS;
// Fused-pass tile: 2^kTileBits amplitudes in shared memory per CTA.
#ifndef QZ_TILE_BITS
#define QZ_TILE_BITS 11
#endif
constexpr uint32_t kTileBits = QZ_TILE_BITS;

// Consecutive gates whose qubits fit kRegBits tile bits: applied in registers.
struct GroupDesc {
    uint32_t gbits[4];     // tile-local bits, ascending; register bit i <-> gbits[i]
    uint32_t first_gate, ngates;   // exact gate list
    uint32_t first_fast, nfast;    // fast-path list (macros folded in)
    uint32_t generic;      // 1: apply on the smem tile with the full formula
    uint32_t pz_stable;    // every gate maps an all-(+0) block to all-(+0)
    uint32_t relaxed;      // holds OP_PDIAG units: no exact path; a block that
                           // cannot take the fast path raises the replay flag
    uint32_t unsafe;       // some of its OP_PDIAG steps are not +0-safe (checked)
};

// A fused pass: gates whose buffer bits all lie in the tile bit set T.
// Case sets of the fused pass kernel: a pass whose fast lists only hold
// PDIAG runs (case ids 0..11), the H-type real GEN1 cases (28, 31, 43, 46,
// 58, 61) and CP5 ops (72..83) gets a kernel (tile_pass_reg<kPassDiagH>)
// whose jump table has only those cases; passes with 1q diagonal gates
// (OP_DIAG ids 12..26) take kPassGen or kPassAll.  Anything outside a set
// would go to the exact path, so the set only affects speed, never results.
// kPassGen: diagonal runs, every 1q case, CX and CX-diagonal ops (QAOA /
// supremacy-style layers).
constexpr int kPassAll = 0, kPassDiagH = 1, kPassGen = 2;
__host__ __device__ constexpr bool case_on(int S, uint32_t c) {
    if (S == kPassDiagH)
        return c <= 11 || c == 28 || c == 31 || c == 43 || c == 46 || c == 58 || c == 61 ||
               (c >= 72 && c <= 83);
    if (S == kPassGen) return c <= 71 || (c >= 84 && c <= 101);
    return true;
}

struct PassDesc {
    uint32_t k;            // tile bits (|T|)
    uint32_t lowbits;      // T ⊇ {0..lowbits-1}
    uint32_t first_group;
    uint32_t ngroups;
    uint32_t first_gate;   // for the smem fallback (k < 4)
    uint32_t ngates;
    uint64_t tmask;        // T as a bit mask over buffer bits
    uint32_t pz_stable;    // all groups pz_stable: an all-(+0) tile is left untouched
    uint32_t kind;         // PASS_TILE, or PASS_SWAPS: a run of disjoint SWAPs as one
                           // bit permutation (perm[b] = image of buffer bit b)
    uint32_t dg0, dg1;     // the stage gates [dg0, dg1) this pass applies
    uint32_t relaxed;      // 0 strict; 1 relaxed, +0-safe units / swap network: in place,
                           // a flag replays the whole window; 2 relaxed with checked
                           // units: out of place, replayed pass by pass
    uint32_t variant;      // kernel case set (host side: kPassAll / kPassDiagH / kPassGen)
    uint32_t wmap;         // register-group thread map: the warp index spells the LOWEST
                           // non-register tile bits (lanes the higher ones), so blocks that
                           // differ only in low bits — the all-(+0) blocks of sparse states —
                           // fall on whole warps, which then skip the group uniformly
    uint8_t perm[48];
    // buffer bits outside T that are fresh (in a basis value) at the pass's
    // start, and their values: a tile whose fixed bits differ from zval on
    // zmask is all +0 and — pz_stable, in place — is never visited
    uint64_t zmask, zval;
    // every buffer bit fresh at the pass's start and its value: an element
    // off zval on fmask is +0 and is zero-filled instead of loaded (the
    // window may not hold it: the decode skips statically-(+0) chunks)
    uint64_t fmask, fval;
    // PASS_TILE: the swap network that followed is fused into the store —
    // out of place, element e written to perm(e) (perm[] as for PASS_SWAPS)
    uint32_t permute;
    // one non-generic register group, no permuted store, >= 32 contiguous low
    // tile bits: registers load / store global memory directly (lanes on the
    // lowest bits: coalesced), no shared-memory tile, no barriers
    uint32_t direct;
};

enum PassKind : uint32_t { PASS_TILE = 0, PASS_SWAPS = 1 };

} // namespace qz
