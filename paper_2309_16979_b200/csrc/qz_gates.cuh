// qz_gates.cuh — gate matrices, fused gate passes and the tile kernel API.
#pragma once

#include <memory>
#include <vector>

#include "qz_common.cuh"
#include "qz_gate_types.cuh"

namespace qz {

// One gate with its host-computed matrix (gates.cpp:114-182) on buffer bits.
struct DevGate {
    uint32_t nq;       // 1 or 2
    uint32_t b0, b1;   // buffer bits (b0 = first listed = matrix high bit)
    uint32_t dim;
    uint64_t kinds;    // 4 bits per entry, row-major
    uint32_t sgn;      // 2 bits per entry: bit 2e = sign(re), 2e+1 = sign(im)
    uint32_t op;       // GateOp: structure used by the zero-free fast path
    double2 m[16];     // row-major, dim = 2 or 4
};

struct GatePlan {
    std::vector<PassDesc> passes;
    std::vector<GroupDesc> groups;
    std::vector<TileGate> gates;
};

// Host: matrix for a qzc_gate, bit-identical to qzsim::gate_matrix.
void gate_matrix_host(const qzc_gate &g, double2 *m, uint32_t *dim);
uint32_t gate_arity(uint32_t kind);
uint32_t gate_nparams(uint32_t kind);

// Host: greedy in-order fusion of gates (already on buffer bits) into passes
// over a buffer of 2^nbits amplitudes with tiles of at most 2^kmax.
// relax: diagonal units do not need their qubits in the tile set (OP_PDIAG);
// such a plan can raise the replay flag and must then be replayed strictly
// from the same input (see run_passes).
// fresh: buffer bits in a basis value at the start (see Fresh): tiles leave
// them out where no gate needs them, and tiles on their +0 side are skipped.
struct Fresh;
// fuse_perm: a swap network right after a tile pass becomes that pass's
// permuted out-of-place store (PassDesc::permute) when its tile can hold the
// network's images of the low bits.
GatePlan build_passes(const std::vector<DevGate> &gates, uint32_t nbits, uint32_t kmax,
                      bool fuse, int relax_level = 0, const Fresh *fresh = nullptr, bool fuse_perm = false);

DevGate make_dev_gate(const qzc_gate &g);
DevGate make_dev_gate_matrix(const double2 *m, uint32_t dim, uint32_t b0, uint32_t b1);

// Device-resident copy of a GatePlan.
struct DevPlan {
    TileGate *gates = nullptr;
    GroupDesc *groups = nullptr;
    size_t ngates = 0, ngroups = 0;
    std::vector<PassDesc> host_passes;
    bool relaxed = false;   // some pass may raise the replay flag
    size_t cap_gates = 0, cap_groups = 0;   // device capacity (grow-only reuse)
    // strict replay plan: passes [replay_range[p].first, .second) of `replay`
    // re-apply relaxed pass p's gates with every qubit in the tile
    std::vector<std::pair<uint32_t, uint32_t>> replay_range;
    // per pass: its runtime-specialised kernel (qz_jit.cuh) or null
    std::vector<std::shared_ptr<struct JitPass>> jit;
};
// Stream-ordered upload into `out`, reusing its device buffers when they are
// large enough (no allocator calls on the steady-state stage loop).
// The plan's passes with their launch fields set (kernel variant, thread map).
std::vector<PassDesc> launch_passes(const GatePlan &plan);

// Buffer bits statically in a basis value ("fresh": no non-diagonal gate has
// touched them since |0...0>): every amplitude whose bit b (in mask) differs
// from val's bit b is +0.  The runtime-specialised passes skip products on
// registers that are +0 this way (qz_jit.cu).
struct Fresh {
    uint64_t mask = 0, val = 0;
};
bool gate_diagonal(const DevGate &g);
// every row maps an all-(+0) input to +0 (zeros keep their sign)
bool gate_keeps_pos_zero(const DevGate &g);
// Fresh state after gates [g0, g1): a non-diagonal gate ends its qubits'
// freshness, a gate that may turn +0 into -0 ends all of it.
Fresh fresh_after(const std::vector<DevGate> &dg, size_t g0, size_t g1, Fresh f);
Fresh fresh_after_gate(Fresh f, const DevGate &g);
// one gate (buffer bits b0, b1): X / CX / SWAP permute basis states and keep
// fresh bits fresh (values updated); other non-diagonal gates end them
Fresh fresh_gate(Fresh f, uint32_t op, uint32_t nq, uint32_t b0, uint32_t b1, uint64_t kinds, bool diagonal);
// jit_bits > 0: also queue runtime-specialised kernels for the plan's
// full-tile passes over 2^jit_bits windows (used once built).
// (fresh: per pass, the fresh state at its start; empty = none)
void upload_plan(const GatePlan &plan, DevPlan &out, cudaStream_t s, uint32_t jit_bits = 0,
                 const std::vector<Fresh> &fresh = {});
void free_plan(DevPlan &p);   // releases the device buffers

// Per-chunk-slot "may be nonzero" words of a window (slot = amplitude >> cbits):
// 0 = known all-(+0) (from the decode index), so in-place passes whose groups
// keep all-(+0) blocks fixed skip such tiles without loading them; every
// processed tile marks its slots (keeping the zero-slot count exact, and a
// pass that starts with no zero slot does no map work); a swap pass resets it.
struct NzMap {
    uint32_t *slot = nullptr;   // nslots words + the zero-slot count
    uint32_t cbits = 0;
};

// Launch every pass of a strict `plan` in place over buf (2^nbits
// amplitudes).  Returns the number of kernel launches.
uint64_t run_passes(const DevPlan &plan, double2 *buf, uint32_t nbits, cudaStream_t s,
                    const uint32_t *cond = nullptr, NzMap nz = {});
// Count a replay and clear the flag (stream-ordered).
void flag_done(uint32_t *flag, uint64_t *replays, cudaStream_t s);

// Relaxed plan (built with relax = true) and its strict replay plan (upload_replay):
// relaxed passes run out of place, buf -> alt, and raise *flag when a tile
// cannot be evaluated exactly (a zero / -0 where partners outside the tile
// would decide the bytes, or -0 under a swap network); the pass is then
// re-applied from its untouched input by the strict sub-plan (launches that
// are no-ops unless *flag), and *flag is cleared (replays counted in
// *replays).  Returns the buffer holding the result (buf or alt).
// Passes with relaxed == 1 run in place and raise *win_flag (sticky; the
// caller replays the whole window from its payloads when set).
double2 *run_relaxed(const DevPlan &plan, const DevPlan &replay, double2 *buf, double2 *alt,
                     uint32_t nbits, cudaStream_t s, uint32_t *flag, uint32_t *win_flag,
                     uint64_t *replays, bool force_replay, uint64_t &launches, NzMap nz = {});

// Strict sub-plans of every relaxed pass of `relaxed`, concatenated into
// `out` (ranges recorded in relaxed_dev.replay_range).
void upload_replay(const std::vector<DevGate> &gates, uint32_t nbits, uint32_t kmax,
                   DevPlan &relaxed_dev, DevPlan &out, cudaStream_t s);
void dump_debug_counters();

} // namespace qz
