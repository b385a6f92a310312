// qz_jit.cuh — runtime-specialised fused gate passes.
//
// A fused pass's fast-path op list is known on the host when the stage is
// planned; the AOT kernel interprets it (one switch per op, descriptors read
// from global memory per op and thread).  For large windows the engine also
// builds the pass as its own kernel: the same device code (qz_gates_dev.cuh),
// with the op sequence as straight-line calls and the op descriptors as
// compile-time constants, compiled for sm_100a by NVRTC on a host thread pool
// while earlier work runs, cached by source.  Results are identical by
// construction (the same per-op device functions in the same order); only
// dispatch and descriptor loads disappear.  QZ_JIT=0 disables it,
// QZ_JIT_MIN_BITS (default 24) sets the smallest window it is used for.
#pragma once

#include <memory>
#include <string>

#include "qz_gates.cuh"

namespace qz {

struct JitPass;

// Queue the specialised kernel for pass `pd` of `plan` over 2^nbits windows;
// nullptr when the JIT is off or the pass does not qualify.
// fresh: the pass's fresh buffer bits at its start (registers statically +0
// skip their products).
std::shared_ptr<JitPass> jit_request(const GatePlan &plan, const PassDesc &pd, uint32_t nbits,
                                     Fresh fresh = {});

// The kernel is built (or failed: then false).  Never waits unless
// QZ_JIT_SYNC=1 — until a compile finishes its pass runs the AOT kernel.
bool jit_ready(JitPass &j);

// Block until every queued compile has finished (and, with load, load the
// kernels into the current context); returns how many built.
size_t jit_wait_all(bool load = false);

// Launch it with tile_pass_reg's arguments; false when it could not be built
// (the caller then launches the AOT kernel — same results).
bool jit_launch(JitPass &j, unsigned grid, unsigned threads, size_t smem, cudaStream_t s, void **args);

// The generated source of a pass (tests / inspection).
std::string jit_source(const GatePlan &plan, const PassDesc &pd, Fresh fresh = {});

} // namespace qz
