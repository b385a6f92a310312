// qzsim/kernels.hpp — gate application on a dense buffer (drop-in for the
// reference header of the same name).  Runs the fused sm_100a gate passes
// (qzc_apply_gates_host); results are bit-identical to the reference loops.
#pragma once

#include <span>

#include "qzsim/gates.hpp"

namespace qzsim {

/// One-qubit matrix on buffer bit `bit`, pair range [pair_begin, pair_end).
void apply_single_qubit(std::span<Amplitude> buffer, uint32_t bit, const GateMatrix &mat,
                        uint64_t pair_begin, uint64_t pair_end);

/// Two-qubit matrix; bit0 is the first listed qubit (high matrix bit).
void apply_two_qubit(std::span<Amplitude> buffer, uint32_t bit0, uint32_t bit1,
                     const GateMatrix &mat, uint64_t group_begin, uint64_t group_end);

void apply_gate(std::span<Amplitude> buffer, const Gate &gate);
void apply_gates(std::span<Amplitude> buffer, std::span<const Gate> gates);

} // namespace qzsim
