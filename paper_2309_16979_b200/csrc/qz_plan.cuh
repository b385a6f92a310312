// qz_plan.cuh — host planner (greedy stages over high qubits).
#pragma once

#include <string>
#include <vector>

#include "qz_common.cuh"

namespace qz {

// Reference: planner.hpp:31-71, planner.cpp:22-141.
struct Stage {
    size_t first_gate = 0;
    size_t ngates = 0;
    std::vector<uint32_t> high;  // sorted, padded to min(m-c, n-c)
};

// Empty string = valid (gates.cpp:193-221 subset used by plan()).
std::string validate_gates(uint32_t n, const qzc_gate *gates, uint64_t ngates);

// Throws Failure(QZC_EPLAN) on the reference's preconditions (planner.cpp:51-59).
std::vector<Stage> plan_stages(uint32_t n, const qzc_gate *gates, uint64_t ngates, uint32_t c,
                               uint32_t m);

// Buffer bit of qubit q in a stage (Stage::buffer_bit, planner.cpp:22-28); -1 if unmapped.
int buffer_bit(const Stage &st, uint32_t q, uint32_t c);

} // namespace qz
