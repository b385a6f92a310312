// qzsim/generators.hpp — benchmark circuits (drop-in for the reference
// header of the same name; same gate lists for the same arguments).
#pragma once

#include "qzsim/gates.hpp"

namespace qzsim {

Circuit make_ghz(uint32_t num_qubits);
Circuit make_qft(uint32_t num_qubits);
Circuit make_random(uint32_t num_qubits, uint32_t depth, uint64_t seed);

} // namespace qzsim
