// qzsim/oracle.hpp — uncompressed fp64 state for fidelity (drop-in for the
// reference header of the same name).  simulate_dense() runs the same gate
// kernels on an uncompressed GPU buffer (qzc_dense_run) instead of the
// reference's host loop, so it reaches n beyond the reference's 24-qubit cap
// when HBM allows.
#pragma once

#include "qzsim/gates.hpp"
#include "qzsim/store.hpp"

namespace qzsim {

constexpr uint32_t kOracleLimit = 24;

struct DenseState {
    uint32_t num_qubits = 0;
    std::vector<Amplitude> amplitudes;
};

DenseState make_basis_state(uint32_t num_qubits);
void apply_gate_dense(DenseState &state, const Gate &gate);
DenseState simulate_dense(const Circuit &circuit, uint32_t limit = kOracleLimit);
double fidelity(const DenseState &a, const DenseState &b);
double fidelity(const DenseState &a, const ChunkStore &store);
double dense_norm(const DenseState &state);

} // namespace qzsim
