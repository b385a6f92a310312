// kernels.cpp — qzsim gate application on the GPU (qzc_apply_*_host).
#include "qzsim/kernels.hpp"

#include <cstring>

#include "engine_ctx.hpp"

namespace qzsim {

namespace {

uint32_t log2_exact(uint64_t n) {
    if (n == 0 || (n & (n - 1))) throw Error("buffer length must be a power of two");
    uint32_t b = 0;
    while ((uint64_t(1) << b) < n) ++b;
    return b;
}

qzc_matrix_gate as_matrix_gate(const GateMatrix &mat, uint32_t b0, uint32_t b1) {
    qzc_matrix_gate g;
    std::memset(&g, 0, sizeof g);
    g.dim = mat.dim;
    g.qubits[0] = b0;
    g.qubits[1] = b1;
    for (uint32_t e = 0; e < mat.dim * mat.dim; ++e) {
        g.m[2 * e] = mat.m[e].real();
        g.m[2 * e + 1] = mat.m[e].imag();
    }
    return g;
}

} // namespace

void apply_single_qubit(std::span<Amplitude> buffer, uint32_t bit, const GateMatrix &mat,
                        uint64_t pair_begin, uint64_t pair_end) {
    const qzc_matrix_gate g = as_matrix_gate(mat, bit, 0);
    b200::check(qzc_apply_matrix_range_host(b200::ctx(), reinterpret_cast<double *>(buffer.data()),
                                            log2_exact(buffer.size()), &g, pair_begin, pair_end));
}

void apply_two_qubit(std::span<Amplitude> buffer, uint32_t bit0, uint32_t bit1, const GateMatrix &mat,
                     uint64_t group_begin, uint64_t group_end) {
    const qzc_matrix_gate g = as_matrix_gate(mat, bit0, bit1);
    b200::check(qzc_apply_matrix_range_host(b200::ctx(), reinterpret_cast<double *>(buffer.data()),
                                            log2_exact(buffer.size()), &g, group_begin, group_end));
}

void apply_gate(std::span<Amplitude> buffer, const Gate &gate) {
    apply_gates(buffer, std::span<const Gate>(&gate, 1));
}

void apply_gates(std::span<Amplitude> buffer, std::span<const Gate> gates) {
    if (gates.empty()) return;
    const uint32_t nbits = log2_exact(buffer.size());
    const std::vector<qzc_gate> abi = b200::to_abi(gates);
    b200::check(qzc_apply_gates_host(b200::ctx(), reinterpret_cast<double *>(buffer.data()), nbits, abi.data(),
                                     abi.size()));
}

} // namespace qzsim
