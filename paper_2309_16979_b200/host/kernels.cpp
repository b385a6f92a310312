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

// Pairs/groups are independent, so a sub-range update = the full update
// restricted to the range; apply on a copy and write back only the range.
template <class IndexFn>
void apply_range(std::span<Amplitude> buffer, const qzc_matrix_gate &g, uint64_t begin, uint64_t end,
                 uint64_t total, IndexFn indices) {
    const uint32_t nbits = log2_exact(buffer.size());
    if (begin == 0 && end == total) {
        b200::check(qzc_apply_matrices_host(b200::ctx(), reinterpret_cast<double *>(buffer.data()), nbits,
                                            &g, 1));
        return;
    }
    std::vector<Amplitude> work(buffer.begin(), buffer.end());
    b200::check(qzc_apply_matrices_host(b200::ctx(), reinterpret_cast<double *>(work.data()), nbits, &g, 1));
    for (uint64_t p = begin; p < end; ++p) indices(p, [&](uint64_t i) { buffer[i] = work[i]; });
}

} // namespace

void apply_single_qubit(std::span<Amplitude> buffer, uint32_t bit, const GateMatrix &mat,
                        uint64_t pair_begin, uint64_t pair_end) {
    const qzc_matrix_gate g = as_matrix_gate(mat, bit, 0);
    apply_range(buffer, g, pair_begin, pair_end, buffer.size() / 2, [&](uint64_t p, auto put) {
        const uint64_t i = insert_zero_bit(p, bit);
        put(i);
        put(i | (uint64_t(1) << bit));
    });
}

void apply_two_qubit(std::span<Amplitude> buffer, uint32_t bit0, uint32_t bit1, const GateMatrix &mat,
                     uint64_t group_begin, uint64_t group_end) {
    const qzc_matrix_gate g = as_matrix_gate(mat, bit0, bit1);
    const uint32_t lo = std::min(bit0, bit1), hi = std::max(bit0, bit1);
    apply_range(buffer, g, group_begin, group_end, buffer.size() / 4, [&](uint64_t q, auto put) {
        const uint64_t b = insert_zero_bit(insert_zero_bit(q, lo), hi);
        const uint64_t s0 = uint64_t(1) << bit0, s1 = uint64_t(1) << bit1;
        put(b);
        put(b | s1);
        put(b | s0);
        put(b | s0 | s1);
    });
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
