// oracle.cpp — uncompressed fp64 state for the fidelity report.  The state
// is simulated on the GPU with the engine's exact kernels (qzc_dense_run);
// the overlap is reduced on the host with compensated sums in index order
// (oracle.cpp:79-113 of the reference).
#include "qzsim/oracle.hpp"

#include <cmath>

#include "engine_ctx.hpp"

namespace qzsim {

DenseState make_basis_state(uint32_t num_qubits) {
    if (num_qubits > kOracleLimit)
        throw Error("oracle limit exceeded: n=" + std::to_string(num_qubits) + " > " +
                    std::to_string(kOracleLimit));
    DenseState s{num_qubits, std::vector<Amplitude>(uint64_t(1) << num_qubits)};
    s.amplitudes[0] = Amplitude{1.0, 0.0};
    return s;
}

void apply_gate_dense(DenseState &state, const Gate &gate) {
    if (state.amplitudes.empty()) return;
    const qzc_gate g = b200::to_abi(gate);
    b200::check(qzc_apply_gates_host(b200::ctx(), reinterpret_cast<double *>(state.amplitudes.data()),
                                     state.num_qubits, &g, 1));
}

DenseState simulate_dense(const Circuit &circuit, uint32_t limit) {
    if (circuit.num_qubits > limit)
        throw Error("oracle limit exceeded: n=" + std::to_string(circuit.num_qubits) + " > " +
                    std::to_string(limit));
    if (const auto errs = validate(circuit); !errs.empty()) throw Error("invalid circuit: " + errs.front());
    const std::vector<qzc_gate> abi = b200::to_abi(circuit.gates);
    double *dev = nullptr;
    qzc_context *c = b200::ctx();
    b200::check(qzc_dense_run(c, circuit.num_qubits, abi.data(), abi.size(), &dev));
    DenseState s{circuit.num_qubits, std::vector<Amplitude>(uint64_t(1) << circuit.num_qubits)};
    const int rc = qzc_copy_d2h(c, reinterpret_cast<double *>(s.amplitudes.data()), dev, 0,
                                s.amplitudes.size());
    qzc_synchronize(c);
    qzc_dense_free(c, dev);
    b200::check(rc);
    return s;
}

namespace {
double overlap(const std::vector<Amplitude> &a, const std::vector<Amplitude> &b, uint64_t base,
               KahanSum &re, KahanSum &im, KahanSum &na, KahanSum &nb) {
    for (uint64_t j = 0; j < b.size(); ++j) {
        const Amplitude p = std::conj(a[base + j]) * b[j];
        re.add(p.real());
        im.add(p.imag());
        na.add(std::norm(a[base + j]));
        nb.add(std::norm(b[j]));
    }
    return 0.0;
}
double finish(const KahanSum &re, const KahanSum &im, const KahanSum &na, const KahanSum &nb) {
    if (na.sum == 0.0 || nb.sum == 0.0) return 0.0;
    return (re.sum * re.sum + im.sum * im.sum) / (na.sum * nb.sum);
}
} // namespace

double fidelity(const DenseState &a, const DenseState &b) {
    if (a.num_qubits != b.num_qubits) throw Error("fidelity dimension mismatch");
    KahanSum re, im, na, nb;
    overlap(a.amplitudes, b.amplitudes, 0, re, im, na, nb);
    return finish(re, im, na, nb);
}

double fidelity(const DenseState &a, const ChunkStore &store) {
    if (a.num_qubits != store.num_qubits()) throw Error("fidelity dimension mismatch");
    KahanSum re, im, na, nb;
    for (uint64_t ci = 0; ci < store.chunk_count(); ++ci)
        overlap(a.amplitudes, store.load_chunk(ci), ci * store.chunk_size(), re, im, na, nb);
    return finish(re, im, na, nb);
}

double dense_norm(const DenseState &state) {
    KahanSum acc;
    for (const Amplitude &x : state.amplitudes) acc.add(std::norm(x));
    return acc.sum;
}

} // namespace qzsim
