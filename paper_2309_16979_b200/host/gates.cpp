// gates.cpp — circuit IR helpers; gate_matrix() asks the engine for the exact
// doubles its kernels use (qzc_gate_matrix).
#include "qzsim/gates.hpp"

#include <complex>
#include <cstring>

#include "engine_ctx.hpp"

namespace qzsim {

namespace {
struct KindInfo {
    const char *name;
    uint32_t arity, params;
};
constexpr KindInfo kKinds[] = {
    {"h", 1, 0},  {"x", 1, 0},  {"y", 1, 0},  {"z", 1, 0},  {"s", 1, 0},  {"sdg", 1, 0},
    {"t", 1, 0},  {"tdg", 1, 0}, {"rx", 1, 1}, {"ry", 1, 1}, {"rz", 1, 1}, {"u1", 1, 1},
    {"u2", 1, 2}, {"u3", 1, 3}, {"cx", 2, 0}, {"cz", 2, 0}, {"swap", 2, 0},
};
const KindInfo &info(GateKind k) { return kKinds[static_cast<size_t>(k)]; }
} // namespace

uint32_t gate_arity(GateKind kind) { return info(kind).arity; }
uint32_t gate_param_count(GateKind kind) { return info(kind).params; }
std::string_view gate_name(GateKind kind) { return info(kind).name; }

std::optional<GateKind> gate_kind_from_name(std::string_view name) {
    for (size_t i = 0; i < std::size(kKinds); ++i)
        if (name == kKinds[i].name) return static_cast<GateKind>(i);
    return std::nullopt;
}

GateMatrix gate_matrix(const Gate &gate) {
    if (gate.params.size() < gate_param_count(gate.kind))
        throw Error("gate " + std::string(gate_name(gate.kind)) + " needs " +
                    std::to_string(gate_param_count(gate.kind)) + " params");
    qzc_gate g = b200::to_abi(gate);
    g.nqubits = gate_arity(gate.kind);
    double m[32];
    uint32_t dim = 0;
    b200::check(qzc_gate_matrix(&g, m, &dim));
    GateMatrix out{};
    out.dim = dim;
    for (uint32_t e = 0; e < 16; ++e) out.m[e] = Amplitude(m[2 * e], m[2 * e + 1]);
    return out;
}

GateMatrix adjoint(const GateMatrix &mat) {
    GateMatrix out{};
    out.dim = mat.dim;
    for (uint32_t r = 0; r < mat.dim; ++r)
        for (uint32_t c = 0; c < mat.dim; ++c) out.m[c * mat.dim + r] = std::conj(mat.m[r * mat.dim + c]);
    return out;
}

std::vector<std::string> validate(const Circuit &circuit) {
    std::vector<std::string> errs;
    for (size_t i = 0; i < circuit.gates.size(); ++i) {
        const Gate &g = circuit.gates[i];
        const std::string at = "gate " + std::to_string(i) + " (" + std::string(gate_name(g.kind)) + "): ";
        if (g.qubits.size() != gate_arity(g.kind))
            errs.push_back(at + "expected " + std::to_string(gate_arity(g.kind)) + " qubits, got " +
                           std::to_string(g.qubits.size()));
        if (g.params.size() != gate_param_count(g.kind))
            errs.push_back(at + "expected " + std::to_string(gate_param_count(g.kind)) +
                           " params, got " + std::to_string(g.params.size()));
        for (uint32_t q : g.qubits)
            if (q >= circuit.num_qubits) errs.push_back(at + "qubit " + std::to_string(q) + " out of range");
        if (g.qubits.size() == 2 && g.qubits[0] == g.qubits[1])
            errs.push_back(at + "duplicate qubit " + std::to_string(g.qubits[0]));
    }
    return errs;
}

} // namespace qzsim
