// qz_plan.cpp — host planner for the staged pipeline.
//
// Semantics follow planner.cpp:46-96: a gate joins the open stage while the
// union of its qubits >= c stays within m - c; otherwise the stage closes,
// is padded with the smallest unused qubits >= c (planner.cpp:32-42), and a
// new stage opens with this gate.  Batch membership (planner.cpp:105-129) is
// evaluated on the device from the stage's bit masks (qz_codec.cu).
#include <algorithm>
#include <set>

#include "qz_gates.cuh"
#include "qz_plan.cuh"

namespace qz {

std::string validate_gates(uint32_t n, const qzc_gate *gates, uint64_t ngates) {
    for (uint64_t i = 0; i < ngates; ++i) {
        const qzc_gate &g = gates[i];
        const bool ok = g.kind <= QZC_SWAP && g.nqubits == gate_arity(g.kind) && g.qubits[0] < n &&
                        (g.nqubits == 1 || (g.qubits[1] < n && g.qubits[0] != g.qubits[1]));
        if (ok) continue;   // message only on the failing gate (no per-gate strings)
        const std::string where = "gate " + std::to_string(i) + ": ";
        if (g.kind > QZC_SWAP) return where + "unknown gate kind";
        if (g.nqubits != gate_arity(g.kind))
            return where + "expected " + std::to_string(gate_arity(g.kind)) + " qubits, got " +
                   std::to_string(g.nqubits);
        for (uint32_t k = 0; k < g.nqubits; ++k)
            if (g.qubits[k] >= n) return where + "qubit " + std::to_string(g.qubits[k]) + " out of range";
        if (g.nqubits == 2 && g.qubits[0] == g.qubits[1])
            return where + "duplicate qubit " + std::to_string(g.qubits[0]);
    }
    return {};
}

std::vector<Stage> plan_stages(uint32_t n, const qzc_gate *gates, uint64_t ngates, uint32_t c,
                               uint32_t m) {
    if (c < 1) throw Failure(QZC_EPLAN, "chunk qubits must be >= 1");
    if (m < c + 2)
        throw Failure(QZC_EPLAN, "batch qubits must be >= chunk qubits + 2, got m=" +
                                     std::to_string(m) + ", c=" + std::to_string(c));
    if (m > n)
        throw Failure(QZC_EPLAN, "batch qubits exceed circuit qubits: m=" + std::to_string(m) +
                                     ", n=" + std::to_string(n));
    if (std::string e = validate_gates(n, gates, ngates); !e.empty())
        throw Failure(QZC_EPLAN, "invalid circuit: " + e);

    const uint32_t capacity = m - c, target = std::min(m - c, n - c);
    std::vector<Stage> out;
    Stage cur;
    if (n <= 64) {
        // the open stage's qubits >= c as a bit mask (one word: no per-gate set copies)
        uint64_t high = 0;
        auto close = [&]() {
            if (cur.ngates == 0) return;
            for (uint32_t q = c; uint32_t(__builtin_popcountll(high)) < target && q < n; ++q)
                high |= uint64_t(1) << q;
            for (uint64_t h = high; h; h &= h - 1) cur.high.push_back(uint32_t(__builtin_ctzll(h)));
            out.push_back(cur);
            cur = Stage{};
            high = 0;
        };
        for (uint64_t i = 0; i < ngates; ++i) {
            uint64_t gm = 0;
            for (uint32_t k = 0; k < gates[i].nqubits; ++k)
                if (gates[i].qubits[k] >= c) gm |= uint64_t(1) << gates[i].qubits[k];
            if (uint32_t(__builtin_popcountll(high | gm)) > capacity) {
                close();
                high = gm;
            } else {
                high |= gm;
            }
            if (cur.ngates == 0) cur.first_gate = i;
            ++cur.ngates;
        }
        close();
        return out;
    }
    std::set<uint32_t> high;
    auto close = [&]() {
        if (cur.ngates == 0) return;
        for (uint32_t q = c; high.size() < target && q < n; ++q) high.insert(q);
        cur.high.assign(high.begin(), high.end());
        out.push_back(cur);
        cur = Stage{};
        high.clear();
    };
    for (uint64_t i = 0; i < ngates; ++i) {
        std::set<uint32_t> merged = high;
        for (uint32_t k = 0; k < gates[i].nqubits; ++k)
            if (gates[i].qubits[k] >= c) merged.insert(gates[i].qubits[k]);
        if (merged.size() > capacity) {
            close();
            for (uint32_t k = 0; k < gates[i].nqubits; ++k)
                if (gates[i].qubits[k] >= c) high.insert(gates[i].qubits[k]);
        } else {
            high.swap(merged);
        }
        if (cur.ngates == 0) cur.first_gate = i;
        ++cur.ngates;
    }
    close();
    return out;
}

int buffer_bit(const Stage &st, uint32_t q, uint32_t c) {
    if (q < c) return int(q);
    auto it = std::lower_bound(st.high.begin(), st.high.end(), q);
    if (it == st.high.end() || *it != q) return -1;
    return int(c + (it - st.high.begin()));
}

} // namespace qz
