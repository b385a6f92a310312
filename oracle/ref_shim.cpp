// ref_shim.cpp — extern "C" bindings over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled together with the reference
// sources straight from /root/reference/proj/src (oracle/Makefile) into
// oracle/_ref/libqzref.so, which is never committed.  It lets the Python
// tests and bench.py's reference arm call the reference's own public API
// (qzsim::compress / decompress / apply_gates / gate_matrix / plan / run)
// with plain C types.  Nothing here reimplements reference behaviour.
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>

#include "qzsim/codec.hpp"
#include "qzsim/generators.hpp"
#include "qzsim/kernels.hpp"
#include "qzsim/pipeline.hpp"
#include "qzsim/planner.hpp"
#include "qzsim/qasm.hpp"

#include "../include/qzcuda.h"

using namespace qzsim;

namespace {

thread_local std::string g_err;

Gate to_gate(const qzc_gate &g) {
    Gate out{static_cast<GateKind>(g.kind), {}, {}};
    for (uint32_t k = 0; k < g.nqubits; ++k) out.qubits.push_back(g.qubits[k]);
    for (uint32_t k = 0; k < gate_param_count(out.kind); ++k)
        out.params.push_back(g.params[k]);
    return out;
}

qzc_gate from_gate(const Gate &g) {
    qzc_gate out;
    std::memset(&out, 0, sizeof out);
    out.kind = static_cast<uint32_t>(g.kind);
    out.nqubits = static_cast<uint32_t>(g.qubits.size());
    for (size_t k = 0; k < g.qubits.size() && k < 2; ++k) out.qubits[k] = g.qubits[k];
    for (size_t k = 0; k < g.params.size() && k < 3; ++k) out.params[k] = g.params[k];
    return out;
}

Circuit to_circuit(uint32_t n, const qzc_gate *gates, uint64_t ngates) {
    Circuit c;
    c.num_qubits = n;
    for (uint64_t i = 0; i < ngates; ++i) c.gates.push_back(to_gate(gates[i]));
    return c;
}

uint64_t export_gates(const Circuit &c, qzc_gate *out, uint64_t cap) {
    for (uint64_t i = 0; i < c.gates.size() && i < cap; ++i) out[i] = from_gate(c.gates[i]);
    return c.gates.size();
}

} // namespace

extern "C" {

const char *qzref_last_error(void) { return g_err.c_str(); }

int qzref_gate_matrix(const qzc_gate *g, double *m, uint32_t *dim) {
    try {
        GateMatrix mat = gate_matrix(to_gate(*g));
        *dim = mat.dim;
        std::memcpy(m, mat.m.data(), sizeof(double) * 32);
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

int64_t qzref_compress(const double *amps, uint64_t n, double eb,
                       const uint64_t *forced, uint64_t nforced, uint8_t *out,
                       uint64_t cap, uint32_t *crc) {
    try {
        std::span<const Amplitude> a(reinterpret_cast<const Amplitude *>(amps), n);
        CompressedChunk cc = compress(0, a, eb, std::span<const uint64_t>(forced, nforced));
        if (cc.payload.size() > cap) {
            g_err = "capacity";
            return -4;
        }
        std::memcpy(out, cc.payload.data(), cc.payload.size());
        *crc = cc.checksum;
        return static_cast<int64_t>(cc.payload.size());
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

int qzref_decompress(const uint8_t *p, uint64_t len, uint32_t crc, uint64_t n,
                     uint64_t chunk_index, double *out) {
    try {
        CompressedChunk cc;
        cc.chunk_index = chunk_index;
        cc.payload.assign(p, p + len);
        cc.checksum = crc;
        cc.element_count = static_cast<uint32_t>(n);
        cc.codec_id = len ? static_cast<CodecId>(p[0]) : CodecId::LosslessRLE;
        if (len >= 9) std::memcpy(&cc.error_bound, p + 1, 8);
        std::vector<Amplitude> v = decompress(cc);
        std::memcpy(out, v.data(), v.size() * sizeof(Amplitude));
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

int qzref_apply_gates(double *amps, uint64_t count, const qzc_gate *gates,
                      uint64_t ngates) {
    try {
        std::span<Amplitude> buf(reinterpret_cast<Amplitude *>(amps), count);
        for (uint64_t i = 0; i < ngates; ++i) apply_gate(buf, to_gate(gates[i]));
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

uint64_t qzref_make_qft(uint32_t n, qzc_gate *out, uint64_t cap) {
    return export_gates(make_qft(n), out, cap);
}
uint64_t qzref_make_ghz(uint32_t n, qzc_gate *out, uint64_t cap) {
    return export_gates(make_ghz(n), out, cap);
}
uint64_t qzref_make_random(uint32_t n, uint32_t depth, uint64_t seed,
                           qzc_gate *out, uint64_t cap) {
    return export_gates(make_random(n, depth, seed), out, cap);
}

// plan(): stage count, per-stage gate counts and padded high sets
// (high_out: stages x 64 entries, nhigh_out: per stage).
int qzref_plan(uint32_t n, const qzc_gate *gates, uint64_t ngates, uint32_t c,
               uint32_t m, uint64_t *nstages, uint64_t *stage_ngates,
               uint32_t *nhigh_out, uint32_t *high_out, uint64_t cap) {
    try {
        ExecutionPlan p = plan(to_circuit(n, gates, ngates), c, m);
        *nstages = p.stages.size();
        for (size_t s = 0; s < p.stages.size() && s < cap; ++s) {
            stage_ngates[s] = p.stages[s].gates.size();
            nhigh_out[s] = static_cast<uint32_t>(p.stages[s].high_set.size());
            for (size_t k = 0; k < p.stages[s].high_set.size() && k < 64; ++k)
                high_out[s * 64 + k] = p.stages[s].high_set[k];
        }
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

struct qzref_result {
    uint64_t digest;
    double norm;
    double wall_seconds;
    double ratio;
    uint64_t current_bytes;
    uint64_t peak_bytes;
    uint64_t stages;
    uint64_t total_payload;
    double fidelity; // -1 when absent
};

// qzsim::run with the given knobs.  workers = 0 → hardware_concurrency.
// strategy: 0 sync, 1 per-element, 2 buffered.  payload_out/sizes_out
// optional: final store in chunk order.
int qzref_run(uint32_t n, const qzc_gate *gates, uint64_t ngates, uint32_t c,
              uint32_t m, double eb, uint32_t workers, uint32_t depth,
              uint32_t strategy, uint32_t oracle_limit, qzref_result *res,
              uint8_t *payload_out, uint64_t cap, uint32_t *sizes_out) {
    try {
        if (workers == 0) workers = std::max(1u, std::thread::hardware_concurrency());
        PipelineConfig cfg;
        cfg.chunk_qubits = c;
        cfg.batch_qubits = m;
        cfg.error_bound = eb;
        cfg.strategy = static_cast<Strategy>(strategy);
        cfg.decompress_workers = workers;
        cfg.recompress_workers = workers;
        cfg.kernel_workers = workers;
        cfg.pipeline_depth = depth;
        cfg.oracle_limit = oracle_limit;
        auto [store, rep] = run(to_circuit(n, gates, ngates), cfg);
        res->digest = rep.digest;
        res->norm = rep.norm;
        res->wall_seconds = rep.wall_seconds;
        res->ratio = rep.footprint.ratio;
        res->current_bytes = rep.footprint.current_bytes;
        res->peak_bytes = rep.footprint.peak_bytes;
        res->stages = rep.stage_batch_counts.size();
        res->fidelity = rep.fidelity ? *rep.fidelity : -1.0;
        uint64_t total = 0;
        // Payload bytes are exported through the reference's own QZST
        // save() format (store.cpp:152-175).
        if (payload_out || sizes_out) {
            std::string path = "/tmp/qzref_export_" + std::to_string(::getpid()) + ".qzst";
            store.save(path);
            FILE *f = std::fopen(path.c_str(), "rb");
            if (!f) throw Error("export failed");
            char magic[4];
            uint32_t nn, cc;
            double ebb;
            if (std::fread(magic, 1, 4, f) != 4 || std::fread(&nn, 4, 1, f) != 1 ||
                std::fread(&cc, 4, 1, f) != 1 || std::fread(&ebb, 8, 1, f) != 1)
                throw Error("export read failed");
            for (uint64_t ci = 0; ci < store.chunk_count(); ++ci) {
                uint32_t len, crc;
                if (std::fread(&len, 4, 1, f) != 1 || std::fread(&crc, 4, 1, f) != 1)
                    throw Error("export read failed");
                if (payload_out) {
                    if (total + len > cap) throw Error("export capacity");
                    if (std::fread(payload_out + total, 1, len, f) != len)
                        throw Error("export read failed");
                } else {
                    std::fseek(f, len, SEEK_CUR);
                }
                if (sizes_out) sizes_out[ci] = len;
                total += len;
            }
            std::fclose(f);
            std::remove(path.c_str());
        }
        res->total_payload = total;
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

// pretty_print(circuit) for exchanging circuits as QASM (qasm.cpp:304-308).
int64_t qzref_pretty_print(uint32_t n, const qzc_gate *gates, uint64_t ngates,
                           char *out, uint64_t cap) {
    std::string s = pretty_print(to_circuit(n, gates, ngates));
    if (s.size() + 1 > cap) return -static_cast<int64_t>(s.size() + 1);
    std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<int64_t>(s.size());
}

} // extern "C"
