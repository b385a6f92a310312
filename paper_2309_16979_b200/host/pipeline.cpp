// pipeline.cpp — qzsim::run on the B200 engine.
//
// Same contract as the reference (pipeline.cpp:128-314): validate, plan,
// start from |0...0>, one codec round trip per chunk per stage, report.  The
// stage loop itself is qzc_sim_run: the compressed store stays in HBM, every
// window of whole batches is decoded, updated by fused gate passes and
// re-encoded on the GPU.  The final payloads are exported to a host
// ChunkStore, byte-identical to the reference's (same digest).
#include "qzsim/pipeline.hpp"

#include <cmath>
#include <cstdio>
#include <sstream>

#include "engine_ctx.hpp"
#include "qzsim/kernels.hpp"
#include "qzsim/oracle.hpp"

namespace qzsim {

namespace {

void check_config(const PipelineConfig &cfg, uint32_t num_qubits) {
    if (!(cfg.host_fraction >= 0.0 && cfg.host_fraction <= 1.0))
        throw Error("host fraction must lie in [0, 1]");
    if (cfg.pipeline_depth < 1) throw Error("pipeline depth must be >= 1");
    if (cfg.decompress_workers < 1 || cfg.recompress_workers < 1 || cfg.kernel_workers < 1)
        throw Error("worker counts must be >= 1");
    if (!(cfg.error_bound >= 0.0) || !std::isfinite(cfg.error_bound))
        throw Error("error bound must be finite and non-negative");
    if (num_qubits == 0) throw Error("circuit has no qubits");
}

struct Sim {
    qzc_sim *h = nullptr;
    ~Sim() {
        if (h) qzc_sim_destroy(h);
    }
};

} // namespace

std::pair<ChunkStore, SimulationReport> run(const Circuit &circuit, const PipelineConfig &cfg) {
    check_config(cfg, circuit.num_qubits);
    if (const auto errs = validate(circuit); !errs.empty()) throw Error("invalid circuit: " + errs.front());
    const uint32_t n = circuit.num_qubits, c = cfg.chunk_qubits;
    const ExecutionPlan p = plan(circuit, c, cfg.batch_qubits);
    if (c < 1 || c > n)
        throw StoreError("chunk qubits must satisfy 1 <= c <= n, got c=" + std::to_string(c) +
                         ", n=" + std::to_string(n));
    if (n > ChunkStore::kMaxQubits) throw StoreError("qubit count exceeds configured address width (40)");

    qzc_context *ctx = b200::ctx();
    qzc_sim_config sc{};
    sc.num_qubits = n;
    sc.chunk_qubits = c;
    sc.batch_qubits = cfg.batch_qubits;
    sc.error_bound = cfg.error_bound;
    sc.fuse_gates = 1;
    Sim sim;
    b200::check(qzc_sim_create(ctx, &sc, &sim.h));
    b200::check(qzc_sim_init_basis(sim.h));
    const std::vector<qzc_gate> abi = b200::to_abi(circuit.gates);
    Timer wall;
    try {
        b200::check(qzc_sim_run(sim.h, abi.data(), abi.size()));
    } catch (const Error &e) {
        throw Error(e.what());
    }
    double run_seconds = wall.seconds();

    qzc_sim_stats st{};
    b200::check(qzc_sim_stats_get(sim.h, &st));
    uint64_t total = 0;
    b200::check(qzc_sim_payload_bytes(sim.h, &total));
    const uint64_t nchunks = uint64_t(1) << (n - c);
    std::vector<uint8_t> payloads(total + 1);
    std::vector<uint32_t> sizes(nchunks), crcs(nchunks);
    b200::check(qzc_sim_export(sim.h, payloads.data(), payloads.size(), sizes.data(), crcs.data()));
    ChunkStore store = ChunkStore::from_payloads(n, c, cfg.error_bound, payloads.data(), sizes.data(),
                                                 crcs.data(), st.peak_bytes);

    SimulationReport rep;
    rep.config = cfg;
    for (const Stage &s : p.stages) rep.stage_batch_counts.push_back(batch_count(s, n, c));
    if (cfg.renormalize) {
        Timer t;
        const double nn = store_norm(store);
        if (nn > 0.0) {
            const double scale = 1.0 / std::sqrt(nn);
            for (uint64_t ci = 0; ci < store.chunk_count(); ++ci) {
                std::vector<Amplitude> v = store.load_chunk(ci);
                for (Amplitude &a : v) a *= scale;
                store.store_chunk(ci, v);
            }
        }
        run_seconds += t.seconds();
    }
    rep.wall_seconds = run_seconds;
    rep.phases.decompress = st.decode_seconds;
    rep.phases.kernel = st.gate_seconds;
    rep.phases.recompress = st.encode_seconds;
    rep.phases.h2d = st.h2d_seconds;
    rep.phases.d2h = st.d2h_seconds;
    rep.transfer.kernel_seconds = st.gate_seconds;
    rep.transfer.h2d_seconds = st.h2d_seconds;
    rep.transfer.d2h_seconds = st.d2h_seconds;
    rep.transfer.bytes_moved = 0;  // the store never leaves HBM during the run
    rep.overlap_efficiency = rep.wall_seconds > 0 ? rep.phases.kernel / rep.wall_seconds : 0.0;
    rep.transient_peak_bytes = 0;  // no host-side decompressed batches on this path
    rep.chunk_decompress_count = st.chunk_decompress_count;
    rep.chunk_recompress_count = st.chunk_recompress_count;
    rep.footprint = store.footprint();
    double norm = 0.0;
    b200::check(qzc_sim_norm(sim.h, &norm));
    rep.norm = cfg.renormalize ? store_norm(store) : norm;
    rep.digest = store.digest();
    if (n <= cfg.oracle_limit && n <= kOracleLimit) {
        const DenseState ref = simulate_dense(circuit);
        rep.fidelity = fidelity(ref, store);
    }
    return {std::move(store), std::move(rep)};
}

void host_apply_batch(ChunkStore &store, const Stage &stage, const BatchDescriptor &batch,
                      const HostPhaseClocks &clocks) {
    const uint64_t len = store.chunk_size();
    std::vector<Amplitude> buf(batch.chunk_indices.size() * len);
    {
        Timer t;
        for (size_t j = 0; j < batch.chunk_indices.size(); ++j) {
            const std::vector<Amplitude> v = store.load_chunk(batch.chunk_indices[j]);
            std::copy(v.begin(), v.end(), buf.begin() + j * len);
        }
        if (clocks.decompress) clocks.decompress->add(t.seconds());
    }
    {
        Timer t;
        std::vector<Gate> remapped;
        for (const Gate &g : stage.gates) remapped.push_back(remap_gate(g, stage, store.chunk_qubits()));
        apply_gates(buf, remapped);
        if (clocks.host_apply) clocks.host_apply->add(t.seconds());
    }
    {
        Timer t;
        for (size_t j = 0; j < batch.chunk_indices.size(); ++j)
            store.store_chunk(batch.chunk_indices[j], std::span<const Amplitude>(buf.data() + j * len, len));
        if (clocks.recompress) clocks.recompress->add(t.seconds());
    }
}

double store_norm(const ChunkStore &store) {
    // one batched GPU decode of every chunk, then the reference's compensated
    // sum in chunk order (pipeline.cpp:119-126)
    const uint64_t count = store.chunk_count(), len = store.chunk_size();
    std::vector<uint8_t> blob;
    std::vector<uint64_t> offs(count);
    std::vector<uint32_t> sizes(count), crcs(count);
    for (uint64_t i = 0; i < count; ++i) {
        const CompressedChunk &c = store.chunk(i);
        offs[i] = blob.size();
        sizes[i] = static_cast<uint32_t>(c.payload.size());
        crcs[i] = c.checksum;
        blob.insert(blob.end(), c.payload.begin(), c.payload.end());
    }
    std::vector<Amplitude> all(count * len);
    b200::check(qzc_decompress_host(b200::ctx(), blob.data(), offs.data(), sizes.data(), crcs.data(), count,
                                    len, 0, reinterpret_cast<double *>(all.data())));
    KahanSum acc;
    for (const Amplitude &a : all) acc.add(std::norm(a));
    return acc.sum;
}

namespace {
std::string num(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}
} // namespace

std::string report_to_json(const SimulationReport &r) {
    std::ostringstream o;
    o << "{\n  \"norm\": " << num(r.norm) << ",\n";
    if (r.fidelity) o << "  \"fidelity\": " << num(*r.fidelity) << ",\n";
    o << "  \"phase_seconds\": {\"decompress\": " << num(r.phases.decompress) << ", \"h2d\": "
      << num(r.phases.h2d) << ", \"kernel\": " << num(r.phases.kernel) << ", \"d2h\": " << num(r.phases.d2h)
      << ", \"host_apply\": " << num(r.phases.host_apply) << ", \"recompress\": " << num(r.phases.recompress)
      << "},\n";
    o << "  \"wall_seconds\": " << num(r.wall_seconds) << ",\n";
    o << "  \"overlap_efficiency\": " << num(r.overlap_efficiency) << ",\n";
    o << "  \"footprint\": {\"current_bytes\": " << r.footprint.current_bytes << ", \"peak_bytes\": "
      << r.footprint.peak_bytes << ", \"dense_bytes\": " << r.footprint.dense_bytes << ", \"ratio\": "
      << num(r.footprint.ratio) << "},\n";
    o << "  \"stage_batch_counts\": [";
    for (size_t i = 0; i < r.stage_batch_counts.size(); ++i) o << (i ? ", " : "") << r.stage_batch_counts[i];
    o << "],\n";
    o << "  \"transient_peak_bytes\": " << r.transient_peak_bytes << ",\n";
    o << "  \"chunk_decompress_count\": " << r.chunk_decompress_count << ",\n";
    o << "  \"chunk_recompress_count\": " << r.chunk_recompress_count << ",\n";
    o << "  \"transfer\": {\"h2d_seconds\": " << num(r.transfer.h2d_seconds) << ", \"d2h_seconds\": "
      << num(r.transfer.d2h_seconds) << ", \"kernel_seconds\": " << num(r.transfer.kernel_seconds)
      << ", \"h2d_op_count\": " << r.transfer.h2d_op_count << ", \"d2h_op_count\": " << r.transfer.d2h_op_count
      << ", \"bytes_moved\": " << r.transfer.bytes_moved << "},\n";
    char hex[17];
    std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(r.digest));
    o << "  \"digest\": \"" << hex << "\",\n";
    const PipelineConfig &c = r.config;
    o << "  \"config\": {\"chunk_qubits\": " << c.chunk_qubits << ", \"batch_qubits\": " << c.batch_qubits
      << ", \"error_bound\": " << num(c.error_bound) << ", \"strategy\": \"" << strategy_name(c.strategy)
      << "\", \"decompress_workers\": " << c.decompress_workers << ", \"recompress_workers\": "
      << c.recompress_workers << ", \"kernel_workers\": " << c.kernel_workers << ", \"host_fraction\": "
      << num(c.host_fraction) << ", \"pipeline_depth\": " << c.pipeline_depth << ", \"renormalize\": "
      << (c.renormalize ? "true" : "false") << ", \"seed\": " << c.seed << ", \"oracle_limit\": "
      << c.oracle_limit << "}\n}";
    return o.str();
}

} // namespace qzsim
