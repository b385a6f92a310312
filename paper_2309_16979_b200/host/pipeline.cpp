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

} // namespace

std::pair<ChunkStore, SimulationReport> run(const Circuit &circuit, const PipelineConfig &cfg) {
    check_config(cfg, circuit.num_qubits);
    const uint32_t n = circuit.num_qubits, c = cfg.chunk_qubits;
    // plan() validates the circuit and the (c, m) preconditions (PlanError)
    const ExecutionPlan p = plan(circuit, c, cfg.batch_qubits);
    if (c < 1 || c > n)
        throw StoreError("chunk qubits must satisfy 1 <= c <= n, got c=" + std::to_string(c) +
                         ", n=" + std::to_string(n));
    if (n > ChunkStore::kMaxQubits) throw StoreError("qubit count exceeds configured address width (40)");

    qzc_sim_config sc{};
    sc.num_qubits = n;
    sc.chunk_qubits = c;
    sc.batch_qubits = cfg.batch_qubits;
    sc.error_bound = cfg.error_bound;
    sc.fuse_gates = 1;
    sc.renormalize = cfg.renormalize ? 1u : 0u;
    qzc_sim *h = nullptr;
    b200::check(qzc_sim_create(b200::ctx(), &sc, &h));
    // the store owns the engine simulator from here on (freed on any throw)
    ChunkStore store = ChunkStore::adopt(h, n, c, cfg.error_bound);
    b200::check(qzc_sim_init_basis(h));
    const std::vector<qzc_gate> abi = b200::to_abi(circuit.gates);
    Timer wall;
    b200::check(qzc_sim_run(h, abi.data(), abi.size()));
    const double run_seconds = wall.seconds();

    qzc_sim_stats st{};
    b200::check(qzc_sim_stats_get(h, &st));
    SimulationReport rep;
    rep.config = cfg;
    for (const Stage &s : p.stages) rep.stage_batch_counts.push_back(batch_count(s, n, c));
    rep.wall_seconds = run_seconds;
    rep.phases.decompress = st.decode_seconds;
    rep.phases.kernel = st.gate_seconds;
    rep.phases.recompress = st.encode_seconds;
    rep.phases.h2d = st.h2d_seconds;
    rep.phases.d2h = st.d2h_seconds;
    rep.transfer.kernel_seconds = st.gate_seconds;
    rep.transfer.h2d_seconds = st.h2d_seconds;
    rep.transfer.d2h_seconds = st.d2h_seconds;
    rep.transfer.bytes_moved = st.h2d_bytes + st.d2h_bytes;
    rep.overlap_efficiency = rep.wall_seconds > 0 ? rep.phases.kernel / rep.wall_seconds : 0.0;
    rep.transient_peak_bytes = 0;  // no host-side decompressed batches on this path
    rep.chunk_decompress_count = st.chunk_decompress_count;
    rep.chunk_recompress_count = st.chunk_recompress_count;
    rep.footprint = store.footprint();
    rep.norm = store_norm(store);
    rep.digest = store.digest();
    if (n <= cfg.oracle_limit && n <= kOracleLimit) {
        const DenseState ref = simulate_dense(circuit);
        rep.fidelity = fidelity(ref, store);
    }
    return {std::move(store), std::move(rep)};
}

void host_apply_batch(ChunkStore &store, const Stage &stage, const BatchDescriptor &batch,
                      const HostPhaseClocks &clocks) {
    // the batch's chunks decoded into one device buffer, the stage's remapped
    // gates applied there, the chunks re-encoded (device codec and kernels;
    // the same bytes as the batch inside qzc_sim_run)
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
    // compensated sum over the decoded store, on the device (qzc_sim_norm)
    double nn = 0.0;
    b200::check(qzc_sim_norm(store.engine_store(), &nn));
    return nn;
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
