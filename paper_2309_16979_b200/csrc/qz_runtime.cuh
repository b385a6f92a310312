// qz_runtime.cuh — engine-private runtime types shared by the runtime's
// translation units (qz_runtime.cu: context, stage pipeline, C ABI;
// qz_store_io.cu: chunk-range import/export, QZST checkpoints, sharded
// exchange).  Not part of the C ABI.
#pragma once

#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "qz_codec.cuh"
#include "qz_gates.cuh"

namespace qz {

std::string &last_error();
struct XPlan;   // sharded-exchange plan (qz_store_io.cu)

inline constexpr uint64_t kPerChunkOverhead = 48;   // ChunkStore::kPerChunkOverhead (store.hpp:48)

// Grow-only device buffer.
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    void ensure(size_t bytes) {
        if (bytes <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        QZ_CUDA(cudaMalloc(&p, bytes ? bytes : 1));
        cap = bytes;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T> T *as() const { return static_cast<T *>(p); }
};

inline const char *status_text(int code) {
    switch (code) {
    case QZS_CRC: return "checksum mismatch on chunk ";
    case QZS_HEADER: return "malformed payload: bad header on chunk ";
    case QZS_RLE_TRUNC: return "malformed payload: truncated RLE stream on chunk ";
    case QZS_RLE_RUN: return "malformed payload: bad RLE run length on chunk ";
    case QZS_RAW_MISSING: return "malformed payload: missing raw values on chunk ";
    case QZS_RAW_UNDER: return "malformed payload: raw value underflow on chunk ";
    case QZS_RAW_UNUSED: return "malformed payload: unused raw values on chunk ";
    case QZS_ARENA: return "compressed arena capacity exhausted, needed bytes ";
    default: return "device error ";
    }
}

// Scratch set for one window of codec work.
struct Window {
    DevBuf amps, scratch, meta, idx, slot_chunk, sizes, reloff, base, cub, delta, maxd;
    DevBuf replay;   // uint32 flag raised by a relaxed gate pass
    DevBuf alt;      // second dense buffer: relaxed passes run out of place
    DevBuf nzslot;   // per slot: may be nonzero (0 = known all-(+0) after decode)
    // host-staged residency: HBM staging of the window's payloads
    DevBuf stage_in, stage_out, lt_off, lt_len, lt_crc, padded, soff, lused, hbase;
    uint64_t slots = 0, stage_in_cap = 0, stage_out_cap = 0;
    ChunkTable local() {
        return ChunkTable{lt_off.as<uint64_t>(), lt_len.as<uint32_t>(), lt_crc.as<uint32_t>()};
    }
    // host-staged pipeline: the second input set (slot map, staged
    // payloads, slot-indexed table, decode cursors) of a single window
    void reserve_input(const CodecGeom &g, uint64_t nslots) {
        const uint64_t bound = payload_bound(g.N, g.lossy ? 1.0 : 0.0);
        slots = nslots;
        stage_in_cap = nslots * (bound + 48) + 64;
        stage_in.ensure(stage_in_cap);
        lt_off.ensure(8 * nslots);
        lt_len.ensure(4 * nslots);
        lt_crc.ensure(4 * nslots);
        padded.ensure(8 * nslots);
        soff.ensure(8 * nslots);
        slot_chunk.ensure(sizeof(uint64_t) * nslots);
        idx.ensure(sizeof(DecIdx) * nslots);
        size_t t1 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, t1, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                      (int)std::min<uint64_t>(nslots, INT32_MAX));
        cub.ensure(t1 + 256);
    }
    DevBuf out_off, out_len, out_crc;   // encode output table (pipelined host-staged)
    ChunkTable out_local() {
        return ChunkTable{out_off.as<uint64_t>(), out_len.as<uint32_t>(), out_crc.as<uint32_t>()};
    }
    void reserve_staging(const CodecGeom &g, uint64_t nslots) {
        const uint64_t bound = payload_bound(g.N, g.lossy ? 1.0 : 0.0);
        stage_in_cap = nslots * (bound + 48) + 64;
        stage_out_cap = nslots * bound + 64;
        stage_in.ensure(stage_in_cap);
        stage_out.ensure(stage_out_cap);
        out_off.ensure(8 * nslots);
        out_len.ensure(4 * nslots);
        out_crc.ensure(4 * nslots);
        lt_off.ensure(8 * nslots);
        lt_len.ensure(4 * nslots);
        lt_crc.ensure(4 * nslots);
        padded.ensure(8 * nslots);
        soff.ensure(8 * nslots);
        lused.ensure(16);
        hbase.ensure(16);
    }
    void reserve(const CodecGeom &g, uint64_t nslots) {
        amps.ensure(sizeof(double2) * nslots * g.N);
        nzslot.ensure(4 * (nslots + 1) + 16);
        QZ_CUDA(cudaMemset(nzslot.p, 0, 4 * (nslots + 1)));   // count 0: map unused until a decode
        scratch.ensure(2 * nslots * g.half_stride + 64);   // warp_copy reads up to 8 B past a stream
        meta.ensure(sizeof(EncHalf) * 2 * nslots);
        idx.ensure(sizeof(DecIdx) * nslots);
        slot_chunk.ensure(sizeof(uint64_t) * nslots);
        sizes.ensure(sizeof(uint64_t) * nslots);
        reloff.ensure(sizeof(uint64_t) * nslots);
        delta.ensure(sizeof(int64_t) * nslots);
        base.ensure(sizeof(uint64_t) * 2);
        maxd.ensure(sizeof(int64_t) * 2);
        if (!replay.p) {
            replay.ensure(16);
            QZ_CUDA(cudaMemset(replay.p, 0, 16));
        }
        size_t t1 = 0, t2 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, t1, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                      (int)std::min<uint64_t>(nslots, INT32_MAX));
        cub::DeviceScan::InclusiveSum(nullptr, t2, (int64_t *)nullptr, (int64_t *)nullptr,
                                      (int)std::min<uint64_t>(nslots, INT32_MAX));
        size_t t3 = 0;
        cub::DeviceReduce::Max(nullptr, t3, (int64_t *)nullptr, (int64_t *)nullptr,
                               (int)std::min<uint64_t>(nslots, INT32_MAX));
        cub.ensure(std::max({t1, t2, t3}) + 256);
        slots = std::max(slots, nslots);
    }
    void release() {
        for (DevBuf *b : {&amps, &scratch, &meta, &idx, &slot_chunk, &sizes, &reloff, &base, &cub,
                          &delta, &maxd, &stage_in, &stage_out, &lt_off, &lt_len, &lt_crc, &padded,
                          &soff, &lused, &hbase, &out_off, &out_len, &out_crc, &replay, &alt, &nzslot})
            b->release();
    }
};

} // namespace qz

// ============================================================== context ====
// the ABI structs live in the global namespace (include/qzcuda.h)
using namespace qz;


struct qzc_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint64_t budget = 0;
    CodecTables tabs;
    DevStatus *status = nullptr;      // device
    DevStatus *status_host = nullptr; // pinned
    uint64_t launches = 0;
    Window win;                       // scratch for the host codec / gate entry points
    DevBuf arena, table_off, table_len, table_crc, forced, used;
    std::mutex mu;
    cudaEvent_t t_begin = nullptr, t_end = nullptr;
    uint64_t last_needed = 0;   // arena bytes a QZS_ARENA failure asked for

    void check_status(uint64_t index_base = 0) {
        QZ_CUDA(cudaMemcpyAsync(status_host, status, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream));
        QZ_CUDA(cudaStreamSynchronize(stream));
        if (status_host->code != 0) {
            const int code = status_host->code;
            const uint64_t idx = status_host->index;
            if (code == QZS_ARENA) last_needed = idx;
            QZ_CUDA(cudaMemsetAsync(status, 0, sizeof(DevStatus), stream));
            QZ_CUDA(cudaStreamSynchronize(stream));
            throw Failure(code == QZS_ARENA ? QZC_ENOMEM : QZC_ECODEC,
                          std::string(status_text(code)) + std::to_string(idx + (code == QZS_ARENA ? 0 : index_base)));
        }
    }
};

// ============================================================ simulator ====

struct qzc_sim {
    qzc_context *ctx = nullptr;
    qzc_sim_config cfg{};
    uint32_t n = 0, c = 0, m = 0;
    double eb = 0;
    uint64_t N = 0, nchunks = 0;
    CodecGeom geom{};
    DevBuf arena[2], off[2], len[2], crc[2];
    // host-staged residency: the arenas live in mapped page-locked host memory
    bool host_res = false;
    uint8_t *harena[2] = {nullptr, nullptr};      // host view
    uint8_t *harena_dev[2] = {nullptr, nullptr};  // device view of the same bytes
    DevBuf io_bytes;  // uint64[2]: host->HBM and HBM->host payload bytes
    DevBuf replays;   // uint64: windows replayed with the strict plan
    DevBuf small;     // uint64[4] scratch for init_basis (slot / forced lists)
    DevPlan plans[3]; // stage plans (relaxed / per-pass replay / whole strict), device buffers reused
    DevBuf used;   // uint64[2] bump pointers
    DevBuf acct;   // int64[2] current / peak
    uint64_t arena_cap = 0;   // bytes per arena (host-staged: the larger of hcap)
    uint64_t hcap[2] = {0, 0}; // host-staged arena capacities (grown on overflow)
    int cur = 0;
    uint64_t win_amps = 0;   // amplitudes per pipeline window
    Window win;              // window set 0 (also used by the host entry points)
    Window win2;             // window set 1: second stream of the stage pipeline
    bool two_windows = false;
    int relax = 1;              // 1: +0-safe diagonal units relaxed; 2: checked units too
    bool force_replay = false;  // debug_flags bit 0
    cudaStream_t streams[3] = {nullptr, nullptr, nullptr};   // [2]: host-staged write-back
    bool pipelined = false;   // host-staged, one window: gather / compute / write-back streams
    bool sparse_store = false;   // store = the init state (zero-chunk aliases): decode with run fills
    DevBuf gcub;              // scan scratch of the gather stream
    std::vector<cudaEvent_t> pevents;
    cudaEvent_t acct_ev[2] = {nullptr, nullptr};
    qzc_sim_stats stats{};
    bool initialized = false;
    // the |0...0> store's two payloads (zero chunk, basis chunk) as the first
    // init_basis produced them: later inits copy them back (no codec round trip)
    struct InitCache {
        bool valid = false;
        std::vector<uint8_t> bytes;   // the arena's first `used` bytes
        uint64_t used = 0, off[2] = {0, 0};
        uint32_t len[2] = {0, 0}, crc[2] = {0, 0};
    } init_cache;
    // qubits statically |0> (untouched by any non-diagonal gate since
    // init_basis, every gate keeping +0 zeros +0): Fresh for the stage plans
    uint64_t fresh_q = 0, fresh_v = 0;   // ... and their basis values
    uint64_t payload_now = 0;   // store payload bytes (host copy, refreshed per stage)
    std::shared_ptr<XPlan> xplan;   // last sharded-exchange plan (qz_store_io.cu)
    std::vector<cudaEvent_t> events;

    ChunkTable table(int i) {
        return ChunkTable{off[i].as<uint64_t>(), len[i].as<uint32_t>(), crc[i].as<uint32_t>()};
    }
    cudaStream_t st() const { return ctx->stream; }
    uint8_t *arena_ptr(int i) { return host_res ? harena_dev[i] : arena[i].as<uint8_t>(); }
    uint64_t *used_ptr(int i) { return used.as<uint64_t>() + i; }
    uint64_t cap(int i) const { return host_res ? hcap[i] : arena_cap; }
};

#define QZ_API_BEGIN try {
#define QZ_API_END                                                                             \
    }                                                                                          \
    catch (const Failure &f) {                                                                 \
        qz::last_error() = f.what();                                                               \
        return f.code;                                                                         \
    }                                                                                          \
    catch (const std::exception &e) {                                                          \
        qz::last_error() = e.what();                                                               \
        return QZC_EINVAL;                                                                     \
    }                                                                                          \
    return QZC_OK;

