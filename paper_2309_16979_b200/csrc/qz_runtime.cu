// qz_runtime.cu — context, HBM-resident compressed store, stage pipeline and
// the C ABI (include/qzcuda.h).
//
// Replaces qzsim::run (pipeline.cpp:128-314) + ChunkStore (store.cpp:26-217)
// + ReferenceDevice (device.cpp:98-503) for the hot path.  Per stage, the
// store is swept window by window: every chunk of the window's batches is
// CRC-verified and decoded straight into its batch slot, the stage's fused
// gate passes run over the whole window (batches stacked along the high
// buffer bits, which no gate touches), and every chunk is re-encoded into the
// other arena.  One codec round trip per chunk per stage, as the reference
// (SPEC.md:367), so payload bytes and the FNV digest match it exactly.
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <functional>
#include <vector>

#include "qz_codec.cuh"
#include "qz_gates.cuh"
#include "qz_kprof.cuh"
#include "qz_plan.cuh"
#include "qz_runtime.cuh"

using namespace qz;

namespace qz {
std::string &last_error() {
    thread_local std::string e;
    return e;
}
} // namespace qz

namespace {

// ---- accounting kernels ---------------------------------------------------
// delta[s] = new_size[s] - old_len[chunk(s)]  (ChunkStore::account_store order)
__global__ void k_delta(const uint64_t *sizes, const uint64_t *slot_chunk, const uint32_t *old_len,
                        uint64_t nslots, int64_t *delta) {
    const uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s < nslots) delta[s] = int64_t(sizes[s]) - int64_t(old_len[slot_chunk ? slot_chunk[s] : s]);
}
// acct[0] = current bytes, acct[1] = peak; prefix = inclusive scan of delta
__global__ void k_account(int64_t *acct, const int64_t *prefix, const int64_t *maxp,
                          uint64_t nslots) {
    const int64_t cur = acct[0];
    const int64_t peak_cand = cur + *maxp;
    if (peak_cand > acct[1]) acct[1] = peak_cand;
    acct[0] = cur + prefix[nslots - 1];
}

// Export: copy every chunk's payload to its place in chunk order (warp per
// chunk, 16 B vector stores where aligned).
__global__ void k_pack_payloads(const uint8_t *__restrict__ arena, ChunkTable t, const uint64_t *__restrict__ dst_off,
                                uint64_t nchunks, uint8_t *__restrict__ out) {
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (w >= nchunks) return;
    const uint8_t *src = arena + t.off[w];
    uint8_t *dst = out + dst_off[w];
    const uint32_t n = t.len[w];
    for (uint32_t i = lane; i < n; i += 32) dst[i] = src[i];
}

__global__ void k_io_count(const uint64_t *soff, const uint64_t *padded, uint64_t nslots,
                           uint64_t *io) {
    atomicAdd((unsigned long long *)&io[0], (unsigned long long)(soff[nslots - 1] + padded[nslots - 1]));
}
__global__ void k_io_count_out(const uint64_t *used_local, uint64_t *io) {
    atomicAdd((unsigned long long *)&io[1], (unsigned long long)((*used_local + 15) / 16 * 16));
}

__global__ void k_fill_init(ChunkTable t, uint64_t nchunks, uint64_t zoff, uint32_t zlen,
                            uint32_t zcrc, uint64_t boff, uint32_t blen, uint32_t bcrc) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nchunks) return;
    t.off[i] = i ? zoff : boff;
    t.len[i] = i ? zlen : blen;
    t.crc[i] = i ? zcrc : bcrc;
}

// per-slot compensated partial sums: out[4s..4s+3] = Re<a|b>, Im<a|b>, |a|^2, |b|^2
// (b = the store, a = dense reference or null for the norm)
__global__ void k_partials(const double2 *win, uint64_t nslots, uint64_t N, const double2 *dense,
                           uint64_t dense_first, double *out) {
    const uint64_t s = uint64_t(blockIdx.x) * blockDim.y + threadIdx.y;
    if (s >= nslots) return;
    double acc[4] = {0, 0, 0, 0}, cmp[4] = {0, 0, 0, 0};
    auto kadd = [&](int i, double x) {
        const double y = x - cmp[i], t = acc[i] + y;
        cmp[i] = (t - acc[i]) - y;
        acc[i] = t;
    };
    // Each warp lane takes a strided subset, then the lanes are combined in
    // lane order (deterministic).
    const uint32_t lane = threadIdx.x;
    for (uint64_t j = lane; j < N; j += 32) {
        const double2 b = win[s * N + j];
        kadd(3, __dadd_rn(__dmul_rn(b.x, b.x), __dmul_rn(b.y, b.y)));
        if (dense) {
            const double2 a = dense[(dense_first + s) * N + j];
            // conj(a) * b
            kadd(0, __dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)));
            kadd(1, __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
            kadd(2, __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)));
        }
    }
    for (int i = 0; i < 4; ++i) {
        double v = acc[i];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        if (lane == 0) out[4 * s + i] = v;
    }
}

// apply_single_qubit / apply_two_qubit over pair (group) indices
// [begin, end) with the reference's formula (kernels.cpp:20-54): complex
// products (ac - bd, ad + bc) separately rounded, rows summed left to right.
__global__ void k_apply_range(double2 *buf, uint32_t dim, uint32_t b0, uint32_t b1, const double2 *m,
                              uint64_t begin, uint64_t end) {
    const uint64_t p = begin + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= end) return;
    auto prod = [](double2 a, double2 v) {
        return make_double2(__dsub_rn(__dmul_rn(a.x, v.x), __dmul_rn(a.y, v.y)),
                            __dadd_rn(__dmul_rn(a.x, v.y), __dmul_rn(a.y, v.x)));
    };
    auto add = [](double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); };
    if (dim == 2) {
        const uint64_t i = insert_zero_bit(p, b0), j = i | (uint64_t(1) << b0);
        const double2 a = buf[i], b = buf[j];
        buf[i] = add(prod(m[0], a), prod(m[1], b));
        buf[j] = add(prod(m[2], a), prod(m[3], b));
        return;
    }
    const uint32_t lo = b0 < b1 ? b0 : b1, hi = b0 < b1 ? b1 : b0;
    const uint64_t base = insert_zero_bit(insert_zero_bit(p, lo), hi);
    const uint64_t s0 = uint64_t(1) << b0, s1 = uint64_t(1) << b1;
    const uint64_t idx[4] = {base, base | s1, base | s0, base | s0 | s1};
    double2 in[4];
    for (int c = 0; c < 4; ++c) in[c] = buf[idx[c]];
    for (int r = 0; r < 4; ++r) {
        double2 acc = prod(m[4 * r], in[0]);
        for (int c = 1; c < 4; ++c) acc = add(acc, prod(m[4 * r + c], in[c]));
        buf[idx[r]] = acc;
    }
}

// a *= scale for std::complex<double> and a real scale: componentwise
// products (complex x real, no cross terms), pipeline.cpp:283
__global__ void k_scale(double2 *buf, uint64_t n, double scale) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double2 a = buf[i];
        buf[i] = make_double2(__dmul_rn(a.x, scale), __dmul_rn(a.y, scale));
    }
}

__global__ void k_basis(double2 *buf, uint64_t n) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) buf[i] = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
}

struct Kahan {
    double s = 0, c = 0;
    void add(double x) {
        const double y = x - c, t = s + y;
        c = (t - s) - y;
        s = t;
    }
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

} // namespace

namespace {

// Encode win slots [0, nslots) into arena `a` / table `t` via slot_chunk map.
void encode_window(qzc_context *ctx, Window &w, const CodecGeom &g, uint64_t nslots,
                   const uint64_t *slot_chunk, const uint64_t *forced, uint32_t nforced,
                   uint8_t *arena, uint64_t *used, uint64_t cap, ChunkTable t,
                   const uint32_t *old_len, int64_t *acct, uint64_t &launches,
                   cudaStream_t s = nullptr, cudaEvent_t acct_prev = nullptr,
                   cudaEvent_t acct_done = nullptr, const uint64_t *acct_map = nullptr) {
    if (!s) s = ctx->stream;
    if (!acct_map) acct_map = slot_chunk;
    launch_encode(w.amps.as<double2>(), nslots, g, forced, nforced, w.scratch.as<uint8_t>(),
                  w.meta.as<EncHalf>(), s);
    const int tail = kprof_begin(s);
    launch_enc_sizes(w.meta.as<EncHalf>(), nslots, g, w.sizes.as<uint64_t>(), s);
    size_t tb = w.cub.cap;
    QZ_CUDA(cub::DeviceScan::ExclusiveSum(w.cub.p, tb, w.sizes.as<uint64_t>(), w.reloff.as<uint64_t>(),
                                          (int)nslots, s));
    launch_arena_alloc(w.reloff.as<uint64_t>(), w.sizes.as<uint64_t>(), nslots, used, cap,
                       w.base.as<uint64_t>(), ctx->status, s);
    if (acct && old_len) {
        k_delta<<<(unsigned)ceil_div(nslots, 256), 256, 0, s>>>(w.sizes.as<uint64_t>(), acct_map,
                                                                old_len, nslots, w.delta.as<int64_t>());
        QZ_CHECK_LAUNCH();
        tb = w.cub.cap;
        QZ_CUDA(cub::DeviceScan::InclusiveSum(w.cub.p, tb, w.delta.as<int64_t>(),
                                              w.delta.as<int64_t>(), (int)nslots, s));
        tb = w.cub.cap;
        QZ_CUDA(cub::DeviceReduce::Max(w.cub.p, tb, w.delta.as<int64_t>(), w.maxd.as<int64_t>(),
                                       (int)nslots, s));
        // footprint accounting is a running sum in batch order: chain the
        // windows of concurrent streams through events
        if (acct_prev) QZ_CUDA(cudaStreamWaitEvent(s, acct_prev, 0));
        k_account<<<1, 1, 0, s>>>(acct, w.delta.as<int64_t>(), w.maxd.as<int64_t>(), nslots);
        QZ_CHECK_LAUNCH();
        if (acct_done) QZ_CUDA(cudaEventRecord(acct_done, s));
        launches += 5;
    }
    kprof_end(tail, s, "enc_sizes+scan+alloc", 0, 0.0);
    const int asm_h = kprof_begin(s);
    launch_assemble(w.scratch.as<uint8_t>(), w.meta.as<EncHalf>(), w.reloff.as<uint64_t>(),
                    w.sizes.as<uint64_t>(), w.base.as<uint64_t>(), slot_chunk, nslots, g, arena, t,
                    ctx->status, s);
    kprof_end(asm_h, s, "k_assemble", 0, 0.0);
    launch_crc(ctx->tabs, arena, t, slot_chunk, nslots, false, ctx->status, s);
    launches += 6;
}

void decode_window(qzc_context *ctx, Window &w, const CodecGeom &g, uint64_t nslots,
                   const uint64_t *slot_chunk, const uint8_t *arena, ChunkTable t,
                   uint64_t &launches, cudaStream_t s = nullptr, bool sparse = false) {
    if (!s) s = ctx->stream;
    launch_crc(ctx->tabs, arena, t, slot_chunk, nslots, true, ctx->status, s);
    launch_dec_index(arena, t, slot_chunk, nslots, g, w.idx.as<DecIdx>(), ctx->status, s,
                     w.nzslot.as<uint32_t>());
    launch_decode(arena, w.idx.as<DecIdx>(), slot_chunk, nslots, g, w.amps.as<double2>(),
                  ctx->status, s, nullptr, sparse);
    launches += 3;
}

// decode_window with an explicit cursor array and target window
void decode_into(qzc_context *ctx, DecIdx *idx, double2 *amps, const CodecGeom &g, uint64_t nslots,
                 const uint64_t *slot_chunk, const uint8_t *arena, ChunkTable t, uint64_t &launches,
                 cudaStream_t s, bool sparse = false, uint32_t *nzslot = nullptr) {
    launch_crc(ctx->tabs, arena, t, slot_chunk, nslots, true, ctx->status, s);
    launch_dec_index(arena, t, slot_chunk, nslots, g, idx, ctx->status, s, nzslot);
    launch_decode(arena, idx, slot_chunk, nslots, g, amps, ctx->status, s, nullptr, sparse);
    launches += 3;
}

// The stage's fused passes over window W: relaxed passes run out of place
// between W.amps and W.alt with their per-pass strict replay; the result is
// left in W.amps (the two buffers swap roles when needed).
void run_window_passes(qzc_sim *sim, Window &W, const DevPlan &dp, const DevPlan &dsub, const DevPlan &dfull,
                       uint32_t wbits, cudaStream_t S,
                       const std::function<void(double2 *, const uint32_t *)> &redecode,
                       const std::function<bool(cudaStream_t)> &ensure_dfull, bool host_decides = false);

uint32_t log2u(uint64_t x) {
    uint32_t r = 0;
    while ((uint64_t(1) << r) < x) ++r;
    return r;
}

uint64_t host_ram() {
    return uint64_t(sysconf(_SC_PHYS_PAGES)) * uint64_t(sysconf(_SC_PAGE_SIZE));
}

void alloc_host_arena(qzc_sim *sim, int i, uint64_t cap) {
    if (sim->harena[i]) QZ_CUDA(cudaFreeHost(sim->harena[i]));
    sim->harena[i] = sim->harena_dev[i] = nullptr;
    void *h = nullptr, *d = nullptr;
    QZ_CUDA(cudaHostAlloc(&h, cap + 64, cudaHostAllocMapped | cudaHostAllocPortable));
    QZ_CUDA(cudaHostGetDevicePointer(&d, h, 0));
    sim->harena[i] = static_cast<uint8_t *>(h);
    sim->harena_dev[i] = static_cast<uint8_t *>(d);
    sim->hcap[i] = cap;
}

// Output arena b overflowed (needed >= the failing allocation's end): give it
// at least twice the room (bounded by the worst case and 40% of host RAM).
// Returns false when it cannot grow.
bool grow_host_arena(qzc_sim *sim, int b, uint64_t needed) {
    const uint64_t worst = std::max<uint64_t>(sim->nchunks, 2) * payload_bound(sim->N, sim->eb) + 4096;
    const uint64_t limit = std::min<uint64_t>(worst, host_ram() * 2 / 5);
    const uint64_t want = std::min<uint64_t>(limit, std::max<uint64_t>(2 * sim->hcap[b], needed + needed / 2));
    if (want <= sim->hcap[b]) return false;
    QZ_CUDA(cudaDeviceSynchronize());
    alloc_host_arena(sim, b, want);
    sim->arena_cap = std::max(sim->hcap[0], sim->hcap[1]);
    return true;
}

void sim_alloc(qzc_sim *sim) {
    qzc_context *ctx = sim->ctx;
    const uint64_t tbl_entries = std::max<uint64_t>(sim->nchunks, 2);
    sim->replays.ensure(8);
    QZ_CUDA(cudaMemset(sim->replays.p, 0, 8));
    sim->small.ensure(64);
    for (int i = 0; i < 2; ++i) {
        sim->off[i].ensure(8 * tbl_entries);
        sim->len[i].ensure(4 * tbl_entries);
        sim->crc[i].ensure(4 * tbl_entries);
        QZ_CUDA(cudaMemset(sim->len[i].p, 0, 4 * tbl_entries));
    }
    sim->used.ensure(16);
    sim->acct.ensure(16);
    QZ_CUDA(cudaMemset(sim->used.p, 0, 16));
    QZ_CUDA(cudaMemset(sim->acct.p, 0, 16));

    // window: whole batches, power of two, bounded by the HBM budget
    size_t free_b = 0, total_b = 0;
    QZ_CUDA(cudaMemGetInfo(&free_b, &total_b));
    uint64_t budget = ctx->budget ? std::min<uint64_t>(ctx->budget, free_b) : free_b;
    budget = budget > (uint64_t(3) << 30) ? budget - (uint64_t(3) << 30) : budget / 2;
    // dense + encode scratch + metadata (+ payload staging when host-staged:
    // two input sets and one output)
    const uint64_t per_amp = 16 + (sim->relax == 2 ? 16 : 0) + 2 * sim->geom.half_stride / sim->N + 8 +
                             (sim->host_res ? 3 * (payload_bound(sim->N, sim->eb) + 48) / sim->N + 1 : 0);
    const uint64_t state_amps = uint64_t(1) << sim->n;
    uint64_t wa = sim->cfg.window_amps;
    if (!wa) {
        // HBM-resident: half the budget stays for the arenas
        const uint64_t cap_amps = std::max<uint64_t>(budget / (sim->host_res ? 1 : 2) / per_amp, sim->N);
        wa = uint64_t(1) << (63 - __builtin_clzll(cap_amps));
        wa = std::min(wa, state_amps);
    }
    if (wa & (wa - 1)) wa = uint64_t(1) << log2u(wa);
    // at least one whole batch (2^m amplitudes) and two chunk slots
    // (skip_reencode: size for one stage over the whole state)
    const uint64_t batch_amps = uint64_t(1) << (sim->cfg.skip_reencode ? sim->n : std::min(sim->m, sim->n));
    wa = std::max<uint64_t>(std::min<uint64_t>(wa, state_amps), std::max<uint64_t>(batch_amps, 2 * sim->N));
    // two half-size windows on two streams when the window holds >= 2
    // batches: decode / gate passes / encode of neighbouring windows overlap
    sim->two_windows = wa >= 2 * batch_amps && wa >= 4 * sim->N;
    if (sim->two_windows) wa /= 2;
    sim->win_amps = wa;
    const uint64_t win_slots = std::max<uint64_t>(wa / sim->N, 2);
    sim->win.reserve(sim->geom, win_slots);
    if (sim->two_windows) sim->win2.reserve(sim->geom, win_slots);
    if (sim->relax == 2) {
        // out-of-place passes for checked units
        sim->win.alt.ensure(sizeof(double2) * win_slots * sim->N);
        if (sim->two_windows) sim->win2.alt.ensure(sizeof(double2) * win_slots * sim->N);
    }
    for (int i = 0; i < 2; ++i) {
        QZ_CUDA(cudaStreamCreateWithFlags(&sim->streams[i], cudaStreamNonBlocking));
        QZ_CUDA(cudaEventCreateWithFlags(&sim->acct_ev[i], cudaEventDisableTiming));
    }
    QZ_CUDA(cudaStreamCreateWithFlags(&sim->streams[2], cudaStreamNonBlocking));

    // arenas: worst case if it fits, else what is left
    QZ_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t worst = tbl_entries * payload_bound(sim->N, sim->eb) + 4096;
    uint64_t avail = free_b > (uint64_t(2) << 30) ? free_b - (uint64_t(2) << 30) : free_b / 2;
    if (ctx->budget) {
        const uint64_t spent = wa * per_amp;
        avail = std::min<uint64_t>(avail, ctx->budget > spent ? ctx->budget - spent : 0);
    }
    sim->arena_cap = std::min<uint64_t>(worst, avail / 2);
    if (!sim->host_res && sim->arena_cap < 4096)
        throw Failure(QZC_ENOMEM, "not enough HBM for the compressed store");
    if (sim->host_res) {
        // page-locked, mapped host arenas (the store leaves HBM; windows
        // stream their payloads through it).  Sized for a compression ratio
        // of 2.5 to start (at least 1 GiB, at most the worst case and 40% of
        // host RAM each) and grown when a stage's output overflows
        // (grow_host_arena) instead of pinning worst-case arenas up front.
        const uint64_t dense = (uint64_t(1) << sim->n) * 16;
        sim->arena_cap = std::min<uint64_t>({worst, host_ram() * 2 / 5, std::max<uint64_t>(dense / 5 * 2, uint64_t(1) << 30)});
        if (const char *e = getenv("QZ_HOST_ARENA_START"))   // test hook: force the growth path
            sim->arena_cap = std::max<uint64_t>(4096, std::strtoull(e, nullptr, 10));
        for (int i = 0; i < 2; ++i) alloc_host_arena(sim, i, sim->arena_cap);
        sim->win.reserve_staging(sim->geom, sim->win.slots);
        if (sim->two_windows) {
            sim->win2.reserve_staging(sim->geom, sim->win2.slots);
        } else {
            // one window: overlap the next window's gather and this window's
            // write-back with its decode / passes / encode
            sim->pipelined = true;
            sim->win2.reserve_input(sim->geom, sim->win.slots);
            size_t t1 = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, t1, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                          (int)std::min<uint64_t>(sim->win.slots, INT32_MAX));
            sim->gcub.ensure(t1 + 256);
        }
        sim->io_bytes.ensure(16);
        QZ_CUDA(cudaMemset(sim->io_bytes.p, 0, 16));
    } else {
        // +64: the decoder's RLE readers fetch 16 bytes ahead
        for (int i = 0; i < 2; ++i) sim->arena[i].ensure(sim->arena_cap + 64);
    }
}

// Elements off `val` on `mask` (window bits still fresh at a stage's end) <- +0.
__global__ void k_fill_dead(double2 *win, uint64_t n, uint64_t mask, uint64_t val) {
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += uint64_t(gridDim.x) * blockDim.x)
        if ((e & mask) != val) win[e] = make_double2(0.0, 0.0);
}

void run_window_passes(qzc_sim *sim, Window &W, const DevPlan &dp, const DevPlan &dsub, const DevPlan &dfull,
                       uint32_t wbits, cudaStream_t S,
                       const std::function<void(double2 *, const uint32_t *)> &redecode,
                       const std::function<bool(cudaStream_t)> &ensure_dfull, bool host_decides) {
    qzc_context *ctx = sim->ctx;
    const NzMap nz{W.nzslot.as<uint32_t>(), sim->c};
    if (!dp.relaxed) {
        ctx->launches += run_passes(dp, W.amps.as<double2>(), wbits, S, nullptr, nz);
        return;
    }
    uint32_t *pflag = W.replay.as<uint32_t>(), *wflag = pflag + 1;
    double2 *res = run_relaxed(dp, dsub, W.amps.as<double2>(), W.alt.p ? W.alt.as<double2>() : nullptr, wbits, S,
                               pflag, wflag, sim->replays.as<uint64_t>(), sim->force_replay, ctx->launches, nz);
    // host_decides (a stage's only window): wait for the relaxed passes and
    // read the flag, so the strict replay is queued only when it is needed
    // (instead of ~55 device-side no-op launches per stage)
    if (host_decides) {
        uint32_t raised = 0;
        QZ_CUDA(cudaStreamSynchronize(S));
        QZ_CUDA(cudaMemcpy(&raised, wflag, 4, cudaMemcpyDeviceToHost));
        if (raised && ensure_dfull(S)) {
            redecode(res, wflag);
            ctx->launches += 1 + run_passes(dfull, res, wbits, S, wflag);
            flag_done(wflag, sim->replays.as<uint64_t>(), S);
            ++ctx->launches;
        }
    } else if (ensure_dfull(S)) {
    // (the strict plan is built while the relaxed passes run on the device)
        // a +0-safe relaxed pass flagged: decode the window again from its
        // untouched payloads and run the strict plan (no-ops unless flagged)
        redecode(res, wflag);
        ctx->launches += 1 + run_passes(dfull, res, wbits, S, wflag);
        flag_done(wflag, sim->replays.as<uint64_t>(), S);
        ++ctx->launches;
    }
    if (res != W.amps.as<double2>()) std::swap(W.amps, W.alt);   // stream-ordered: later kernels see the swap
}

// PipelineConfig::renormalize (pipeline.cpp:278-288): norm = store_norm —
// the reference's Kahan sum over |a|^2 in chunk order (pipeline.cpp:119-126),
// a sequential compensated recurrence, so it runs on the host over decoded
// windows streamed from the device (its bits decide the scale and hence the
// payload bytes) — then every chunk is decoded, scaled on the device and
// re-encoded in chunk order (store_chunk's footprint accounting order).
void renormalize(qzc_sim *sim) {
    qzc_context *ctx = sim->ctx;
    cudaStream_t s = ctx->stream;
    Window &w = sim->win;
    const uint64_t per = std::max<uint64_t>(1, w.slots);
    const uint64_t mask = (uint64_t(1) << (sim->n - sim->c)) - 1;
    std::vector<double2> host(per * sim->N);
    double sum = 0.0, comp = 0.0;
    for (uint64_t f = 0; f < sim->nchunks; f += per) {
        const uint64_t k = std::min(per, sim->nchunks - f);
        launch_slot_chunks(w.slot_chunk.as<uint64_t>(), k, f, 0, mask, 0, s);
        decode_window(ctx, w, sim->geom, k, w.slot_chunk.as<uint64_t>(), sim->arena_ptr(sim->cur),
                      sim->table(sim->cur), ctx->launches, s, sim->sparse_store);
        ctx->check_status();
        QZ_CUDA(cudaMemcpyAsync(host.data(), w.amps.p, 16 * k * sim->N, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaStreamSynchronize(s));
        for (uint64_t i = 0; i < k * sim->N; ++i) {
            const double x = host[i].x * host[i].x + host[i].y * host[i].y;   // std::norm
            const double y = x - comp, t = sum + y;
            comp = (t - sum) - y;
            sum = t;
        }
    }
    if (!(sum > 0.0)) return;
    const double scale = 1.0 / std::sqrt(sum);
    const int a = sim->cur, b = 1 - a;
    QZ_CUDA(cudaMemsetAsync(sim->used_ptr(b), 0, 8, s));
    for (uint64_t f = 0; f < sim->nchunks; f += per) {
        const uint64_t k = std::min(per, sim->nchunks - f);
        launch_slot_chunks(w.slot_chunk.as<uint64_t>(), k, f, 0, mask, 0, s);
        decode_window(ctx, w, sim->geom, k, w.slot_chunk.as<uint64_t>(), sim->arena_ptr(a), sim->table(a),
                      ctx->launches, s, sim->sparse_store);
        k_scale<<<(unsigned)std::min<uint64_t>(ceil_div(k * sim->N, 256), kNumSMs * 16), 256, 0, s>>>(
            w.amps.as<double2>(), k * sim->N, scale);
        QZ_CHECK_LAUNCH();
        ++ctx->launches;
        encode_window(ctx, w, sim->geom, k, w.slot_chunk.as<uint64_t>(), nullptr, 0, sim->arena_ptr(b),
                      sim->used_ptr(b), sim->cap(b), sim->table(b), sim->len[a].as<uint32_t>(),
                      sim->acct.as<int64_t>(), ctx->launches, s);
    }
    ctx->check_status();
    sim->cur = b;
    sim->sparse_store = false;
    sim->stats.chunk_decompress_count += 2 * sim->nchunks;
    sim->stats.chunk_recompress_count += sim->nchunks;
}

} // namespace

// ================================================================== C ABI ==

extern "C" {

const char *qzc_last_error(void) { return qz::last_error().c_str(); }
const char *qzc_version(void) { return "qzcuda 0.1 sm_100a"; }

int qzc_gate_matrix(const qzc_gate *gate, double *mat_out, uint32_t *dim_out) {
    QZ_API_BEGIN
    if (!gate || !mat_out || !dim_out) throw Failure(QZC_EINVAL, "null argument");
    double2 m[16];
    gate_matrix_host(*gate, m, dim_out);
    std::memcpy(mat_out, m, sizeof m);
    QZ_API_END
}

uint32_t qzc_crc32(const uint8_t *bytes, uint64_t len) { return crc32_host(bytes, len); }
uint64_t qzc_fnv1a64(const uint8_t *bytes, uint64_t len, uint64_t state) {
    return fnv1a64_host(bytes, len, state);
}
uint64_t qzc_payload_bound(uint64_t elements, double error_bound) {
    return payload_bound(elements, error_bound);
}

int qzc_context_create(int device, uint64_t hbm_budget_bytes, qzc_context **out) {
    QZ_API_BEGIN
    if (!out) throw Failure(QZC_EINVAL, "null out");
    int count = 0;
    QZ_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
        throw Failure(QZC_EDEVICE, "no CUDA device " + std::to_string(device));
    QZ_CUDA(cudaSetDevice(device));
    auto *ctx = new qzc_context;
    ctx->device = device;
    ctx->budget = hbm_budget_bytes;
    QZ_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    init_codec_tables(ctx->tabs);
    QZ_CUDA(cudaMalloc(&ctx->status, sizeof(DevStatus)));
    QZ_CUDA(cudaMemset(ctx->status, 0, sizeof(DevStatus)));
    QZ_CUDA(cudaMallocHost(&ctx->status_host, sizeof(DevStatus)));
    // L2 fetch granularity hint (QZ_L2_FETCH bytes, tuning): the sparse
    // opening passes read one 16 B element per 128 B line
    if (const char *e = getenv("QZ_L2_FETCH")) QZ_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, size_t(atoi(e))));
    // load the stage loop's kernels now (CUDA loads a kernel's module at its
    // first launch): two tiny runs, lossy and lossless, multi-stage, so no
    // timed run pays for module loading (QZ_NO_WARMUP=1 skips)
    if (!getenv("QZ_NO_WARMUP")) {
        auto g = [](uint32_t kind, uint32_t a, int b = -1, double p = 0.0) {
            qzc_gate x{};
            x.kind = kind;
            x.nqubits = b < 0 ? 1 : 2;
            x.qubits[0] = a;
            x.qubits[1] = b < 0 ? 0 : uint32_t(b);
            x.params[0] = p;
            return x;
        };
        std::vector<qzc_gate> circ;
        for (uint32_t q = 0; q < 8; ++q) circ.push_back(g(QZC_H, q));
        for (const qzc_gate &x : {g(QZC_CX, 0, 1), g(QZC_CZ, 2, 3), g(QZC_U1, 4, -1, 0.3), g(QZC_X, 1),
                                  g(QZC_RY, 2, -1, 0.4), g(QZC_T, 3), g(QZC_CX, 6, 2), g(QZC_SWAP, 5, 6),
                                  g(QZC_SWAP, 0, 7), g(QZC_H, 7), g(QZC_U1, 7, -1, 2.5), g(QZC_CX, 7, 0)})
            circ.push_back(x);
        for (double eb : {1e-5, 0.0})
            for (uint32_t m : {8u, 6u}) {
                qzc_sim_config sc{};
                sc.num_qubits = 8;
                sc.chunk_qubits = 4;
                sc.batch_qubits = m;
                sc.error_bound = eb;
                sc.fuse_gates = 1;
                qzc_sim *sim = nullptr;
                if (qzc_sim_create(ctx, &sc, &sim) == QZC_OK) {
                    qzc_sim_init_basis(sim);
                    qzc_sim_run(sim, circ.data(), circ.size());
                    qzc_sim_destroy(sim);
                }
            }
        QZ_CUDA(cudaDeviceSynchronize());
        ctx->launches = 0;
        last_error().clear();
    }
    *out = ctx;
    QZ_API_END
}

void qzc_context_destroy(qzc_context *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->win.release();
    for (DevBuf *b : {&ctx->arena, &ctx->table_off, &ctx->table_len, &ctx->table_crc, &ctx->forced, &ctx->used})
        b->release();
    free_codec_tables(ctx->tabs);
    if (ctx->t_begin) cudaEventDestroy(ctx->t_begin);
    if (ctx->t_end) cudaEventDestroy(ctx->t_end);
    cudaFree(ctx->status);
    cudaFreeHost(ctx->status_host);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int qzc_synchronize(qzc_context *ctx) {
    QZ_API_BEGIN
    QZ_CUDA(cudaStreamSynchronize(ctx->stream));
    QZ_API_END
}

uint64_t qzc_kernel_launches(const qzc_context *ctx) { return ctx ? ctx->launches : 0; }

int qzc_timer_begin(qzc_context *ctx) {
    QZ_API_BEGIN
    QZ_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->t_begin) {
        QZ_CUDA(cudaEventCreate(&ctx->t_begin));
        QZ_CUDA(cudaEventCreate(&ctx->t_end));
    }
    QZ_CUDA(cudaEventRecord(ctx->t_begin, ctx->stream));
    QZ_API_END
}

int qzc_timer_end(qzc_context *ctx, double *seconds_out) {
    QZ_API_BEGIN
    if (!ctx->t_begin) throw Failure(QZC_EINVAL, "timer not started");
    QZ_CUDA(cudaEventRecord(ctx->t_end, ctx->stream));
    QZ_CUDA(cudaEventSynchronize(ctx->t_end));
    float ms = 0;
    QZ_CUDA(cudaEventElapsedTime(&ms, ctx->t_begin, ctx->t_end));
    *seconds_out = ms * 1e-3;
    QZ_API_END
}

// ---- codec entry points ----------------------------------------------------

int qzc_compress_host(qzc_context *ctx, const double *amps, uint64_t count, uint64_t elements,
                      double error_bound, const uint64_t *forced_raw, uint64_t n_forced,
                      uint8_t *payload_out, uint64_t payload_cap, uint64_t *offsets,
                      uint32_t *sizes, uint32_t *crcs) {
    QZ_API_BEGIN
    std::lock_guard<std::mutex> lk(ctx->mu);
    QZ_CUDA(cudaSetDevice(ctx->device));
    if (elements == 0 || (elements & (elements - 1)))
        throw Failure(QZC_ECODEC, "chunk length must be a power of two, got " + std::to_string(elements));
    if (!(error_bound >= 0.0) || !std::isfinite(error_bound))
        throw Failure(QZC_ECODEC, "error bound must be finite and non-negative");
    if (count == 0) return QZC_OK;
    const CodecGeom g = make_geom(elements, error_bound);
    std::vector<uint64_t> fr(forced_raw, forced_raw + n_forced);
    for (uint64_t f : fr)
        if (f >= 2 * elements) throw Failure(QZC_ECODEC, "forced raw index out of range");
    std::sort(fr.begin(), fr.end());
    cudaStream_t s = ctx->stream;
    // process in windows of at most ~1 GiB dense
    const uint64_t per = std::max<uint64_t>(1, std::min<uint64_t>(count, (uint64_t(1) << 26) / elements));
    ctx->win.reserve(g, per);
    const uint64_t bound = payload_bound(elements, error_bound);
    ctx->arena.ensure(per * bound + 64);
    ctx->table_off.ensure(8 * per);
    ctx->table_len.ensure(4 * per);
    ctx->table_crc.ensure(4 * per);
    ctx->used.ensure(8);
    ctx->forced.ensure(8 * std::max<size_t>(fr.size(), 1));
    if (!fr.empty())
        QZ_CUDA(cudaMemcpyAsync(ctx->forced.p, fr.data(), 8 * fr.size(), cudaMemcpyHostToDevice, s));
    ChunkTable t{ctx->table_off.as<uint64_t>(), ctx->table_len.as<uint32_t>(), ctx->table_crc.as<uint32_t>()};
    std::vector<uint64_t> hoff(per);
    std::vector<uint32_t> hlen(per), hcrc(per);
    uint64_t written = 0;
    for (uint64_t first = 0; first < count; first += per) {
        const uint64_t k = std::min(per, count - first);
        QZ_CUDA(cudaMemcpyAsync(ctx->win.amps.p, amps + 2 * first * elements, 16 * k * elements,
                                cudaMemcpyHostToDevice, s));
        QZ_CUDA(cudaMemsetAsync(ctx->used.p, 0, 8, s));
        encode_window(ctx, ctx->win, g, k, nullptr, ctx->forced.as<uint64_t>(), (uint32_t)fr.size(),
                      ctx->arena.as<uint8_t>(), ctx->used.as<uint64_t>(), ctx->arena.cap, t, nullptr,
                      nullptr, ctx->launches);
        ctx->check_status();
        QZ_CUDA(cudaMemcpyAsync(hoff.data(), t.off, 8 * k, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaMemcpyAsync(hlen.data(), t.len, 4 * k, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaMemcpyAsync(hcrc.data(), t.crc, 4 * k, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaStreamSynchronize(s));
        uint64_t total = 0;
        for (uint64_t i = 0; i < k; ++i) total += hlen[i];
        if (written + total > payload_cap) throw Failure(QZC_EINVAL, "payload buffer too small");
        // arena order == slot order (single window, identity mapping)
        QZ_CUDA(cudaMemcpyAsync(payload_out + written, ctx->arena.p, total, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaStreamSynchronize(s));
        for (uint64_t i = 0; i < k; ++i) {
            offsets[first + i] = written + hoff[i];
            sizes[first + i] = hlen[i];
            crcs[first + i] = hcrc[i];
        }
        written += total;
    }
    QZ_API_END
}

int qzc_decompress_host(qzc_context *ctx, const uint8_t *payloads, const uint64_t *offsets,
                        const uint32_t *sizes, const uint32_t *crcs, uint64_t count,
                        uint64_t elements, uint64_t chunk_index_base, double *amps_out) {
    QZ_API_BEGIN
    std::lock_guard<std::mutex> lk(ctx->mu);
    QZ_CUDA(cudaSetDevice(ctx->device));
    if (elements == 0 || (elements & (elements - 1)))
        throw Failure(QZC_ECODEC, "chunk length must be a power of two");
    if (count == 0) return QZC_OK;
    cudaStream_t s = ctx->stream;
    // codec id comes from the first payload's header byte (CompressedChunk::codec_id)
    uint64_t span = 0;
    for (uint64_t i = 0; i < count; ++i) span = std::max<uint64_t>(span, offsets[i] + sizes[i]);
    const uint8_t id = sizes[0] ? payloads[offsets[0]] : 2;
    CodecGeom g = make_geom(elements, id == 1 ? 1.0 : 0.0);
    uint64_t total = 0;
    for (uint64_t i = 0; i < count; ++i) total += sizes[i];
    g.dense_hint = total > count * elements ? 1u : 0u;   // compresses less than 16x
    g.enc_dense = g.dense_hint;
    ctx->win.reserve(g, count);
    ctx->arena.ensure(span + 64);
    ctx->table_off.ensure(8 * count);
    ctx->table_len.ensure(4 * count);
    ctx->table_crc.ensure(4 * count);
    QZ_CUDA(cudaMemcpyAsync(ctx->arena.p, payloads, span, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(ctx->table_off.p, offsets, 8 * count, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(ctx->table_len.p, sizes, 4 * count, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(ctx->table_crc.p, crcs, 4 * count, cudaMemcpyHostToDevice, s));
    ChunkTable t{ctx->table_off.as<uint64_t>(), ctx->table_len.as<uint32_t>(), ctx->table_crc.as<uint32_t>()};
    // CRC first, exactly like codec.cpp:188 (a bad checksum must not reach the parser)
    launch_crc(ctx->tabs, ctx->arena.as<uint8_t>(), t, nullptr, count, true, ctx->status, s);
    ctx->check_status(chunk_index_base);
    decode_window(ctx, ctx->win, g, count, nullptr, ctx->arena.as<uint8_t>(), t, ctx->launches);
    ctx->check_status(chunk_index_base);
    QZ_CUDA(cudaMemcpyAsync(amps_out, ctx->win.amps.p, 16 * count * elements, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaStreamSynchronize(s));
    QZ_API_END
}

// ---- gate entry points ------------------------------------------------------

static void check_bits(uint32_t nq, const uint32_t *q, uint32_t nbits) {
    for (uint32_t k = 0; k < nq; ++k)
        if (q[k] >= nbits)
            throw Failure(QZC_EDEVICE, "buffer bit " + std::to_string(q[k]) +
                                           " out of range for batch of 2^" + std::to_string(nbits) +
                                           " amplitudes");
}

static void run_dev_gates(qzc_context *ctx, double *amps_dev, uint32_t nbits,
                          const std::vector<DevGate> &dg, bool fuse = true);

static void apply_gates_device(qzc_context *ctx, double *amps_dev, uint32_t nbits,
                               const qzc_gate *gates, uint64_t ngates, bool fuse = true) {
    std::vector<DevGate> dg;
    dg.reserve(ngates);
    for (uint64_t i = 0; i < ngates; ++i) {
        const qzc_gate &g = gates[i];
        if (g.kind > QZC_SWAP) throw Failure(QZC_EINVAL, "unknown gate kind");
        if (g.nqubits != gate_arity(g.kind)) throw Failure(QZC_EINVAL, "gate arity mismatch");
        check_bits(g.nqubits, g.qubits, nbits);
        dg.push_back(make_dev_gate(g));
    }
    run_dev_gates(ctx, amps_dev, nbits, dg, fuse);
}

static void run_dev_gates(qzc_context *ctx, double *amps_dev, uint32_t nbits,
                          const std::vector<DevGate> &dg, bool fuse) {
    if (dg.empty()) return;
    GatePlan plan = build_passes(dg, nbits, kTileBits, fuse);
    DevPlan dp;
    upload_plan(plan, dp, ctx->stream);
    ctx->launches += run_passes(dp, reinterpret_cast<double2 *>(amps_dev), nbits, ctx->stream);
    QZ_CUDA(cudaStreamSynchronize(ctx->stream));
    free_plan(dp);
}

static std::vector<DevGate> matrix_gates(const qzc_matrix_gate *gates, uint64_t ngates,
                                         uint32_t nbits) {
    std::vector<DevGate> dg;
    for (uint64_t i = 0; i < ngates; ++i) {
        const qzc_matrix_gate &g = gates[i];
        check_bits(g.dim == 4 ? 2 : 1, g.qubits, nbits);
        dg.push_back(make_dev_gate_matrix(reinterpret_cast<const double2 *>(g.m), g.dim, g.qubits[0],
                                          g.qubits[1]));
    }
    return dg;
}

int qzc_apply_matrices_dev(qzc_context *ctx, double *amps_dev, uint32_t nbits,
                           const qzc_matrix_gate *gates, uint64_t ngates) {
    QZ_API_BEGIN
    std::lock_guard<std::mutex> lk(ctx->mu);
    QZ_CUDA(cudaSetDevice(ctx->device));
    run_dev_gates(ctx, amps_dev, nbits, matrix_gates(gates, ngates, nbits));
    QZ_API_END
}

int qzc_apply_matrices_host(qzc_context *ctx, double *amps, uint32_t nbits,
                            const qzc_matrix_gate *gates, uint64_t ngates) {
    QZ_API_BEGIN
    std::lock_guard<std::mutex> lk(ctx->mu);
    QZ_CUDA(cudaSetDevice(ctx->device));
    const std::vector<DevGate> dg = matrix_gates(gates, ngates, nbits);
    const uint64_t bytes = 16ull << nbits;
    DevBuf buf;
    buf.ensure(bytes);
    QZ_CUDA(cudaMemcpyAsync(buf.p, amps, bytes, cudaMemcpyHostToDevice, ctx->stream));
    run_dev_gates(ctx, buf.as<double>(), nbits, dg);
    QZ_CUDA(cudaMemcpyAsync(amps, buf.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    QZ_CUDA(cudaStreamSynchronize(ctx->stream));
    buf.release();
    QZ_API_END
}

int qzc_apply_matrix_range_host(qzc_context *ctx, double *amps, uint32_t nbits, const qzc_matrix_gate *gate,
                                uint64_t begin, uint64_t end) {
    QZ_API_BEGIN
    if (!ctx || !amps || !gate) throw Failure(QZC_EINVAL, "null argument");
    if (gate->dim != 2 && gate->dim != 4) throw Failure(QZC_EINVAL, "matrix dimension must be 2 or 4");
    const uint32_t nq = gate->dim == 2 ? 1 : 2;
    for (uint32_t k = 0; k < nq; ++k)
        if (gate->qubits[k] >= nbits)
            throw Failure(QZC_EDEVICE, "buffer bit " + std::to_string(gate->qubits[k]) + " out of range");
    if (nq == 2 && gate->qubits[0] == gate->qubits[1]) throw Failure(QZC_EINVAL, "duplicate qubit");
    const uint64_t units = uint64_t(1) << (nbits - nq);
    if (begin > end || end > units) throw Failure(QZC_EINVAL, "range outside the buffer's pairs / groups");
    if (begin == end) return QZC_OK;
    std::lock_guard<std::mutex> lk(ctx->mu);
    QZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    // the touched amplitudes lie in the index span of the range's first /
    // last unit shifted by each partner offset: copy only those spans
    const uint32_t b0 = gate->qubits[0], b1 = nq == 2 ? gate->qubits[1] : 0;
    auto first_index = [&](uint64_t u) {
        if (nq == 1) return insert_zero_bit(u, b0);
        const uint32_t lo = std::min(b0, b1), hi = std::max(b0, b1);
        return insert_zero_bit(insert_zero_bit(u, lo), hi);
    };
    const uint64_t f0 = first_index(begin), f1 = first_index(end - 1);
    std::vector<uint64_t> offs{0, uint64_t(1) << b0};
    if (nq == 2) offs = {0, uint64_t(1) << b0, uint64_t(1) << b1, (uint64_t(1) << b0) | (uint64_t(1) << b1)};
    std::vector<std::pair<uint64_t, uint64_t>> spans;
    for (uint64_t o : offs) spans.push_back({f0 + o, f1 + o + 1});
    std::sort(spans.begin(), spans.end());
    std::vector<std::pair<uint64_t, uint64_t>> merged;
    for (auto sp : spans) {
        if (!merged.empty() && sp.first <= merged.back().second) merged.back().second = std::max(merged.back().second, sp.second);
        else merged.push_back(sp);
    }
    DevBuf buf, mat;
    buf.ensure(16ull << nbits);
    mat.ensure(16 * 16);
    double2 m[16];
    for (uint32_t e = 0; e < gate->dim * gate->dim; ++e) m[e] = make_double2(gate->m[2 * e], gate->m[2 * e + 1]);
    QZ_CUDA(cudaMemcpyAsync(mat.p, m, sizeof m, cudaMemcpyHostToDevice, s));
    double2 *d = buf.as<double2>();
    const double2 *h = reinterpret_cast<const double2 *>(amps);
    for (auto sp : merged)
        QZ_CUDA(cudaMemcpyAsync(d + sp.first, h + sp.first, 16 * (sp.second - sp.first), cudaMemcpyHostToDevice, s));
    k_apply_range<<<(unsigned)ceil_div(end - begin, 256), 256, 0, s>>>(d, gate->dim, b0, b1, mat.as<double2>(), begin,
                                                                       end);
    QZ_CHECK_LAUNCH();
    ++ctx->launches;
    for (auto sp : merged)
        QZ_CUDA(cudaMemcpyAsync(reinterpret_cast<double2 *>(amps) + sp.first, d + sp.first,
                                16 * (sp.second - sp.first), cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaStreamSynchronize(s));
    QZ_API_END
}

int qzc_apply_gates_dev(qzc_context *ctx, double *amps_dev, uint32_t nbits, const qzc_gate *gates,
                        uint64_t ngates) {
    QZ_API_BEGIN
    std::lock_guard<std::mutex> lk(ctx->mu);
    QZ_CUDA(cudaSetDevice(ctx->device));
    apply_gates_device(ctx, amps_dev, nbits, gates, ngates);
    QZ_API_END
}

int qzc_apply_gates_host(qzc_context *ctx, double *amps, uint32_t nbits, const qzc_gate *gates,
                         uint64_t ngates) {
    QZ_API_BEGIN
    std::lock_guard<std::mutex> lk(ctx->mu);
    QZ_CUDA(cudaSetDevice(ctx->device));
    const uint64_t bytes = 16ull << nbits;
    DevBuf buf;
    buf.ensure(bytes);
    QZ_CUDA(cudaMemcpyAsync(buf.p, amps, bytes, cudaMemcpyHostToDevice, ctx->stream));
    apply_gates_device(ctx, buf.as<double>(), nbits, gates, ngates);
    QZ_CUDA(cudaMemcpyAsync(amps, buf.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    QZ_CUDA(cudaStreamSynchronize(ctx->stream));
    buf.release();
    QZ_API_END
}

// ---- device buffers ---------------------------------------------------------------

namespace {
__global__ void k_copy(double2 *dst, const double2 *src, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}
} // namespace

int qzc_buffer_alloc(qzc_context *ctx, uint64_t amps, double **dev_out) {
    QZ_API_BEGIN
    QZ_CUDA(cudaSetDevice(ctx->device));
    void *p = nullptr;
    QZ_CUDA(cudaMalloc(&p, 16 * std::max<uint64_t>(amps, 1)));
    *dev_out = static_cast<double *>(p);
    QZ_API_END
}

void qzc_buffer_free(qzc_context *ctx, double *dev) {
    if (ctx) cudaSetDevice(ctx->device);
    cudaFree(dev);
}

int qzc_copy_h2d(qzc_context *ctx, double *dev, uint64_t dev_offset, const double *host,
                 uint64_t amps) {
    QZ_API_BEGIN
    QZ_CUDA(cudaMemcpyAsync(dev + 2 * dev_offset, host, 16 * amps, cudaMemcpyHostToDevice,
                            ctx->stream));
    QZ_API_END
}

int qzc_copy_d2h(qzc_context *ctx, double *host, const double *dev, uint64_t dev_offset,
                 uint64_t amps) {
    QZ_API_BEGIN
    QZ_CUDA(cudaMemcpyAsync(host, dev + 2 * dev_offset, 16 * amps, cudaMemcpyDeviceToHost,
                            ctx->stream));
    QZ_API_END
}

int qzc_permute(qzc_context *ctx, double *dst, const double *src, uint64_t amps) {
    QZ_API_BEGIN
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(amps, 256), kNumSMs * 32);
    k_copy<<<std::max(grid, 1u), 256, 0, ctx->stream>>>(reinterpret_cast<double2 *>(dst),
                                                     reinterpret_cast<const double2 *>(src), amps);
    QZ_CHECK_LAUNCH();
    ++ctx->launches;
    QZ_API_END
}

int qzc_host_alloc(qzc_context *ctx, uint64_t bytes, void **host_out) {
    QZ_API_BEGIN
    QZ_CUDA(cudaSetDevice(ctx->device));
    QZ_CUDA(cudaMallocHost(host_out, std::max<uint64_t>(bytes, 1)));
    QZ_API_END
}

void qzc_host_free(qzc_context *ctx, void *host) {
    (void)ctx;
    cudaFreeHost(host);
}

int qzc_event_record(qzc_context *ctx, void **event_out) {
    QZ_API_BEGIN
    cudaEvent_t e;
    QZ_CUDA(cudaEventCreate(&e));
    QZ_CUDA(cudaEventRecord(e, ctx->stream));
    *event_out = e;
    QZ_API_END
}

int qzc_event_elapsed(qzc_context *ctx, void *start, void *end, double *seconds_out) {
    QZ_API_BEGIN
    (void)ctx;
    QZ_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(end)));
    float ms = 0;
    QZ_CUDA(cudaEventElapsedTime(&ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(end)));
    *seconds_out = ms * 1e-3;
    QZ_API_END
}

int qzc_event_done(qzc_context *ctx, void *event) {
    (void)ctx;
    return cudaEventQuery(static_cast<cudaEvent_t>(event)) == cudaSuccess ? 1 : 0;
}

void qzc_event_destroy(qzc_context *ctx, void *event) {
    (void)ctx;
    if (event) cudaEventDestroy(static_cast<cudaEvent_t>(event));
}

// ---- simulator -----------------------------------------------------------------

int qzc_sim_create(qzc_context *ctx, const qzc_sim_config *cfg, qzc_sim **out) {
    QZ_API_BEGIN
    if (!ctx || !cfg || !out) throw Failure(QZC_EINVAL, "null argument");
    QZ_CUDA(cudaSetDevice(ctx->device));
    const uint32_t n = cfg->num_qubits, c = cfg->chunk_qubits;
    // ChunkStore::init_basis_state geometry checks (store.cpp:29-35)
    if (c < 1 || c > n)
        throw Failure(QZC_ESTORE, "chunk qubits must satisfy 1 <= c <= n, got c=" + std::to_string(c) +
                                      ", n=" + std::to_string(n));
    if (n > 40) throw Failure(QZC_ESTORE, "qubit count exceeds configured address width (40)");
    if (!(cfg->error_bound >= 0.0) || !std::isfinite(cfg->error_bound))
        throw Failure(QZC_EINVAL, "error bound must be finite and non-negative");
    if (cfg->residency > 1) throw Failure(QZC_EINVAL, "residency must be 0 (HBM) or 1 (host-staged)");
    if (cfg->fuse_gates > 3) throw Failure(QZC_EINVAL, "fuse_gates must be 0, 1, 2 or 3");
    auto *sim = new qzc_sim;
    sim->ctx = ctx;
    sim->cfg = *cfg;
    sim->relax = cfg->fuse_gates == 1 ? 1 : (cfg->fuse_gates == 3 ? 2 : 0);
    sim->force_replay = (cfg->debug_flags & 1u) != 0;
    sim->n = n;
    sim->c = c;
    sim->m = cfg->batch_qubits;
    sim->eb = cfg->error_bound;
    sim->N = uint64_t(1) << c;
    sim->nchunks = uint64_t(1) << (n - c);
    sim->geom = make_geom(sim->N, sim->eb);
    sim->host_res = cfg->residency == 1;
    try {
        sim_alloc(sim);
    } catch (...) {
        delete sim;
        throw;
    }
    *out = sim;
    QZ_API_END
}

void qzc_sim_destroy(qzc_sim *sim) {
    if (!sim) return;
    cudaSetDevice(sim->ctx->device);
    cudaStreamSynchronize(sim->ctx->stream);
    for (int i = 0; i < 3; ++i)
        if (sim->streams[i]) cudaStreamSynchronize(sim->streams[i]);
    for (int i = 0; i < 2; ++i)
        for (DevBuf *b : {&sim->arena[i], &sim->off[i], &sim->len[i], &sim->crc[i]}) b->release();
    sim->used.release();
    sim->acct.release();
    sim->io_bytes.release();
    sim->replays.release();
    sim->small.release();
    sim->gcub.release();
    for (DevPlan &p : sim->plans) free_plan(p);
    for (int i = 0; i < 2; ++i)
        if (sim->harena[i]) cudaFreeHost(sim->harena[i]);
    sim->win.release();
    sim->win2.release();
    for (int i = 0; i < 3; ++i) {
        if (sim->streams[i]) {
            cudaStreamSynchronize(sim->streams[i]);
            cudaStreamDestroy(sim->streams[i]);
        }
    }
    for (int i = 0; i < 2; ++i)
        if (sim->acct_ev[i]) cudaEventDestroy(sim->acct_ev[i]);
    for (cudaEvent_t e : sim->events) cudaEventDestroy(e);
    for (cudaEvent_t e : sim->pevents) cudaEventDestroy(e);
    delete sim;
}

namespace {
// |0...0> (basis = true, store.cpp:26-81) or the zero vector (every chunk the
// zero-chunk payload: the non-zero ranks of a sharded |0...0>).
void init_store(qzc_sim *sim, bool basis);
} // namespace

int qzc_sim_init_basis(qzc_sim *sim) {
    QZ_API_BEGIN
    init_store(sim, true);
    QZ_API_END
}

int qzc_sim_init_zero(qzc_sim *sim) {
    QZ_API_BEGIN
    init_store(sim, false);
    QZ_API_END
}

namespace {
void init_store(qzc_sim *sim, bool basis) {
    qzc_context *ctx = sim->ctx;
    sim->fresh_q = basis ? ((sim->n >= 64 ? ~uint64_t(0) : (uint64_t(1) << sim->n) - 1)) : 0;
    sim->fresh_v = 0;
    QZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    Window &w = sim->win;
    const uint64_t N = sim->N;
    const int a = sim->cur;
    static const bool trace = getenv("QZ_TRACE") && *getenv("QZ_TRACE") == '1';
    const double ti0 = now_s();
    kprof_set_stage(0xFFFFFFFFu);   // init launches are tagged apart from the stages
    QZ_CUDA(cudaMemsetAsync(sim->used.p, 0, 16, s));
    static const bool no_cache = getenv("QZ_NO_INIT_CACHE") != nullptr;
    if (basis && sim->init_cache.valid && !no_cache) {
        // the same two payloads as the first init produced (same bytes, CRCs
        // and offsets): copy them back instead of re-encoding
        const auto &ic = sim->init_cache;
        const int a = sim->cur;
        QZ_CUDA(cudaMemcpyAsync(sim->arena_ptr(a), ic.bytes.data(), ic.bytes.size(), cudaMemcpyHostToDevice, s));
        QZ_CUDA(cudaMemcpyAsync(sim->used_ptr(a), &ic.used, 8, cudaMemcpyHostToDevice, s));
        k_fill_init<<<(unsigned)ceil_div(sim->nchunks, 256), 256, 0, s>>>(
            sim->table(a), sim->nchunks, ic.off[0], ic.len[0], ic.crc[0], ic.off[1], ic.len[1], ic.crc[1]);
        QZ_CHECK_LAUNCH();
        const int64_t bytes = int64_t(ic.len[1] + kPerChunkOverhead) +
                              int64_t(sim->nchunks - 1) * int64_t(ic.len[0] + kPerChunkOverhead);
        const int64_t acct[2] = {bytes, bytes};
        QZ_CUDA(cudaMemcpyAsync(sim->acct.p, acct, 16, cudaMemcpyHostToDevice, s));
        if (sim->host_res) QZ_CUDA(cudaMemsetAsync(sim->io_bytes.p, 0, 16, s));
        QZ_CUDA(cudaMemsetAsync(sim->replays.p, 0, 8, s));
        QZ_CUDA(cudaStreamSynchronize(s));   // (the pageable sources above)
        sim->initialized = true;
        sim->sparse_store = true;
        sim->stats = qzc_sim_stats{};
        sim->payload_now = uint64_t(bytes) - kPerChunkOverhead * sim->nchunks;
        return;
    }
    // slot 0 = zero chunk, slot 1 = basis chunk (store.cpp:46-51)
    QZ_CUDA(cudaMemsetAsync(w.amps.p, 0, 32 * N, s));
    const double one[2] = {1.0, 0.0};
    QZ_CUDA(cudaMemcpyAsync(w.amps.as<double2>() + N, one, 16, cudaMemcpyHostToDevice, s));
    ChunkTable t = sim->table(a);
    encode_window(ctx, w, sim->geom, 2, nullptr, nullptr, 0, sim->arena_ptr(a),
                  sim->used_ptr(a), sim->cap(a), t, nullptr, nullptr, ctx->launches);
    ctx->check_status();
    const double ti1 = now_s();
    if (sim->eb > 0.0) {
        // decode the basis chunk; route {0,1} through the raw path if the
        // quantiser perturbed it (store.cpp:52-67)
        static const uint64_t kSmall[4] = {1, 0, 1, 0};   // slot list {1}, forced list {0, 1}
        QZ_CUDA(cudaMemcpyAsync(sim->small.p, kSmall, sizeof kSmall, cudaMemcpyHostToDevice, s));
        const uint64_t *sc = sim->small.as<uint64_t>();
        decode_window(ctx, w, sim->geom, 1, sc, sim->arena_ptr(a), t, ctx->launches);
        ctx->check_status();
        std::vector<double2> r(N);
        QZ_CUDA(cudaMemcpyAsync(r.data(), w.amps.p, 16 * N, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaStreamSynchronize(s));
        bool exact = std::fabs(r[0].x - 1.0) <= 1e-12;
        for (uint64_t i = 0; exact && i < N; ++i)
            if (r[i].y != 0.0 || (i > 0 && r[i].x != 0.0)) exact = false;
        if (!exact) {
            QZ_CUDA(cudaMemsetAsync(w.amps.p, 0, 16 * N, s));
            QZ_CUDA(cudaMemcpyAsync(w.amps.p, one, 16, cudaMemcpyHostToDevice, s));
            encode_window(ctx, w, sim->geom, 1, sc, sc + 1, N > 1 ? 2u : 1u,
                          sim->arena_ptr(a), sim->used_ptr(a), sim->cap(a), t, nullptr,
                          nullptr, ctx->launches);
            ctx->check_status();
        }
    }
    uint64_t off2[2];
    uint32_t len2[2], crc2[2];
    QZ_CUDA(cudaMemcpyAsync(off2, t.off, 16, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaMemcpyAsync(len2, t.len, 8, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaMemcpyAsync(crc2, t.crc, 8, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaStreamSynchronize(s));
    if (!basis) {
        off2[1] = off2[0];
        len2[1] = len2[0];
        crc2[1] = crc2[0];
    }
    k_fill_init<<<(unsigned)ceil_div(sim->nchunks, 256), 256, 0, s>>>(
        t, sim->nchunks, off2[0], len2[0], crc2[0], off2[1], len2[1], crc2[1]);
    QZ_CHECK_LAUNCH();
    if (basis && !sim->init_cache.valid) {
        auto &ic = sim->init_cache;
        QZ_CUDA(cudaMemcpyAsync(&ic.used, sim->used_ptr(a), 8, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaStreamSynchronize(s));
        ic.bytes.resize(ic.used);
        if (ic.used) QZ_CUDA(cudaMemcpy(ic.bytes.data(), sim->arena_ptr(a), ic.used, cudaMemcpyDeviceToHost));
        for (int i = 0; i < 2; ++i) {
            ic.off[i] = off2[i];
            ic.len[i] = len2[i];
            ic.crc[i] = crc2[i];
        }
        ic.valid = ic.used <= (uint64_t(1) << 20);   // (two chunk payloads: small)
    }
    const int64_t bytes = int64_t(len2[1] + kPerChunkOverhead) +
                          int64_t(sim->nchunks - 1) * int64_t(len2[0] + kPerChunkOverhead);
    const int64_t acct[2] = {bytes, bytes};
    QZ_CUDA(cudaMemcpyAsync(sim->acct.p, acct, 16, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaStreamSynchronize(s));
    sim->initialized = true;
    sim->sparse_store = true;
    sim->stats = qzc_sim_stats{};
    sim->payload_now = uint64_t(bytes) - kPerChunkOverhead * sim->nchunks;
    if (sim->host_res) QZ_CUDA(cudaMemset(sim->io_bytes.p, 0, 16));
    QZ_CUDA(cudaMemset(sim->replays.p, 0, 8));
    if (trace)
        fprintf(stderr, "qz trace: init encode %.2f ms total %.2f ms\n", 1e3 * (ti1 - ti0),
                1e3 * (now_s() - ti0));
}
} // namespace

int qzc_pass_plan_stats(const qzc_gate *gates, uint64_t ngates, uint32_t nbits,
                        uint32_t fuse_mode, uint64_t *out) {
    QZ_API_BEGIN
    if (fuse_mode > 3 || nbits > 40) throw Failure(QZC_EINVAL, "bad fuse mode / buffer width");
    const std::string err = validate_gates(nbits, gates, ngates);
    if (!err.empty()) throw Failure(QZC_EINVAL, err);
    std::vector<DevGate> dg;
    for (uint64_t i = 0; i < ngates; ++i) dg.push_back(make_dev_gate(gates[i]));
    // QZ_PLAN_FRESH=1 (inspection): plan as for a store fresh from init_basis
    Fresh fr;
    if (getenv("QZ_PLAN_FRESH")) fr.mask = (uint64_t(1) << nbits) - 1;
    const GatePlan p = build_passes(dg, nbits, kTileBits, fuse_mode != 0,
                                    fuse_mode == 1 ? 1 : (fuse_mode == 3 ? 2 : 0), &fr,
                                    getenv("QZ_PLAN_PERM") != nullptr);
    uint64_t relaxed = 0, fast = 0, pdiag = 0;
    for (const GroupDesc &g : p.groups) {
        relaxed += g.relaxed;
        fast += g.nfast;
        for (uint32_t q = 0; q < g.nfast; ++q) pdiag += p.gates[g.first_fast + q].op == OP_PDIAG;
    }
    out[0] = p.passes.size();
    out[1] = p.groups.size();
    out[2] = relaxed;
    out[3] = ngates;
    out[4] = fast;
    out[5] = pdiag;
    QZ_API_END
}

int qzc_plan_export(uint32_t num_qubits, uint32_t chunk_qubits, uint32_t batch_qubits,
                    const qzc_gate *gates, uint64_t ngates, uint64_t *nstages,
                    uint64_t *first_gate, uint64_t *stage_ngates, uint32_t *nhigh,
                    uint32_t *high, uint64_t cap) {
    QZ_API_BEGIN
    const std::vector<Stage> st = plan_stages(num_qubits, gates, ngates, chunk_qubits, batch_qubits);
    *nstages = st.size();
    for (size_t i = 0; i < st.size() && i < cap; ++i) {
        first_gate[i] = st[i].first_gate;
        stage_ngates[i] = st[i].ngates;
        nhigh[i] = uint32_t(st[i].high.size());
        for (size_t k = 0; k < st[i].high.size() && k < 64; ++k) high[64 * i + k] = st[i].high[k];
    }
    QZ_API_END
}

int qzc_sim_plan_stages(const qzc_sim *sim, const qzc_gate *gates, uint64_t ngates,
                        uint64_t *stages_out) {
    QZ_API_BEGIN
    *stages_out = plan_stages(sim->n, gates, ngates, sim->c, sim->m).size();
    QZ_API_END
}

int qzc_sim_run(qzc_sim *sim, const qzc_gate *gates, uint64_t ngates) {
    QZ_API_BEGIN
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    if (!sim->initialized) throw Failure(QZC_ESTORE, "store not initialised");
    // non-parity fast mode: the whole circuit as one stage when the dense
    // state fits the window (else the reference's stage semantics)
    const bool one_stage = sim->cfg.skip_reencode && !sim->host_res && sim->win_amps >= (uint64_t(1) << sim->n);
    const std::vector<Stage> stages = plan_stages(sim->n, gates, ngates, sim->c, one_stage ? sim->n : sim->m);
    cudaStream_t s = ctx->stream;
    const uint32_t n = sim->n, c = sim->c;
    const uint64_t chunk_bits_mask = (uint64_t(1) << (n - c)) - 1;
    const uint64_t launches0 = ctx->launches;
    const double t0 = now_s();
    static const bool trace = getenv("QZ_TRACE") && *getenv("QZ_TRACE") == '1';
    // 4 events per window, recycled per stage
    auto ev = [&](size_t i) {
        while (sim->events.size() <= i) {
            cudaEvent_t e;
            QZ_CUDA(cudaEventCreate(&e));
            sim->events.push_back(e);
        }
        return sim->events[i];
    };
    for (size_t si = 0; si < stages.size(); ++si) {
        const Stage &st = stages[si];
        kprof_set_stage(uint32_t(sim->stats.stages));
        // decoder choice for this stage's input: dense stores (ratio < 16)
        // take the segmented kernel, sparse ones the run-filling warp kernel
        sim->geom.dense_hint = sim->payload_now > (uint64_t(1) << sim->n) ? 1u : 0u;
        const uint32_t hs = (uint32_t)st.high.size();
        const uint32_t mb = c + hs;  // buffer bits of one batch
        uint64_t smask = 0;
        for (uint32_t q : st.high) smask |= uint64_t(1) << (q - c);
        const uint64_t fmask = chunk_bits_mask & ~smask;
        const uint64_t nbatches = uint64_t(1) << ((n - c) - hs);
        uint64_t bpw = std::max<uint64_t>(1, sim->win_amps >> mb);
        bpw = std::min(bpw, nbatches);
        const uint32_t wbits = mb + log2u(bpw);
        // A stage that ends in a network of disjoint SWAPs (permutation pi of
        // qubits) whose moved qubits are all fresh with pi-symmetric values:
        // the live amplitudes are fixed by pi, so the decoded window is also
        // the window laid out with qubit q on buffer bit pi(q).  Run the stage
        // in that layout and the network is only a relabelling: at the stage's
        // end the window holds the state in the natural layout (no permutation
        // pass).  QFT from |0...0>: the bit reversal, and the qubits it opens
        // last sit on the high buffer bits (contiguous live data throughout).
        std::vector<uint32_t> relabel(n);
        for (uint32_t q = 0; q < n; ++q) relabel[q] = q;
        size_t ngates_run = st.ngates;
        {
            static const bool no_absorb = getenv("QZ_NO_ABSORB") != nullptr || getenv("QZ_NO_FRESH") != nullptr;
            uint64_t used_q = 0;
            size_t first = st.ngates;
            while (first > 0) {
                const qzc_gate &g = gates[st.first_gate + first - 1];
                if (g.kind != QZC_SWAP || g.nqubits != 2) break;
                const uint64_t m2 = (uint64_t(1) << g.qubits[0]) | (uint64_t(1) << g.qubits[1]);
                if ((used_q & m2) || g.qubits[0] == g.qubits[1]) break;
                used_q |= m2;
                --first;
            }
            bool ok = !no_absorb && first < st.ngates;
            for (size_t i = first; ok && i < st.ngates; ++i) {
                const qzc_gate &g = gates[st.first_gate + i];
                const uint32_t a = g.qubits[0], b = g.qubits[1];
                ok = buffer_bit(st, a, c) >= 0 && buffer_bit(st, b, c) >= 0 && ((sim->fresh_q >> a) & 1) &&
                     ((sim->fresh_q >> b) & 1) && (((sim->fresh_v >> a) ^ (sim->fresh_v >> b)) & 1) == 0;
            }
            if (ok) {
                for (size_t i = first; i < st.ngates; ++i) {
                    const qzc_gate &g = gates[st.first_gate + i];
                    relabel[g.qubits[0]] = g.qubits[1];
                    relabel[g.qubits[1]] = g.qubits[0];
                }
                ngates_run = first;
            }
        }
        // relaxed plan (diagonal units need no tile bits) + the strict plan
        // it is replayed with, device-side, when a window raises the flag
        const double tp0 = now_s();
        // fresh buffer bits at the stage's start (qubits still |0>)
        Fresh stage_fresh;
        static const bool no_fresh = getenv("QZ_NO_FRESH") != nullptr;   // control
        for (uint32_t q = 0; q < n && !no_fresh; ++q)
            if ((sim->fresh_q >> q) & 1) {
                const int bq = buffer_bit(st, relabel[q], c);
                if (bq >= 0) {
                    stage_fresh.mask |= uint64_t(1) << bq;
                    stage_fresh.val |= ((sim->fresh_v >> q) & 1) << bq;
                }
            }
        const uint64_t nwin = nbatches / bpw;
        const uint64_t nslots = bpw << hs;
        CodecGeom dgeom = sim->geom;
        Fresh end_fresh;
        bool dead_chunks = false;
        {
            // out-of-place checked passes exist only with relax level 2
            const bool out_of_place = sim->relax == 2;
            // chunk-index bits of the stage's fresh high qubits (only those:
            // the passes know the stage's buffer bits alone)
            uint64_t fq = 0, fv = 0;
            for (uint32_t q : st.high)
                if ((sim->fresh_q >> q) & 1) {
                    fq |= uint64_t(1) << (q - c);
                    fv |= ((sim->fresh_v >> q) & 1) << (q - c);
                }
            dead_chunks = !no_fresh && !sim->host_res && !out_of_place && fq && wbits >= 5;
            if (dead_chunks) {
                dgeom.dead_mask = fq;
                dgeom.dead_val = fv;
            }
        }
        // HBM store, one stream per window: the first window's decode does
        // not depend on the plan, so it is issued before planning and runs
        // while the host plans
        const bool pre_decode = !sim->host_res && !sim->pipelined;
        if (pre_decode) {
            Window &W0 = sim->win;
            cudaStream_t S0 = sim->streams[0];
            QZ_CUDA(cudaEventRecord(ev(0), S0));
            launch_slot_chunks(W0.slot_chunk.as<uint64_t>(), nslots, 0, hs, fmask, smask, S0);
            decode_window(ctx, W0, dgeom, nslots, W0.slot_chunk.as<uint64_t>(), sim->arena_ptr(sim->cur),
                          sim->table(sim->cur), ctx->launches, S0, sim->sparse_store);
            QZ_CUDA(cudaEventRecord(ev(1), S0));
        }
        // (the gate list is built while the first window decodes)
        // remap the stage's gates to buffer bits (remap_gate, planner.cpp:131-141)
        std::vector<DevGate> dg;
        dg.reserve(ngates_run);
        for (size_t i = 0; i < ngates_run; ++i) {
            qzc_gate g = gates[st.first_gate + i];
            for (uint32_t k = 0; k < g.nqubits; ++k) {
                const int b = buffer_bit(st, relabel[g.qubits[k]], c);
                if (b < 0) throw Failure(QZC_EPLAN, "qubit not mapped by the stage layout");
                g.qubits[k] = uint32_t(b);
            }
            dg.push_back(make_dev_gate(g));
        }
        {
            // encoder choice for this stage's output: dense when the input
            // is, or when some qubit sees >= 4 mixing gates (a row with two
            // nonzero entries: H, sqrt-X, U3 ...; random-circuit layers)
            uint32_t mix[64] = {}, most = 0;
            for (const DevGate &d : dg) {
                bool mixing = false;
                for (uint32_t r = 0; r < d.dim && !mixing; ++r) {
                    uint32_t nz = 0;
                    for (uint32_t k = 0; k < d.dim; ++k)
                        nz += ((d.kinds >> (4 * (r * d.dim + k))) & 15u) != CK_ZERO;
                    mixing = nz > 1;
                }
                if (!mixing) continue;
                most = std::max(most, ++mix[d.b0]);
                if (d.nq == 2) most = std::max(most, ++mix[d.b1]);
            }
            sim->geom.enc_dense = sim->geom.dense_hint || most >= 4 ? 1u : 0u;
        }
        if (dead_chunks) end_fresh = fresh_after(dg, 0, dg.size(), stage_fresh);
        if (trace)
            fprintf(stderr, "qz trace: stage %zu dead-chunk mask %#llx val %#llx end-fresh %#llx pipelined %d\n", si,
                    (unsigned long long)dgeom.dead_mask, (unsigned long long)dgeom.dead_val,
                    (unsigned long long)end_fresh.mask, int(sim->pipelined));
        // a swap network after a tile pass is fused into its store (out of
        // place: needs the second window buffer; QZ_NO_PERM_FUSE=1 keeps the
        // separate swap pass)
        static const bool no_perm = getenv("QZ_NO_PERM_FUSE") != nullptr;
        GatePlan gp = build_passes(dg, wbits, kTileBits, sim->cfg.fuse_gates != 0, sim->relax, &stage_fresh,
                                   !no_perm);
        {
            bool perm = false;
            for (const PassDesc &pd : gp.passes) perm |= pd.permute != 0;
            if (perm) {
                try {
                    sim->win.alt.ensure(sim->win.amps.cap);
                    if (sim->two_windows) sim->win2.alt.ensure(sim->win2.amps.cap);
                } catch (const Failure &) {
                    (void)cudaGetLastError();   // out of memory: the unfused plan
                    gp = build_passes(dg, wbits, kTileBits, sim->cfg.fuse_gates != 0, sim->relax, &stage_fresh, false);
                }
            }
        }
        DevPlan &dp = sim->plans[0], &dsub = sim->plans[1], &dfull = sim->plans[2];
        std::vector<Fresh> pass_fresh;
        {
            Fresh f = stage_fresh;
            size_t at = 0;
            for (const PassDesc &pd : gp.passes) {
                f = fresh_after(dg, at, pd.dg0, f);
                at = pd.dg0;
                pass_fresh.push_back(f);
            }
        }
        upload_plan(gp, dp, s, wbits, pass_fresh);
        dsub.host_passes.clear();
        dfull.host_passes.clear();
        bool need_dfull = false;
        if (dp.relaxed) {
            upload_replay(dg, wbits, kTileBits, dp, dsub, s);
            for (const PassDesc &pd : dp.host_passes) need_dfull |= pd.relaxed == 1;
        }
        // the whole-window strict plan (replayed device-side only when a +0-safe
        // relaxed pass flags): built lazily, once the first window's relaxed
        // passes are queued, so the host builds it while they run
        bool dfull_built = false;
        cudaEvent_t dfull_ready = ev(4 * nwin + 1);
        auto ensure_dfull = [&](cudaStream_t S) -> bool {
            if (!need_dfull) return false;
            if (!dfull_built) {
                upload_plan(build_passes(dg, wbits, kTileBits, true, false), dfull, S);
                QZ_CUDA(cudaEventRecord(dfull_ready, S));
                dfull_built = true;
            }
            QZ_CUDA(cudaStreamWaitEvent(S, dfull_ready, 0));
            return true;
        };
        const int a = sim->cur, b = 1 - sim->cur;
        // host-staged stores start with arenas sized for a typical ratio and
        // grow on demand: a stage whose output overflows its arena is re-run
        // from its (untouched) input arena after the output arena grew
        int64_t acct_before[2] = {0, 0};
        if (sim->host_res) QZ_CUDA(cudaMemcpy(acct_before, sim->acct.p, 16, cudaMemcpyDeviceToHost));
        // statically-(+0) chunks (fresh high qubits) are not decoded: every
        // pass zero-fills what it reads of them (PassDesc::fmask) and the
        // elements still +0 at the stage's end are zero-filled before the
        // encode.  Not with out-of-place passes (their replays read the
        // window as decoded) or the host-staged store.
        for (int attempt = 0;; ++attempt) {
        QZ_CUDA(cudaMemsetAsync(sim->used_ptr(b), 0, 8, s));
        // the stage's plan upload and arena reset happen on the context
        // stream; both window streams start after them
        cudaEvent_t ready = ev(4 * nwin);
        QZ_CUDA(cudaEventRecord(ready, s));
        const double tp1 = now_s();
        // pipeline events: 3 per window (gathered, encoded, written back)
        auto pev = [&](uint64_t i) {
            while (sim->pevents.size() <= i) {
                cudaEvent_t e;
                QZ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                sim->pevents.push_back(e);
            }
            return sim->pevents[i];
        };
        for (uint64_t w = 0; w < nwin && sim->pipelined; ++w) {
            // host-staged, one window: input set w&1 (slot map, staged payloads,
            // slot table, cursors) cycles gather -> decode -> write-back; the
            // window, scratch and output staging are shared and serialised
            Window &W = sim->win;
            Window &In = (w & 1) ? sim->win2 : sim->win;
            cudaStream_t SG = sim->streams[1], S = sim->streams[0], SO = sim->streams[2];
            // gather (H2D) of window w on SG, after the write-back of window
            // w-2 released this input set
            if (w < 2) QZ_CUDA(cudaStreamWaitEvent(SG, ready, 0));
            else QZ_CUDA(cudaStreamWaitEvent(SG, pev(3 * (w - 2) + 2), 0));
            launch_slot_chunks(In.slot_chunk.as<uint64_t>(), nslots, w * bpw, hs, fmask, smask, SG);
            launch_stage_sizes(sim->table(a), In.slot_chunk.as<uint64_t>(), nslots, In.padded.as<uint64_t>(), SG);
            size_t tb = sim->gcub.cap;
            QZ_CUDA(cub::DeviceScan::ExclusiveSum(sim->gcub.p, tb, In.padded.as<uint64_t>(), In.soff.as<uint64_t>(),
                                                  (int)nslots, SG));
            launch_gather(sim->arena_ptr(a), sim->table(a), In.slot_chunk.as<uint64_t>(), In.soff.as<uint64_t>(),
                          nslots, In.stage_in.as<uint8_t>(), In.local(), SG);
            k_io_count<<<1, 1, 0, SG>>>(In.soff.as<uint64_t>(), In.padded.as<uint64_t>(), nslots,
                                         sim->io_bytes.as<uint64_t>());
            QZ_CHECK_LAUNCH();
            ctx->launches += 5;
            QZ_CUDA(cudaEventRecord(pev(3 * w), SG));
            // decode / passes / encode of window w on S
            if (w == 0) QZ_CUDA(cudaStreamWaitEvent(S, ready, 0));
            QZ_CUDA(cudaStreamWaitEvent(S, pev(3 * w), 0));
            QZ_CUDA(cudaEventRecord(ev(4 * w), S));
            decode_into(ctx, In.idx.as<DecIdx>(), W.amps.as<double2>(), sim->geom, nslots, nullptr,
                        In.stage_in.as<uint8_t>(), In.local(), ctx->launches, S, sim->sparse_store,
                        W.nzslot.as<uint32_t>());
            QZ_CUDA(cudaEventRecord(ev(4 * w + 1), S));
            run_window_passes(sim, W, dp, dsub, dfull, wbits, S, [&](double2 *dst, const uint32_t *cond) {
                launch_decode(In.stage_in.as<uint8_t>(), In.idx.as<DecIdx>(), nullptr, nslots, sim->geom, dst,
                              ctx->status, S, cond, sim->sparse_store);
            }, ensure_dfull);
            QZ_CUDA(cudaEventRecord(ev(4 * w + 2), S));
            // the output staging / table of window w-1 must be written back
            if (w) QZ_CUDA(cudaStreamWaitEvent(S, pev(3 * (w - 1) + 2), 0));
            QZ_CUDA(cudaMemsetAsync(W.lused.p, 0, 8, S));
            encode_window(ctx, W, sim->geom, nslots, nullptr, nullptr, 0, W.stage_out.as<uint8_t>(),
                          W.lused.as<uint64_t>(), W.stage_out_cap, W.out_local(), sim->len[a].as<uint32_t>(),
                          sim->acct.as<int64_t>(), ctx->launches, S, nullptr, nullptr,
                          In.slot_chunk.as<uint64_t>());
            QZ_CUDA(cudaEventRecord(ev(4 * w + 3), S));
            QZ_CUDA(cudaEventRecord(pev(3 * w + 1), S));
            // write-back (D2H) of window w on SO
            QZ_CUDA(cudaStreamWaitEvent(SO, pev(3 * w + 1), 0));
            launch_copy_out(W.stage_out.as<uint8_t>(), W.lused.as<uint64_t>(), sim->used_ptr(b), sim->cap(b),
                            W.hbase.as<uint64_t>(), sim->arena_ptr(b), W.out_local(), In.slot_chunk.as<uint64_t>(),
                            nslots, sim->table(b), ctx->status, SO);
            k_io_count_out<<<1, 1, 0, SO>>>(W.lused.as<uint64_t>(), sim->io_bytes.as<uint64_t>());
            QZ_CHECK_LAUNCH();
            ctx->launches += 4;
            QZ_CUDA(cudaEventRecord(pev(3 * w + 2), SO));
        }
        for (uint64_t w = 0; w < nwin && !sim->pipelined; ++w) {
            const int ws = sim->two_windows ? int(w & 1) : 0;
            Window &W = ws ? sim->win2 : sim->win;
            cudaStream_t S = sim->streams[ws];
            if (w < 2) QZ_CUDA(cudaStreamWaitEvent(S, ready, 0));
            if (!(w == 0 && pre_decode)) {   // (window 0's decode was issued before planning)
            QZ_CUDA(cudaEventRecord(ev(4 * w), S));
            launch_slot_chunks(W.slot_chunk.as<uint64_t>(), nslots, w * bpw, hs, fmask, smask, S);
            if (sim->host_res) {
                // host arena -> HBM staging (zero-copy 16 B reads), then decode
                // from the staging copy with the slot-indexed local table
                launch_stage_sizes(sim->table(a), W.slot_chunk.as<uint64_t>(), nslots,
                                   W.padded.as<uint64_t>(), S);
                size_t tb = W.cub.cap;
                QZ_CUDA(cub::DeviceScan::ExclusiveSum(W.cub.p, tb, W.padded.as<uint64_t>(),
                                                      W.soff.as<uint64_t>(), (int)nslots, S));
                launch_gather(sim->arena_ptr(a), sim->table(a), W.slot_chunk.as<uint64_t>(),
                              W.soff.as<uint64_t>(), nslots, W.stage_in.as<uint8_t>(), W.local(), S);
                k_io_count<<<1, 1, 0, S>>>(W.soff.as<uint64_t>(), W.padded.as<uint64_t>(), nslots,
                                            sim->io_bytes.as<uint64_t>());
                QZ_CHECK_LAUNCH();
                ctx->launches += 5;
                decode_window(ctx, W, sim->geom, nslots, nullptr, W.stage_in.as<uint8_t>(), W.local(),
                              ctx->launches, S, sim->sparse_store);
            } else {
                decode_window(ctx, W, dgeom, nslots, W.slot_chunk.as<uint64_t>(),
                              sim->arena_ptr(a), sim->table(a), ctx->launches, S, sim->sparse_store);
            }
            QZ_CUDA(cudaEventRecord(ev(4 * w + 1), S));
            }
            run_window_passes(sim, W, dp, dsub, dfull, wbits, S, [&](double2 *dst, const uint32_t *cond) {
                if (sim->host_res)
                    launch_decode(W.stage_in.as<uint8_t>(), W.idx.as<DecIdx>(), nullptr, nslots, sim->geom, dst,
                                  ctx->status, S, cond, sim->sparse_store);
                else
                    launch_decode(sim->arena_ptr(a), W.idx.as<DecIdx>(), W.slot_chunk.as<uint64_t>(), nslots,
                                  sim->geom, dst, ctx->status, S, cond, sim->sparse_store);
            }, ensure_dfull, nwin == 1 && !sim->two_windows);
            QZ_CUDA(cudaEventRecord(ev(4 * w + 2), S));
            if (sim->host_res) {
                QZ_CUDA(cudaMemsetAsync(W.lused.p, 0, 8, S));
                encode_window(ctx, W, sim->geom, nslots, nullptr, nullptr, 0, W.stage_out.as<uint8_t>(),
                              W.lused.as<uint64_t>(), W.stage_out_cap, W.local(),
                              sim->len[a].as<uint32_t>(), sim->acct.as<int64_t>(), ctx->launches, S,
                              w ? sim->acct_ev[(w - 1) & 1] : nullptr, sim->acct_ev[w & 1],
                              W.slot_chunk.as<uint64_t>());
                // HBM -> host arena (zero-copy 16 B writes) + chunk table
                launch_copy_out(W.stage_out.as<uint8_t>(), W.lused.as<uint64_t>(), sim->used_ptr(b),
                                sim->cap(b), W.hbase.as<uint64_t>(), sim->arena_ptr(b), W.local(),
                                W.slot_chunk.as<uint64_t>(), nslots, sim->table(b), ctx->status, S);
                k_io_count_out<<<1, 1, 0, S>>>(W.lused.as<uint64_t>(), sim->io_bytes.as<uint64_t>());
                QZ_CHECK_LAUNCH();
                ctx->launches += 4;
            } else {
                if (end_fresh.mask) {
                    k_fill_dead<<<kNumSMs * 8, 256, 0, S>>>(W.amps.as<double2>(), uint64_t(1) << wbits,
                                                             end_fresh.mask, end_fresh.val);
                    QZ_CHECK_LAUNCH();
                    ++ctx->launches;
                }
                encode_window(ctx, W, sim->geom, nslots, W.slot_chunk.as<uint64_t>(), nullptr, 0,
                              sim->arena_ptr(b), sim->used_ptr(b), sim->cap(b),
                              sim->table(b), sim->len[a].as<uint32_t>(), sim->acct.as<int64_t>(),
                              ctx->launches, S, w ? sim->acct_ev[(w - 1) & 1] : nullptr,
                              sim->acct_ev[w & 1]);
            }
            QZ_CUDA(cudaEventRecord(ev(4 * w + 3), S));
        }
        const double tp2 = now_s();
        for (int i = 0; i < 3; ++i) QZ_CUDA(cudaStreamSynchronize(sim->streams[i]));
        if (trace)
            fprintf(stderr, "qz trace: stage %zu plan %.2f ms launch %.2f ms sync %.2f ms (%zu passes)\n", si,
                    1e3 * (tp1 - tp0), 1e3 * (tp2 - tp1), 1e3 * (now_s() - tp2), gp.passes.size());
        try {
            ctx->check_status();
        } catch (const Failure &f) {
            if (f.code == QZC_ENOMEM && sim->host_res && attempt < 4 && grow_host_arena(sim, b, ctx->last_needed)) {
                QZ_CUDA(cudaMemcpy(sim->acct.p, acct_before, 16, cudaMemcpyHostToDevice));
                continue;
            }
            throw Failure(f.code, "stage " + std::to_string(si) + ": " + f.what());
        }
        break;
        }
        for (uint64_t w = 0; w < nwin; ++w) {
            float ms[3];
            for (int k = 0; k < 3; ++k) QZ_CUDA(cudaEventElapsedTime(&ms[k], ev(4 * w + k), ev(4 * w + k + 1)));
            sim->stats.decode_seconds += ms[0] * 1e-3;
            sim->stats.gate_seconds += ms[1] * 1e-3;
            sim->stats.encode_seconds += ms[2] * 1e-3;
        }
        {
            // compressed bytes decoded / encoded by this stage (store payload
            // totals before and after it; footprint minus per-chunk overhead)
            int64_t acct[2];
            QZ_CUDA(cudaMemcpy(acct, sim->acct.p, 16, cudaMemcpyDeviceToHost));
            const uint64_t out_bytes = uint64_t(acct[0]) - kPerChunkOverhead * sim->nchunks;
            sim->stats.payload_in_bytes += sim->payload_now;
            sim->stats.payload_out_bytes += out_bytes;
            sim->payload_now = out_bytes;
        }
        sim->cur = b;
        sim->sparse_store = false;   // after a stage the payload density is unknown
        {
            // qubits the stage's gates leave fresh
            bool keeps_zero = true;
            for (const DevGate &g : dg) keeps_zero &= gate_keeps_pos_zero(g);
            const Fresh f = fresh_after(dg, 0, dg.size(), stage_fresh);
            uint64_t keep = 0;
            for (uint32_t q = 0; q < n; ++q) {
                const int bq = buffer_bit(st, q, c);
                // a stage's gates act only on its buffer bits (X / CX / SWAP
                // may have changed a fresh qubit's value)
                if (bq < 0) {
                    keep |= uint64_t(1) << q;
                } else if ((f.mask >> bq) & 1) {
                    keep |= uint64_t(1) << q;
                    sim->fresh_v = (sim->fresh_v & ~(uint64_t(1) << q)) | (((f.val >> bq) & 1) << q);
                }
            }
            // the lossy codec reconstructs a zero that shares a chunk with
            // nonzero amplitudes only within the error bound (all-zero chunks
            // stay exact): chunk-local qubits are no longer fresh
            if (sim->geom.lossy) keep &= ~((uint64_t(1) << c) - 1);
            sim->fresh_q = keeps_zero ? (sim->fresh_q & keep) : 0;
            sim->fresh_v &= sim->fresh_q;
        }
        sim->stats.stages += 1;
        sim->stats.batches += nbatches;
        sim->stats.windows += nwin;
        sim->stats.gate_passes += gp.passes.size() * nwin;
        sim->stats.chunk_decompress_count += sim->nchunks;
        sim->stats.chunk_recompress_count += sim->nchunks;
    }
    QZ_CUDA(cudaStreamSynchronize(s));
    if (sim->cfg.renormalize) {
        renormalize(sim);   // re-encodes every chunk (see the stage loop)
        if (sim->geom.lossy) sim->fresh_q &= ~((uint64_t(1) << c) - 1);
    }
    sim->stats.wall_seconds += now_s() - t0;
    dump_debug_counters();
    sim->stats.kernel_launches += ctx->launches - launches0;
    QZ_API_END
}

int qzc_sim_stats_get(const qzc_sim *sim, qzc_sim_stats *out) {
    QZ_API_BEGIN
    *out = sim->stats;
    int64_t acct[2];
    QZ_CUDA(cudaMemcpy(acct, sim->acct.p, 16, cudaMemcpyDeviceToHost));
    out->current_bytes = uint64_t(acct[0]);
    out->peak_bytes = uint64_t(acct[1]);
    if (sim->host_res) {
        uint64_t io[2];
        QZ_CUDA(cudaMemcpy(io, sim->io_bytes.p, 16, cudaMemcpyDeviceToHost));
        out->h2d_bytes += io[0];
        out->d2h_bytes += io[1];
    }
    out->dense_bytes = (uint64_t(1) << sim->n) * 16;
    out->replays = 0;
    if (sim->replays.p) QZ_CUDA(cudaMemcpy(&out->replays, sim->replays.p, 8, cudaMemcpyDeviceToHost));
    QZ_API_END
}

int qzc_sim_chunk_count(const qzc_sim *sim, uint64_t *count_out) {
    QZ_API_BEGIN
    *count_out = sim->nchunks;
    QZ_API_END
}

namespace {
// Host copy of the live table and the arena prefix it references.
void pull_store(qzc_sim *sim, std::vector<uint64_t> &off, std::vector<uint32_t> &len,
                std::vector<uint32_t> &crc, std::vector<uint8_t> &arena) {
    cudaStream_t s = sim->ctx->stream;
    const int a = sim->cur;
    off.resize(sim->nchunks);
    len.resize(sim->nchunks);
    crc.resize(sim->nchunks);
    uint64_t used = 0;
    QZ_CUDA(cudaMemcpyAsync(off.data(), sim->off[a].p, 8 * sim->nchunks, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaMemcpyAsync(len.data(), sim->len[a].p, 4 * sim->nchunks, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaMemcpyAsync(crc.data(), sim->crc[a].p, 4 * sim->nchunks, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaMemcpyAsync(&used, sim->used_ptr(a), 8, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaStreamSynchronize(s));
    arena.resize(used);
    if (sim->host_res)
        std::memcpy(arena.data(), sim->harena[a], used);
    else
        QZ_CUDA(cudaMemcpyAsync(arena.data(), sim->arena[a].p, used, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaStreamSynchronize(s));
    sim->stats.d2h_bytes += used + 16 * sim->nchunks;
}
} // namespace

int qzc_sim_digest(qzc_sim *sim, uint64_t *digest_out) {
    QZ_API_BEGIN
    QZ_CUDA(cudaSetDevice(sim->ctx->device));
    std::vector<uint64_t> off;
    std::vector<uint32_t> len, crc;
    std::vector<uint8_t> arena;
    pull_store(sim, off, len, crc, arena);
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint64_t i = 0; i < sim->nchunks; ++i) h = fnv1a64_host(arena.data() + off[i], len[i], h);
    *digest_out = h;
    QZ_API_END
}

int qzc_sim_payload_bytes(qzc_sim *sim, uint64_t *total_out) {
    QZ_API_BEGIN
    std::vector<uint32_t> len(sim->nchunks);
    QZ_CUDA(cudaMemcpy(len.data(), sim->len[sim->cur].p, 4 * sim->nchunks, cudaMemcpyDeviceToHost));
    uint64_t t = 0;
    for (uint32_t l : len) t += l;
    *total_out = t;
    QZ_API_END
}

int qzc_sim_export(qzc_sim *sim, uint8_t *payload_out, uint64_t cap, uint32_t *sizes, uint32_t *crcs) {
    QZ_API_BEGIN
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int a = sim->cur;
    const uint64_t nc = sim->nchunks;
    std::vector<uint32_t> len(nc), crc(nc);
    QZ_CUDA(cudaMemcpyAsync(len.data(), sim->len[a].p, 4 * nc, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaMemcpyAsync(crc.data(), sim->crc[a].p, 4 * nc, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaStreamSynchronize(s));
    std::vector<uint64_t> dst(nc);
    uint64_t total = 0;
    for (uint64_t i = 0; i < nc; ++i) {
        dst[i] = total;
        total += len[i];
    }
    if (sizes) std::memcpy(sizes, len.data(), 4 * nc);
    if (crcs) std::memcpy(crcs, crc.data(), 4 * nc);
    if (payload_out && total > cap) throw Failure(QZC_EINVAL, "export buffer too small");
    if (payload_out && sim->host_res) {
        // the store already lives in host memory
        std::vector<uint64_t> off(nc);
        QZ_CUDA(cudaMemcpy(off.data(), sim->off[a].p, 8 * nc, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < nc; ++i) std::memcpy(payload_out + dst[i], sim->harena[a] + off[i], len[i]);
    } else if (payload_out) {
        // pack the payloads in chunk order in HBM (the idle window's encode
        // scratch when it is large enough), then one device->host copy
        DevBuf tmp;
        const uint64_t need = ((total + 15) & ~uint64_t(15)) + 8 * nc;
        uint8_t *stage = sim->win.scratch.cap >= need ? sim->win.scratch.as<uint8_t>()
                                                      : (tmp.ensure(need), tmp.as<uint8_t>());
        uint64_t *doff = reinterpret_cast<uint64_t *>(stage + ((total + 15) & ~uint64_t(15)));
        QZ_CUDA(cudaMemcpyAsync(doff, dst.data(), 8 * nc, cudaMemcpyHostToDevice, s));
        k_pack_payloads<<<(unsigned)ceil_div(nc * 32, 256), 256, 0, s>>>(sim->arena_ptr(a), sim->table(a), doff,
                                                                          nc, stage);
        QZ_CHECK_LAUNCH();
        ++ctx->launches;
        QZ_CUDA(cudaMemcpyAsync(payload_out, stage, total, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaStreamSynchronize(s));
        sim->stats.d2h_bytes += total + 8 * nc;
    }
    QZ_API_END
}

int qzc_sim_import(qzc_sim *sim, const uint8_t *payloads, const uint32_t *sizes, const uint32_t *crcs) {
    QZ_API_BEGIN
    sim->fresh_q = 0;
    sim->sparse_store = false;
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    std::vector<uint64_t> off(sim->nchunks);
    uint64_t pos = 0, acct_bytes = 0;
    for (uint64_t i = 0; i < sim->nchunks; ++i) {
        off[i] = pos;
        pos += sizes[i];
        acct_bytes += sizes[i] + kPerChunkOverhead;
    }
    const int a = sim->cur;
    if (pos > sim->cap(a)) throw Failure(QZC_ENOMEM, "store does not fit the arena");
    if (sim->host_res)
        std::memcpy(sim->harena[a], payloads, pos);
    else
        QZ_CUDA(cudaMemcpyAsync(sim->arena[a].p, payloads, pos, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(sim->off[a].p, off.data(), 8 * sim->nchunks, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(sim->len[a].p, sizes, 4 * sim->nchunks, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(sim->crc[a].p, crcs, 4 * sim->nchunks, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(sim->used_ptr(a), &pos, 8, cudaMemcpyHostToDevice, s));
    const int64_t acct[2] = {int64_t(acct_bytes), int64_t(acct_bytes)};
    QZ_CUDA(cudaMemcpyAsync(sim->acct.p, acct, 16, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaStreamSynchronize(s));
    sim->stats.h2d_bytes += pos + 16 * sim->nchunks;
    sim->payload_now = pos;
    sim->initialized = true;
    QZ_API_END
}

int qzc_sim_read_chunks(qzc_sim *sim, uint64_t first, uint64_t count, double *amps_out) {
    QZ_API_BEGIN
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    if (first + count > sim->nchunks)
        throw Failure(QZC_ESTORE, "chunk index out of range: " + std::to_string(first + count - 1));
    cudaStream_t s = ctx->stream;
    const uint64_t per = std::max<uint64_t>(1, sim->win.slots);
    for (uint64_t f = first; f < first + count; f += per) {
        const uint64_t k = std::min(per, first + count - f);
        launch_slot_chunks(sim->win.slot_chunk.as<uint64_t>(), k, f, 0, (uint64_t(1) << (sim->n - sim->c)) - 1, 0, s);
        decode_window(ctx, sim->win, sim->geom, k, sim->win.slot_chunk.as<uint64_t>(),
                      sim->arena_ptr(sim->cur), sim->table(sim->cur), ctx->launches);
        ctx->check_status();
        QZ_CUDA(cudaMemcpyAsync(amps_out + 2 * (f - first) * sim->N, sim->win.amps.p, 16 * k * sim->N,
                                cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaStreamSynchronize(s));
    }
    QZ_API_END
}

int qzc_sim_write_chunk(qzc_sim *sim, uint64_t index, const double *amps) {
    QZ_API_BEGIN
    sim->fresh_q = 0;
    sim->sparse_store = false;
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    if (index >= sim->nchunks) throw Failure(QZC_ESTORE, "chunk index out of range: " + std::to_string(index));
    cudaStream_t s = ctx->stream;
    const int a = sim->cur;
    QZ_CUDA(cudaMemcpyAsync(sim->win.amps.p, amps, 16 * sim->N, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(sim->win.slot_chunk.p, &index, 8, cudaMemcpyHostToDevice, s));
    // the table of the live arena is updated in place; old bytes become garbage
    encode_window(ctx, sim->win, sim->geom, 1, sim->win.slot_chunk.as<uint64_t>(), nullptr, 0,
                  sim->arena_ptr(a), sim->used_ptr(a), sim->cap(a), sim->table(a),
                  sim->len[a].as<uint32_t>(), sim->acct.as<int64_t>(), ctx->launches);
    ctx->check_status();
    int64_t acct[2];
    QZ_CUDA(cudaMemcpy(acct, sim->acct.p, 16, cudaMemcpyDeviceToHost));
    sim->payload_now = uint64_t(acct[0]) - kPerChunkOverhead * sim->nchunks;
    QZ_API_END
}

int qzc_sim_norm(qzc_sim *sim, double *norm_out) {
    QZ_API_BEGIN
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const uint64_t per = std::max<uint64_t>(1, sim->win.slots);
    DevBuf part;
    part.ensure(32 * per);
    std::vector<double> hp(4 * per);
    Kahan k;
    for (uint64_t f = 0; f < sim->nchunks; f += per) {
        const uint64_t cnt = std::min(per, sim->nchunks - f);
        launch_slot_chunks(sim->win.slot_chunk.as<uint64_t>(), cnt, f, 0, (uint64_t(1) << (sim->n - sim->c)) - 1, 0, s);
        decode_window(ctx, sim->win, sim->geom, cnt, sim->win.slot_chunk.as<uint64_t>(),
                      sim->arena_ptr(sim->cur), sim->table(sim->cur), ctx->launches);
        k_partials<<<(unsigned)ceil_div(cnt, 8), dim3(32, 8), 0, s>>>(sim->win.amps.as<double2>(), cnt, sim->N,
                                                                   nullptr, 0, part.as<double>());
        QZ_CHECK_LAUNCH();
        ctx->check_status();
        QZ_CUDA(cudaMemcpyAsync(hp.data(), part.p, 32 * cnt, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaStreamSynchronize(s));
        for (uint64_t i = 0; i < cnt; ++i) k.add(hp[4 * i + 3]);
    }
    part.release();
    *norm_out = k.s;
    QZ_API_END
}

int qzc_sim_fidelity_dev(qzc_sim *sim, const double *dense_dev, double *fidelity_out) {
    QZ_API_BEGIN
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const uint64_t per = std::max<uint64_t>(1, sim->win.slots);
    DevBuf part;
    part.ensure(32 * per);
    std::vector<double> hp(4 * per);
    Kahan re, im, na, nb;
    for (uint64_t f = 0; f < sim->nchunks; f += per) {
        const uint64_t cnt = std::min(per, sim->nchunks - f);
        launch_slot_chunks(sim->win.slot_chunk.as<uint64_t>(), cnt, f, 0, (uint64_t(1) << (sim->n - sim->c)) - 1, 0, s);
        decode_window(ctx, sim->win, sim->geom, cnt, sim->win.slot_chunk.as<uint64_t>(),
                      sim->arena_ptr(sim->cur), sim->table(sim->cur), ctx->launches);
        k_partials<<<(unsigned)ceil_div(cnt, 8), dim3(32, 8), 0, s>>>(
            sim->win.amps.as<double2>(), cnt, sim->N, reinterpret_cast<const double2 *>(dense_dev), f,
            part.as<double>());
        QZ_CHECK_LAUNCH();
        ctx->check_status();
        QZ_CUDA(cudaMemcpyAsync(hp.data(), part.p, 32 * cnt, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaStreamSynchronize(s));
        for (uint64_t i = 0; i < cnt; ++i) {
            re.add(hp[4 * i]);
            im.add(hp[4 * i + 1]);
            na.add(hp[4 * i + 2]);
            nb.add(hp[4 * i + 3]);
        }
    }
    part.release();
    *fidelity_out = (na.s == 0.0 || nb.s == 0.0) ? 0.0 : (re.s * re.s + im.s * im.s) / (na.s * nb.s);
    QZ_API_END
}

int qzc_dense_run(qzc_context *ctx, uint32_t num_qubits, const qzc_gate *gates, uint64_t ngates,
                  double **dense_dev_out) {
    QZ_API_BEGIN
    std::lock_guard<std::mutex> lk(ctx->mu);
    QZ_CUDA(cudaSetDevice(ctx->device));
    const uint64_t count = uint64_t(1) << num_qubits;
    double2 *buf = nullptr;
    QZ_CUDA(cudaMalloc(&buf, 16 * count));
    k_basis<<<(unsigned)ceil_div(count, 256), 256, 0, ctx->stream>>>(buf, count);
    QZ_CHECK_LAUNCH();
    try {
        apply_gates_device(ctx, reinterpret_cast<double *>(buf), num_qubits, gates, ngates);
    } catch (...) {
        cudaFree(buf);
        throw;
    }
    *dense_dev_out = reinterpret_cast<double *>(buf);
    QZ_API_END
}

void qzc_dense_free(qzc_context *ctx, double *dense_dev) {
    if (ctx) cudaSetDevice(ctx->device);
    cudaFree(dense_dev);
}

} // extern "C"
