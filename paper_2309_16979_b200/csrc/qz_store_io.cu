// qz_store_io.cu — the compressed store leaving / entering the device as
// whole payloads (bytes never change, so digests and parity are unaffected):
//
//  * QZST checkpoints (ChunkStore::save / load, store.cpp:152-217): the
//    reference's file format, written from and read back into the device
//    arenas through a page-locked staging buffer, CRCs verified on the device.
//  * Sharded ownership changes (SURVEY §5, §8e — the reference is one
//    process): per-destination record groups packed in HBM from
//    the arena, moved GPU to GPU by the caller's collective (NCCL
//    all_to_all over NVLink), and unpacked in place — the receive buffer
//    becomes the new arena, no host round trip of payload bytes.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "qz_runtime.cuh"

namespace {

// Pack: chunk payloads to their places (warp per chunk, 16 B moves where both
// ends are 16 B aligned, bytes otherwise).
__global__ void k_gather_payloads(const uint8_t *__restrict__ arena, const uint64_t *__restrict__ src_off,
                                  const uint64_t *__restrict__ dst_off, const uint32_t *__restrict__ len,
                                  uint64_t n, uint8_t *__restrict__ out) {
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (w >= n) return;
    const uint8_t *src = arena + src_off[w];
    uint8_t *dst = out + dst_off[w];
    const uint32_t b = len[w];
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        const uint32_t nv = b >> 4;
        for (uint32_t i = lane; i < nv; i += 32)
            reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
        for (uint32_t i = 16 * nv + lane; i < b; i += 32) dst[i] = src[i];
    } else {
        for (uint32_t i = lane; i < b; i += 32) dst[i] = src[i];
    }
}

// One record of a sharded exchange group (see qzc_sim_exchange_plan).
struct XRec {
    uint64_t newidx;   // chunk index in the destination's local store
    uint64_t rel_off;  // payload offset from the group's payload section
    uint32_t len, crc;
};
static_assert(sizeof(XRec) == 24, "record layout");
constexpr uint64_t kGroupHdr = 16;   // u64 record count + u64 pad

__host__ __device__ inline uint64_t round16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

// Unpack one source's group: every record becomes a table entry pointing
// into the receive buffer (which is the new arena).  seen[] catches a chunk
// delivered twice; count[0] totals the records, count[1] the payload bytes.
__global__ void k_unpack_group(const uint8_t *__restrict__ buf, uint64_t group_off, uint64_t group_bytes,
                               uint64_t nlocal, ChunkTable t, uint32_t *__restrict__ seen,
                               unsigned long long *__restrict__ count, DevStatus *status) {
    if (group_bytes < kGroupHdr) return;
    const uint8_t *g = buf + group_off;
    const uint64_t nrec = *reinterpret_cast<const uint64_t *>(g);
    const uint64_t payload0 = group_off + kGroupHdr + round16(sizeof(XRec) * nrec);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nrec;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const XRec r = reinterpret_cast<const XRec *>(g + kGroupHdr)[i];
        if (r.newidx >= nlocal || payload0 + r.rel_off + r.len > group_off + group_bytes) {
            dev_fail(status, QZS_HEADER, r.newidx);
            continue;
        }
        if (atomicExch(&seen[r.newidx], 1u) != 0u) dev_fail(status, QZS_HEADER, r.newidx);
        t.off[r.newidx] = payload0 + r.rel_off;
        t.len[r.newidx] = r.len;
        t.crc[r.newidx] = r.crc;
        atomicAdd(&count[0], 1ull);
        atomicAdd(&count[1], (unsigned long long)r.len);
    }
}

// Bits of the local chunk index y interleaved with the rank bits at the
// owner positions (ascending free positions take y's bits in order).
uint64_t expand_bits(uint64_t y, const std::vector<uint32_t> &pos, uint32_t rank, uint32_t width) {
    uint64_t x = 0;
    uint32_t j = 0;
    for (uint32_t b = 0; b < width; ++b) {
        int owner = -1;
        for (size_t i = 0; i < pos.size(); ++i)
            if (pos[i] == b) owner = int(i);
        if (owner >= 0) x |= uint64_t((rank >> owner) & 1u) << b;
        else x |= ((y >> j++) & 1) << b;
    }
    return x;
}

uint64_t squeeze_bits(uint64_t x, const std::vector<uint32_t> &pos, uint32_t width) {
    uint64_t y = 0;
    uint32_t j = 0;
    for (uint32_t b = 0; b < width; ++b) {
        bool owner = false;
        for (uint32_t p : pos) owner |= p == b;
        if (!owner) y |= ((x >> b) & 1) << j++;
    }
    return y;
}

struct Pinned {
    void *p = nullptr;
    explicit Pinned(size_t n) { QZ_CUDA(cudaMallocHost(&p, n)); }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
    uint8_t *bytes() const { return static_cast<uint8_t *>(p); }
};

void pull_table(qzc_sim *sim, int a, std::vector<uint64_t> &off, std::vector<uint32_t> &len,
                std::vector<uint32_t> &crc) {
    cudaStream_t s = sim->ctx->stream;
    off.resize(sim->nchunks);
    len.resize(sim->nchunks);
    crc.resize(sim->nchunks);
    QZ_CUDA(cudaMemcpyAsync(off.data(), sim->off[a].p, 8 * sim->nchunks, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaMemcpyAsync(len.data(), sim->len[a].p, 4 * sim->nchunks, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaMemcpyAsync(crc.data(), sim->crc[a].p, 4 * sim->nchunks, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(cudaStreamSynchronize(s));
}

// Footprint after a wholesale replacement of the store: current = payload +
// 48 B per chunk; the peak keeps the larger value (account_store semantics).
void set_footprint(qzc_sim *sim, uint64_t payload) {
    int64_t acct[2];
    QZ_CUDA(cudaMemcpy(acct, sim->acct.p, 16, cudaMemcpyDeviceToHost));
    acct[0] = int64_t(payload + kPerChunkOverhead * sim->nchunks);
    acct[1] = std::max(acct[1], acct[0]);
    QZ_CUDA(cudaMemcpy(sim->acct.p, acct, 16, cudaMemcpyHostToDevice));
    sim->payload_now = payload;
}

constexpr char kMagic[4] = {'Q', 'Z', 'S', 'T'};
constexpr uint64_t kStageBytes = uint64_t(256) << 20;   // streaming granule

} // namespace

namespace qz {
// The plan of a sim's last exchange_plan call (held by qzc_sim::xplan).
struct XPlan {
    uint32_t world = 0;
    std::vector<uint64_t> group_off, group_bytes;   // send buffer layout
    std::vector<uint64_t> src_off, dst_off;         // per chunk (arena -> send buffer)
    std::vector<uint32_t> len;
    std::vector<uint8_t> headers;                   // all groups' header sections, concatenated
    std::vector<uint64_t> header_off;               // per group: offset into headers
    std::vector<uint64_t> group_chunks;
    uint64_t total = 0;
};
} // namespace qz

namespace {

// Send layout of an ownership change.  Rank `rank` holds local chunks y of a
// local_bits-bit index; the global chunk index x = y with the rank's bits
// inserted at old_pos; its new owner reads x at new_pos, its new local
// index drops those bits.  Group d (for rank d) = u64 count, u64 pad,
// count 24-byte records (new index, payload offset, len, crc) padded to
// 16 B, the payloads in local chunk order; groups padded to 16 B.
XPlan build_xplan(uint32_t local_bits, uint32_t g, uint32_t rank, const uint32_t *old_pos,
                  const uint32_t *new_pos, const std::vector<uint64_t> &off, const std::vector<uint32_t> &len,
                  const std::vector<uint32_t> &crc) {
    if (g > 6) throw Failure(QZC_EINVAL, "at most 2^6 ranks");
    const uint32_t world = 1u << g;
    if (rank >= world) throw Failure(QZC_EINVAL, "rank out of range");
    const uint32_t width = local_bits + g;   // global chunk-index bits
    std::vector<uint32_t> op(old_pos, old_pos + g), np(new_pos, new_pos + g);
    for (const auto *v : {&op, &np}) {
        std::vector<uint32_t> sorted(*v);
        std::sort(sorted.begin(), sorted.end());
        if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
            throw Failure(QZC_EINVAL, "duplicate owner position");
        for (uint32_t p : *v)
            if (p >= width) throw Failure(QZC_EINVAL, "owner position outside the chunk index");
    }
    const uint64_t nchunks = uint64_t(1) << local_bits;
    XPlan xp;
    xp.world = world;
    std::vector<std::vector<uint64_t>> members(world);
    std::vector<uint64_t> newidx(nchunks);
    for (uint64_t y = 0; y < nchunks; ++y) {
        const uint64_t x = expand_bits(y, op, rank, width);
        uint32_t d = 0;
        for (uint32_t i = 0; i < g; ++i) d |= uint32_t((x >> np[i]) & 1) << i;
        newidx[y] = squeeze_bits(x, np, width);
        members[d].push_back(y);
    }
    xp.src_off.resize(nchunks);
    xp.dst_off.resize(nchunks);
    xp.len.resize(nchunks);
    uint64_t pos = 0, k = 0;
    for (uint32_t d = 0; d < world; ++d) {
        const uint64_t cnt = members[d].size();
        xp.group_off.push_back(pos);
        xp.header_off.push_back(xp.headers.size());
        xp.group_chunks.push_back(cnt);
        const uint64_t hdr = kGroupHdr + round16(sizeof(XRec) * cnt);
        const size_t h0 = xp.headers.size();
        xp.headers.resize(h0 + hdr, 0);
        std::memcpy(xp.headers.data() + h0, &cnt, 8);
        uint64_t rel = 0;
        for (uint64_t i = 0; i < cnt; ++i, ++k) {
            const uint64_t y = members[d][i];
            const XRec r{newidx[y], rel, len[y], crc[y]};
            std::memcpy(xp.headers.data() + h0 + kGroupHdr + sizeof(XRec) * i, &r, sizeof r);
            xp.src_off[k] = off[y];
            xp.dst_off[k] = pos + hdr + rel;
            xp.len[k] = len[y];
            rel += len[y];
        }
        const uint64_t bytes = round16(hdr + rel);
        xp.group_bytes.push_back(bytes);
        pos += bytes;
    }
    xp.total = pos;
    return xp;
}

XPlan &xplan(qzc_sim *sim) {
    if (!sim->xplan) sim->xplan = std::make_shared<XPlan>();
    return *sim->xplan;
}
} // namespace

extern "C" {

int qzc_sim_save(qzc_sim *sim, const char *path) {
    QZ_API_BEGIN
    if (!sim || !path) throw Failure(QZC_EINVAL, "null argument");
    if (!sim->initialized) throw Failure(QZC_ESTORE, "store not initialised");
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int a = sim->cur;
    std::vector<uint64_t> off;
    std::vector<uint32_t> len, crc;
    pull_table(sim, a, off, len, crc);
    std::unique_ptr<FILE, int (*)(FILE *)> f(std::fopen(path, "wb"), &std::fclose);
    if (!f) throw Failure(QZC_ESTORE, std::string("cannot open for writing: ") + path);
    const uint32_t n = sim->n, c = sim->c;
    const double eb = sim->eb;
    bool ok = std::fwrite(kMagic, 1, 4, f.get()) == 4 && std::fwrite(&n, 4, 1, f.get()) == 1 &&
              std::fwrite(&c, 4, 1, f.get()) == 1 && std::fwrite(&eb, 8, 1, f.get()) == 1;
    Pinned host(kStageBytes);
    DevBuf stage, doff, dsrc, dlen;
    uint64_t first = 0;
    while (ok && first < sim->nchunks) {
        // a run of chunks whose payloads fill one staging granule
        uint64_t last = first, bytes = 0;
        while (last < sim->nchunks && (last == first || bytes + len[last] <= kStageBytes)) bytes += len[last++];
        const uint64_t k = last - first;
        if (bytes > kStageBytes) throw Failure(QZC_ESTORE, "chunk payload exceeds the staging buffer");
        if (sim->host_res) {
            uint64_t pos = 0;
            for (uint64_t i = first; i < last; ++i) {
                std::memcpy(host.bytes() + pos, sim->harena[a] + off[i], len[i]);
                pos += len[i];
            }
        } else {
            std::vector<uint64_t> dst(k);
            uint64_t pos = 0;
            for (uint64_t i = 0; i < k; ++i) {
                dst[i] = pos;
                pos += len[first + i];
            }
            stage.ensure(std::max<uint64_t>(bytes, 16));
            doff.ensure(8 * k);
            dsrc.ensure(8 * k);
            dlen.ensure(4 * k);
            QZ_CUDA(cudaMemcpyAsync(doff.p, dst.data(), 8 * k, cudaMemcpyHostToDevice, s));
            QZ_CUDA(cudaMemcpyAsync(dsrc.p, off.data() + first, 8 * k, cudaMemcpyHostToDevice, s));
            QZ_CUDA(cudaMemcpyAsync(dlen.p, len.data() + first, 4 * k, cudaMemcpyHostToDevice, s));
            k_gather_payloads<<<(unsigned)ceil_div(32 * k, 256), 256, 0, s>>>(
                sim->arena_ptr(a), dsrc.as<uint64_t>(), doff.as<uint64_t>(), dlen.as<uint32_t>(), k,
                stage.as<uint8_t>());
            QZ_CHECK_LAUNCH();
            ++ctx->launches;
            QZ_CUDA(cudaMemcpyAsync(host.bytes(), stage.p, bytes, cudaMemcpyDeviceToHost, s));
            QZ_CUDA(cudaStreamSynchronize(s));
            sim->stats.d2h_bytes += bytes;
        }
        uint64_t pos = 0;
        for (uint64_t i = first; ok && i < last; ++i) {
            ok = std::fwrite(&len[i], 4, 1, f.get()) == 1 && std::fwrite(&crc[i], 4, 1, f.get()) == 1 &&
                 std::fwrite(host.bytes() + pos, 1, len[i], f.get()) == len[i];
            pos += len[i];
        }
        first = last;
    }
    if (!ok || std::fflush(f.get()) != 0) throw Failure(QZC_ESTORE, std::string("write failed: ") + path);
    QZ_API_END
}

int qzc_sim_load(qzc_sim *sim, const char *path) {
    QZ_API_BEGIN
    sim->fresh_q = 0;
    if (!sim || !path) throw Failure(QZC_EINVAL, "null argument");
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    std::unique_ptr<FILE, int (*)(FILE *)> f(std::fopen(path, "rb"), &std::fclose);
    if (!f) throw Failure(QZC_ESTORE, std::string("cannot open for reading: ") + path);
    char magic[4];
    uint32_t n = 0, c = 0;
    double eb = 0.0;
    if (std::fread(magic, 1, 4, f.get()) != 4 || std::memcmp(magic, kMagic, 4) != 0)
        throw Failure(QZC_ESTORE, std::string("not a chunk store file: ") + path);
    if (std::fread(&n, 4, 1, f.get()) != 1 || std::fread(&c, 4, 1, f.get()) != 1 ||
        std::fread(&eb, 8, 1, f.get()) != 1 || n > 40 || c > n)
        throw Failure(QZC_ESTORE, std::string("corrupt chunk store header: ") + path);
    if (n != sim->n || c != sim->c || !(eb == sim->eb))
        throw Failure(QZC_ESTORE, "chunk store geometry (n=" + std::to_string(n) + ", c=" + std::to_string(c) +
                                      ") does not match the simulator (n=" + std::to_string(sim->n) +
                                      ", c=" + std::to_string(sim->c) + ", same error bound)");
    const int a = sim->cur;
    std::vector<uint64_t> off(sim->nchunks);
    std::vector<uint32_t> len(sim->nchunks), crc(sim->nchunks);
    Pinned host(kStageBytes);
    uint64_t used = 0, fill = 0, flushed = 0;
    auto flush = [&] {
        if (!fill) return;
        if (used + fill > sim->cap(a)) throw Failure(QZC_ENOMEM, "store does not fit the arena");
        if (sim->host_res) std::memcpy(sim->harena[a] + flushed, host.bytes(), fill);
        else QZ_CUDA(cudaMemcpy(sim->arena[a].as<uint8_t>() + flushed, host.bytes(), fill, cudaMemcpyHostToDevice));
        sim->stats.h2d_bytes += fill;
        flushed += fill;
        fill = 0;
    };
    for (uint64_t i = 0; i < sim->nchunks; ++i) {
        if (std::fread(&len[i], 4, 1, f.get()) != 1 || std::fread(&crc[i], 4, 1, f.get()) != 1)
            throw Failure(QZC_ESTORE, std::string("truncated chunk store: ") + path);
        if (len[i] > kStageBytes) throw Failure(QZC_ESTORE, "chunk payload exceeds the staging buffer");
        if (fill + len[i] > kStageBytes) flush();
        if (std::fread(host.bytes() + fill, 1, len[i], f.get()) != len[i])
            throw Failure(QZC_ESTORE, std::string("truncated chunk store: ") + path);
        off[i] = used;
        used += len[i];
        fill += len[i];
    }
    flush();
    QZ_CUDA(cudaMemcpyAsync(sim->off[a].p, off.data(), 8 * sim->nchunks, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(sim->len[a].p, len.data(), 4 * sim->nchunks, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(sim->crc[a].p, crc.data(), 4 * sim->nchunks, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(sim->used_ptr(a), &used, 8, cudaMemcpyHostToDevice, s));
    // every CRC checked on the device (ChunkStore::load, store.cpp:200-201)
    launch_crc(ctx->tabs, sim->arena_ptr(a), sim->table(a), nullptr, sim->nchunks, true, ctx->status, s);
    ++ctx->launches;
    try {
        ctx->check_status();
    } catch (const Failure &e) {
        std::string m = e.what();
        const auto p = m.find_last_of(' ');
        throw Failure(QZC_ESTORE, "checksum mismatch in chunk " + m.substr(p + 1));
    }
    set_footprint(sim, used);
    sim->initialized = true;
    sim->sparse_store = false;
    QZ_API_END
}

int qzc_sim_exchange_plan(qzc_sim *sim, uint32_t g, uint32_t rank, const uint32_t *old_pos,
                          const uint32_t *new_pos, uint64_t *send_bytes, uint64_t *send_chunks) {
    QZ_API_BEGIN
    if (!sim || (g && (!old_pos || !new_pos)) || !send_bytes) throw Failure(QZC_EINVAL, "null argument");
    if (sim->host_res) throw Failure(QZC_EINVAL, "sharded exchange needs the HBM-resident store");
    if (!sim->initialized) throw Failure(QZC_ESTORE, "store not initialised");
    std::vector<uint64_t> off;
    std::vector<uint32_t> len, crc;
    pull_table(sim, sim->cur, off, len, crc);
    XPlan &xp = xplan(sim);
    xp = build_xplan(sim->n - sim->c, g, rank, old_pos, new_pos, off, len, crc);
    for (uint32_t d = 0; d < xp.world; ++d) {
        send_bytes[d] = xp.group_bytes[d];
        if (send_chunks) send_chunks[d] = xp.group_chunks[d];
    }
    QZ_API_END
}

int qzc_exchange_pack_host(uint32_t local_bits, uint32_t g, uint32_t rank, const uint32_t *old_pos,
                           const uint32_t *new_pos, const uint8_t *payloads, const uint32_t *sizes,
                           const uint32_t *crcs, uint8_t *out, uint64_t cap, uint64_t *send_bytes) {
    QZ_API_BEGIN
    if (!sizes || !crcs || !send_bytes || (g && (!old_pos || !new_pos))) throw Failure(QZC_EINVAL, "null argument");
    if (local_bits > 40) throw Failure(QZC_EINVAL, "local chunk index too wide");
    const uint64_t nchunks = uint64_t(1) << local_bits;
    std::vector<uint64_t> off(nchunks);
    std::vector<uint32_t> len(sizes, sizes + nchunks), crc(crcs, crcs + nchunks);
    uint64_t pos = 0;
    for (uint64_t i = 0; i < nchunks; ++i) {
        off[i] = pos;
        pos += len[i];
    }
    const XPlan xp = build_xplan(local_bits, g, rank, old_pos, new_pos, off, len, crc);
    for (uint32_t d = 0; d < xp.world; ++d) send_bytes[d] = xp.group_bytes[d];
    if (out) {
        if (xp.total > cap) throw Failure(QZC_EINVAL, "exchange buffer too small");
        std::memset(out, 0, xp.total);
        for (uint32_t d = 0; d < xp.world; ++d) {
            const uint64_t hb = (d + 1 < xp.world ? xp.header_off[d + 1] : xp.headers.size()) - xp.header_off[d];
            std::memcpy(out + xp.group_off[d], xp.headers.data() + xp.header_off[d], hb);
        }
        for (uint64_t k = 0; k < nchunks; ++k) std::memcpy(out + xp.dst_off[k], payloads + xp.src_off[k], xp.len[k]);
    }
    QZ_API_END
}

int qzc_exchange_unpack_host(uint32_t world, const uint8_t *recv, const uint64_t *recv_bytes,
                             uint32_t local_bits, uint8_t *payload_out, uint64_t cap, uint32_t *sizes,
                             uint32_t *crcs) {
    QZ_API_BEGIN
    if (!recv_bytes || !sizes || !crcs || local_bits > 40) throw Failure(QZC_EINVAL, "bad argument");
    const uint64_t nchunks = uint64_t(1) << local_bits;
    std::vector<const uint8_t *> src(nchunks, nullptr);
    uint64_t pos = 0;
    for (uint32_t s = 0; s < world; ++s) {
        const uint64_t gb = recv_bytes[s];
        if (gb >= kGroupHdr) {
            uint64_t nrec;
            std::memcpy(&nrec, recv + pos, 8);
            const uint64_t payload0 = pos + kGroupHdr + round16(sizeof(XRec) * nrec);
            for (uint64_t i = 0; i < nrec; ++i) {
                XRec r;
                std::memcpy(&r, recv + pos + kGroupHdr + sizeof(XRec) * i, sizeof r);
                if (r.newidx >= nchunks || payload0 + r.rel_off + r.len > pos + gb || src[r.newidx])
                    throw Failure(QZC_ESTORE, "exchange: malformed or duplicate record for chunk " +
                                                  std::to_string(r.newidx));
                src[r.newidx] = recv + payload0 + r.rel_off;
                sizes[r.newidx] = r.len;
                crcs[r.newidx] = r.crc;
            }
        }
        pos += gb;
    }
    uint64_t out = 0;
    for (uint64_t i = 0; i < nchunks; ++i) {
        if (!src[i]) throw Failure(QZC_ESTORE, "exchange: chunk " + std::to_string(i) + " not delivered");
        if (payload_out) {
            if (out + sizes[i] > cap) throw Failure(QZC_EINVAL, "payload buffer too small");
            std::memcpy(payload_out + out, src[i], sizes[i]);
        }
        out += sizes[i];
    }
    QZ_API_END
}

int qzc_sim_exchange_pack(qzc_sim *sim, void **send_dev_out, uint64_t *bytes_out) {
    QZ_API_BEGIN
    if (!sim || !send_dev_out) throw Failure(QZC_EINVAL, "null argument");
    XPlan &xp = xplan(sim);
    if (!xp.world) throw Failure(QZC_EINVAL, "no exchange planned");
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    // the send groups are staged in the idle window's encode scratch when it
    // is large enough, else in a buffer of the plan's size
    static thread_local DevBuf spill;
    uint8_t *buf;
    const uint64_t meta = 20 * sim->nchunks + 64;
    if (sim->win.scratch.cap >= xp.total + meta) {
        buf = sim->win.scratch.as<uint8_t>();
    } else {
        spill.ensure(xp.total + meta);
        buf = spill.as<uint8_t>();
    }
    uint8_t *mbase = buf + round16(xp.total);
    uint64_t *dsrc = reinterpret_cast<uint64_t *>(mbase);
    uint64_t *ddst = dsrc + sim->nchunks;
    uint32_t *dlen = reinterpret_cast<uint32_t *>(ddst + sim->nchunks);
    QZ_CUDA(cudaMemcpyAsync(dsrc, xp.src_off.data(), 8 * sim->nchunks, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(ddst, xp.dst_off.data(), 8 * sim->nchunks, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaMemcpyAsync(dlen, xp.len.data(), 4 * sim->nchunks, cudaMemcpyHostToDevice, s));
    for (uint32_t d = 0; d < xp.world; ++d) {
        const uint64_t hb = (d + 1 < xp.world ? xp.header_off[d + 1] : xp.headers.size()) - xp.header_off[d];
        QZ_CUDA(cudaMemcpyAsync(buf + xp.group_off[d], xp.headers.data() + xp.header_off[d], hb,
                                cudaMemcpyHostToDevice, s));
    }
    if (sim->nchunks) {
        k_gather_payloads<<<(unsigned)ceil_div(32 * sim->nchunks, 256), 256, 0, s>>>(
            sim->arena_ptr(sim->cur), dsrc, ddst, dlen, sim->nchunks, buf);
        QZ_CHECK_LAUNCH();
        ++ctx->launches;
    }
    QZ_CUDA(cudaStreamSynchronize(s));
    *send_dev_out = buf;
    if (bytes_out) *bytes_out = xp.total;
    QZ_API_END
}

int qzc_sim_exchange_recv_buffer(qzc_sim *sim, uint64_t bytes, void **recv_dev_out) {
    QZ_API_BEGIN
    if (!sim || !recv_dev_out) throw Failure(QZC_EINVAL, "null argument");
    if (bytes > sim->cap(1 - sim->cur)) throw Failure(QZC_ENOMEM, "exchange does not fit the arena");
    QZ_CUDA(cudaSetDevice(sim->ctx->device));
    *recv_dev_out = sim->arena_ptr(1 - sim->cur);
    QZ_API_END
}

int qzc_sim_exchange_unpack(qzc_sim *sim, const uint64_t *recv_bytes) {
    QZ_API_BEGIN
    sim->fresh_q = 0;
    if (!sim || !recv_bytes) throw Failure(QZC_EINVAL, "null argument");
    XPlan &xp = xplan(sim);
    if (!xp.world) throw Failure(QZC_EINVAL, "no exchange planned");
    qzc_context *ctx = sim->ctx;
    QZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int b = 1 - sim->cur;
    // seen flags + counters live in the idle window's slot map scratch
    DevBuf tmp;
    tmp.ensure(4 * sim->nchunks + 32);
    uint32_t *seen = tmp.as<uint32_t>();
    auto *count = reinterpret_cast<unsigned long long *>(tmp.as<uint8_t>() + ((4 * sim->nchunks + 15) & ~uint64_t(15)));
    QZ_CUDA(cudaMemsetAsync(tmp.p, 0, tmp.cap, s));
    uint64_t pos = 0;
    for (uint32_t src = 0; src < xp.world; ++src) {
        if (recv_bytes[src]) {
            const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(sim->nchunks, 256), kNumSMs * 4);
            k_unpack_group<<<std::max(grid, 1u), 256, 0, s>>>(sim->arena_ptr(b), pos, recv_bytes[src], sim->nchunks,
                                                             sim->table(b), seen, count, ctx->status);
            QZ_CHECK_LAUNCH();
            ++ctx->launches;
        }
        pos += recv_bytes[src];
    }
    unsigned long long cnt[2] = {0, 0};
    QZ_CUDA(cudaMemcpyAsync(cnt, count, 16, cudaMemcpyDeviceToHost, s));
    try {
        ctx->check_status();
    } catch (const Failure &e) {
        throw Failure(QZC_ESTORE, std::string("exchange: malformed or duplicate record, ") + e.what());
    }
    if (cnt[0] != sim->nchunks)
        throw Failure(QZC_ESTORE, "exchange delivered " + std::to_string(cnt[0]) + " of " +
                                      std::to_string(sim->nchunks) + " chunks");
    QZ_CUDA(cudaMemcpyAsync(sim->used_ptr(b), &pos, 8, cudaMemcpyHostToDevice, s));
    QZ_CUDA(cudaStreamSynchronize(s));
    sim->cur = b;
    set_footprint(sim, cnt[1]);
    sim->sparse_store = false;
    xp.world = 0;
    QZ_API_END
}

} // extern "C"
