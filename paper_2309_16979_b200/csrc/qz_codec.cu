// qz_codec.cu — bit-exact chunk codec kernels for sm_100a.
//
// Reference: codec.cpp:28-266 (LossyPQ quantiser chain, zigzag, byte-plane
// RLE, LosslessRLE, CRC-32), util.cpp:20-31.
//
// The quantiser / reconstruction chain is strictly sequential per
// (chunk, plane): pred_{i+1} depends on the rounded reconstruction of element
// i (codec.cpp:130-159, 226-246), and fp64 addition is not associative, so
// parallelism comes from chunks: one thread per (chunk, plane) "half".  Each
// CTA stages a [32 chunks x 32 elements] amplitude tile through shared memory
// so every HBM access is a coalesced 512 B row, while the threads walk their
// chains.  The same sequential walk emits the RLE pairs of its half into a
// scratch sub-stream; the real half keeps its last run open and the
// imaginary half holds back its first run, and the assembler merges the two
// at the plane boundary exactly as rle_encode would over the joined plane.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "qz_codec.cuh"
#include "qz_kprof.cuh"

namespace qz {

namespace {

constexpr uint32_t kHdr = 17;
constexpr uint32_t kPoly = 0xEDB88320u;
constexpr int kSlotsPerCta = 32;  // chunks per CTA in the encode/decode kernels
constexpr int kTileElems = 32;    // elements per staged tile row

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }
__host__ __device__ inline uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// ----------------------------------------------------------------- bytes --
__device__ __forceinline__ uint32_t ld_u8(const uint8_t *p) { return p[0]; }
__device__ __forceinline__ uint32_t ld_u32(const uint8_t *p) {
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}
__device__ __forceinline__ uint64_t ld_u64(const uint8_t *p) {
    return uint64_t(ld_u32(p)) | (uint64_t(ld_u32(p + 4)) << 32);
}
__device__ __forceinline__ void st_u32(uint8_t *p, uint32_t v) {
    p[0] = v & 0xff; p[1] = (v >> 8) & 0xff; p[2] = (v >> 16) & 0xff; p[3] = v >> 24;
}
__device__ __forceinline__ void st_u64(uint8_t *p, uint64_t v) {
    st_u32(p, uint32_t(v));
    st_u32(p + 4, uint32_t(v >> 32));
}

__device__ __forceinline__ uint32_t zigzag16(int32_t code) {
    return uint32_t((code << 1) ^ (code >> 15)) & 0xffffu;
}
__device__ __forceinline__ int32_t unzigzag16(uint32_t z) {
    return int32_t(z >> 1) ^ -int32_t(z & 1);
}

// ------------------------------------------------------------- CRC-32 ---
__host__ __device__ inline uint32_t multmodp(uint32_t a, uint32_t b) {
    if (a == 0) return 0;
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}

// x^(8n) mod P: the operator that appends n zero bytes (crc32_combine).
__host__ __device__ inline uint32_t x8nmodp(uint64_t n) {
    uint32_t p = 1u << 31;     // x^0
    uint32_t sq = 1u << 30;    // x^1
    // x^(8n) = x^(n * 2^3): square x three times first
    for (int i = 0; i < 3; ++i) sq = multmodp(sq, sq);
    while (n) {
        if (n & 1) p = multmodp(sq, p);
        n >>= 1;
        if (n) sq = multmodp(sq, sq);
    }
    return p;
}

__device__ uint32_t crc_range(const uint32_t *T, const uint8_t *p, uint64_t n) {
    uint32_t c = 0xFFFFFFFFu;
    // bytes up to an 8-byte boundary, then aligned 8-byte words (slicing-by-8)
    while (n && (reinterpret_cast<uintptr_t>(p) & 7)) {
        c = T[(c ^ *p++) & 0xff] ^ (c >> 8);
        --n;
    }
    const uint2 *w = reinterpret_cast<const uint2 *>(p);
    for (; n >= 8; n -= 8, ++w) {
        const uint2 x = __ldg(w);
        const uint32_t lo = c ^ x.x, hi = x.y;
        c = T[7 * 256 + (lo & 0xff)] ^ T[6 * 256 + ((lo >> 8) & 0xff)] ^
            T[5 * 256 + ((lo >> 16) & 0xff)] ^ T[4 * 256 + (lo >> 24)] ^
            T[3 * 256 + (hi & 0xff)] ^ T[2 * 256 + ((hi >> 8) & 0xff)] ^
            T[1 * 256 + ((hi >> 16) & 0xff)] ^ T[0 * 256 + (hi >> 24)];
    }
    p = reinterpret_cast<const uint8_t *>(w);
    while (n--) c = T[(c ^ *p++) & 0xff] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

// Warp per slot: 32 equal segments, per-lane slicing-by-8, then lane 0
// folds them left to right with crc32_combine.
__global__ void __launch_bounds__(256) k_crc(const uint32_t *__restrict__ tabs,
                                             const uint8_t *__restrict__ arena, ChunkTable table,
                                             const uint64_t *__restrict__ slot_chunk,
                                             uint64_t nslots, int verify, DevStatus *status) {
    __shared__ uint32_t T[8 * 256];
    __shared__ uint32_t X2[32];   // x^(8 * 2^k) mod P
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) T[i] = tabs[i];
    if (threadIdx.x == 0) {
        uint32_t x = x8nmodp(1);
        for (int k = 0; k < 32; ++k) {
            X2[k] = x;
            x = multmodp(x, x);
        }
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t s = warp; s < nslots; s += nwarps) {
        const uint64_t chunk = slot_chunk ? slot_chunk[s] : s;
        const uint64_t len = table.len[chunk];
        const uint8_t *p = arena + table.off[chunk];
        const uint64_t seg = round_up((len + 31) / 32, 8);
        const uint64_t b = umin64(len, lane * seg), e = umin64(len, b + seg);
        const uint32_t c = crc_range(T, p + b, e - b);
        // crc(A||B) = crc(A) * x^(8|B|) ^ crc(B) folds to
        // XOR_i crc_i * x^(8 S_i), S_i = bytes after lane i's segment: every
        // lane shifts its own CRC (powers from X2), then one XOR reduction
        const uint32_t after = uint32_t(len - e);
        uint32_t acc = 0;
        if (e > b) {
            uint32_t f = 0x80000000u;   // x^0
            for (uint32_t r = after; r; r &= r - 1) f = multmodp(X2[__ffs(r) - 1], f);
            acc = multmodp(f, c);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            if (verify) {
                if (acc != table.crc[chunk]) dev_fail(status, QZS_CRC, chunk);
            } else {
                table.crc[chunk] = acc;
            }
        }
    }
}

// ----------------------------------------------------------- decode index --

struct Cursor {
    uint32_t pos, rem, byte;
};

// Warp per chunk.  Each plane's RLE stream is walked 256 pairs per step
// (8 per lane, warp scan of the run sums): validation, the pair / skip where
// the plane's element count crosses N (start of the imaginary half) and the
// per-step element counts (smem) from which every lane then locates its
// 1/32 of the real half and merges the two byte planes there to count the
// sentinel (raw) codes of the real half.  Same results as a sequential walk.
constexpr uint32_t kIdxWarps = 4;
constexpr uint32_t kIdxMaxSteps = 1040;   // >= 4N / 256 + 1 for c <= 17 (lossy: <= 2N pairs per plane)

__global__ void __launch_bounds__(32 * kIdxWarps) k_dec_index_warp(
    const uint8_t *__restrict__ arena, ChunkTable table, const uint64_t *__restrict__ slot_chunk,
    uint64_t nslots, CodecGeom g, DecIdx *__restrict__ out, DevStatus *status, uint32_t *nzslot) {
    __shared__ uint32_t step_prod[kIdxWarps][2][kIdxMaxSteps];   // elements before step j
    const uint32_t lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const uint64_t s = uint64_t(blockIdx.x) * kIdxWarps + wq;
    if (s >= nslots) return;
    const uint64_t chunk = slot_chunk ? slot_chunk[s] : s;
    DecIdx d;
    d.base = table.off[chunk];
    d.len = 0;
    const uint32_t len = table.len[chunk];
    const uint8_t *p = arena + d.base;
    const uint64_t N = g.N, total = 2 * N;
    int err = 0;
    uint32_t count = 0;
    if (len < kHdr) err = QZS_HEADER;
    if (!err) {
        const uint32_t id = ld_u8(p);
        d.eb = __longlong_as_double((long long)ld_u64(p + 1));
        count = ld_u32(p + 9);
        d.raw_count = ld_u32(p + 13);
        if ((id != 1 && id != 2) || id != (g.lossy ? 1u : 2u) || count != N) err = QZS_HEADER;
    }
    uint32_t pos = kHdr;
    uint32_t nsteps[2] = {0, 0}, start[2] = {0, 0};
    bool ff_real[2] = {false, false};   // a 0xFF run touches the real half
    bool nonzero_byte = false;          // some run of plane 0/1 has a byte != 0
    for (uint32_t k = 0; k < g.planes && !err; ++k) {
        uint64_t produced = 0;
        d.pos[k][0] = pos;
        d.skip[k][0] = 0;
        start[k < 2 ? k : 1] = pos;
        bool done = false, found = false;
        uint32_t step = 0;
        while (!done && !err) {
            if (k < 2 && step < kIdxMaxSteps && lane == 0) step_prod[wq][k][step] = uint32_t(produced);
            // this lane's 8 pairs
            const uint32_t p0 = pos + 16 * lane;
            uint32_t runs[8];
            uint32_t mysum = 0, avail = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t q = p0 + 2 * j;
                runs[j] = q + 2 <= len ? uint32_t(__ldg(p + q + 1)) : 0u;
                avail += q + 2 <= len ? 1u : 0u;
                mysum += runs[j];
            }
            // inclusive scan of the lane sums
            uint64_t incl = mysum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= uint32_t(o)) incl += t;
            }
            const uint64_t excl = produced + incl - mysum;
            // the pair that completes the plane, the pair holding element N,
            // the first zero run before the end, the first missing pair
            uint32_t end_pair = ~0u, half_pair = ~0u, half_skip = 0, bad_pair = ~0u;
            uint64_t c = excl;
            bool ff = false, nz = false;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t idx = 8 * lane + j;
                if (j >= int(avail)) { if (bad_pair == ~0u && c < total) bad_pair = idx; continue; }
                if (c >= total) continue;
                const uint32_t r = runs[j];
                const uint32_t bj = __ldg(p + p0 + 2 * j);
                ff |= c < N && bj == 0xFF;
                nz |= bj != 0;
                if (bad_pair == ~0u && (r == 0 || c + r > total)) bad_pair = idx;
                if (half_pair == ~0u && c <= N && N < c + r) { half_pair = idx; half_skip = uint32_t(N - c); }
                if (end_pair == ~0u && c + r == total) end_pair = idx;
                c += r;
            }
            if (k < 2 && __any_sync(0xffffffffu, ff)) ff_real[k] = true;
            if (__any_sync(0xffffffffu, nz)) nonzero_byte = true;
            // warp-wide minima (first occurrence in stream order)
            uint32_t e_end = end_pair, e_half = half_pair, e_bad = bad_pair;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                e_end = min(e_end, __shfl_xor_sync(0xffffffffu, e_end, o));
                e_half = min(e_half, __shfl_xor_sync(0xffffffffu, e_half, o));
                e_bad = min(e_bad, __shfl_xor_sync(0xffffffffu, e_bad, o));
            }
            if (e_half != ~0u && !found) {
                const uint32_t src = e_half >> 3;
                const uint32_t sk = __shfl_sync(0xffffffffu, half_skip, src);
                if (e_bad == ~0u || e_half < e_bad) {
                    d.pos[k][1] = pos + 2 * e_half;
                    d.skip[k][1] = sk;
                    found = true;
                }
            }
            if (e_bad != ~0u && (e_end == ~0u || e_bad <= e_end)) {
                // a zero / overlong run, or the stream ends before 2N elements
                const uint32_t q = pos + 2 * e_bad;
                err = q + 2 > len ? QZS_RLE_TRUNC : QZS_RLE_RUN;
                break;
            }
            if (e_end != ~0u) {
                pos += 2 * (e_end + 1);
                done = true;
            } else {
                produced += __shfl_sync(0xffffffffu, incl, 31);
                pos += 512;
            }
            ++step;
        }
        if (k < 2) nsteps[k] = step;
    }
    if (!err && g.lossy) {
        d.raw_pos = pos;
        if (uint64_t(pos) + uint64_t(d.raw_count) * 8 > len) err = QZS_RAW_MISSING;
    }
    if (!err && g.lossy && (nsteps[0] > kIdxMaxSteps || nsteps[1] > kIdxMaxSteps)) err = QZS_RLE_RUN;
    __syncwarp();
    if (!err && g.lossy) {
        // sentinel codes in [lane * N/32, (lane+1) * N/32): locate both planes'
        // cursors at the segment start, then merge the two run streams
        const uint64_t seg = N / 32 ? N / 32 : 1;
        const uint64_t e0 = uint64_t(lane) * seg, e1 = lane == 31 ? N : umin64(N, e0 + seg);
        uint64_t cnt = 0;
        // a sentinel needs 0xFF in both planes: without 0xFF runs in the real
        // half of either plane there is none (the common dense case)
        if (e0 < e1 && ff_real[0] && ff_real[1]) {
            uint32_t pp[2], rr[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                // last step whose start count <= e0, then walk its pairs
                uint32_t lo = 0, hi = nsteps[k] - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) >> 1;
                    if (step_prod[wq][k][mid] <= e0) lo = mid;
                    else hi = mid - 1;
                }
                uint32_t q = start[k] + 512 * lo;
                uint64_t c = step_prod[wq][k][lo];
                uint32_t r = p[q + 1];
                while (c + r <= e0) {
                    c += r;
                    q += 2;
                    r = p[q + 1];
                }
                pp[k] = q;
                rr[k] = uint32_t(c + r - e0);   // elements of this run at/after e0
            }
            uint64_t i = e0;
            while (i < e1) {
                const uint64_t st = umin64(umin32(rr[0], rr[1]), e1 - i);
                if (p[pp[0]] == 0xFF && p[pp[1]] == 0xFF) cnt += st;
                i += st;
                rr[0] -= uint32_t(st);
                rr[1] -= uint32_t(st);
                if (i < e1) {
                    if (rr[0] == 0) { pp[0] += 2; rr[0] = p[pp[0] + 1]; }
                    if (rr[1] == 0) { pp[1] += 2; rr[1] = p[pp[1] + 1]; }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (cnt > d.raw_count) err = QZS_RAW_UNDER;
        d.raw_re = uint32_t(cnt);
    }
    if (lane == 0) {
        if (err) dev_fail(status, err, chunk);
        else d.len = len;
        out[s] = d;
        if (nzslot) {
            const bool nzs = err || nonzero_byte || d.raw_count != 0;
            nzslot[s] = nzs ? 1u : 0u;
            if (!nzs) atomicAdd(&nzslot[nslots], 1u);
        }
    }
}

__global__ void k_dec_index(const uint8_t *__restrict__ arena, ChunkTable table,
                            const uint64_t *__restrict__ slot_chunk, uint64_t nslots,
                            CodecGeom g, DecIdx *__restrict__ out, DevStatus *status) {
    const uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    const uint64_t chunk = slot_chunk ? slot_chunk[s] : s;
    DecIdx d;
    d.base = table.off[chunk];
    d.len = 0;  // marks "invalid" until the walk succeeds
    const uint32_t len = table.len[chunk];
    const uint8_t *p = arena + d.base;
    const uint64_t N = g.N, total = 2 * N;
    int err = 0;
    if (len < kHdr) err = QZS_HEADER;
    uint32_t id = 0, count = 0;
    if (!err) {
        id = ld_u8(p);
        d.eb = __longlong_as_double((long long)ld_u64(p + 1));
        count = ld_u32(p + 9);
        d.raw_count = ld_u32(p + 13);
        if ((id != 1 && id != 2) || id != (g.lossy ? 1u : 2u) || count != N) err = QZS_HEADER;
    }
    uint32_t pos = kHdr;
    for (uint32_t k = 0; k < g.planes && !err; ++k) {
        uint64_t produced = 0;
        d.pos[k][0] = pos;
        d.skip[k][0] = 0;
        bool found = false;
        while (produced < total) {
            if (pos + 2 > len) { err = QZS_RLE_TRUNC; break; }
            const uint32_t run = p[pos + 1];
            if (run == 0 || produced + run > total) { err = QZS_RLE_RUN; break; }
            if (!found && produced <= N && N < produced + run) {
                d.pos[k][1] = pos;
                d.skip[k][1] = uint32_t(N - produced);
                found = true;
            }
            produced += run;
            pos += 2;
        }
    }
    if (!err && g.lossy) {
        d.raw_pos = pos;
        if (uint64_t(pos) + uint64_t(d.raw_count) * 8 > len) err = QZS_RAW_MISSING;
    }
    if (!err && g.lossy) {
        // sentinel (0xFFFF) codes in the real half: overlap of 0xFF runs in
        // both byte planes over elements [0, N)
        uint32_t pl = d.pos[0][0], ph = d.pos[1][0];
        uint32_t rl = p[pl + 1], rh = p[ph + 1];
        uint64_t i = 0, cnt = 0;
        while (i < N) {
            uint64_t step = umin64(umin32(rl, rh), N - i);
            if (p[pl] == 0xFF && p[ph] == 0xFF) cnt += step;
            i += step;
            rl -= uint32_t(step);
            rh -= uint32_t(step);
            if (i < N) {
                if (rl == 0) { pl += 2; rl = p[pl + 1]; }
                if (rh == 0) { ph += 2; rh = p[ph + 1]; }
            }
        }
        if (cnt > d.raw_count) err = QZS_RAW_UNDER;
        d.raw_re = uint32_t(cnt);
    }
    if (err) dev_fail(status, err, chunk);
    else d.len = len;
    out[s] = d;
}

// ----------------------------------------------------------------- decode --

// Buffered RLE reader for the lossy decoder: 8 (byte, run) pairs are fetched
// at a time (16 independent byte loads, up to 15 bytes past the stream —
// arenas and staging buffers keep >= 64 bytes of slack), so the dependent
// load latency is paid once per 8 pairs instead of once per pair.
struct BCursor {
    uint32_t bpos;      // byte offset of the buffered pairs
    uint32_t k;         // next pair in the buffer (0..8)
    uint32_t byte, rem; // current run
    uint64_t b0, b1;    // pairs 0-3, 4-7
};

__device__ __forceinline__ void bc_fill(BCursor &c, const uint8_t *p) {
    uint64_t x0 = 0, x1 = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x0 |= uint64_t(__ldg(p + c.bpos + i)) << (8 * i);
        x1 |= uint64_t(__ldg(p + c.bpos + 8 + i)) << (8 * i);
    }
    c.b0 = x0;
    c.b1 = x1;
    c.k = 0;
}

__device__ __forceinline__ void bc_take(BCursor &c, const uint8_t *p) {
    if (c.k == 8) {
        c.bpos += 16;
        bc_fill(c, p);
    }
    const uint64_t w = c.k < 4 ? c.b0 : c.b1;
    const uint32_t sh = 16 * (c.k & 3);
    c.byte = uint32_t(w >> sh) & 0xffu;
    c.rem = uint32_t(w >> (sh + 8)) & 0xffu;
    ++c.k;
}

__device__ __forceinline__ void bc_init(BCursor &c, const uint8_t *p, uint32_t pos, uint32_t skip) {
    c.bpos = pos;
    bc_fill(c, p);
    bc_take(c, p);
    c.rem -= skip;
}

__device__ __forceinline__ uint32_t bc_next(BCursor &c, const uint8_t *p) {
    if (c.rem == 0) bc_take(c, p);
    --c.rem;
    return c.byte;
}

__device__ __forceinline__ void cur_init(Cursor &c, const uint8_t *p, uint32_t pos, uint32_t skip) {
    c.pos = pos;
    c.byte = p[pos];
    c.rem = p[pos + 1] - skip;
}

__device__ __forceinline__ uint32_t cur_next(Cursor &c, const uint8_t *p) {
    if (c.rem == 0) {
        c.pos += 2;
        c.byte = p[c.pos];
        c.rem = p[c.pos + 1];
    }
    --c.rem;
    return c.byte;
}

// Tile width for a CTA holding `rows` chunks: kTileElems for a full CTA, wider
// when only a few chunks are coded (init, read-back), so the serial per-chunk
// loop crosses fewer barriers.  rows * (te + 1) <= kSlotsPerCta * (kTileElems + 1).
__device__ __forceinline__ uint32_t tile_width(uint32_t rows, uint64_t N) {
    uint32_t rp = 1;
    while (rp < rows) rp <<= 1;
    return uint32_t(umin64(uint64_t(kTileElems) * (kSlotsPerCta / rp), N));
}

// Tile of kSlotsPerCta rows x kTileElems amplitudes (+1 pad element per row).
struct TileSmem {
    double2 f[kSlotsPerCta * (kTileElems + 1)];   // row r at r * (te + 1)
};

__device__ __forceinline__ void store_tile(TileSmem &t, double2 *win, uint64_t slot0,
                                           uint64_t nslots, uint64_t N, uint64_t e0,
                                           uint32_t te, uint32_t stride) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t r = warp; r < kSlotsPerCta; r += nw) {
        if (slot0 + r >= nslots) break;
        for (uint32_t e = lane; e < te; e += 32) win[(slot0 + r) * N + e0 + e] = t.f[r * stride + e];
    }
}


__device__ __forceinline__ double comp(const double2 &v, uint32_t h) { return h ? v.y : v.x; }
__device__ __forceinline__ void set_comp(double2 &v, uint32_t h, double x) {
    if (h) v.y = x; else v.x = x;
}

// Lossy decode, warp per (slot, half): 32 elements per step.  Each lane
// expands one element's code from the two byte planes (32 pairs fetched per
// plane, warp scan of the runs, binary search by shuffles), raw escapes are
// ranked by ballot and fetched in parallel, d = code * 2eb is formed per lane,
// and only the predictor chain itself — pred = raw ? value : pred + d, the
// reference's sequence of roundings (codec.cpp:217-249) — runs serially over
// the 32 lanes' values.  One chain per warp instead of per thread: enough
// warps to hide latency when a window holds few chunks.
struct PlaneRd {
    uint32_t pp;    // byte offset of the current pair
    uint32_t rem;   // elements left in it
};

__device__ __forceinline__ uint32_t plane_block(PlaneRd &c, const uint8_t *p, uint32_t lane) {
    if (c.rem >= 32) {
        // the whole block lies in the current run
        const uint32_t byte = __ldg(p + c.pp);
        c.rem -= 32;
        if (c.rem == 0) {
            c.pp += 2;
            c.rem = __ldg(p + c.pp + 1);
        }
        return byte;
    }
    const uint32_t q = c.pp + 2 * lane;
    const uint32_t b = __ldg(p + q);
    uint32_t r = __ldg(p + q + 1);
    if (lane == 0) r = c.rem;
    uint32_t S = r;   // inclusive scan of the runs
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, S, o);
        if (lane >= uint32_t(o)) S += t;
    }
    // pair of element `lane`: number of pairs whose scan is <= lane
    uint32_t j = 0;
#pragma unroll
    for (uint32_t step = 16; step; step >>= 1) {
        const uint32_t sv = __shfl_sync(0xffffffffu, S, j + step - 1);
        if (sv <= lane) j += step;
    }
    const uint32_t byte = __shfl_sync(0xffffffffu, b, j);
    // advance past 32 elements
    const uint32_t j31 = __shfl_sync(0xffffffffu, j, 31);
    const uint32_t s31 = __shfl_sync(0xffffffffu, S, j31);
    const uint32_t rnext = __shfl_sync(0xffffffffu, r, (j31 + 1) & 31);
    if (s31 > 32) {
        c.pp += 2 * j31;
        c.rem = s31 - 32;
    } else {
        c.pp += 2 * (j31 + 1);
        c.rem = j31 + 1 < 32 ? rnext : uint32_t(__ldg(p + c.pp + 1));
    }
    return byte;
}

__device__ __forceinline__ bool chunk_dead(const CodecGeom &g, const uint64_t *slot_chunk, uint64_t s) {
    if (!g.dead_mask) return false;
    const uint64_t chunk = slot_chunk ? slot_chunk[s] : s;
    return (chunk & g.dead_mask) != g.dead_val;
}

__global__ void __launch_bounds__(256) k_dec_lossy_warp(
    const uint8_t *__restrict__ arena, const DecIdx *__restrict__ idx,
    const uint64_t *__restrict__ slot_chunk, uint64_t nslots, CodecGeom g,
    double2 *__restrict__ win, DevStatus *status, const uint32_t *cond) {
    if (cond && *cond == 0) return;
    __shared__ double chain[8][64];   // per warp: 32 inputs, 32 predictor values
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wg = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t s = wg >> 1;
    const uint32_t h = uint32_t(wg & 1);
    if (s >= nslots || chunk_dead(g, slot_chunk, s)) return;
    const DecIdx &d = idx[s];
    const uint64_t N = g.N;
    double *out = reinterpret_cast<double *>(win) + 2 * s * N + h;
    if (d.len == 0) {
        for (uint64_t e = lane; e < N; e += 32) __stcs(out + 2 * e, 0.0);
        return;
    }
    const uint8_t *p = arena + d.base;
    PlaneRd lo{d.pos[0][h], 0}, hi{d.pos[1][h], 0};
    lo.rem = uint32_t(__ldg(p + lo.pp + 1)) - d.skip[0][h];
    hi.rem = uint32_t(__ldg(p + hi.pp + 1)) - d.skip[1][h];
    // a zero remainder: the half starts at the next pair
    if (lo.rem == 0) { lo.pp += 2; lo.rem = __ldg(p + lo.pp + 1); }
    if (hi.rem == 0) { hi.pp += 2; hi.rem = __ldg(p + hi.pp + 1); }
    const double twoeb = 2.0 * d.eb;
    uint32_t raw_i = h ? d.raw_re : 0;
    const uint32_t raw_count = d.raw_count, raw_pos = d.raw_pos;
    double pred = 0.0;
    bool bad = false;
    for (uint64_t e0 = 0; e0 < N; e0 += 32) {
        // runs of code 0 in both planes: pred + (+0) = pred (a -0 becomes
        // +0), so whole 32-element blocks are value fills
        if (lo.rem >= 32 && hi.rem >= 32 && (__ldg(p + lo.pp) | __ldg(p + hi.pp)) == 0) {
            const uint32_t nb = uint32_t(umin64(min(lo.rem, hi.rem) / 32, (N - e0) / 32));
            pred = __dadd_rn(pred, 0.0);
            for (uint32_t k = 0; k < nb; ++k) __stcs(out + 2 * (e0 + 32 * k + lane), pred);
            lo.rem -= 32 * nb;
            hi.rem -= 32 * nb;
            if (lo.rem == 0) { lo.pp += 2; lo.rem = __ldg(p + lo.pp + 1); }
            if (hi.rem == 0) { hi.pp += 2; hi.rem = __ldg(p + hi.pp + 1); }
            e0 += 32 * uint64_t(nb) - 32;
            continue;
        }
        const uint32_t z = plane_block(lo, p, lane) | (plane_block(hi, p, lane) << 8);
        if (__all_sync(0xffffffffu, z == 0)) {
            // a block of code 0 across pair boundaries: a value fill
            pred = __dadd_rn(pred, 0.0);
            __stcs(out + 2 * (e0 + lane), pred);
            continue;
        }
        const bool raw = z == 0xFFFFu;
        const uint32_t rm = __ballot_sync(0xffffffffu, raw);
        double val;
        if (raw) {
            const uint32_t k = raw_i + __popc(rm & ((1u << lane) - 1));
            val = k < raw_count ? __longlong_as_double((long long)ld_u64(p + raw_pos + 8ull * k)) : 0.0;
        } else {
            // ((double)code * 2.0) * eb == (double)code * (2 eb) exactly
            val = __dmul_rn(double(unzigzag16(z)), twoeb);
        }
        raw_i += __popc(rm);
        bad |= raw_i > raw_count;
        // the chain through shared memory: broadcast reads of the inputs,
        // uniform writes of the running predictor
        double *cv = chain[threadIdx.x >> 5];
        cv[lane] = val;
        __syncwarp();
        if (rm == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                pred = __dadd_rn(pred, cv[i]);
                cv[32 + i] = pred;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const double x = cv[i];
                pred = ((rm >> i) & 1) ? x : __dadd_rn(pred, x);
                cv[32 + i] = pred;
            }
        }
        __syncwarp();
        __stcs(out + 2 * (e0 + lane), cv[32 + lane]);
        __syncwarp();
    }
    if (lane == 0) {
        if (bad) dev_fail(status, QZS_RAW_UNDER, slot_chunk ? slot_chunk[s] : s);
        else if (h == 1 && raw_i != raw_count) dev_fail(status, QZS_RAW_UNUSED, slot_chunk ? slot_chunk[s] : s);
    }
}

// Lossy decode for dense stores, 8-lane segments (codec.cpp:217-249): a warp
// decodes two chunks at once, one 8-lane segment per (chunk, half) — seg =
// lane / 8, chunk = 2 warp + seg / 2, half = seg % 2 — 8 elements per step.
// Per step every segment expands its 8 codes from the two byte planes
// (segment scan of the run lengths + shuffle search, width-8 shuffles), ranks
// its raw escapes by ballot, forms val = raw ? value : code * 2eb, and runs
// the predictor chain pred = raw ? val : pred + val (the reference's
// sequence of roundings) over its 8 values through shared memory.  Four
// chains share each chain instruction (one per 8 lanes), a quarter of the
// warp-per-chain kernel's serial cost; the real and imaginary segments of a
// chunk meet by shuffle and store whole amplitudes (8 x 16 B contiguous).
constexpr uint32_t kSegW = 8;

__device__ __forceinline__ uint32_t plane_seg(PlaneRd &c, const uint8_t *p, uint32_t sub) {
    const uint32_t q = c.pp + 2 * sub;
    const uint32_t b = __ldg(p + q);
    uint32_t r = __ldg(p + q + 1);
    if (sub == 0) r = c.rem;
    uint32_t S = r;   // inclusive scan of the runs within the segment
#pragma unroll
    for (uint32_t o = 1; o < kSegW; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, S, o, kSegW);
        if (sub >= o) S += t;
    }
    // pair of element `sub`: number of pairs whose scan is <= sub
    uint32_t j = 0;
#pragma unroll
    for (uint32_t step = kSegW / 2; step; step >>= 1) {
        const uint32_t sv = __shfl_sync(0xffffffffu, S, j + step - 1, kSegW);
        if (sv <= sub) j += step;
    }
    const uint32_t byte = __shfl_sync(0xffffffffu, b, j, kSegW);
    // advance past the segment's 8 elements
    const uint32_t jl = __shfl_sync(0xffffffffu, j, kSegW - 1, kSegW);
    const uint32_t sl = __shfl_sync(0xffffffffu, S, jl, kSegW);
    const uint32_t rnext = __shfl_sync(0xffffffffu, r, (jl + 1) & (kSegW - 1), kSegW);
    if (sl > kSegW) {
        c.pp += 2 * jl;
        c.rem = sl - kSegW;
    } else {
        c.pp += 2 * (jl + 1);
        c.rem = jl + 1 < kSegW ? rnext : uint32_t(__ldg(p + c.pp + 1));
    }
    return byte;
}

__global__ void __launch_bounds__(256) k_dec_lossy_seg(
    const uint8_t *__restrict__ arena, const DecIdx *__restrict__ idx,
    const uint64_t *__restrict__ slot_chunk, uint64_t nslots, CodecGeom g,
    double2 *__restrict__ win, DevStatus *status, const uint32_t *cond) {
    if (cond && *cond == 0) return;
    const uint32_t lane = threadIdx.x & 31, seg = lane >> 3, sub = lane & 7;
    const uint64_t s = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 2 + (seg >> 1);
    const uint32_t h = seg & 1;
    if (((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 2 >= nslots) return;   // whole warp
    {
        // both chunks of the warp statically +0: nothing to write
        const uint64_t s0 = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 2;
        if (chunk_dead(g, slot_chunk, s0) && (s0 + 1 >= nslots || chunk_dead(g, slot_chunk, s0 + 1))) return;
    }
    const bool exists = s < nslots;
    const DecIdx &d = idx[exists ? s : 0];
    const bool live = exists && d.len != 0;
    const uint64_t N = g.N;
    // dead segments (no chunk, or an index walk that failed) run on a
    // never-ending run at a valid address and produce zeros
    const uint8_t *p = live ? arena + d.base : arena;
    PlaneRd lo{0, 0x40000000u}, hi{0, 0x40000000u};
    if (live) {
        lo = PlaneRd{d.pos[0][h], uint32_t(__ldg(p + d.pos[0][h] + 1)) - d.skip[0][h]};
        hi = PlaneRd{d.pos[1][h], uint32_t(__ldg(p + d.pos[1][h] + 1)) - d.skip[1][h]};
        // a zero remainder: the half starts at the next pair
        if (lo.rem == 0) { lo.pp += 2; lo.rem = __ldg(p + lo.pp + 1); }
        if (hi.rem == 0) { hi.pp += 2; hi.rem = __ldg(p + hi.pp + 1); }
    }
    const double twoeb = live ? 2.0 * d.eb : 0.0;
    uint32_t raw_i = live && h ? d.raw_re : 0;
    const uint32_t raw_count = live ? d.raw_count : 0, raw_pos = live ? d.raw_pos : 0;
    double pred = 0.0;
    double2 *out = win + (exists ? s : 0) * N;
    for (uint64_t e0 = 0; e0 < N; e0 += kSegW) {
        const uint32_t z = plane_seg(lo, p, sub) | (plane_seg(hi, p, sub) << 8);
        const bool raw = live && z == 0xFFFFu;
        const uint32_t rm = (__ballot_sync(0xffffffffu, raw) >> (8 * seg)) & 0xFFu;
        double val = 0.0;
        if (raw) {
            const uint32_t k = raw_i + __popc(rm & ((1u << sub) - 1));
            val = k < raw_count ? __longlong_as_double((long long)ld_u64(p + raw_pos + 8ull * k)) : 0.0;
        } else if (live) {
            // ((double)code * 2.0) * eb == (double)code * (2 eb) exactly
            val = __dmul_rn(double(unzigzag16(z)), twoeb);
        }
        raw_i += __popc(rm);
        // the segment's chain in order, its values broadcast by shuffles
        // (every lane of the segment runs it; lane `sub` keeps step sub)
        double mine = 0.0;
#pragma unroll
        for (uint32_t i = 0; i < kSegW; ++i) {
            const double x = __shfl_sync(0xffffffffu, val, i, kSegW);
            pred = ((rm >> i) & 1) ? x : __dadd_rn(pred, x);
            if (i == sub) mine = pred;
        }
        const double im = __shfl_down_sync(0xffffffffu, mine, kSegW);
        if (h == 0 && exists) __stcs(out + e0 + sub, make_double2(live ? mine : 0.0, live ? im : 0.0));
    }
    if (live && sub == 0) {
        const uint64_t chunk = slot_chunk ? slot_chunk[s] : s;
        if (raw_i > raw_count) dev_fail(status, QZS_RAW_UNDER, chunk);
        else if (h == 1 && raw_i != raw_count) dev_fail(status, QZS_RAW_UNUSED, chunk);
    }
}

// Lossy decode (codec.cpp:217-249): thread = (slot, half).  WIDE: a launch
// with fewer chunks than one CTA row set uses wide tiles (tile_width).
template <bool WIDE>
__global__ void __launch_bounds__(2 * kSlotsPerCta) k_dec_lossy(
    const uint8_t *__restrict__ arena, const DecIdx *__restrict__ idx,
    const uint64_t *__restrict__ slot_chunk, uint64_t nslots, CodecGeom g,
    double2 *__restrict__ win, DevStatus *status, const uint32_t *cond) {
    if (cond && *cond == 0) return;
    __shared__ TileSmem tile;
    const uint32_t r = threadIdx.x >> 1, h = threadIdx.x & 1;
    const uint64_t slot0 = uint64_t(blockIdx.x) * kSlotsPerCta, s = slot0 + r;
    // every chunk of the CTA statically +0: nothing to write
    if (!__syncthreads_or(s < nslots && !chunk_dead(g, slot_chunk, s))) return;
    const bool active = s < nslots && idx[min(s, nslots - 1)].len != 0;
    const DecIdx *d = &idx[min(s, nslots - 1)];
    const uint8_t *p = arena + d->base;
    BCursor lo{0, 8, 0, 0, 0, 0}, hi{0, 8, 0, 0, 0, 0};
    uint32_t raw_i = 0, raw_count = 0, raw_pos = 0;
    double twoeb = 0.0, pred = 0.0;
    bool bad = false;
    if (active) {
        bc_init(lo, p, d->pos[0][h], d->skip[0][h]);
        bc_init(hi, p, d->pos[1][h], d->skip[1][h]);
        raw_i = h ? d->raw_re : 0;
        raw_count = d->raw_count;
        raw_pos = d->raw_pos;
        twoeb = 2.0 * d->eb;
    }
    const uint64_t N = g.N;
    const uint32_t rows = uint32_t(umin64(kSlotsPerCta, nslots - slot0));
    const uint32_t te = WIDE ? tile_width(rows, N) : uint32_t(umin64(kTileElems, N));
    // rows past the CTA's chunk count have no tile storage (wide tiles)
    double2 *row = tile.f + (WIDE ? min(r, rows - 1) * (te + 1) : r * (kTileElems + 1));
    const bool has_row = !WIDE || r < rows;
    for (uint64_t e0 = 0; e0 < N; e0 += te) {
        for (uint32_t e = 0; e < te && has_row; ++e) {
            if (active) {
                if (lo.rem == 0) bc_take(lo, p);
                if (hi.rem == 0) bc_take(hi, p);
                if ((lo.byte | hi.byte) == 0) {
                    // a stretch of code 0: pred + (+0) = pred (a -0 becomes +0)
                    const uint32_t k = min(min(lo.rem, hi.rem), te - e);
                    if (__double_as_longlong(pred) << 1 == 0) pred = 0.0;
                    for (uint32_t j = 0; j < k; ++j) set_comp(row[e + j], h, pred);
                    lo.rem -= k;
                    hi.rem -= k;
                    e += k - 1;
                    continue;
                }
                const uint32_t z = bc_next(lo, p) | (bc_next(hi, p) << 8);
                if (z == 0xFFFFu) {
                    if (raw_i >= raw_count) {
                        bad = true;
                    } else {
                        pred = __longlong_as_double((long long)ld_u64(p + raw_pos + 8ull * raw_i));
                        ++raw_i;
                    }
                } else {
                    const int32_t code = unzigzag16(z);
                    // ((double)code * 2.0) * eb == (double)code * (2 eb) exactly
                    pred = __dadd_rn(pred, __dmul_rn(double(code), twoeb));
                }
            }
            set_comp(row[e], h, pred);
        }
        __syncthreads();
        store_tile(tile, win, slot0, nslots, N, e0, te, WIDE ? te + 1 : kTileElems + 1);
        __syncthreads();
    }
    if (active) {
        if (bad) dev_fail(status, QZS_RAW_UNDER, slot_chunk ? slot_chunk[s] : s);
        else if (h == 1 && raw_i != raw_count) dev_fail(status, QZS_RAW_UNUSED, slot_chunk ? slot_chunk[s] : s);
    }
}

// Lossless decode (codec.cpp:251-263): 8 byte-plane cursors per half.
__global__ void __launch_bounds__(2 * kSlotsPerCta) k_dec_lossless(
    const uint8_t *__restrict__ arena, const DecIdx *__restrict__ idx, uint64_t nslots,
    CodecGeom g, double2 *__restrict__ win, const uint32_t *cond) {
    if (cond && *cond == 0) return;
    __shared__ TileSmem tile;
    const uint32_t r = threadIdx.x >> 1, h = threadIdx.x & 1;
    const uint64_t slot0 = uint64_t(blockIdx.x) * kSlotsPerCta, s = slot0 + r;
    const bool active = s < nslots && idx[min(s, nslots - 1)].len != 0;
    const DecIdx *d = &idx[min(s, nslots - 1)];
    const uint8_t *p = arena + d->base;
    Cursor cur[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        cur[k] = Cursor{0, 0, 0};
        if (active) cur_init(cur[k], p, d->pos[k][h], d->skip[k][h]);
    }
    const uint64_t N = g.N;
    const uint32_t te = uint32_t(umin64(kTileElems, N));
    double2 *row = tile.f + r * (kTileElems + 1);
    for (uint64_t e0 = 0; e0 < N; e0 += te) {
        for (uint32_t e = 0; e < te; ++e) {
            uint64_t bits = 0;
            if (active) {
#pragma unroll
                for (int k = 0; k < 8; ++k) bits |= uint64_t(cur_next(cur[k], p)) << (8 * k);
            }
            set_comp(row[e], h, __longlong_as_double((long long)bits));
        }
        __syncthreads();
        store_tile(tile, win, slot0, nslots, N, e0, te, kTileElems + 1);
        __syncthreads();
    }
}

// ----------------------------------------------------------------- encode --

// Tiles of kSlotsPerCta rows x kTileElems amplitudes (dynamic shared memory,
// kEncStages deep: the next tile's loads are in flight while the chains walk
// the current one).
constexpr int kEncStages = 2;
constexpr uint32_t kEncTileDoubles2 = kSlotsPerCta * (kTileElems + 1);
// RLE pairs staged per tile: 4 streams (half x plane) per row, up to te + 2
// pairs each (rows * (te + 2) <= kSlotsPerCta * (kTileElems + 2)), double
// buffered, plus per-stream (global start, count) words
constexpr uint32_t kEncPairWords = kSlotsPerCta * (kTileElems + 2) * 4;
constexpr size_t kEncSmem = sizeof(double2) * kEncTileDoubles2 * kEncStages +
                            2 * sizeof(uint16_t) * kEncPairWords + 2 * sizeof(uint32_t) * 2 * 4 * kSlotsPerCta +
                            sizeof(uint16_t *) * 4 * kSlotsPerCta;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// One byte plane's RLE of one half (rle_encode, codec.cpp:52-63, restated as
// a branch-free per-byte step).  The real half keeps its last run open (the
// assembler continues it into the imaginary half); the imaginary half holds
// back its first run (head), which may exceed 255 until the merge.  Pairs
// go straight to the scratch stream (the lossless encoder; the lossy one
// stages its pairs in shared memory, RleT below).
struct RleS {
    uint16_t *dst;
    uint32_t np0;         // pair index of dst[0] (0: dst is the stream)
    uint32_t np;          // pairs emitted
    uint32_t cur, cnt;    // open run (cur = 0x100: none yet)
    uint32_t hold;        // imaginary half, first run not closed yet
    uint32_t head_byte, head_len;
};

__device__ __forceinline__ void rle_start(RleS &s, uint16_t *dst, uint32_t hold) {
    s.dst = dst;
    s.np0 = 0;
    s.np = 0;
    s.cur = 0x100;
    s.cnt = 0;
    s.hold = hold;
    s.head_byte = 0;
    s.head_len = 0;
}

__device__ __forceinline__ void rle_emit(RleS &s, uint32_t v) { s.dst[s.np++ - s.np0] = uint16_t(v); }

// Same pair stream as the reference's greedy split: a run is emitted when it
// closes or reaches 255 (then restarts at 0), one (byte, run) u16 per pair.
__device__ __forceinline__ void rle_step(RleS &s, uint32_t x) {
    const bool diff = x != s.cur;
    if (diff && s.hold && s.cnt) {
        // the imaginary half's first run closes: it is the head
        s.head_byte = s.cur;
        s.head_len = s.cnt;
        s.hold = 0;
        s.cnt = 0;
    }
    const uint32_t c1 = s.cnt + 1;
    const bool emit = diff ? s.cnt != 0 : (c1 == 255 && !s.hold);
    const uint32_t val = s.cur | ((diff ? s.cnt : 255u) << 8);
    if (emit) rle_emit(s, val);
    s.cnt = diff ? 1u : (emit ? 0u : c1);
    s.cur = x;
}

// Close a half: the real half reports its open tail, the imaginary half
// emits its last run (or, still holding, reports the whole half as head).
__device__ __forceinline__ void rle_close(RleS &s, uint32_t h, EncHalf &m, int k) {
    if (h == 0) {
        m.edge_byte[k] = uint8_t(s.cur);
        m.edge_len[k] = s.cnt;
    } else {
        if (s.hold) {
            s.head_byte = s.cur;
            s.head_len = s.cnt;
        } else if (s.cnt > 0) {
            rle_emit(s, s.cur | (s.cnt << 8));
        }
        m.edge_byte[k] = uint8_t(s.head_byte);
        m.edge_len[k] = s.head_len;
    }
    m.npairs[k] = s.np;
}

__device__ __forceinline__ uint8_t *scratch_half(uint8_t *scratch, const CodecGeom &g,
                                                 uint64_t slot, uint32_t h) {
    return scratch + (2 * slot + h) * g.half_stride;
}

constexpr uint32_t kEncFlushWarps = 4;
constexpr uint32_t kEncThreads = 2 * kSlotsPerCta + 32 * kEncFlushWarps;

__device__ __forceinline__ void sts16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;\n" ::"r"(addr), "h"(static_cast<unsigned short>(v)) : "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// The lossy encoder's per-stream RLE state: rle_step's state machine with the
// tile's pairs staged in shared memory (byte address sbase, n staged so far)
// and the hold flag folded into the 255-split limit (lim = ~0 while the
// imaginary half's first run is held back).
struct RleT {
    uint32_t sbase, n;    // staging buffer (shared address), pairs staged this tile
    uint32_t np0;         // pairs of earlier tiles
    uint32_t cur, cnt, lim;
    uint32_t head_byte, head_len;
};

__device__ __forceinline__ void rlet_start(RleT &s, uint32_t hold) {
    s.sbase = 0;
    s.n = 0;
    s.np0 = 0;
    s.cur = 0x100;
    s.cnt = 0;
    s.lim = hold ? ~0u : 255u;
    s.head_byte = 0;
    s.head_len = 0;
}

__device__ __forceinline__ void rlet_step(RleT &s, uint32_t x) {
    const bool diff = x != s.cur;
    if (diff && s.lim == ~0u && s.cnt) {
        // the imaginary half's first run closes: it is the head (once per half)
        s.head_byte = s.cur;
        s.head_len = s.cnt;
        s.lim = 255u;
        s.cnt = 0;
    }
    const uint32_t c1 = s.cnt + 1;
    const bool emit = diff ? s.cnt != 0 : c1 == s.lim;
    const uint32_t val = s.cur | ((diff ? s.cnt : 255u) << 8);
    if (emit) sts16(s.sbase + 2 * s.n++, val);
    s.cnt = diff ? 1u : (emit ? 0u : c1);
    s.cur = x;
}

__device__ __forceinline__ void rlet_step_n(RleT &s, uint32_t x, uint32_t n) {
    if (n == 0) return;
    if (x != s.cur) {
        rlet_step(s, x);
        --n;
    }
    if (s.lim == ~0u) {
        s.cnt += n;
        return;
    }
    uint32_t tot = s.cnt + n;
    while (tot >= 255) {
        sts16(s.sbase + 2 * s.n++, x | (255u << 8));
        tot -= 255;
    }
    s.cnt = tot;
}

// Close a half (rle_close for the staged state; the imaginary half's last
// pair goes straight to the scratch stream out).
__device__ __forceinline__ void rlet_close(RleT &s, uint32_t h, EncHalf &m, int k, uint16_t *out) {
    uint32_t np = s.np0 + s.n;
    if (h == 0) {
        m.edge_byte[k] = uint8_t(s.cur);
        m.edge_len[k] = s.cnt;
    } else {
        if (s.lim == ~0u) {
            s.head_byte = s.cur;
            s.head_len = s.cnt;
        } else if (s.cnt > 0) {
            out[np++] = uint16_t(s.cur | (s.cnt << 8));
        }
        m.edge_byte[k] = uint8_t(s.head_byte);
        m.edge_len[k] = s.head_len;
    }
    m.npairs[k] = np;
}

// Lossy encode (codec.cpp:121-168).  CTA = kSlotsPerCta chunks, 4 warps:
//  * warps 0-1, thread = (slot, half): the sequential quantiser chain and the
//    RLE state machines of the half's two byte planes, staging the pairs in
//    shared memory;
//  * warps 2-3: flush the previous tile's staged pairs to the scratch streams
//    (each stream's new pairs as one contiguous, coalesced warp store);
//  * all 4 warps: cp.async the next tile ([32 chunks x te] amplitudes,
//    coalesced 512 B rows).
// Quantiser (codec.cpp:138-149) on the critical path, division-free and
// branch-free: t = d * fl(1/2eb), k = (t + 1.5*2^52) - 1.5*2^52 (t rounded
// to the nearest integer, ties to even, exact for |t| < 2^51), f = t - k
// (exact).  t differs from the reference's quotient fl(d / 2eb) by at most
// two roundings (|t| 2^-52 < 2^-37 for |t| < 2^15), so whenever
// |f| < 0.4999999 and |t| < 32767, round-half-away(fl(d/2eb)) == k exactly
// and |q| < 32768.  Everything else — a quotient near a half-integer, a
// code near the 16-bit limit, NaN / Inf, a forced raw — takes the exact
// path (the reference's division and std::round).  rec = pred + k * 2eb
// equals reconstruct(pred, code, eb) = pred + (code * 2.0) * eb exactly
// (multiplying by 2 commutes with rounding); k is never -0.
// FORCED: the launch carries forced-raw indices (the basis-state init only).
template <bool FORCED>
__global__ void __launch_bounds__(kEncThreads) k_enc_lossy(
    const double2 *__restrict__ win, uint64_t nslots, CodecGeom g,
    const uint64_t *__restrict__ forced, uint32_t nforced, uint8_t *__restrict__ scratch,
    EncHalf *__restrict__ meta) {
    extern __shared__ __align__(16) unsigned char enc_smem[];
    double2 *tiles = reinterpret_cast<double2 *>(enc_smem);
    uint16_t *pairs = reinterpret_cast<uint16_t *>(tiles + kEncTileDoubles2 * kEncStages);
    uint32_t *sinfo = reinterpret_cast<uint32_t *>(pairs + 2 * kEncPairWords);   // [2][start, count][4 * 32]
    uint16_t **sout = reinterpret_cast<uint16_t **>(sinfo + 2 * 2 * 4 * kSlotsPerCta);   // stream q's scratch
    const bool chain = threadIdx.x < 2 * kSlotsPerCta;
    const uint32_t r = (threadIdx.x >> 1) & (kSlotsPerCta - 1), h = threadIdx.x & 1;
    const uint64_t slot0 = uint64_t(blockIdx.x) * kSlotsPerCta, s = slot0 + r;
    const uint32_t rows = uint32_t(umin64(kSlotsPerCta, nslots - slot0));
    for (uint32_t q = threadIdx.x; q < 4 * rows; q += blockDim.x)
        sout[q] = reinterpret_cast<uint16_t *>(scratch_half(scratch, g, slot0 + (q >> 2), (q >> 1) & 1) +
                                               (q & 1) * g.scap);
    const bool active = chain && r < rows;
    const uint64_t N = g.N;
    const uint32_t te = tile_width(rows, N), lte = 31 - __clz(te);
    const uint64_t ntiles = N / te;
    const uint32_t pcap = te + 2;   // staged pairs per stream per tile
    // stream q = 4 r + 2 h + plane; its staging slice in buffer b
    auto stage = [&](int b, uint32_t q) { return pairs + b * kEncPairWords + q * pcap; };
    uint8_t *base = scratch_half(scratch, g, active ? s : 0, h);
    RleT lo, hi;
    rlet_start(lo, h);
    rlet_start(hi, h);
    double *raws = reinterpret_cast<double *>(base + 2 * g.scap);
    uint32_t nraw = 0;
    // forced raw cursor (sorted flat indices, codec.cpp:124-129)
    uint32_t fc = 0;
    uint64_t next_forced = ~uint64_t(0);
    if (FORCED) {
        while (active && fc < nforced && forced[fc] < h * N) ++fc;
        next_forced = fc < nforced ? forced[fc] : ~uint64_t(0);
    }
    const double eb = g.eb, twoeb = g.twoeb, inv = g.inv2eb;
    const double kRne = 6755399441055744.0;   // 1.5 * 2^52
    const double thr = __dmul_rn(0.99, eb);
    double pred = 0.0;
    auto tile = [&](uint64_t i) -> double2 * { return tiles + (i % kEncStages) * kEncTileDoubles2; };
    auto issue = [&](uint64_t i) {
        if (i < ntiles) {
            double2 *dst = tile(i);
            const uint64_t e0 = i * te;
            for (uint32_t j = threadIdx.x; j < rows * te; j += blockDim.x) {
                const uint32_t rr = j >> lte, e = j & (te - 1);
                cp_async16(dst + rr * (te + 1) + e, win + (slot0 + rr) * N + e0 + e);
            }
        }
        cp_async_commit();   // (empty groups keep the wait count uniform)
    };
    // flush warps: copy buffer b's staged pairs of every stream to scratch
    auto flush = [&](int b) {
        const uint32_t lane = threadIdx.x & 31, fw = (threadIdx.x >> 5) - 2;
        const uint32_t *info = sinfo + b * 2 * 4 * kSlotsPerCta;
        for (uint32_t q = fw; q < 4 * rows; q += kEncFlushWarps) {
            const uint32_t cnt = info[4 * kSlotsPerCta + q];
            if (cnt == 0) continue;
            uint16_t *out = sout[q] + info[q];
            const uint16_t *src = stage(b, q);
            for (uint32_t i = lane; i < cnt; i += 32) out[i] = src[i];
        }
    };
    issue(0);
    for (uint64_t ti = 0; ti < ntiles; ++ti) {
        const int pb = int(ti & 1);
        issue(ti + 1);
        cp_async_wait<1>();
        // (the barrier also tells whether the previous tile staged any pair:
        // fast-forwarded tiles of sparse states stage none, so the flush
        // warps skip their stream loop)
        const int staged = __syncthreads_or(active && (lo.n | hi.n) != 0);
        if (!chain) {
            if (ti && staged) flush(pb ^ 1);
        } else if (active) {
            const double *rowc = reinterpret_cast<const double *>(tile(ti) + r * (te + 1)) + h;
            const uint64_t tile0 = h * N + ti * te;
            lo.np0 += lo.n;
            hi.np0 += hi.n;
            lo.n = hi.n = 0;
            lo.sbase = smem_addr(stage(pb, 4 * r + 2 * h));
            hi.sbase = smem_addr(stage(pb, 4 * r + 2 * h + 1));
            // fast-forward: every value of the tile within 0.99 eb of the
            // predictor quantises to code 0 with the predictor fixed (rec =
            // pred + (+0), a -0 predictor becomes +0): two runs of byte 0
            bool ff = (!FORCED || next_forced >= tile0 + te) && fabs(__dsub_rn(rowc[0], pred)) < thr;
            if (ff) {
                bool all = true;
#pragma unroll 8
                for (uint32_t e = 1; e < te; ++e) all &= fabs(__dsub_rn(rowc[2 * e], pred)) < thr;
                ff = all;
                if (ff) {
                    rlet_step_n(lo, 0, te);
                    rlet_step_n(hi, 0, te);
                    pred = __dadd_rn(pred, 0.0);
                }
            }
            if (!ff) {
                uint32_t fr = ~0u;
                if (FORCED) fr = next_forced - tile0 < te ? uint32_t(next_forced - tile0) : ~0u;
#pragma unroll 4
                for (uint32_t e = 0; e < te; ++e) {
                    const double v = rowc[2 * e];
                    const double d = __dsub_rn(v, pred);
                    const double t = __dmul_rn(d, inv);
                    double q = __dsub_rn(__dadd_rn(t, kRne), kRne);
                    const double f = __dsub_rn(t, q);
                    bool raw = false;
                    if (!(fabs(f) < 0.4999999 && fabs(t) < 32767.0) || (FORCED && e == fr)) {
                        if (FORCED && e == fr) {
                            raw = true;
                            const uint64_t flat = tile0 + e;
                            do { ++fc; } while (fc < nforced && forced[fc] == flat);
                            next_forced = fc < nforced ? forced[fc] : ~uint64_t(0);
                            fr = next_forced - tile0 < te ? uint32_t(next_forced - tile0) : ~0u;
                        } else {
                            // the reference's quotient and std::round (half away)
                            q = round(__ddiv_rn(d, twoeb));
                            if (!(fabs(q) < 32768.0)) raw = true;
                            else q = __dadd_rn(q, 0.0);   // code 0 from -0
                        }
                    }
                    const double rec = __dadd_rn(pred, __dmul_rn(q, twoeb));
                    raw = raw || !(fabs(__dsub_rn(rec, v)) <= eb);
                    pred = raw ? v : rec;
                    const uint32_t z = raw ? 0xFFFFu : zigzag16(int32_t(q));
                    if (raw) raws[nraw++] = v;
                    rlet_step(lo, z & 0xffu);
                    rlet_step(hi, z >> 8);
                }
            }
            uint32_t *info = sinfo + pb * 2 * 4 * kSlotsPerCta;
            info[4 * r + 2 * h] = lo.np0;
            info[4 * r + 2 * h + 1] = hi.np0;
            info[4 * kSlotsPerCta + 4 * r + 2 * h] = lo.n;
            info[4 * kSlotsPerCta + 4 * r + 2 * h + 1] = hi.n;
        }
        __syncthreads();  // tile and staging buffers are reused next round
    }
    cp_async_wait<0>();
    if (__syncthreads_or(active && (lo.n | hi.n) != 0) && !chain && ntiles) flush(int((ntiles - 1) & 1));
    if (active) {
        EncHalf &m = meta[2 * s + h];
        rlet_close(lo, h, m, 0, reinterpret_cast<uint16_t *>(base));
        rlet_close(hi, h, m, 1, reinterpret_cast<uint16_t *>(base + g.scap));
        m.nraw = nraw;
    }
}

// RLE state machine writing its pairs straight to the scratch stream, four
// pairs per aligned 8-byte store (the stream starts 8-byte aligned).  Same
// pair stream as RleT / rle_step.
struct RleD {
    uint16_t *out;
    uint32_t np;          // pairs emitted
    uint64_t acc;         // pairs np & ~3 .. np - 1, not yet stored
    uint32_t cur, cnt, lim;
    uint32_t head_byte, head_len;
};

__device__ __forceinline__ void rled_start(RleD &s, uint16_t *out, uint32_t hold) {
    s.out = out;
    s.np = 0;
    s.acc = 0;
    s.cur = 0x100;
    s.cnt = 0;
    s.lim = hold ? ~0u : 255u;
    s.head_byte = 0;
    s.head_len = 0;
}

__device__ __forceinline__ void rled_emit(RleD &s, uint32_t v) {
    s.acc |= uint64_t(v & 0xffffu) << (16 * (s.np & 3));
    if ((s.np & 3) == 3) {
        *reinterpret_cast<uint64_t *>(s.out + (s.np & ~3u)) = s.acc;
        s.acc = 0;
    }
    ++s.np;
}

__device__ __forceinline__ void rled_step(RleD &s, uint32_t x) {
    const bool diff = x != s.cur;
    if (diff && s.lim == ~0u && s.cnt) {
        s.head_byte = s.cur;
        s.head_len = s.cnt;
        s.lim = 255u;
        s.cnt = 0;
    }
    const uint32_t c1 = s.cnt + 1;
    const bool emit = diff ? s.cnt != 0 : c1 == s.lim;
    const uint32_t val = s.cur | ((diff ? s.cnt : 255u) << 8);
    if (emit) rled_emit(s, val);
    s.cnt = diff ? 1u : (emit ? 0u : c1);
    s.cur = x;
}

__device__ __forceinline__ void rled_step_n(RleD &s, uint32_t x, uint32_t n) {
    if (n == 0) return;
    if (x != s.cur) {
        rled_step(s, x);
        --n;
    }
    if (s.lim == ~0u) {
        s.cnt += n;
        return;
    }
    uint32_t tot = s.cnt + n;
    while (tot >= 255) {
        rled_emit(s, x | (255u << 8));
        tot -= 255;
    }
    s.cnt = tot;
}

__device__ __forceinline__ void rled_close(RleD &s, uint32_t h, EncHalf &m, int k) {
    if (h == 0) {
        m.edge_byte[k] = uint8_t(s.cur);
        m.edge_len[k] = s.cnt;
    } else {
        if (s.lim == ~0u) {
            s.head_byte = s.cur;
            s.head_len = s.cnt;
        } else if (s.cnt > 0) {
            rled_emit(s, s.cur | (s.cnt << 8));
        }
        m.edge_byte[k] = uint8_t(s.head_byte);
        m.edge_len[k] = s.head_len;
    }
    // the stored-so-far words end at np & ~3: the rest pair by pair
    for (uint32_t i = s.np & ~3u; i < s.np; ++i) s.out[i] = uint16_t(s.acc >> (16 * (i & 3)));
    m.npairs[k] = s.np;
}

// Lossy encode, direct-output variant (round 2): CTA = 32
// chunks, 64 threads = (chunk, half); tiles staged by cp.async as in
// k_enc_lossy, but every thread writes its two RLE streams itself (RleD,
// 8-byte stores of four pairs) — no staging of pairs, no flush warps, a
// third of the shared memory, so more chains per SM.  Same payload bytes.
constexpr uint32_t kEncDThreads = 2 * kSlotsPerCta;
constexpr size_t kEncDSmem = sizeof(double2) * kEncTileDoubles2 * kEncStages;

template <bool FORCED>
__global__ void __launch_bounds__(kEncDThreads) k_enc_lossy_direct(
    const double2 *__restrict__ win, uint64_t nslots, CodecGeom g,
    const uint64_t *__restrict__ forced, uint32_t nforced, uint8_t *__restrict__ scratch,
    EncHalf *__restrict__ meta) {
    extern __shared__ __align__(16) unsigned char enc_smem[];
    double2 *tiles = reinterpret_cast<double2 *>(enc_smem);
    const uint32_t r = threadIdx.x >> 1, h = threadIdx.x & 1;
    const uint64_t slot0 = uint64_t(blockIdx.x) * kSlotsPerCta, s = slot0 + r;
    const uint32_t rows = uint32_t(umin64(kSlotsPerCta, nslots - slot0));
    const bool active = r < rows;
    const uint64_t N = g.N;
    const uint32_t te = tile_width(rows, N), lte = 31 - __clz(te);
    const uint64_t ntiles = N / te;
    uint8_t *base = scratch_half(scratch, g, active ? s : 0, h);
    RleD lo, hi;
    rled_start(lo, reinterpret_cast<uint16_t *>(base), h);
    rled_start(hi, reinterpret_cast<uint16_t *>(base + g.scap), h);
    double *raws = reinterpret_cast<double *>(base + 2 * g.scap);
    uint32_t nraw = 0;
    uint32_t fc = 0;
    uint64_t next_forced = ~uint64_t(0);
    if (FORCED) {
        while (active && fc < nforced && forced[fc] < h * N) ++fc;
        next_forced = fc < nforced ? forced[fc] : ~uint64_t(0);
    }
    const double eb = g.eb, twoeb = g.twoeb, inv = g.inv2eb;
    const double kRne = 6755399441055744.0;   // 1.5 * 2^52
    const double thr = __dmul_rn(0.99, eb);
    double pred = 0.0;
    auto tile = [&](uint64_t i) -> double2 * { return tiles + (i % kEncStages) * kEncTileDoubles2; };
    auto issue = [&](uint64_t i) {
        if (i < ntiles) {
            double2 *dst = tile(i);
            const uint64_t e0 = i * te;
            for (uint32_t j = threadIdx.x; j < rows * te; j += blockDim.x) {
                const uint32_t rr = j >> lte, e = j & (te - 1);
                cp_async16(dst + rr * (te + 1) + e, win + (slot0 + rr) * N + e0 + e);
            }
        }
        cp_async_commit();
    };
    issue(0);
    for (uint64_t ti = 0; ti < ntiles; ++ti) {
        issue(ti + 1);
        cp_async_wait<1>();
        __syncthreads();
        if (active) {
            const double *rowc = reinterpret_cast<const double *>(tile(ti) + r * (te + 1)) + h;
            const uint64_t tile0 = h * N + ti * te;
            bool ff = (!FORCED || next_forced >= tile0 + te) && fabs(__dsub_rn(rowc[0], pred)) < thr;
            if (ff) {
                bool all = true;
#pragma unroll 8
                for (uint32_t e = 1; e < te; ++e) all &= fabs(__dsub_rn(rowc[2 * e], pred)) < thr;
                ff = all;
                if (ff) {
                    rled_step_n(lo, 0, te);
                    rled_step_n(hi, 0, te);
                    pred = __dadd_rn(pred, 0.0);
                }
            }
            if (!ff) {
                uint32_t fr = ~0u;
                if (FORCED) fr = next_forced - tile0 < te ? uint32_t(next_forced - tile0) : ~0u;
#pragma unroll 4
                for (uint32_t e = 0; e < te; ++e) {
                    const double v = rowc[2 * e];
                    const double d = __dsub_rn(v, pred);
                    const double t = __dmul_rn(d, inv);
                    double q = __dsub_rn(__dadd_rn(t, kRne), kRne);
                    const double f = __dsub_rn(t, q);
                    bool raw = false;
                    if (!(fabs(f) < 0.4999999 && fabs(t) < 32767.0) || (FORCED && e == fr)) {
                        if (FORCED && e == fr) {
                            raw = true;
                            const uint64_t flat = tile0 + e;
                            do { ++fc; } while (fc < nforced && forced[fc] == flat);
                            next_forced = fc < nforced ? forced[fc] : ~uint64_t(0);
                            fr = next_forced - tile0 < te ? uint32_t(next_forced - tile0) : ~0u;
                        } else {
                            q = round(__ddiv_rn(d, twoeb));
                            if (!(fabs(q) < 32768.0)) raw = true;
                            else q = __dadd_rn(q, 0.0);   // code 0 from -0
                        }
                    }
                    const double rec = __dadd_rn(pred, __dmul_rn(q, twoeb));
                    raw = raw || !(fabs(__dsub_rn(rec, v)) <= eb);
                    pred = raw ? v : rec;
                    const uint32_t z = raw ? 0xFFFFu : zigzag16(int32_t(q));
                    if (raw) raws[nraw++] = v;
                    rled_step(lo, z & 0xffu);
                    rled_step(hi, z >> 8);
                }
            }
        }
        __syncthreads();   // the tile buffer is refilled next round
    }
    cp_async_wait<0>();
    if (active) {
        EncHalf &m = meta[2 * s + h];
        rled_close(lo, h, m, 0);
        rled_close(hi, h, m, 1);
        m.nraw = nraw;
    }
}

// Lossless encode (codec.cpp:169-181): thread = (slot, half, byte plane).
constexpr int kLLSlots = 16;
__global__ void __launch_bounds__(16 * kLLSlots) k_enc_lossless(
    const double2 *__restrict__ win, uint64_t nslots, CodecGeom g,
    uint8_t *__restrict__ scratch, EncHalf *__restrict__ meta) {
    __shared__ double2 tile[kLLSlots][kTileElems + 1];
    const uint32_t r = threadIdx.x >> 4, h = (threadIdx.x >> 3) & 1, k = threadIdx.x & 7;
    const uint64_t slot0 = uint64_t(blockIdx.x) * kLLSlots, s = slot0 + r;
    const bool active = s < nslots;
    const uint64_t N = g.N;
    RleS st;
    rle_start(st, reinterpret_cast<uint16_t *>(scratch_half(scratch, g, active ? s : 0, h) + k * g.scap), h);
    const uint32_t te = uint32_t(umin64(kTileElems, N));
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint64_t e0 = 0; e0 < N; e0 += te) {
        __syncthreads();
        for (uint32_t rr = warp; rr < kLLSlots; rr += nw)
            if (slot0 + rr < nslots && lane < te)
                tile[rr][lane] = __ldcs(win + (slot0 + rr) * N + e0 + lane);
        __syncthreads();
        if (!active) continue;
        for (uint32_t e = 0; e < te; ++e) {
            const uint64_t bits = (uint64_t)__double_as_longlong(comp(tile[r][e], h));
            rle_step(st, uint32_t(bits >> (8 * k)) & 0xff);
        }
    }
    if (active) {
        EncHalf &m = meta[2 * s + h];
        rle_close(st, h, m, k);
        if (k == 0) m.nraw = 0;
    }
}

// Pairs produced where the real half's open tail meets the imaginary half's
// held head (same split-at-255 phase as rle_encode over the joined plane).
__host__ __device__ __forceinline__ uint32_t boundary_pairs(uint32_t tb, uint32_t tc, uint32_t hb,
                                                            uint32_t hl) {
    if (tc > 0 && tb == hb) {
        const uint32_t t = tc + hl;
        return t / 255 + (t % 255 != 0);
    }
    return (tc > 0) + hl / 255 + (hl % 255 != 0);
}

__device__ __forceinline__ void boundary_pair(uint32_t i, uint32_t tb, uint32_t tc, uint32_t hb,
                                              uint32_t hl, uint32_t &b, uint32_t &run) {
    if (tc > 0 && tb == hb) {
        const uint32_t t = tc + hl, full = t / 255;
        b = hb;
        run = i < full ? 255 : t % 255;
        return;
    }
    if (tc > 0) {
        if (i == 0) { b = tb; run = tc; return; }
        --i;
    }
    b = hb;
    run = i < hl / 255 ? 255 : hl % 255;
}

__global__ void k_enc_sizes(const EncHalf *__restrict__ meta, uint64_t nslots, CodecGeom g,
                            uint64_t *__restrict__ sizes) {
    const uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    const EncHalf &a = meta[2 * s], &b = meta[2 * s + 1];
    uint64_t size = kHdr;
    for (uint32_t k = 0; k < g.planes; ++k)
        size += 2ull * (a.npairs[k] + b.npairs[k] +
                        boundary_pairs(a.edge_byte[k], a.edge_len[k], b.edge_byte[k], b.edge_len[k]));
    if (g.lossy) size += 8ull * (a.nraw + b.nraw);
    sizes[s] = size;
}

__global__ void k_arena_alloc(const uint64_t *rel_off, const uint64_t *sizes, uint64_t nslots,
                              uint64_t *used, uint64_t capacity, uint64_t *base_out,
                              DevStatus *status) {
    // atomic bump: windows on concurrent streams share one output arena
    const uint64_t total = rel_off[nslots - 1] + sizes[nslots - 1];
    const uint64_t base = atomicAdd((unsigned long long *)used, (unsigned long long)total);
    if (base + total > capacity) {
        dev_fail(status, QZS_ARENA, base + total);
        *base_out = 0;
        return;
    }
    *base_out = base;
}

// Warp copy of n bytes, any alignment: head bytes up to an 8-byte boundary
// of dst, then 8 bytes per lane (two aligned source words funnel-shifted into
// place), tail bytes.  Reads up to 8 bytes past the source range (scratch
// buffers keep >= 64 bytes of slack).
__device__ __forceinline__ void warp_copy(uint8_t *dst, const uint8_t *src, uint64_t n,
                                          uint32_t lane) {
    const uint64_t head = umin64((8 - (reinterpret_cast<uintptr_t>(dst) & 7)) & 7, n);
    if (lane < head) dst[lane] = src[lane];
    dst += head;
    src += head;
    n -= head;
    const uint64_t words = n >> 3;
    const uint32_t sh = uint32_t(reinterpret_cast<uintptr_t>(src) & 7);
    const uint64_t *s8 = reinterpret_cast<const uint64_t *>(src - sh);
    uint64_t *d8 = reinterpret_cast<uint64_t *>(dst);
    if (sh == 0) {
        for (uint64_t i = lane; i < words; i += 32) d8[i] = s8[i];
    } else {
        for (uint64_t i = lane; i < words; i += 32) {
            const uint64_t w0 = s8[i], w1 = s8[i + 1];
            d8[i] = (w0 >> (8 * sh)) | (w1 << (64 - 8 * sh));
        }
    }
    const uint64_t t0 = words << 3;
    if (t0 + lane < n) dst[t0 + lane] = src[t0 + lane];
}

// Warp per slot: header, merged planes, raws (codec.cpp:115-168).
__global__ void __launch_bounds__(256) k_assemble(
    const uint8_t *__restrict__ scratch, const EncHalf *__restrict__ meta,
    const uint64_t *__restrict__ rel_off, const uint64_t *__restrict__ sizes,
    const uint64_t *__restrict__ base_p, const uint64_t *__restrict__ slot_chunk, uint64_t nslots,
    CodecGeom g, uint8_t *__restrict__ arena, ChunkTable table, const DevStatus *status) {
    if (status->code == QZS_ARENA) return;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t base = *base_p;
    for (uint64_t s = warp; s < nslots; s += nwarps) {
        const EncHalf &a = meta[2 * s], &b = meta[2 * s + 1];
        uint8_t *dst = arena + base + rel_off[s];
        if (lane == 0) {
            dst[0] = g.lossy ? 1 : 2;
            st_u64(dst + 1, (uint64_t)__double_as_longlong(g.eb));
            st_u32(dst + 9, uint32_t(g.N));
            st_u32(dst + 13, g.lossy ? a.nraw + b.nraw : 0);
        }
        uint64_t pos = kHdr;
        const uint8_t *ha = scratch + (2 * s) * g.half_stride;
        const uint8_t *hb = ha + g.half_stride;
        for (uint32_t k = 0; k < g.planes; ++k) {
            warp_copy(dst + pos, ha + k * g.scap, 2ull * a.npairs[k], lane);
            pos += 2ull * a.npairs[k];
            const uint32_t tb = a.edge_byte[k], tc = a.edge_len[k];
            const uint32_t hbyte = b.edge_byte[k], hl = b.edge_len[k];
            const uint32_t nb = boundary_pairs(tb, tc, hbyte, hl);
            for (uint32_t i = lane; i < nb; i += 32) {
                uint32_t byte, run;
                boundary_pair(i, tb, tc, hbyte, hl, byte, run);
                dst[pos + 2 * i] = uint8_t(byte);
                dst[pos + 2 * i + 1] = uint8_t(run);
            }
            pos += 2ull * nb;
            warp_copy(dst + pos, hb + k * g.scap, 2ull * b.npairs[k], lane);
            pos += 2ull * b.npairs[k];
        }
        if (g.lossy) {
            warp_copy(dst + pos, ha + 2 * g.scap, 8ull * a.nraw, lane);
            pos += 8ull * a.nraw;
            warp_copy(dst + pos, hb + 2 * g.scap, 8ull * b.nraw, lane);
        }
        if (lane == 0) {
            const uint64_t chunk = slot_chunk ? slot_chunk[s] : s;
            table.off[chunk] = base + rel_off[s];
            table.len[chunk] = uint32_t(sizes[s]);
        }
    }
}

__global__ void k_slot_chunks(uint64_t *out, uint64_t nslots, uint64_t first_batch,
                              uint32_t log_members, uint64_t free_mask, uint64_t member_mask) {
    const uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    const uint64_t b = first_batch + (s >> log_members);
    const uint64_t j = s & ((uint64_t(1) << log_members) - 1);
    out[s] = deposit_bits(b, free_mask) | deposit_bits(j, member_mask);
}

// ---- host-staged residency: move window payloads between a mapped
// page-locked host arena and HBM with coalesced 16-byte zero-copy accesses ----

// Staging size per slot: payload + room to keep (dst - src) % 16 == 0.
__global__ void k_stage_sizes(ChunkTable table, const uint64_t *__restrict__ slot_chunk,
                              uint64_t nslots, uint64_t *__restrict__ padded) {
    const uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    padded[s] = round_up(uint64_t(table.len[slot_chunk[s]]) + 31, 16);
}

// Warp per slot: copy the 16-byte words covering the payload from the host
// arena into the HBM staging area; fill the slot-indexed local table.
__global__ void __launch_bounds__(256) k_gather(const uint8_t *__restrict__ host_arena, ChunkTable table,
                                                const uint64_t *__restrict__ slot_chunk,
                                                const uint64_t *__restrict__ soff, uint64_t nslots,
                                                uint8_t *__restrict__ stage, ChunkTable local) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t s = warp; s < nslots; s += nwarps) {
        const uint64_t chunk = slot_chunk[s];
        const uint64_t src = table.off[chunk];
        const uint32_t len = table.len[chunk];
        const uint64_t words = (uint64_t((src & 15) + len) + 15) / 16;
        const uint4 *in = reinterpret_cast<const uint4 *>(host_arena + (src & ~uint64_t(15)));
        uint4 *out = reinterpret_cast<uint4 *>(stage + soff[s]);
        // 8 x 16 B zero-copy reads in flight per lane: a few CTAs keep the
        // host link busy and leave the SMs to the decode / gate kernels
        uint64_t w = lane;
        for (; w + 7 * 32 < words; w += 8 * 32) {
            uint4 r[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = in[w + 32 * j];
#pragma unroll
            for (int j = 0; j < 8; ++j) out[w + 32 * j] = r[j];
        }
        for (; w < words; w += 32) out[w] = in[w];
        if (lane == 0) {
            local.off[s] = soff[s] + (src & 15);
            local.len[s] = len;
            local.crc[s] = table.crc[chunk];
        }
    }
}

// Reserve a 16-byte aligned block of the host arena for a window's output.
__global__ void k_host_alloc(const uint64_t *__restrict__ used_local, uint64_t *host_used, uint64_t cap,
                             uint64_t *base_out, DevStatus *status) {
    const uint64_t total = round_up(*used_local, 16);
    const uint64_t base = atomicAdd((unsigned long long *)host_used, (unsigned long long)total);
    if (base + total > cap) {
        dev_fail(status, QZS_ARENA, base + total);
        *base_out = ~uint64_t(0);
        return;
    }
    *base_out = base;
}

// Copy the window's contiguous output bytes HBM -> host arena (16 B words).
__global__ void k_copy_out(const uint8_t *__restrict__ stage, const uint64_t *__restrict__ used_local,
                           const uint64_t *__restrict__ base, uint8_t *__restrict__ host_arena) {
    if (*base == ~uint64_t(0)) return;
    const uint64_t words = round_up(*used_local, 16) / 16;
    const uint4 *in = reinterpret_cast<const uint4 *>(stage);
    uint4 *out = reinterpret_cast<uint4 *>(host_arena + *base);
    const uint64_t nth = uint64_t(gridDim.x) * blockDim.x;
    uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; w + 7 * nth < words; w += 8 * nth) {
        uint4 r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = in[w + nth * j];
#pragma unroll
        for (int j = 0; j < 8; ++j) out[w + nth * j] = r[j];
    }
    for (; w < words; w += nth) out[w] = in[w];
}

// Publish the window's entries in the global (chunk-indexed) table.
__global__ void k_table_out(ChunkTable local, const uint64_t *__restrict__ slot_chunk,
                            const uint64_t *__restrict__ base, uint64_t nslots, ChunkTable table) {
    const uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= nslots || *base == ~uint64_t(0)) return;
    const uint64_t chunk = slot_chunk[s];
    table.off[chunk] = *base + local.off[s];
    table.len[chunk] = local.len[s];
    table.crc[chunk] = local.crc[s];
}

unsigned grid_for(uint64_t n, unsigned threads) { return (unsigned)ceil_div(n, threads); }

} // namespace

// ------------------------------------------------------------------ host --

uint64_t payload_bound(uint64_t N, double eb) {
    // lossy: 2 planes x 2N pairs x 2 B + 2N raws x 8 B; lossless: 8 x 4N
    return kHdr + (eb > 0.0 ? 24 * N : 32 * N);
}

CodecGeom make_geom(uint64_t N, double eb) {
    CodecGeom g;
    g.N = N;
    g.lossy = eb > 0.0;
    g.planes = g.lossy ? 2 : 8;
    g.eb = eb;
    g.twoeb = 2.0 * eb;
    g.inv2eb = eb > 0.0 ? 1.0 / g.twoeb : 0.0;
    {
        int ex = 0;
        const double mant = std::frexp(g.twoeb, &ex);
        // exact reciprocal: power of two whose inverse is a normal double
        g.exact_inv = eb > 0.0 && mant == 0.5 && ex > -1020 && ex < 1020 ? 1u : 0u;
    }
    g.dense_hint = 0;
    g.enc_dense = 0;
    g.scap = round_up(2 * N, 8);
    g.half_stride = round_up(g.lossy ? 2 * g.scap + 8 * N : 8 * g.scap, 16);
    g.dead_mask = g.dead_val = 0;
    return g;
}

void init_codec_tables(CodecTables &t) {
    uint32_t T[8][256];
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? kPoly ^ (c >> 1) : c >> 1;
        T[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
        for (int k = 1; k < 8; ++k) T[k][i] = (T[k - 1][i] >> 8) ^ T[0][T[k - 1][i] & 0xff];
    QZ_CUDA(cudaMalloc(&t.crc8, sizeof T));
    QZ_CUDA(cudaMemcpy(t.crc8, T, sizeof T, cudaMemcpyHostToDevice));
}

void free_codec_tables(CodecTables &t) {
    if (t.crc8) cudaFree(t.crc8);
    t.crc8 = nullptr;
}

void launch_slot_chunks(uint64_t *slot_chunk, uint64_t nslots, uint64_t first_batch,
                        uint32_t log_members, uint64_t free_mask, uint64_t member_mask,
                        cudaStream_t s) {
    k_slot_chunks<<<grid_for(nslots, 256), 256, 0, s>>>(slot_chunk, nslots, first_batch,
                                                         log_members, free_mask, member_mask);
    QZ_CHECK_LAUNCH();
}

void launch_crc(const CodecTables &tabs, const uint8_t *arena, ChunkTable table,
                const uint64_t *slot_chunk, uint64_t nslots, bool verify, DevStatus *status,
                cudaStream_t s) {
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(nslots, 8), kNumSMs * 64);
    KProfScope prof(s, verify ? "k_crc(verify)" : "k_crc", 0, 0.0);
    k_crc<<<grid, 256, 0, s>>>(tabs.crc8, arena, table, slot_chunk, nslots, verify ? 1 : 0, status);
    QZ_CHECK_LAUNCH();
}

void launch_dec_index(const uint8_t *arena, ChunkTable table, const uint64_t *slot_chunk,
                      uint64_t nslots, const CodecGeom &g, DecIdx *idx, DevStatus *status,
                      cudaStream_t s, uint32_t *nzslot) {
    KProfScope prof(s, "k_dec_index", 0, 0.0);
    if (nzslot) QZ_CUDA(cudaMemsetAsync(nzslot + nslots, 0, 4, s));
    if (g.lossy && g.N >= 64 && 4 * g.N / 256 + 1 <= kIdxMaxSteps)
        k_dec_index_warp<<<grid_for(nslots, kIdxWarps), 32 * kIdxWarps, 0, s>>>(arena, table, slot_chunk,
                                                                              nslots, g, idx, status, nzslot);
    else {
        k_dec_index<<<grid_for(nslots, 64), 64, 0, s>>>(arena, table, slot_chunk, nslots, g, idx,
                                                        status);
        if (nzslot) QZ_CUDA(cudaMemsetAsync(nzslot, 1, 4 * nslots, s));   // unknown: nonzero
    }
    QZ_CHECK_LAUNCH();
}

void launch_decode(const uint8_t *arena, const DecIdx *idx, const uint64_t *slot_chunk,
                   uint64_t nslots, const CodecGeom &g, double2 *win, DevStatus *status,
                   cudaStream_t s, const uint32_t *cond, bool sparse) {
    const unsigned grid = grid_for(nslots, kSlotsPerCta);
    // bytes written: the live chunks only (a window's chunks cover every
    // value of the stage's dead-mask bits equally)
    const double dense = 16.0 * double(g.N) * double(nslots) / double(uint64_t(1) << __builtin_popcountll(g.dead_mask));
    // with statically-(+0) chunks skipped, the few live ones of a sparse
    // store decode warp-parallel (the run-filling kernel's per-CTA tail
    // would dominate)
    if (g.dead_mask) sparse = false;
    // QZ_DEC_KERNEL=warp|seg forces the dense-store kernel choice (tests)
    static const int force = getenv("QZ_DEC_KERNEL") ? (std::string(getenv("QZ_DEC_KERNEL")) == "seg" ? 1
                                                         : std::string(getenv("QZ_DEC_KERNEL")) == "thread" ? 2 : 0)
                                                      : -1;
    if (force == 2) sparse = true;   // (the thread-per-chain kernel on any store)
    const bool seg = g.lossy && g.N >= 64 && !sparse && (force >= 0 ? force == 1 : g.dense_hint != 0);
    KProfScope prof(s, cond ? "replay_decode" : seg ? "k_dec_lossy_seg" : (g.lossy && g.N >= 32 && !sparse) ? "k_dec_lossy_warp"
                                            : g.lossy ? "k_dec_lossy" : "k_dec_lossless", 0, cond ? 0.0 : dense);
    // dense payloads: warp per chunk-half (parallel RLE expansion, serial
    // predictor chain only); a store known to be mostly zero runs (right
    // after init): thread per chunk-half with run fills
    if (seg) {
        // dense store: 8-lane segments, two chunks per warp, 16 per CTA
        k_dec_lossy_seg<<<grid_for(nslots, 16), 256, 0, s>>>(arena, idx, slot_chunk, nslots, g, win, status, cond);
    } else if (g.lossy && g.N >= 32 && !sparse) {
        // warp per (slot, half): 4 slots per 256-thread CTA
        k_dec_lossy_warp<<<grid_for(nslots, 4), 256, 0, s>>>(arena, idx, slot_chunk, nslots, g, win,
                                                              status, cond);
    } else if (g.lossy && nslots < uint64_t(kSlotsPerCta))
        k_dec_lossy<true><<<grid, 2 * kSlotsPerCta, 0, s>>>(arena, idx, slot_chunk, nslots, g, win,
                                                             status, cond);
    else if (g.lossy)
        k_dec_lossy<false><<<grid, 2 * kSlotsPerCta, 0, s>>>(arena, idx, slot_chunk, nslots, g, win,
                                                              status, cond);
    else
        k_dec_lossless<<<grid, 2 * kSlotsPerCta, 0, s>>>(arena, idx, nslots, g, win, cond);
    QZ_CHECK_LAUNCH();
}

void launch_encode(const double2 *win, uint64_t nslots, const CodecGeom &g,
                   const uint64_t *forced, uint32_t nforced, uint8_t *scratch, EncHalf *meta,
                   cudaStream_t s) {
    static const int force_k = getenv("QZ_ENC_KERNEL") ? (std::string(getenv("QZ_ENC_KERNEL")) == "direct" ? 1 : 0) : -1;
    const bool direct_k = g.lossy && (force_k >= 0 ? force_k == 1 : g.enc_dense == 0);
    KProfScope prof(s, direct_k ? "k_enc_lossy_direct" : g.lossy ? "k_enc_lossy" : "k_enc_lossless", 0,
                    16.0 * double(g.N) * double(nslots));
    static bool attr = false;
    if (!attr) {
        QZ_CUDA(cudaFuncSetAttribute(k_enc_lossy<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kEncSmem)));
        QZ_CUDA(cudaFuncSetAttribute(k_enc_lossy<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kEncSmem)));
        QZ_CUDA(cudaFuncSetAttribute(k_enc_lossy_direct<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kEncDSmem)));
        QZ_CUDA(cudaFuncSetAttribute(k_enc_lossy_direct<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kEncDSmem)));
        attr = true;
    }
    // QZ_ENC_KERNEL=staged|direct forces the choice (tests); default: the
    // staged kernel when the stage's output is expected dense (its coalesced
    // pair flushes win when most elements emit pairs: supremacy-30 15.7 vs
    // 23.6 ms), the direct one otherwise (less per-tile overhead on
    // fast-forwarded tiles: QFT-30 3.7 vs 4.3 ms)
    const bool direct = direct_k;
    if (direct && nforced)
        k_enc_lossy_direct<true><<<grid_for(nslots, kSlotsPerCta), kEncDThreads, kEncDSmem, s>>>(
            win, nslots, g, forced, nforced, scratch, meta);
    else if (direct)
        k_enc_lossy_direct<false><<<grid_for(nslots, kSlotsPerCta), kEncDThreads, kEncDSmem, s>>>(
            win, nslots, g, forced, nforced, scratch, meta);
    else if (g.lossy && nforced)
        k_enc_lossy<true><<<grid_for(nslots, kSlotsPerCta), kEncThreads, kEncSmem, s>>>(
            win, nslots, g, forced, nforced, scratch, meta);
    else if (g.lossy)
        k_enc_lossy<false><<<grid_for(nslots, kSlotsPerCta), kEncThreads, kEncSmem, s>>>(
            win, nslots, g, forced, nforced, scratch, meta);
    else
        k_enc_lossless<<<grid_for(nslots, kLLSlots), 16 * kLLSlots, 0, s>>>(win, nslots, g,
                                                                           scratch, meta);
    QZ_CHECK_LAUNCH();
}

void launch_enc_sizes(const EncHalf *meta, uint64_t nslots, const CodecGeom &g, uint64_t *sizes,
                      cudaStream_t s) {
    k_enc_sizes<<<grid_for(nslots, 256), 256, 0, s>>>(meta, nslots, g, sizes);
    QZ_CHECK_LAUNCH();
}

void launch_arena_alloc(const uint64_t *rel_off, const uint64_t *sizes, uint64_t nslots,
                        uint64_t *used, uint64_t capacity, uint64_t *base_out,
                        DevStatus *status, cudaStream_t s) {
    k_arena_alloc<<<1, 1, 0, s>>>(rel_off, sizes, nslots, used, capacity, base_out, status);
    QZ_CHECK_LAUNCH();
}

void launch_assemble(const uint8_t *scratch, const EncHalf *meta, const uint64_t *rel_off,
                     const uint64_t *sizes, const uint64_t *base, const uint64_t *slot_chunk,
                     uint64_t nslots, const CodecGeom &g, uint8_t *arena, ChunkTable table,
                     const DevStatus *status, cudaStream_t s) {
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(nslots, 8), kNumSMs * 64);
    k_assemble<<<grid, 256, 0, s>>>(scratch, meta, rel_off, sizes, base, slot_chunk, nslots, g,
                                    arena, table, status);
    QZ_CHECK_LAUNCH();
}

void launch_stage_sizes(ChunkTable table, const uint64_t *slot_chunk, uint64_t nslots,
                        uint64_t *padded, cudaStream_t s) {
    k_stage_sizes<<<grid_for(nslots, 256), 256, 0, s>>>(table, slot_chunk, nslots, padded);
    QZ_CHECK_LAUNCH();
}

void launch_gather(const uint8_t *host_arena, ChunkTable table, const uint64_t *slot_chunk,
                   const uint64_t *soff, uint64_t nslots, uint8_t *stage, ChunkTable local,
                   cudaStream_t s) {
    // a small grid: the transfer is link-bound, the SMs stay with the compute stream
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(nslots, 8), 64);
    k_gather<<<grid, 256, 0, s>>>(host_arena, table, slot_chunk, soff, nslots, stage, local);
    QZ_CHECK_LAUNCH();
}

void launch_copy_out(const uint8_t *stage, const uint64_t *used_local, uint64_t *host_used,
                     uint64_t cap, uint64_t *base, uint8_t *host_arena, ChunkTable local,
                     const uint64_t *slot_chunk, uint64_t nslots, ChunkTable table,
                     DevStatus *status, cudaStream_t s) {
    k_host_alloc<<<1, 1, 0, s>>>(used_local, host_used, cap, base, status);
    QZ_CHECK_LAUNCH();
    k_copy_out<<<64, 256, 0, s>>>(stage, used_local, base, host_arena);
    QZ_CHECK_LAUNCH();
    k_table_out<<<grid_for(nslots, 256), 256, 0, s>>>(local, slot_chunk, base, nslots, table);
    QZ_CHECK_LAUNCH();
}

uint32_t crc32_host(const uint8_t *p, uint64_t n) {
    static uint32_t T[256];
    static bool ready = false;
    if (!ready) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? kPoly ^ (c >> 1) : c >> 1;
            T[i] = c;
        }
        ready = true;
    }
    uint32_t c = 0xFFFFFFFFu;
    for (uint64_t i = 0; i < n; ++i) c = T[(c ^ p[i]) & 0xff] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

uint64_t fnv1a64_host(const uint8_t *p, uint64_t n, uint64_t state) {
    for (uint64_t i = 0; i < n; ++i) {
        state ^= p[i];
        state *= 0x100000001b3ULL;
    }
    return state;
}

} // namespace qz
