// qz_codec.cuh — device codec: bit-exact LossyPQ / LosslessRLE chunk payloads.
//
// Payload format (codec.hpp:36-41, codec.cpp:95-185), little-endian:
//   u8 codec_id | f64 error_bound | u32 element_count | u32 raw_count |
//   RLE(plane 0) | ... | RLE(plane P-1) | raw f64 values (lossy only)
// Lossy: P = 2 byte planes (low / high byte of the 16-bit zigzag code) over
// the 2N components (real plane then imaginary plane).  Lossless: P = 8 byte
// planes of the raw fp64 bits.  RLE = (byte, run) pairs, run in [1, 255],
// runs may cross the real→imaginary boundary.
#pragma once

#include "qz_common.cuh"

namespace qz {

// Compressed-chunk table in HBM (one entry per logical chunk index).
struct ChunkTable {
    uint64_t *off = nullptr;  // byte offset of the payload in its arena
    uint32_t *len = nullptr;  // payload bytes
    uint32_t *crc = nullptr;  // CRC-32 of the payload (CompressedChunk::checksum)
};

// Per-(slot, half) output of the encoder's sequential pass.
struct EncHalf {
    uint32_t npairs[8];     // complete pairs written to the scratch stream
    uint32_t edge_len[8];   // real half: open tail count [0,254]; imag half: head run
    uint8_t edge_byte[8];
    uint32_t nraw;
    uint32_t pad;
};

// Per-slot decode cursors derived from the payload (or from the encoder).
struct DecIdx {
    uint64_t base;          // arena offset
    double eb;              // error bound from the payload header
    uint32_t len;
    uint32_t raw_pos;       // payload-relative offset of the raw section
    uint32_t raw_count;
    uint32_t raw_re;        // raws consumed by the real half
    uint32_t pos[8][2];     // per stream, per half: payload offset of the pair
    uint32_t skip[8][2];    // elements of that pair used before the half starts
};

// Geometry of one codec call.
struct CodecGeom {
    uint64_t N;             // elements per chunk (2^c)
    uint32_t lossy;         // error_bound > 0
    uint32_t planes;        // 2 or 8
    double eb, twoeb;       // store error bound, 2*eb
    double inv2eb;          // fl(1 / (2 eb)) for the division-free quantiser
    uint32_t exact_inv;     // 2 eb is a power of two: the reciprocal is exact
    uint32_t dense_hint;    // the store compresses less than 16x: decode with the
                            // segmented kernel (set per stage by the runtime)
    uint32_t enc_dense;     // the stage's output is expected dense (dense input or a
                            // qubit mixed >= 4 times): staged encoder, else direct
    uint64_t scap;          // bytes per scratch stream (>= 2N, multiple of 8)
    uint64_t half_stride;   // scratch bytes per (slot, half)
    // decode only: chunks whose index differs from dead_val on dead_mask are
    // statically all +0 (fresh high qubits) and are not written — every
    // later reader zero-fills them (qz_gates PassDesc::fmask, the runtime's
    // dead fill before the encode)
    uint64_t dead_mask, dead_val;
};

CodecGeom make_geom(uint64_t N, double eb);
uint64_t payload_bound(uint64_t N, double eb);

// Device tables (CRC slicing tables + x^(2^k) mod P) — one per context.
struct CodecTables {
    uint32_t *crc8 = nullptr;   // 8 x 256 slicing-by-8 tables
};
void init_codec_tables(CodecTables &t);
void free_codec_tables(CodecTables &t);

// ---- launchers (all stream-ordered) --------------------------------------

// slot -> logical chunk index for a window of a stage:
//   chunk = deposit(first_batch + (s >> log_members), free_mask) |
//           deposit(s & (members-1), member_mask)
void launch_slot_chunks(uint64_t *slot_chunk, uint64_t nslots, uint64_t first_batch,
                        uint32_t log_members, uint64_t free_mask, uint64_t member_mask,
                        cudaStream_t s);

// CRC-32 of each slot's payload.  verify=true compares with table.crc and
// flags QZS_CRC; verify=false writes table.crc.
void launch_crc(const CodecTables &tabs, const uint8_t *arena, ChunkTable table,
                const uint64_t *slot_chunk, uint64_t nslots, bool verify,
                DevStatus *status, cudaStream_t s);

// Parse payload headers / RLE streams into decode cursors.
// nzslot (optional, nslots + 1 words): per slot 0 when the payload is known
// to decode to all (+0) (lossy, no raws, both byte planes only byte-0 runs),
// else nonzero; nzslot[nslots] = number of zero slots.
void launch_dec_index(const uint8_t *arena, ChunkTable table, const uint64_t *slot_chunk,
                      uint64_t nslots, const CodecGeom &g, DecIdx *idx, DevStatus *status,
                      cudaStream_t s, uint32_t *nzslot = nullptr);

// Decode every slot into win[slot*N .. (slot+1)*N).  cond != nullptr: the
// launch does nothing unless *cond != 0 (device-side replay, see run_passes).
void launch_decode(const uint8_t *arena, const DecIdx *idx, const uint64_t *slot_chunk,
                   uint64_t nslots, const CodecGeom &g, double2 *win, DevStatus *status,
                   cudaStream_t s, const uint32_t *cond = nullptr, bool sparse = false);

// Sequential encoder pass: codes, RLE sub-streams and raws into scratch.
void launch_encode(const double2 *win, uint64_t nslots, const CodecGeom &g,
                   const uint64_t *forced, uint32_t nforced, uint8_t *scratch,
                   EncHalf *meta, cudaStream_t s);

// Payload size per slot from the encoder metadata.
void launch_enc_sizes(const EncHalf *meta, uint64_t nslots, const CodecGeom &g,
                      uint64_t *sizes, cudaStream_t s);

// Reserve sum(sizes) bytes in an arena: *base_out = *used; *used += total.
void launch_arena_alloc(const uint64_t *rel_off, const uint64_t *sizes, uint64_t nslots,
                        uint64_t *used, uint64_t capacity, uint64_t *base_out,
                        DevStatus *status, cudaStream_t s);

// Write payloads at arena[*base + rel_off[slot]] and fill table entries.
void launch_assemble(const uint8_t *scratch, const EncHalf *meta, const uint64_t *rel_off,
                     const uint64_t *sizes, const uint64_t *base, const uint64_t *slot_chunk,
                     uint64_t nslots, const CodecGeom &g, uint8_t *arena, ChunkTable table,
                     const DevStatus *status, cudaStream_t s);

// Host-staged residency (mapped page-locked host arena):
//   padded[s] = staging bytes of slot s; soff = exclusive scan of padded;
//   gather copies payloads into `stage` and fills the slot-indexed `local`
//   table; copy_out moves a window's encoded bytes (stage[0, *used_local))
//   to the host arena and publishes the chunk-indexed table entries.
void launch_stage_sizes(ChunkTable table, const uint64_t *slot_chunk, uint64_t nslots,
                        uint64_t *padded, cudaStream_t s);
void launch_gather(const uint8_t *host_arena, ChunkTable table, const uint64_t *slot_chunk,
                   const uint64_t *soff, uint64_t nslots, uint8_t *stage, ChunkTable local,
                   cudaStream_t s);
void launch_copy_out(const uint8_t *stage, const uint64_t *used_local, uint64_t *host_used,
                     uint64_t cap, uint64_t *base, uint8_t *host_arena, ChunkTable local,
                     const uint64_t *slot_chunk, uint64_t nslots, ChunkTable table,
                     DevStatus *status, cudaStream_t s);

// Host-side CRC-32 / FNV-1a (util.cpp:20-31).
uint32_t crc32_host(const uint8_t *p, uint64_t n);
uint64_t fnv1a64_host(const uint8_t *p, uint64_t n, uint64_t state);

} // namespace qz
