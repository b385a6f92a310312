/*
 * qzcuda.h — C ABI of the B200-native compressed-chunk state-vector engine.
 *
 * This is the drop-in boundary for the MEMQSim hot path (reference:
 * /root/reference/proj, C++ library `qzsim`).  The reference has no FFI of its
 * own; its accelerator extension point is the abstract `qzsim::Device`
 * (include/qzsim/device.hpp:76-95) driven by `qzsim::run`
 * (src/pipeline.cpp:128-314), plus the chunk codec
 * (include/qzsim/codec.hpp:61-70).  Every entry point below replaces one of
 * those interfaces and cites it.  Plain C types only: pointers, sizes,
 * doubles, status ints.  The C++ host library (the qzsim headers under
 * include/qzsim in this repo) and the Python package both bind exactly these symbols.
 *
 * Conventions
 *   - Every function returns QZC_OK (0) or a negative QZC_E* status; the
 *     message of the last failure on the calling thread is qzc_last_error().
 *     The C++ layer maps status classes onto the reference's exception
 *     hierarchy (CodecError/StoreError/PlanError/DeviceError, util.hpp:34-37).
 *   - Amplitudes are interleaved complex<double> (re, im), 16 bytes each,
 *     exactly std::complex<double> / qzsim::Amplitude (util.hpp:32).
 *   - Payload bytes, CRC-32 and FNV-1a digests are bit-identical to the
 *     reference (codec.cpp:95-266, util.cpp:20-31, store.cpp:129-136).
 *   - "host" pointers may be pageable or pinned; "dev" pointers are CUDA
 *     device pointers on the context's device.
 */
#ifndef QZCUDA_H
#define QZCUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define QZC_OK 0
#define QZC_EINVAL (-1)   /* bad argument (reference: Error / PlanError)     */
#define QZC_ECODEC (-2)   /* malformed or corrupt payload (CodecError)        */
#define QZC_ESTORE (-3)   /* store geometry / index error (StoreError)        */
#define QZC_EPLAN (-4)    /* planner precondition (PlanError)                 */
#define QZC_EDEVICE (-5)  /* device bound / bad buffer bit (DeviceError)      */
#define QZC_ECUDA (-6)    /* CUDA runtime failure                             */
#define QZC_ENOMEM (-7)   /* HBM / arena capacity exhausted                   */

const char *qzc_last_error(void);
const char *qzc_version(void);

/* ---- gates -------------------------------------------------------------- */
/* Gate kinds in the reference's enum order (include/qzsim/gates.hpp:27-45). */
enum qzc_gate_kind {
    QZC_H = 0, QZC_X, QZC_Y, QZC_Z, QZC_S, QZC_SDG, QZC_T, QZC_TDG,
    QZC_RX, QZC_RY, QZC_RZ, QZC_U1, QZC_U2, QZC_U3,
    QZC_CX, QZC_CZ, QZC_SWAP
};

/* One gate (reference qzsim::Gate, gates.hpp:49-55).  For two-qubit kinds
 * qubits[0] is the control / higher-order matrix bit. */
typedef struct qzc_gate {
    uint32_t kind;
    uint32_t nqubits;
    uint32_t qubits[2];
    double params[3];
} qzc_gate;

/* Unitary of a gate, row-major, interleaved complex; dim 2 or 4.
 * Bit-identical to qzsim::gate_matrix (gates.cpp:114-182). */
int qzc_gate_matrix(const qzc_gate *gate, double *mat_out /* 32 doubles */,
                    uint32_t *dim_out);

/* ---- context ------------------------------------------------------------ */
typedef struct qzc_context qzc_context;

/* One context per GPU.  hbm_budget_bytes = 0 means "all free HBM minus a
 * safety margin".  Replaces make_reference_device's memory bound
 * (device.hpp:36-40, device.cpp:273-299). */
int qzc_context_create(int device, uint64_t hbm_budget_bytes,
                       qzc_context **out);
void qzc_context_destroy(qzc_context *ctx);
int qzc_synchronize(qzc_context *ctx);
/* Number of engine kernels launched on this context so far. */
uint64_t qzc_kernel_launches(const qzc_context *ctx);
/* CUDA-event timer on the context stream: begin records an event, end
 * records a second one, synchronizes and returns the elapsed seconds. */
int qzc_timer_begin(qzc_context *ctx);
int qzc_timer_end(qzc_context *ctx, double *seconds_out);

/* Per-launch kernel timing (the reference's OpBegin/OpEnd brackets,
 * device.cpp:308-321, 358-390, at kernel granularity).  When enabled, every
 * fused gate pass and codec kernel the engine launches is bracketed by two
 * CUDA events on its own stream.  Records: kernel name, tag (pass index
 * within the stage plan; 0 for codec kernels), stage index, seconds and the
 * launch's algorithmic bytes (32 B per window amplitude for a gate pass,
 * 16 B per dense amplitude for codec kernels — payload bytes excluded).
 * enable() clears the records; read() synchronizes the device, returns the
 * count in *count and, when out != NULL, copies up to cap records and
 * clears them.  Process-wide (one engine device per process). */
typedef struct qzc_kprof_record {
    char name[32];
    uint32_t tag;
    uint32_t stage;
    double seconds;
    double bytes;
} qzc_kprof_record;
int qzc_kprof_enable(qzc_context *ctx, int on);
int qzc_kprof_read(qzc_context *ctx, qzc_kprof_record *out, uint64_t cap, uint64_t *count);

/* Runtime-specialised gate passes (NVRTC; QZ_JIT=0 disables).  Full-tile
 * passes over windows of >= 2^QZ_JIT_MIN_BITS amplitudes are also compiled
 * as straight-line kernels on host threads and used once built; results are
 * identical to the AOT kernels.  qzc_jit_wait blocks until every queued
 * compile finished (returns how many built); qzc_jit_selftest compiles the
 * widest pass of `gates` (on buffer bits of a 2^nbits window) with NVRTC,
 * no GPU needed: QZC_OK or an error carrying NVRTC's log. */
uint64_t qzc_jit_wait(void);
int qzc_jit_selftest(const qzc_gate *gates, uint64_t ngates, uint32_t nbits);

/* ---- chunk codec (replaces codec.hpp:61-70) ----------------------------- */
/* Worst-case payload bytes for one chunk of `elements` amplitudes. */
uint64_t qzc_payload_bound(uint64_t elements, double error_bound);

/* Compress `count` chunks of `elements` amplitudes each (host arrays).
 * Chunk k's amplitudes are amps[k*elements .. (k+1)*elements).  Payloads are
 * written back to back into payload_out (capacity payload_cap) with
 * offsets[k], sizes[k] and crcs[k] (CRC-32 of the payload).  forced_raw lists
 * flat component indices (real plane [0,N), imaginary [N,2N)) forced onto the
 * raw path for EVERY chunk of the call (codec.hpp:55-64).
 * Reference: qzsim::compress, codec.cpp:95-185. */
int qzc_compress_host(qzc_context *ctx, const double *amps, uint64_t count,
                      uint64_t elements, double error_bound,
                      const uint64_t *forced_raw, uint64_t n_forced,
                      uint8_t *payload_out, uint64_t payload_cap,
                      uint64_t *offsets, uint32_t *sizes, uint32_t *crcs);

/* Decompress `count` payloads (host arrays) into amps_out.  Verifies each
 * CRC first; on failure returns QZC_ECODEC and names the chunk index
 * (chunk_index_base + k) in qzc_last_error(), like codec.cpp:187-190.
 * Reference: qzsim::decompress, codec.cpp:187-266. */
int qzc_decompress_host(qzc_context *ctx, const uint8_t *payloads,
                        const uint64_t *offsets, const uint32_t *sizes,
                        const uint32_t *crcs, uint64_t count,
                        uint64_t elements, uint64_t chunk_index_base,
                        double *amps_out);

/* CRC-32 (zlib polynomial) and FNV-1a-64 of a host byte span
 * (util.cpp:20-31).  Host helpers for the report path. */
uint32_t qzc_crc32(const uint8_t *bytes, uint64_t len);
uint64_t qzc_fnv1a64(const uint8_t *bytes, uint64_t len, uint64_t state);

/* ---- gate kernels (replaces kernels.hpp:24-38 / Device::apply_gates) ---- */
/* Apply gates (already remapped to buffer bits) in order to a host buffer of
 * 2^nbits amplitudes.  Bit-exact with qzsim::apply_gates. */
int qzc_apply_gates_host(qzc_context *ctx, double *amps, uint32_t nbits,
                         const qzc_gate *gates, uint64_t ngates);
/* Same on a device buffer (stream-ordered on the context stream). */
int qzc_apply_gates_dev(qzc_context *ctx, double *amps_dev, uint32_t nbits,
                        const qzc_gate *gates, uint64_t ngates);

/* A gate given by an explicit matrix (qzsim::GateMatrix, gates.hpp:64-71):
 * dim 2 or 4, row-major interleaved complex, qubits[0] = high matrix bit. */
typedef struct qzc_matrix_gate {
    uint32_t dim;
    uint32_t qubits[2];
    uint32_t reserved;
    double m[32];
} qzc_matrix_gate;
/* apply_single_qubit / apply_two_qubit with caller matrices (kernels.cpp:20-54). */
int qzc_apply_matrices_host(qzc_context *ctx, double *amps, uint32_t nbits,
                            const qzc_matrix_gate *gates, uint64_t ngates);
int qzc_apply_matrices_dev(qzc_context *ctx, double *amps_dev, uint32_t nbits,
                           const qzc_matrix_gate *gates, uint64_t ngates);
/* One gate over pair (dim 2) or group (dim 4) indices [begin, end) only —
 * the sub-range arguments of apply_single_qubit / apply_two_qubit
 * (kernels.cpp:20-54) that the reference uses to split a gate among its
 * kernel workers.  Only the amplitudes the range touches cross the link. */
int qzc_apply_matrix_range_host(qzc_context *ctx, double *amps, uint32_t nbits,
                                const qzc_matrix_gate *gate, uint64_t begin, uint64_t end);

/* ---- device buffers (replaces ReferenceDevice's buffer / staging,
 *      device.cpp:120-255, 404-449) --------------------------------------- */
/* All operations are stream-ordered on the context stream (the in-order
 * command queue of device.hpp:59-60); qzc_synchronize() waits for them. */
int qzc_buffer_alloc(qzc_context *ctx, uint64_t amps, double **dev_out);
void qzc_buffer_free(qzc_context *ctx, double *dev);
/* Copy `amps` amplitudes host -> device at dev[dev_offset ...]. */
int qzc_copy_h2d(qzc_context *ctx, double *dev, uint64_t dev_offset, const double *host,
                 uint64_t amps);
/* Copy `amps` amplitudes device -> host from dev[dev_offset ...]. */
int qzc_copy_d2h(qzc_context *ctx, double *host, const double *dev, uint64_t dev_offset,
                 uint64_t amps);
/* Device-side mapping pass dst[i] = src[i] (the Buffered strategy's
 * permutation, an identity over the gather layout, device.cpp:436-449). */
int qzc_permute(qzc_context *ctx, double *dst, const double *src, uint64_t amps);
/* Page-locked host memory for staging (cudaMallocHost). */
int qzc_host_alloc(qzc_context *ctx, uint64_t bytes, void **host_out);
void qzc_host_free(qzc_context *ctx, void *host);
/* Event-timed region on the context stream, for TransferStats. */
int qzc_event_record(qzc_context *ctx, void **event_out);
int qzc_event_elapsed(qzc_context *ctx, void *start, void *end, double *seconds_out);
void qzc_event_destroy(qzc_context *ctx, void *event);
/* 1 if the event has completed, 0 if work before it is still pending. */
int qzc_event_done(qzc_context *ctx, void *event);

/* ---- planner (plan(), planner.cpp:46-96) — host only, no context ---------- */
/* Stage partition of a circuit: stage s covers gates [first_gate[s],
 * first_gate[s] + stage_ngates[s]); its padded high set is
 * high[64*s .. 64*s + nhigh[s]).  Returns the stage count in *nstages; at
 * most `cap` stages are written. */
/* Fused-pass plan summary for gates already on buffer bits of a 2^nbits
 * window (host only, no GPU): out[0] passes, [1] register groups,
 * [2] relaxed groups, [3] gates, [4] fast-path ops (macros folded),
 * [5] OP_PDIAG ops.  fuse_mode as qzc_sim_config.fuse_gates (0..3).
 * (Engine-internal scheduling; no reference counterpart.) */
int qzc_pass_plan_stats(const qzc_gate *gates, uint64_t ngates, uint32_t nbits,
                        uint32_t fuse_mode, uint64_t *out);

int qzc_plan_export(uint32_t num_qubits, uint32_t chunk_qubits, uint32_t batch_qubits,
                    const qzc_gate *gates, uint64_t ngates, uint64_t *nstages,
                    uint64_t *first_gate, uint64_t *stage_ngates, uint32_t *nhigh,
                    uint32_t *high, uint64_t cap);

/* ---- simulator (replaces qzsim::run, pipeline.cpp:128-314) -------------- */
typedef struct qzc_sim qzc_sim;

typedef struct qzc_sim_config {
    uint32_t num_qubits;     /* n                                             */
    uint32_t chunk_qubits;   /* c  (PipelineConfig::chunk_qubits)             */
    uint32_t batch_qubits;   /* m  (PipelineConfig::batch_qubits)             */
    uint32_t skip_reencode;  /* NON-PARITY fast mode (the
                                reference re-encodes every chunk once per
                                stage): when the whole dense
                                state fits one HBM window, the circuit runs
                                as ONE stage (one decode and one encode per
                                run, m = n) — fewer lossy round trips, so
                                payload bytes differ from the reference and
                                numbers are reported apart from parity runs.
                                0 = the reference's semantics (default).   */
    double error_bound;      /* 0 selects the lossless codec                  */
    uint64_t window_amps;    /* dense amplitudes per device window; 0 = auto  */
    uint32_t residency;      /* 0 = compressed store in HBM, 1 = pinned host  */
    uint32_t renormalize;    /* PipelineConfig::renormalize                   */
    uint32_t fuse_gates;     /* 0 = one pass per gate; 1 = fused passes where
                                +0-safe diagonal units may keep qubits outside
                                the tile (default); 2 = fused, every gate
                                qubit inside the tile; 3 = as 1, plus checked
                                diagonal units (Z, S, CZ ...) in out-of-place
                                passes replayed pass by pass on a zero        */
    uint32_t debug_flags;    /* bit 0: always take the strict replay (test)   */
} qzc_sim_config;

/* Per-run statistics (SimulationReport subset, pipeline.hpp:53-67, plus
 * device-event phase times). */
typedef struct qzc_sim_stats {
    double wall_seconds;         /* stage loop, host clock                   */
    double decode_seconds;       /* CUDA-event phase sums                    */
    double gate_seconds;
    double encode_seconds;
    double h2d_seconds;
    double d2h_seconds;
    uint64_t stages;
    uint64_t batches;
    uint64_t gate_passes;
    uint64_t chunk_decompress_count;
    uint64_t chunk_recompress_count;
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    uint64_t kernel_launches;
    uint64_t current_bytes;      /* Footprint (store.hpp:31-36)              */
    uint64_t peak_bytes;
    uint64_t dense_bytes;
    uint64_t windows;
    uint64_t replays;            /* relaxed gate passes that met a zero / -0
                                    they could not evaluate without amplitudes
                                    outside their tile and were re-applied by
                                    their strict sub-plan (device-side, same
                                    bytes)                                    */
    uint64_t payload_in_bytes;   /* compressed bytes the stages decoded
                                    (sum over stages of the store's payload
                                    total at stage start)                    */
    uint64_t payload_out_bytes;  /* compressed bytes the stages encoded      */
} qzc_sim_stats;

int qzc_sim_create(qzc_context *ctx, const qzc_sim_config *cfg,
                   qzc_sim **out);
void qzc_sim_destroy(qzc_sim *sim);
/* |0...0> through the reference's init (store.cpp:26-81). */
int qzc_sim_init_basis(qzc_sim *sim);
/* The zero vector: every chunk is the reference's zero-chunk payload (the
 * ranks that do not hold amplitude 0 of a sharded |0...0>). */
int qzc_sim_init_zero(qzc_sim *sim);
/* Execute a circuit through the staged, batched, compressed pipeline. */
int qzc_sim_run(qzc_sim *sim, const qzc_gate *gates, uint64_t ngates);
int qzc_sim_stats_get(const qzc_sim *sim, qzc_sim_stats *out);
/* Number of stages the planner produces (plan(), planner.cpp:46-96). */
int qzc_sim_plan_stages(const qzc_sim *sim, const qzc_gate *gates,
                        uint64_t ngates, uint64_t *stages_out);
/* FNV-1a over payloads in chunk order (store.cpp:129-136). */
int qzc_sim_digest(qzc_sim *sim, uint64_t *digest_out);
/* Σ|a|^2, compensated (pipeline.cpp:119-126). */
int qzc_sim_norm(qzc_sim *sim, double *norm_out);
/* Total payload bytes and per-chunk sizes (chunk order). */
int qzc_sim_chunk_count(const qzc_sim *sim, uint64_t *count_out);
int qzc_sim_payload_bytes(qzc_sim *sim, uint64_t *total_out);
/* Copy all payloads to host in chunk order (the reference's ChunkStore
 * contents): payload_out gets the concatenation, sizes/crcs per chunk. */
int qzc_sim_export(qzc_sim *sim, uint8_t *payload_out, uint64_t cap,
                   uint32_t *sizes, uint32_t *crcs);
/* Replace the store with host payloads (QZST load / store_chunk path). */
int qzc_sim_import(qzc_sim *sim, const uint8_t *payloads,
                   const uint32_t *sizes, const uint32_t *crcs);
/* Decompress chunk range [first, first+count) to host amplitudes. */
int qzc_sim_read_chunks(qzc_sim *sim, uint64_t first, uint64_t count,
                        double *amps_out);
/* Compress host amplitudes into chunk `index` (ChunkStore::store_chunk). */
int qzc_sim_write_chunk(qzc_sim *sim, uint64_t index, const double *amps);
/* Normalised |<dense|store>|^2 against a dense device state of 2^n
 * amplitudes (oracle.cpp:95-113). */
int qzc_sim_fidelity_dev(qzc_sim *sim, const double *dense_dev,
                         double *fidelity_out);

/* ---- checkpoint / resume (ChunkStore::save / load, store.cpp:152-217) ---- */
/* The reference's QZST file: "QZST", n:u32, c:u32, eb:f64, then per chunk in
 * index order len:u32, crc:u32, payload.  save streams the payloads out of
 * the device arenas through a page-locked buffer; load streams them back in,
 * verifies every CRC on the device (QZC_ESTORE "checksum mismatch in chunk
 * i", store.cpp:200-201) and needs the simulator's n, c and error bound.
 * Saving between two qzc_sim_run calls that split a circuit at a stage
 * boundary of its plan and resuming from the file reproduces the unsplit
 * run's bytes (each stage is one codec round trip). */
int qzc_sim_save(qzc_sim *sim, const char *path);
int qzc_sim_load(qzc_sim *sim, const char *path);

/* ---- sharded runs: ownership change by chunk exchange --- */
/* No reference counterpart (the reference is one process).  A
 * rank's simulator holds the 2^(n-g-c) chunks whose global chunk index has
 * the rank's bits at the g owner positions (global qubit - c).  To move to
 * new owner positions:
 *   1. exchange_plan: per destination rank, the bytes (send_bytes[2^g]) and
 *      chunk count of its record group (host metadata only);
 *   2. exchange_pack: packs every group into a device buffer (engine-owned,
 *      valid until the next engine call on this sim; *send_dev_out), group d
 *      at the prefix sum of send_bytes — a group is a u64 record count, a
 *      padded array of 24-byte records (new local index, payload offset,
 *      len, crc) and the payloads, copied from the arena on the device;
 *   3. the caller moves the groups GPU to GPU (all_to_all over NCCL) into
 *      exchange_recv_buffer(total received bytes), source s at the prefix
 *      sum of recv_bytes;
 *   4. exchange_unpack: the received groups become the store in place (the
 *      receive buffer is the other arena; every local chunk must arrive
 *      exactly once, else QZC_ESTORE).
 * Payload bytes and CRCs are never re-encoded, so digests are unchanged. */
int qzc_sim_exchange_plan(qzc_sim *sim, uint32_t g, uint32_t rank, const uint32_t *old_pos,
                          const uint32_t *new_pos, uint64_t *send_bytes, uint64_t *send_chunks);
int qzc_sim_exchange_pack(qzc_sim *sim, void **send_dev_out, uint64_t *bytes_out);
int qzc_sim_exchange_recv_buffer(qzc_sim *sim, uint64_t bytes, void **recv_dev_out);
int qzc_sim_exchange_unpack(qzc_sim *sim, const uint64_t *recv_bytes);
/* The same record layout built / parsed on the host from a store given as
 * payloads in local chunk order (2^local_bits chunks) — the exchange's index
 * and format logic without a GPU (CPU tests over gloo).  pack_host writes
 * the groups into out (NULL: sizes only) and send_bytes[2^g]; unpack_host
 * turns received groups back into payloads / sizes / crcs in local order. */
int qzc_exchange_pack_host(uint32_t local_bits, uint32_t g, uint32_t rank, const uint32_t *old_pos,
                           const uint32_t *new_pos, const uint8_t *payloads, const uint32_t *sizes,
                           const uint32_t *crcs, uint8_t *out, uint64_t cap, uint64_t *send_bytes);
int qzc_exchange_unpack_host(uint32_t world, const uint8_t *recv, const uint64_t *recv_bytes,
                             uint32_t local_bits, uint8_t *payload_out, uint64_t cap, uint32_t *sizes,
                             uint32_t *crcs);

/* ---- dense fp64 reference run on the GPU (fidelity baseline) ------------ */
/* Uncompressed double-precision state on the device, same gate kernels.
 * Used for fidelity at n beyond the CPU oracle (oracle.hpp:21). */
int qzc_dense_run(qzc_context *ctx, uint32_t num_qubits, const qzc_gate *gates,
                  uint64_t ngates, double **dense_dev_out);
void qzc_dense_free(qzc_context *ctx, double *dense_dev);

#ifdef __cplusplus
}
#endif
#endif /* QZCUDA_H */
