/*
 * qz_oracle.h — CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as the checker.
 * The product (libqzcuda.so) never links or calls it.
 *
 * Each function restates one reference function and cites it
 * (/root/reference/proj/...).  Parity is pinned against the reference itself
 * (oracle/_ref built from the reference sources, see oracle/Makefile) and the
 * golden fixtures under tests/golden/ (tests/golden/make_golden.py).
 *
 * Build flags matter: no FMA contraction (-ffp-contract=off, no -march), so
 * complex products round exactly like the reference build.
 */
#ifndef QZ_ORACLE_H
#define QZ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/qzcuda.h" /* qzc_gate layout only (plain struct) */

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double re, im;
} qzo_amp;

uint32_t qzo_gate_arity(uint32_t kind);
uint32_t qzo_gate_nparams(uint32_t kind);
/* gates.cpp:114-182 */
int qzo_gate_matrix(const qzc_gate *g, qzo_amp *m /*16*/, uint32_t *dim);

/* kernels.cpp:20-68 */
void qzo_apply_1q(qzo_amp *buf, uint32_t bit, const qzo_amp *m,
                  uint64_t pair_begin, uint64_t pair_end);
void qzo_apply_2q(qzo_amp *buf, uint32_t bit0, uint32_t bit1, const qzo_amp *m,
                  uint64_t group_begin, uint64_t group_end);
int qzo_apply_gates(qzo_amp *buf, uint64_t count, const qzc_gate *gates,
                    uint64_t ngates);

/* util.cpp:20-31 (zlib crc32 restated with a table) */
uint32_t qzo_crc32(const uint8_t *p, size_t n);
uint64_t qzo_fnv1a64(const uint8_t *p, size_t n, uint64_t state);

/* codec.cpp:95-185.  Returns payload length or a negative error. */
uint64_t qzo_payload_bound(uint64_t n);
int64_t qzo_compress(const qzo_amp *a, uint64_t n, double eb,
                     const uint64_t *forced, uint64_t nforced, uint8_t *out,
                     uint64_t cap, uint32_t *crc);
/* codec.cpp:187-266.  0 on success; <0 on error (message in errbuf). */
int qzo_decompress(const uint8_t *payload, uint64_t len, uint32_t crc,
                   uint64_t n, qzo_amp *out, char *errbuf, size_t errlen);

/* planner.cpp:22-141 */
typedef struct {
    uint64_t first_gate; /* index into the circuit */
    uint64_t ngates;
    uint32_t nhigh;
    uint32_t high[64]; /* sorted, padded */
} qzo_stage;
int qzo_plan(uint32_t n, const qzc_gate *gates, uint64_t ngates, uint32_t c,
             uint32_t m, qzo_stage *stages, uint64_t cap, uint64_t *nstages);
void qzo_batch_members(const qzo_stage *st, uint32_t n, uint32_t c,
                       uint64_t batch, uint64_t *members);
int qzo_remap(const qzo_stage *st, uint32_t c, const qzc_gate *in,
              qzc_gate *out);

/* Whole pipeline run (pipeline.cpp:128-314 semantics, single-threaded):
 * store init (store.cpp:26-81), every stage decompresses / applies /
 * recompresses each batch once.  Outputs the final store as concatenated
 * payloads (chunk order) when payload_out != NULL. */
typedef struct {
    uint64_t digest;
    double norm;
    uint64_t current_bytes;
    uint64_t peak_bytes;
    uint64_t dense_bytes;
    uint64_t stages;
    uint64_t total_payload;
    double seconds;
} qzo_run_result;
int qzo_run(uint32_t n, const qzc_gate *gates, uint64_t ngates, uint32_t c,
            uint32_t m, double eb, qzo_run_result *res, uint8_t *payload_out,
            uint64_t cap, uint32_t *sizes_out);

/* Dense state (oracle.cpp:20-119; uses the kernel formula, not the oracle's
 * 0+ accumulation, so it is bit-comparable to apply_gates). */
int qzo_dense(uint32_t n, const qzc_gate *gates, uint64_t ngates,
              qzo_amp *out);
double qzo_fidelity(const qzo_amp *a, const qzo_amp *b, uint64_t count);

/* circuit generators (generators.cpp:21-57) */
uint64_t qzo_make_ghz(uint32_t n, qzc_gate *out, uint64_t cap);
uint64_t qzo_make_qft(uint32_t n, qzc_gate *out, uint64_t cap);

#ifdef __cplusplus
}
#endif
#endif
