/*
 * qz_oracle.c — CPU restatement of the MEMQSim (qzsim) hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see qz_oracle.h).  Written from the reference's
 * behaviour, one function per reference function, each citing the file:line
 * it restates under /root/reference/proj.  Compile WITHOUT FMA contraction.
 */
#include "qz_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---------------------------------------------------------------- gates -- */

/* gates.cpp:26-51 */
uint32_t qzo_gate_arity(uint32_t kind) {
    return (kind == QZC_CX || kind == QZC_CZ || kind == QZC_SWAP) ? 2u : 1u;
}

uint32_t qzo_gate_nparams(uint32_t kind) {
    switch (kind) {
    case QZC_RX: case QZC_RY: case QZC_RZ: case QZC_U1: return 1;
    case QZC_U2: return 2;
    case QZC_U3: return 3;
    default: return 0;
    }
}

static qzo_amp A(double re, double im) {
    qzo_amp a = {re, im};
    return a;
}

/* std::exp(complex(x, y)) in the reference is glibc cexp of the same pair. */
static qzo_amp cexp_of(double x, double y) {
    double complex z = cexp(CMPLX(x, y));
    return A(creal(z), cimag(z));
}

/* complex<double> * double == (re*d, im*d) */
static qzo_amp scale(qzo_amp a, double d) { return A(a.re * d, a.im * d); }

/* i * x as std::complex computes it: (0*x, 1*x) */
static qzo_amp exp_i(double x) { return cexp_of(0.0 * x, 1.0 * x); }
/* (-i) * x: (-0*x, -1*x) */
static qzo_amp exp_minus_i(double x) { return cexp_of(-0.0 * x, -1.0 * x); }

static void set2(qzo_amp *m, qzo_amp a, qzo_amp b, qzo_amp c, qzo_amp d) {
    m[0] = a;
    m[1] = b;
    m[2] = c;
    m[3] = d;
}

/* u3_matrix, gates.cpp:105-110 */
static void u3(qzo_amp *m, double theta, double phi, double lambda) {
    double ct = cos(theta / 2.0), st = sin(theta / 2.0);
    qzo_amp el = exp_i(lambda);
    qzo_amp neg_el = A(-el.re, -el.im);
    set2(m, A(ct, 0.0), scale(neg_el, st), scale(exp_i(phi), st),
         scale(exp_i(phi + lambda), ct));
}

/* gate_matrix, gates.cpp:114-182 */
int qzo_gate_matrix(const qzc_gate *g, qzo_amp *m, uint32_t *dim) {
    const double h = 0.7071067811865475244008443621048490;
    for (int i = 0; i < 16; ++i) m[i] = A(0.0, 0.0);
    *dim = 2;
    switch (g->kind) {
    case QZC_H: set2(m, A(h, 0), A(h, 0), A(h, 0), A(-h, 0)); return 0;
    case QZC_X: set2(m, A(0, 0), A(1, 0), A(1, 0), A(0, 0)); return 0;
    case QZC_Y: set2(m, A(0, 0), A(-0.0, -1.0), A(0.0, 1.0), A(0, 0)); return 0;
    case QZC_Z: set2(m, A(1, 0), A(0, 0), A(0, 0), A(-1, 0)); return 0;
    case QZC_S: set2(m, A(1, 0), A(0, 0), A(0, 0), A(0.0, 1.0)); return 0;
    case QZC_SDG: set2(m, A(1, 0), A(0, 0), A(0, 0), A(-0.0, -1.0)); return 0;
    case QZC_T: set2(m, A(1, 0), A(0, 0), A(0, 0), exp_i(M_PI / 4.0)); return 0;
    case QZC_TDG:
        set2(m, A(1, 0), A(0, 0), A(0, 0), exp_minus_i(M_PI / 4.0));
        return 0;
    case QZC_RX: {
        double hh = g->params[0] / 2.0;
        double c = cos(hh), s = sin(hh);
        qzo_amp off = A(-0.0 * s, -1.0 * s);
        set2(m, A(c, 0), off, off, A(c, 0));
        return 0;
    }
    case QZC_RY: {
        double hh = g->params[0] / 2.0;
        double c = cos(hh), s = sin(hh);
        set2(m, A(c, 0), A(-s, 0), A(s, 0), A(c, 0));
        return 0;
    }
    case QZC_RZ: {
        double hh = g->params[0] / 2.0;
        set2(m, exp_minus_i(hh), A(0, 0), A(0, 0), exp_i(hh));
        return 0;
    }
    case QZC_U1: set2(m, A(1, 0), A(0, 0), A(0, 0), exp_i(g->params[0])); return 0;
    case QZC_U2: u3(m, M_PI / 2.0, g->params[0], g->params[1]); return 0;
    case QZC_U3: u3(m, g->params[0], g->params[1], g->params[2]); return 0;
    case QZC_CX:
        *dim = 4;
        m[0] = m[5] = m[11] = m[14] = A(1, 0);
        return 0;
    case QZC_CZ:
        *dim = 4;
        m[0] = m[5] = m[10] = A(1, 0);
        m[15] = A(-1, 0);
        return 0;
    case QZC_SWAP:
        *dim = 4;
        m[0] = m[6] = m[9] = m[15] = A(1, 0);
        return 0;
    default: return -1;
    }
}

/* -------------------------------------------------------------- kernels -- */

/* complex<double> operator* (no FMA, separate roundings) */
static inline qzo_amp cmul(qzo_amp m, qzo_amp a) {
    qzo_amp r;
    r.re = m.re * a.re - m.im * a.im;
    r.im = m.re * a.im + m.im * a.re;
    return r;
}
static inline qzo_amp cadd(qzo_amp x, qzo_amp y) { return A(x.re + y.re, x.im + y.im); }

/* util.hpp:47-50 */
static inline uint64_t insert_zero_bit(uint64_t x, uint32_t bit) {
    uint64_t low = x & ((1ull << bit) - 1);
    return ((x >> bit) << (bit + 1)) | low;
}

/* kernels.cpp:20-34 */
void qzo_apply_1q(qzo_amp *buf, uint32_t bit, const qzo_amp *m,
                  uint64_t pair_begin, uint64_t pair_end) {
    const uint64_t stride = 1ull << bit;
    for (uint64_t p = pair_begin; p < pair_end; ++p) {
        uint64_t i = insert_zero_bit(p, bit), j = i | stride;
        qzo_amp a = buf[i], b = buf[j];
        buf[i] = cadd(cmul(m[0], a), cmul(m[1], b));
        buf[j] = cadd(cmul(m[2], a), cmul(m[3], b));
    }
}

/* kernels.cpp:36-54 */
void qzo_apply_2q(qzo_amp *buf, uint32_t bit0, uint32_t bit1, const qzo_amp *m,
                  uint64_t group_begin, uint64_t group_end) {
    uint32_t lo = bit0 < bit1 ? bit0 : bit1, hi = bit0 < bit1 ? bit1 : bit0;
    uint64_t s0 = 1ull << bit0, s1 = 1ull << bit1;
    for (uint64_t g = group_begin; g < group_end; ++g) {
        uint64_t base = insert_zero_bit(insert_zero_bit(g, lo), hi);
        uint64_t idx[4] = {base, base | s1, base | s0, base | s0 | s1};
        qzo_amp in[4];
        for (int k = 0; k < 4; ++k) in[k] = buf[idx[k]];
        for (int r = 0; r < 4; ++r) {
            qzo_amp acc = cmul(m[r * 4 + 0], in[0]);
            acc = cadd(acc, cmul(m[r * 4 + 1], in[1]));
            acc = cadd(acc, cmul(m[r * 4 + 2], in[2]));
            acc = cadd(acc, cmul(m[r * 4 + 3], in[3]));
            buf[idx[r]] = acc;
        }
    }
}

/* kernels.cpp:56-68 */
int qzo_apply_gates(qzo_amp *buf, uint64_t count, const qzc_gate *gates,
                    uint64_t ngates) {
    for (uint64_t k = 0; k < ngates; ++k) {
        qzo_amp m[16];
        uint32_t dim;
        if (qzo_gate_matrix(&gates[k], m, &dim)) return -1;
        if (dim == 2)
            qzo_apply_1q(buf, gates[k].qubits[0], m, 0, count / 2);
        else
            qzo_apply_2q(buf, gates[k].qubits[0], gates[k].qubits[1], m, 0,
                         count / 4);
    }
    return 0;
}

/* ------------------------------------------------------ crc32 / fnv1a64 -- */

static uint32_t crc_table[256];
static int crc_ready = 0;

static void crc_init(void) {
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
        crc_table[i] = c;
    }
    crc_ready = 1;
}

/* util.cpp:28-31 → zlib crc32(0, p, n) */
uint32_t qzo_crc32(const uint8_t *p, size_t n) {
    if (!crc_ready) crc_init();
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; ++i) c = crc_table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

/* util.cpp:20-26 */
uint64_t qzo_fnv1a64(const uint8_t *p, size_t n, uint64_t state) {
    for (size_t i = 0; i < n; ++i) {
        state ^= p[i];
        state *= 0x100000001b3ULL;
    }
    return state;
}

/* ---------------------------------------------------------------- codec -- */

#define HDR 17u

typedef struct {
    uint8_t *p;
    uint64_t len, cap;
    int overflow;
} sink;

static void put(sink *s, const void *src, uint64_t n) {
    if (s->len + n > s->cap) {
        s->overflow = 1;
        return;
    }
    memcpy(s->p + s->len, src, n);
    s->len += n;
}

/* rle_encode, codec.cpp:52-63: (byte, run) pairs, run in [1, 255] */
static void rle(sink *s, const uint8_t *b, uint64_t n) {
    uint64_t i = 0;
    while (i < n) {
        uint8_t v = b[i];
        uint64_t run = 1;
        while (run < 255 && i + run < n && b[i + run] == v) ++run;
        uint8_t pair[2] = {v, (uint8_t)run};
        put(s, pair, 2);
        i += run;
    }
}

static uint16_t zigzag(int32_t code) { return (uint16_t)((code << 1) ^ (code >> 15)); }
static int32_t unzigzag(uint16_t z) { return (int32_t)(z >> 1) ^ -(int32_t)(z & 1); }

uint64_t qzo_payload_bound(uint64_t n) {
    /* lossless: 8 planes * 2n bytes, each pair covers >= 1 byte; lossy is
     * smaller (2 planes + 8 bytes per raw component). */
    return HDR + 32 * n + 16;
}

/* compress, codec.cpp:95-185 */
int64_t qzo_compress(const qzo_amp *a, uint64_t n, double eb,
                     const uint64_t *forced, uint64_t nforced, uint8_t *out,
                     uint64_t cap, uint32_t *crc) {
    if (n == 0 || (n & (n - 1))) return -1;
    if (!(eb >= 0.0) || !isfinite(eb)) return -2;
    const uint64_t total = 2 * n;
    sink s = {out, 0, cap, 0};
    uint8_t id = eb > 0.0 ? 1 : 2;
    uint32_t n32 = (uint32_t)n;
    put(&s, &id, 1);
    put(&s, &eb, 8);
    put(&s, &n32, 4);
    uint8_t *plane = (uint8_t *)malloc(total);
    if (id == 1) {
        uint16_t *zz = (uint16_t *)malloc(total * 2);
        double *raws = (double *)malloc(total * 8);
        uint8_t *fr = (uint8_t *)calloc(total, 1);
        uint64_t nraw = 0;
        for (uint64_t k = 0; k < nforced; ++k) {
            if (forced[k] >= total) {
                free(zz); free(raws); free(fr); free(plane);
                return -3;
            }
            fr[forced[k]] = 1;
        }
        for (int pl = 0; pl < 2; ++pl) {
            double pred = 0.0;
            for (uint64_t j = 0; j < n; ++j) {
                uint64_t flat = pl * n + j;
                double v = pl == 0 ? a[j].re : a[j].im;
                int raw = fr[flat];
                int32_t code = 0;
                if (!raw) {
                    double q = round((v - pred) / (2.0 * eb));
                    if (!(fabs(q) < 32768.0)) {
                        raw = 1;
                    } else {
                        code = (int32_t)q;
                        double r = pred + (double)code * 2.0 * eb;
                        if (!(fabs(r - v) <= eb)) raw = 1;
                        else pred = r;
                    }
                }
                if (raw) {
                    raws[nraw++] = v;
                    pred = v;
                    zz[flat] = zigzag(-32768);
                } else {
                    zz[flat] = zigzag(code);
                }
            }
        }
        uint32_t nr32 = (uint32_t)nraw;
        put(&s, &nr32, 4);
        for (uint64_t i = 0; i < total; ++i) plane[i] = (uint8_t)(zz[i] & 0xFF);
        rle(&s, plane, total);
        for (uint64_t i = 0; i < total; ++i) plane[i] = (uint8_t)(zz[i] >> 8);
        rle(&s, plane, total);
        for (uint64_t i = 0; i < nraw; ++i) put(&s, &raws[i], 8);
        free(zz);
        free(raws);
        free(fr);
    } else {
        uint32_t zero = 0;
        put(&s, &zero, 4);
        for (int k = 0; k < 8; ++k) {
            for (uint64_t i = 0; i < total; ++i) {
                double v = i < n ? a[i].re : a[i - n].im;
                uint64_t bits;
                memcpy(&bits, &v, 8);
                plane[i] = (uint8_t)(bits >> (8 * k));
            }
            rle(&s, plane, total);
        }
    }
    free(plane);
    if (s.overflow) return -4;
    if (crc) *crc = qzo_crc32(out, s.len);
    return (int64_t)s.len;
}

static int fail(char *errbuf, size_t errlen, const char *msg) {
    if (errbuf && errlen) snprintf(errbuf, errlen, "%s", msg);
    return -1;
}

/* rle_decode, codec.cpp:65-79 */
static int unrle(const uint8_t *p, uint64_t len, uint64_t *pos, uint8_t *out,
                 uint64_t count, char *eb, size_t el) {
    uint64_t produced = 0;
    while (produced < count) {
        if (*pos + 2 > len) return fail(eb, el, "malformed payload: truncated RLE stream");
        uint8_t b = p[*pos], run = p[*pos + 1];
        *pos += 2;
        if (run == 0 || produced + run > count)
            return fail(eb, el, "malformed payload: bad RLE run length");
        memset(out + produced, b, run);
        produced += run;
    }
    return 0;
}

/* decompress, codec.cpp:187-266 */
int qzo_decompress(const uint8_t *p, uint64_t len, uint32_t crc, uint64_t n,
                   qzo_amp *out, char *eb, size_t el) {
    if (qzo_crc32(p, len) != crc) return fail(eb, el, "checksum mismatch");
    if (len < HDR) return fail(eb, el, "malformed payload: truncated header");
    uint8_t id = p[0];
    double bound;
    uint32_t count, nraw;
    memcpy(&bound, p + 1, 8);
    memcpy(&count, p + 9, 4);
    memcpy(&nraw, p + 13, 4);
    if (id != 1 && id != 2) return fail(eb, el, "malformed payload: unknown codec id");
    if (count != n) return fail(eb, el, "payload header disagrees with chunk metadata");
    uint64_t pos = HDR, total = 2 * n;
    int rc = 0;
    if (id == 1) {
        uint8_t *lo = (uint8_t *)malloc(total), *hi = (uint8_t *)malloc(total);
        double *planes = (double *)malloc(total * 8);
        if ((rc = unrle(p, len, &pos, lo, total, eb, el)) == 0 &&
            (rc = unrle(p, len, &pos, hi, total, eb, el)) == 0) {
            if (pos + (uint64_t)nraw * 8 > len) {
                rc = fail(eb, el, "malformed payload: missing raw values");
            } else {
                uint64_t used = 0;
                for (int pl = 0; pl < 2 && rc == 0; ++pl) {
                    double pred = 0.0;
                    for (uint64_t j = 0; j < n; ++j) {
                        uint64_t flat = pl * n + j;
                        int32_t code = unzigzag((uint16_t)(lo[flat] | (hi[flat] << 8)));
                        if (code == -32768) {
                            if (used >= nraw) {
                                rc = fail(eb, el, "malformed payload: raw value underflow");
                                break;
                            }
                            memcpy(&pred, p + pos + used * 8, 8);
                            ++used;
                        } else {
                            pred = pred + (double)code * 2.0 * bound;
                        }
                        planes[flat] = pred;
                    }
                }
                if (rc == 0 && used != nraw)
                    rc = fail(eb, el, "malformed payload: unused raw values");
                if (rc == 0)
                    for (uint64_t j = 0; j < n; ++j) out[j] = A(planes[j], planes[n + j]);
            }
        }
        free(lo);
        free(hi);
        free(planes);
    } else {
        uint64_t *bits = (uint64_t *)calloc(total, 8);
        uint8_t *pb = (uint8_t *)malloc(total);
        for (int k = 0; k < 8 && rc == 0; ++k) {
            rc = unrle(p, len, &pos, pb, total, eb, el);
            for (uint64_t i = 0; rc == 0 && i < total; ++i) bits[i] |= (uint64_t)pb[i] << (8 * k);
        }
        if (rc == 0)
            for (uint64_t j = 0; j < n; ++j) {
                memcpy(&out[j].re, &bits[j], 8);
                memcpy(&out[j].im, &bits[n + j], 8);
            }
        free(bits);
        free(pb);
    }
    return rc;
}

/* -------------------------------------------------------------- planner -- */

static int contains(const uint32_t *s, uint32_t k, uint32_t q) {
    for (uint32_t i = 0; i < k; ++i)
        if (s[i] == q) return 1;
    return 0;
}

static void sort_u32(uint32_t *s, uint32_t k) {
    for (uint32_t i = 1; i < k; ++i)
        for (uint32_t j = i; j > 0 && s[j - 1] > s[j]; --j) {
            uint32_t t = s[j];
            s[j] = s[j - 1];
            s[j - 1] = t;
        }
}

/* pad_high_set, planner.cpp:32-42: smallest free qubits >= c */
static void pad(qzo_stage *st, uint32_t n, uint32_t c, uint32_t m) {
    uint32_t target = (m - c) < (n - c) ? (m - c) : (n - c);
    for (uint32_t q = c; st->nhigh < target && q < n; ++q)
        if (!contains(st->high, st->nhigh, q)) st->high[st->nhigh++] = q;
    sort_u32(st->high, st->nhigh);
}

/* plan, planner.cpp:46-96 */
int qzo_plan(uint32_t n, const qzc_gate *gates, uint64_t ngates, uint32_t c,
             uint32_t m, qzo_stage *stages, uint64_t cap, uint64_t *nstages) {
    if (c < 1 || m < c + 2 || m > n) return -1;
    for (uint64_t i = 0; i < ngates; ++i) {
        const qzc_gate *g = &gates[i];
        if (g->nqubits != qzo_gate_arity(g->kind)) return -2;
        for (uint32_t k = 0; k < g->nqubits; ++k)
            if (g->qubits[k] >= n) return -2;
        if (g->nqubits == 2 && g->qubits[0] == g->qubits[1]) return -2;
    }
    const uint32_t capacity = m - c;
    uint64_t ns = 0;
    qzo_stage cur;
    memset(&cur, 0, sizeof cur);
    int open = 0;
    for (uint64_t i = 0; i < ngates; ++i) {
        const qzc_gate *g = &gates[i];
        uint32_t merged[64], k = cur.nhigh;
        memcpy(merged, cur.high, sizeof(uint32_t) * k);
        for (uint32_t t = 0; t < g->nqubits; ++t)
            if (g->qubits[t] >= c && !contains(merged, k, g->qubits[t])) merged[k++] = g->qubits[t];
        if (k > capacity) {
            /* close the stage, start a new one with this gate's high qubits */
            if (ns >= cap) return -3;
            pad(&cur, n, c, m);
            stages[ns++] = cur;
            memset(&cur, 0, sizeof cur);
            cur.first_gate = i;
            for (uint32_t t = 0; t < g->nqubits; ++t)
                if (g->qubits[t] >= c && !contains(cur.high, cur.nhigh, g->qubits[t]))
                    cur.high[cur.nhigh++] = g->qubits[t];
        } else {
            if (!open) cur.first_gate = i;
            memcpy(cur.high, merged, sizeof(uint32_t) * k);
            cur.nhigh = k;
        }
        open = 1;
        cur.ngates++;
    }
    if (open && cur.ngates) {
        if (ns >= cap) return -3;
        pad(&cur, n, c, m);
        stages[ns++] = cur;
    }
    *nstages = ns;
    return 0;
}

/* make_batch, planner.cpp:105-129 */
void qzo_batch_members(const qzo_stage *st, uint32_t n, uint32_t c,
                       uint64_t batch, uint64_t *members) {
    uint32_t chunk_bits = n - c, sp[64], fp[64], ns = 0, nf = 0;
    for (uint32_t i = 0; i < st->nhigh; ++i) sp[ns++] = st->high[i] - c;
    for (uint32_t b = 0; b < chunk_bits; ++b)
        if (!contains(sp, ns, b)) fp[nf++] = b;
    uint64_t base = 0;
    for (uint32_t i = 0; i < nf; ++i)
        if ((batch >> i) & 1) base |= 1ull << fp[i];
    for (uint64_t s = 0; s < (1ull << ns); ++s) {
        uint64_t idx = base;
        for (uint32_t i = 0; i < ns; ++i)
            if ((s >> i) & 1) idx |= 1ull << sp[i];
        members[s] = idx;
    }
}

/* remap_gate + Stage::buffer_bit, planner.cpp:22-28, 131-141 */
int qzo_remap(const qzo_stage *st, uint32_t c, const qzc_gate *in,
              qzc_gate *out) {
    *out = *in;
    for (uint32_t k = 0; k < in->nqubits; ++k) {
        uint32_t q = in->qubits[k];
        if (q < c) continue;
        uint32_t r = 0;
        while (r < st->nhigh && st->high[r] != q) ++r;
        if (r == st->nhigh) return -1;
        out->qubits[k] = c + r;
    }
    return 0;
}

/* ------------------------------------------------------------- pipeline -- */

typedef struct {
    uint8_t *p;
    uint32_t len, crc;
} chunk_t;

static int store_chunk(chunk_t *ch, const qzo_amp *vals, uint64_t len,
                       double eb, uint8_t *tmp, uint64_t tmpcap) {
    uint32_t crc;
    int64_t r = qzo_compress(vals, len, eb, NULL, 0, tmp, tmpcap, &crc);
    if (r < 0) return -1;
    free(ch->p);
    ch->p = (uint8_t *)malloc(r ? r : 1);
    memcpy(ch->p, tmp, r);
    ch->len = (uint32_t)r;
    ch->crc = crc;
    return 0;
}

/* run, pipeline.cpp:128-314 (device path, no host fraction; scheduling
 * knobs do not affect results). */
int qzo_run(uint32_t n, const qzc_gate *gates, uint64_t ngates, uint32_t c,
            uint32_t m, double eb, qzo_run_result *res, uint8_t *payload_out,
            uint64_t cap, uint32_t *sizes_out) {
    struct timespec t0, t1;
    if (c < 1 || c > n || n > 40) return -1;
    uint64_t max_stages = ngates + 1;
    qzo_stage *stages = (qzo_stage *)malloc(sizeof(qzo_stage) * max_stages);
    uint64_t ns = 0;
    if (qzo_plan(n, gates, ngates, c, m, stages, max_stages, &ns)) {
        free(stages);
        return -2;
    }
    const uint64_t nchunks = 1ull << (n - c), len = 1ull << c;
    const uint64_t tmpcap = qzo_payload_bound(len);
    uint8_t *tmp = (uint8_t *)malloc(tmpcap);
    chunk_t *chunks = (chunk_t *)calloc(nchunks, sizeof(chunk_t));
    qzo_amp *zeros = (qzo_amp *)calloc(len, sizeof(qzo_amp));

    /* init_basis_state, store.cpp:26-81 */
    uint32_t zcrc, bcrc;
    int64_t zlen = qzo_compress(zeros, len, eb, NULL, 0, tmp, tmpcap, &zcrc);
    uint8_t *zp = (uint8_t *)malloc(zlen);
    memcpy(zp, tmp, zlen);
    zeros[0].re = 1.0;
    int64_t blen = qzo_compress(zeros, len, eb, NULL, 0, tmp, tmpcap, &bcrc);
    if (eb > 0.0) {
        qzo_amp *r = (qzo_amp *)malloc(sizeof(qzo_amp) * len);
        qzo_decompress(tmp, blen, bcrc, len, r, NULL, 0);
        int exact = fabs(r[0].re - 1.0) <= 1e-12;
        for (uint64_t i = 0; exact && i < len; ++i)
            if (r[i].im != 0.0 || (i > 0 && r[i].re != 0.0)) exact = 0;
        free(r);
        if (!exact) {
            uint64_t fr[2] = {0, 1};
            blen = qzo_compress(zeros, len, eb, fr, len > 1 ? 2 : 1, tmp, tmpcap, &bcrc);
        }
    }
    zeros[0].re = 0.0;
    chunks[0].p = (uint8_t *)malloc(blen);
    memcpy(chunks[0].p, tmp, blen);
    chunks[0].len = (uint32_t)blen;
    chunks[0].crc = bcrc;
    for (uint64_t i = 1; i < nchunks; ++i) {
        chunks[i].p = (uint8_t *)malloc(zlen);
        memcpy(chunks[i].p, zp, zlen);
        chunks[i].len = (uint32_t)zlen;
        chunks[i].crc = zcrc;
    }
    uint64_t cur = 0;
    for (uint64_t i = 0; i < nchunks; ++i) cur += chunks[i].len + 48;
    uint64_t peak = cur;

    clock_gettime(CLOCK_MONOTONIC, &t0);
    int rc = 0;
    for (uint64_t si = 0; si < ns && rc == 0; ++si) {
        const qzo_stage *st = &stages[si];
        uint64_t members = 1ull << st->nhigh;
        uint64_t batches = 1ull << ((n - c) - st->nhigh);
        qzc_gate *rg = (qzc_gate *)malloc(sizeof(qzc_gate) * (st->ngates + 1));
        for (uint64_t k = 0; k < st->ngates; ++k) qzo_remap(st, c, &gates[st->first_gate + k], &rg[k]);
        uint64_t *mem = (uint64_t *)malloc(8 * members);
        qzo_amp *buf = (qzo_amp *)malloc(sizeof(qzo_amp) * members * len);
        for (uint64_t b = 0; b < batches && rc == 0; ++b) {
            qzo_batch_members(st, n, c, b, mem);
            for (uint64_t j = 0; j < members && rc == 0; ++j) {
                chunk_t *ch = &chunks[mem[j]];
                rc = qzo_decompress(ch->p, ch->len, ch->crc, len, buf + j * len, NULL, 0);
            }
            qzo_apply_gates(buf, members * len, rg, st->ngates);
            for (uint64_t j = 0; j < members && rc == 0; ++j) {
                chunk_t *ch = &chunks[mem[j]];
                uint64_t old = ch->len;
                rc = store_chunk(ch, buf + j * len, len, eb, tmp, tmpcap);
                cur = cur - old + ch->len;
                if (cur > peak) peak = cur;
            }
        }
        free(rg);
        free(mem);
        free(buf);
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);

    if (rc == 0) {
        /* report: digest (store.cpp:129-136), norm (pipeline.cpp:119-126) */
        uint64_t h = 0xcbf29ce484222325ULL, total = 0;
        double sum = 0.0, comp = 0.0;
        qzo_amp *vals = (qzo_amp *)malloc(sizeof(qzo_amp) * len);
        for (uint64_t i = 0; i < nchunks; ++i) {
            h = qzo_fnv1a64(chunks[i].p, chunks[i].len, h);
            if (payload_out) {
                if (total + chunks[i].len > cap) {
                    rc = -5;
                    break;
                }
                memcpy(payload_out + total, chunks[i].p, chunks[i].len);
            }
            if (sizes_out) sizes_out[i] = chunks[i].len;
            total += chunks[i].len;
            qzo_decompress(chunks[i].p, chunks[i].len, chunks[i].crc, len, vals, NULL, 0);
            for (uint64_t j = 0; j < len; ++j) {
                /* std::norm: re*re + im*im; KahanSum::add, util.hpp:57-66 */
                double x = vals[j].re * vals[j].re + vals[j].im * vals[j].im;
                double y = x - comp, t = sum + y;
                comp = (t - sum) - y;
                sum = t;
            }
        }
        free(vals);
        res->digest = h;
        res->norm = sum;
        res->current_bytes = cur;
        res->peak_bytes = peak;
        res->dense_bytes = (1ull << n) * 16;
        res->stages = ns;
        res->total_payload = total;
        res->seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    }
    for (uint64_t i = 0; i < nchunks; ++i) free(chunks[i].p);
    free(chunks);
    free(zp);
    free(zeros);
    free(tmp);
    free(stages);
    return rc;
}

/* Dense run with the kernel formula (simulate_dense semantics,
 * oracle.cpp:67-77). */
int qzo_dense(uint32_t n, const qzc_gate *gates, uint64_t ngates,
              qzo_amp *out) {
    uint64_t count = 1ull << n;
    memset(out, 0, sizeof(qzo_amp) * count);
    out[0].re = 1.0;
    return qzo_apply_gates(out, count, gates, ngates);
}

/* fidelity, oracle.cpp:79-93 (Kahan sums of <a|b>, |a|^2, |b|^2) */
typedef struct {
    double s, c;
} kahan;
static void kadd(kahan *k, double x) {
    double y = x - k->c, t = k->s + y;
    k->c = (t - k->s) - y;
    k->s = t;
}

double qzo_fidelity(const qzo_amp *a, const qzo_amp *b, uint64_t count) {
    kahan re = {0, 0}, im = {0, 0}, na = {0, 0}, nb = {0, 0};
    for (uint64_t i = 0; i < count; ++i) {
        qzo_amp ca = {a[i].re, -a[i].im};
        qzo_amp p = cmul(ca, b[i]);
        kadd(&re, p.re);
        kadd(&im, p.im);
        kadd(&na, a[i].re * a[i].re + a[i].im * a[i].im);
        kadd(&nb, b[i].re * b[i].re + b[i].im * b[i].im);
    }
    if (na.s == 0.0 || nb.s == 0.0) return 0.0;
    return (re.s * re.s + im.s * im.s) / (na.s * nb.s);
}

/* ----------------------------------------------------------- generators -- */

static void push(qzc_gate *out, uint64_t cap, uint64_t *k, uint32_t kind,
                 uint32_t q0, uint32_t q1, double p0) {
    if (*k < cap) {
        qzc_gate g;
        memset(&g, 0, sizeof g);
        g.kind = kind;
        g.nqubits = qzo_gate_arity(kind);
        g.qubits[0] = q0;
        g.qubits[1] = g.nqubits == 2 ? q1 : 0;
        g.params[0] = p0;
        out[*k] = g;
    }
    ++*k;
}

/* make_ghz, generators.cpp:21-28 */
uint64_t qzo_make_ghz(uint32_t n, qzc_gate *out, uint64_t cap) {
    uint64_t k = 0;
    push(out, cap, &k, QZC_H, 0, 0, 0.0);
    for (uint32_t t = 1; t < n; ++t) push(out, cap, &k, QZC_CX, 0, t, 0.0);
    return k;
}

/* make_qft with push_controlled_phase, generators.cpp:32-59 */
uint64_t qzo_make_qft(uint32_t n, qzc_gate *out, uint64_t cap) {
    uint64_t k = 0;
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t target = n - 1 - i;
        push(out, cap, &k, QZC_H, target, 0, 0.0);
        for (uint32_t j = 0; j < target; ++j) {
            uint32_t control = target - 1 - j;
            double lambda = M_PI / (double)(1ull << (j + 1));
            push(out, cap, &k, QZC_U1, control, 0, lambda / 2.0);
            push(out, cap, &k, QZC_CX, control, target, 0.0);
            push(out, cap, &k, QZC_U1, target, 0, -lambda / 2.0);
            push(out, cap, &k, QZC_CX, control, target, 0.0);
            push(out, cap, &k, QZC_U1, target, 0, lambda / 2.0);
        }
    }
    for (uint32_t i = 0; i < n / 2; ++i) push(out, cap, &k, QZC_SWAP, i, n - 1 - i, 0.0);
    return k;
}
