// qz_gates.cu — gate matrices and fused, bit-exact gate passes for sm_100a.
//
// Reference semantics: kernels.cpp:20-68 (apply_single_qubit /
// apply_two_qubit: dense 2x2 / 4x4 complex updates, left-to-right sums, no
// FMA) and gates.cpp:114-182 (gate_matrix).  Every amplitude receives exactly
// the reference's operation sequence for every gate, in circuit order, so the
// buffer is bit-identical to qzsim::apply_gates.
//
// B200 design: a stage's gates are grouped greedily (in order) into passes
// whose buffer bits fit a tile of 2^k amplitudes (k <= 12: 64 KB smem).  One
// pass = one HBM read + write of the buffer (32 B/amplitude); all gates of
// the pass run on the tile in shared memory.  Tiles always contain the low
// buffer bits 0..2 so every global access is a >= 128 B contiguous segment
// of 16 B double2 loads.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <complex>
#include <cstring>

#include "qz_gates.cuh"
#include "qz_jit.cuh"
#include "qz_kprof.cuh"

namespace qz {

// ----------------------------------------------------------- host matrices --

uint32_t gate_arity(uint32_t kind) {
    return (kind == QZC_CX || kind == QZC_CZ || kind == QZC_SWAP) ? 2u : 1u;
}

uint32_t gate_nparams(uint32_t kind) {
    switch (kind) {
    case QZC_RX: case QZC_RY: case QZC_RZ: case QZC_U1: return 1;
    case QZC_U2: return 2;
    case QZC_U3: return 3;
    default: return 0;
    }
}

namespace {

using cd = std::complex<double>;

// The unitaries are evaluated with the same std::complex expressions as the
// reference (gates.cpp:95-182) so the doubles handed to the device are
// bit-identical; tests/test_engine.py pins them against the golden fixture.
const cd kI{0.0, 1.0};

void put2(double2 *m, cd a, cd b, cd c, cd d) {
    cd v[4] = {a, b, c, d};
    for (int i = 0; i < 4; ++i) m[i] = make_double2(v[i].real(), v[i].imag());
}

void u3(double2 *m, double theta, double phi, double lambda) {
    const double ct = std::cos(theta / 2.0), st = std::sin(theta / 2.0);
    put2(m, ct, -std::exp(kI * lambda) * st, std::exp(kI * phi) * st,
         std::exp(kI * (phi + lambda)) * ct);
}

} // namespace

void gate_matrix_host(const qzc_gate &g, double2 *m, uint32_t *dim) {
    const double r2 = 0.7071067811865475244008443621048490;
    for (int i = 0; i < 16; ++i) m[i] = make_double2(0.0, 0.0);
    *dim = 2;
    const double *p = g.params;
    switch (g.kind) {
    case QZC_H: put2(m, r2, r2, r2, -r2); return;
    case QZC_X: put2(m, 0, 1, 1, 0); return;
    case QZC_Y: put2(m, 0, -kI, kI, 0); return;
    case QZC_Z: put2(m, 1, 0, 0, -1); return;
    case QZC_S: put2(m, 1, 0, 0, kI); return;
    case QZC_SDG: put2(m, 1, 0, 0, -kI); return;
    case QZC_T: put2(m, 1, 0, 0, std::exp(kI * (M_PI / 4.0))); return;
    case QZC_TDG: put2(m, 1, 0, 0, std::exp(-kI * (M_PI / 4.0))); return;
    case QZC_RX: {
        const double h = p[0] / 2.0;
        put2(m, std::cos(h), -kI * std::sin(h), -kI * std::sin(h), std::cos(h));
        return;
    }
    case QZC_RY: {
        const double h = p[0] / 2.0;
        put2(m, std::cos(h), -std::sin(h), std::sin(h), std::cos(h));
        return;
    }
    case QZC_RZ: {
        const double h = p[0] / 2.0;
        put2(m, std::exp(-kI * h), 0, 0, std::exp(kI * h));
        return;
    }
    case QZC_U1: put2(m, 1, 0, 0, std::exp(kI * p[0])); return;
    case QZC_U2: u3(m, M_PI / 2.0, p[0], p[1]); return;
    case QZC_U3: u3(m, p[0], p[1], p[2]); return;
    case QZC_CX:
        *dim = 4;
        m[0] = m[5] = m[11] = m[14] = make_double2(1.0, 0.0);
        return;
    case QZC_CZ:
        *dim = 4;
        m[0] = m[5] = m[10] = make_double2(1.0, 0.0);
        m[15] = make_double2(-1.0, 0.0);
        return;
    case QZC_SWAP:
        *dim = 4;
        m[0] = m[6] = m[9] = m[15] = make_double2(1.0, 0.0);
        return;
    default:
        throw Failure(QZC_EINVAL, "unknown gate kind " + std::to_string(g.kind));
    }
}


static uint32_t coef_kind(double2 v) {
    if (v.x == 0.0 && v.y == 0.0) return CK_ZERO;
    if (v.y == 0.0) {
        if (v.x == 1.0) return CK_ONE;
        if (v.x == -1.0) return CK_NEG;
        return CK_REAL;
    }
    if (v.x == 0.0) return CK_IMAG;
    return CK_CPLX;
}

DevGate make_dev_gate(const qzc_gate &g) {
    double2 m[16];
    uint32_t dim = 0;
    gate_matrix_host(g, m, &dim);
    return make_dev_gate_matrix(m, dim, g.qubits[0], dim == 4 ? g.qubits[1] : 0);
}

DevGate make_dev_gate_matrix(const double2 *mat, uint32_t dim, uint32_t b0, uint32_t b1) {
    if (dim != 2 && dim != 4) throw Failure(QZC_EINVAL, "gate matrix dim must be 2 or 4");
    DevGate d;
    std::memset(&d, 0, sizeof d);
    for (uint32_t e = 0; e < dim * dim; ++e) d.m[e] = mat[e];
    d.dim = dim;
    d.nq = dim == 2 ? 1 : 2;
    d.b0 = b0;
    d.b1 = d.nq == 2 ? b1 : 0;
    if (d.nq == 2 && b0 == b1) throw Failure(QZC_EINVAL, "duplicate qubit in two-qubit gate");
    for (uint32_t e = 0; e < dim * dim; ++e) {
        d.kinds |= uint64_t(coef_kind(d.m[e])) << (4 * e);
        d.sgn |= uint32_t(std::signbit(d.m[e].x)) << (2 * e);
        d.sgn |= uint32_t(std::signbit(d.m[e].y)) << (2 * e + 1);
    }
    auto is = [&](int e, double re) { return d.m[e].x == re && d.m[e].y == 0.0; };
    auto zero_except = [&](std::initializer_list<int> keep) {
        for (int e = 0; e < 16; ++e) {
            bool k = false;
            for (int x : keep) k |= x == e;
            if (!k && !(d.m[e].x == 0.0 && d.m[e].y == 0.0)) return false;
        }
        return true;
    };
    if (d.nq == 1) {
        const bool diag = d.m[1].x == 0.0 && d.m[1].y == 0.0 && d.m[2].x == 0.0 && d.m[2].y == 0.0;
        d.op = diag ? OP_DIAG : OP_GEN1;
    } else if (is(0, 1) && is(5, 1) && is(11, 1) && is(14, 1) && zero_except({0, 5, 11, 14})) {
        d.op = OP_CX;
    } else if (is(0, 1) && is(5, 1) && is(10, 1) && is(15, -1) && zero_except({0, 5, 10, 15})) {
        d.op = OP_CZ;
    } else if (is(0, 1) && is(6, 1) && is(9, 1) && is(15, 1) && zero_except({0, 6, 9, 15})) {
        d.op = OP_SWAP;
    } else {
        d.op = OP_GEN2;
    }
    return d;
}

// ------------------------------------------------------------- pass builder --

// Does an all-(+0) input produce all-(+0) outputs?  With every input +0 the
// product signs are the coefficient signs, so row r's real part is -0 iff
// every entry has (sign re, sign im) = (1, 0) and its imaginary part iff
// every entry has (1, 1) (IEEE: a sum of zeros is -0 only if all are -0).
static bool maps_pos_zero(const DevGate &g) {
    for (uint32_t r = 0; r < g.dim; ++r) {
        uint32_t nre = 1, nim = 1;
        for (uint32_t c = 0; c < g.dim; ++c) {
            const uint32_t e = r * g.dim + c;
            const uint32_t smr = (g.sgn >> (2 * e)) & 1, smi = (g.sgn >> (2 * e + 1)) & 1;
            nre &= smr & (smi ^ 1);
            nim &= smr & smi;
        }
        if (nre | nim) return false;
    }
    return true;
}

// Row r is "+0-safe" if it has a structural entry whose product can only be
// a +0 zero when its input has no -0 component: kind ONE, REAL or CPLX with
// a real part of sign 0 (then m_r*(+0) = +0 and x - (±0), x + (±0) keep +0).
// The row's exact value is then either nonzero (and equal to the shortcut
// sum) or +0, which the shortcut also yields.  Gates with a nonzero
// coefficient part below 2^-100 get no safe rows (products must not
// underflow for the argument to hold).
static uint32_t safe_rows(const DevGate &g) {
    for (uint32_t e = 0; e < g.dim * g.dim; ++e) {
        const double re = std::fabs(g.m[e].x), im = std::fabs(g.m[e].y);
        if ((re != 0.0 && re < 0x1p-100) || (im != 0.0 && im < 0x1p-100)) return 0;
    }
    uint32_t out = 0;
    for (uint32_t r = 0; r < g.dim; ++r)
        for (uint32_t c = 0; c < g.dim; ++c) {
            const uint32_t e = r * g.dim + c;
            const uint32_t kd = uint32_t(g.kinds >> (4 * e)) & 15;
            if ((kd == CK_ONE || kd == CK_REAL || kd == CK_CPLX) && !std::signbit(g.m[e].x))
                out |= 1u << r;
        }
    return out;
}

static bool is_signed_perm(const DevGate &g) {
    for (uint32_t r = 0; r < g.dim; ++r) {
        int nz = 0;
        for (uint32_t c = 0; c < g.dim; ++c) {
            const uint32_t kd = uint32_t(g.kinds >> (4 * (r * g.dim + c))) & 15;
            if (kd == CK_ZERO) continue;
            ++nz;
            if (kd != CK_ONE && kd != CK_NEG) return false;
        }
        if (nz != 1) return false;
    }
    return true;
}

// A diagonal unit: a run of gates whose net effect is diagonal (1q diagonal,
// CZ, or the CP5 / CXD runs) — only these may leave qubits outside a pass.
struct Unit {
    size_t first;
    uint32_t count;
    bool diag;
    uint64_t bits;   // buffer bits of all its gates
    bool swaps = false;   // a run of >= 2 pairwise disjoint SWAPs (PASS_SWAPS)
};

static uint64_t gate_bits(const DevGate &g) {
    uint64_t m = uint64_t(1) << g.b0;
    if (g.nq == 2) m |= uint64_t(1) << g.b1;
    return m;
}

static std::vector<Unit> make_units(const std::vector<DevGate> &G, bool relax) {
    std::vector<Unit> out;
    auto diag1 = [&](size_t i) {
        return G[i].nq == 1 && G[i].op == OP_DIAG && (uint32_t(G[i].kinds) & 15u) != CK_ZERO &&
               (uint32_t(G[i].kinds >> 12) & 15u) != CK_ZERO;
    };
    auto u1_on = [&](size_t i, uint32_t b) {
        return diag1(i) && G[i].b0 == b && (uint32_t(G[i].kinds) & 15u) == CK_ONE;
    };
    auto cx_on = [&](size_t i, uint32_t a, uint32_t b) {
        return G[i].nq == 2 && G[i].op == OP_CX && G[i].b0 == a && G[i].b1 == b;
    };
    for (size_t i = 0; i < G.size();) {
        Unit u{i, 1, false, gate_bits(G[i])};
        if (relax && G[i].nq == 2 && G[i].op == OP_SWAP) {
            uint64_t used = 0;
            size_t j = i;
            while (j < G.size() && G[j].nq == 2 && G[j].op == OP_SWAP && !(gate_bits(G[j]) & used)) {
                used |= gate_bits(G[j]);
                ++j;
            }
            if (j - i >= 2) {
                u = Unit{i, uint32_t(j - i), false, used};
                u.swaps = true;
                out.push_back(u);
                i = j;
                continue;
            }
        }
        if (relax) {
            if (i + 5 <= G.size() && u1_on(i, G[i].b0) && G[i + 1].nq == 2 &&
                cx_on(i + 1, G[i].b0, G[i + 1].b1) && u1_on(i + 2, G[i + 1].b1) &&
                cx_on(i + 3, G[i].b0, G[i + 1].b1) && u1_on(i + 4, G[i + 1].b1)) {
                u = Unit{i, 5, true, gate_bits(G[i + 1])};
            } else if (i + 3 <= G.size() && G[i].nq == 2 && G[i].op == OP_CX && diag1(i + 1) &&
                       G[i + 1].b0 == G[i].b1 && cx_on(i + 2, G[i].b0, G[i].b1)) {
                u = Unit{i, 3, true, gate_bits(G[i])};
            } else if (diag1(i) || (G[i].nq == 2 && G[i].op == OP_CZ)) {
                u.diag = true;
            }
        }
        out.push_back(u);
        i += u.count;
    }
    return out;
}

// +0-safe single step (see safe_rows): a structural coefficient of kind
// ONE / REAL / CPLX with a real part of sign 0, no part below 2^-100.
static bool safe_coef(uint32_t kind, double2 m) {
    const double re = std::fabs(m.x), im = std::fabs(m.y);
    if ((re != 0.0 && re < 0x1p-100) || (im != 0.0 && im < 0x1p-100)) return false;
    return (kind == CK_ONE || kind == CK_REAL || kind == CK_CPLX) && !std::signbit(m.x);
}

// Per-basis-state step chain of a diagonal unit: follow the basis state
// through the unit's gates (CX moves it, diagonal entries multiply it).
struct Step {
    uint32_t kind;
    double2 m;
};
static std::vector<Step> unit_chain(const std::vector<DevGate> &G, const Unit &u, uint64_t state) {
    std::vector<Step> ch;
    const uint64_t start = state;
    for (size_t i = u.first; i < u.first + u.count; ++i) {
        const DevGate &g = G[i];
        const uint32_t s0 = uint32_t(state >> g.b0) & 1;
        if (g.nq == 1) {
            const uint32_t e = s0 * 3;
            const uint32_t kd = uint32_t(g.kinds >> (4 * e)) & 15u;
            if (kd != CK_ONE) ch.push_back(Step{kd, g.m[e]});
        } else if (g.op == OP_CX) {
            if (s0) state ^= uint64_t(1) << g.b1;
        } else {   // CZ
            const uint32_t st = (s0 << 1) | (uint32_t(state >> g.b1) & 1);
            const uint32_t e = st * 5;
            const uint32_t kd = uint32_t(g.kinds >> (4 * e)) & 15u;
            if (kd != CK_ONE) ch.push_back(Step{kd, g.m[e]});
        }
    }
    if (state != start || ch.size() > 2) throw Failure(QZC_EDEVICE, "diagonal unit: bad chain");
    return ch;
}

// A unit may be relaxed only if every step of every basis state's chain is
// +0-safe: then a relaxed group needs no zero checks at all, and the only
// way it can fail is a block with a -0 / tiny component at group entry.
static bool unit_safe(const std::vector<DevGate> &G, const Unit &u) {
    uint32_t q[2], nq = 0;
    for (uint64_t r = u.bits; r; r &= r - 1) q[nq++] = (uint32_t)__builtin_ctzll(r);
    for (uint32_t st = 0; st < (1u << nq); ++st) {
        uint64_t state = 0;
        for (uint32_t i = 0; i < nq; ++i)
            if ((st >> i) & 1) state |= uint64_t(1) << q[i];
        for (const Step &s : unit_chain(G, u, state))
            if (!safe_coef(s.kind, s.m)) return false;
    }
    return true;
}

// Case id of a fast-list op: mirrors the device switch in fast_case().
static uint32_t case_id(const TileGate &t) {
    static const uint32_t gen_codes[14] = {3, 4, 5, 13, 14, 15, 21, 22, 23, 24, 31, 32, 33, 34};
    auto pair_idx = [](uint32_t a, uint32_t b) {
        static const uint32_t P[3][3] = {{99, 0, 1}, {2, 99, 3}, {4, 5, 99}};
        return P[a][b];
    };
    auto lohi_idx = [](uint32_t a, uint32_t b) {
        const uint32_t lo = std::min(a, b), hi = std::max(a, b);
        return lo == 0 ? (hi == 1 ? 0u : 1u) : 2u;
    };
    switch (t.op) {
    case OP_PDIAG: {
        const uint32_t R = t.nq ? t.r0 : 3;
        if (t.run) return t.pad4[0];
        return 4 + R * 2 + (t.pad2 == 8 ? 1 : 0);
    }
    case OP_DIAG: {
        const uint32_t vi = t.pad2 == 1 ? 0 : t.pad2 == 2 ? 1 : t.pad2 == 11 ? 2 : t.pad2 == 12 ? 3 : 4;
        return 12 + t.r0 * 5 + vi;
    }
    case OP_GEN1: {
        uint32_t gi = 14;
        for (uint32_t i = 0; i < 14; ++i)
            if (t.pad2 == gen_codes[i]) gi = i;
        return 27 + t.r0 * 15 + gi;
    }
    case OP_CP5: return 72 + pair_idx(t.r0, t.r1) * 2 + (t.pad2 == 6 ? 1 : 0);
    case OP_CXD: return 84 + pair_idx(t.r0, t.r1) * 2 + (t.pad2 == 7 ? 1 : 0);
    case OP_CX: return 96 + pair_idx(t.r0, t.r1);
    case OP_CZ: return 102 + lohi_idx(t.r0, t.r1);
    case OP_SWAP: return 105 + lohi_idx(t.r0, t.r1);
    default: return 1000;   // exact path only
    }
}

GatePlan build_passes(const std::vector<DevGate> &gates, uint32_t nbits, uint32_t kmax, bool fuse,
                      int relax_level, const Fresh *fresh, bool fuse_perm) {
    bool relax = relax_level > 0;
    GatePlan plan;
    const uint32_t k = std::min(kmax, nbits);
    // bits always in the tile (global segments of 2^low amplitudes)
    static const uint32_t kLow = getenv("QZ_TILE_LOW") ? uint32_t(atoi(getenv("QZ_TILE_LOW"))) : 3u;
    const uint32_t low = std::min<uint32_t>(kLow, k);
    const uint64_t low_mask = (uint64_t(1) << low) - 1;
    relax = relax && fuse && nbits > k;
    std::vector<Unit> units = make_units(gates, relax);
    // level 2: units with steps that are not +0-safe are relaxed too (their
    // steps are zero-checked and a zero raises the pass's replay flag) — a
    // win for zero-free states, a loss where lossy coding leaves exact zeros
    if (relax_level < 2)
        for (Unit &u : units)
            if (u.diag && !unit_safe(gates, u)) u.diag = false;
    std::vector<size_t> members;   // unit indices of the open pass
    // fresh state at the open pass's start / after its members so far: fresh
    // low bits are not forced into T (a tile over them would be mostly +0)
    Fresh fpass = fresh ? *fresh : Fresh{}, fcur = fpass;
    uint64_t tmask = low_mask & ~fpass.mask;
    // a pass "opens" at most kOpen of its start's fresh bits (non-diagonal
    // gates on them): the ops before an opening run on a mostly-(+0) tile
    // where few warps have work, so a long run of openings is split into
    // passes whose live tiles are dense
    static const uint32_t kOpen = getenv("QZ_FRESH_OPEN") ? uint32_t(atoi(getenv("QZ_FRESH_OPEN"))) : 3u;
    uint64_t opened = 0;
    // the bit permutation of a swap network unit (an involution)
    auto unit_perm = [&](const Unit &u, uint8_t *perm) {
        for (uint32_t b = 0; b < 48; ++b) perm[b] = uint8_t(b);
        for (size_t i = u.first; i < u.first + u.count; ++i) {
            perm[gates[i].b0] = uint8_t(gates[i].b1);
            perm[gates[i].b1] = uint8_t(gates[i].b0);
        }
    };
    // close the open pass; with `perm_unit`, try to fuse that swap network
    // into its store (returns whether it did)
    auto close = [&](const Unit *perm_unit = nullptr) -> bool {
        if (members.empty()) return false;
        uint8_t perm[48];
        bool fusing = false;
        if (perm_unit && nbits <= 48) {
            // the stored tile needs the images of the low bits (coalesced
            // output runs) among its bits
            unit_perm(*perm_unit, perm);
            uint64_t need_o = 0;
            for (uint32_t b = 0; b < low; ++b) need_o |= uint64_t(1) << perm[b];
            if ((uint32_t)__builtin_popcountll(tmask | need_o) <= k && low > 0) {
                tmask |= need_o;
                fusing = true;
            }
        }
        // a fused store: alternately the lowest non-fresh input bit (the live
        // elements' input runs) and the image of the next output bit (output
        // runs), while they are not fresh
        if (fusing) {
            // QZ_FUSE_PAD (tuning): 0 alternate (default), 1 input runs first, 2 output runs first
            static const int mode = getenv("QZ_FUSE_PAD") ? atoi(getenv("QZ_FUSE_PAD")) : 0;
            uint32_t ib = 0, ob = low;
            for (bool more = true; more && (uint32_t)__builtin_popcountll(tmask) < k;) {
                more = false;
                if (mode != 2) {
                    while (ib < nbits && (((tmask >> ib) & 1) || ((fpass.mask >> ib) & 1))) ++ib;
                    if (ib < nbits) {
                        tmask |= uint64_t(1) << ib;
                        more = true;
                        if (mode == 1) continue;
                    }
                }
                if ((uint32_t)__builtin_popcountll(tmask) >= k) break;
                while (ob < nbits && ((tmask >> perm[ob]) & 1)) ++ob;
                if (ob < nbits && !((fpass.mask >> perm[ob]) & 1)) {
                    tmask |= uint64_t(1) << perm[ob];
                    more = true;
                }
            }
        }
        // pad T to exactly k bits with the lowest free bits (longer contiguous
        // global segments), bits fresh at the pass's start last
        for (int round = 0; round < 2; ++round)
            for (uint32_t b = 0; b < nbits && (uint32_t)__builtin_popcountll(tmask) < k; ++b)
                if (round || !((fpass.mask >> b) & 1)) tmask |= uint64_t(1) << b;
        PassDesc pd;
        std::memset(&pd, 0, sizeof pd);
        pd.k = k;
        uint32_t lowbits = 0;
        while (lowbits < 64 && ((tmask >> lowbits) & 1)) ++lowbits;
        pd.lowbits = std::min(lowbits, k);
        pd.tmask = tmask;
        pd.zmask = fpass.mask & ~tmask;
        pd.zval = fpass.val & pd.zmask;
        pd.fmask = fpass.mask;
        pd.fval = fpass.val & fpass.mask;
        pd.first_gate = (uint32_t)plan.gates.size();
        pd.ngates = (uint32_t)members.size();
        pd.dg0 = (uint32_t)units[members.front()].first;
        pd.dg1 = (uint32_t)(units[members.back()].first + units[members.back()].count);
        pd.first_group = (uint32_t)plan.groups.size();
        auto local = [&](uint32_t b) {
            return (uint32_t)__builtin_popcountll(tmask & ((uint64_t(1) << b) - 1));
        };
        // register groups: consecutive gates whose tile bits fit kRegBits bits
        uint32_t gmask = 0;
        std::vector<int64_t> gentries;   // gate index, or -(unit + 1) for a relaxed unit
        std::vector<size_t> gmembers;    // the group's plain gates (exact list)
        auto close_group = [&]() {
            if (gentries.empty()) return;
            for (uint32_t b = 0; b < k && __builtin_popcount(gmask) < kRegBits; ++b) gmask |= 1u << b;
            auto is_reg = [&](uint32_t b) {   // buffer bit b is one of the group's register bits
                return ((tmask >> b) & 1) && ((gmask >> local(b)) & 1);
            };
            {
                // diagonal units entirely on register bits stay plain gates
                std::vector<int64_t> ents;
                for (int64_t e : gentries) {
                    if (e < 0) {
                        const Unit &u = units[size_t(-(e + 1))];
                        bool all_reg = true;
                        for (uint64_t r = u.bits; r; r &= r - 1) all_reg &= is_reg((uint32_t)__builtin_ctzll(r));
                        if (all_reg) {
                            for (size_t i = u.first; i < u.first + u.count; ++i) ents.push_back(int64_t(i));
                            continue;
                        }
                    }
                    ents.push_back(e);
                }
                gentries.swap(ents);
                gmembers.clear();
                for (int64_t e : gentries)
                    if (e >= 0) gmembers.push_back(size_t(e));
            }
            GroupDesc gd;
            std::memset(&gd, 0, sizeof gd);
            gd.generic = 0;
            gd.pz_stable = 1;
            gd.relaxed = 0;
            for (size_t gi : gmembers) gd.pz_stable &= maps_pos_zero(gates[gi]) ? 1u : 0u;
            int i = 0;
            for (uint32_t b = 0; b < k; ++b)
                if ((gmask >> b) & 1) gd.gbits[i++] = b;
            for (; i < 4; ++i) gd.gbits[i] = 0;   // unused slots
            gd.first_gate = (uint32_t)plan.gates.size();
            gd.ngates = (uint32_t)gmembers.size();
            auto reg = [&](uint32_t lb) {
                return (uint32_t)__builtin_popcount(gmask & ((1u << lb) - 1));
            };
            for (size_t gi : gmembers) {
                const DevGate &g = gates[gi];
                TileGate t;
                std::memset(&t, 0, sizeof t);
                t.nq = g.nq;
                t.t0 = local(g.b0);
                t.t1 = g.nq == 2 ? local(g.b1) : 0;
                t.r0 = reg(t.t0);
                t.r1 = g.nq == 2 ? reg(t.t1) : 0;
                t.kinds = g.kinds;
                t.sgn = g.sgn;
                t.zm = 0;
                t.smask = 0;
                for (uint32_t e = 0; e < g.dim * g.dim; ++e) {
                    t.zm |= uint32_t(g.m[e].x == 0.0) << e;
                    t.zm |= uint32_t(g.m[e].y == 0.0) << (16 + e);
                    t.smask |= uint32_t(std::signbit(g.m[e].x)) << e;
                    t.smask |= uint32_t(std::signbit(g.m[e].y)) << (16 + e);
                }
                t.op = g.op;
                t.srow = safe_rows(g);
                t.pad2 = 0;
                t.pad = 0;   // bit r: row r maps all-(+0) inputs to (+0, +0)
                for (uint32_t r = 0; r < g.dim; ++r) {
                    uint32_t nre = 1, nim = 1;
                    for (uint32_t c = 0; c < g.dim; ++c) {
                        const uint32_t e = r * g.dim + c;
                        const uint32_t smr = (g.sgn >> (2 * e)) & 1, smi = (g.sgn >> (2 * e + 1)) & 1;
                        nre &= smr & (smi ^ 1);
                        nim &= smr & smi;
                    }
                    if (!(nre | nim)) t.pad |= 1u << r;
                }
                t.cls = TG_GEN;
                {
                    const uint32_t dim = g.dim;
                    bool perm = true, diag = g.nq == 1;
                    uint32_t code = 0;
                    for (uint32_t r = 0; r < dim && perm; ++r) {
                        int nz = 0;
                        for (uint32_t c = 0; c < dim; ++c) {
                            const uint32_t kd = uint32_t(g.kinds >> (4 * (r * dim + c))) & 15;
                            if (kd == CK_ZERO) continue;
                            ++nz;
                            if (kd != CK_ONE && kd != CK_NEG) perm = false;
                            code |= (c | (kd == CK_NEG ? 4u : 0u)) << (3 * r);
                            if (c != r) diag = false;
                        }
                        if (nz != 1) perm = false;
                    }
                    if (g.nq == 1 && !(uint32_t(g.kinds >> 4) & 15) && !(uint32_t(g.kinds >> 8) & 15))
                        diag = true;
                    else if (g.nq == 1)
                        diag = false;
                    if (perm) {
                        t.cls = TG_PERM;
                        t.perm = code;
                    } else if (diag) {
                        t.cls = TG_DIAG;
                    }
                }
                std::memcpy(t.m, g.m, sizeof t.m);
                plan.gates.push_back(t);
            }
            // fast list: the same gates with macro-able runs folded, relaxed
            // units in their place in the order
            gd.first_fast = (uint32_t)plan.gates.size();
            uint32_t exact_pos = gd.first_gate;
            for (size_t ei = 0; ei < gentries.size();) {
                if (gentries[ei] < 0) {
                    const Unit &u = units[size_t(-(gentries[ei] + 1))];
                    TileGate t;
                    std::memset(&t, 0, sizeof t);
                    t.op = OP_PDIAG;
                    uint64_t in = 0;
                    for (uint64_t r = u.bits; r; r &= r - 1)
                        if (is_reg((uint32_t)__builtin_ctzll(r))) in |= r & (0 - r);
                    const uint64_t outb = u.bits & ~in;
                    t.nq = __builtin_popcountll(in);   // 0 or 1 register bits
                    if (t.nq) {
                        const uint32_t b = (uint32_t)__builtin_ctzll(in);
                        t.r0 = reg(local(b));
                        t.t0 = b;
                    }
                    t.ob0 = (uint32_t)__builtin_ctzll(outb);
                    const uint64_t rest = outb & (outb - 1);
                    t.ob1 = rest ? (uint32_t)__builtin_ctzll(rest) : 63u;
                    bool spec = true, pz = true;
                    for (uint32_t var = 0; var < 4; ++var) {
                        if (!rest && var >= 2) break;
                        for (uint32_t st = 0; st < (t.nq ? 2u : 1u); ++st) {
                            uint64_t state = 0;
                            if (var & 1) state |= uint64_t(1) << t.ob0;
                            if (var & 2) state |= uint64_t(1) << t.ob1;
                            if (t.nq && st) state |= in;
                            const std::vector<Step> ch = unit_chain(gates, u, state);
                            for (size_t j = 0; j < ch.size(); ++j) {
                                const uint32_t e = 4 * var + 2 * st + (uint32_t)j;
                                t.kinds |= uint64_t(ch[j].kind) << (4 * e);
                                t.m[e] = ch[j].m;
                                const bool sf = safe_coef(ch[j].kind, ch[j].m);
                                t.srow |= uint32_t(sf) << e;
                                spec &= sf && ch[j].kind == CK_CPLX;
                                pz &= sf;
                            }
                        }
                    }
                    t.pad2 = spec ? 8u : 0u;
                    for (uint32_t e = 0; e < 16; ++e)
                        if ((t.kinds >> (4 * e)) & 15u) t.steps |= 1u << e;
                    gd.pz_stable &= pz ? 1u : 0u;
                    gd.unsafe |= pz ? 0u : 1u;
                    gd.relaxed = 1;
                    plan.gates.push_back(t);
                    ++ei;
                    continue;
                }
                size_t ej = ei;
                while (ej < gentries.size() && gentries[ej] >= 0) ++ej;
                const uint32_t e0 = exact_pos, e1 = exact_pos + uint32_t(ej - ei);
                exact_pos = e1;
                ei = ej;
                for (uint32_t i = e0; i < e1;) {
                    const TileGate *G = &plan.gates[0];
                    auto u1_on = [&](uint32_t k, uint32_t r) {
                        return G[k].nq == 1 && G[k].op == OP_DIAG && G[k].r0 == r &&
                               (uint32_t(G[k].kinds) & 15u) == CK_ONE;
                    };
                    auto cx_on = [&](uint32_t k, uint32_t a, uint32_t b) {
                        return G[k].nq == 2 && G[k].op == OP_CX && G[k].r0 == a && G[k].r1 == b;
                    };
                    if (i + 5 <= e1 && u1_on(i, G[i].r0) && G[i + 1].nq == 2 &&
                        cx_on(i + 1, G[i].r0, G[i + 1].r1) && u1_on(i + 2, G[i + 1].r1) &&
                        cx_on(i + 3, G[i].r0, G[i + 1].r1) && u1_on(i + 4, G[i + 1].r1)) {
                        TileGate mg = G[i + 1];
                        mg.op = OP_CP5;
                        mg.m[0] = G[i].m[3];
                        mg.m[1] = G[i + 2].m[3];
                        mg.m[2] = G[i + 4].m[3];
                        mg.kinds = (uint64_t(G[i].kinds >> 12) & 15) | ((uint64_t(G[i + 2].kinds >> 12) & 15) << 4) |
                                   ((uint64_t(G[i + 4].kinds >> 12) & 15) << 8);
                        mg.srow = ((G[i].srow >> 1) & 1) | (((G[i + 2].srow >> 1) & 1) << 1) |
                                  (((G[i + 4].srow >> 1) & 1) << 2);
                        plan.gates.push_back(mg);
                        i += 5;
                        continue;
                    }
                    if (i + 3 <= e1 && G[i].nq == 2 && G[i].op == OP_CX && G[i + 1].nq == 1 &&
                        G[i + 1].op == OP_DIAG && G[i + 1].r0 == G[i].r1 && cx_on(i + 2, G[i].r0, G[i].r1)) {
                        TileGate mg = G[i];
                        mg.op = OP_CXD;
                        mg.m[0] = G[i + 1].m[0];
                        mg.m[1] = G[i + 1].m[3];
                        mg.kinds = (uint64_t(G[i + 1].kinds) & 15) | ((uint64_t(G[i + 1].kinds >> 12) & 15) << 4);
                        mg.srow = G[i + 1].srow & 3;
                        plan.gates.push_back(mg);
                        i += 3;
                        continue;
                    }
                    const TileGate same = plan.gates[i];
                    plan.gates.push_back(same);
                    ++i;
                }
            }
            for (size_t k = gd.first_fast; k < plan.gates.size(); ++k) {
                TileGate &t = plan.gates[k];
                if (t.op == OP_PDIAG) continue;
                const uint32_t kd = uint32_t(t.kinds);
                auto K = [&](int e) { return (kd >> (4 * e)) & 15u; };
                t.pad2 = 0;
                // 1-5: compile-time kinds, rows +0-safe (no checks);
                // 11-15: the same kinds with run-time row checks
                const uint32_t chk = (t.srow & 3) == 3 ? 0u : 10u;
                if (t.op == OP_DIAG) {
                    if (K(0) == CK_ONE && K(3) == CK_CPLX) t.pad2 = 1 + chk;
                    else if (K(0) == CK_CPLX && K(3) == CK_CPLX) t.pad2 = 2 + chk;
                } else if (t.op == OP_GEN1) {
                    if (K(0) == CK_REAL && K(1) == CK_IMAG && K(2) == CK_IMAG && K(3) == CK_REAL) t.pad2 = 3 + chk;
                    else if (K(0) == CK_REAL && K(1) == CK_REAL && K(2) == CK_REAL && K(3) == CK_REAL) t.pad2 = 4 + chk;
                    else if (K(0) == CK_CPLX && K(1) == CK_CPLX && K(2) == CK_CPLX && K(3) == CK_CPLX) t.pad2 = 5 + chk;
                    // X, Y, U3 / U2 shapes
                    else if (K(0) == CK_ZERO && K(1) == CK_ONE && K(2) == CK_ONE && K(3) == CK_ZERO) t.pad2 = 21 + chk;
                    else if (K(0) == CK_ZERO && K(1) == CK_IMAG && K(2) == CK_IMAG && K(3) == CK_ZERO) t.pad2 = 22 + chk;
                    else if (K(0) == CK_REAL && K(1) == CK_CPLX && K(2) == CK_CPLX && K(3) == CK_CPLX) t.pad2 = 23 + chk;
                    else if (K(0) == CK_REAL && K(1) == CK_CPLX && K(2) == CK_REAL && K(3) == CK_CPLX) t.pad2 = 24 + chk;
                } else if (t.op == OP_CP5 && (t.srow & 7) == 7 && K(0) == CK_CPLX && K(1) == CK_CPLX &&
                           K(2) == CK_CPLX) {
                    t.pad2 = 6;
                } else if (t.op == OP_CXD && (t.srow & 3) == 3 && K(0) == CK_CPLX && K(1) == CK_CPLX) {
                    t.pad2 = 7;
                }
            }
            // runs of specialised OP_PDIAG ops whose register selectors are
            // "uniform" or one common bit R (the kernel's tight loop); the
            // run's selector is kept in pad4[0]
            for (size_t q = plan.gates.size(); q-- > gd.first_fast;) {
                TileGate &t = plan.gates[q];
                t.run = 0;
                if (t.op == OP_PDIAG && t.pad2 == 8) {
                    const uint32_t rs = t.nq ? t.r0 : kRegBits;
                    t.run = 1;
                    t.pad4[0] = rs;
                    if (q + 1 < plan.gates.size()) {
                        const TileGate &u = plan.gates[q + 1];
                        const uint32_t ru = u.pad4[0];
                        if (u.run && (rs == kRegBits || ru == kRegBits || rs == ru)) {
                            t.run += u.run;
                            t.pad4[0] = rs == kRegBits ? ru : rs;
                        }
                    }
                }
            }
            for (size_t q = gd.first_fast; q < plan.gates.size(); ++q) plan.gates[q].cid = case_id(plan.gates[q]);
            plan.groups.push_back(gd);
            plan.groups.back().nfast = (uint32_t)plan.gates.size() - gd.first_fast;
            gmembers.clear();
            gentries.clear();
            gmask = 0;
        };
        for (size_t ui : members) {
            const Unit &u = units[ui];
            if (relax && u.diag) {
                // diagonal unit: needs no register bit; at close_group its
                // qubits outside the group's register bits become per-thread
                // constants (OP_PDIAG), unless all of them are register bits
                gentries.push_back(-int64_t(ui) - 1);
                continue;
            }
            for (size_t i = u.first; i < u.first + u.count; ++i) {
                const DevGate &g = gates[i];
                uint32_t need = 1u << local(g.b0);
                if (g.nq == 2) need |= 1u << local(g.b1);
                const bool generic = g.nq == 2 && !is_signed_perm(g);
                if (generic || __builtin_popcount(gmask | need) > kRegBits || k <= (uint32_t)kRegBits)
                    close_group();
                gmask |= need;
                gmembers.push_back(i);
                gentries.push_back(int64_t(i));
                if (generic) {
                    close_group();
                    plan.groups.back().generic = 1;
                }
            }
        }
        close_group();
        pd.ngroups = (uint32_t)plan.groups.size() - pd.first_group;
        pd.pz_stable = 1;
        for (uint32_t gi = pd.first_group; gi < pd.first_group + pd.ngroups; ++gi) {
            pd.pz_stable &= plan.groups[gi].pz_stable;
            if (plan.groups[gi].relaxed) pd.relaxed = std::max<uint32_t>(pd.relaxed, plan.groups[gi].unsafe ? 2u : 1u);
        }
        // (out-of-place checked passes keep their own replay scheme)
        const bool fused = fusing && pd.relaxed != 2;
        if (fused) {
            pd.permute = 1;
            std::memcpy(pd.perm, perm, sizeof perm);
            pd.dg1 = (uint32_t)(perm_unit->first + perm_unit->count);
        }
        plan.passes.push_back(pd);
        members.clear();
        fpass = fcur;
        tmask = low_mask & ~fpass.mask;
        opened = 0;
        return fused;
    };
    auto advance = [&](const Unit &u) {   // fcur through the unit's gates
        for (size_t i = u.first; i < u.first + u.count && fcur.mask; ++i) fcur = fresh_after_gate(fcur, gates[i]);
    };
    for (size_t ui = 0; ui < units.size(); ++ui) {
        const Unit &u = units[ui];
        if (u.bits >> nbits) throw Failure(QZC_EDEVICE, "gate bit outside buffer");
        if (u.swaps) {
            // fused into the open pass's store, or one in-place
            // bit-permutation pass of its own
            if (close(fuse_perm ? &u : nullptr)) {
                advance(u);
                fpass = fcur;
                tmask = low_mask & ~fpass.mask;
                continue;
            }
            PassDesc pd;
            std::memset(&pd, 0, sizeof pd);
            pd.kind = PASS_SWAPS;
            pd.first_gate = (uint32_t)u.first;
            pd.ngates = u.count;
            pd.dg0 = (uint32_t)u.first;
            pd.dg1 = (uint32_t)(u.first + u.count);
            pd.relaxed = 1;
            for (uint32_t b = 0; b < 48; ++b) pd.perm[b] = uint8_t(b);
            for (size_t i = u.first; i < u.first + u.count; ++i) {
                pd.perm[gates[i].b0] = uint8_t(gates[i].b1);
                pd.perm[gates[i].b1] = uint8_t(gates[i].b0);
            }
            pd.pz_stable = 1;
            plan.passes.push_back(pd);
            advance(u);
            fpass = fcur;
            tmask = low_mask & ~fpass.mask;
            opened = 0;
            continue;
        }
        const uint64_t need = u.diag ? 0 : u.bits;
        const uint64_t merged = tmask | need;
        if (!fuse || (uint32_t)__builtin_popcountll(merged) > k ||
            (opened && (uint32_t)__builtin_popcountll(opened | (need & fpass.mask)) > kOpen))
            close();
        tmask |= need;
        opened |= need & fpass.mask;
        members.push_back(ui);
        advance(u);
    }
    close();
    if (getenv("QZ_TRACE") && getenv("QZ_TRACE")[0] == '2') {
        for (const PassDesc &pd : plan.passes) {
            uint32_t nf = 0, npd = 0, nrel = 0, nuns = 0;
            for (uint32_t gi = pd.first_group; gi < pd.first_group + pd.ngroups; ++gi) {
                nf += plan.groups[gi].nfast;
                nrel += plan.groups[gi].relaxed;
                nuns += plan.groups[gi].unsafe;
                for (uint32_t q = 0; q < plan.groups[gi].nfast; ++q)
                    npd += plan.gates[plan.groups[gi].first_fast + q].op == OP_PDIAG;
            }
            fprintf(stderr, "qz plan: kind %u tmask %#llx groups %u (relaxed %u, unsafe %u) fast ops %u pdiag %u "
                            "gates %u pass relaxed %u zmask %#llx fmask %#llx permute %u\n",
                    pd.kind, (unsigned long long)pd.tmask, pd.ngroups, nrel, nuns, nf, npd, pd.ngates, pd.relaxed,
                    (unsigned long long)pd.zmask, (unsigned long long)pd.fmask, pd.permute);
        }
    }
    return plan;
}

std::vector<PassDesc> launch_passes(const GatePlan &plan) {
    std::vector<PassDesc> out = plan.passes;
    // kernel case set per pass: the narrow one when every fast-list entry of
    // every group is in it (and no group needs the shared-memory generic path)
    static const bool narrow_off = getenv("QZ_NO_NARROW") != nullptr;
    static const bool wmap_off = getenv("QZ_NO_WMAP") != nullptr;
    static const bool direct_off = getenv("QZ_NO_DIRECT") != nullptr;
    for (PassDesc &pd : out) {
        pd.wmap = wmap_off ? 0u : 1u;
        pd.direct = !direct_off && pd.kind == PASS_TILE && pd.ngroups == 1 && !plan.groups[pd.first_group].generic &&
                    !pd.permute && pd.lowbits >= 5 && pd.k >= (uint32_t)kRegBits + 1 ? 1u : 0u;
        pd.variant = kPassAll;
        for (int S : {kPassDiagH, kPassGen}) {
            bool narrow = !narrow_off && pd.kind != PASS_SWAPS;
            for (uint32_t gi = 0; narrow && gi < pd.ngroups; ++gi) {
                const GroupDesc &G = plan.groups[pd.first_group + gi];
                if (G.generic) narrow = false;
                for (uint32_t q = 0; narrow && q < G.nfast; ++q)
                    narrow = case_on(S, plan.gates[G.first_fast + q].cid);
            }
            if (narrow) {
                pd.variant = uint32_t(S);
                break;
            }
        }
        static const bool dump = getenv("QZ_CID_DUMP") != nullptr;
        if (dump && pd.kind != PASS_SWAPS) {
            uint32_t hist[128] = {0};
            for (uint32_t gi = 0; gi < pd.ngroups; ++gi) {
                const GroupDesc &G = plan.groups[pd.first_group + gi];
                for (uint32_t q = 0; q < G.nfast; ++q) ++hist[plan.gates[G.first_fast + q].cid & 127];
            }
            fprintf(stderr, "qz pass k=%u groups=%u variant=%u cids:", pd.k, pd.ngroups, pd.variant);
            for (int c = 0; c < 128; ++c)
                if (hist[c]) fprintf(stderr, " %d:%u", c, hist[c]);
            fprintf(stderr, "\n");
        }
    }
    return out;
}

bool gate_diagonal(const DevGate &g) {
    for (uint32_t r = 0; r < g.dim; ++r)
        for (uint32_t c = 0; c < g.dim; ++c)
            if (r != c && ((g.kinds >> (4 * (r * g.dim + c))) & 15u) != CK_ZERO) return false;
    return true;
}

bool gate_keeps_pos_zero(const DevGate &g) { return maps_pos_zero(g); }

Fresh fresh_gate(Fresh f, uint32_t op, uint32_t nq, uint32_t b0, uint32_t b1, uint64_t kinds, bool diagonal) {
    auto bit = [](uint64_t x, uint32_t b) { return (x >> b) & 1; };
    const uint64_t m0 = uint64_t(1) << b0, m1 = nq == 2 ? uint64_t(1) << b1 : 0;
    if (diagonal) return f;
    if (nq == 2 && op == OP_CX) {
        // basis states to basis states: a fresh control keeps the target's
        // freshness (and flips its value when 1); a superposed one ends it
        if (bit(f.mask, b0)) {
            if (bit(f.val, b0)) f.val ^= m1;
        } else {
            f.mask &= ~m1;
        }
    } else if (nq == 2 && op == OP_SWAP) {
        const uint64_t a = bit(f.mask, b0), b = bit(f.mask, b1), va = bit(f.val, b0), vb = bit(f.val, b1);
        f.mask = (f.mask & ~(m0 | m1)) | (b << b0) | (a << b1);
        f.val = (f.val & ~(m0 | m1)) | (vb << b0) | (va << b1);
    } else if (nq == 1 && op == OP_GEN1 && (kinds & 0xFFFF) == ((uint64_t(CK_ONE) << 4) | (uint64_t(CK_ONE) << 8))) {
        f.val ^= m0;   // X
    } else {
        f.mask &= ~(m0 | m1);
    }
    f.val &= f.mask;
    return f;
}

Fresh fresh_after_gate(Fresh f, const DevGate &g) {
    if (!f.mask) return f;
    // amplitudes on the +0 side of a fresh qubit the gate does not touch
    // form all-(+0) orbits: they stay +0 iff the gate maps all-(+0) to +0
    if (!maps_pos_zero(g)) return Fresh{};
    const uint64_t gm = (uint64_t(1) << g.b0) | (g.nq == 2 ? uint64_t(1) << g.b1 : 0);
    if (!(f.mask & gm)) return f;
    if (gate_diagonal(g)) {
        // a +0-side row (a touched fresh bit on its +0 side) sums m_rr * (+0)
        // with structural-zero products of live amplitudes (zeros of any
        // sign): +0 only when m_rr is sign-safe; else those bits are lost
        for (uint32_t r = 0; r < g.dim; ++r) {
            const uint32_t v0 = g.nq == 2 ? (r >> 1) & 1 : r & 1, v1 = r & 1;
            const bool zside = (((f.mask >> g.b0) & 1) && v0 != ((f.val >> g.b0) & 1)) ||
                               (g.nq == 2 && ((f.mask >> g.b1) & 1) && v1 != ((f.val >> g.b1) & 1));
            const uint32_t e = r * g.dim + r;
            if (zside && !safe_coef(uint32_t(g.kinds >> (4 * e)) & 15u, g.m[e])) {
                f.mask &= ~gm;
                break;
            }
        }
        f.val &= f.mask;
        return f;
    }
    // X / CX / SWAP: the +0 side maps through a 1 * (+0) term (stays +0)
    return fresh_gate(f, g.op, g.nq, g.b0, g.b1, g.kinds, false);
}

Fresh fresh_after(const std::vector<DevGate> &dg, size_t g0, size_t g1, Fresh f) {
    for (size_t i = g0; i < g1 && f.mask; ++i) f = fresh_after_gate(f, dg[i]);
    return f;
}

void upload_plan(const GatePlan &plan, DevPlan &out, cudaStream_t s, uint32_t jit_bits,
                 const std::vector<Fresh> &fresh) {
    out.ngates = plan.gates.size();
    out.ngroups = plan.groups.size();
    out.host_passes = launch_passes(plan);
    out.jit.assign(out.host_passes.size(), nullptr);
    if (jit_bits)
        for (size_t p = 0; p < out.host_passes.size(); ++p)
            out.jit[p] = jit_request(plan, out.host_passes[p], jit_bits, p < fresh.size() ? fresh[p] : Fresh{});
    out.relaxed = false;
    for (const PassDesc &pd : plan.passes) out.relaxed |= pd.relaxed != 0 || pd.permute != 0;   // (run_relaxed)
    out.replay_range.clear();
    if (out.ngates > out.cap_gates) {
        if (out.gates) QZ_CUDA(cudaFree(out.gates));
        out.cap_gates = std::max<size_t>(out.ngates * 2, 256);
        QZ_CUDA(cudaMalloc(&out.gates, sizeof(TileGate) * out.cap_gates));
    }
    if (out.ngroups > out.cap_groups) {
        if (out.groups) QZ_CUDA(cudaFree(out.groups));
        out.cap_groups = std::max<size_t>(out.ngroups * 2, 64);
        QZ_CUDA(cudaMalloc(&out.groups, sizeof(GroupDesc) * out.cap_groups));
    }
    if (out.ngates)
        QZ_CUDA(cudaMemcpyAsync(out.gates, plan.gates.data(), sizeof(TileGate) * out.ngates,
                                cudaMemcpyHostToDevice, s));
    if (out.ngroups)
        QZ_CUDA(cudaMemcpyAsync(out.groups, plan.groups.data(), sizeof(GroupDesc) * out.ngroups,
                                cudaMemcpyHostToDevice, s));
    // (pageable source: staged by the driver before the call returns)
}

void free_plan(DevPlan &p) {
    if (p.gates) cudaFree(p.gates);
    if (p.groups) cudaFree(p.groups);
    p.gates = nullptr;
    p.groups = nullptr;
    p.ngates = p.ngroups = 0;
    p.cap_gates = p.cap_groups = 0;
    p.host_passes.clear();
    p.jit.clear();
    p.relaxed = false;
}

#include "qz_gates_dev.cuh"

// QZ_DEBUG_COUNTERS=1: count tile skips and per-group paths
// [0] tiles skipped, [1] +0 groups skipped, [2] sign-mask, [3] fast,
// [4] exact (zero at entry), [5] fast then exact
unsigned long long *debug_counters() {
    static unsigned long long *ptr = nullptr;
    static bool init = false;
    if (!init) {
        init = true;
        const char *e = getenv("QZ_DEBUG_COUNTERS");
        if (e && *e == '1') {
            QZ_CUDA(cudaMalloc(&ptr, 8 * 16));
            QZ_CUDA(cudaMemset(ptr, 0, 8 * 16));
        }
    }
    return ptr;
}

void dump_debug_counters() {
    unsigned long long *p = debug_counters();
    if (!p) return;
    unsigned long long h[16];
    QZ_CUDA(cudaMemcpy(h, p, sizeof h, cudaMemcpyDeviceToHost));
    if (h[8] | h[9] | h[15])
        fprintf(stderr, "qz group clocks (CTA-thread-0 cycles): load+census=%llu g0=%llu g1=%llu g2=%llu g3=%llu "
                        "g4=%llu g5+=%llu store=%llu\n", h[8], h[9], h[10], h[11], h[12], h[13], h[14], h[15]);
    fprintf(stderr, "qz counters: tiles_skipped=%llu grp_pz_skip=%llu grp_mask=%llu grp_fast=%llu "
                    "grp_exact=%llu grp_fast_then_exact=%llu zero_filled=%llu loaded=%llu\n",
            h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    QZ_CUDA(cudaMemset(p, 0, sizeof h));
}

namespace {

// Count a replayed pass and clear the flag for the next relaxed pass.
__global__ void k_flag_done(uint32_t *flag, uint64_t *count) {
    if (count) *count += *flag;
    *flag = 0;
}

void set_attrs() {
    static bool attr_set = false;
    if (!attr_set) {
        QZ_CUDA(cudaFuncSetAttribute(tile_pass_reg<kPassAll>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
        QZ_CUDA(cudaFuncSetAttribute(tile_pass_reg<kPassDiagH>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
        QZ_CUDA(cudaFuncSetAttribute(tile_pass_reg<kPassGen>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
        attr_set = true;
    }
}

// Chunks moved (swap network, permuted store): the zero map no longer
// describes the slots.
void reset_nz(NzMap nz, uint32_t nbits, cudaStream_t s) {
    if (nz.slot && nbits > nz.cbits) {
        const size_t ns = size_t(1) << (nbits - nz.cbits);
        QZ_CUDA(cudaMemsetAsync(nz.slot, 1, 4 * ns, s));
        QZ_CUDA(cudaMemsetAsync(nz.slot + ns, 0, 4, s));
    }
}

// QZ_DEBUG_COUNTERS=1 QZ_COUNTERS_PER_PASS=1: counters after every pass (synchronous)
void dump_pass_counters(const PassDesc &pd, uint32_t tag, const uint32_t *cond, cudaStream_t s) {
    static const bool per_pass = getenv("QZ_COUNTERS_PER_PASS") != nullptr;
    if (!per_pass || !debug_counters()) return;
    QZ_CUDA(cudaStreamSynchronize(s));
    fprintf(stderr, "qz pass %u (k=%u groups=%u%s):\n", tag, pd.k, pd.ngroups, cond ? ", replay" : "");
    dump_debug_counters();
}

void launch_pass(const DevPlan &plan, const PassDesc &pd, const double2 *src, double2 *dst,
                 uint32_t nbits, cudaStream_t s, uint32_t *flag, const uint32_t *cond, NzMap nz,
                 uint32_t tag) {
    // replay launches (cond != nullptr) are device-side no-ops unless flagged:
    // they are not timed as passes
    static const char *const kName[3] = {"tile_pass_reg<All>", "tile_pass_reg<DiagH>", "tile_pass_reg<Gen>"};
    static const char *const kJitName[3] = {"tile_pass_jit<All>", "tile_pass_jit<DiagH>", "tile_pass_jit<Gen>"};
    // `tag` is the pass's index in `plan`
    JitPass *jit = tag < plan.jit.size() && plan.jit[tag] && jit_ready(*plan.jit[tag]) ? plan.jit[tag].get() : nullptr;
    // algorithmic bytes: 16 B per element loaded (live tiles, minus the
    // statically-(+0) elements a pass zero-fills) + 16 B per element stored;
    // replays are no-ops unless flagged
    double pbytes = 32.0 * double(uint64_t(1) << nbits);
    if (pd.kind == PASS_TILE && pd.k >= (uint32_t)kRegBits + 1) {
        const double live = double(uint64_t(1) << nbits) /
                            ((pd.zmask && pd.pz_stable && src == dst) ? double(uint64_t(1) << __builtin_popcountll(pd.zmask)) : 1.0);
        pbytes = 16.0 * live * (1.0 + 1.0 / double(uint64_t(1) << __builtin_popcountll(pd.fmask & pd.tmask)));
    }
    KProfScope prof(s, cond ? "replay_pass" : pd.kind == PASS_SWAPS ? "tile_swaps" : (jit ? kJitName : kName)[pd.variant % 3],
                    tag, cond ? 0.0 : pbytes);
    if (pd.kind == PASS_SWAPS) {
        const uint64_t tiles = uint64_t(1) << (nbits > 2 * kSwapLow ? nbits - 2 * kSwapLow : 0);
        const uint64_t grid = std::min<uint64_t>(std::max<uint64_t>(tiles, 1), uint64_t(kNumSMs) * 8);
        tile_swaps<<<(unsigned)grid, 256, 0, s>>>(src, dst, nbits, pd, flag, cond);
        reset_nz(nz, nbits, s);
    } else if (pd.k < (uint32_t)kRegBits + 1) {
        // tile == whole buffer (nbits < 4): never relaxed, in place
        if (src != dst) throw Failure(QZC_EDEVICE, "tiny pass out of place");
        tile_pass_tiny<<<1, 32, 0, s>>>(dst, nbits, pd, plan.groups, plan.gates, cond);
    } else {
        const uint32_t tile = 1u << pd.k;
        const uint64_t ntiles = uint64_t(1) << (nbits - pd.k);
        const uint32_t threads = tile >> kRegBits;
        size_t smem = sizeof(double2) * tile + sizeof(uint64_t) * (tile >> pd.lowbits);
        if (pd.permute) {
            // output offsets + the output-order slot map (tile_pass_body)
            uint64_t ot = 0;
            for (uint32_t b = 0; b < 48; ++b)
                if ((pd.tmask >> b) & 1) ot |= uint64_t(1) << pd.perm[b];
            uint32_t lo = 0;
            while (lo < pd.k && ((ot >> lo) & 1)) ++lo;
            smem += sizeof(uint64_t) * (tile >> lo) + sizeof(uint16_t) * tile;
            if (src == dst) throw Failure(QZC_EDEVICE, "permuted pass in place");
        }
        // live tiles (tile_pass_body's fresh-bit skip)
        const uint64_t live = (pd.zmask && pd.pz_stable && src == dst) ? ntiles >> __builtin_popcountll(pd.zmask)
                                                                       : ntiles;
        const uint64_t grid = std::min<uint64_t>(std::max<uint64_t>(live, 1), uint64_t(kNumSMs) * 2 * 8);
        // the map is only used for passes inside one window of whole slots
        static const bool off = getenv("QZ_NO_NZMAP") != nullptr;
        const bool usable = nz.slot && nbits > nz.cbits && !off && !pd.permute;
        if (jit) {
            const double2 *a_src = src;
            double2 *a_dst = dst;
            uint32_t a_nbits = nbits, a_cbits = nz.cbits;
            PassDesc a_pd = pd;
            const GroupDesc *a_groups = plan.groups;
            const TileGate *a_gates = plan.gates;
            uint64_t a_ntiles = ntiles;
            unsigned long long *a_ctr = debug_counters();
            uint32_t *a_flag = flag;
            const uint32_t *a_cond = cond;
            uint32_t *a_nz = usable ? nz.slot : nullptr;
            void *args[] = {&a_src, &a_dst, &a_nbits, &a_pd, &a_groups, &a_gates, &a_ntiles,
                            &a_ctr, &a_flag, &a_cond, &a_nz, &a_cbits};
            if (jit_launch(*jit, (unsigned)grid, threads, smem, s, args)) {
                QZ_CHECK_LAUNCH();
                if (pd.permute) reset_nz(nz, nbits, s);
                dump_pass_counters(pd, tag, cond, s);
                return;
            }
        }
        auto kern = pd.variant == kPassDiagH ? tile_pass_reg<kPassDiagH>
                    : pd.variant == kPassGen ? tile_pass_reg<kPassGen>
                                             : tile_pass_reg<kPassAll>;
        kern<<<(unsigned)grid, threads, smem, s>>>(src, dst, nbits, pd, plan.groups, plan.gates, ntiles,
                                                   debug_counters(), flag, cond,
                                                   usable ? nz.slot : nullptr, nz.cbits);
        if (pd.permute) reset_nz(nz, nbits, s);
    }
    QZ_CHECK_LAUNCH();
    dump_pass_counters(pd, tag, cond, s);
}

} // namespace

uint64_t run_passes(const DevPlan &plan, double2 *buf, uint32_t nbits, cudaStream_t s,
                    const uint32_t *cond, NzMap nz) {
    if (plan.relaxed) throw Failure(QZC_EDEVICE, "relaxed plan run without its replay plan");
    for (const PassDesc &pd : plan.host_passes)
        if (pd.permute) throw Failure(QZC_EDEVICE, "permuted pass in an in-place plan");
    set_attrs();
    for (size_t p = 0; p < plan.host_passes.size(); ++p)
        launch_pass(plan, plan.host_passes[p], buf, buf, nbits, s, nullptr, cond, nz, uint32_t(p));
    return plan.host_passes.size();
}

void flag_done(uint32_t *flag, uint64_t *replays, cudaStream_t s) {
    k_flag_done<<<1, 1, 0, s>>>(flag, replays);
    QZ_CHECK_LAUNCH();
}

double2 *run_relaxed(const DevPlan &plan, const DevPlan &replay, double2 *buf, double2 *alt,
                     uint32_t nbits, cudaStream_t s, uint32_t *flag, uint32_t *win_flag,
                     uint64_t *replays, bool force_replay, uint64_t &launches, NzMap nz) {
    set_attrs();
    double2 *cur = buf, *oth = alt;
    for (size_t p = 0; p < plan.host_passes.size(); ++p) {
        const PassDesc &pd = plan.host_passes[p];
        if (pd.permute) {
            // fused swap network: out of place into the other buffer
            if (pd.relaxed && force_replay) QZ_CUDA(cudaMemsetAsync(win_flag, 1, 1, s));
            launch_pass(plan, pd, cur, oth, nbits, s, pd.relaxed ? win_flag : nullptr, nullptr, nz, uint32_t(p));
            ++launches;
            std::swap(cur, oth);
            continue;
        }
        if (pd.relaxed != 2) {
            if (pd.relaxed && force_replay) QZ_CUDA(cudaMemsetAsync(win_flag, 1, 1, s));
            launch_pass(plan, pd, cur, cur, nbits, s, pd.relaxed ? win_flag : nullptr, nullptr, nz, uint32_t(p));
            ++launches;
            continue;
        }
        if (force_replay) QZ_CUDA(cudaMemsetAsync(flag, 1, 1, s));
        launch_pass(plan, pd, cur, oth, nbits, s, flag, nullptr, nz, uint32_t(p));
        // strict replay of this pass from its untouched input (no-ops unless flagged)
        const auto &rr = plan.replay_range.at(p);
        for (uint32_t q = rr.first; q < rr.second; ++q)
            launch_pass(replay, replay.host_passes[q], q == rr.first ? cur : oth, oth, nbits, s, nullptr, flag, nz,
                        uint32_t(q));
        k_flag_done<<<1, 1, 0, s>>>(flag, replays);
        QZ_CHECK_LAUNCH();
        launches += 2 + (rr.second - rr.first);
        std::swap(cur, oth);
    }
    return cur;
}

void upload_replay(const std::vector<DevGate> &gates, uint32_t nbits, uint32_t kmax,
                   DevPlan &relaxed_dev, DevPlan &out, cudaStream_t s) {
    GatePlan all;
    relaxed_dev.replay_range.assign(relaxed_dev.host_passes.size(), {0u, 0u});
    for (size_t p = 0; p < relaxed_dev.host_passes.size(); ++p) {
        const PassDesc &pd = relaxed_dev.host_passes[p];
        if (pd.relaxed != 2) continue;
        const std::vector<DevGate> sub(gates.begin() + pd.dg0, gates.begin() + pd.dg1);
        const GatePlan gp = build_passes(sub, nbits, kmax, true, false);
        const uint32_t goff = (uint32_t)all.gates.size(), groff = (uint32_t)all.groups.size();
        relaxed_dev.replay_range[p].first = (uint32_t)all.passes.size();
        for (PassDesc q : gp.passes) {
            q.first_group += groff;
            q.first_gate += goff;
            q.dg0 += pd.dg0;
            q.dg1 += pd.dg0;
            all.passes.push_back(q);
        }
        relaxed_dev.replay_range[p].second = (uint32_t)all.passes.size();
        for (GroupDesc g : gp.groups) {
            g.first_gate += goff;
            g.first_fast += goff;
            all.groups.push_back(g);
        }
        all.gates.insert(all.gates.end(), gp.gates.begin(), gp.gates.end());
    }
    upload_plan(all, out, s);
}

} // namespace qz
