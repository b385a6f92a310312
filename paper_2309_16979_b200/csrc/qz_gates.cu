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
                      int relax_level) {
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
    uint64_t tmask = low_mask;
    auto close = [&]() {
        if (members.empty()) return;
        // pad T to exactly k bits with the lowest free bits (longer contiguous
        // global segments)
        for (uint32_t b = 0; b < nbits && (uint32_t)__builtin_popcountll(tmask) < k; ++b)
            tmask |= uint64_t(1) << b;
        PassDesc pd;
        std::memset(&pd, 0, sizeof pd);
        pd.k = k;
        uint32_t lowbits = 0;
        while (lowbits < 64 && ((tmask >> lowbits) & 1)) ++lowbits;
        pd.lowbits = std::min(lowbits, k);
        pd.tmask = tmask;
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
        plan.passes.push_back(pd);
        members.clear();
        tmask = low_mask;
    };
    for (size_t ui = 0; ui < units.size(); ++ui) {
        const Unit &u = units[ui];
        if (u.bits >> nbits) throw Failure(QZC_EDEVICE, "gate bit outside buffer");
        if (u.swaps) {
            // the whole swap network is one in-place bit-permutation pass
            close();
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
            continue;
        }
        const uint64_t need = u.diag ? 0 : u.bits;
        const uint64_t merged = tmask | need;
        if (!fuse || (uint32_t)__builtin_popcountll(merged) > k) close();
        tmask |= need;
        members.push_back(ui);
    }
    close();
    if (getenv("QZ_TRACE") && getenv("QZ_TRACE")[0] == '2') {
        for (const PassDesc &pd : plan.passes) {
            uint32_t nf = 0, npd = 0, nrel = 0;
            for (uint32_t gi = pd.first_group; gi < pd.first_group + pd.ngroups; ++gi) {
                nf += plan.groups[gi].nfast;
                nrel += plan.groups[gi].relaxed;
                for (uint32_t q = 0; q < plan.groups[gi].nfast; ++q)
                    npd += plan.gates[plan.groups[gi].first_fast + q].op == OP_PDIAG;
            }
            fprintf(stderr, "qz plan: kind %u tmask %#llx groups %u (relaxed %u) fast ops %u pdiag %u gates %u\n",
                    pd.kind, (unsigned long long)pd.tmask, pd.ngroups, nrel, nf, npd, pd.ngates);
        }
    }
    return plan;
}

void upload_plan(const GatePlan &plan, DevPlan &out, cudaStream_t s) {
    out.ngates = plan.gates.size();
    out.ngroups = plan.groups.size();
    out.host_passes = plan.passes;
    // kernel case set per pass: the narrow one when every fast-list entry of
    // every group is in it (and no group needs the shared-memory generic path)
    static const bool narrow_off = getenv("QZ_NO_NARROW") != nullptr;
    static const bool wmap_off = getenv("QZ_NO_WMAP") != nullptr;
    for (PassDesc &pd : out.host_passes) {
        pd.wmap = wmap_off ? 0u : 1u;
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
    out.relaxed = false;
    for (const PassDesc &pd : plan.passes) out.relaxed |= pd.relaxed != 0;
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
    p.relaxed = false;
}

// ============================================================ device math ==
//
// Exactness argument (every path is bit-identical to the dense formula of
// kernels.cpp:31-32 / 49-50):
//  * A product with a coefficient whose real or imaginary part is exactly
//    ±0 contributes ±0 to that component; x ± 0 == x for x != 0 and
//    ±0 + y == y for y != 0, so dropping those terms (and using 1*x == x,
//    -1*x == -x) can change a left-to-right sum only when the final value is
//    zero, and then only its sign.  Any output component that comes out zero
//    is recomputed: by IEEE sign rules if every input is ±0 (all products
//    are then ±0), else by the full dense formula in the reference order.
//  * A thread's 16-amplitude register block is closed under its group's
//    gates, so an all-zero block stays all-zero; only the zero signs evolve
//    and are tracked as two 16-bit masks.
//  * Non-finite amplitudes are outside the domain (a unitary circuit from
//    |0..0> never produces them).
namespace {

constexpr int NB = 1 << kRegBits;   // amplitudes per thread register block

__device__ __forceinline__ bool dz(double x) { return (__double_as_longlong(x) << 1) == 0; }
__device__ __forceinline__ bool zc(double2 v) { return dz(v.x) | dz(v.y); }
// a -0 component: the fast path's +0-safe rows may not see it (group redo)
__device__ __forceinline__ bool nz0(double2 v) {
    return (__double_as_longlong(v.x) == (long long)0x8000000000000000ULL) |
           (__double_as_longlong(v.y) == (long long)0x8000000000000000ULL);
}
__device__ __forceinline__ double dneg(double x) {
    return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL);
}
__device__ __forceinline__ double2 pm(double2 v, uint32_t neg) {
    return neg ? make_double2(dneg(v.x), dneg(v.y)) : v;
}
// +0, or exponent field in [123, 2046]: no -0, tiny, inf or nan component.
__device__ __forceinline__ uint32_t comp_ok(double x) {
    const uint64_t b = (uint64_t)__double_as_longlong(x);
    const uint32_t e = uint32_t(b >> 52) & 0x7ff;
    return uint32_t(b == 0) | uint32_t(e - 123u < 1924u);
}
__device__ __forceinline__ uint32_t sbit(double x) {
    return uint32_t((unsigned long long)__double_as_longlong(x) >> 63);
}
__device__ __forceinline__ double signed_zero(uint32_t neg) { return neg ? -0.0 : 0.0; }

__host__ __device__ constexpr int izb(int x, int bit) {
    return ((x >> bit) << (bit + 1)) | (x & ((1 << bit) - 1));
}

// Full reference row, columns in reference order, separate roundings.
__device__ double2 full_row(const TileGate &g, int r, int nc, const double2 *in) {
    double sr = 0, si = 0;
    for (int c = 0; c < nc; ++c) {
        const double2 m = g.m[r * nc + c];
        const double tr = __dsub_rn(__dmul_rn(m.x, in[c].x), __dmul_rn(m.y, in[c].y));
        const double ti = __dadd_rn(__dmul_rn(m.x, in[c].y), __dmul_rn(m.y, in[c].x));
        sr = c == 0 ? tr : __dadd_rn(sr, tr);
        si = c == 0 ? ti : __dadd_rn(si, ti);
    }
    return make_double2(sr, si);
}

// Exact recomputation of one output row whose fast value had a zero
// component; `in` is in reference column order.  If every input is ±0 all
// products are ±0 and IEEE sign rules decide (x - y: -0 iff x=-0, y=+0;
// x + y: -0 iff both -0); otherwise the full formula is evaluated.
__device__ double2 exact_row(const TileGate &g, int r, int nc, const double2 *in) {
    // per component: are all its products zero (a zero factor each)?
    bool zre = true, zim = true;
    uint32_t nre = 1, nim = 1;
    for (int c = 0; c < nc; ++c) {
        const int e = r * nc + c;
        const bool mrz = (g.zm >> e) & 1, miz = (g.zm >> (16 + e)) & 1;
        const bool vrz = dz(in[c].x), viz = dz(in[c].y);
        zre = zre && (mrz || vrz) && (miz || viz);
        zim = zim && (mrz || viz) && (miz || vrz);
        const uint32_t smr = (g.sgn >> (2 * e)) & 1, smi = (g.sgn >> (2 * e + 1)) & 1;
        const uint32_t svr = sbit(in[c].x), svi = sbit(in[c].y);
        nre &= (smr ^ svr) & ~(smi ^ svi);   // mr*vr - mi*vi
        nim &= (smr ^ svi) & (smi ^ svr);    // mr*vi + mi*vr
    }
    double2 o;
    if (zre && zim) return make_double2(signed_zero(nre & 1), signed_zero(nim & 1));
    o = full_row(g, r, nc, in);
    if (zre) o.x = signed_zero(nre & 1);
    if (zim) o.y = signed_zero(nim & 1);
    return o;
}

__device__ __noinline__ double2 slow2(const TileGate &g, int r, double2 a, double2 b) {
    const double2 in[2] = {a, b};
    return exact_row(g, r, 2, in);
}

__device__ __noinline__ double2 slow4(const TileGate &g, int r, double2 a, double2 b, double2 c,
                                      double2 d) {
    const double2 in[4] = {a, b, c, d};
    return exact_row(g, r, 4, in);
}

// One nonzero term, kind uniform across the warp.
__device__ __forceinline__ double2 term(uint32_t kind, double2 m, double2 v) {
    if (kind == CK_ONE) return v;
    if (kind == CK_NEG) return make_double2(dneg(v.x), dneg(v.y));
    if (kind == CK_REAL) return make_double2(__dmul_rn(m.x, v.x), __dmul_rn(m.x, v.y));
    if (kind == CK_IMAG) return make_double2(dneg(__dmul_rn(m.y, v.y)), __dmul_rn(m.y, v.x));
    return make_double2(__dsub_rn(__dmul_rn(m.x, v.x), __dmul_rn(m.y, v.y)),
                        __dadd_rn(__dmul_rn(m.x, v.y), __dmul_rn(m.y, v.x)));
}

// Compile-time-kind term (K < 0: run-time kind).
template <int K>
__device__ __forceinline__ double2 termk(uint32_t kind, double2 m, double2 v) {
    if constexpr (K < 0) {
        return term(kind, m, v);
    } else if constexpr (K == CK_ONE) {
        return v;
    } else if constexpr (K == CK_NEG) {
        return make_double2(dneg(v.x), dneg(v.y));
    } else if constexpr (K == CK_REAL) {
        return make_double2(__dmul_rn(m.x, v.x), __dmul_rn(m.x, v.y));
    } else if constexpr (K == CK_IMAG) {
        return make_double2(dneg(__dmul_rn(m.y, v.y)), __dmul_rn(m.y, v.x));
    } else {
        return make_double2(__dsub_rn(__dmul_rn(m.x, v.x), __dmul_rn(m.y, v.y)),
                            __dadd_rn(__dmul_rn(m.x, v.y), __dmul_rn(m.y, v.x)));
    }
}

__device__ __forceinline__ double2 sum2(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

// ---- 1-qubit gates on register bit R ----
template <int R>
__device__ __forceinline__ void reg_apply1(double2 (&v)[NB], const TileGate &g) {
    constexpr int sh = 1 << R;
    const uint32_t kd = uint32_t(g.kinds);
    const uint32_t k00 = kd & 15u, k01 = (kd >> 4) & 15u, k10 = (kd >> 8) & 15u, k11 = (kd >> 12) & 15u;
    const double2 m00 = g.m[0], m01 = g.m[1], m10 = g.m[2], m11 = g.m[3];
    const uint32_t cls = g.cls, pc = g.perm;
#pragma unroll
    for (int p = 0; p < NB / 2; ++p) {
        const int i = izb(p, R), j = i | sh;
        const double2 a = v[i], b = v[j];
        double2 oi, oj;
        if (cls == TG_PERM) {
            oi = pm((pc & 1) ? b : a, (pc >> 2) & 1);
            oj = pm(((pc >> 3) & 1) ? b : a, (pc >> 5) & 1);
        } else if (cls == TG_DIAG) {
            oi = term(k00, m00, a);
            oj = term(k11, m11, b);
        } else {
            oi = k00 == CK_ZERO ? term(k01, m01, b)
                                : (k01 == CK_ZERO ? term(k00, m00, a) : sum2(term(k00, m00, a), term(k01, m01, b)));
            oj = k10 == CK_ZERO ? term(k11, m11, b)
                                : (k11 == CK_ZERO ? term(k10, m10, a) : sum2(term(k10, m10, a), term(k11, m11, b)));
        }
        if (zc(oi) | zc(oj)) {
            // both inputs +0 and the row maps (+0,+0) to +0: the common case
            // in sparse states, no call needed
            const bool pz = ((__double_as_longlong(a.x) | __double_as_longlong(a.y) |
                              __double_as_longlong(b.x) | __double_as_longlong(b.y)) == 0);
            if (zc(oi)) oi = (pz && (g.pad & 1)) ? make_double2(0.0, 0.0) : slow2(g, 0, a, b);
            if (zc(oj)) oj = (pz && (g.pad & 2)) ? make_double2(0.0, 0.0) : slow2(g, 1, a, b);
        }
        v[i] = oi;
        v[j] = oj;
    }
}

// ---- 2-qubit signed permutations (CX CZ SWAP) on register bits (R0, R1) ----
template <int R0, int R1>
__device__ __forceinline__ void reg_apply2(double2 (&v)[NB], const TileGate &g) {
    constexpr int lo = R0 < R1 ? R0 : R1, hi = R0 < R1 ? R1 : R0;
    constexpr int s0 = 1 << R0, s1 = 1 << R1;
    const uint32_t pc = g.perm;
#pragma unroll
    for (int q = 0; q < NB / 4; ++q) {
        const int b = izb(izb(q, lo), hi);
        const double2 in0 = v[b], in1 = v[b | s1], in2 = v[b | s0], in3 = v[b | s0 | s1];
        double2 o[4];
        bool anyz = false;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t c = (pc >> (3 * r)) & 3, ng = (pc >> (3 * r + 2)) & 1;
            o[r] = pm(c == 0 ? in0 : c == 1 ? in1 : c == 2 ? in2 : in3, ng);
            anyz |= zc(o[r]);
        }
        if (anyz) {
            const bool pz = ((__double_as_longlong(in0.x) | __double_as_longlong(in0.y) |
                              __double_as_longlong(in1.x) | __double_as_longlong(in1.y) |
                              __double_as_longlong(in2.x) | __double_as_longlong(in2.y) |
                              __double_as_longlong(in3.x) | __double_as_longlong(in3.y)) == 0);
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (zc(o[r]))
                    o[r] = (pz && ((g.pad >> r) & 1)) ? make_double2(0.0, 0.0)
                                                      : slow4(g, r, in0, in1, in2, in3);
        }
        v[b] = o[0];
        v[b | s1] = o[1];
        v[b | s0] = o[2];
        v[b | s0 | s1] = o[3];
    }
}

#if QZ_REG_BITS == 3
#define QZ_R1_CASES(X) X(0) X(1) X(2)
#define QZ_R2_CASES(X) X(0, 1) X(0, 2) X(1, 0) X(1, 2) X(2, 0) X(2, 1)
#else
#define QZ_R1_CASES(X) X(0) X(1) X(2) X(3)
#define QZ_R2_CASES(X)                                                               \
    X(0, 1) X(0, 2) X(0, 3) X(1, 0) X(1, 2) X(1, 3) X(2, 0) X(2, 1) X(2, 3) X(3, 0)   \
    X(3, 1) X(3, 2)
#endif

// ---- zero-free fast path ----------------------------------------------------
// Valid while every component in the block is nonzero: moves are exact, and
// the shortcut products are exact for nonzero results.  Any zero output sets
// `bad`; the caller then redoes the whole group on the exact path.
// SPEC = 1: every row +0-safe and the kinds are the template's (no checks,
// no kind branches); SPEC = 0: run-time kinds and safety.
template <int R, int K0 = -1, int K1 = -1, int SPEC = 0>
__device__ __forceinline__ void fast_diag(double2 (&v)[NB], const TileGate &g, bool &bad) {
    constexpr int sh = 1 << R;
    const uint32_t k00 = uint32_t(g.kinds) & 15u, k11 = uint32_t(g.kinds >> 12) & 15u;
    const double2 m00 = g.m[0], m11 = g.m[3];
    const bool u0 = SPEC != 1 && !(g.srow & 1), u1 = SPEC != 1 && !(g.srow & 2);
#pragma unroll
    for (int p = 0; p < NB / 2; ++p) {
        const int i = izb(p, R), j = i | sh;
        const double2 a = v[i], b = v[j];
        // a zero in a row that is not +0-safe: that row's exact value
        if (K0 == CK_ONE || (K0 < 0 && k00 == CK_ONE)) {
        } else {
            double2 o = termk<K0>(k00, m00, a);
            if (u0 && zc(o)) {
                o = slow2(g, 0, a, b);
                bad |= nz0(o);
            }
            v[i] = o;
        }
        if (K1 == CK_ONE || (K1 < 0 && k11 == CK_ONE)) {
        } else {
            double2 o = termk<K1>(k11, m11, b);
            if (u1 && zc(o)) {
                o = slow2(g, 1, a, b);
                bad |= nz0(o);
            }
            v[j] = o;
        }
    }
}

template <int R, int K00 = -1, int K01 = -1, int K10 = -1, int K11 = -1, int SPEC = 0>
__device__ __forceinline__ void fast_gen1(double2 (&v)[NB], const TileGate &g, bool &bad) {
    constexpr int sh = 1 << R;
    const uint32_t kd = uint32_t(g.kinds);
    const uint32_t k00 = kd & 15u, k01 = (kd >> 4) & 15u, k10 = (kd >> 8) & 15u, k11 = (kd >> 12) & 15u;
    const double2 m00 = g.m[0], m01 = g.m[1], m10 = g.m[2], m11 = g.m[3];
#pragma unroll
    for (int p = 0; p < NB / 2; ++p) {
        const int i = izb(p, R), j = i | sh;
        const double2 a = v[i], b = v[j];
        double2 oi, oj;
        if constexpr (SPEC) {
            if constexpr (K00 == CK_ZERO) oi = termk<K01>(k01, m01, b);
            else if constexpr (K01 == CK_ZERO) oi = termk<K00>(k00, m00, a);
            else oi = sum2(termk<K00>(k00, m00, a), termk<K01>(k01, m01, b));
            if constexpr (K10 == CK_ZERO) oj = termk<K11>(k11, m11, b);
            else if constexpr (K11 == CK_ZERO) oj = termk<K10>(k10, m10, a);
            else oj = sum2(termk<K10>(k10, m10, a), termk<K11>(k11, m11, b));
            if constexpr (SPEC == 2) {   // compile-time kinds, rows not all +0-safe
                if (!(g.srow & 1) && zc(oi)) {
                    oi = slow2(g, 0, a, b);
                    bad |= nz0(oi);
                }
                if (!(g.srow & 2) && zc(oj)) {
                    oj = slow2(g, 1, a, b);
                    bad |= nz0(oj);
                }
            }
        } else {
            oi = k00 == CK_ZERO ? term(k01, m01, b)
               : (k01 == CK_ZERO ? term(k00, m00, a) : sum2(term(k00, m00, a), term(k01, m01, b)));
            oj = k10 == CK_ZERO ? term(k11, m11, b)
               : (k11 == CK_ZERO ? term(k10, m10, a) : sum2(term(k10, m10, a), term(k11, m11, b)));
            if (!(g.srow & 1) && zc(oi)) {
                oi = slow2(g, 0, a, b);
                bad |= nz0(oi);
            }
            if (!(g.srow & 2) && zc(oj)) {
                oj = slow2(g, 1, a, b);
                bad |= nz0(oj);
            }
        }
        v[i] = oi;
        v[j] = oj;
    }
}

template <int C, int T>
__device__ __forceinline__ void fast_cx(double2 (&v)[NB]) {
#pragma unroll
    for (int i = 0; i < NB; ++i)
        if (((i >> C) & 1) && !((i >> T) & 1)) {
            const double2 t = v[i];
            v[i] = v[i | (1 << T)];
            v[i | (1 << T)] = t;
        }
}

template <int A, int B>
__device__ __forceinline__ void fast_cz(double2 (&v)[NB], const TileGate &g, bool &bad) {
#pragma unroll
    for (int i = 0; i < NB; ++i)
        if (((i >> A) & 1) && ((i >> B) & 1)) {
            const double2 o = make_double2(dneg(v[i].x), dneg(v[i].y));
            if (zc(o)) {
                // the -1 row is not +0-safe: its exact value (the other three
                // products are +-0; their order does not matter for zeros)
                const int i00 = i & ~((1 << A) | (1 << B));
                v[i] = slow4(g, 3, v[i00], v[i00 | (1 << A)], v[i00 | (1 << B)], v[i]);
                bad |= nz0(v[i]);
            } else {
                v[i] = o;
            }
        }
}

template <int A, int B>
__device__ __forceinline__ void fast_swap(double2 (&v)[NB]) {
#pragma unroll
    for (int i = 0; i < NB; ++i)
        if (((i >> A) & 1) && !((i >> B) & 1)) {
            const int j = (i & ~(1 << A)) | (1 << B);
            const double2 t = v[i];
            v[i] = v[j];
            v[j] = t;
        }
}

// CP5 on (A, B): p01 <- m3(m2 v01), p10 <- m2(m1 v10), p11 <- m3(m1 v11)
// (the CX swaps folded into the indexing; same products, same order).
template <int A, int B, int SPEC = 0>
__device__ __forceinline__ void fast_cp5(double2 (&v)[NB], const TileGate &g, bool &bad) {
    const uint32_t k1 = uint32_t(g.kinds) & 15u, k2 = uint32_t(g.kinds >> 4) & 15u,
                   k3 = uint32_t(g.kinds >> 8) & 15u;
    const double2 m1 = g.m[0], m2 = g.m[1], m3 = g.m[2];
    const bool u1 = !SPEC && !(g.srow & 1), u2 = !SPEC && !(g.srow & 2), u3 = !SPEC && !(g.srow & 4);
    constexpr int KC = SPEC ? int(CK_CPLX) : -1;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        if (((i >> A) & 1) || ((i >> B) & 1)) continue;
        const int i01 = i | (1 << B), i10 = i | (1 << A), i11 = i | (1 << A) | (1 << B);
        double2 x01 = termk<KC>(k2, m2, v[i01]);
        if (u2) bad |= zc(x01);
        x01 = termk<KC>(k3, m3, x01);
        if (u3) bad |= zc(x01);
        double2 x10 = termk<KC>(k1, m1, v[i10]);
        if (u1) bad |= zc(x10);
        x10 = termk<KC>(k2, m2, x10);
        if (u2) bad |= zc(x10);
        double2 x11 = termk<KC>(k1, m1, v[i11]);
        if (u1) bad |= zc(x11);
        x11 = termk<KC>(k3, m3, x11);
        if (u3) bad |= zc(x11);
        v[i01] = x01;
        v[i10] = x10;
        v[i11] = x11;
    }
}

// CXD on (A, B), D = diag(d0, d1) on B: p00 <- d0 v00, p01 <- d1 v01,
// p10 <- d1 v10, p11 <- d0 v11.
template <int A, int B, int SPEC = 0>
__device__ __forceinline__ void fast_cxd(double2 (&v)[NB], const TileGate &g, bool &bad) {
    const uint32_t k0 = uint32_t(g.kinds) & 15u, k1 = uint32_t(g.kinds >> 4) & 15u;
    const double2 d0 = g.m[0], d1 = g.m[1];
    const bool u0 = !SPEC && !(g.srow & 1), u1 = !SPEC && !(g.srow & 2);
    constexpr int KC = SPEC ? int(CK_CPLX) : -1;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        if (((i >> A) & 1) || ((i >> B) & 1)) continue;
        const int i01 = i | (1 << B), i10 = i | (1 << A), i11 = i | (1 << A) | (1 << B);
        const double2 x00 = termk<KC>(k0, d0, v[i]), x01 = termk<KC>(k1, d1, v[i01]);
        const double2 x10 = termk<KC>(k1, d1, v[i10]), x11 = termk<KC>(k0, d0, v[i11]);
        if (u0) bad |= zc(x00) | zc(x11);
        if (u1) bad |= zc(x01) | zc(x10);
        v[i] = x00;
        v[i01] = x01;
        v[i10] = x10;
        v[i11] = x11;
    }
}

// OP_PDIAG resolved for this tile's outside-bit values `var`: step chains on
// register bit R (R == kRegBits: one chain for the whole block).
// SPEC = 1: every step CPLX and +0-safe (no kind branches, no checks).
template <int R, int SPEC = 0>
__device__ __forceinline__ void fast_pdiag(double2 (&v)[NB], const TileGate &g, uint32_t var,
                                           bool &bad) {
    const uint32_t kd = uint32_t(g.kinds >> (16 * var));
    const uint32_t sf = g.srow >> (4 * var);
    constexpr int KC = SPEC ? int(CK_CPLX) : -1;
#pragma unroll
    for (int st = 0; st < (R < kRegBits ? 2 : 1); ++st) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint32_t e = 2 * st + j;
            const uint32_t kind = (kd >> (4 * e)) & 15u;
            if (kind == CK_ZERO) continue;
            const double2 m = g.m[4 * var + e];
            const bool chk = !SPEC && !((sf >> e) & 1);
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                if (R < kRegBits && ((i >> R) & 1) != st) continue;
                v[i] = termk<KC>(kind, m, v[i]);
                if (chk) bad |= zc(v[i]);
            }
        }
    }
}

// Run of specialised OP_PDIAG ops: every step a CPLX +0-safe product, no
// checks; per op only the thread's variant and register bit are resolved.
template <int R>
__device__ __forceinline__ void pdiag_spec(double2 (&v)[NB], const double2 *__restrict__ mm,
                                           uint32_t act) {
#pragma unroll
    for (int st = 0; st < (R < kRegBits ? 2 : 1); ++st) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int e = 2 * st + j;
            if (!((act >> e) & 1)) continue;
            const double2 m = mm[e];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                if (R < kRegBits && ((i >> R) & 1) != st) continue;
                v[i] = termk<CK_CPLX>(CK_CPLX, m, v[i]);
            }
        }
    }
}

#if QZ_REG_BITS == 3
#define QZ_PAIRS(X) X(0, 1) X(0, 2) X(1, 2)
#else
#define QZ_PAIRS(X) X(0, 1) X(0, 2) X(0, 3) X(1, 2) X(1, 3) X(2, 3)
#endif

// Flat dispatch: one jump table over a host-computed case id (case_id(),
// which mirrors this switch), so every op leaves the register block in the
// same registers.  Returns the number of fast-list entries consumed.
__device__ __forceinline__ uint32_t pdiag_var(const TileGate &g, uint64_t gidx) {
    return uint32_t((gidx >> g.ob0) & 1) | (uint32_t((gidx >> g.ob1) & 1) << 1);
}

// A run mixes uniform ops (no register bit) with ops on register bit R.
template <int R>
__device__ __forceinline__ void run_pdiag_r(double2 (&v)[NB], const TileGate *__restrict__ gp,
                                            uint32_t n, uint64_t gidx) {
    for (uint32_t q = 0; q < n; ++q) {
        const TileGate &g = gp[q];
        const uint32_t var = pdiag_var(g, gidx);
        const uint32_t act = (g.steps >> (4 * var)) & 15u;
        if (R == kRegBits || g.nq == 0) pdiag_spec<kRegBits>(v, g.m + 4 * var, act);
        else pdiag_spec<R>(v, g.m + 4 * var, act);
    }
}

template <int S>
__device__ __forceinline__ uint32_t fast_case(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q,
                                              uint64_t gidx, bool &bad) {
    const TileGate &g = fp[q];
    switch (g.cid) {
    case 0: if constexpr (case_on(S, 0)) { run_pdiag_r<0>(v, fp + q, g.run, gidx); return g.run; } else { bad = true; return 1; }
    case 1: if constexpr (case_on(S, 1)) { run_pdiag_r<1>(v, fp + q, g.run, gidx); return g.run; } else { bad = true; return 1; }
    case 2: if constexpr (case_on(S, 2)) { run_pdiag_r<2>(v, fp + q, g.run, gidx); return g.run; } else { bad = true; return 1; }
    case 3: if constexpr (case_on(S, 3)) { run_pdiag_r<3>(v, fp + q, g.run, gidx); return g.run; } else { bad = true; return 1; }
    case 4: if constexpr (case_on(S, 4)) { fast_pdiag<0, 0>(v, g, pdiag_var(g, gidx), bad); return 1; } else { bad = true; return 1; }
    case 5: if constexpr (case_on(S, 5)) { fast_pdiag<0, 1>(v, g, pdiag_var(g, gidx), bad); return 1; } else { bad = true; return 1; }
    case 6: if constexpr (case_on(S, 6)) { fast_pdiag<1, 0>(v, g, pdiag_var(g, gidx), bad); return 1; } else { bad = true; return 1; }
    case 7: if constexpr (case_on(S, 7)) { fast_pdiag<1, 1>(v, g, pdiag_var(g, gidx), bad); return 1; } else { bad = true; return 1; }
    case 8: if constexpr (case_on(S, 8)) { fast_pdiag<2, 0>(v, g, pdiag_var(g, gidx), bad); return 1; } else { bad = true; return 1; }
    case 9: if constexpr (case_on(S, 9)) { fast_pdiag<2, 1>(v, g, pdiag_var(g, gidx), bad); return 1; } else { bad = true; return 1; }
    case 10: if constexpr (case_on(S, 10)) { fast_pdiag<3, 0>(v, g, pdiag_var(g, gidx), bad); return 1; } else { bad = true; return 1; }
    case 11: if constexpr (case_on(S, 11)) { fast_pdiag<3, 1>(v, g, pdiag_var(g, gidx), bad); return 1; } else { bad = true; return 1; }
    case 12: if constexpr (case_on(S, 12)) { fast_diag<0, CK_ONE, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 13: if constexpr (case_on(S, 13)) { fast_diag<0, CK_CPLX, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 14: if constexpr (case_on(S, 14)) { fast_diag<0, CK_ONE, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 15: if constexpr (case_on(S, 15)) { fast_diag<0, CK_CPLX, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 16: if constexpr (case_on(S, 16)) { fast_diag<0>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 17: if constexpr (case_on(S, 17)) { fast_diag<1, CK_ONE, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 18: if constexpr (case_on(S, 18)) { fast_diag<1, CK_CPLX, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 19: if constexpr (case_on(S, 19)) { fast_diag<1, CK_ONE, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 20: if constexpr (case_on(S, 20)) { fast_diag<1, CK_CPLX, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 21: if constexpr (case_on(S, 21)) { fast_diag<1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 22: if constexpr (case_on(S, 22)) { fast_diag<2, CK_ONE, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 23: if constexpr (case_on(S, 23)) { fast_diag<2, CK_CPLX, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 24: if constexpr (case_on(S, 24)) { fast_diag<2, CK_ONE, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 25: if constexpr (case_on(S, 25)) { fast_diag<2, CK_CPLX, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 26: if constexpr (case_on(S, 26)) { fast_diag<2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 27: if constexpr (case_on(S, 27)) { fast_gen1<0, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 28: if constexpr (case_on(S, 28)) { fast_gen1<0, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 29: if constexpr (case_on(S, 29)) { fast_gen1<0, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 30: if constexpr (case_on(S, 30)) { fast_gen1<0, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 31: if constexpr (case_on(S, 31)) { fast_gen1<0, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 32: if constexpr (case_on(S, 32)) { fast_gen1<0, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 33: if constexpr (case_on(S, 33)) { fast_gen1<0, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 34: if constexpr (case_on(S, 34)) { fast_gen1<0, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 35: if constexpr (case_on(S, 35)) { fast_gen1<0, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 36: if constexpr (case_on(S, 36)) { fast_gen1<0, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 37: if constexpr (case_on(S, 37)) { fast_gen1<0, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 38: if constexpr (case_on(S, 38)) { fast_gen1<0, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 39: if constexpr (case_on(S, 39)) { fast_gen1<0, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 40: if constexpr (case_on(S, 40)) { fast_gen1<0, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 41: if constexpr (case_on(S, 41)) { fast_gen1<0>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 42: if constexpr (case_on(S, 42)) { fast_gen1<1, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 43: if constexpr (case_on(S, 43)) { fast_gen1<1, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 44: if constexpr (case_on(S, 44)) { fast_gen1<1, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 45: if constexpr (case_on(S, 45)) { fast_gen1<1, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 46: if constexpr (case_on(S, 46)) { fast_gen1<1, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 47: if constexpr (case_on(S, 47)) { fast_gen1<1, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 48: if constexpr (case_on(S, 48)) { fast_gen1<1, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 49: if constexpr (case_on(S, 49)) { fast_gen1<1, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 50: if constexpr (case_on(S, 50)) { fast_gen1<1, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 51: if constexpr (case_on(S, 51)) { fast_gen1<1, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 52: if constexpr (case_on(S, 52)) { fast_gen1<1, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 53: if constexpr (case_on(S, 53)) { fast_gen1<1, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 54: if constexpr (case_on(S, 54)) { fast_gen1<1, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 55: if constexpr (case_on(S, 55)) { fast_gen1<1, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 56: if constexpr (case_on(S, 56)) { fast_gen1<1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 57: if constexpr (case_on(S, 57)) { fast_gen1<2, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 58: if constexpr (case_on(S, 58)) { fast_gen1<2, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 59: if constexpr (case_on(S, 59)) { fast_gen1<2, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 60: if constexpr (case_on(S, 60)) { fast_gen1<2, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 61: if constexpr (case_on(S, 61)) { fast_gen1<2, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 62: if constexpr (case_on(S, 62)) { fast_gen1<2, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 63: if constexpr (case_on(S, 63)) { fast_gen1<2, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 64: if constexpr (case_on(S, 64)) { fast_gen1<2, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 65: if constexpr (case_on(S, 65)) { fast_gen1<2, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 66: if constexpr (case_on(S, 66)) { fast_gen1<2, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 67: if constexpr (case_on(S, 67)) { fast_gen1<2, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 68: if constexpr (case_on(S, 68)) { fast_gen1<2, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 69: if constexpr (case_on(S, 69)) { fast_gen1<2, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 70: if constexpr (case_on(S, 70)) { fast_gen1<2, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 71: if constexpr (case_on(S, 71)) { fast_gen1<2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 72: if constexpr (case_on(S, 72)) { fast_cp5<0, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 73: if constexpr (case_on(S, 73)) { fast_cp5<0, 1, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 74: if constexpr (case_on(S, 74)) { fast_cp5<0, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 75: if constexpr (case_on(S, 75)) { fast_cp5<0, 2, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 76: if constexpr (case_on(S, 76)) { fast_cp5<1, 0>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 77: if constexpr (case_on(S, 77)) { fast_cp5<1, 0, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 78: if constexpr (case_on(S, 78)) { fast_cp5<1, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 79: if constexpr (case_on(S, 79)) { fast_cp5<1, 2, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 80: if constexpr (case_on(S, 80)) { fast_cp5<2, 0>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 81: if constexpr (case_on(S, 81)) { fast_cp5<2, 0, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 82: if constexpr (case_on(S, 82)) { fast_cp5<2, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 83: if constexpr (case_on(S, 83)) { fast_cp5<2, 1, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 84: if constexpr (case_on(S, 84)) { fast_cxd<0, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 85: if constexpr (case_on(S, 85)) { fast_cxd<0, 1, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 86: if constexpr (case_on(S, 86)) { fast_cxd<0, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 87: if constexpr (case_on(S, 87)) { fast_cxd<0, 2, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 88: if constexpr (case_on(S, 88)) { fast_cxd<1, 0>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 89: if constexpr (case_on(S, 89)) { fast_cxd<1, 0, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 90: if constexpr (case_on(S, 90)) { fast_cxd<1, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 91: if constexpr (case_on(S, 91)) { fast_cxd<1, 2, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 92: if constexpr (case_on(S, 92)) { fast_cxd<2, 0>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 93: if constexpr (case_on(S, 93)) { fast_cxd<2, 0, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 94: if constexpr (case_on(S, 94)) { fast_cxd<2, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 95: if constexpr (case_on(S, 95)) { fast_cxd<2, 1, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 96: if constexpr (case_on(S, 96)) { fast_cx<0, 1>(v); return 1; } else { bad = true; return 1; }
    case 97: if constexpr (case_on(S, 97)) { fast_cx<0, 2>(v); return 1; } else { bad = true; return 1; }
    case 98: if constexpr (case_on(S, 98)) { fast_cx<1, 0>(v); return 1; } else { bad = true; return 1; }
    case 99: if constexpr (case_on(S, 99)) { fast_cx<1, 2>(v); return 1; } else { bad = true; return 1; }
    case 100: if constexpr (case_on(S, 100)) { fast_cx<2, 0>(v); return 1; } else { bad = true; return 1; }
    case 101: if constexpr (case_on(S, 101)) { fast_cx<2, 1>(v); return 1; } else { bad = true; return 1; }
    case 102: if constexpr (case_on(S, 102)) { fast_cz<0, 1>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 103: if constexpr (case_on(S, 103)) { fast_cz<0, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 104: if constexpr (case_on(S, 104)) { fast_cz<1, 2>(v, g, bad); return 1; } else { bad = true; return 1; }
    case 105: if constexpr (case_on(S, 105)) { fast_swap<0, 1>(v); return 1; } else { bad = true; return 1; }
    case 106: if constexpr (case_on(S, 106)) { fast_swap<0, 2>(v); return 1; } else { bad = true; return 1; }
    case 107: if constexpr (case_on(S, 107)) { fast_swap<1, 2>(v); return 1; } else { bad = true; return 1; }
    default: bad = true; return 1;   // other 2q matrices: exact path only
    }
}

#if QZ_REG_BITS != 3
#error "the flat fast-path dispatch (fast_case / case_id) is generated for QZ_REG_BITS == 3"
#endif

// ---- sign-mask mode for all-zero register blocks ----
__host__ __device__ constexpr uint32_t low_positions(int R) {
    uint32_t m = 0;
    for (int i = 0; i < NB; ++i)
        if (!((i >> R) & 1)) m |= 1u << i;
    return m;
}

__device__ __forceinline__ void zero_terms(uint32_t sgn, int e, uint32_t xr, uint32_t xi,
                                           uint32_t &re, uint32_t &im) {
    const uint32_t mr = 0u - ((sgn >> (2 * e)) & 1u);
    const uint32_t mi = 0u - ((sgn >> (2 * e + 1)) & 1u);
    re &= (xr ^ mr) & ~(xi ^ mi);
    im &= (xi ^ mr) & (xr ^ mi);
}

template <int R>
__device__ __forceinline__ void mask_apply1(uint32_t &SR, uint32_t &SI, const TileGate &g) {
    constexpr uint32_t LOW = low_positions(R);
    constexpr int sh = 1 << R;
    const uint32_t ar = SR & LOW, ai = SI & LOW;
    const uint32_t br = (SR >> sh) & LOW, bi = (SI >> sh) & LOW;
    uint32_t r0 = LOW, i0 = LOW, r1 = LOW, i1 = LOW;
    zero_terms(g.sgn, 0, ar, ai, r0, i0);
    zero_terms(g.sgn, 1, br, bi, r0, i0);
    zero_terms(g.sgn, 2, ar, ai, r1, i1);
    zero_terms(g.sgn, 3, br, bi, r1, i1);
    SR = (r0 & LOW) | ((r1 & LOW) << sh);
    SI = (i0 & LOW) | ((i1 & LOW) << sh);
}

template <int R0, int R1>
__device__ __forceinline__ void mask_apply2(uint32_t &SR, uint32_t &SI, const TileGate &g) {
    constexpr uint32_t BASE = low_positions(R0) & low_positions(R1);
    constexpr int s0 = 1 << R0, s1 = 1 << R1;
    const int off[4] = {0, s1, s0, s0 | s1};
    uint32_t xr[4], xi[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        xr[c] = (SR >> off[c]) & BASE;
        xi[c] = (SI >> off[c]) & BASE;
    }
    uint32_t nr = 0, ni = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        uint32_t re = BASE, im = BASE;
#pragma unroll
        for (int c = 0; c < 4; ++c) zero_terms(g.sgn, 4 * r + c, xr[c], xi[c], re, im);
        nr |= (re & BASE) << off[r];
        ni |= (im & BASE) << off[r];
    }
    SR = nr;
    SI = ni;
}


__device__ __forceinline__ void reg_apply(double2 (&v)[NB], const TileGate &g) {
    if (g.nq == 1) {
        switch (g.r0) {
#define X(a)                                                                                 \
    case a: reg_apply1<a>(v, g); break;
            QZ_R1_CASES(X)
#undef X
        default: break;
        }
        return;
    }
    switch (g.r0 * 4 + g.r1) {
#define X(a, b)                                                                              \
    case a * 4 + b: reg_apply2<a, b>(v, g); break;
        QZ_R2_CASES(X)
#undef X
    default: break;
    }
}

__device__ __forceinline__ void mask_apply(uint32_t &SR, uint32_t &SI, const TileGate &g) {
    if (g.nq == 1) {
        switch (g.r0) {
#define X(a)                                                                                 \
    case a: mask_apply1<a>(SR, SI, g); break;
            QZ_R1_CASES(X)
#undef X
        default: break;
        }
        return;
    }
    switch (g.r0 * 4 + g.r1) {
#define X(a, b)                                                                              \
    case a * 4 + b: mask_apply2<a, b>(SR, SI, g); break;
        QZ_R2_CASES(X)
#undef X
    default: break;
    }
}

// Bank-conflict swizzle of the 16 B shared-memory slots inside each 128 B row.
// Shared-memory slot of tile element l: its low 3 bits XOR bits 3-5 and 6-8
// (a bijection), so 16-byte accesses whose lanes differ in bits 3-8 — the
// contiguous tile fill, a register group's block under either thread map —
// spread over all 8 bank groups.
__device__ __forceinline__ uint32_t swz(uint32_t l) { return l ^ ((l >> 3) & 7u) ^ ((l >> 6) & 7u); }


__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Generic gate straight on the shared-memory tile (any matrix; used for
// 2-qubit gates that are not signed permutations — none in the reference
// gate set — and kept exact with the full formula).
__device__ void smem_generic(double2 *s, uint32_t tile, const TileGate &g) {
    const uint32_t tid = threadIdx.x, nth = blockDim.x;
    if (g.nq == 1) {
        for (uint32_t p = tid; p < tile / 2; p += nth) {
            const uint32_t i = insert_zero_bit32(p, g.t0), j = i | (1u << g.t0);
            const double2 in[2] = {s[swz(i)], s[swz(j)]};
            s[swz(i)] = full_row(g, 0, 2, in);
            s[swz(j)] = full_row(g, 1, 2, in);
        }
    } else {
        const uint32_t lo = min(g.t0, g.t1), hi = max(g.t0, g.t1);
        const uint32_t s0 = 1u << g.t0, s1 = 1u << g.t1;
        for (uint32_t p = tid; p < tile / 4; p += nth) {
            const uint32_t b = insert_zero_bit32(insert_zero_bit32(p, lo), hi);
            const uint32_t idx[4] = {b, b | s1, b | s0, b | s0 | s1};
            double2 in[4];
            for (int c = 0; c < 4; ++c) in[c] = s[swz(idx[c])];
            for (int r = 0; r < 4; ++r) s[swz(idx[r])] = full_row(g, r, 4, in);
        }
    }
}

#ifndef QZ_MIN_CTAS
#define QZ_MIN_CTAS 3
#endif

// One fused pass: tile of 2^k amplitudes (k >= kRegBits) in shared memory;
// each group is applied by 2^(k-kRegBits) threads holding NB amplitudes in
// registers.  Every thread moves exactly NB amplitudes per tile in each
// direction, all issued before any is consumed (cp.async in, batched stores).
template <int S>
__global__ void __launch_bounds__(1 << (kTileBits - kRegBits), (kTileBits >= 12 ? 1 : (kTileBits == 11 ? QZ_MIN_CTAS : 4))) tile_pass_reg(const double2 *__restrict__ src, double2 *__restrict__ dst, uint32_t nbits,
                                                         PassDesc pd,
                                                         const GroupDesc *__restrict__ groups,
                                                         const TileGate *__restrict__ gates,
                                                         uint64_t ntiles,
                                                         unsigned long long *__restrict__ counters,
                                                         uint32_t *__restrict__ flag,
                                                         const uint32_t *__restrict__ cond,
                                                         uint32_t *__restrict__ nzslot, uint32_t cbits) {
    if (cond && *cond == 0) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *s = reinterpret_cast<double2 *>(smem_raw);
    const uint32_t k = pd.k, L = pd.lowbits;
    const uint32_t tile = 1u << k;
    uint64_t *offhi = reinterpret_cast<uint64_t *>(s + tile);
    const uint32_t nhi = 1u << (k - L);
    const uint64_t all = (uint64_t(1) << nbits) - 1;
    const uint64_t ntmask = all & ~pd.tmask;
    const uint64_t himask = pd.tmask & ~((uint64_t(1) << L) - 1);
    const uint32_t lowmask = (1u << L) - 1;
    const uint32_t tid = threadIdx.x, nth = blockDim.x;   // nth == tile / NB
    // register-group position of this thread (PassDesc::wmap)
    const uint32_t tmap = (pd.wmap && nth >= 64) ? (tid >> 5) | ((tid & 31u) << (31 - __clz(nth >> 5))) : tid;
    for (uint32_t h = tid; h < nhi; h += nth) offhi[h] = deposit_bits(h, himask);
    // the zero-slot count, read once per CTA (other CTAs update it)
    __shared__ uint32_t s_zc;
    if (tid == 0) s_zc = nzslot ? nzslot[uint64_t(1) << (nbits - cbits)] : 0u;
    __syncthreads();
    // tile bases: deposit(t) advanced by deposit(gridDim.x) with the carry
    // running through the tile-bit positions
    const uint64_t dstep = deposit_bits(gridDim.x, ntmask);
    uint64_t base = deposit_bits(blockIdx.x, ntmask);
    // known all-(+0) chunk slots: tiles made only of them are fixed points of
    // a pz_stable in-place pass (no load, no store)
    // the map is consulted / maintained only while it still holds zero slots
    if (s_zc == 0) nzslot = nullptr;
    const bool use_nz = nzslot && pd.pz_stable && src == dst && L <= cbits;
    for (uint64_t t = blockIdx.x; t < ntiles;
         t += gridDim.x, base = ((base | ~ntmask) + dstep) & ntmask) {
        if (use_nz) {
            uint32_t nzt = 0;
            for (uint32_t h = tid; h < nhi; h += nth) nzt |= nzslot[(base + offhi[h]) >> cbits];
            if (!__syncthreads_or(nzt)) {
                if (counters && tid == 0) atomicAdd(&counters[0], 1ull);
                continue;
            }
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const uint32_t l = tid + i * nth;
            cp_async16(s + swz(l), src + base + offhi[l >> L] + (l & lowmask));
        }
        cp_async_wait_all();
        __syncthreads();
        // tile census: any nonzero bit (all-(+0) skip) and "clean" = no -0,
        // tiny, inf or nan component (the fast path's precondition, then
        // kept by every group that stays on the fast path)
        unsigned long long any = 0;
        uint32_t okv = 1;
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const double2 x = s[swz(tid + i * nth)];
            any |= (unsigned long long)__double_as_longlong(x.x) |
                   (unsigned long long)__double_as_longlong(x.y);
            okv &= comp_ok(x.x) & comp_ok(x.y);
        }
        if (pd.pz_stable && !__syncthreads_or(any != 0)) {
            // an all-(+0) tile is a fixed point of the whole pass: skip it
            // (out of place: the output still needs the zeros)
            if (counters && tid == 0) atomicAdd(&counters[0], 1ull);
            if (src != dst) {
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    const uint32_t l = tid + i * nth;
                    __stcs(dst + base + offhi[l >> L] + (l & lowmask), make_double2(0.0, 0.0));
                }
            }
            continue;
        }
        bool clean = __syncthreads_and(okv) != 0;
        for (uint32_t gi = 0; gi < pd.ngroups; ++gi) {
            const GroupDesc &G = groups[pd.first_group + gi];
            const TileGate *gp = gates + G.first_gate;
            if (G.generic) {
                for (uint32_t q = 0; q < G.ngates; ++q) {
                    smem_generic(s, tile, gp[q]);
                    __syncthreads();
                }
                clean = false;
                continue;
            }
            uint32_t bm[kRegBits], gm = 0;
#pragma unroll
            for (int i = 0; i < kRegBits; ++i) {
                bm[i] = 1u << G.gbits[i];
                gm |= bm[i];
            }
            // thread id with zeros inserted at the (ascending) register bits
            // == deposit into the tile bits outside gm; under pd.wmap the
            // warp index takes the lowest of those bits
            uint32_t mybase = tmap;
#pragma unroll
            for (int i = 0; i < kRegBits; ++i) {
                const uint32_t b = G.gbits[i];
                mybase = ((mybase >> b) << (b + 1)) | (mybase & ((1u << b) - 1));
            }
            // buffer index of the thread's register-0 amplitude: the values of
            // every non-register bit (OP_PDIAG variants)
            const uint64_t gidx = G.relaxed ? base + offhi[mybase >> L] + (mybase & lowmask) : 0;
            uint32_t addr[NB];
#pragma unroll
            for (int r = 0; r < NB; ++r) {
                uint32_t a = mybase;
#pragma unroll
                for (int i = 0; i < kRegBits; ++i)
                    if ((r >> i) & 1) a |= bm[i];
                addr[r] = swz(a);
            }
            double2 v[NB];
#pragma unroll
            for (int r = 0; r < NB; ++r) v[r] = s[addr[r]];
            unsigned long long nz = 0, raw = 0;
#pragma unroll
            for (int r = 0; r < NB; ++r) {
                raw |= (unsigned long long)__double_as_longlong(v[r].x) |
                       (unsigned long long)__double_as_longlong(v[r].y);
                nz |= ((unsigned long long)__double_as_longlong(v[r].x) << 1) |
                      ((unsigned long long)__double_as_longlong(v[r].y) << 1);
            }
            int path = 1;
            if (raw == 0 && G.pz_stable) {
                // all-(+0) block, every gate keeps it all-(+0): nothing to do
            } else if (G.relaxed && nz == 0) {
                *flag = 1u;   // partner values outside the tile would be needed
            } else if (nz == 0) {
                path = 2;
                // all-zero block: stays zero, track the zero signs only
                uint32_t SR = 0, SI = 0;
#pragma unroll
                for (int r = 0; r < NB; ++r) {
                    SR |= sbit(v[r].x) << r;
                    SI |= sbit(v[r].y) << r;
                }
                for (uint32_t q = 0; q < G.ngates; ++q) mask_apply(SR, SI, gp[q]);
#pragma unroll
                for (int r = 0; r < NB; ++r)
                    v[r] = make_double2(signed_zero((SR >> r) & 1), signed_zero((SI >> r) & 1));
            } else {
                // fast path precondition: no -0 component and every nonzero
                // component in [2^-900, 2^1023] (no underflow, no inf/nan)
                uint32_t okg = 1;
                if (!clean) {
#pragma unroll
                    for (int r = 0; r < NB; ++r) okg &= comp_ok(v[r].x) & comp_ok(v[r].y);
                }
                const bool okblk = okg != 0;
                bool bad = !okblk;
                path = okblk ? 3 : 4;
                const TileGate *fp = gates + G.first_fast;
                for (uint32_t q = 0; q < G.nfast && !bad;) q += fast_case<S>(v, fp, q, gidx, bad);
                if (bad && okblk) path = 5;
                if (bad && G.relaxed) {
                    *flag = 1u;   // the exact path needs partners outside the tile
                } else if (bad) {
                    // a zero is (or became) present: redo the group exactly
#pragma unroll
                    for (int r = 0; r < NB; ++r) v[r] = s[addr[r]];
                    for (uint32_t q = 0; q < G.ngates; ++q) reg_apply(v, gp[q]);
                }
            }
            if (!(raw == 0 && G.pz_stable)) {
#pragma unroll
                for (int r = 0; r < NB; ++r) s[addr[r]] = v[r];
            }
            if (counters) atomicAdd(&counters[path], 1ull);
            // the sign-mask and exact paths may leave -0 behind
            clean = __syncthreads_and(path == 1 || path == 3) != 0;
        }
        double2 out[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) out[i] = s[swz(tid + i * nth)];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const uint32_t l = tid + i * nth;
            __stcs(dst + base + offhi[l >> L] + (l & lowmask), out[i]);
        }
        if (nzslot) {
            // every slot the tile covers (the low tile bits span 2^(L - cbits)
            // consecutive slots when L > cbits)
            const uint32_t span = L > cbits ? 1u << (L - cbits) : 1u;
            uint32_t *zcount = nzslot + (uint64_t(1) << (nbits - cbits));
            for (uint32_t i = tid; i < nhi * span; i += nth) {
                uint32_t *w = nzslot + ((base + offhi[i / span]) >> cbits) + (i % span);
                if (*w == 0 && atomicExch(w, 1u) == 0) atomicSub(zcount, 1u);
            }
        }
        __syncthreads();
    }
}

// PASS_SWAPS: a run of pairwise disjoint SWAPs applied as the bit permutation
// pi (an involution): psi'[j] = psi[pi(j)].  Each SWAP row is 1*v + 0*(others)
// (kernels.cpp:49-50), which equals v exactly unless v has a -0 component;
// a tile pair holding a -0 raises the replay flag instead.
// Tile = buffer bits S = {0..4} u pi({0..4}) (512 B contiguous segments on
// both the read and the write side); tiles pair up as (base, pi(base)) and
// one CTA moves both, in place.
constexpr uint32_t kSwapLow = 5;

__device__ __forceinline__ uint64_t permute_bits(uint64_t x, const uint8_t *perm, uint32_t nbits) {
    uint64_t y = 0;
    for (uint32_t b = 0; b < nbits; ++b) y |= ((x >> b) & 1) << perm[b];
    return y;
}

// smem slot of local index l in a swap tile: XOR the low 5 bits with the
// bit-reversed next 5, so the contiguous fill and the gather of a
// bit-reversal-type permutation (low <-> high tile bits, the QFT's swap
// network) both hit 8 distinct 16-byte bank groups per phase
__device__ __forceinline__ uint32_t swz10(uint32_t l) {
    return l ^ (__brev((l >> kSwapLow) & 31u) >> 27);
}

__global__ void __launch_bounds__(256) tile_swaps(const double2 *__restrict__ src, double2 *__restrict__ dst,
                                                  uint32_t nbits,
                                                  PassDesc pd, uint32_t *__restrict__ flag,
                                                  const uint32_t *__restrict__ cond) {
    if (cond && *cond == 0) return;
    constexpr uint32_t kMaxTile = 1u << (2 * kSwapLow);
    constexpr uint32_t kChunks = 8;   // tile index split in 5-bit chunks (<= 40 bits)
    __shared__ uint8_t perm[48];
    __shared__ uint16_t lperm[kMaxTile];
    __shared__ uint64_t loff[kMaxTile];
    __shared__ uint64_t dtab[kChunks][32], ptab[kChunks][32];   // deposit / permuted deposit
    __shared__ __align__(16) double2 ta[kMaxTile], tb[kMaxTile];
    const uint32_t tid = threadIdx.x, nth = blockDim.x;
    const uint32_t L = min(kSwapLow, nbits);
    uint64_t smask = (uint64_t(1) << L) - 1;
    for (uint32_t b = 0; b < L; ++b) smask |= uint64_t(1) << pd.perm[b];
    const uint32_t ks = __popcll(smask), tile = 1u << ks;
    const uint64_t cmask = ((uint64_t(1) << nbits) - 1) & ~smask;
    if (tid < 48) perm[tid] = pd.perm[tid];
    __syncthreads();
    // local bit permutation induced on S
    for (uint32_t l = tid; l < tile; l += nth) {
        const uint64_t off = deposit_bits(l, smask);
        const uint64_t img = permute_bits(off, perm, nbits);
        uint32_t li = 0, i = 0;
        for (uint64_t m = smask; m; m &= m - 1, ++i)
            if (img & (m & (0 - m))) li |= 1u << i;
        lperm[l] = uint16_t(li);
        loff[l] = off;
    }
    // tile index -> base / partner base, 5 index bits per table (GF(2)-linear)
    for (uint32_t e = tid; e < kChunks * 32; e += nth) {
        const uint32_t c = e >> 5, v = e & 31;
        const uint64_t dep = deposit_bits(uint64_t(v) << (5 * c), cmask);
        dtab[c][v] = dep;
        ptab[c][v] = permute_bits(dep, perm, nbits);
    }
    __syncthreads();
    const uint64_t ntiles = uint64_t(1) << (nbits - ks);
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        uint64_t base = 0, pbase = 0;
#pragma unroll
        for (uint32_t c = 0; c < kChunks; ++c) {
            const uint32_t v = uint32_t(t >> (5 * c)) & 31u;
            base |= dtab[c][v];
            pbase |= ptab[c][v];
        }
        if (pbase < base) continue;   // the partner tile's CTA moves this pair
        const bool pair = pbase != base;
        uint32_t neg0 = 0;
        // all loads of the pair issued before any is consumed (8 x 16 B per thread)
        constexpr uint32_t kPer = kMaxTile / 256;
        double2 ra[kPer], rb[kPer];
#pragma unroll
        for (uint32_t i = 0; i < kPer; ++i) {
            const uint32_t l = tid + i * nth;
            ra[i] = rb[i] = make_double2(0.0, 0.0);
            if (l < tile) {
                const uint64_t off = loff[l];
                ra[i] = __ldcs(src + base + off);
                if (pair) rb[i] = __ldcs(src + pbase + off);
            }
        }
#pragma unroll
        for (uint32_t i = 0; i < kPer; ++i) {
            const uint32_t l = tid + i * nth;
            if (l < tile) {
                ta[swz10(l)] = ra[i];
                tb[swz10(l)] = rb[i];
            }
            neg0 |= uint32_t(nz0(ra[i])) | uint32_t(nz0(rb[i]));
        }
        if (__syncthreads_or(neg0)) {
            if (tid == 0) *flag = 1u;
        }
#pragma unroll
        for (uint32_t i = 0; i < kPer; ++i) {
            const uint32_t l = tid + i * nth;
            if (l >= tile) break;
            const uint64_t off = loff[l];
            const uint32_t srcl = swz10(lperm[l]);
            if (pair) {
                __stcs(dst + base + off, tb[srcl]);
                __stcs(dst + pbase + off, ta[srcl]);
            } else {
                __stcs(dst + base + off, ta[srcl]);
            }
        }
        __syncthreads();
    }
}

// Buffers below 16 amplitudes: one thread, dense formula.
__global__ void tile_pass_tiny(double2 *buf, uint32_t nbits, PassDesc pd,
                               const GroupDesc *__restrict__ groups,
                               const TileGate *__restrict__ gates, const uint32_t *cond) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (cond && *cond == 0) return;
    const uint32_t n = 1u << nbits;
    for (uint32_t gi = 0; gi < pd.ngroups; ++gi)
    for (uint32_t q = 0; q < groups[pd.first_group + gi].ngates; ++q) {
        const TileGate &g = gates[groups[pd.first_group + gi].first_gate + q];
        if (g.nq == 1) {
            for (uint32_t p = 0; p < n / 2; ++p) {
                const uint32_t i = insert_zero_bit32(p, g.t0), j = i | (1u << g.t0);
                const double2 in[2] = {buf[i], buf[j]};
                buf[i] = full_row(g, 0, 2, in);
                buf[j] = full_row(g, 1, 2, in);
            }
        } else {
            const uint32_t lo = min(g.t0, g.t1), hi = max(g.t0, g.t1);
            const uint32_t s0 = 1u << g.t0, s1 = 1u << g.t1;
            for (uint32_t p = 0; p < n / 4; ++p) {
                const uint32_t b = insert_zero_bit32(insert_zero_bit32(p, lo), hi);
                const uint32_t idx[4] = {b, b | s1, b | s0, b | s0 | s1};
                const double2 in[4] = {buf[idx[0]], buf[idx[1]], buf[idx[2]], buf[idx[3]]};
                for (int r = 0; r < 4; ++r) buf[idx[r]] = full_row(g, r, 4, in);
            }
        }
    }
}

} // namespace

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
            QZ_CUDA(cudaMalloc(&ptr, 8 * 8));
            QZ_CUDA(cudaMemset(ptr, 0, 8 * 8));
        }
    }
    return ptr;
}

void dump_debug_counters() {
    unsigned long long *p = debug_counters();
    if (!p) return;
    unsigned long long h[8];
    QZ_CUDA(cudaMemcpy(h, p, sizeof h, cudaMemcpyDeviceToHost));
    fprintf(stderr, "qz counters: tiles_skipped=%llu grp_pz_skip=%llu grp_mask=%llu grp_fast=%llu "
                    "grp_exact=%llu grp_fast_then_exact=%llu\n",
            h[0], h[1], h[2], h[3], h[4], h[5]);
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

void launch_pass(const DevPlan &plan, const PassDesc &pd, const double2 *src, double2 *dst,
                 uint32_t nbits, cudaStream_t s, uint32_t *flag, const uint32_t *cond, NzMap nz,
                 uint32_t tag) {
    // replay launches (cond != nullptr) are device-side no-ops unless flagged:
    // they are not timed as passes
    static const char *const kName[3] = {"tile_pass_reg<All>", "tile_pass_reg<DiagH>", "tile_pass_reg<Gen>"};
    KProfScope prof(s, cond ? "replay_pass" : pd.kind == PASS_SWAPS ? "tile_swaps" : kName[pd.variant % 3],
                    tag, 32.0 * double(uint64_t(1) << nbits));
    if (pd.kind == PASS_SWAPS) {
        const uint64_t tiles = uint64_t(1) << (nbits > 2 * kSwapLow ? nbits - 2 * kSwapLow : 0);
        const uint64_t grid = std::min<uint64_t>(std::max<uint64_t>(tiles, 1), uint64_t(kNumSMs) * 8);
        tile_swaps<<<(unsigned)grid, 256, 0, s>>>(src, dst, nbits, pd, flag, cond);
        // chunks moved: the zero map no longer describes the slots
        if (nz.slot && nbits > nz.cbits) {
            const size_t ns = size_t(1) << (nbits - nz.cbits);
            QZ_CUDA(cudaMemsetAsync(nz.slot, 1, 4 * ns, s));
            QZ_CUDA(cudaMemsetAsync(nz.slot + ns, 0, 4, s));
        }
    } else if (pd.k < (uint32_t)kRegBits + 1) {
        // tile == whole buffer (nbits < 4): never relaxed, in place
        if (src != dst) throw Failure(QZC_EDEVICE, "tiny pass out of place");
        tile_pass_tiny<<<1, 32, 0, s>>>(dst, nbits, pd, plan.groups, plan.gates, cond);
    } else {
        const uint32_t tile = 1u << pd.k;
        const uint64_t ntiles = uint64_t(1) << (nbits - pd.k);
        const uint32_t threads = tile >> kRegBits;
        const size_t smem = sizeof(double2) * tile + sizeof(uint64_t) * (tile >> pd.lowbits);
        const uint64_t grid = std::min<uint64_t>(ntiles, uint64_t(kNumSMs) * 2 * 8);
        // the map is only used for passes inside one window of whole slots
        static const bool off = getenv("QZ_NO_NZMAP") != nullptr;
        const bool usable = nz.slot && nbits > nz.cbits && !off;
        auto kern = pd.variant == kPassDiagH ? tile_pass_reg<kPassDiagH>
                    : pd.variant == kPassGen ? tile_pass_reg<kPassGen>
                                             : tile_pass_reg<kPassAll>;
        kern<<<(unsigned)grid, threads, smem, s>>>(src, dst, nbits, pd, plan.groups, plan.gates, ntiles,
                                                   debug_counters(), flag, cond,
                                                   usable ? nz.slot : nullptr, nz.cbits);
    }
    QZ_CHECK_LAUNCH();
}

} // namespace

uint64_t run_passes(const DevPlan &plan, double2 *buf, uint32_t nbits, cudaStream_t s,
                    const uint32_t *cond, NzMap nz) {
    if (plan.relaxed) throw Failure(QZC_EDEVICE, "relaxed plan run without its replay plan");
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
