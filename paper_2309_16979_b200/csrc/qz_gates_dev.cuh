// qz_gates_dev.cuh — device side of the fused gate passes: exact register
// fast path, exact fallbacks, tile_pass_body and the AOT pass kernels.
// Included by qz_gates.cu inside namespace qz, and — with QZ_JIT_SOURCE
// defined — by the runtime-specialised pass sources qz_jit.cu builds with
// NVRTC (no standard library, no host code in here).
#pragma once

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
// zm (every op below): registers statically +0 at op entry (runtime-specialised
// passes over fresh qubits, qz_jit.cu; the op maps all-(+0) inputs to +0):
// their products are skipped.  A compile-time constant where it is nonzero.
template <int R, int K0 = -1, int K1 = -1, int SPEC = 0>
__device__ __forceinline__ void fast_diag(double2 (&v)[NB], const TileGate &g, bool &bad, uint32_t zm = 0) {
    constexpr int sh = 1 << R;
    const uint32_t k00 = uint32_t(g.kinds) & 15u, k11 = uint32_t(g.kinds >> 12) & 15u;
    const double2 m00 = g.m[0], m11 = g.m[3];
    const bool u0 = SPEC != 1 && !(g.srow & 1), u1 = SPEC != 1 && !(g.srow & 2);
#pragma unroll
    for (int p = 0; p < NB / 2; ++p) {
        const int i = izb(p, R), j = i | sh;
        const double2 a = v[i], b = v[j];
        // a zero in a row that is not +0-safe: that row's exact value
        if (K0 == CK_ONE || (K0 < 0 && k00 == CK_ONE) || ((zm >> i) & 1)) {
        } else {
            double2 o = termk<K0>(k00, m00, a);
            if (u0 && zc(o)) {
                o = slow2(g, 0, a, b);
                bad |= nz0(o);
            }
            v[i] = o;
        }
        if (K1 == CK_ONE || (K1 < 0 && k11 == CK_ONE) || ((zm >> j) & 1)) {
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
__device__ __forceinline__ void fast_gen1(double2 (&v)[NB], const TileGate &g, bool &bad, uint32_t zm = 0) {
    constexpr int sh = 1 << R;
    const uint32_t kd = uint32_t(g.kinds);
    const uint32_t k00 = kd & 15u, k01 = (kd >> 4) & 15u, k10 = (kd >> 8) & 15u, k11 = (kd >> 12) & 15u;
    const double2 m00 = g.m[0], m01 = g.m[1], m10 = g.m[2], m11 = g.m[3];
#pragma unroll
    for (int p = 0; p < NB / 2; ++p) {
        const int i = izb(p, R), j = i | sh;
        if ((zm >> i) & (zm >> j) & 1) continue;
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
__device__ __forceinline__ void fast_cz(double2 (&v)[NB], const TileGate &g, bool &bad, uint32_t zm = 0) {
#pragma unroll
    for (int i = 0; i < NB; ++i)
        if (((i >> A) & 1) && ((i >> B) & 1) && !((zm >> i) & 1)) {
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
__device__ __forceinline__ void fast_cp5(double2 (&v)[NB], const TileGate &g, bool &bad, uint32_t zm = 0) {
    const uint32_t k1 = uint32_t(g.kinds) & 15u, k2 = uint32_t(g.kinds >> 4) & 15u,
                   k3 = uint32_t(g.kinds >> 8) & 15u;
    const double2 m1 = g.m[0], m2 = g.m[1], m3 = g.m[2];
    const bool u1 = !SPEC && !(g.srow & 1), u2 = !SPEC && !(g.srow & 2), u3 = !SPEC && !(g.srow & 4);
    constexpr int KC = SPEC ? int(CK_CPLX) : -1;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        if (((i >> A) & 1) || ((i >> B) & 1)) continue;
        const int i01 = i | (1 << B), i10 = i | (1 << A), i11 = i | (1 << A) | (1 << B);
        if (!((zm >> i01) & 1)) {
            double2 x01 = termk<KC>(k2, m2, v[i01]);
            if (u2) bad |= zc(x01);
            x01 = termk<KC>(k3, m3, x01);
            if (u3) bad |= zc(x01);
            v[i01] = x01;
        }
        if (!((zm >> i10) & 1)) {
            double2 x10 = termk<KC>(k1, m1, v[i10]);
            if (u1) bad |= zc(x10);
            x10 = termk<KC>(k2, m2, x10);
            if (u2) bad |= zc(x10);
            v[i10] = x10;
        }
        if (!((zm >> i11) & 1)) {
            double2 x11 = termk<KC>(k1, m1, v[i11]);
            if (u1) bad |= zc(x11);
            x11 = termk<KC>(k3, m3, x11);
            if (u3) bad |= zc(x11);
            v[i11] = x11;
        }
    }
}

// CXD on (A, B), D = diag(d0, d1) on B: p00 <- d0 v00, p01 <- d1 v01,
// p10 <- d1 v10, p11 <- d0 v11.
template <int A, int B, int SPEC = 0>
__device__ __forceinline__ void fast_cxd(double2 (&v)[NB], const TileGate &g, bool &bad, uint32_t zm = 0) {
    const uint32_t k0 = uint32_t(g.kinds) & 15u, k1 = uint32_t(g.kinds >> 4) & 15u;
    const double2 d0 = g.m[0], d1 = g.m[1];
    const bool u0 = !SPEC && !(g.srow & 1), u1 = !SPEC && !(g.srow & 2);
    constexpr int KC = SPEC ? int(CK_CPLX) : -1;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        if (((i >> A) & 1) || ((i >> B) & 1)) continue;
        const int i01 = i | (1 << B), i10 = i | (1 << A), i11 = i | (1 << A) | (1 << B);
        if (!((zm >> i) & 1)) {
            const double2 x00 = termk<KC>(k0, d0, v[i]);
            if (u0) bad |= zc(x00);
            v[i] = x00;
        }
        if (!((zm >> i01) & 1)) {
            const double2 x01 = termk<KC>(k1, d1, v[i01]);
            if (u1) bad |= zc(x01);
            v[i01] = x01;
        }
        if (!((zm >> i10) & 1)) {
            const double2 x10 = termk<KC>(k1, d1, v[i10]);
            if (u1) bad |= zc(x10);
            v[i10] = x10;
        }
        if (!((zm >> i11) & 1)) {
            const double2 x11 = termk<KC>(k0, d0, v[i11]);
            if (u0) bad |= zc(x11);
            v[i11] = x11;
        }
    }
}

// OP_PDIAG resolved for this tile's outside-bit values `var`: step chains on
// register bit R (R == kRegBits: one chain for the whole block).
// SPEC = 1: every step CPLX and +0-safe (no kind branches, no checks).
template <int R, int SPEC = 0>
__device__ __forceinline__ void fast_pdiag(double2 (&v)[NB], const TileGate &g, uint32_t var,
                                           bool &bad, uint32_t zm = 0) {
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
                if ((zm >> i) & 1) continue;
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
                                           uint32_t act, uint32_t zm = 0) {
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
                if ((zm >> i) & 1) continue;
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
                                            uint32_t n, uint64_t gidx, uint32_t zm = 0) {
    for (uint32_t q = 0; q < n; ++q) {
        const TileGate &g = gp[q];
        const uint32_t var = pdiag_var(g, gidx);
        const uint32_t act = (g.steps >> (4 * var)) & 15u;
        if (R == kRegBits || g.nq == 0) pdiag_spec<kRegBits>(v, g.m + 4 * var, act, zm);
        else pdiag_spec<R>(v, g.m + 4 * var, act, zm);
    }
}

// Fast-path op bodies by case id (host case_id()); the AOT kernels reach
// them through fast_case's switch, the runtime-specialised passes call
// them directly in the plan's order.
template <int C>
__device__ __forceinline__ uint32_t fast_cid(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q,
                                             uint64_t gidx, bool &bad, uint32_t zm = 0);
template <> __device__ __forceinline__ uint32_t fast_cid<0>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; run_pdiag_r<0>(v, fp + q, g.run, gidx, zm); return g.run;
}
template <> __device__ __forceinline__ uint32_t fast_cid<1>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; run_pdiag_r<1>(v, fp + q, g.run, gidx, zm); return g.run;
}
template <> __device__ __forceinline__ uint32_t fast_cid<2>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; run_pdiag_r<2>(v, fp + q, g.run, gidx, zm); return g.run;
}
template <> __device__ __forceinline__ uint32_t fast_cid<3>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; run_pdiag_r<3>(v, fp + q, g.run, gidx, zm); return g.run;
}
template <> __device__ __forceinline__ uint32_t fast_cid<4>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_pdiag<0, 0>(v, g, pdiag_var(g, gidx), bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<5>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_pdiag<0, 1>(v, g, pdiag_var(g, gidx), bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<6>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_pdiag<1, 0>(v, g, pdiag_var(g, gidx), bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<7>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_pdiag<1, 1>(v, g, pdiag_var(g, gidx), bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<8>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_pdiag<2, 0>(v, g, pdiag_var(g, gidx), bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<9>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_pdiag<2, 1>(v, g, pdiag_var(g, gidx), bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<10>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_pdiag<3, 0>(v, g, pdiag_var(g, gidx), bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<11>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_pdiag<3, 1>(v, g, pdiag_var(g, gidx), bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<12>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<0, CK_ONE, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<13>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<0, CK_CPLX, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<14>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<0, CK_ONE, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<15>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<0, CK_CPLX, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<16>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<0>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<17>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<1, CK_ONE, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<18>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<1, CK_CPLX, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<19>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<1, CK_ONE, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<20>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<1, CK_CPLX, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<21>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<22>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<2, CK_ONE, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<23>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<2, CK_CPLX, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<24>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<2, CK_ONE, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<25>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<2, CK_CPLX, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<26>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_diag<2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<27>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<28>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<29>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<30>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<31>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<32>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<33>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<34>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<35>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<36>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<37>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<38>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<39>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<40>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<41>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<0>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<42>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<43>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<44>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<45>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<46>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<47>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<48>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<49>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<50>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<51>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<52>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<53>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<54>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<55>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<56>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<57>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<58>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<59>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<60>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_REAL, CK_IMAG, CK_IMAG, CK_REAL, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<61>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_REAL, CK_REAL, CK_REAL, CK_REAL, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<62>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_CPLX, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<63>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<64>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<65>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<66>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<67>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_ZERO, CK_ONE, CK_ONE, CK_ZERO, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<68>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_ZERO, CK_IMAG, CK_IMAG, CK_ZERO, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<69>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_REAL, CK_CPLX, CK_CPLX, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<70>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2, CK_REAL, CK_CPLX, CK_REAL, CK_CPLX, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<71>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_gen1<2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<72>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<0, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<73>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<0, 1, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<74>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<0, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<75>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<0, 2, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<76>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<1, 0>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<77>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<1, 0, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<78>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<1, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<79>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<1, 2, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<80>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<2, 0>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<81>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<2, 0, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<82>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<2, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<83>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cp5<2, 1, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<84>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<0, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<85>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<0, 1, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<86>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<0, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<87>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<0, 2, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<88>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<1, 0>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<89>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<1, 0, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<90>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<1, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<91>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<1, 2, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<92>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<2, 0>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<93>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<2, 0, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<94>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<2, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<95>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cxd<2, 1, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<96>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; (void)zm; fast_cx<0, 1>(v); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<97>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; (void)zm; fast_cx<0, 2>(v); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<98>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; (void)zm; fast_cx<1, 0>(v); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<99>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; (void)zm; fast_cx<1, 2>(v); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<100>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; (void)zm; fast_cx<2, 0>(v); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<101>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; (void)zm; fast_cx<2, 1>(v); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<102>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cz<0, 1>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<103>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cz<0, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<104>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; fast_cz<1, 2>(v, g, bad, zm); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<105>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; (void)zm; fast_swap<0, 1>(v); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<106>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; (void)zm; fast_swap<0, 2>(v); return 1;
}
template <> __device__ __forceinline__ uint32_t fast_cid<107>(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q, uint64_t gidx, bool &bad, uint32_t zm) {
    const TileGate &g = fp[q]; (void)g; (void)gidx; (void)bad; (void)zm; fast_swap<1, 2>(v); return 1;
}

template <int S>
__device__ __forceinline__ uint32_t fast_case(double2 (&v)[NB], const TileGate *__restrict__ fp, uint32_t q,
                                              uint64_t gidx, bool &bad) {
    switch (fp[q].cid) {
    case 0: if constexpr (case_on(S, 0)) return fast_cid<0>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 1: if constexpr (case_on(S, 1)) return fast_cid<1>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 2: if constexpr (case_on(S, 2)) return fast_cid<2>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 3: if constexpr (case_on(S, 3)) return fast_cid<3>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 4: if constexpr (case_on(S, 4)) return fast_cid<4>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 5: if constexpr (case_on(S, 5)) return fast_cid<5>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 6: if constexpr (case_on(S, 6)) return fast_cid<6>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 7: if constexpr (case_on(S, 7)) return fast_cid<7>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 8: if constexpr (case_on(S, 8)) return fast_cid<8>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 9: if constexpr (case_on(S, 9)) return fast_cid<9>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 10: if constexpr (case_on(S, 10)) return fast_cid<10>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 11: if constexpr (case_on(S, 11)) return fast_cid<11>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 12: if constexpr (case_on(S, 12)) return fast_cid<12>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 13: if constexpr (case_on(S, 13)) return fast_cid<13>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 14: if constexpr (case_on(S, 14)) return fast_cid<14>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 15: if constexpr (case_on(S, 15)) return fast_cid<15>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 16: if constexpr (case_on(S, 16)) return fast_cid<16>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 17: if constexpr (case_on(S, 17)) return fast_cid<17>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 18: if constexpr (case_on(S, 18)) return fast_cid<18>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 19: if constexpr (case_on(S, 19)) return fast_cid<19>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 20: if constexpr (case_on(S, 20)) return fast_cid<20>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 21: if constexpr (case_on(S, 21)) return fast_cid<21>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 22: if constexpr (case_on(S, 22)) return fast_cid<22>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 23: if constexpr (case_on(S, 23)) return fast_cid<23>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 24: if constexpr (case_on(S, 24)) return fast_cid<24>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 25: if constexpr (case_on(S, 25)) return fast_cid<25>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 26: if constexpr (case_on(S, 26)) return fast_cid<26>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 27: if constexpr (case_on(S, 27)) return fast_cid<27>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 28: if constexpr (case_on(S, 28)) return fast_cid<28>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 29: if constexpr (case_on(S, 29)) return fast_cid<29>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 30: if constexpr (case_on(S, 30)) return fast_cid<30>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 31: if constexpr (case_on(S, 31)) return fast_cid<31>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 32: if constexpr (case_on(S, 32)) return fast_cid<32>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 33: if constexpr (case_on(S, 33)) return fast_cid<33>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 34: if constexpr (case_on(S, 34)) return fast_cid<34>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 35: if constexpr (case_on(S, 35)) return fast_cid<35>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 36: if constexpr (case_on(S, 36)) return fast_cid<36>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 37: if constexpr (case_on(S, 37)) return fast_cid<37>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 38: if constexpr (case_on(S, 38)) return fast_cid<38>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 39: if constexpr (case_on(S, 39)) return fast_cid<39>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 40: if constexpr (case_on(S, 40)) return fast_cid<40>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 41: if constexpr (case_on(S, 41)) return fast_cid<41>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 42: if constexpr (case_on(S, 42)) return fast_cid<42>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 43: if constexpr (case_on(S, 43)) return fast_cid<43>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 44: if constexpr (case_on(S, 44)) return fast_cid<44>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 45: if constexpr (case_on(S, 45)) return fast_cid<45>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 46: if constexpr (case_on(S, 46)) return fast_cid<46>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 47: if constexpr (case_on(S, 47)) return fast_cid<47>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 48: if constexpr (case_on(S, 48)) return fast_cid<48>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 49: if constexpr (case_on(S, 49)) return fast_cid<49>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 50: if constexpr (case_on(S, 50)) return fast_cid<50>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 51: if constexpr (case_on(S, 51)) return fast_cid<51>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 52: if constexpr (case_on(S, 52)) return fast_cid<52>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 53: if constexpr (case_on(S, 53)) return fast_cid<53>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 54: if constexpr (case_on(S, 54)) return fast_cid<54>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 55: if constexpr (case_on(S, 55)) return fast_cid<55>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 56: if constexpr (case_on(S, 56)) return fast_cid<56>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 57: if constexpr (case_on(S, 57)) return fast_cid<57>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 58: if constexpr (case_on(S, 58)) return fast_cid<58>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 59: if constexpr (case_on(S, 59)) return fast_cid<59>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 60: if constexpr (case_on(S, 60)) return fast_cid<60>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 61: if constexpr (case_on(S, 61)) return fast_cid<61>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 62: if constexpr (case_on(S, 62)) return fast_cid<62>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 63: if constexpr (case_on(S, 63)) return fast_cid<63>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 64: if constexpr (case_on(S, 64)) return fast_cid<64>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 65: if constexpr (case_on(S, 65)) return fast_cid<65>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 66: if constexpr (case_on(S, 66)) return fast_cid<66>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 67: if constexpr (case_on(S, 67)) return fast_cid<67>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 68: if constexpr (case_on(S, 68)) return fast_cid<68>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 69: if constexpr (case_on(S, 69)) return fast_cid<69>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 70: if constexpr (case_on(S, 70)) return fast_cid<70>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 71: if constexpr (case_on(S, 71)) return fast_cid<71>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 72: if constexpr (case_on(S, 72)) return fast_cid<72>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 73: if constexpr (case_on(S, 73)) return fast_cid<73>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 74: if constexpr (case_on(S, 74)) return fast_cid<74>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 75: if constexpr (case_on(S, 75)) return fast_cid<75>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 76: if constexpr (case_on(S, 76)) return fast_cid<76>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 77: if constexpr (case_on(S, 77)) return fast_cid<77>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 78: if constexpr (case_on(S, 78)) return fast_cid<78>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 79: if constexpr (case_on(S, 79)) return fast_cid<79>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 80: if constexpr (case_on(S, 80)) return fast_cid<80>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 81: if constexpr (case_on(S, 81)) return fast_cid<81>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 82: if constexpr (case_on(S, 82)) return fast_cid<82>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 83: if constexpr (case_on(S, 83)) return fast_cid<83>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 84: if constexpr (case_on(S, 84)) return fast_cid<84>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 85: if constexpr (case_on(S, 85)) return fast_cid<85>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 86: if constexpr (case_on(S, 86)) return fast_cid<86>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 87: if constexpr (case_on(S, 87)) return fast_cid<87>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 88: if constexpr (case_on(S, 88)) return fast_cid<88>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 89: if constexpr (case_on(S, 89)) return fast_cid<89>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 90: if constexpr (case_on(S, 90)) return fast_cid<90>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 91: if constexpr (case_on(S, 91)) return fast_cid<91>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 92: if constexpr (case_on(S, 92)) return fast_cid<92>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 93: if constexpr (case_on(S, 93)) return fast_cid<93>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 94: if constexpr (case_on(S, 94)) return fast_cid<94>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 95: if constexpr (case_on(S, 95)) return fast_cid<95>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 96: if constexpr (case_on(S, 96)) return fast_cid<96>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 97: if constexpr (case_on(S, 97)) return fast_cid<97>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 98: if constexpr (case_on(S, 98)) return fast_cid<98>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 99: if constexpr (case_on(S, 99)) return fast_cid<99>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 100: if constexpr (case_on(S, 100)) return fast_cid<100>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 101: if constexpr (case_on(S, 101)) return fast_cid<101>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 102: if constexpr (case_on(S, 102)) return fast_cid<102>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 103: if constexpr (case_on(S, 103)) return fast_cid<103>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 104: if constexpr (case_on(S, 104)) return fast_cid<104>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 105: if constexpr (case_on(S, 105)) return fast_cid<105>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 106: if constexpr (case_on(S, 106)) return fast_cid<106>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    case 107: if constexpr (case_on(S, 107)) return fast_cid<107>(v, fp, q, gidx, bad); else { bad = true; return 1; }
    default: bad = true; return 1;   // other 2q matrices: exact path only
    }
}

// The AOT fast-list interpreter: group gi's fast ops through the switch.
template <int S>
struct FastInterp {
    static __device__ __forceinline__ void run(uint32_t gi, const TileGate *__restrict__ fp, uint32_t nfast,
                                               double2 (&v)[NB], uint64_t gidx, bool &bad) {
        (void)gi;
        for (uint32_t q = 0; q < nfast && !bad;) q += fast_case<S>(v, fp, q, gidx, bad);
    }
};

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

// Image of the bit set x under a bit permutation (PassDesc::perm).
__device__ __forceinline__ uint64_t permute_bits(uint64_t x, const uint8_t (&perm)[48]) {
    uint64_t r = 0;
    while (x) {
        const uint32_t b = __ffsll((long long)x) - 1;
        x &= x - 1;
        r |= uint64_t(1) << perm[b];
    }
    return r;
}


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
template <int S, class FP>
__device__ __forceinline__ void tile_pass_body(const double2 *__restrict__ src, double2 *__restrict__ dst, uint32_t nbits,
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
    // permuted store (PassDesc::permute): the output tile spans perm(T); it
    // is written in output order (runs of 2^Lo contiguous elements), element
    // l_out taken from tile slot lmap[l_out]
    uint64_t *offo = offhi + nhi;
    uint16_t *lmap = nullptr;
    uint32_t Lo = 0;
    if (pd.permute) {
        const uint64_t otmask = permute_bits(pd.tmask, pd.perm);
        while (Lo < k && ((otmask >> Lo) & 1)) ++Lo;
        const uint64_t ohimask = otmask & ~((uint64_t(1) << Lo) - 1);
        lmap = reinterpret_cast<uint16_t *>(offo + (1u << (k - Lo)));
        for (uint32_t h = tid; h < (1u << (k - Lo)); h += nth) offo[h] = deposit_bits(h, ohimask);
        // output tile bit j (ascending in perm(T)) is input tile bit rank[j]
        uint32_t rank[16];
        {
            uint64_t om = otmask;
            for (uint32_t j = 0; j < k; ++j) {
                const uint32_t ob = __ffsll((long long)om) - 1;
                om &= om - 1;
                const uint32_t ib = pd.perm[ob];
                rank[j] = __popcll(pd.tmask & ((uint64_t(1) << ib) - 1));
            }
        }
        for (uint32_t l = tid; l < tile; l += nth) {
            uint32_t li = 0;
            for (uint32_t j = 0; j < k; ++j) li |= ((l >> j) & 1u) << rank[j];
            lmap[l] = uint16_t(li);
        }
    }
    const uint32_t lomask = (1u << Lo) - 1;
    // the zero-slot count, read once per CTA (other CTAs update it)
    __shared__ uint32_t s_zc;
    if (tid == 0) s_zc = nzslot ? nzslot[uint64_t(1) << (nbits - cbits)] : 0u;
    __syncthreads();
    // live tiles only: those on the nonzero side of the pass's fresh outside
    // bits (the others are all +0 and stay so: pz_stable, in place)
    const bool zskip = pd.zmask && pd.pz_stable && src == dst;
    const uint64_t ltmask = zskip ? ntmask & ~pd.zmask : ntmask;
    const uint64_t zv = zskip ? pd.zval : 0;
    if (zskip) ntiles >>= __popcll(pd.zmask);
    // tile bases: deposit(t) advanced by deposit(gridDim.x) with the carry
    // running through the tile-bit positions
    const uint64_t dstep = deposit_bits(gridDim.x, ltmask);
    uint64_t base = deposit_bits(blockIdx.x, ltmask) | zv;
    // known all-(+0) chunk slots: tiles made only of them are fixed points of
    // a pz_stable in-place pass (no load, no store)
    // the map is consulted / maintained only while it still holds zero slots
    if (s_zc == 0) nzslot = nullptr;
    // fresh bits inside the tile: elements this pass may open are not yet in
    // the window, so every visited tile is stored (no skip without a store)
    const bool opens = (pd.fmask & pd.tmask) != 0;
    const bool use_nz = nzslot && pd.pz_stable && src == dst && L <= cbits && !opens;
    if (pd.direct) {
        // register-direct pass (PassDesc::direct): the single group's block
        // of 8 amplitudes per thread comes straight from global memory
        const GroupDesc &G = groups[pd.first_group];
        const TileGate *gp = gates + G.first_gate;
        uint32_t mybase = tid;   // plain map: lanes on the lowest non-register tile bits
#pragma unroll
        for (int i = 0; i < kRegBits; ++i) {
            const uint32_t b = G.gbits[i];
            mybase = ((mybase >> b) << (b + 1)) | (mybase & ((1u << b) - 1));
        }
        uint32_t lidx[NB];
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            uint32_t a = mybase;
#pragma unroll
            for (int i = 0; i < kRegBits; ++i)
                if ((r >> i) & 1) a |= 1u << G.gbits[i];
            lidx[r] = a;
        }
        const uint32_t span = L > cbits ? 1u << (L - cbits) : 1u;
        for (uint64_t t = blockIdx.x; t < ntiles;
             t += gridDim.x, base = ((((base & ~zv) | ~ltmask) + dstep) & ltmask) | zv) {
            uint64_t ea[NB];
            double2 v[NB];
#pragma unroll
            for (int r = 0; r < NB; ++r) {
                ea[r] = base + offhi[lidx[r] >> L] + (lidx[r] & lowmask);
                v[r] = (ea[r] & pd.fmask) != pd.fval ? make_double2(0.0, 0.0) : src[ea[r]];
            }
            const uint64_t gidx = G.relaxed ? base + offhi[mybase >> L] + (mybase & lowmask) : 0;
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
            } else if (G.relaxed && nz == 0) {
                *flag = 1u;
            } else if (nz == 0) {
                path = 2;
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
                uint32_t okg = 1;
#pragma unroll
                for (int r = 0; r < NB; ++r) okg &= comp_ok(v[r].x) & comp_ok(v[r].y);
                const bool okblk = okg != 0;
                bool bad = !okblk;
                path = okblk ? 3 : 4;
                FP::run(0, gates + G.first_fast, G.nfast, v, gidx, bad);
                if (bad && okblk) path = 5;
                if (bad && G.relaxed) {
                    *flag = 1u;
                } else if (bad) {
#pragma unroll
                    for (int r = 0; r < NB; ++r)
                        v[r] = (ea[r] & pd.fmask) != pd.fval ? make_double2(0.0, 0.0) : src[ea[r]];
                    for (uint32_t q = 0; q < G.ngates; ++q) reg_apply(v, gp[q]);
                }
            }
            if (!(raw == 0 && G.pz_stable) || opens || src != dst) {
#pragma unroll
                for (int r = 0; r < NB; ++r) __stcs(dst + ea[r], v[r]);
            }
#ifndef QZ_GROUP_CLOCKS
            if (counters) atomicAdd(&counters[path], 1ull);
#endif
            if (nzslot) {
                uint32_t *zcount = nzslot + (uint64_t(1) << (nbits - cbits));
                for (uint32_t i = tid; i < nhi * span; i += nth) {
                    uint32_t *w = nzslot + ((base + offhi[i / span]) >> cbits) + (i % span);
                    if (*w == 0 && atomicExch(w, 1u) == 0) atomicSub(zcount, 1u);
                }
            }
        }
        return;
    }
    for (uint64_t t = blockIdx.x; t < ntiles;
         t += gridDim.x, base = ((((base & ~zv) | ~ltmask) + dstep) & ltmask) | zv) {
        if (use_nz) {
            uint32_t nzt = 0;
            for (uint32_t h = tid; h < nhi; h += nth) nzt |= nzslot[(base + offhi[h]) >> cbits];
            if (!__syncthreads_or(nzt)) {
                if (counters && tid == 0) atomicAdd(&counters[0], 1ull);
                continue;
            }
        }
#ifdef QZ_GROUP_CLOCKS
        const long long ck_t0 = clock64();
#endif
        uint32_t loaded = 0;   // elements this thread loads (the others are statically +0)
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const uint32_t l = tid + i * nth;
            const uint64_t e = base + offhi[l >> L] + (l & lowmask);
            if ((e & pd.fmask) != pd.fval) {
                s[swz(l)] = make_double2(0.0, 0.0);
            } else {
                cp_async16(s + swz(l), src + e);
                loaded |= 1u << i;
            }
#ifdef QZ_COUNT_FILL
            if (counters) atomicAdd(&counters[((e & pd.fmask) != pd.fval) ? 6 : 7], 1ull);
#endif
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
            if (!((loaded >> i) & 1)) continue;   // a zero-filled +0: clean, zero
            const double2 x = s[swz(tid + i * nth)];
            any |= (unsigned long long)__double_as_longlong(x.x) |
                   (unsigned long long)__double_as_longlong(x.y);
            okv &= comp_ok(x.x) & comp_ok(x.y);
        }
        if (pd.pz_stable && !__syncthreads_or(any != 0)) {
            // an all-(+0) tile is a fixed point of the whole pass: skip it
            // (out of place: the output still needs the zeros)
            if (counters && tid == 0) atomicAdd(&counters[0], 1ull);
            if (src != dst || opens) {
                const uint64_t pbase = pd.permute ? permute_bits(base, pd.perm) : 0;
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    const uint32_t l = tid + i * nth;
                    __stcs(pd.permute ? dst + pbase + offo[l >> Lo] + (l & lomask)
                                      : dst + base + offhi[l >> L] + (l & lowmask),
                           make_double2(0.0, 0.0));
                }
            }
            continue;
        }
        bool clean = __syncthreads_and(okv) != 0;
#ifdef QZ_GROUP_CLOCKS
        // inspection: CTA time per phase (thread 0's view, barrier to barrier)
        // counters[8] load+census, [9 + gi] group gi, [15] store
        long long ck = clock64();
        if (counters && tid == 0) atomicAdd(&counters[8], (unsigned long long)(ck - ck_t0));
#endif
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
                FP::run(gi, gates + G.first_fast, G.nfast, v, gidx, bad);
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
#ifndef QZ_GROUP_CLOCKS
            if (counters) atomicAdd(&counters[path], 1ull);
#endif
            // the sign-mask and exact paths may leave -0 behind
            clean = __syncthreads_and(path == 1 || path == 3) != 0;
#ifdef QZ_GROUP_CLOCKS
            {
                const long long c2 = clock64();
                if (counters && tid == 0) atomicAdd(&counters[9 + (gi < 6 ? gi : 5)], (unsigned long long)(c2 - ck));
                ck = c2;
            }
#endif
        }
        double2 out[NB];
        if (pd.permute) {
            const uint64_t pbase = permute_bits(base, pd.perm);
#pragma unroll
            for (int i = 0; i < NB; ++i) out[i] = s[swz(lmap[tid + i * nth])];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const uint32_t l = tid + i * nth;
                __stcs(dst + pbase + offo[l >> Lo] + (l & lomask), out[i]);
            }
        } else {
#pragma unroll
            for (int i = 0; i < NB; ++i) out[i] = s[swz(tid + i * nth)];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const uint32_t l = tid + i * nth;
                __stcs(dst + base + offhi[l >> L] + (l & lowmask), out[i]);
            }
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
#ifdef QZ_GROUP_CLOCKS
        if (counters && tid == 0) atomicAdd(&counters[15], (unsigned long long)(clock64() - ck));
#endif
    }
}

template <int S>
__global__ void __launch_bounds__(1 << (kTileBits - kRegBits), (kTileBits >= 12 ? 1 : QZ_MIN_CTAS))
tile_pass_reg(const double2 *__restrict__ src, double2 *__restrict__ dst, uint32_t nbits, PassDesc pd,
              const GroupDesc *__restrict__ groups, const TileGate *__restrict__ gates, uint64_t ntiles,
              unsigned long long *__restrict__ counters, uint32_t *__restrict__ flag,
              const uint32_t *__restrict__ cond, uint32_t *__restrict__ nzslot, uint32_t cbits) {
    tile_pass_body<S, FastInterp<S>>(src, dst, nbits, pd, groups, gates, ntiles, counters, flag, cond, nzslot,
                                     cbits);
}

#ifndef QZ_JIT_SOURCE
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

#endif  // QZ_JIT_SOURCE

} // namespace
