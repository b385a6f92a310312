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
#include <complex>
#include <cstring>

#include "qz_gates.cuh"

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

static bool is_zero(double2 v) { return v.x == 0.0 && v.y == 0.0; }

DevGate make_dev_gate(const qzc_gate &g) {
    DevGate d;
    std::memset(&d, 0, sizeof d);
    uint32_t dim = 0;
    gate_matrix_host(g, d.m, &dim);
    d.nq = dim == 2 ? 1 : 2;
    d.b0 = g.qubits[0];
    d.b1 = d.nq == 2 ? g.qubits[1] : 0;
    d.cls = GC_DENSE;
    if (d.nq == 1) {
        if (is_zero(d.m[1]) && is_zero(d.m[2])) d.cls = GC_DIAG;
        else if (is_zero(d.m[0]) && is_zero(d.m[3])) d.cls = GC_ANTI;
    } else {
        bool perm = true;
        for (int r = 0; r < 4 && perm; ++r) {
            int nz = 0;
            for (int c = 0; c < 4; ++c) nz += !is_zero(d.m[r * 4 + c]);
            perm = nz == 1;
        }
        if (perm) {
            // bits 8.. hold the nonzero column of each row (2 bits per row)
            uint32_t cols = 0;
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c)
                    if (!is_zero(d.m[r * 4 + c])) cols |= uint32_t(c) << (2 * r);
            d.cls = GC_PERM4 | (cols << 8);
        }
    }
    return d;
}

// ------------------------------------------------------------- pass builder --

GatePlan build_passes(const std::vector<DevGate> &gates, uint32_t nbits,
                      uint32_t kmax, bool fuse) {
    GatePlan plan;
    const uint32_t k = std::min(kmax, nbits);
    const uint32_t low = std::min<uint32_t>(3, k);
    const uint64_t low_mask = (uint64_t(1) << low) - 1;
    auto bits_of = [](const DevGate &g) {
        uint64_t m = uint64_t(1) << g.b0;
        if (g.nq == 2) m |= uint64_t(1) << g.b1;
        return m;
    };
    std::vector<size_t> members;
    uint64_t tmask = low_mask;
    auto close = [&]() {
        if (members.empty()) return;
        // pad T to exactly k bits with the lowest free bits (longer
        // contiguous runs, better coalescing)
        for (uint32_t b = 0; b < nbits && (uint32_t)__builtin_popcountll(tmask) < k; ++b)
            tmask |= uint64_t(1) << b;
        PassDesc pd;
        pd.k = k;
        uint32_t lowbits = 0;
        while (lowbits < 64 && ((tmask >> lowbits) & 1)) ++lowbits;
        pd.lowbits = std::min(lowbits, k);
        pd.first_gate = (uint32_t)plan.gates.size();
        pd.ngates = (uint32_t)members.size();
        pd.tmask = tmask;
        // local position of buffer bit b inside T
        auto local = [&](uint32_t b) {
            return (uint32_t)__builtin_popcountll(tmask & ((uint64_t(1) << b) - 1));
        };
        for (size_t i : members) {
            const DevGate &g = gates[i];
            TileGate t;
            t.nq = g.nq;
            t.t0 = local(g.b0);
            t.t1 = g.nq == 2 ? local(g.b1) : 0;
            t.cls = g.cls;
            std::memcpy(t.m, g.m, sizeof t.m);
            plan.gates.push_back(t);
        }
        plan.passes.push_back(pd);
        members.clear();
        tmask = low_mask;
    };
    for (size_t i = 0; i < gates.size(); ++i) {
        const uint64_t need = bits_of(gates[i]);
        if (need >> nbits) throw Failure(QZC_EDEVICE, "gate bit outside buffer");
        const uint64_t merged = tmask | need;
        if (!fuse || (uint32_t)__builtin_popcountll(merged) > k) close();
        tmask |= need;
        members.push_back(i);
    }
    close();
    return plan;
}

void upload_plan(const GatePlan &plan, DevPlan &out, cudaStream_t s) {
    free_plan(out);
    out.npasses = plan.passes.size();
    out.ngates = plan.gates.size();
    out.host_passes = plan.passes;
    if (out.ngates) {
        QZ_CUDA(cudaMalloc(&out.gates, sizeof(TileGate) * out.ngates));
        QZ_CUDA(cudaMemcpyAsync(out.gates, plan.gates.data(), sizeof(TileGate) * out.ngates,
                                cudaMemcpyHostToDevice, s));
    }
}

void free_plan(DevPlan &p) {
    if (p.gates) cudaFree(p.gates);
    if (p.passes) cudaFree(p.passes);
    p.gates = nullptr;
    p.passes = nullptr;
    p.npasses = p.ngates = 0;
    p.host_passes.clear();
}

// ------------------------------------------------------------ tile kernel --

namespace {

__device__ __forceinline__ double2 to2(cplx c) { return make_double2(c.re, c.im); }

__device__ __forceinline__ bool has_zero(cplx c) { return c.re == 0.0 || c.im == 0.0; }

// Dense 1q formula: out = m_r0*a + m_r1*b (kernels.cpp:31-32).
__device__ __forceinline__ cplx row2(const double2 *m, int r, double2 a, double2 b) {
    cplx x = cmul(m[2 * r].x, m[2 * r].y, a);
    cplx y = cmul(m[2 * r + 1].x, m[2 * r + 1].y, b);
    return cplx{__dadd_rn(x.re, y.re), __dadd_rn(x.im, y.im)};
}

// Dense 4x4 row: ((m0*i0 + m1*i1) + m2*i2) + m3*i3 (kernels.cpp:49-50).
__device__ __forceinline__ cplx row4(const double2 *m, int r, const double2 *in) {
    cplx acc = cmul(m[4 * r].x, m[4 * r].y, in[0]);
#pragma unroll
    for (int c = 1; c < 4; ++c) {
        cplx t = cmul(m[4 * r + c].x, m[4 * r + c].y, in[c]);
        acc.re = __dadd_rn(acc.re, t.re);
        acc.im = __dadd_rn(acc.im, t.im);
    }
    return acc;
}

__device__ __forceinline__ void apply1(double2 *s, uint32_t half, uint32_t t,
                                       const TileGate &g, uint32_t tid, uint32_t nth) {
    const double2 *m = g.m;
    const uint32_t stride = 1u << t;
    for (uint32_t p = tid; p < half; p += nth) {
        const uint32_t i = insert_zero_bit32(p, t), j = i | stride;
        const double2 a = s[i], b = s[j];
        cplx oi, oj;
        const uint32_t cls = g.cls & 0xff;
        if (cls == GC_DIAG) {
            oi = cmul(m[0].x, m[0].y, a);
            oj = cmul(m[3].x, m[3].y, b);
            if (has_zero(oi) || has_zero(oj)) {
                oi = row2(m, 0, a, b);
                oj = row2(m, 1, a, b);
            }
        } else if (cls == GC_ANTI) {
            oi = cmul(m[1].x, m[1].y, b);
            oj = cmul(m[2].x, m[2].y, a);
            if (has_zero(oi) || has_zero(oj)) {
                oi = row2(m, 0, a, b);
                oj = row2(m, 1, a, b);
            }
        } else {
            oi = row2(m, 0, a, b);
            oj = row2(m, 1, a, b);
        }
        s[i] = to2(oi);
        s[j] = to2(oj);
    }
}

__device__ __forceinline__ void apply2(double2 *s, uint32_t quarter, const TileGate &g,
                                       uint32_t tid, uint32_t nth) {
    const double2 *m = g.m;
    const uint32_t lo = min(g.t0, g.t1), hi = max(g.t0, g.t1);
    const uint32_t s0 = 1u << g.t0, s1 = 1u << g.t1;
    for (uint32_t q = tid; q < quarter; q += nth) {
        const uint32_t base = insert_zero_bit32(insert_zero_bit32(q, lo), hi);
        const uint32_t idx[4] = {base, base | s1, base | s0, base | s0 | s1};
        double2 in[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) in[k] = s[idx[k]];
        cplx out[4];
        bool full = (g.cls & 0xff) != GC_PERM4;
        if (!full) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int c = (g.cls >> (8 + 2 * r)) & 3;  // the row's nonzero column
                out[r] = cmul(m[4 * r + c].x, m[4 * r + c].y, in[c]);
                full |= has_zero(out[r]);
            }
        }
        if (full) {
#pragma unroll
            for (int r = 0; r < 4; ++r) out[r] = row4(m, r, in);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) s[idx[r]] = to2(out[r]);
    }
}

__global__ void __launch_bounds__(256) tile_pass_kernel(double2 *__restrict__ buf,
                                                        uint32_t nbits, PassDesc pd,
                                                        const TileGate *__restrict__ gates,
                                                        uint64_t ntiles) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *s = reinterpret_cast<double2 *>(smem_raw);
    const uint32_t k = pd.k, L = pd.lowbits;
    const uint32_t tile = 1u << k;
    uint64_t *offhi = reinterpret_cast<uint64_t *>(s + tile);
    const uint32_t nhi = 1u << (k - L);
    const uint64_t all = nbits >= 64 ? ~uint64_t(0) : ((uint64_t(1) << nbits) - 1);
    const uint64_t ntmask = all & ~pd.tmask;
    const uint64_t himask = pd.tmask & ~((uint64_t(1) << L) - 1);
    const uint32_t lowmask = (1u << L) - 1;
    const uint32_t tid = threadIdx.x, nth = blockDim.x;
    for (uint32_t h = tid; h < nhi; h += nth) offhi[h] = deposit_bits(h, himask);
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t base = deposit_bits(t, ntmask);
        __syncthreads();
        for (uint32_t l = tid; l < tile; l += nth)
            s[l] = __ldcs(buf + base + offhi[l >> L] + (l & lowmask));
        __syncthreads();
        for (uint32_t gi = 0; gi < pd.ngates; ++gi) {
            const TileGate &g = gates[pd.first_gate + gi];
            if (g.nq == 1) apply1(s, tile >> 1, g.t0, g, tid, nth);
            else apply2(s, tile >> 2, g, tid, nth);
            __syncthreads();
        }
        for (uint32_t l = tid; l < tile; l += nth)
            __stcs(buf + base + offhi[l >> L] + (l & lowmask), s[l]);
    }
}

} // namespace

uint64_t run_passes(const DevPlan &plan, double2 *buf, uint32_t nbits, cudaStream_t s) {
    uint64_t launches = 0;
    for (const PassDesc &pd : plan.host_passes) {
        const uint32_t tile = 1u << pd.k;
        const uint64_t ntiles = uint64_t(1) << (nbits - pd.k);
        const uint32_t threads = std::max<uint32_t>(32, std::min<uint32_t>(256, tile / 2));
        const size_t smem = sizeof(double2) * tile + sizeof(uint64_t) * (tile >> pd.lowbits);
        static bool attr_set = false;
        if (!attr_set) {
            QZ_CUDA(cudaFuncSetAttribute(tile_pass_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         96 * 1024));
            attr_set = true;
        }
        const uint64_t grid = std::min<uint64_t>(ntiles, uint64_t(kNumSMs) * 16);
        tile_pass_kernel<<<(unsigned)grid, threads, smem, s>>>(buf, nbits, pd, plan.gates, ntiles);
        QZ_CHECK_LAUNCH();
        ++launches;
    }
    return launches;
}

} // namespace qz
