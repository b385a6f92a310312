// qz_jit.cu — runtime-specialised fused gate passes (see qz_jit.cuh).
//
// NVRTC and the driver's module API are reached at run time (dlopen /
// cudaGetDriverEntryPoint), so the library still loads where no GPU driver
// exists (the CPU test suite) and nothing here runs unless a pass asks.
#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <future>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "qz_jit.cuh"

#ifndef QZ_MIN_CTAS
#define QZ_MIN_CTAS 3   // as in qz_gates_dev.cuh
#endif

namespace qz {

constexpr int NB_HOST = 1 << kRegBits;

namespace {

// The device headers, embedded at build time (Makefile: jit_headers.inc).
#include "jit_headers.inc"

struct Nvrtc {
    bool ok = false;
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) log = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) cubin = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
};

void drain_pool_at_exit();

const Nvrtc &nvrtc() {
    static Nvrtc n = [] {
        Nvrtc r;
        void *h = nullptr;
        for (const char *name : {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"})
            if (!h) h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
        if (!h) return r;
        // registered after libnvrtc's own exit handlers: runs before them, so
        // no compile is still inside NVRTC while it is torn down
        std::atexit(drain_pool_at_exit);
        r.create = reinterpret_cast<decltype(r.create)>(dlsym(h, "nvrtcCreateProgram"));
        r.compile = reinterpret_cast<decltype(r.compile)>(dlsym(h, "nvrtcCompileProgram"));
        r.log_size = reinterpret_cast<decltype(r.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
        r.log = reinterpret_cast<decltype(r.log)>(dlsym(h, "nvrtcGetProgramLog"));
        r.cubin_size = reinterpret_cast<decltype(r.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
        r.cubin = reinterpret_cast<decltype(r.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
        r.destroy = reinterpret_cast<decltype(r.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
        r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
        return r;
    }();
    return n;
}

struct Driver {
    bool ok = false;
    CUresult (*load)(CUmodule *, const void *) = nullptr;
    CUresult (*get_fn)(CUfunction *, CUmodule, const char *) = nullptr;
    CUresult (*set_attr)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                       CUstream, void **, void **) = nullptr;
};

const Driver &driver() {
    static Driver d = [] {
        Driver r;
        auto get = [](const char *name, void **fn) {
            cudaDriverEntryPointQueryResult st;
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &st) == cudaSuccess &&
                   st == cudaDriverEntryPointSuccess && *fn;
        };
        void *p[4] = {nullptr, nullptr, nullptr, nullptr};
        r.ok = get("cuModuleLoadData", &p[0]) && get("cuModuleGetFunction", &p[1]) &&
               get("cuFuncSetAttribute", &p[2]) && get("cuLaunchKernel", &p[3]);
        r.load = reinterpret_cast<decltype(r.load)>(p[0]);
        r.get_fn = reinterpret_cast<decltype(r.get_fn)>(p[1]);
        r.set_attr = reinterpret_cast<decltype(r.set_attr)>(p[2]);
        r.launch = reinterpret_cast<decltype(r.launch)>(p[3]);
        return r;
    }();
    return d;
}

// Compile jobs run on a few host threads while the GPU works.
class Pool {
  public:
    Pool() {
        const unsigned n = std::max(2u, std::min(16u, std::thread::hardware_concurrency()));
        for (unsigned i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
    }
    ~Pool() { shutdown(); }
    // queued compiles are dropped, running ones finish (idempotent)
    void shutdown() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            q_.clear();
        }
        cv_.notify_all();
        std::lock_guard<std::mutex> lk(join_mu_);
        for (auto &t : threads_)
            if (t.joinable()) t.join();
    }
    void submit(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back(std::move(f));
        }
        cv_.notify_one();
    }

  private:
    void loop() {
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
                if (q_.empty()) return;
                f = std::move(q_.front());
                q_.pop_front();
            }
            f();
        }
    }
    std::mutex mu_, join_mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    std::vector<std::thread> threads_;
    bool stop_ = false;
};

Pool &pool() {
    static Pool p;
    return p;
}

void drain_pool_at_exit() { pool().shutdown(); }

void put_double(std::string &o, double x) {
    char b[40];
    std::snprintf(b, sizeof b, "%a", x);
    o += b;
}

void put_gate(std::string &o, const TileGate &t) {
    char b[512];
    std::snprintf(b, sizeof b, "{%uu,%uu,%uu,%uu,%uu,%uu,%lluull,%uu,%uu,%uu,%uu,%uu,%uu,%uu,%uu,%uu,%uu,%uu,%uu,%uu,{%uu,%uu,%uu},{",
                  t.nq, t.r0, t.r1, t.t0, t.t1, t.sgn, (unsigned long long)t.kinds, t.cls, t.perm, t.zm, t.smask, t.op,
                  t.pad, t.srow, t.pad2, t.ob0, t.ob1, t.run, t.steps, t.cid, t.pad4[0], t.pad4[1], t.pad4[2]);
    o += b;
    for (int e = 0; e < 16; ++e) {
        o += e ? ",{" : "{";
        put_double(o, t.m[e].x);
        o += ",";
        put_double(o, t.m[e].y);
        o += "}";
    }
    o += "}}";
}

uint32_t min_bits() {
    static const uint32_t v = getenv("QZ_JIT_MIN_BITS") ? uint32_t(atoi(getenv("QZ_JIT_MIN_BITS"))) : 24u;
    return v;
}

bool jit_enabled() {
    static const bool v = !(getenv("QZ_JIT") && getenv("QZ_JIT")[0] == '0');
    return v;
}

} // namespace

struct JitPass {
    std::string source;
    std::mutex mu;
    std::condition_variable cv;
    bool compiled = false;   // the compile job finished (cubin or failure)
    std::string cubin, log;
    bool loaded = false, failed = false;
    CUfunction fn = nullptr;
};

namespace {
std::mutex g_cache_mu;
std::unordered_map<std::string, std::shared_ptr<JitPass>> g_cache;

void compile_job(const std::shared_ptr<JitPass> &j) {
    const Nvrtc &n = nvrtc();
    if (const char *dir = getenv("QZ_JIT_DUMP")) {   // inspection: write the source
        static std::atomic<int> seq{0};
        const std::string path = std::string(dir) + "/qz_jit_" + std::to_string(seq++) + ".cu";
        if (FILE *f = std::fopen(path.c_str(), "w")) {
            std::fputs(j->source.c_str(), f);
            std::fclose(f);
        }
    }
    std::string cubin, log;
    bool ok = n.ok;
    if (ok) {
        nvrtcProgram prog;
        ok = n.create(&prog, j->source.c_str(), "qz_jit_pass.cu", kJitHeaderCount, kJitHeaderSrc, kJitHeaderNames) ==
             NVRTC_SUCCESS;
        if (ok) {
            // the build's tile geometry (the device headers' macros)
            static const std::string ctas =
                std::string("-DQZ_MIN_CTAS=") +
                (getenv("QZ_JIT_MIN_CTAS") ? std::string(getenv("QZ_JIT_MIN_CTAS")) : std::to_string(QZ_MIN_CTAS));
            static const std::string tbits = "-DQZ_TILE_BITS=" + std::to_string(kTileBits);
            // inspection builds: QZ_JIT_DEFINE=<macro> (e.g. QZ_GROUP_CLOCKS)
            static const std::string extra =
                std::string("-D") + (getenv("QZ_JIT_DEFINE") ? getenv("QZ_JIT_DEFINE") : "QZ_JIT_NODEF");
            const char *opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo",
                                  "-DQZ_JIT_SOURCE=1", ctas.c_str(), tbits.c_str(), extra.c_str()};
            const nvrtcResult rc = n.compile(prog, 8, opts);
            size_t ls = 0;
            n.log_size(prog, &ls);
            log.resize(ls);
            if (ls) n.log(prog, &log[0]);
            ok = rc == NVRTC_SUCCESS;
            if (ok) {
                size_t cs = 0;
                ok = n.cubin_size(prog, &cs) == NVRTC_SUCCESS && cs > 0;
                if (ok) {
                    cubin.resize(cs);
                    ok = n.cubin(prog, &cubin[0]) == NVRTC_SUCCESS;
                }
            }
            n.destroy(&prog);
        }
    } else {
        log = "libnvrtc not found";
    }
    {
        std::lock_guard<std::mutex> lk(j->mu);
        j->cubin = ok ? std::move(cubin) : std::string();
        j->log = std::move(log);
        j->compiled = true;
        if (!ok) j->failed = true;
    }
    j->cv.notify_all();
}
} // namespace

// Registers statically +0 under `f` for a group whose register bits sit on
// buffer bits bb[]: some fresh register bit holds the value whose amplitudes
// are all +0.
static uint32_t static_zero_regs(const Fresh &f, const uint32_t (&bb)[kRegBits]) {
    uint32_t zm = 0;
    for (uint32_t r = 0; r < uint32_t(NB_HOST); ++r)
        for (int i = 0; i < kRegBits; ++i)
            if (((f.mask >> bb[i]) & 1) && ((r >> i) & 1) != ((f.val >> bb[i]) & 1)) zm |= 1u << r;
    return zm;
}

std::string jit_source(const GatePlan &plan, const PassDesc &pd, Fresh fresh) {
    std::string o;
    o.reserve(1 << 16);
    o += "#include \"qz_rtc_types.cuh\"\n#include \"qz_gate_types.cuh\"\n#include \"qz_bits.cuh\"\n";
    o += "namespace qz {\n#include \"qz_gates_dev.cuh\"\n}\n";
    o += "namespace qz { namespace {\n";
    // the pass's fast-list descriptors, in group order
    std::vector<uint32_t> goff(pd.ngroups);
    uint32_t total = 0;
    for (uint32_t gi = 0; gi < pd.ngroups; ++gi) {
        goff[gi] = total;
        total += plan.groups[pd.first_group + gi].nfast;
    }
    o += "__device__ const TileGate kG[" + std::to_string(std::max(total, 1u)) + "] = {";
    bool first = true;
    for (uint32_t gi = 0; gi < pd.ngroups; ++gi) {
        const GroupDesc &G = plan.groups[pd.first_group + gi];
        for (uint32_t q = 0; q < G.nfast; ++q) {
            if (!first) o += ",\n";
            first = false;
            put_gate(o, plan.gates[G.first_fast + q]);
        }
    }
    if (first) o += "{}";
    o += "};\n";
    o += "struct Prog {\n  static __device__ __forceinline__ void run(uint32_t gi, const TileGate *__restrict__, "
         "uint32_t, double2 (&v)[NB], uint64_t gidx, bool &bad) {\n    switch (gi) {\n";
    // tile bit t of this pass is buffer bit tb[t]
    std::vector<uint32_t> tb;
    for (uint32_t b = 0; b < 64; ++b)
        if ((pd.tmask >> b) & 1) tb.push_back(b);
    for (uint32_t gi = 0; gi < pd.ngroups; ++gi) {
        const GroupDesc &G = plan.groups[pd.first_group + gi];
        if (G.generic || G.nfast == 0) {
            fresh = Fresh{};   // (conservative)
            continue;
        }
        uint32_t bb[kRegBits];
        for (int i = 0; i < kRegBits; ++i) bb[i] = G.gbits[i] < tb.size() ? tb[G.gbits[i]] : 63u;
        // statically +0 registers are skipped only where every gate keeps
        // all-(+0) blocks all-(+0) (then they stay +0, sign included)
        const bool use = G.pz_stable && fresh.mask;
        o += "    case " + std::to_string(gi) + ": {\n      const TileGate *f = kG + " + std::to_string(goff[gi]) + ";\n";
        for (uint32_t q = 0; q < G.nfast;) {
            const TileGate &t = plan.gates[G.first_fast + q];
            uint32_t zm = use ? static_zero_regs(fresh, bb) : 0u;
            // PDIAG / DIAG / CZ and the fused CP5 / CXD are diagonal: a +0
            // register they touch through a fresh bit sums m_rr * (+0) with
            // structural zeros of live amplitudes, +0 only for sign-safe rows
            const bool diag = t.op == OP_PDIAG || t.op == OP_DIAG || t.op == OP_CZ || t.op == OP_CP5 ||
                              t.op == OP_CXD;
            if (diag) {
                uint64_t touched = 0;
                if (t.op == OP_PDIAG) {
                    if (t.nq) touched |= uint64_t(1) << bb[t.r0];
                } else {
                    touched |= uint64_t(1) << bb[t.r0];
                    if (t.nq == 2) touched |= uint64_t(1) << bb[t.r1];
                }
                const bool safe = t.op == OP_DIAG  ? (t.srow & 3u) == 3u
                                  : t.op == OP_CP5 ? (t.srow & 7u) == 7u
                                  : t.op == OP_CXD ? (t.srow & 3u) == 3u
                                  : t.op == OP_PDIAG ? (t.srow & t.steps) == t.steps
                                                     : false;
                if ((fresh.mask & touched) && !safe) {
                    zm = 0;
                    fresh.mask &= ~touched;
                    fresh.val &= fresh.mask;
                }
            }
            o += "      if (!bad) fast_cid<" + std::to_string(t.cid) + ">(v, f, " + std::to_string(q) + "u, gidx, bad, " +
                 std::to_string(zm) + "u);\n";
            // freshness after a non-diagonal op
            if (t.op == OP_GEN1 || t.op == OP_CX || t.op == OP_SWAP)
                fresh = fresh_gate(fresh, t.op, t.nq, bb[t.r0], t.nq == 2 ? bb[t.r1] : 0u, t.kinds, false);
            else if (!diag)
                fresh = Fresh{};
            // PDIAG runs (case ids 0..3) cover `run` ops, everything else one
            q += (t.cid <= 3 && t.run) ? t.run : 1;
        }
        if (!G.pz_stable) fresh = Fresh{};   // zeros may have turned -0
        o += "      break;\n    }\n";
    }
    o += "    default: break;\n    }\n  }\n};\n} }\n";
    o += "extern \"C\" __global__ void __launch_bounds__(1 << (qz::kTileBits - qz::kRegBits), QZ_MIN_CTAS)\n"
         "qz_jit_pass(const double2 *__restrict__ src, double2 *__restrict__ dst, uint32_t nbits, qz::PassDesc pd,\n"
         "            const qz::GroupDesc *__restrict__ groups, const qz::TileGate *__restrict__ gates, uint64_t ntiles,\n"
         "            unsigned long long *__restrict__ counters, uint32_t *__restrict__ flag,\n"
         "            const uint32_t *__restrict__ cond, uint32_t *__restrict__ nzslot, uint32_t cbits) {\n"
         "  qz::tile_pass_body<" + std::to_string(pd.variant) + ", qz::Prog>(src, dst, nbits, pd, groups, gates, ntiles, "
         "counters, flag, cond, nzslot, cbits);\n}\n";
    return o;
}

namespace {
// Cache key: the bytes the source is generated from (cheaper than the
// source itself on the per-stage upload path).
std::string cache_key(const GatePlan &plan, const PassDesc &pd, const Fresh &fresh) {
    std::string k;
    k.push_back(char(pd.variant));
    const uint64_t hdr0[3] = {pd.tmask, fresh.mask, fresh.val};
    k.append(reinterpret_cast<const char *>(hdr0), sizeof hdr0);
    for (uint32_t gi = 0; gi < pd.ngroups; ++gi) {
        const GroupDesc &G = plan.groups[pd.first_group + gi];
        const uint32_t hdr[6] = {G.generic ? 0xFFFFFFFFu : G.nfast, gi, G.pz_stable, G.gbits[0], G.gbits[1],
                                 G.gbits[2]};
        k.append(reinterpret_cast<const char *>(hdr), sizeof hdr);
        k.append(reinterpret_cast<const char *>(&plan.gates[G.first_fast]), sizeof(TileGate) * G.nfast);
    }
    return k;
}

std::shared_ptr<JitPass> request(const GatePlan &plan, const PassDesc &pd, const Fresh &fresh) {
    std::string key = cache_key(plan, pd, fresh);
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) return it->second;
    auto j = std::make_shared<JitPass>();
    j->source = jit_source(plan, pd, fresh);
    g_cache.emplace(std::move(key), j);
    pool().submit([j] { compile_job(j); });
    return j;
}
} // namespace

std::shared_ptr<JitPass> jit_request(const GatePlan &plan, const PassDesc &pd, uint32_t nbits, Fresh fresh) {
    if (!jit_enabled() || nbits < min_bits() || pd.kind != PASS_TILE || pd.k != kTileBits) return nullptr;
    static const bool no_fresh = getenv("QZ_NO_FRESH") != nullptr;   // control: no static skipping
    return request(plan, pd, no_fresh ? Fresh{} : fresh);
}

std::string &last_error();   // qz_runtime.cu

bool jit_ready(JitPass &j) {
    static const bool sync = getenv("QZ_JIT_SYNC") && getenv("QZ_JIT_SYNC")[0] == '1';
    std::unique_lock<std::mutex> lk(j.mu);
    if (sync) j.cv.wait(lk, [&] { return j.compiled; });
    return j.compiled && !j.failed;
}

namespace {
// Load a compiled pass into the current context (caller holds j.mu).
bool load_locked(JitPass &j) {
    if (j.failed) return false;
    if (j.loaded) return true;
    const Driver &d = driver();
    CUmodule mod = nullptr;
    if (!d.ok || d.load(&mod, j.cubin.data()) != CUDA_SUCCESS ||
        d.get_fn(&j.fn, mod, "qz_jit_pass") != CUDA_SUCCESS ||
        d.set_attr(j.fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, 110 * 1024) != CUDA_SUCCESS) {
        j.failed = true;
        static bool warned = false;
        if (!warned) {
            warned = true;
            std::fprintf(stderr, "qz: specialised pass could not be loaded; using the AOT kernel\n");
        }
        return false;
    }
    j.loaded = true;
    j.cubin.clear();
    return true;
}
} // namespace

size_t jit_wait_all(bool load) {
    std::vector<std::shared_ptr<JitPass>> all;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (auto &kv : g_cache) all.push_back(kv.second);
    }
    size_t built = 0;
    for (auto &j : all) {
        std::unique_lock<std::mutex> lk(j->mu);
        j->cv.wait(lk, [&] { return j->compiled; });
        if (load) load_locked(*j);
        built += !j->failed;
    }
    return built;
}

bool jit_launch(JitPass &j, unsigned grid, unsigned threads, size_t smem, cudaStream_t s, void **args) {
    std::unique_lock<std::mutex> lk(j.mu);
    j.cv.wait(lk, [&] { return j.compiled; });
    if (!load_locked(j)) return false;
    return driver().launch(j.fn, grid, 1, 1, threads, 1, 1, unsigned(smem), reinterpret_cast<CUstream>(s), args,
                           nullptr) == CUDA_SUCCESS;
}

} // namespace qz

using namespace qz;

extern "C" {

// Compile the widest pass of a gate list (on buffer bits of a 2^nbits
// window) with NVRTC on the host — no GPU needed: 0 when the specialised-pass
// toolchain works here; else -1 with NVRTC's log in qzc_last_error().
int qzc_jit_selftest(const qzc_gate *gates, uint64_t ngates, uint32_t nbits) {
    try {
        std::vector<DevGate> dg;
        for (uint64_t i = 0; i < ngates; ++i) dg.push_back(make_dev_gate(gates[i]));
        const GatePlan gp = build_passes(dg, nbits, kTileBits, true, 1);
        static const bool all = getenv("QZ_JIT_SELFTEST_ALL") != nullptr;   // every pass (inspection)
        std::vector<std::shared_ptr<JitPass>> jobs;
        // QZ_JIT_SELFTEST_FRESH=1: as after init_basis (every bit fresh at the start)
        Fresh f;
        if (getenv("QZ_JIT_SELFTEST_FRESH")) f.mask = nbits >= 64 ? ~uint64_t(0) : (uint64_t(1) << nbits) - 1;
        size_t at = 0;
        for (const PassDesc &pd : launch_passes(gp)) {
            f = fresh_after(dg, at, pd.dg0, f);
            at = pd.dg0;
            if (pd.kind != PASS_TILE || pd.k != kTileBits) continue;
            jobs.push_back(request(gp, pd, f));
            if (!all) break;
        }
        if (jobs.empty()) {
            qz::last_error() = "jit: no full-tile pass in the plan";
            return QZC_EINVAL;
        }
        for (auto &j : jobs) {
            std::unique_lock<std::mutex> lk(j->mu);
            j->cv.wait(lk, [&] { return j->compiled; });
            if (j->failed) {
                qz::last_error() = "jit: " + j->log;
                return QZC_EDEVICE;
            }
        }
        return QZC_OK;
    } catch (const std::exception &e) {
        qz::last_error() = e.what();
        return QZC_EINVAL;
    }
}

// Wait for the specialised passes queued so far (e.g. after a warm-up run);
// returns how many were built.
uint64_t qzc_jit_wait(void) {
    // loads the built kernels into the calling thread's current context when
    // it has one (the engine's device), so no later launch pays for it
    CUcontext cur = nullptr;
    static auto get_cur = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult st;
        return cudaGetDriverEntryPoint("cuCtxGetCurrent", &fn, cudaEnableDefault, &st) == cudaSuccess &&
                       st == cudaDriverEntryPointSuccess
                   ? reinterpret_cast<CUresult (*)(CUcontext *)>(fn)
                   : nullptr;
    }();
    const bool has_ctx = get_cur && get_cur(&cur) == CUDA_SUCCESS && cur != nullptr;
    return jit_wait_all(has_ctx);
}

} // extern "C"
