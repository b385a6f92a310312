// qz_kprof.cu — per-launch event timing (see qz_kprof.cuh) and its C ABI.
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "qz_common.cuh"
#include "qz_kprof.cuh"

namespace qz {
namespace {

struct Rec {
    const char *name;
    uint32_t tag, stage;
    double bytes;
    int a, b;   // event pool indices
    bool closed;
};

struct KProf {
    bool on = false;
    uint32_t stage = 0;
    std::vector<cudaEvent_t> pool;
    size_t next = 0;
    std::vector<Rec> recs;
    std::mutex mu;

    int event() {
        if (next == pool.size()) {
            cudaEvent_t e;
            QZ_CUDA(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return int(next++);
    }
    void reset() {
        recs.clear();
        next = 0;
    }
};

KProf &kp() {
    static KProf k;
    return k;
}

} // namespace

int kprof_begin(cudaStream_t s) {
    KProf &k = kp();
    if (!k.on) return -1;
    std::lock_guard<std::mutex> g(k.mu);
    const int a = k.event();
    QZ_CUDA(cudaEventRecord(k.pool[a], s));
    k.recs.push_back(Rec{nullptr, 0, k.stage, 0.0, a, -1, false});
    return int(k.recs.size() - 1);
}

void kprof_end(int h, cudaStream_t s, const char *name, uint32_t tag, double bytes) {
    if (h < 0) return;
    KProf &k = kp();
    std::lock_guard<std::mutex> g(k.mu);
    if (size_t(h) >= k.recs.size()) return;   // records were read in between
    Rec &r = k.recs[h];
    r.b = k.event();
    QZ_CUDA(cudaEventRecord(k.pool[r.b], s));
    r.name = name;
    r.tag = tag;
    r.bytes = bytes;
    r.closed = true;
}

void kprof_set_stage(uint32_t stage) { kp().stage = stage; }

} // namespace qz

using namespace qz;


extern "C" {

int qzc_kprof_enable(qzc_context *, int on) {
    KProf &k = kp();
    std::lock_guard<std::mutex> g(k.mu);
    k.on = on != 0;
    k.reset();
    k.stage = 0;
    return QZC_OK;
}

int qzc_kprof_read(qzc_context *, qzc_kprof_record *out, uint64_t cap, uint64_t *count) {
    KProf &k = kp();
    std::lock_guard<std::mutex> g(k.mu);
    uint64_t n = 0;
    if (cudaDeviceSynchronize() != cudaSuccess) return QZC_ECUDA;
    for (const Rec &r : k.recs) {
        if (!r.closed) continue;
        if (out && n < cap) {
            qzc_kprof_record &o = out[n];
            std::memset(&o, 0, sizeof o);
            std::strncpy(o.name, r.name ? r.name : "?", sizeof o.name - 1);
            o.tag = r.tag;
            o.stage = r.stage;
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, k.pool[r.a], k.pool[r.b]) != cudaSuccess) return QZC_ECUDA;
            o.seconds = 1e-3 * double(ms);
            o.bytes = r.bytes;
        }
        ++n;
    }
    *count = n;
    if (out) k.reset();
    return QZC_OK;
}

} // extern "C"
