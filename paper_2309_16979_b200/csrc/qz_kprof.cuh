// qz_kprof.cuh — per-launch CUDA-event timing of the engine's own kernels.
//
// When enabled (qzc_kprof_enable), every fused gate pass and every codec
// kernel launch is bracketed by two events recorded on the stream the kernel
// is launched on, tagged with its name, the stage / pass index and its
// algorithmic bytes (32 B per window amplitude for a gate pass,
// 16 B per decoded / encoded amplitude for the codec kernels; payload bytes
// are added by the caller from qzc_sim_stats).  bench.py reads the records of
// its timed region to report the dominant launch's roofline.  Process-wide
// (the engine drives one device per process).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace qz {

// Returns a handle (or -1 when profiling is off).
int kprof_begin(cudaStream_t s);
// Closes handle h: records the end event on s and the record's metadata.
void kprof_end(int h, cudaStream_t s, const char *name, uint32_t tag, double bytes);
// Stage index stored with subsequent records.
void kprof_set_stage(uint32_t stage);

// RAII form for launches with a single exit.
struct KProfScope {
    int h;
    cudaStream_t s;
    const char *name;
    uint32_t tag;
    double bytes;
    KProfScope(cudaStream_t s_, const char *n, uint32_t t, double b)
        : h(kprof_begin(s_)), s(s_), name(n), tag(t), bytes(b) {}
    ~KProfScope() { kprof_end(h, s, name, tag, bytes); }
};

} // namespace qz
