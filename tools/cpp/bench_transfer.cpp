// bench_transfer — the reference CLI's `bench-transfer` (tools/qzsim.cpp:
// 231-317) over the CUDA device of the drop-in: the paper's Table 1
// measured on a B200 across real PCIe.  Per amplitude
// exponent and strategy: gather (H2D) and scatter (D2H) of 2^e amplitudes in
// chunks of 2^c, median / min / max over the repetitions, ratio vs
// Synchronous.  The device's own TransferStats (CUDA events on the engine
// stream) are the timer, like the reference's OpBegin / OpEnd brackets.
//
//   bench_transfer [exponents=20,25] [reps=3] [c=16] [per_element_max_exp=25]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "qzsim/device.hpp"

using namespace qzsim;

static double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

int main(int argc, char **argv) {
    std::vector<uint32_t> exps{20, 25};
    if (argc > 1) {
        exps.clear();
        std::stringstream ss(argv[1]);
        for (std::string t; std::getline(ss, t, ',');) exps.push_back(uint32_t(std::stoul(t)));
    }
    const uint32_t reps = argc > 2 ? uint32_t(std::atoi(argv[2])) : 3;
    const uint32_t cq = argc > 3 ? uint32_t(std::atoi(argv[3])) : 16;
    const uint32_t pe_max = argc > 4 ? uint32_t(std::atoi(argv[4])) : 25;
    std::printf("{\"repetitions\": %u, \"chunk_qubits\": %u, \"cpu_threads\": %u, \"device\": \"cuda\", \"results\": [",
                reps, cq, std::thread::hardware_concurrency());
    bool first_row = true;
    for (uint32_t e : exps) {
        const uint32_t c = std::min(cq, e);
        const uint64_t len = uint64_t(1) << c, chunks = uint64_t(1) << (e - c);
        std::mt19937_64 rng(7);
        std::uniform_real_distribution<double> dist(-1.0, 1.0);
        std::vector<std::vector<Amplitude>> data(chunks);
        for (auto &ch : data) {
            ch.resize(len);
            for (Amplitude &a : ch) a = {dist(rng), dist(rng)};
        }
        std::printf("%s\n  {\"amplitude_exponent\": %u", first_row ? "" : ",", e);
        first_row = false;
        double sync_h = 0, sync_d = 0;
        for (Strategy st : {Strategy::Synchronous, Strategy::PerElement, Strategy::Buffered}) {
            const uint32_t r = st == Strategy::PerElement ? (e > pe_max ? 0u : std::min(reps, e >= 25 ? 1u : reps))
                                                          : reps;
            if (!r) continue;
            DeviceConfig dc;
            dc.strategy = st;
            dc.memory_limit_bytes = (uint64_t(1) << e) * 16 * 2;
            auto dev = make_cuda_device(dc);
            std::vector<double> h2d, d2h;
            for (uint32_t k = 0; k < r; ++k) {
                std::vector<const Amplitude *> in;
                std::vector<Amplitude *> out;
                for (auto &ch : data) {
                    in.push_back(ch.data());
                    out.push_back(ch.data());
                }
                const TransferStats a = dev->stats();
                dev->wait(dev->gather(std::move(in), len));
                const TransferStats b = dev->stats();
                dev->wait(dev->scatter(std::move(out), len));
                const TransferStats d = dev->stats();
                h2d.push_back(b.h2d_seconds - a.h2d_seconds);
                d2h.push_back(d.d2h_seconds - b.d2h_seconds);
            }
            const double mh = median(h2d), md = median(d2h);
            if (st == Strategy::Synchronous) {
                sync_h = mh;
                sync_d = md;
            }
            std::printf(", \"%s\": {\"h2d_median_seconds\": %.6g, \"h2d_min_seconds\": %.6g, \"h2d_max_seconds\": %.6g, "
                        "\"d2h_median_seconds\": %.6g, \"d2h_min_seconds\": %.6g, \"d2h_max_seconds\": %.6g, "
                        "\"h2d_ratio_vs_sync\": %.6g, \"d2h_ratio_vs_sync\": %.6g, \"repetitions\": %u}",
                        std::string(strategy_name(st)).c_str(), mh, *std::min_element(h2d.begin(), h2d.end()),
                        *std::max_element(h2d.begin(), h2d.end()), md, *std::min_element(d2h.begin(), d2h.end()),
                        *std::max_element(d2h.begin(), d2h.end()), sync_h > 0 ? mh / sync_h : 1.0,
                        sync_d > 0 ? md / sync_d : 1.0, r);
            std::fflush(stdout);
        }
        std::printf("}");
    }
    std::printf("\n]}\n");
    return 0;
}
