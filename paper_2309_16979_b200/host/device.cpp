// device.cpp — qzsim::Device on the B200 (make_cuda_device).
//
// The reference's ReferenceDevice (device.cpp:98-503) is an in-process worker
// thread with a per-command doorbell.  Here the in-order queue is the
// engine's CUDA stream: every command is enqueued through the C ABI and
// completes in submission order; handles wrap CUDA events; the memory bound
// and buffer-bit checks fail at submission like the reference.  The three
// transfer strategies are real host<->device traffic:
//   Synchronous : one copy per chunk
//   PerElement  : one copy per amplitude (the paper's slow async path)
//   Buffered    : pack into page-locked staging on the host, one bulk copy,
//                 then a device-side mapping pass (qzc_permute)
#include <algorithm>
#include <cstring>
#include <deque>
#include <thread>

#include "engine_ctx.hpp"
#include "qzsim/device.hpp"

namespace qzsim {

std::string_view strategy_name(Strategy s) {
    switch (s) {
    case Strategy::Synchronous: return "synchronous";
    case Strategy::PerElement: return "per-element";
    case Strategy::Buffered: return "buffered";
    }
    return "?";
}

std::optional<Strategy> strategy_from_name(std::string_view name) {
    if (name == "synchronous" || name == "sync") return Strategy::Synchronous;
    if (name == "per-element" || name == "per_element") return Strategy::PerElement;
    if (name == "buffered") return Strategy::Buffered;
    return std::nullopt;
}

namespace detail {
struct CommandState {
    void *event = nullptr;
    ~CommandState() {
        if (event) qzc_event_destroy(b200::ctx(), event);
    }
};
} // namespace detail

CommandStatus CommandHandle::status() const {
    if (!state_ || !state_->event) return CommandStatus::Done;
    return qzc_event_done(b200::ctx(), state_->event) ? CommandStatus::Done : CommandStatus::Pending;
}

namespace {
enum class Op { H2D, D2H, Kernel };

// Copy chunk-sized pieces between pageable chunk memory and the pinned
// staging area on several host threads (the host half of the Buffered
// strategy; one thread for small batches).
template <class Fn> void parallel_chunks(size_t count, uint64_t bytes_each, Fn fn) {
    const uint64_t total = count * bytes_each;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nt = total < (uint64_t(4) << 20) ? 1u : std::min<unsigned>(hw, 8u);
    if (nt == 1 || count < 2) {
        for (size_t j = 0; j < count; ++j) fn(j);
        return;
    }
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < nt; ++t)
        ts.emplace_back([&, t] {
            for (size_t j = t; j < count; j += nt) fn(j);
        });
    for (std::thread &t : ts) t.join();
}
} // namespace

class CudaDevice final : public Device {
  public:
    explicit CudaDevice(const DeviceConfig &cfg) : cfg_(cfg) {
        if (cfg.kernel_workers < 1) throw DeviceError("kernel worker count must be >= 1");
        b200::ctx();
    }

    ~CudaDevice() override {
        qzc_synchronize(b200::ctx());
        drain_timers();
        if (buffer_) qzc_buffer_free(b200::ctx(), buffer_);
        if (staging_) qzc_buffer_free(b200::ctx(), staging_);
        if (pinned_) qzc_host_free(b200::ctx(), pinned_);
    }

    CommandHandle gather(std::vector<const Amplitude *> chunks, uint64_t chunk_len) override {
        const uint64_t total = chunks.size() * chunk_len;
        reserve(total);
        qzc_context *c = b200::ctx();
        if (cfg_.strategy == Strategy::Buffered) {
            void *t0 = mark();
            parallel_chunks(chunks.size(), chunk_len * sizeof(Amplitude), [&](size_t j) {
                std::memcpy(pinned_ + j * chunk_len, chunks[j], chunk_len * sizeof(Amplitude));
            });
            b200::check(qzc_copy_h2d(c, staging_, 0, reinterpret_cast<const double *>(pinned_), total));
            ++stats_.h2d_op_count;
            stats_.bytes_moved += total * sizeof(Amplitude);
            void *t1 = mark();
            timers_.push_back({Op::H2D, t0, t1});
            b200::check(qzc_permute(c, buffer_, staging_, total));
            void *t2 = mark();
            timers_.push_back({Op::Kernel, t1, t2});
            amps_ = total;
            return handle();
        }
        void *t0 = mark();
        for (size_t j = 0; j < chunks.size(); ++j) {
            const double *src = reinterpret_cast<const double *>(chunks[j]);
            if (cfg_.strategy == Strategy::Synchronous) {
                b200::check(qzc_copy_h2d(c, buffer_, j * chunk_len, src, chunk_len));
                ++stats_.h2d_op_count;
            } else {
                for (uint64_t e = 0; e < chunk_len; ++e)
                    b200::check(qzc_copy_h2d(c, buffer_, j * chunk_len + e, src + 2 * e, 1));
                stats_.h2d_op_count += chunk_len;
            }
            stats_.bytes_moved += chunk_len * sizeof(Amplitude);
        }
        timers_.push_back({Op::H2D, t0, mark()});
        amps_ = total;
        return handle();
    }

    CommandHandle apply_gates(std::vector<Gate> gates) override {
        uint32_t bits = 0;
        while ((uint64_t(1) << bits) < amps_) ++bits;
        for (const Gate &g : gates)
            for (uint32_t q : g.qubits)
                if (q >= bits)
                    throw DeviceError("buffer bit " + std::to_string(q) + " out of range for batch of 2^" +
                                      std::to_string(bits) + " amplitudes");
        void *t0 = mark();
        if (!gates.empty()) {
            const std::vector<qzc_gate> abi = b200::to_abi(gates);
            b200::check(qzc_apply_gates_dev(b200::ctx(), buffer_, bits, abi.data(), abi.size()));
        }
        timers_.push_back({Op::Kernel, t0, mark()});
        return handle();
    }

    CommandHandle scatter(std::vector<Amplitude *> chunks, uint64_t chunk_len) override {
        const uint64_t total = chunks.size() * chunk_len;
        if (total != amps_) throw DeviceError("scatter size disagrees with gathered batch");
        qzc_context *c = b200::ctx();
        if (cfg_.strategy == Strategy::Buffered) {
            void *t0 = mark();
            b200::check(qzc_permute(c, staging_, buffer_, total));
            void *t1 = mark();
            timers_.push_back({Op::Kernel, t0, t1});
            b200::check(qzc_copy_d2h(c, reinterpret_cast<double *>(pinned_), staging_, 0, total));
            b200::check(qzc_synchronize(c));
            parallel_chunks(chunks.size(), chunk_len * sizeof(Amplitude), [&](size_t j) {
                std::memcpy(chunks[j], pinned_ + j * chunk_len, chunk_len * sizeof(Amplitude));
            });
            ++stats_.d2h_op_count;
            stats_.bytes_moved += total * sizeof(Amplitude);
            timers_.push_back({Op::D2H, t1, mark()});
            return handle();
        }
        void *t0 = mark();
        for (size_t j = 0; j < chunks.size(); ++j) {
            double *dst = reinterpret_cast<double *>(chunks[j]);
            if (cfg_.strategy == Strategy::Synchronous) {
                b200::check(qzc_copy_d2h(c, dst, buffer_, j * chunk_len, chunk_len));
                ++stats_.d2h_op_count;
            } else {
                for (uint64_t e = 0; e < chunk_len; ++e)
                    b200::check(qzc_copy_d2h(c, dst + 2 * e, buffer_, j * chunk_len + e, 1));
                stats_.d2h_op_count += chunk_len;
            }
            stats_.bytes_moved += chunk_len * sizeof(Amplitude);
        }
        timers_.push_back({Op::D2H, t0, mark()});
        return handle();
    }

    void wait(const CommandHandle &h) override {
        if (!h.state_) return;
        b200::check(qzc_synchronize(b200::ctx()));
    }

    TransferStats stats() const override {
        const_cast<CudaDevice *>(this)->drain_timers();
        return stats_;
    }

  private:
    struct Timed {
        Op op;
        void *start, *end;
    };

    void *mark() {
        void *e = nullptr;
        b200::check(qzc_event_record(b200::ctx(), &e));
        return e;
    }

    CommandHandle handle() {
        auto st = std::make_shared<detail::CommandState>();
        st->event = mark();
        return CommandHandle(std::move(st));
    }

    void drain_timers() {
        qzc_context *c = b200::ctx();
        for (const Timed &t : timers_) {
            double s = 0;
            if (qzc_event_elapsed(c, t.start, t.end, &s) == QZC_OK) {
                if (t.op == Op::H2D) stats_.h2d_seconds += s;
                else if (t.op == Op::D2H) stats_.d2h_seconds += s;
                else stats_.kernel_seconds += s;
            }
        }
        // events are shared between consecutive timers: destroy each once
        std::vector<void *> seen;
        for (const Timed &t : timers_)
            for (void *e : {t.start, t.end})
                if (std::find(seen.begin(), seen.end(), e) == seen.end()) seen.push_back(e);
        for (void *e : seen) qzc_event_destroy(c, e);
        timers_.clear();
    }

    void reserve(uint64_t total) {
        uint64_t need = total * sizeof(Amplitude);
        if (cfg_.strategy == Strategy::Buffered) need *= 2;
        if (need > cfg_.memory_limit_bytes)
            throw DeviceError("batch exceeds device memory limit: needs " + std::to_string(need) +
                              " bytes, limit " + std::to_string(cfg_.memory_limit_bytes));
        if (total <= cap_) return;
        qzc_context *c = b200::ctx();
        b200::check(qzc_synchronize(c));
        if (buffer_) qzc_buffer_free(c, buffer_);
        if (staging_) qzc_buffer_free(c, staging_);
        if (pinned_) qzc_host_free(c, pinned_);
        buffer_ = staging_ = nullptr;
        pinned_ = nullptr;
        b200::check(qzc_buffer_alloc(c, total, &buffer_));
        if (cfg_.strategy == Strategy::Buffered) {
            b200::check(qzc_buffer_alloc(c, total, &staging_));
            void *h = nullptr;
            b200::check(qzc_host_alloc(c, total * sizeof(Amplitude), &h));
            pinned_ = static_cast<Amplitude *>(h);
        }
        cap_ = total;
    }

    DeviceConfig cfg_;
    double *buffer_ = nullptr, *staging_ = nullptr;
    Amplitude *pinned_ = nullptr;
    uint64_t cap_ = 0, amps_ = 0;
    std::vector<Timed> timers_;
    mutable TransferStats stats_;
};

std::unique_ptr<Device> make_cuda_device(const DeviceConfig &config) {
    return std::make_unique<CudaDevice>(config);
}

std::unique_ptr<Device> make_reference_device(const DeviceConfig &config) {
    return make_cuda_device(config);
}

} // namespace qzsim
