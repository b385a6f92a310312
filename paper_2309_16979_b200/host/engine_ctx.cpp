// engine_ctx.cpp — see engine_ctx.hpp.
#include "engine_ctx.hpp"

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "qzsim/codec.hpp"
#include "qzsim/device.hpp"
#include "qzsim/planner.hpp"
#include "qzsim/store.hpp"

namespace qzsim::b200 {

namespace {
struct Holder {
    qzc_context *c = nullptr;
    ~Holder() {
        if (c) qzc_context_destroy(c);
    }
};
} // namespace

qzc_context *ctx() {
    static Holder h;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *dev = std::getenv("QZSIM_DEVICE");
        const int rc = qzc_context_create(dev ? std::atoi(dev) : 0, 0, &h.c);
        if (rc != QZC_OK) throw DeviceError(std::string("no CUDA device for qzsim: ") + qzc_last_error());
    });
    if (!h.c) throw DeviceError("no CUDA device for qzsim");
    return h.c;
}

void check(int rc) {
    if (rc == QZC_OK) return;
    const std::string msg = qzc_last_error();
    switch (rc) {
    case QZC_ECODEC: throw CodecError(msg);
    case QZC_ESTORE: throw StoreError(msg);
    case QZC_EPLAN: throw PlanError(msg);
    case QZC_EDEVICE: throw DeviceError(msg);
    default: throw Error(msg);
    }
}

qzc_gate to_abi(const Gate &g) {
    qzc_gate out;
    std::memset(&out, 0, sizeof out);
    out.kind = static_cast<uint32_t>(g.kind);
    out.nqubits = static_cast<uint32_t>(g.qubits.size());
    for (size_t k = 0; k < g.qubits.size() && k < 2; ++k) out.qubits[k] = g.qubits[k];
    for (size_t k = 0; k < g.params.size() && k < 3; ++k) out.params[k] = g.params[k];
    return out;
}

std::vector<qzc_gate> to_abi(std::span<const Gate> gates) {
    std::vector<qzc_gate> out;
    out.reserve(gates.size());
    for (const Gate &g : gates) out.push_back(to_abi(g));
    return out;
}

} // namespace qzsim::b200
