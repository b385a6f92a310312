// engine_ctx.hpp — process-wide libqzcuda context for the C++ drop-in layer
// and the translation of C-ABI status codes into the qzsim exception types.
#pragma once

#include <vector>

#include "../../include/qzcuda.h"
#include "qzsim/gates.hpp"

namespace qzsim::b200 {

/// The context every drop-in call uses (device from $QZSIM_DEVICE, default 0).
qzc_context *ctx();

/// Throw the qzsim exception matching a non-zero qzc status.
void check(int rc);

qzc_gate to_abi(const Gate &g);
std::vector<qzc_gate> to_abi(std::span<const Gate> gates);

} // namespace qzsim::b200
