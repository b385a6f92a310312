// codec.cpp — qzsim::compress / decompress on the sm_100a codec kernels.
#include "qzsim/codec.hpp"

#include <cmath>
#include <cstring>

#include "engine_ctx.hpp"

namespace qzsim {

CompressedChunk compress(uint64_t chunk_index, std::span<const Amplitude> amplitudes,
                         double error_bound, std::span<const uint64_t> forced_raw) {
    const uint64_t n = amplitudes.size();
    if (n == 0 || (n & (n - 1)))
        throw CodecError("chunk length must be a power of two, got " + std::to_string(n));
    if (!(error_bound >= 0.0) || !std::isfinite(error_bound))
        throw CodecError("error bound must be finite and non-negative");
    CompressedChunk out;
    out.chunk_index = chunk_index;
    out.codec_id = error_bound > 0.0 ? CodecId::LossyPQ : CodecId::LosslessRLE;
    out.error_bound = error_bound;
    out.element_count = static_cast<uint32_t>(n);
    std::vector<uint8_t> buf(qzc_payload_bound(n, error_bound) + 64);
    uint64_t off = 0;
    uint32_t size = 0, crc = 0;
    b200::check(qzc_compress_host(b200::ctx(), reinterpret_cast<const double *>(amplitudes.data()),
                                  1, n, error_bound, forced_raw.data(), forced_raw.size(), buf.data(),
                                  buf.size(), &off, &size, &crc));
    out.payload.assign(buf.begin() + off, buf.begin() + off + size);
    out.checksum = crc;
    return out;
}

std::vector<Amplitude> decompress(const CompressedChunk &chunk) {
    // metadata checks that do not need the payload body (codec.cpp:187-211)
    if (crc32_of(chunk.payload) != chunk.checksum)
        throw CodecError("checksum mismatch on chunk " + std::to_string(chunk.chunk_index));
    if (chunk.payload.size() < 17) throw CodecError("malformed payload: truncated header");
    const uint8_t id = chunk.payload[0];
    uint32_t count = 0;
    std::memcpy(&count, chunk.payload.data() + 9, 4);
    if (id != 1 && id != 2) throw CodecError("malformed payload: unknown codec id");
    if (id != static_cast<uint8_t>(chunk.codec_id) || count != chunk.element_count)
        throw CodecError("payload header disagrees with chunk metadata");
    std::vector<Amplitude> out(count);
    const uint64_t off = 0;
    const uint32_t size = static_cast<uint32_t>(chunk.payload.size());
    b200::check(qzc_decompress_host(b200::ctx(), chunk.payload.data(), &off, &size, &chunk.checksum, 1,
                                    count, chunk.chunk_index, reinterpret_cast<double *>(out.data())));
    return out;
}

double ratio(const CompressedChunk &chunk) {
    return static_cast<double>(chunk.element_count) * 16.0 / static_cast<double>(chunk.payload.size());
}

} // namespace qzsim
