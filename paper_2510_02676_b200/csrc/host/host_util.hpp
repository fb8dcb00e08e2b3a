// host_util.hpp -- glue between the C++ API and the C ABI (internal).
#pragma once

#include <stdexcept>
#include <string>

#include "ecf8/codec.hpp"
#include "ecf8/container.hpp"
#include "ecf8/errors.hpp"
#include "ecf8_cuda.h"

namespace ecf8::host {

// Rethrow a C-ABI status as the exception type the reference API uses.
inline void check(int status) {
  if (status == ECF8_OK) return;
  const std::string msg = ecf8_last_error();
  switch (status) {
    case ECF8_EINVAL: throw std::invalid_argument(msg);
    case ECF8_EFORMAT: throw FormatError(msg);
    case ECF8_EIO: throw IoError(msg);
    default: throw std::runtime_error("ecf8: " + msg);
  }
}

inline ecf8_sections sections_of(const EncodedTensor& t) {
  ecf8_sections s{};
  s.n_elem = t.stream.n_elem;
  s.threads_per_block = t.stream.geometry.threads_per_block;
  for (int i = 0; i < 16; ++i) s.lengths[i] = t.stream.lengths[i];
  s.encoded = t.stream.encoded.data();
  s.encoded_len = t.stream.encoded.size();
  s.gaps = t.stream.gaps.data();
  s.gaps_len = t.stream.gaps.size();
  s.outpos = t.stream.outpos.data();
  s.n_outpos = t.stream.outpos.size();
  s.packed = t.packed.data();
  s.packed_len = t.packed.size();
  return s;
}

// The cascade's last subtable is the symbol -> length map (lut.hpp).
inline void lengths_from_lut(const CascadedLut& lut, std::uint8_t lengths[16]) {
  if (lut.n_luts < 2 || lut.entries.size() < std::size_t{256} * lut.n_luts)
    throw std::invalid_argument("invalid length vector");
  const std::uint8_t* m = lut.entries.data() + std::size_t{256} * (lut.n_luts - 1);
  for (int s = 0; s < 16; ++s) lengths[s] = m[s];
}

// decompress_streaming straight from container bytes (no parse copies).
DecompressStats decompress_bytes(std::span<const std::uint8_t> bytes, std::ostream& out);

}  // namespace ecf8::host
