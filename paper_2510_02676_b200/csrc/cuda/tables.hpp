// tables.hpp -- device decode tables derived from a tensor's code lengths.
//
// Built on the host once per distinct length vector (cached), uploaded with
// the tensor.  Replaces the per-symbol cascade walk of the reference
// (lut.hpp:43-49) with a multi-symbol table:
//
//   fast[i], i = next kFastBits stream bits (MSB first), one uint32:
//     bits  0..4   b  -- total bits consumed by the decoded symbols
//     bits  5..7   n  -- symbols decoded (0..6); 0 = first word is longer
//                        than kFastBits or not determined by them
//     bits  8..31  up to six 4-bit symbols, first symbol lowest
//
// A symbol enters an entry only if the reference cascade would return the
// same (symbol, length) for EVERY completion of the bits not yet seen, and
// its word ends inside the index.  So a fast-table step is bit-for-bit the
// reference's decode_one sequence, fallback symbols for garbage windows
// included.  n == 0 defers to the reference cascade itself (kept in shared
// memory) on a 16-bit window.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

namespace ecf8::dev {

inline constexpr int kFastBits = 12;
inline constexpr int kFastEntries = 1 << kFastBits;
inline constexpr int kMaxPerEntry = 6;

struct DecodeTables {
  std::array<std::uint8_t, 16> lengths{};
  std::vector<std::uint32_t> fast;     // kFastEntries
  std::vector<std::uint8_t> cascade;   // n_luts * 256, reference layout
  std::uint32_t n_luts = 0;
  std::uint64_t lenpack = 0;           // 4 bits per symbol: length & 15 (16 -> 0)
};

// Throws std::invalid_argument("invalid length vector") like the reference.
std::shared_ptr<const DecodeTables> tables_for(const std::uint8_t lengths[16]);

// Uncached builder (tests).
DecodeTables build_tables(const std::uint8_t lengths[16]);

}  // namespace ecf8::dev
