// ecf8/lut.hpp -- host-side cascaded decode table (reference layout).
//
// API of /root/reference/proj/include/ecf8/lut.hpp, kept so existing callers
// and tests that inspect the table keep working: a flat n_luts x 256 byte
// array -- subtable 0 indexed by the first window byte, continuation
// subtables for the <= 16 long-code prefixes (pointer entries 255, 254, ...
// in first-appearance order), the symbol -> length map last; unmatched
// windows resolve to the lowest present symbol.
//
// The B200 kernels do NOT walk this cascade per symbol.  They decode with a
// multi-symbol table (up to six symbols per shared-memory load) derived from
// the same code, and use this cascade only for code words too long for the
// fast table.  Both forms give identical (symbol, bits) for every window --
// tests/test_tables.py checks all 65 536 windows.
#pragma once

#include <cstdint>
#include <vector>

#include "ecf8/huffman.hpp"

namespace ecf8 {

struct CascadedLut {
  std::vector<std::uint8_t> entries;
  std::uint32_t n_luts = 0;
};

inline constexpr std::uint32_t kMaxLuts = 18;
inline constexpr std::uint32_t kFirstPointer = 240;

CascadedLut build_lut(const CodeTable& t);

struct DecodeStep {
  std::uint8_t symbol;
  std::uint8_t bits;
};

// Code word at the head of a 16-bit MSB-aligned window.
inline DecodeStep decode_one(const CascadedLut& lut, std::uint16_t window) {
  const std::uint8_t* tab = lut.entries.data();
  unsigned v = tab[window >> 8];
  if (v >= kFirstPointer) v = tab[((256u - v) << 8) | (window & 0xFFu)];
  return DecodeStep{static_cast<std::uint8_t>(v), tab[((lut.n_luts - 1) << 8) + v]};
}

}  // namespace ecf8
