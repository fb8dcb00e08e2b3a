// tables.hpp -- device decode tables derived from a tensor's code lengths.
//
// Built on the host once per distinct length vector (cached), uploaded once
// per device.  Replaces the per-symbol cascade walk of the reference
// (lut.hpp:43-49) with a multi-symbol table indexed by the next kFastBits
// stream bits (MSB first):
//
//   fast[i] (uint32)
//     bits  0..4   b   -- bits consumed by the decoded symbols (<= 12)
//     bits  5..9   n4  -- 4 * symbols decoded (0..5 symbols); 0 = the first
//                         word is longer than kFastBits or undetermined
//     bits 12..31  up to five 4-bit symbols, first symbol lowest
//   smask[i] (uint16)  bit j set iff one of those symbols starts at offset j
//
// A symbol enters an entry only if the reference cascade returns the same
// (symbol, length) for EVERY completion of the bits not yet seen and its word
// ends inside the index, so a fast step is bit-for-bit the reference's
// decode_one sequence, garbage-window fallback symbols included.  smask lets
// the kernel take exactly the symbols that start before a window's 64-bit
// boundary (the reference's count/emit rule, codec.cpp:143-160) in one
// popcount.  n4 == 0 defers to the reference cascade (kept in shared memory)
// on a 16-bit window.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

namespace ecf8::dev {

inline constexpr int kFastBits = 12;
inline constexpr int kFsmStates = 16;  // internal nodes of a complete 16-symbol code tree: <= 15
inline constexpr int kFastEntries = 1 << kFastBits;
inline constexpr int kMaxPerEntry = 5;

struct DecodeTables {
  std::array<std::uint8_t, 16> lengths{};
  std::vector<std::uint32_t> fast;     // kFastEntries
  std::vector<std::uint16_t> smask;    // kFastEntries
  std::vector<std::uint8_t> cascade;   // n_luts * 256, reference layout
  std::uint32_t n_luts = 0;
  std::uint64_t lenpack = 0;           // 4 bits per symbol: length & 15 (16 -> 0)
  // Byte-step decoder (finite-state machine over the code tree), available
  // when the code is complete (Kraft sum 1: every bit string parses) and
  // every word is >= 2 bits (<= 4 words complete per input byte).  A state is
  // an internal node of the code tree (the pending prefix; 0 = root, i.e. at
  // a code boundary).  fsm[state * 256 + byte] (uint32):
  //   bits  0..4   n4 = 4 * (code words completed by the byte, MSB first), <= 16
  //   bits  8..11  next state
  //   bits 16..31  the completed words' symbols, first lowest (4 bits each)
  // fsm_cm[state * 256 + byte]: bit i set iff a word completes at bit i of
  // the byte (bit 0 = the byte's most significant bit).
  bool fsm_ok = false;
  std::vector<std::uint32_t> fsm;     // kFsmStates * 256 (zeros when !fsm_ok)
  std::vector<std::uint8_t> fsm_cm;   // kFsmStates * 256
  // The same state machine for complete codes with a 1-bit word (up to 8
  // words per byte): fsm64[state * 256 + byte] (uint64)
  //   bits  0..31  the completed words' symbols, first lowest (4 bits each)
  //   bits 32..37  n4 = 4 * words completed (<= 32)
  //   bits 40..43  next state
  bool fsm64_ok = false;
  std::vector<std::uint64_t> fsm64;   // kFsmStates * 256 (empty when !fsm64_ok)
};

// Throws std::invalid_argument("invalid length vector") like the reference.
std::shared_ptr<const DecodeTables> tables_for(const std::uint8_t lengths[16]);

// Uncached builder (tests).
DecodeTables build_tables(const std::uint8_t lengths[16]);

}  // namespace ecf8::dev
