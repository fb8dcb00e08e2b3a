// tables.cpp -- host builder for the device decode tables (see tables.hpp).
#include "tables.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <stdexcept>

#include "ecf8/huffman.hpp"
#include "ecf8/lut.hpp"

namespace ecf8::dev {

namespace {
constexpr std::uint16_t kUndetermined = 0xFFFF;

inline std::uint16_t pack_step(unsigned sym, unsigned len) {
  return static_cast<std::uint16_t>(sym | (len << 4));
}
// The byte-step state machine of tables.hpp: walk the code tree bit by bit
// (MSB first), emitting a symbol at every leaf.  The tree is the canonical
// code's (huffman.cpp:131-157 word assignment), so a complete code parses
// any bit string exactly as the reference's decode_one chain does
// (lut.hpp:43-49; every 16-bit window then starts with a whole code word).
void build_fsm(const CodeTable& code, DecodeTables& t) {
  t.fsm.assign(kFsmStates * 256, 0);
  t.fsm_cm.assign(kFsmStates * 256, 0);
  t.fsm_ok = false;
  t.fsm64_ok = false;
  t.fsm64.clear();
  // leaf[(len, word)] = symbol; node ids for proper prefixes of words
  std::map<std::pair<int, std::uint32_t>, int> leaf, node;
  double kraft = 0;
  int lmin = 17, present = 0;
  for (int s = 0; s < 16; ++s) {
    const int l = code.lengths[s];
    if (!l) continue;
    ++present;
    lmin = std::min(lmin, l);
    kraft += std::ldexp(1.0, -l);
    leaf[{l, code.codes[s]}] = s;
  }
  if (present < 2 || kraft != 1.0) return;
  const bool wide = lmin < 2;  // a 1-bit word: up to 8 words per byte -> 64-bit entries
  if (wide) t.fsm64.assign(kFsmStates * 256, 0);
  node[{0, 0}] = 0;
  for (int l = 1; l <= 16; ++l)  // breadth-first ids
    for (const auto& [k, s] : leaf)
      if (k.first > l) {
        const std::pair<int, std::uint32_t> pre{l, k.second >> (k.first - l)};
        if (!node.count(pre)) node.emplace(pre, static_cast<int>(node.size()));
      }
  if (node.size() > static_cast<std::size_t>(kFsmStates)) return;
  for (const auto& [pre, id] : node) {
    for (std::uint32_t b = 0; b < 256; ++b) {
      int l = pre.first;
      std::uint32_t v = pre.second, syms = 0, cm = 0, n = 0;
      for (int i = 0; i < 8; ++i) {
        ++l;
        v = (v << 1) | ((b >> (7 - i)) & 1u);
        auto f = leaf.find({l, v});
        if (f != leaf.end()) {
          if (!wide && n == 4) return;  // cannot happen with words >= 2 bits
          syms |= static_cast<std::uint32_t>(f->second) << (4 * n);
          cm |= 1u << i;
          ++n;
          l = 0;
          v = 0;
        } else if (!node.count({l, v})) {
          return;  // not a prefix of any word: the code is incomplete
        }
      }
      const std::uint32_t next = static_cast<std::uint32_t>(node.at({l, v}));
      if (wide)
        t.fsm64[id * 256 + b] = syms | (std::uint64_t{4 * n} << 32) | (std::uint64_t{next} << 40);
      else
        t.fsm[id * 256 + b] = (4 * n) | (next << 8) | (syms << 16);
      t.fsm_cm[id * 256 + b] = static_cast<std::uint8_t>(cm);
    }
  }
  if (wide) t.fsm64_ok = true;
  else t.fsm_ok = true;
}
}  // namespace

DecodeTables build_tables(const std::uint8_t lengths[16]) {
  std::array<std::uint8_t, 16> len{};
  for (int s = 0; s < 16; ++s) len[s] = lengths[s];
  const CodeTable code = canonical_codes(len);  // validates cap + Kraft
  const CascadedLut lut = build_lut(code);

  DecodeTables t;
  t.lengths = len;
  t.cascade = lut.entries;
  t.n_luts = lut.n_luts;
  for (int s = 0; s < 16; ++s) t.lenpack |= std::uint64_t{len[s] & 15u} << (4 * s);

  // same[r][v]: the cascade's (symbol, length) common to every 16-bit window
  // whose first r bits are v, or kUndetermined.  r = 16 is the cascade
  // itself; coarser prefixes agree when both halves agree.
  std::vector<std::vector<std::uint16_t>> same(17);
  same[16].resize(1u << 16);
  for (std::uint32_t w = 0; w < (1u << 16); ++w) {
    const DecodeStep d = decode_one(lut, static_cast<std::uint16_t>(w));
    same[16][w] = pack_step(d.symbol, d.bits);
  }
  for (int r = 15; r >= 1; --r) {
    same[r].resize(1u << r);
    const auto& fine = same[r + 1];
    for (std::uint32_t v = 0; v < (1u << r); ++v) {
      const std::uint16_t a = fine[2 * v], b = fine[2 * v + 1];
      same[r][v] = (a == b) ? a : kUndetermined;
    }
  }

  build_fsm(code, t);

  t.fast.resize(kFastEntries);
  t.smask.resize(kFastEntries);
  for (std::uint32_t idx = 0; idx < static_cast<std::uint32_t>(kFastEntries); ++idx) {
    unsigned pos = 0, n = 0;
    std::uint32_t syms = 0, starts = 0;
    while (n < kMaxPerEntry && pos < static_cast<unsigned>(kFastBits)) {
      const unsigned r = kFastBits - pos;            // visible bits left
      const std::uint32_t v = idx & ((1u << r) - 1);  // they are idx's low r bits
      const std::uint16_t st = same[r][v];
      if (st == kUndetermined) break;
      const unsigned sym = st & 15, l = st >> 4;
      if (l == 0 || l > r) break;  // word runs past what the index shows
      syms |= sym << (4 * n);
      starts |= 1u << pos;
      ++n;
      pos += l;
    }
    t.fast[idx] = pos | ((4 * n) << 5) | (syms << 12);
    t.smask[idx] = static_cast<std::uint16_t>(starts);
  }
  return t;
}

std::shared_ptr<const DecodeTables> tables_for(const std::uint8_t lengths[16]) {
  static std::mutex mu;
  static std::map<std::array<std::uint8_t, 16>, std::shared_ptr<const DecodeTables>> cache;
  std::array<std::uint8_t, 16> key{};
  for (int s = 0; s < 16; ++s) key[s] = lengths[s];
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  auto built = std::make_shared<const DecodeTables>(build_tables(lengths));
  std::lock_guard<std::mutex> lock(mu);
  return cache.emplace(key, std::move(built)).first->second;
}

}  // namespace ecf8::dev
