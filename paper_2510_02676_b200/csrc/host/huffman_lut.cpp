// huffman_lut.cpp -- code construction and the host cascaded table.
//
// build_code: length-limited optimal lengths by the coin-collector form of
// package-merge.  Tie rule and pairing follow /root/reference/proj/src/
// huffman.cpp:43-107 exactly (singletons ordered by (count, symbol); at each
// of the 15 coarser levels adjacent items pair up, an odd leftover drops,
// and a package sorts before a singleton of equal weight), so the lengths --
// and hence containers -- are byte-identical to the reference's.
// build_lut: lut.cpp:47-97 layout (see ecf8/lut.hpp).
#include <algorithm>
#include <iterator>
#include <stdexcept>
#include <vector>

#include "ecf8/huffman.hpp"
#include "ecf8/lut.hpp"
#include "package_merge.hpp"

namespace ecf8 {

int CodeTable::present_count() const {
  return static_cast<int>(std::count_if(lengths.begin(), lengths.end(),
                                        [](std::uint8_t l) { return l != 0; }));
}

int CodeTable::max_length() const { return *std::max_element(lengths.begin(), lengths.end()); }

namespace {

std::array<std::uint8_t, kNumSymbols> coin_collector_lengths(const ExponentHistogram& h) {
  std::array<std::uint64_t, kNumSymbols> c{};
  for (int s = 0; s < kNumSymbols; ++s) c[s] = h.counts[s];
  return host::package_merge_lengths<kNumSymbols, kMaxCodeLength>(c);
}

}  // namespace

CodeTable build_code(const ExponentHistogram& h) {
  if (h.total() == 0) throw std::invalid_argument("empty input");
  int present = 0, last = -1;
  for (int s = 0; s < kNumSymbols; ++s)
    if (h.counts[s]) {
      ++present;
      last = s;
    }
  std::array<std::uint8_t, kNumSymbols> len{};
  if (present == 1)
    len[last] = 1;  // a zero-length word would never advance a decoder
  else
    len = coin_collector_lengths(h);
  return canonical_codes(len);
}

CodeTable canonical_codes(const std::array<std::uint8_t, kNumSymbols>& lengths) {
  std::uint64_t kraft = 0;  // units of 2^-16
  bool any = false;
  for (std::uint8_t l : lengths) {
    if (l == 0) continue;
    if (l > kMaxCodeLength) throw std::invalid_argument("invalid length vector");
    kraft += std::uint64_t{1} << (kMaxCodeLength - l);
    any = true;
  }
  if (!any || kraft > (std::uint64_t{1} << kMaxCodeLength))
    throw std::invalid_argument("invalid length vector");

  CodeTable t;
  t.lengths = lengths;
  std::uint32_t next = 0;  // next free word at the current length
  int cur_len = 0;
  for (int l = 1; l <= kMaxCodeLength; ++l) {
    for (int s = 0; s < kNumSymbols; ++s) {
      if (lengths[s] != l) continue;
      if (cur_len != 0) next <<= (l - cur_len);
      cur_len = l;
      t.codes[s] = static_cast<std::uint16_t>(next);
      ++next;
    }
  }
  return t;
}

double expected_length(const CodeTable& t, const ExponentHistogram& h) {
  const std::uint64_t n = h.total();
  if (n == 0) throw std::invalid_argument("empty input");
  std::uint64_t bits = 0;
  for (int s = 0; s < kNumSymbols; ++s) {
    if (!h.counts[s]) continue;
    if (!t.has(static_cast<unsigned>(s))) throw std::invalid_argument("symbol absent from code table");
    bits += h.counts[s] * t.lengths[s];
  }
  return static_cast<double>(bits) / static_cast<double>(n);
}

// ----------------------------------------------------------- cascaded LUT

CascadedLut build_lut(const CodeTable& t) {
  int fallback = -1;
  std::uint64_t kraft = 0;
  for (int s = 0; s < kNumSymbols; ++s) {
    const int l = t.lengths[s];
    if (!l) continue;
    if (l > kMaxCodeLength) throw std::invalid_argument("invalid length vector");
    kraft += std::uint64_t{1} << (kMaxCodeLength - l);
    if (fallback < 0) fallback = s;
  }
  if (fallback < 0 || kraft > (std::uint64_t{1} << kMaxCodeLength))
    throw std::invalid_argument("invalid length vector");

  // Fill the root by painting each short word over the bytes it prefixes
  // (lowest symbol wins, as in a first-match scan), then mark long-word
  // first bytes as pointers in byte order.
  std::array<int, 256> root;
  root.fill(-1);
  for (int s = kNumSymbols - 1; s >= 0; --s) {
    const int l = t.lengths[s];
    if (l < 1 || l > 8) continue;
    const unsigned lo = static_cast<unsigned>(t.codes[s]) << (8 - l);
    for (unsigned b = lo; b < lo + (1u << (8 - l)); ++b) root[b] = s;
  }
  std::array<bool, 256> long_first{};
  for (int s = 0; s < kNumSymbols; ++s) {
    const int l = t.lengths[s];
    if (l > 8) long_first[t.codes[s] >> (l - 8)] = true;
  }
  std::vector<unsigned> prefix;  // continuation subtables in byte order
  std::array<std::uint8_t, 256> rootb{};
  for (unsigned b = 0; b < 256; ++b) {
    if (root[b] >= 0) {
      rootb[b] = static_cast<std::uint8_t>(root[b]);
    } else if (long_first[b]) {
      prefix.push_back(b);
      if (prefix.size() > 16) throw std::runtime_error("pointer space exhausted");
      rootb[b] = static_cast<std::uint8_t>(256 - prefix.size());  // 255, 254, ...
    } else {
      rootb[b] = static_cast<std::uint8_t>(fallback);
    }
  }

  CascadedLut lut;
  lut.n_luts = static_cast<std::uint32_t>(prefix.size() + 2);
  lut.entries.assign(std::size_t{256} * lut.n_luts, 0);
  std::copy(rootb.begin(), rootb.end(), lut.entries.begin());
  for (std::size_t i = 0; i < prefix.size(); ++i) {
    std::uint8_t* sub = lut.entries.data() + 256 * (i + 1);
    std::fill(sub, sub + 256, static_cast<std::uint8_t>(fallback));
    for (int s = kNumSymbols - 1; s >= 0; --s) {
      const int l = t.lengths[s];
      if (l <= 8 || static_cast<unsigned>(t.codes[s] >> (l - 8)) != prefix[i]) continue;
      const unsigned tail = t.codes[s] & ((1u << (l - 8)) - 1);
      const unsigned lo = tail << (16 - l);
      for (unsigned b2 = lo; b2 < lo + (1u << (16 - l)); ++b2) sub[b2] = static_cast<std::uint8_t>(s);
    }
  }
  std::uint8_t* len_map = lut.entries.data() + 256 * (lut.n_luts - 1);
  for (int s = 0; s < kNumSymbols; ++s) len_map[s] = t.lengths[s];
  return lut;
}

}  // namespace ecf8
