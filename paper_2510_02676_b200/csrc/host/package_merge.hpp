// package_merge.hpp -- length-limited optimal code lengths over N symbols by
// the coin-collector form of package-merge, with the reference's tie rules
// (/root/reference/proj/src/huffman.cpp:43-107): singletons ordered by
// (count, symbol); at each of the L - 1 coarser levels adjacent items pair
// up, an odd leftover drops, and a package sorts before a singleton of equal
// weight.  N = 16 is the reference's E4M3 alphabet (huffman_lut.cpp);
// N = 32 the native E5M2 variant's (e5m2.cpp).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <iterator>
#include <stdexcept>
#include <utility>
#include <vector>

namespace ecf8::host {

template <int N, int L>
std::array<std::uint8_t, N> package_merge_lengths(const std::array<std::uint64_t, N>& counts) {
  struct Coin {
    std::uint64_t weight = 0;
    std::array<std::uint8_t, N> mult{};  // leaf multiplicity per symbol
  };
  std::vector<std::pair<std::uint64_t, int>> live;
  for (int s = 0; s < N; ++s)
    if (counts[s]) live.emplace_back(counts[s], s);
  std::sort(live.begin(), live.end());

  std::vector<Coin> leaves(live.size());
  for (std::size_t i = 0; i < live.size(); ++i) {
    leaves[i].weight = live[i].first;
    leaves[i].mult[live[i].second] = 1;
  }
  const auto lighter = [](const Coin& a, const Coin& b) { return a.weight < b.weight; };
  std::vector<Coin> row = leaves, pairs, merged;
  for (int pass = 1; pass < L; ++pass) {
    pairs.clear();
    for (std::size_t i = 1; i < row.size(); i += 2) {
      Coin c;
      c.weight = row[i - 1].weight + row[i].weight;
      for (int s = 0; s < N; ++s) c.mult[s] = static_cast<std::uint8_t>(row[i - 1].mult[s] + row[i].mult[s]);
      pairs.push_back(c);
    }
    // std::merge keeps the first range ahead on ties: packages win.
    merged.clear();
    std::merge(pairs.begin(), pairs.end(), leaves.begin(), leaves.end(), std::back_inserter(merged), lighter);
    row.swap(merged);
  }
  std::array<std::uint8_t, N> len{};
  const std::size_t keep = 2 * (live.size() - 1);
  if (row.size() < keep) throw std::logic_error("package-merge list too short");
  for (std::size_t i = 0; i < keep; ++i)
    for (int s = 0; s < N; ++s) len[s] = static_cast<std::uint8_t>(len[s] + row[i].mult[s]);
  return len;
}

}  // namespace ecf8::host
