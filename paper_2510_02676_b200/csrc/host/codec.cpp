// codec.cpp -- host encoder, the reference-API sequential oracle, and the
// C++ wrappers that route every parallel decode through the B200 C ABI.
//
// Bitstream semantics (must stay byte-identical to the reference encoder,
// /root/reference/proj/src/codec.cpp:49-98): codes concatenated MSB-first,
// tail zero-padded to whole windows plus 2 lookahead bytes; window w's gap
// is the in-window start bit of the first code that *starts* in w (0 when
// none does); outpos[b+1] counts the codes starting in windows of blocks
// <= b.
#include <algorithm>
#include <bit>
#include <stdexcept>

#include "ecf8/codec.hpp"
#include "ecf8/errors.hpp"
#include "ecf8_cuda.h"
#include "host_util.hpp"

namespace ecf8 {

BlockGeometry make_geometry(std::uint64_t bitstream_bytes, std::uint32_t threads_per_block) {
  if (threads_per_block < 1 || threads_per_block > 1024 || !std::has_single_bit(threads_per_block))
    throw std::invalid_argument("threads per block must be a power of two in [1, 1024]");
  BlockGeometry g;
  g.threads_per_block = threads_per_block;
  const std::uint64_t bb = g.block_bytes();
  g.n_blocks = bitstream_bytes / bb + (bitstream_bytes % bb != 0);
  return g;
}

EncodedStream encode(std::span<const ExponentSymbol> exponents, const CodeTable& table,
                     std::uint32_t threads_per_block) {
  std::uint64_t bits = 0;
  for (ExponentSymbol s : exponents) {
    if (!table.has(s)) throw std::invalid_argument("symbol absent from code table");
    bits += table.lengths[s];
  }
  EncodedStream out;
  out.n_elem = exponents.size();
  out.lengths = table.lengths;
  out.geometry = make_geometry((bits + 7) / 8, threads_per_block);
  const std::uint32_t T = out.geometry.threads_per_block;
  const std::uint64_t windows = out.geometry.thread_count();
  out.encoded.assign(out.geometry.window_bytes() + BlockGeometry::kLookaheadBytes, 0);
  out.gaps.assign((windows + 1) / 2, 0);
  out.outpos.assign(out.geometry.n_blocks + 1, 0);

  // 64-bit MSB-first accumulator flushed a byte at a time.
  std::uint64_t buf = 0;
  unsigned fill = 0;
  std::uint8_t* dst = out.encoded.data();
  std::uint64_t pos = 0;
  std::uint64_t owner = ~std::uint64_t{0};
  for (ExponentSymbol s : exponents) {
    const std::uint64_t w = pos >> 6;
    if (w != owner) {
      owner = w;
      out.gaps[w >> 1] |= static_cast<std::uint8_t>((pos & 63) << ((w & 1) ? 0 : 4));
    }
    out.outpos[w / T + 1] += 1;
    const unsigned len = table.lengths[s];
    buf = (buf << len) | table.codes[s];
    fill += len;
    pos += len;
    while (fill >= 8) {
      fill -= 8;
      *dst++ = static_cast<std::uint8_t>(buf >> fill);
    }
  }
  if (fill) *dst = static_cast<std::uint8_t>(buf << (8 - fill));
  for (std::size_t b = 1; b < out.outpos.size(); ++b) out.outpos[b] += out.outpos[b - 1];
  return out;
}

EncodedTensor encode_tensor(std::span<const Fp8Byte> fp8, const CodeTable& table,
                            std::uint32_t threads_per_block) {
  std::vector<ExponentSymbol> x;
  std::vector<SignMantissaNibble> q;
  split_bytes(fp8, x, q);
  EncodedTensor t;
  t.stream = encode(x, table, threads_per_block);
  t.packed = pack_nibbles(q);
  return t;
}

std::vector<ExponentSymbol> decode_sequential(const EncodedStream& s, const CascadedLut& lut) {
  std::vector<ExponentSymbol> out(s.n_elem);
  const std::uint8_t* buf = s.encoded.data();
  const std::uint64_t nbytes = s.encoded.size();
  const std::uint64_t cap = nbytes * 8;
  std::uint64_t pos = 0;
  for (std::uint64_t i = 0; i < s.n_elem; ++i) {
    if (pos >= cap) throw FormatError("truncated stream");
    const std::uint64_t k = pos >> 3;
    std::uint32_t w24 = 0;
    for (std::uint64_t j = 0; j < 3; ++j) w24 = (w24 << 8) | (k + j < nbytes ? buf[k + j] : 0u);
    const DecodeStep d = decode_one(lut, static_cast<std::uint16_t>(w24 >> (8 - (pos & 7))));
    out[i] = d.symbol;
    pos += d.bits;
  }
  return out;
}

std::vector<Fp8Byte> decode_reference(const EncodedTensor& t, const CascadedLut& lut) {
  const std::vector<ExponentSymbol> x = decode_sequential(t.stream, lut);
  std::vector<Fp8Byte> out(x.size());
  for (std::uint64_t i = 0; i < out.size(); ++i) out[i] = assemble(x[i], nibble_high(t.packed, i));
  return out;
}

// ------------------------------------------------- B200-routed functions

std::uint32_t count_phase(std::span<const std::uint8_t, 10> window10, unsigned gap,
                          const CascadedLut& lut) {
  std::uint8_t lengths[16];
  host::lengths_from_lut(lut, lengths);
  std::uint32_t c = 0;
  host::check(ecf8_count_window(window10.data(), gap, lengths, &c));
  return c;
}

void BlockScratch::resize(const BlockGeometry& g) {
  counts.resize(g.threads_per_block);
  accum.resize(g.threads_per_block);
  staging.resize(std::size_t{g.threads_per_block} * BlockGeometry::kMaxSymbolsPerWindow);
}

void decode_block(const EncodedTensor& t, const CascadedLut& lut, std::uint64_t block,
                  std::span<Fp8Byte> out, BlockScratch& scratch,
                  std::span<const std::uint32_t> phase1_order,
                  std::span<const std::uint32_t> phase2_order) {
  (void)lut;  // the device rebuilds its tables from the stream's lengths
  (void)scratch;
  const std::uint32_t T = t.stream.geometry.threads_per_block;
  for (auto order : {phase1_order, phase2_order}) {
    if (order.empty()) continue;
    std::vector<bool> seen(T, false);
    if (order.size() != T) throw std::invalid_argument("thread order must be a permutation");
    for (std::uint32_t v : order) {
      if (v >= T || seen[v]) throw std::invalid_argument("thread order must be a permutation");
      seen[v] = true;
    }
  }
  const ecf8_sections sec = host::sections_of(t);
  host::check(ecf8_decode_block_host(&sec, block, out.data(), out.size()));
}

void decode_parallel_into(const EncodedTensor& t, const CascadedLut& lut, std::span<Fp8Byte> out) {
  // The reference decodes with the caller's LUT (codec.cpp:256-273); the
  // device rebuilds the same tables from the LUT's symbol->length map.
  ecf8_sections sec = host::sections_of(t);
  host::lengths_from_lut(lut, sec.lengths);
  host::check(ecf8_decode_host(&sec, out.data(), out.size()));
}

std::vector<Fp8Byte> decode_parallel(const EncodedTensor& t, const CascadedLut& lut) {
  std::vector<Fp8Byte> out(t.stream.n_elem);
  decode_parallel_into(t, lut, out);
  return out;
}

}  // namespace ecf8
