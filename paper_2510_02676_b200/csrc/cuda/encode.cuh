// encode.cuh -- the ECF8 encoder and exponent histogram on the device
// (SURVEY §8f row 4): make_stats' histogram (container.cpp:386-413) and
// encode (codec.cpp:49-98), byte-identical to the host encoder.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ecf8::dev {

constexpr std::uint32_t kEncChunkElems = 4096;  // elements per encode CTA (256 threads x 16)

// counts[16] (device, u64) += exponent histogram of fp8[0, n).
cudaError_t launch_exponent_histogram(const std::uint8_t* fp8, std::uint64_t n, unsigned long long* counts,
                                      cudaStream_t s);

// Pass 1: chunk_bits[c] = code bits of chunk c; *bad |= 1 if a symbol has no
// code.  Pass 2: chunk_start = exclusive scan (u64), *total = sum.
cudaError_t launch_encode_sizes(const std::uint8_t* fp8, std::uint64_t n, const std::uint8_t* lengths16,
                                std::uint32_t* chunk_bits, std::uint64_t* chunk_start, unsigned long long* total,
                                std::uint32_t* bad, cudaStream_t s);

struct EncodeArgs {
  const std::uint8_t* fp8;
  std::uint64_t n;
  const std::uint64_t* chunk_start;
  std::uint32_t* encoded;  // zeroed, 4-byte aligned
  std::uint32_t* gaps;     // zeroed, 4-byte aligned, padded to whole words
  std::uint64_t* outpos;   // zeroed, n_blocks + 1
  std::uint8_t* packed;    // 8-byte aligned
  std::uint64_t n_blocks;
  std::uint32_t log2T;
  std::uint32_t lc[16];  // code << (32 - length) | length (0 for absent symbols)
};
// Pass 3: bitstream, gaps, outpos and packed nibbles.
cudaError_t launch_encode_emit(const EncodeArgs& a, cudaStream_t s);

// Row-major [n, k] FP8 bytes <-> the fused GEMM's tiled, swizzled layout.
cudaError_t launch_fused_layout(const std::uint8_t* in, std::uint64_t n, std::uint64_t k, std::uint8_t* out,
                                bool inverse, cudaStream_t s);

}  // namespace ecf8::dev
