// decode.cuh -- device descriptors and launchers for the ECF8 decode kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ecf8::dev {

// One tensor (or one block range of it) in a decode launch.  All pointers
// are device memory.  encoded / gaps / packed carry >= 64 zero bytes of
// padding so the kernels may over-read by whole 16-byte vectors.
struct TensorDesc {
  const std::uint8_t* encoded;
  const std::uint8_t* gaps;
  const std::uint64_t* outpos;
  const std::uint8_t* packed;
  const std::uint32_t* fast;     // tables.hpp fast table
  const std::uint16_t* smask;    // tables.hpp start masks
  const std::uint8_t* cascade;   // reference cascade (slow path)
  std::uint8_t* out;             // element i lands at out[i - out_offset]
  std::uint64_t out_offset;      // multiple of 16
  std::uint64_t n_elem;
  std::uint64_t blk_begin;       // decode blocks [blk_begin, blk_end)
  std::uint64_t blk_end;
  std::uint64_t lenpack;
  std::uint64_t tile_begin;      // first tile of this desc within its launch
  std::uint32_t T;
  std::uint32_t n_luts;
  std::uint32_t lmin;  // shortest code length (selects the variant)
};

constexpr int kThreads = 256;  // threads of one tile group (a CTA runs several groups)
constexpr std::uint64_t kPad = 64;

// Kernel variant.  A thread decodes KWIN consecutive windows (always inside
// one reference block) into a private slot of SLOTW 32-bit words; a tile is
// kThreads * KWIN windows.  A window holds at most ceil(64 / Lmin) symbols
// (every code word, garbage fallbacks included, is >= Lmin bits), so the
// shortest code length of the tensor bounds the slot: Lmin >= 2 allows four
// windows in the slot that two windows need when Lmin == 1.
struct Variant {
  int kwin;
  int slotw;
  int id;  // index into the compiled variants
};

inline Variant variant_for(std::uint32_t T, std::uint32_t lmin) {
  if (T == 1) return {1, 8, 0};
  if (T == 2) return {2, 16, 1};
  if (lmin >= 2) return {4, 16, 2};
  if (T == 1024) return {4, 32, 3};
  return {2, 16, 1};
}

inline std::uint64_t blocks_per_tile(std::uint32_t T, int kwin) {
  const std::uint64_t w = static_cast<std::uint64_t>(kThreads) * kwin;
  return T >= w ? 1 : w / T;
}

inline std::uint64_t tiles_of(std::uint32_t T, int kwin, std::uint64_t n_blocks) {
  const std::uint64_t m = blocks_per_tile(T, kwin);
  return (n_blocks + m - 1) / m;
}

// Kernel parameters: either a device array of descriptors (batched, tile
// ranges given by tile_begin) or, when descs == nullptr, one descriptor
// passed by value (no host->device copy on the single-tensor path).
struct LaunchArgs {
  const TensorDesc* descs;
  int n_desc;
  std::uint64_t total_tiles;
  TensorDesc inline_desc;
};

// One decode launch; every descriptor was prepared for variant `variant`.
cudaError_t launch_decode(const LaunchArgs& args, int variant, cudaStream_t stream);

// count_phase on one window (window10 staged as 16 bytes in device memory).
cudaError_t launch_count_window(const std::uint8_t* d_window16, unsigned gap,
                                const std::uint32_t* d_fast, const std::uint16_t* d_smask,
                                const std::uint8_t* d_cascade, std::uint32_t n_luts,
                                std::uint32_t* d_count, cudaStream_t stream);

}  // namespace ecf8::dev
