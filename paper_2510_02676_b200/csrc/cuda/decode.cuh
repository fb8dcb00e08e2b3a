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
  const std::uint32_t* tile_ok;  // bit v: gaps of windows [256v, 256v+256) verified (nullptr: none)
  const std::uint32_t* fsm;      // tables.hpp byte-step decoder (nullptr: the code has none)
  const std::uint8_t* fsm_cm;    // its completion masks
  const std::uint64_t* fsm64;    // 64-bit byte-step decoder for 1-bit codes; set only when every tile is direct (variant 6)
  const std::uint8_t* endgap;    // per window, gap layout: where its reference walk stops, minus 64 (upload check)
  const std::uint16_t* lane_start;   // per 4-window group: first output element, relative to its block's outpos
  const std::uint32_t* tile_direct;  // bit v: tile v's blocks (but the tensor's last) decode to exactly their ranges
  std::uint8_t* out;             // element i lands at out[i - out_offset]
  std::uint64_t out_offset;      // multiple of 16
  std::uint64_t n_elem;
  std::uint64_t blk_begin;       // decode blocks [blk_begin, blk_end)
  std::uint64_t blk_end;
  std::uint64_t lenpack;
  std::uint64_t tile_begin;      // first tile of this desc within its launch
  // Tiled weights (fused layout, 128 x 128 swizzled tiles) decoded back to
  // row-major: out_tiled_k = the row length k (0: elements land linearly);
  // element e goes to its row-major place under `out`, written only for e in
  // [out_lo, out_hi) (the rows a call asked for).
  std::uint64_t out_lo, out_hi;
  std::uint32_t out_tiled_k;
  std::uint32_t all_direct;      // every tile of the tensor is direct (upload check): variant 7
  std::uint32_t T;
  std::uint32_t n_luts;
  std::uint32_t lmin;  // shortest code length (selects the variant)
};

constexpr int kThreads = 256;  // threads of one tile group (a CTA runs several groups)
constexpr std::uint64_t kPad = 64;
// Largest tile of any variant: 1024 windows -> 8 KB encoded, <= 64 Ki elements.
constexpr std::uint64_t kTileBytesMax = 1024 * 8;
constexpr std::uint64_t kTileElemsMax = 1024 * 64;

// Kernel variant.  A thread decodes KWIN consecutive windows (always inside
// one reference block) into a private slot of SLOTW 32-bit words; a tile is
// kThreads * KWIN windows.  A window holds at most ceil(64 / Lmin) symbols
// (every code word, garbage fallbacks included, is >= Lmin bits), so the
// shortest code length of the tensor bounds the slot: Lmin >= 2 allows four
// windows in the slot that two windows need when Lmin == 1.
//
// Variant 4 is the warp-autonomous kernel (decode_warp.cu): one warp owns a
// 256-window tile, eight windows per lane; it needs T in [8, 256] (whole
// blocks per tile, whole lanes per block) and Lmin >= 2.  Variant 5 is the
// same kernel for 1-bit codes: 64-symbol windows double a lane's slot and
// the staging tile, so 12 warps per SM.  Variant 7 is variant 4 for tensors
// whose every tile passed the upload check's direct-placement test: no
// fallback path, the staging tile is the warp's only shared memory.
struct Variant {
  int kwin;
  int slotw;
  int id;        // index into the compiled variants
  int tile_win;  // windows per tile
};

bool warp_variant_enabled();  // false when ECF8_NO_WARP_KERNEL=1 (A/B runs)

// fsm: the code has a byte-step decoder (tables.hpp; complete, Lmin >= 2),
// which variant 4 needs; fsm64: a complete code with a 1-bit word whose
// tensor passed the upload check on every tile (variant 6, byte steps with
// 64-bit entries); other codes with T in [8, 256] take variant 5.
inline Variant variant_for(std::uint32_t T, std::uint32_t lmin, bool fsm = true, bool fsm64 = false, bool direct = false) {
  if (lmin >= 2 && fsm && direct && T >= 8 && T <= 256 && warp_variant_enabled()) return {8, 32, 7, 256};
  if (lmin >= 2 && fsm && T >= 8 && T <= 256 && warp_variant_enabled()) return {8, 32, 4, 256};
  if (lmin == 1 && fsm64 && T >= 8 && T <= 256 && warp_variant_enabled()) return {8, 64, 6, 256};
  if (lmin >= 1 && T >= 8 && T <= 256 && warp_variant_enabled()) return {8, 64, 5, 256};
  if (T == 1) return {1, 8, 0, kThreads};
  if (T == 2) return {2, 16, 1, 2 * kThreads};
  if (lmin >= 2) return {4, 16, 2, 4 * kThreads};
  if (T == 1024) return {4, 32, 3, 4 * kThreads};
  return {2, 16, 1, 2 * kThreads};
}

inline Variant variant_of(const TensorDesc& d) {
  return variant_for(d.T, d.lmin, d.fsm != nullptr, d.fsm64 != nullptr, d.all_direct != 0);
}

inline std::uint64_t blocks_per_tile(std::uint32_t T, int tile_win) {
  const std::uint64_t w = static_cast<std::uint64_t>(tile_win);
  return T >= w ? 1 : w / T;
}

inline std::uint64_t tiles_of(std::uint32_t T, int tile_win, std::uint64_t n_blocks) {
  const std::uint64_t m = blocks_per_tile(T, tile_win);
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

// Gap check of blocks [d.blk_begin, d.blk_end) (whole 256-window tiles;
// tile_ok / endgap indexed by global window number): writes every window's
// end nibble (window_end - 64, endgap) and clears bit v of tile_ok (pre-set
// to all ones) unless every window w in [256v, 256v + 256) that is not the
// last of an 8-window group (w % 8 != 7) ends where window w + 1's gap says.
// Also (T in [8, 256]): every 4-window group's output offset within its
// block (lane_start: the reference's per-block scan, codec.cpp:227-237,
// taken per group of 4 windows), and tile_direct bit v cleared unless every
// block of tile v except the tensor's last (nb_total - 1) decodes to no more
// symbols than its outpos range.
cudaError_t launch_verify_gaps(const TensorDesc& d, std::uint64_t nb_total, std::uint32_t* tile_ok,
                               std::uint8_t* endgap, std::uint16_t* lane_start, std::uint32_t* tile_direct,
                               cudaStream_t stream);

// count_phase on one window (window10 staged as 16 bytes in device memory).
// Only the table fields of `tables` are used.
cudaError_t launch_count_window(const std::uint8_t* d_window16, unsigned gap, const TensorDesc& tables,
                                std::uint32_t* d_count, cudaStream_t stream);

}  // namespace ecf8::dev
