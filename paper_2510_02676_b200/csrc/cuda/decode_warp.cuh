// decode_warp.cuh -- the per-warp ECF8 tile decode shared by the standalone
// decode kernel (decode_warp.cu) and the decode-fused GEMM (fused_gemm.cu).
//
// A warp owns a tile of 32 * LW consecutive 64-bit windows = 32*LW/T whole
// reference blocks, LW windows per lane.  A window holds at most
// ceil(64 / Lmin) symbols, so a lane's 32-word (256-nibble) slot takes
//   LW = 8 windows when the shortest code Lmin >= 2 (T in [8, 256]),
//   LW = 4 windows when Lmin == 1 (T in [4, 128]).
// warp_decode_scan() walks each lane's windows into its nibble slot and
// returns the lane's clamped output run relative to the tile's first element
// -- codec.cpp:201-253 (count, scan, clamp) restated per warp with the block
// offsets taken from outpos[].
#pragma once

#include <cstdint>

#include "decode.cuh"
#include "decode_common.cuh"

namespace ecf8::dev {

constexpr int kLaneWin = 8;     // windows per lane (Lmin >= 2)
constexpr int kSlotWords = 32;  // 256 nibbles: 8 windows x 32 or 4 x 64 symbols

template <int LW>
struct WarpInT {
  uint4 w01, w23, w45, w67;  // window bytes (little-endian 32-bit words)
  uint2 w8;                  // first 8 bytes of the next window (lookahead)
  std::uint32_t gaps;        // 8 gap nibbles, window 2j in the high nibble of byte j
  std::uint64_t A, E;        // tile output range
  std::uint64_t o0, o1;      // my reference block's output range
  std::uint32_t nblk, nwin;
  std::uint64_t b0;
};
using WarpIn = WarpInT<kLaneWin>;

// A tile's inputs in two halves: the window words and gaps (issued early,
// they fly while the previous tile is written back), and the block offsets.
template <int LW>
__device__ __forceinline__ void load_tile_words(const TensorDesc& d, std::uint64_t tile, std::uint32_t log2T,
                                                int lane, WarpInT<LW>& in) {
  const std::uint32_t m = (32u * LW) >> log2T;  // blocks per tile
  in.b0 = d.blk_begin + (tile - d.tile_begin) * m;
  in.nblk = static_cast<std::uint32_t>(d.blk_end - in.b0 < m ? d.blk_end - in.b0 : m);
  in.nwin = in.nblk << log2T;
  const std::uint64_t w0g = in.b0 << log2T;
  const std::uint32_t wl = static_cast<std::uint32_t>(lane) * LW;
  if (wl < in.nwin) {
    const uint4* src = reinterpret_cast<const uint4*>(d.encoded + 8 * (w0g + wl));
    in.w01 = __ldg(src);
    in.w23 = __ldg(src + 1);
    if constexpr (LW == 8) {
      in.w45 = __ldg(src + 2);
      in.w67 = __ldg(src + 3);
      in.w8 = __ldg(reinterpret_cast<const uint2*>(src + 4));
      in.gaps = __ldg(reinterpret_cast<const std::uint32_t*>(d.gaps + (w0g >> 1)) + lane);
    } else {
      static_assert(LW == 4, "4 or 8 windows per lane");
      in.w8 = __ldg(reinterpret_cast<const uint2*>(src + 2));
      in.gaps = __ldg(reinterpret_cast<const std::uint16_t*>(d.gaps + (w0g >> 1)) + lane);
    }
  }
}

template <int LW>
__device__ __forceinline__ void load_tile_meta(const TensorDesc& d, std::uint32_t log2T, int lane, WarpInT<LW>& in) {
  const std::uint32_t wl = static_cast<std::uint32_t>(lane) * LW;
  in.A = __ldg(d.outpos + in.b0);
  in.E = __ldg(d.outpos + in.b0 + in.nblk);
  if (wl < in.nwin) {
    const std::uint32_t bl = wl >> log2T;
    in.o0 = __ldg(d.outpos + in.b0 + bl);
    in.o1 = __ldg(d.outpos + in.b0 + bl + 1);
  } else {
    in.o0 = in.o1 = in.E;
  }
}

template <int LW>
__device__ __forceinline__ void load_warp_tile(const TensorDesc& d, std::uint64_t tile, std::uint32_t log2T,
                                               int lane, WarpInT<LW>& in) {
  load_tile_words(d, tile, log2T, lane, in);
  load_tile_meta(d, log2T, lane, in);
}

// Were the gaps of the windows of this warp tile verified (verify_gaps_kernel)?
// tile_ok bit v covers the boundaries after windows [256v, 256v + 256).
template <int LW>
__device__ __forceinline__ bool tile_verified(const TensorDesc& d, const WarpInT<LW>& in, std::uint32_t log2T) {
  if (!d.tile_ok || in.nwin == 0) return false;
  const std::uint64_t w0 = in.b0 << log2T;
  const std::uint64_t v0 = w0 >> 8, v1 = (w0 + in.nwin - 1) >> 8;
  const std::uint32_t a = __ldg(d.tile_ok + (v0 >> 5)) >> (v0 & 31);
  const std::uint32_t b = __ldg(d.tile_ok + (v1 >> 5)) >> (v1 & 31);
  return (a & b & 1u) != 0;
}

struct LaneRun {
  std::uint32_t cnt;    // symbols this lane decoded (reference count rule)
  std::uint32_t start;  // first output element, relative to the tile's A
  std::uint32_t len;    // symbols kept after the block clamp
};

// Decode this lane's windows into its slot (word j of the run at shared
// address slot_base + j * WS; nibble i of the run in bits 4(i%8).. of word
// i/8), then scan + clamp across the warp.  verified (the tile passed the
// upload-time gap check): one continuous walk over the lane's windows;
// otherwise, or when the walk met a flagged entry, window by window with the
// reference's per-window semantics (fast table, exact walk where flagged).
template <int LW, int WS = 4>
__device__ __forceinline__ LaneRun warp_decode_scan(const WarpInT<LW>& in, std::uint32_t log2T,
                                                   std::uint32_t len_off, const Tables& tb, std::uint32_t slot_base,
                                                   int lane, bool verified = false) {
  const std::uint32_t wl0 = static_cast<std::uint32_t>(lane) * LW;
  const bool active = wl0 < in.nwin;
  SlotSinkT<WS> sink{slot_base};
  if (active) {
    std::uint32_t w[2 * LW + 2];
    w[0] = bswap32(in.w01.x), w[1] = bswap32(in.w01.y), w[2] = bswap32(in.w01.z), w[3] = bswap32(in.w01.w);
    w[4] = bswap32(in.w23.x), w[5] = bswap32(in.w23.y), w[6] = bswap32(in.w23.z), w[7] = bswap32(in.w23.w);
    if constexpr (LW == 8) {
      w[8] = bswap32(in.w45.x), w[9] = bswap32(in.w45.y), w[10] = bswap32(in.w45.z), w[11] = bswap32(in.w45.w);
      w[12] = bswap32(in.w67.x), w[13] = bswap32(in.w67.y), w[14] = bswap32(in.w67.z), w[15] = bswap32(in.w67.w);
    }
    w[2 * LW] = bswap32(in.w8.x), w[2 * LW + 1] = bswap32(in.w8.y);
    const std::uint32_t n = min(in.nwin - wl0, static_cast<std::uint32_t>(LW));
    bool windowed = true;
    if (verified) {
      const SlotSinkT<WS> saved = sink;
      const std::uint32_t gap0 = (in.gaps >> 4) & 15u;  // window 0: high nibble of byte 0
      windowed = !decode_lane_continuous<LW>(w, n, gap0, smem_addr(tb.fast), smem_addr(tb.smask), sink);
      if (windowed) sink = saved;
    }
    if (windowed) {
#pragma unroll
      for (int i = 0; i < LW; ++i) {
        if (static_cast<std::uint32_t>(i) < n) {
          // byte j of the gap word: window 2j in the high nibble, 2j + 1 low
          const std::uint32_t gap = (in.gaps >> (8 * (i >> 1) + ((i & 1) ? 0 : 4))) & 15u;
          if (verified)  // a flagged entry: the exact walk straight away
            decode_window_exact(w[2 * i], w[2 * i + 1], w[2 * i + 2], w[2 * i + 3], gap, tb, len_off, sink);
          else
            decode_window(w[2 * i], w[2 * i + 1], w[2 * i + 2], w[2 * i + 3], gap, tb, len_off, sink);
        }
      }
    }
  }
  const std::uint32_t cnt = sink.finish(slot_base);

  // warp scan, segmented by reference block (2^(log2T-3) lanes each)
  std::uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const std::uint32_t excl = incl - cnt;
  constexpr std::uint32_t kLog2LW = LW == 8 ? 3 : 2;
  const std::uint32_t lpb_mask = (1u << (log2T - kLog2LW)) - 1;  // lanes per block - 1
  const std::uint32_t first_excl = __shfl_sync(0xffffffffu, excl, static_cast<std::uint32_t>(lane) & ~lpb_mask);
  const std::uint32_t start_rel = static_cast<std::uint32_t>(in.o0 - in.A) + excl - first_excl;
  const std::uint32_t lim_rel = static_cast<std::uint32_t>(in.o1 - in.A);
  const std::uint32_t cc = (active && start_rel < lim_rel) ? min(cnt, lim_rel - start_rel) : 0u;
  return LaneRun{cnt, start_rel, cc};
}

}  // namespace ecf8::dev
