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
#ifndef ECF8_WB_ALL_LOADS
#define ECF8_WB_ALL_LOADS 0  // 1: GPK write-back issues a pass of packed loads at once (A/B: spills, -4..-13 %)
#endif
#ifndef ECF8_WB_PASS
#define ECF8_WB_PASS 8
#endif
#ifndef ECF8_PF_WINDOWS_ONLY
#define ECF8_PF_WINDOWS_ONLY 0
#endif
#ifndef ECF8_COUNTED
#define ECF8_COUNTED 1  // verified direct tiles: runs end by the group offsets (0: by the completion masks)
#endif
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
  std::uint32_t ok_a, ok_b;  // tile_ok words of the tile's first / last window (loaded one tile ahead)
  std::uint32_t gnext;       // the lane's endgap word (gap layout) -- byte-step decoder only
  std::uint32_t ls;          // its two 4-window groups' output offsets in their block (lane_start) -- byte-step only
  std::uint32_t dir;         // the tile's tile_direct word -- byte-step decoder only
};
using WarpIn = WarpInT<kLaneWin>;

// A tile's inputs in two halves: the window words and gaps (issued early,
// they fly while the previous tile is written back), and the block offsets.
template <int LW, bool NEXT = false, bool GNEXT = true>
__device__ __forceinline__ void load_tile_words(const TensorDesc& d, std::uint64_t tile, std::uint32_t log2T,
                                                int lane, WarpInT<LW>& in) {
  constexpr bool kGnext = NEXT && GNEXT;
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
      if constexpr (kGnext)  // (no byte-step decoder -> no recorded ends)
        in.gnext = d.endgap ? __ldg(reinterpret_cast<const std::uint32_t*>(d.endgap + (w0g >> 1)) + lane) : 0u;
    } else {
      static_assert(LW == 4, "4 or 8 windows per lane");
      in.w8 = __ldg(reinterpret_cast<const uint2*>(src + 2));
      in.gaps = __ldg(reinterpret_cast<const std::uint16_t*>(d.gaps + (w0g >> 1)) + lane);
      if constexpr (kGnext)
        in.gnext = d.endgap ? __ldg(reinterpret_cast<const std::uint16_t*>(d.endgap + (w0g >> 1)) + lane) : 0u;
    }
  }
}

template <int LW, bool NEXT = false, bool DIR = true>
__device__ __forceinline__ void load_tile_meta(const TensorDesc& d, std::uint32_t log2T, int lane, WarpInT<LW>& in) {
  const std::uint32_t wl = static_cast<std::uint32_t>(lane) * LW;
  in.A = __ldg(d.outpos + in.b0);
  in.E = __ldg(d.outpos + in.b0 + in.nblk);
  // my block's bounds (lanes past the tile's windows read the last block's:
  // unused, their run is empty) -- no select on E, which would wait for it here
  const std::uint32_t bl = min(wl >> log2T, in.nblk - 1);
  in.o0 = __ldg(d.outpos + in.b0 + bl);
  in.o1 = __ldg(d.outpos + in.b0 + bl + 1);
  in.ok_a = in.ok_b = 0;
  if (d.tile_ok && in.nwin) {
    const std::uint64_t w0 = in.b0 << log2T;
    in.ok_a = __ldg(d.tile_ok + (w0 >> 13));
    in.ok_b = __ldg(d.tile_ok + ((w0 + in.nwin - 1) >> 13));
  }
  if constexpr (NEXT) {
    in.ls = in.dir = 0;
    if (d.lane_start && in.nwin) {
      const std::uint64_t w0 = in.b0 << log2T;
      if constexpr (DIR) in.dir = __ldg(d.tile_direct + (w0 >> 13));
      if (wl < in.nwin) {
        if constexpr (LW == 8) in.ls = __ldg(reinterpret_cast<const std::uint32_t*>(d.lane_start + (w0 >> 2)) + lane);
        else in.ls = __ldg(d.lane_start + (w0 >> 2) + lane);
      }
    }
  }
}

// GNEXT: load the lanes' endgap words with the tile (the 8-window direct
// tiles load them only when a tile is unverified: load_gnext); DIR: the
// tile's tile_direct word (not needed where every tile is direct).
template <int LW, bool NEXT = false, bool GNEXT = true, bool DIR = true>
__device__ __forceinline__ void load_warp_tile(const TensorDesc& d, std::uint64_t tile, std::uint32_t log2T,
                                               int lane, WarpInT<LW>& in) {
  load_tile_words<LW, NEXT, GNEXT>(d, tile, log2T, lane, in);
  load_tile_meta<LW, NEXT, DIR>(d, log2T, lane, in);
}

// The lane's endgap word of an 8-window tile, on demand.
__device__ __forceinline__ std::uint32_t load_gnext(const TensorDesc& d, const WarpInT<8>& in, int lane) {
  const std::uint32_t log2T = 31 - __clz(d.T);
  const std::uint64_t w0g = in.b0 << log2T;
  if (!d.endgap || static_cast<std::uint32_t>(lane) * 8 >= in.nwin) return 0u;
  return __ldg(reinterpret_cast<const std::uint32_t*>(d.endgap + (w0g >> 1)) + lane);
}

// A warp tile's input sections -> L2 (bulk prefetches, lanes 0-4): its
// windows, gap and end nibbles, group offsets and block offsets.  The packed
// bytes are fetched by the tile itself (cp.async during the decode).
__device__ __forceinline__ void prefetch_l2(const void* p, std::uint64_t bytes) {
  const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(p) & ~std::uintptr_t{15};
  const std::uint32_t n = static_cast<std::uint32_t>((reinterpret_cast<std::uintptr_t>(p) + bytes - a + 15) & ~std::uint64_t{15});
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
}
// Lanes 0-4 issue one section each (the descriptor reads and the address
// math run side by side instead of one after another).
// ntiles consecutive tiles at once: their sections are contiguous.
__device__ __forceinline__ void prefetch_tile_l2(const TensorDesc& d, std::uint64_t tile, std::uint32_t log2T,
                                                 int lane, std::uint32_t ntiles = 1) {
  const std::uint32_t m1 = 256u >> log2T, m = m1 * ntiles;
  const std::uint64_t b0 = d.blk_begin + (tile - d.tile_begin) * m1;
  const std::uint64_t nb = d.blk_end - b0 < m ? d.blk_end - b0 : m;
  const std::uint64_t w0 = b0 << log2T, nw = nb << log2T;
  // branch-free: lane i picks section i (0 windows, 1 gaps, 2 block offsets,
  // 3 end nibbles, 4 group offsets)
  const std::uint8_t* p = d.encoded + 8 * w0;
  std::uint64_t n = 8 * nw + 8;
#if ECF8_PF_WINDOWS_ONLY  // A/B: only the windows (the small sections load from HBM at the tile's start)
  if (lane == 0) prefetch_l2(p, n);
  return;
#endif
  p = lane == 1 ? d.gaps + (w0 >> 1) : p;
  p = lane == 2 ? reinterpret_cast<const std::uint8_t*>(d.outpos + b0) : p;
  p = lane == 3 ? (d.endgap ? d.endgap + (w0 >> 1) : nullptr) : p;
  p = lane == 4 ? (d.lane_start ? reinterpret_cast<const std::uint8_t*>(d.lane_start + (w0 >> 2)) : nullptr) : p;
  n = lane == 2 ? 8 * (nb + 1) : lane >= 1 ? nw >> 1 : n;
  if (p && n) prefetch_l2(p, n);
}

// The same prefetches from a per-segment table (ECF8_PF_TAB): lane i < 5
// takes its section's base pointer, byte shift per block and extra bytes
// (prefetch_sections) -- one shared load instead of five candidate pointers
// and a select chain.  Section i of blocks [b0, b0 + nb): base + (b0 << sh),
// (nb << sh) + add bytes.
struct PfSec {
  std::uint64_t base;  // 0: the section is absent
  std::uint32_t sh, add;
};
__device__ __forceinline__ PfSec pf_section(const TensorDesc& d, int i, std::uint32_t log2T) {
  const void* p = i == 0 ? static_cast<const void*>(d.encoded)
                  : i == 1 ? static_cast<const void*>(d.gaps)
                  : i == 2 ? static_cast<const void*>(d.outpos)
                  : i == 3 ? static_cast<const void*>(d.endgap)
                           : static_cast<const void*>(d.lane_start);
  // encoded: 8 T bytes per block (+ the 8-byte lookahead); gaps, end nibbles,
  // group offsets: T / 2 bytes per block; outpos: 8 bytes per block (+ 1 entry)
  const std::uint32_t sh = i == 0 ? log2T + 3 : i == 2 ? 3u : log2T - 1;
  return PfSec{reinterpret_cast<std::uint64_t>(p), sh, (i == 0 || i == 2) ? 8u : 0u};
}
__device__ __forceinline__ void prefetch_tile_l2_tab(const TensorDesc& d, const PfSec* tab, std::uint64_t tile,
                                                     std::uint32_t log2T, int lane) {
  const std::uint32_t m1 = 256u >> log2T;
  const std::uint64_t b0 = d.blk_begin + (tile - d.tile_begin) * m1;
  const std::uint64_t nb = d.blk_end - b0 < m1 ? d.blk_end - b0 : m1;
  const PfSec s = tab[lane];
  if (s.base) prefetch_l2(reinterpret_cast<const void*>(s.base + (b0 << s.sh)), (nb << s.sh) + s.add);
}

// Were the gaps of the windows of this warp tile verified (verify_gaps_kernel)?
// tile_ok bit v covers the boundaries after windows [256v, 256v + 256).
template <int LW>
__device__ __forceinline__ bool tile_verified(const TensorDesc&, const WarpInT<LW>& in, std::uint32_t log2T) {
  const std::uint64_t w0 = in.b0 << log2T;
  const std::uint32_t v0 = static_cast<std::uint32_t>(w0 >> 8), v1 = static_cast<std::uint32_t>((w0 + in.nwin - 1) >> 8);
  return ((in.ok_a >> (v0 & 31)) & (in.ok_b >> (v1 & 31)) & 1u) != 0;  // ok words are 0 when unverified
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
// FSM (the tensor's code has a byte-step decoder, staged at kFsmAt): a
// verified tile's lanes decode their LW windows in one pass, the others
// window by window, each up to its recorded end (decode_windows_fsm).
template <int LW, int WS = 4, bool OR_BASE = false, class TV, bool FSM = false>
__device__ __forceinline__ LaneRun warp_decode_scan(const WarpInT<LW>& in, std::uint32_t log2T,
                                                   std::uint32_t len_off, const TV& tb, std::uint32_t slot_base,
                                                   int lane, bool verified = false) {
  const std::uint32_t wl0 = static_cast<std::uint32_t>(lane) * LW;
  const bool active = wl0 < in.nwin;
  SlotSinkT<WS> sink{slot_base};
  PairSink<WS> psink{slot_base};  // byte-step path (the other sink then stays empty)
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
    if constexpr (FSM) {
      windowed = false;
      if (verified) {
        decode_windows_fsm<LW, WS>(w, (in.gaps >> 4) & 15u, (in.gnext >> (8 * ((LW - 1) >> 1))) & 15u, psink);
      } else {
#pragma unroll
        for (int i = 0; i < LW; ++i) {
          const int sh = 8 * (i >> 1) + ((i & 1) ? 0 : 4);  // window 2j: high nibble of byte j
          decode_windows_fsm<1, WS>(w + 2 * i, (in.gaps >> sh) & 15u, (in.gnext >> sh) & 15u, psink);
        }
      }
    } else if (!TV::kGlobal && verified) {
      const SlotSinkT<WS> saved = sink;
      const std::uint32_t gap0 = (in.gaps >> 4) & 15u;  // window 0: high nibble of byte 0
      // n == LW: tiles are whole blocks of T >= LW windows, so every active lane owns LW windows
      windowed = !decode_lane_continuous<LW, SlotSinkT<WS>, OR_BASE, TV, true>(w, n, gap0, tb.fast_addr(), tb, sink);
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
            decode_window<OR_BASE>(w[2 * i], w[2 * i + 1], w[2 * i + 2], w[2 * i + 3], gap, tb, len_off, sink);
        }
      }
    }
  }
  const std::uint32_t cnt = FSM ? psink.finish(slot_base) : sink.finish(slot_base);

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

// ---- compaction + write-back (shared by the decode kernel and the fused GEMM)

// Per-warp shared memory of the tile pipeline: the lanes' nibble slots
// (interleaved word by word: word j of lane L at slot[32 j + L]) and the
// staging tile the runs are compacted into.  After compaction the slots hold
// the tile's sign/mantissa bytes.
template <int SLOT_ROWS, int STAGE_WORDS>
struct WarpPipeSmem {
  static constexpr int kSlotRows = SLOT_ROWS;
  std::uint32_t slot[SLOT_ROWS * 32];
  alignas(16) std::uint32_t stage[STAGE_WORDS];
};

// Write the tile's output elements [A, E) from the staging tile (exponent
// nibbles at nibble off + i for element A + i) and the packed bytes copied
// to the slots (from the 16-byte aligned pk_a): full 16-element chunks as
// lane-interleaved 16-byte stores, the ragged first / last chunk byte-wise.
// GPK: the packed bytes are read from global memory (gpk = d.packed; L2
// after the tile's bulk prefetch) instead of the slots -- the fused GEMM,
// whose shared memory goes to the A ring.
template <int UNROLL, bool GPK = false, class WSm, class Out>
__device__ __forceinline__ void write_back(std::uint64_t S0, std::uint32_t off, std::uint32_t data_end,
                                           std::uint64_t pk_a, const WSm& ws, int lane, Out& out,
                                           const std::uint8_t* gpk = nullptr) {
  const std::uint32_t nch = (data_end + 15) >> 4;
  const std::uint32_t full_lo = (off + 15) >> 4, full_hi = data_end >> 4;
  const std::uint32_t nfull = full_hi > full_lo ? full_hi - full_lo : 0u;
  const std::uint64_t pk_lo = (S0 >> 1) + 8 * full_lo;
  out.wait();
  const uint2* sl = reinterpret_cast<const uint2*>(ws.stage) + full_lo + lane;
  const uint2* pl = GPK ? reinterpret_cast<const uint2*>(gpk + pk_lo) + lane
                        : reinterpret_cast<const uint2*>(reinterpret_cast<const std::uint8_t*>(ws.slot) + (pk_lo - pk_a)) + lane;
  std::uint32_t k = lane;
#if ECF8_WB_ALL_LOADS
  if constexpr (GPK) {
    // the packed bytes come from L2: every load of a pass is issued before
    // its first merge, so a pass waits out one L2 round trip
    constexpr int kPass = ECF8_WB_PASS;  // chunks per lane per pass
    for (std::uint32_t base = 0; base < nfull; base += 32 * kPass, sl += 32 * kPass, pl += 32 * kPass) {
      uint2 q[kPass];
#pragma unroll
      for (int u = 0; u < kPass; ++u)
        if (base + lane + 32u * u < nfull) q[u] = __ldg(pl + 32 * u);
#pragma unroll
      for (int u = 0; u < kPass; ++u) {
        const std::uint32_t kk = base + lane + 32u * u;
        if (kk < nfull) {
          const uint2 sv = sl[32 * u];
          uint4 r;
          merge8(sv.x, q[u].x, r.x, r.y);
          merge8(sv.y, q[u].y, r.z, r.w);
          out.chunk(full_lo + kk, r);
        }
      }
    }
    k = nfull + lane;  // the loops below find nothing left
  }
#endif
#if ECF8_WB_PRED
  if constexpr (GPK) {
    // groups of UNROLL chunks per lane with per-chunk predicates: a tile's
    // ~12 chunks per lane take ceil(12 / UNROLL) L2 round trips, with no
    // one-chunk-at-a-time remainder loop
    for (; k < nfull; k += 32 * UNROLL, sl += 32 * UNROLL, pl += 32 * UNROLL) {
      uint2 sv[UNROLL], q[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (k + 32u * u < nfull) sv[u] = sl[32 * u], q[u] = __ldg(pl + 32 * u);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (k + 32u * u < nfull) {
          uint4 r;
          merge8(sv[u].x, q[u].x, r.x, r.y);
          merge8(sv[u].y, q[u].y, r.z, r.w);
          out.chunk(full_lo + k + 32 * u, r);
        }
      }
    }
  }
#endif
#if ECF8_WB_PIPE
  if constexpr (GPK) {
    // the packed bytes come from L2: the next group's loads are issued before
    // this group's merges (two groups in flight per lane)
    uint2 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (k + 32u * u < nfull) q[u] = __ldg(pl + 32 * u);
    for (; k < nfull; k += 32 * UNROLL, sl += 32 * UNROLL, pl += 32 * UNROLL) {
      uint2 qn[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (k + 32u * (UNROLL + u) < nfull) qn[u] = __ldg(pl + 32 * (UNROLL + u));
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (k + 32u * u < nfull) {
          const uint2 sv = sl[32 * u];
          uint4 r;
          merge8(sv.x, q[u].x, r.x, r.y);
          merge8(sv.y, q[u].y, r.z, r.w);
          out.chunk(full_lo + k + 32 * u, r);
        }
        q[u] = qn[u];
      }
    }
  }
#endif
  for (; k + 32 * (UNROLL - 1) < nfull; k += 32 * UNROLL, sl += 32 * UNROLL, pl += 32 * UNROLL) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint2 s = sl[32 * u], q = GPK ? __ldg(pl + 32 * u) : pl[32 * u];
      uint4 r;
      merge8(s.x, q.x, r.x, r.y);
      merge8(s.y, q.y, r.z, r.w);
      out.chunk(full_lo + k + 32 * u, r);
    }
  }
#if ECF8_WB_STEPS
  // the rest in groups of UNROLL / 2, / 4: a lane's loads of a group are in
  // flight together (one L2 round trip per group, not per chunk)
  if constexpr (UNROLL >= 8) {
    constexpr int U2 = UNROLL / 2;
    for (; k + 32 * (U2 - 1) < nfull; k += 32 * U2, sl += 32 * U2, pl += 32 * U2) {
#pragma unroll
      for (int u = 0; u < U2; ++u) {
        const uint2 s = sl[32 * u], q = GPK ? __ldg(pl + 32 * u) : pl[32 * u];
        uint4 r;
        merge8(s.x, q.x, r.x, r.y);
        merge8(s.y, q.y, r.z, r.w);
        out.chunk(full_lo + k + 32 * u, r);
      }
    }
  }
  if constexpr (UNROLL >= 4) {
    constexpr int U4 = UNROLL >= 8 ? UNROLL / 4 : 2;
    for (; k + 32 * (U4 - 1) < nfull; k += 32 * U4, sl += 32 * U4, pl += 32 * U4) {
#pragma unroll
      for (int u = 0; u < U4; ++u) {
        const uint2 s = sl[32 * u], q = GPK ? __ldg(pl + 32 * u) : pl[32 * u];
        uint4 r;
        merge8(s.x, q.x, r.x, r.y);
        merge8(s.y, q.y, r.z, r.w);
        out.chunk(full_lo + k + 32 * u, r);
      }
    }
  }
#endif
  for (; k < nfull; k += 32, sl += 32, pl += 32) {
    const uint2 s = *sl, q = GPK ? __ldg(pl) : *pl;
    uint4 r;
    merge8(s.x, q.x, r.x, r.y);
    merge8(s.y, q.y, r.z, r.w);
    out.chunk(full_lo + k, r);
  }
  // partial edge chunks, one byte per lane: lanes 0-15 the first chunk,
  // lanes 16-31 the last one
  const std::uint32_t i = lane < 16 ? static_cast<std::uint32_t>(lane) : 16 * (nch - 1) + (lane - 16);
  const bool edge = lane < 16 ? (full_lo > 0 && i >= off && i < data_end)
                              : (full_hi < nch && !(nch == 1 && full_lo > 0) && i < data_end);
  if (edge) {
    const std::uint32_t x = (ws.stage[i >> 3] >> (4 * (i & 7))) & 15u;
    const std::uint8_t qb = GPK ? __ldg(gpk + (S0 >> 1) + (i >> 1))
                                : (reinterpret_cast<const std::uint8_t*>(ws.slot) + ((S0 >> 1) - pk_a))[i >> 1];
    out.byte(i, merge1(x, qb, i & 1));
  }
  out.done();
}

// The tile's packed sign/mantissa bytes [S0 / 2, (S0 + data_end + 1) / 2) into
// the slots by 16-byte async copies from the 16-byte aligned address pk_a
// (the slots must hold the tile's packed bytes + 16: (8192 + 30) / 2 + 16 <=
// 33 x 128 bytes).  Returns pk_a.
template <class WSm>
__device__ __forceinline__ std::uint64_t fetch_packed(const TensorDesc& d, std::uint64_t S0, std::uint32_t data_end,
                                                      WSm& ws, int lane) {
  const std::uint64_t pk_a = (S0 >> 1) & ~std::uint64_t{15};
  const std::uint32_t n16 = static_cast<std::uint32_t>((((S0 + data_end + 1) >> 1) - pk_a + 15) >> 4);
  const std::uint32_t dst = smem_addr(ws.slot);
  for (std::uint32_t i = lane; i < n16; i += 32)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * i), "l"(d.packed + pk_a + 16 * i)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
  return pk_a;
}

// Compact the lanes' runs (slot nibbles, LaneRun from warp_decode_scan) into
// the staging tile, then write the tile's output elements [A, E) -- FP8
// bytes = exponent nibble + sign/mantissa nibble (fp8.hpp:42-57) -- through
// `out`:
//   out.wait()               once, before the first store
//   out.chunk(c, r)          16 bytes for elements [S0 + 16c, +16), S0 = A & ~15
//   out.byte(i, b)           one byte for element S0 + i
//   out.done()               after the last store
// Full 16-element chunks go out as 16-byte stores, lane-interleaved
// (coalesced); the ragged first and last chunks byte by byte.  The
// sign/mantissa bytes of the full chunks come into the (then free) slots by
// 16-byte async copies issued right after compaction: one round trip per tile
// (the slots must hold the tile's packed bytes + 16: (8192 + 30) / 2 + 16 <=
// 33 x 128 bytes).
template <int UNROLL, class WSm, class Out>
__device__ __forceinline__ void compact_write(const TensorDesc& d, std::uint64_t A, std::uint64_t E,
                                              const LaneRun& run, WSm& ws, int lane, Out& out) {
  const std::uint32_t* const my_slot = ws.slot + lane;
  const std::uint32_t cc = run.len;
  const std::uint32_t off = static_cast<std::uint32_t>(A & 15);  // staging nibble of element A
  const std::uint32_t d0 = run.start + off, dend = d0 + cc;
  const std::uint32_t data_end = off + static_cast<std::uint32_t>(E - A);
  const std::uint64_t S0 = A - off;
  __syncwarp();  // previous tile's write-back is done with the staging and the slots' packed bytes

  // ---- move my nibbles to their final place; publish partial words
  std::uint32_t headv = 0, tailv = 0;
  const std::uint32_t fw = d0 >> 3, lw = (dend - 1) >> 3;
  const std::uint32_t f4 = (d0 & 7) * 4, lastn = ((dend - 1) & 7) + 1;
  if (cc) {
    std::uint32_t prev = my_slot[0];
    const std::uint32_t v0 = prev << f4;
    if (fw == lw) {
      const std::uint32_t v = v0 & low_nibbles(lastn);
      if (f4 == 0 && lastn == 8) ws.stage[fw] = v;
      else headv = v;
    } else {
      if (f4 == 0) ws.stage[fw] = v0;
      else headv = v0;
      std::uint32_t j = 1;
#pragma unroll 4
      for (std::uint32_t k = fw + 1; k < lw; ++k, ++j) {
        const std::uint32_t c = my_slot[32 * j];
        ws.stage[k] = __funnelshift_l(prev, c, f4);
        prev = c;
      }
      const std::uint32_t v = __funnelshift_l(prev, my_slot[32 * j], f4) & low_nibbles(lastn);
      if (lastn == 8) ws.stage[lw] = v;
      else tailv = v;
    }
  }
  __syncwarp();

  // ---- the slots are free: sign/mantissa bytes of the full chunks into them
  // (16-byte pieces from the 16-byte aligned address at or below the first
  // full chunk's bytes: <= 8 nfull + 16 bytes)
  // all of the tile's packed bytes [S0 / 2, (S0 + data_end + 1) / 2), edge chunks included
  const std::uint64_t pk_a = fetch_packed(d, S0, data_end, ws, lane);

  // ---- owners assemble words shared between lanes: the start owner of my
  // first word / my tail word OR in the partial head words of the following
  // lanes until the word is covered (lane bounds and heads by shuffle; runs
  // are contiguous, so this takes one or two steps)
  const bool start_owner = cc && (f4 == 0 || d0 == off) && !(f4 == 0 && (fw < lw || lastn == 8));
  const bool tail_owner = cc && fw != lw && lastn != 8;
  std::uint32_t vs = headv, vt = tailv, cov_s = dend, cov_t = dend;
  const std::uint32_t wend_s = min(8 * fw + 8, data_end), wend_t = min(8 * lw + 8, data_end);
  for (std::uint32_t o = 1; o < 32; ++o) {
    const bool need_s = start_owner && cov_s < wend_s, need_t = tail_owner && cov_t < wend_t;
    if (!__any_sync(0xffffffffu, need_s || need_t)) break;
    const std::uint32_t rj = __shfl_down_sync(0xffffffffu, d0, o);
    const std::uint32_t ej = __shfl_down_sync(0xffffffffu, cc ? dend : d0, o);
    const std::uint32_t hj = __shfl_down_sync(0xffffffffu, headv, o);
    if (static_cast<std::uint32_t>(lane) + o < 32 && ej > rj) {
      if (need_s) vs |= hj, cov_s = ej;
      if (need_t) vt |= hj, cov_t = ej;
    }
  }
  if (start_owner) ws.stage[fw] = vs;
  if (tail_owner) ws.stage[lw] = vt;
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();

  // ---- write-back
  write_back<UNROLL>(S0, off, data_end, pk_a, ws, lane, out);
}

// ---- direct tile (byte-step decoder, tile_direct set): every lane's output
// offset is known before decoding (lane_start, from the upload check), so
// the byte steps append straight into the zeroed staging tile at the lane's
// final place -- no slot, no scan, no compaction.  Each lane runs two
// independent chains (its 4-window groups, each from its own known offset),
// interleaved: two table-probe chains in flight per lane.  Full words are
// plain stores (each belongs to one chain); a chain's partial last word is
// OR-ed in after every chain's first word (which may share it) is stored.
// The tile's packed bytes stream into the slots while the lanes decode.
// mk_out() builds the output sink (out.wait / chunk / byte / done, see
// compact_write) after the decode: its state is not live across the byte steps.
template <int UNROLL, int LW, bool GPK = false, class WSm, class MkOut, class FT = FsmPinned>
__device__ __forceinline__ void direct_tile(const TensorDesc& d, const WarpInT<LW>& in, WSm& ws, int lane,
                                            const MkOut& mk_out, bool verified, const FT& ft = FT{}) {
  const std::uint32_t off = static_cast<std::uint32_t>(in.A & 15);  // staging nibble of element A
  const std::uint32_t data_end = off + static_cast<std::uint32_t>(in.E - in.A);
  const std::uint64_t S0 = in.A - off;
  __syncwarp();  // previous tile's write-back is done with the staging and the slots' packed bytes
  std::uint32_t ta_addr = 0, ta = 0, tb_addr = 0, tb = 0;
  const std::uint32_t base = static_cast<std::uint32_t>(in.o0 - in.A) + off;
#if ECF8_COUNTED
  // run ends from the group offsets: group A ends where group B starts, group
  // B where the next lane's group A starts (same reference block), else at
  // the block's end; every run clamped to its block's outpos range
  // (codec.cpp:239-246: only the tensor's last block can decode past it)
  std::uint32_t end_a = 0, end_b = 0;
  if constexpr (LW == 8) {
    const std::uint32_t blk_end = static_cast<std::uint32_t>(in.o1 - in.A) + off;
    const std::uint32_t da = base + (in.ls & 0xFFFFu), db = base + (in.ls >> 16);
    const std::uint32_t next_da = __shfl_down_sync(0xffffffffu, da, 1);
    const std::uint32_t lpb_mask = (d.T >> 3) - 1;  // lanes per reference block - 1 (T >= 8)
    const std::uint32_t nl = static_cast<std::uint32_t>(lane) + 1;
    const bool next_same = nl < 32 && (nl & lpb_mask) != 0 && nl * 8 < in.nwin;
    end_a = min(max(db, da), blk_end);
    end_b = min(max(next_same ? next_da : blk_end, db), blk_end);
    end_a = max(end_a, min(da, blk_end));
    end_b = max(end_b, min(db, blk_end));
  }
#endif
  {
    const std::uint32_t st = smem_addr(ws.stage);
#if ECF8_COUNTED
    if constexpr (LW == 8) {
      // direct tiles cover [A, E) with the lanes' runs, back to back (every
      // block decodes to exactly its range, the upload check): a word is
      // either plain-stored by a run that fills it, or it holds a run's end
      // and gets OR-ed -- only those end words need zeroes
      if (static_cast<std::uint32_t>(lane) * LW < in.nwin) {
        sts32(st + 4 * (end_a >> 3), 0u);
        sts32(st + 4 * (end_b >> 3), 0u);
      }
    } else
#endif
    {
      constexpr std::uint32_t n16 = sizeof(ws.stage) / 16;
      for (std::uint32_t i = lane; i < n16; i += 32)
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(st + 16 * i), "r"(0u) : "memory");
    }
  }
  const std::uint64_t pk_a = GPK ? 0 : fetch_packed(d, S0, data_end, ws, lane);
  __syncwarp();  // the zeroes are in place
  if (static_cast<std::uint32_t>(lane) * LW < in.nwin) {
    std::uint32_t w[2 * LW + 2];
    w[0] = bswap32(in.w01.x), w[1] = bswap32(in.w01.y), w[2] = bswap32(in.w01.z), w[3] = bswap32(in.w01.w);
    w[4] = bswap32(in.w23.x), w[5] = bswap32(in.w23.y), w[6] = bswap32(in.w23.z), w[7] = bswap32(in.w23.w);
    if constexpr (LW == 8) {
      w[8] = bswap32(in.w45.x), w[9] = bswap32(in.w45.y), w[10] = bswap32(in.w45.z), w[11] = bswap32(in.w45.w);
      w[12] = bswap32(in.w67.x), w[13] = bswap32(in.w67.y), w[14] = bswap32(in.w67.z), w[15] = bswap32(in.w67.w);
    }
    w[2 * LW] = bswap32(in.w8.x), w[2 * LW + 1] = bswap32(in.w8.y);
    if constexpr (LW == 8) {
      // two chains: windows 0-3 and 4-7, each from its group's known offset
      const std::uint32_t da = base + (in.ls & 0xFFFFu), db = base + (in.ls >> 16);
      PairSink<4> sa{smem_addr(ws.stage) + 4 * (da >> 3)}, sb{smem_addr(ws.stage) + 4 * (db >> 3)};
      sa.q4 = 4 * (da & 7);
      sb.q4 = 4 * (db & 7);
      if (verified) {
#if ECF8_COUNTED
        const std::uint32_t st = smem_addr(ws.stage);
        std::uint32_t xa, xb;
        decode_two_fsm_counted<4, 4, FT>(w, (in.gaps >> 4) & 15u, end_a, sa, xa, w + 8, (in.gaps >> 20) & 15u, end_b,
                                         sb, xb, st, ft);
        // the end words (OR-ed in below, after every run's plain stores)
        ta_addr = st + 4 * (end_a >> 3);
        ta = xa;
        tb_addr = st + 4 * (end_b >> 3);
        tb = xb;
        goto stored;
#else
        const std::uint32_t gn = load_gnext(d, in, lane);
        decode_two_fsm<4, 4, FT>(w, (in.gaps >> 4) & 15u, (gn >> 8) & 15u, sa, w + 8, (in.gaps >> 20) & 15u,
                                 (gn >> 24) & 15u, sb, ft);
#endif
      } else {
        const std::uint32_t gn = load_gnext(d, in, lane);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int sh = 8 * (i >> 1) + ((i & 1) ? 0 : 4);  // window 2j: high nibble of byte j
          decode_two_fsm<1, 4, FT>(w + 2 * i, (in.gaps >> sh) & 15u, (gn >> sh) & 15u, sa, w + 8 + 2 * i,
                                   (in.gaps >> (16 + sh)) & 15u, (gn >> (16 + sh)) & 15u, sb, ft);
        }
      }
      tb_addr = sb.addr;
      tb = (sb.q4 & 31u) ? sb.lo : 0u;
      ta_addr = sa.addr;
      ta = (sa.q4 & 31u) ? sa.lo : 0u;
#if ECF8_COUNTED
    stored:;
#endif
    } else {
      // one chain: the lane's 4-window group
      const std::uint32_t da = base + in.ls;
      PairSink<4> sa{smem_addr(ws.stage) + 4 * (da >> 3)};
      sa.q4 = 4 * (da & 7);
      if (verified) {
        decode_windows_fsm<4, 4, FT>(w, (in.gaps >> 4) & 15u, (in.gnext >> 8) & 15u, sa, ft);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int sh = 8 * (i >> 1) + ((i & 1) ? 0 : 4);
          decode_windows_fsm<1, 4, FT>(w + 2 * i, (in.gaps >> sh) & 15u, (in.gnext >> sh) & 15u, sa, ft);
        }
      }
      ta_addr = sa.addr;
      ta = (sa.q4 & 31u) ? sa.lo : 0u;
    }
  }
  __syncwarp();  // every full word and every lane's first word is stored
  if (ta) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(ta_addr), "r"(ta) : "memory");
  if (tb) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(tb_addr), "r"(tb) : "memory");
  if constexpr (!GPK) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
  auto out = mk_out();
  write_back<UNROLL, GPK>(S0, off, data_end, pk_a, ws, lane, out, d.packed);
}

// ---- direct tile, 64-bit byte steps (variant 6: codes with a 1-bit word;
// every tile of the tensor passed the upload check, so every lane's run is
// placed directly and ends by its group offsets).  Windows hold up to 64
// symbols: the staging tile holds 16384 nibbles.
template <int UNROLL, class WSm, class MkOut>
__device__ __forceinline__ void direct_tile64(const TensorDesc& d, const WarpInT<8>& in, WSm& ws, int lane,
                                              const MkOut& mk_out, const Fsm64At& ft) {
  const std::uint32_t off = static_cast<std::uint32_t>(in.A & 15);
  const std::uint32_t data_end = off + static_cast<std::uint32_t>(in.E - in.A);
  const std::uint64_t S0 = in.A - off;
  __syncwarp();  // previous tile's write-back is done with the staging tile
  const std::uint32_t st = smem_addr(ws.stage);
  const std::uint32_t base = static_cast<std::uint32_t>(in.o0 - in.A) + off;
  const std::uint32_t blk_end = static_cast<std::uint32_t>(in.o1 - in.A) + off;
  const std::uint32_t da = base + (in.ls & 0xFFFFu), db = base + (in.ls >> 16);
  const std::uint32_t next_da = __shfl_down_sync(0xffffffffu, da, 1);
  const std::uint32_t nl = static_cast<std::uint32_t>(lane) + 1;
  const bool next_same = nl < 32 && (nl & ((d.T >> 3) - 1)) != 0 && nl * 8 < in.nwin;
  const std::uint32_t end_a = max(min(max(db, da), blk_end), min(da, blk_end));
  const std::uint32_t end_b = max(min(max(next_same ? next_da : blk_end, db), blk_end), min(db, blk_end));
  const bool active = static_cast<std::uint32_t>(lane) * 8 < in.nwin;
  if (active) {  // only the runs' end words need zeroes (see direct_tile)
    sts32(st + 4 * (end_a >> 3), 0u);
    sts32(st + 4 * (end_b >> 3), 0u);
  }
  __syncwarp();
  std::uint32_t ta = 0, tb = 0;
  if (active) {
    std::uint32_t w[18];
    w[0] = bswap32(in.w01.x), w[1] = bswap32(in.w01.y), w[2] = bswap32(in.w01.z), w[3] = bswap32(in.w01.w);
    w[4] = bswap32(in.w23.x), w[5] = bswap32(in.w23.y), w[6] = bswap32(in.w23.z), w[7] = bswap32(in.w23.w);
    w[8] = bswap32(in.w45.x), w[9] = bswap32(in.w45.y), w[10] = bswap32(in.w45.z), w[11] = bswap32(in.w45.w);
    w[12] = bswap32(in.w67.x), w[13] = bswap32(in.w67.y), w[14] = bswap32(in.w67.z), w[15] = bswap32(in.w67.w);
    w[16] = bswap32(in.w8.x), w[17] = bswap32(in.w8.y);
    PairSink<4> sa{st + 4 * (da >> 3)}, sb{st + 4 * (db >> 3)};
    sa.q4 = 4 * (da & 7);
    sb.q4 = 4 * (db & 7);
    decode_two_fsm64_counted<4, 4>(w, (in.gaps >> 4) & 15u, end_a, sa, ta, w + 8, (in.gaps >> 20) & 15u, end_b, sb, tb,
                                   st, ft);
  }
  __syncwarp();  // every run's plain stores are in place
  if (ta) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(st + 4 * (end_a >> 3)), "r"(ta) : "memory");
  if (tb) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(st + 4 * (end_b >> 3)), "r"(tb) : "memory");
  __syncwarp();
  auto out = mk_out();
  write_back<UNROLL, true>(S0, off, data_end, 0, ws, lane, out, d.packed);
}

}  // namespace ecf8::dev
