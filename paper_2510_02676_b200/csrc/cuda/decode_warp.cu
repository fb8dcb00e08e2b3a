// decode_warp.cu -- warp-autonomous ECF8 decode kernel (sm_100a).
//
// Variant for the common case T in [8, 256] and shortest code length >= 2
// (every FP8 weight tensor we have seen): one warp owns a tile of 256
// consecutive 64-bit windows = 256/T whole reference blocks, eight windows
// per lane.  A window then holds at most 32 symbols, so a lane's slot is 32
// words and the tile's output at most 8192 nibbles.  Everything after the
// table staging is warp-synchronous: no CTA or group barriers, no cross-warp
// scan -- the reference block's offsets come straight from outpos[]
// (codec.cpp:212-253 restated per warp).  Phases per tile:
//
//   decode   each lane walks its 8 windows (decode_common.cuh fast walk,
//            exact walk for flagged windows) into its nibble slot;
//   scan     5-step warp shuffle scan of the lane counts, segmented by
//            reference block, clamped to outpos limits (codec.cpp:239-246);
//   compact  funnel-shift copy of each lane's nibbles to their final place
//            in the warp's staging tile; shared words assembled by owners;
//   write    16 output bytes per lane-step (SWAR merge with the
//            sign/mantissa nibbles, prefetched into L2 by one bulk TMA
//            prefetch), tile edges byte-wise.
//
// The next tile's window words, gaps and outpos bounds are loaded into
// registers one tile ahead.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "decode.cuh"
#include "decode_common.cuh"
#include "decode_warp.cuh"

namespace ecf8::dev {

namespace {

struct WarpSmem {
  static constexpr int kSlotW = kSlotWords;
  static constexpr int kStride = kSlotW + 1;
  static constexpr int kStageWords = 32 * kSlotW + 8;
  std::uint32_t slot[32 * kStride];
  alignas(16) std::uint32_t stage[kStageWords];
  std::uint32_t rs[32];
  std::uint32_t re[32];
  std::uint32_t head[32];
};

__shared__ Tables g_tb;
__shared__ unsigned long long g_next_tile;  // CTA-local work queue of the current segment

template <bool CONT>
__device__ __forceinline__ void warp_tile(const TensorDesc& d, const WarpIn& in, std::uint32_t log2T,
                                          std::uint32_t len_off, WarpSmem& ws, int lane) {
  std::uint32_t* const my_slot = ws.slot + lane * WarpSmem::kStride;
  const LaneRun run = warp_decode_scan<kLaneWin, CONT>(in, log2T, len_off, g_tb, my_slot, lane);
  const std::uint32_t cc = run.len;
  const std::uint32_t off = static_cast<std::uint32_t>(in.A & 15);  // staging nibble of element A
  const std::uint32_t d0 = run.start + off, dend = d0 + cc;
  const std::uint32_t data_end = off + static_cast<std::uint32_t>(in.E - in.A);
  __syncwarp();  // previous tile's write-back is done with the staging
  ws.rs[lane] = d0;
  ws.re[lane] = dend;

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
        const std::uint32_t c = my_slot[j];
        ws.stage[k] = __funnelshift_l(prev, c, f4);
        prev = c;
      }
      const std::uint32_t v = __funnelshift_l(prev, my_slot[j], f4) & low_nibbles(lastn);
      if (lastn == 8) ws.stage[lw] = v;
      else tailv = v;
    }
  }
  ws.head[lane] = headv;
  __syncwarp();

  // ---- owners assemble words shared between lanes
  if (cc) {
    const bool start_owner = (f4 == 0 || d0 == off) && !(f4 == 0 && (fw < lw || lastn == 8));
    const bool tail_owner = fw != lw && lastn != 8;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 0 ? !start_owner : !tail_owner) continue;
      const std::uint32_t k = pass == 0 ? fw : lw;
      std::uint32_t v = pass == 0 ? headv : tailv;
      const std::uint32_t wend = min(8 * k + 8, data_end);
      std::uint32_t covered = dend;
      for (int j = lane + 1; covered < wend && j < 32; ++j) {
        const std::uint32_t rj = ws.rs[j], ej = ws.re[j];
        if (ej > rj) {
          v |= ws.head[j];
          covered = ej;
        }
      }
      ws.stage[k] = v;
    }
  }
  __syncwarp();

  // ---- write-back
  const std::uint64_t S0 = in.A - off;
  std::uint8_t* const out = d.out + (S0 - d.out_offset);
  const std::uint8_t* const pk = d.packed + (S0 >> 1);
  const std::uint32_t nch = (data_end + 15) >> 4;
  const std::uint32_t full_lo = (off + 15) >> 4, full_hi = data_end >> 4;
  const uint2* sp = reinterpret_cast<const uint2*>(ws.stage);
  const uint2* pp = reinterpret_cast<const uint2*>(pk);
  uint4* op = reinterpret_cast<uint4*>(out);
  const std::uint32_t nfull = full_hi > full_lo ? full_hi - full_lo : 0u;
  const uint2* sl = sp + full_lo + lane;
  const uint2* pl = pp + full_lo + lane;
  uint4* ol = op + full_lo + lane;
  std::uint32_t k = lane;
  for (; k + 96 < nfull; k += 128, sl += 128, pl += 128, ol += 128) {
    uint2 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) q[u] = __ldg(pl + 32 * u);  // four L2 round trips overlap
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint2 s = sl[32 * u];
      uint4 r;
      merge8(s.x, q[u].x, r.x, r.y);
      merge8(s.y, q[u].y, r.z, r.w);
      ol[32 * u] = r;
    }
  }
  for (; k < nfull; k += 32, sl += 32, pl += 32, ol += 32) {
    const uint2 q = __ldg(pl);
    const uint2 s = *sl;
    uint4 r;
    merge8(s.x, q.x, r.x, r.y);
    merge8(s.y, q.y, r.z, r.w);
    *ol = r;
  }
  // partial edge chunks, one byte per lane: lanes 0-15 the first chunk,
  // lanes 16-31 the last one
  const std::uint32_t i = lane < 16 ? static_cast<std::uint32_t>(lane) : 16 * (nch - 1) + (lane - 16);
  const bool edge = lane < 16 ? (full_lo > 0 && i >= off && i < data_end)
                              : (full_hi < nch && !(nch == 1 && full_lo > 0) && i < data_end);
  if (edge) {
    const std::uint32_t x = (ws.stage[i >> 3] >> (4 * (i & 7))) & 15u;
    out[i] = merge1(x, pk[i >> 1], i & 1);
  }
}

template <int NW, bool CONT>
__global__ void __launch_bounds__(NW * 32, 1) decode_warp_kernel(const LaunchArgs args) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpSmem& ws = reinterpret_cast<WarpSmem*>(smem_raw)[warp];
  const std::uint64_t total_tiles = args.total_tiles;
  const std::uint64_t t_lo = total_tiles * blockIdx.x / gridDim.x;
  const std::uint64_t t_hi = total_tiles * (blockIdx.x + 1) / gridDim.x;

  for (std::uint64_t seg = t_lo; seg < t_hi;) {
    TensorDesc d;
    std::uint64_t seg_end;
    if (args.descs) {
      const int di = find_desc(args.descs, args.n_desc, seg);
      d = args.descs[di];
      seg_end = (di + 1 < args.n_desc) ? args.descs[di + 1].tile_begin : total_tiles;
    } else {
      d = args.inline_desc;
      seg_end = total_tiles;
    }
    if (seg_end > t_hi) seg_end = t_hi;
    const std::uint32_t log2T = 31 - __clz(d.T);
    __syncthreads();  // every warp is done with the previous tables
    stage_tables(d, g_tb, threadIdx.x, NW * 32);
    const std::uint32_t len_off = (d.n_luts - 1) << 8;
    if (threadIdx.x == 0) g_next_tile = seg + NW;
    __syncthreads();

    // Tiles are handed out dynamically inside the CTA (warp w starts with
    // tile seg + w, then takes the next unclaimed one), so the warps of a
    // segment finish within one tile of each other whatever the per-tile
    // cost.  The next tile is claimed and its inputs loaded one tile ahead.
    WarpIn nxt;
    std::uint64_t tile = seg + warp;
    if (tile < seg_end) load_warp_tile(d, tile, log2T, lane, nxt);
    while (tile < seg_end) {
      const WarpIn cur = nxt;
      if (lane == 0) {  // sign/mantissa bytes of this tile -> L2 (one bulk TMA prefetch)
        const std::uint64_t p0 = (cur.A >> 1) & ~std::uint64_t{15};
        const std::uint32_t bytes = static_cast<std::uint32_t>((((cur.E + 1) >> 1) - p0 + 15) & ~std::uint64_t{15});
        if (bytes)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(d.packed + p0), "r"(bytes) : "memory");
      }
      unsigned long long claim = 0;
      if (lane == 0) claim = atomicAdd(&g_next_tile, 1ull);
      const std::uint64_t next = __shfl_sync(0xffffffffu, claim, 0);
      if (next < seg_end) load_warp_tile(d, next, log2T, lane, nxt);
      warp_tile<CONT>(d, cur, log2T, len_off, ws, lane);
      tile = next;
    }
    seg = seg_end;
  }
}

template <int NW, bool CONT>
cudaError_t launch_nw(const LaunchArgs& args, cudaStream_t s) {
  static int grid_cap = 0;
  const int smem = static_cast<int>(sizeof(WarpSmem)) * NW;
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(decode_warp_kernel<NW, CONT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_warp_kernel<NW, CONT>, NW * 32, smem);
    if (e != cudaSuccess) return e;
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const std::uint64_t want = (args.total_tiles + NW - 1) / NW;
  const std::uint64_t grid = want < static_cast<std::uint64_t>(grid_cap) ? want : grid_cap;
  if (grid == 0) return cudaSuccess;
  decode_warp_kernel<NW, CONT><<<static_cast<unsigned>(grid), NW * 32, smem, s>>>(args);
  return cudaGetLastError();
}

}  // namespace

// Warps per CTA: 20 (default; 95 registers, no spills, 20 x 8.7 KB of warp
// state + 28.6 KB of tables) or 16 (ECF8_WARPS=16, <= 128 registers).
// Measured (8 x 14336x4096, T 256): 20 warps 2995 GB/s, 16 warps 2821 GB/s.
cudaError_t launch_decode_warp(const LaunchArgs& args, cudaStream_t s) {
  static const int nw = [] {
    const char* e = std::getenv("ECF8_WARPS");
    return e ? std::atoi(e) : 20;
  }();
  return nw == 16 ? launch_nw<16, false>(args, s) : launch_nw<20, false>(args, s);
}

// Variant 5: the same kernel walking each lane's windows continuously, for
// tensors whose gaps ecf8_tensor_upload verified (decode_lane_continuous).
cudaError_t launch_decode_warp_cont(const LaunchArgs& args, cudaStream_t s) {
  static const int nw = [] {
    const char* e = std::getenv("ECF8_WARPS");
    return e ? std::atoi(e) : 20;
  }();
  return nw == 16 ? launch_nw<16, true>(args, s) : launch_nw<20, true>(args, s);
}

}  // namespace ecf8::dev
