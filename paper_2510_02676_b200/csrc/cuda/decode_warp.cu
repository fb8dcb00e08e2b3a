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
//   decode   each lane walks its 8 windows into its nibble slot: one
//            continuous walk when the tile passed the upload-time gap check
//            (verify_gaps_kernel), else window by window (decode_common.cuh;
//            exact walk for flagged windows);
//   scan     5-step warp shuffle scan of the lane counts, segmented by
//            reference block, clamped to outpos limits (codec.cpp:239-246);
//   compact  funnel-shift copy of each lane's nibbles to their final place
//            in the warp's staging tile; shared words assembled by owners;
//            meanwhile the tile's sign/mantissa bytes stream into the freed
//            slots (cp.async, one round trip);
//   write    16 output bytes per lane-step (SWAR merge of exponent and
//            sign/mantissa nibbles), coalesced 128-bit stores, tile edges
//            byte-wise.
//
// The next tile's window words, gaps and outpos bounds are loaded into
// registers one tile ahead; the sign/mantissa bytes are prefetched into L2
// by one bulk prefetch per tile.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "decode.cuh"
#include "decode_common.cuh"
#include "decode_warp.cuh"

namespace ecf8::dev {

namespace {

// 33 slot rows: a lane's run is <= 256 nibbles (32 words); the staging tile
// holds 8192 nibbles + the 16-byte alignment offset.  With 1-bit codes (WIDE)
// both double: 512 nibbles per lane, 16384 per tile.
template <bool WIDE>
using WarpSmemT = WarpPipeSmem<WIDE ? 65 : 33, (WIDE ? 2 : 1) * 32 * kSlotWords + 8>;
// Direct-only tiles (every tile of the launch placed directly, the packed
// bytes from L2): the staging tile alone.
using DirectWarpSmem = WarpPipeSmem<1, 32 * kSlotWords + 8>;
template <bool WIDE, bool DIRECT>
using KernelWarpSmem = std::conditional_t<DIRECT, DirectWarpSmem, WarpSmemT<WIDE>>;

// Static shared memory: the tile queue, the current segment's descriptor
// (read field by field where used: a register copy would pin ~30 registers
// for the whole tile loop) and the decode tables, laid out so that the fast
// table starts at shared address kFastAt = 0x4000 (the CTA window begins 1 KB
// in, after the reserved area): a probe address is offset + constant.  The
// kernel traps if the toolchain ever places it elsewhere.
struct StaticSmem {
  unsigned next_tile;  // CTA-local work queue of the current segment (relative)
  TensorDesc desc;     // the current segment's tensor
  unsigned char pad[0x4000 - 0x400 - offsetof(Tables, fast) - 8 - sizeof(TensorDesc)];
  Tables tb;
};
static_assert(offsetof(StaticSmem, tb) + offsetof(Tables, fast) == 0x4000 - 0x400, "fast table offset");
__shared__ __align__(1024) StaticSmem g_s;

#define g_tb g_s.tb

// The byte-step variant (Lmin >= 2): the staged tables are the byte-step
// decoder (16 KB + 4 KB of completion masks), pinned at kFsmAt; windows off
// the verified path read the fast / cascade tables through L1.
struct StaticSmemFsm {
  unsigned next_tile;
  TensorDesc desc;
  PfSec pf[5];  // the segment's section table for the L2 prefetches (ECF8_PF_TAB)
  unsigned char pad[kFsmAt - 0x400 - 8 - sizeof(TensorDesc) - 5 * sizeof(PfSec)];
  std::uint32_t fsm[256 * kFsmStates];
  std::uint8_t cm[256 * kFsmStates];
};
static_assert(offsetof(StaticSmemFsm, fsm) == kFsmAt - 0x400, "fsm table offset");
static_assert(offsetof(StaticSmemFsm, cm) == kFsmCmAt - 0x400, "fsm mask offset");
__shared__ __align__(1024) StaticSmemFsm g_f;

__device__ __forceinline__ void stage_fsm(const TensorDesc& d, int tid, int nthreads) {
  if (!d.fsm) return;
  const uint4* f4 = reinterpret_cast<const uint4*>(d.fsm);
  uint4* sf4 = reinterpret_cast<uint4*>(g_f.fsm);
  for (int i = tid; i < 256 * kFsmStates / 4; i += nthreads) sf4[i] = __ldg(f4 + i);
  const uint4* c4 = reinterpret_cast<const uint4*>(d.fsm_cm);
  uint4* sc4 = reinterpret_cast<uint4*>(g_f.cm);
  for (int i = tid; i < 256 * kFsmStates / 16; i += nthreads) sc4[i] = __ldg(c4 + i);
}

#ifndef ECF8_WB_UNROLL
#define ECF8_WB_UNROLL 8  // A/B (r3e, r3f): 8 +0.8-1.8 % over 4; 6, 12 and the stepped remainder (ECF8_WB_STEPS) less
#endif
constexpr int kWbUnroll = ECF8_WB_UNROLL;
#ifndef ECF8_STATIC_TILES
#define ECF8_STATIC_TILES 0
#endif
#ifndef ECF8_CLAIM_AHEAD
#define ECF8_CLAIM_AHEAD 0  // 1: claim the next tile one tile early (A/B: slower)
#endif
#ifndef ECF8_PF_GROUP
#define ECF8_PF_GROUP 1  // >1: the sections of G tiles per L2 prefetch, AHEAD tiles ahead (A/B: slower, lower clocks)
#endif
#ifndef ECF8_PF_TAB
#define ECF8_PF_TAB 1  // the next tile's L2 prefetch addresses from a per-segment section table (A/B r3n: +1.3-1.6 %)
#endif
#ifndef ECF8_PF_AHEAD
#define ECF8_PF_AHEAD 32  // tiles between a claim and the group it prefetches (a multiple of ECF8_PF_GROUP)
#endif  // write-back chunks per lane and loop step

// Output to global memory (d.out).  Launched with programmatic stream
// serialization, this grid may start while the previous one finishes; its
// inputs are immutable, so only the stores wait for the previous grid (a
// no-op once it has completed).
#ifndef ECF8_STG
#define ECF8_STG 1  // 0: generic stores (ptxas then keeps the write-back's shared loads behind them)
#endif
struct GlobalOut {
  std::uint8_t* base;  // element S0
  __device__ __forceinline__ void wait() const { asm volatile("griddepcontrol.wait;" ::: "memory"); }
  __device__ __forceinline__ void chunk(std::uint32_t c, const uint4& r) const {
#if ECF8_STG
    // st.global: a store ptxas knows cannot alias shared memory, so the next
    // chunks' stage / packed loads may be issued ahead of it
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(reinterpret_cast<uint4*>(base) + c), "r"(r.x),
                 "r"(r.y), "r"(r.z), "r"(r.w));
#else
    reinterpret_cast<uint4*>(base)[c] = r;
#endif
  }
  __device__ __forceinline__ void byte(std::uint32_t i, std::uint8_t b) const { base[i] = b; }
  __device__ __forceinline__ void done() const {}
};

// Output of a tiled weight (fused layout) to row-major rows: element e of
// tile t = e / 16384 (tile (nt, kt) = (t / KT, t % KT)) at offset o = e %
// 16384 is row 128 nt + o / 128, 16-byte chunk ((o / 16) ^ (o / 128 % 8)) of
// K tile kt (the 128B swizzle undone); 16-element chunks stay contiguous.  A
// warp tile spans at most two weight tiles: their row bases are computed
// once.  Only elements in [lo, hi) are written.
struct TiledOut {
  std::uint8_t* rb0;      // row-major address of weight tile t0's (row 0, column 0)
  std::uint8_t* rb1;      // ... of tile t0 + 1
  std::uint64_t S0, bnd;  // element of chunk 0; first element of tile t0 + 1
  std::uint64_t lo, hi;
  std::uint32_t k;
  __device__ __forceinline__ void wait() const { asm volatile("griddepcontrol.wait;" ::: "memory"); }
  __device__ __forceinline__ std::uint8_t* at(std::uint64_t e) const {
    const std::uint32_t o = static_cast<std::uint32_t>(e) & 16383u, r = o >> 7;
    return (e >= bnd ? rb1 : rb0) + static_cast<std::uint64_t>(r) * k + ((((o >> 4) ^ r) & 7u) << 4) + (o & 15u);
  }
  __device__ __forceinline__ void chunk(std::uint32_t c, const uint4& v) const {
    const std::uint64_t e = S0 + 16 * static_cast<std::uint64_t>(c);
    if (e < lo || e >= hi) return;
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(at(e)), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
  }
  __device__ __forceinline__ void byte(std::uint32_t i, std::uint8_t b) const {
    const std::uint64_t e = S0 + i;
    if (e < lo || e >= hi) return;
    *at(e) = b;
  }
  __device__ __forceinline__ void done() const {}
};

__device__ __forceinline__ TiledOut tiled_out(const TensorDesc& d, std::uint64_t A) {
  TiledOut t;
  t.S0 = A & ~std::uint64_t{15};
  const std::uint64_t kt_n = d.out_tiled_k >> 7, t0 = t.S0 >> 14;
  const std::uint64_t nt = t0 / kt_n, kt = t0 - nt * kt_n;
  const std::uint64_t nt1 = kt + 1 == kt_n ? nt + 1 : nt, kt1 = kt + 1 == kt_n ? 0 : kt + 1;
  t.rb0 = d.out + (nt * 128) * d.out_tiled_k + kt * 128;
  t.rb1 = d.out + (nt1 * 128) * d.out_tiled_k + kt1 * 128;
  t.bnd = (t0 + 1) << 14;
  t.lo = d.out_lo;
  t.hi = d.out_hi;
  t.k = d.out_tiled_k;
  return t;
}

// One tile: decode + scan, compact, write back.
template <bool WIDE, bool TILED = false, bool DIRECT = false, class WSm>
__device__ __forceinline__ void warp_tile(const TensorDesc& d, const WarpIn& in, std::uint32_t log2T,
                                          std::uint32_t len_off, WSm& ws, int lane) {
  if constexpr (DIRECT) {
    direct_tile<kWbUnroll, kLaneWin, true>(
        d, in, ws, lane, [&] { return GlobalOut{d.out + ((in.A & ~std::uint64_t{15}) - d.out_offset)}; },
        tile_verified(d, in, log2T));
    return;
  } else {

  // slots interleaved word by word (word j of lane L at slot[32 j + L]): the
  // lanes' slot stores and reads hit 32 different banks
  const std::uint32_t slot = smem_addr(ws.slot + lane);
  LaneRun run;
  if constexpr (WIDE) {
    run = warp_decode_scan<kLaneWin, 128, true>(in, log2T, len_off, SmemTables{g_tb}, slot, lane,
                                                tile_verified(d, in, log2T));
  } else if (d.fsm && d.endgap) {  // byte steps: whole lanes on verified tiles, else window by window
    const bool verified = tile_verified(d, in, log2T);
    const std::uint32_t v = static_cast<std::uint32_t>((in.b0 << log2T) >> 8);  // the tile's verification tile
    if ((in.dir >> (v & 31)) & 1u) {  // every lane's output offset known: decode in place
      // the packed sign/mantissa bytes come from L2 at write-back (prefetched at the tile's start)
      if constexpr (TILED)  // a tiled weight back to row-major rows (ecf8_fused_decode_rows)
        direct_tile<kWbUnroll, kLaneWin, true>(d, in, ws, lane, [&] { return tiled_out(d, in.A); }, verified);
      else
        direct_tile<kWbUnroll, kLaneWin, true>(
            d, in, ws, lane, [&] { return GlobalOut{d.out + ((in.A & ~std::uint64_t{15}) - d.out_offset)}; }, verified);
      return;
    }
    if constexpr (TILED) __trap();  // row-major output of tiled weights needs direct tiles (checked by the caller)
    // the lanes' endgap words (loaded with the tile only where a direct tile
    // does not need them): `in` is the caller's mutable tile (the byte-step loop)
    const_cast<WarpIn&>(in).gnext = load_gnext(d, in, lane);
    run = warp_decode_scan<kLaneWin, 128, false, GlobalTables, true>(in, log2T, len_off, GlobalTables{d}, slot, lane,
                                                                     verified);
  } else {  // an incomplete code (no encoder writes one): the reference walk per window, tables through L1
    run = warp_decode_scan<kLaneWin, 128, false, GlobalTables, false>(in, log2T, len_off, GlobalTables{d}, slot, lane,
                                                                      false);
  }
  GlobalOut out{d.out + ((in.A & ~std::uint64_t{15}) - d.out_offset)};
  compact_write<kWbUnroll>(d, in.A, in.E, run, ws, lane, out);
  }
}

template <int NW, bool WIDE, bool TILED = false, bool DIRECT = false>
__global__ void __launch_bounds__(NW * 32, 1) decode_warp_kernel(const LaunchArgs args) {
  using WarpSmem = KernelWarpSmem<WIDE, DIRECT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpSmem& ws = reinterpret_cast<WarpSmem*>(smem_raw)[warp];
  unsigned& next_tile = WIDE ? g_s.next_tile : g_f.next_tile;
  TensorDesc& desc = WIDE ? g_s.desc : g_f.desc;
  asm volatile("griddepcontrol.launch_dependents;");  // the next decode may claim SMs as ours free up
  const std::uint64_t total_tiles = args.total_tiles;
  const std::uint64_t t_lo = total_tiles * blockIdx.x / gridDim.x;
  const std::uint64_t t_hi = total_tiles * (blockIdx.x + 1) / gridDim.x;

  for (std::uint64_t seg = t_lo; seg < t_hi;) {
    std::uint64_t seg_end;
    int di = 0;
    if (args.descs) {
      if (args.n_desc <= 32) {  // one parallel probe instead of a dependent binary search
        const bool le = lane < args.n_desc && args.descs[lane].tile_begin <= seg;
        di = 31 - __clz(__ballot_sync(0xffffffffu, le) | 1u);
      } else {
        di = find_desc(args.descs, args.n_desc, seg);
      }
      seg_end = (di + 1 < args.n_desc) ? args.descs[di + 1].tile_begin : total_tiles;
    } else {
      seg_end = total_tiles;
    }
    if (seg_end > t_hi) seg_end = t_hi;
    __syncthreads();  // every warp is done with the previous tables and descriptor
    // The segment's descriptor lives in shared memory, read field by field
    // where used: ~30 registers a register copy would pin for the whole loop.
    // Warp 0 copies it 8 bytes per lane.
    if (warp == 0) {
      static_assert(sizeof(TensorDesc) % 8 == 0 && sizeof(TensorDesc) <= 32 * 8, "descriptor copy");
      const auto* src = reinterpret_cast<const unsigned long long*>(args.descs ? &args.descs[di] : &args.inline_desc);
      if (lane < static_cast<int>(sizeof(TensorDesc) / 8)) reinterpret_cast<unsigned long long*>(&desc)[lane] = src[lane];
    }
    __syncthreads();
    const TensorDesc& d = desc;
    const std::uint32_t log2T = 31 - __clz(d.T);
    if constexpr (WIDE) {
      if (threadIdx.x == 0 && smem_addr(g_tb.fast) != kFastAt) __trap();  // the walk addresses the table at kFastAt
      stage_tables(d, g_tb, threadIdx.x, NW * 32);
    } else {
      if (threadIdx.x == 0 && smem_addr(g_f.fsm) != kFsmAt) __trap();  // the byte steps address the table at kFsmAt
      stage_fsm(d, threadIdx.x, NW * 32);
    }
    const std::uint32_t len_off = (d.n_luts - 1) << 8;
    if (threadIdx.x == 0) next_tile = NW;
#if ECF8_PF_TAB
    if constexpr (!WIDE)
      if (threadIdx.x < 5) g_f.pf[threadIdx.x] = pf_section(d, threadIdx.x, log2T);
#endif
    __syncthreads();

    // Tiles are handed out dynamically inside the CTA (warp w starts with
    // tile seg + w, then takes the next unclaimed one), so the warps of a
    // segment finish within one tile of each other whatever the per-tile
    // cost.  WIDE: the next tile is claimed and its inputs loaded into
    // registers one tile ahead.  Byte-step variant: the registers go to the
    // two decode paths instead; the next tile's inputs are prefetched into L2
    // (bulk prefetches, one tile ahead) and loaded at the tile's start.
    std::uint64_t tile = seg + warp;
    if constexpr (WIDE) {
      WarpIn nxt;
      if (tile < seg_end) load_warp_tile(d, tile, log2T, lane, nxt);
      while (tile < seg_end) {
        const WarpIn cur = nxt;
        if (lane == 0) {  // sign/mantissa bytes of this tile -> L2 (one bulk TMA prefetch)
          const std::uint64_t p0 = (cur.A >> 1) & ~std::uint64_t{15};
          const std::uint32_t bytes = static_cast<std::uint32_t>((((cur.E + 1) >> 1) - p0 + 15) & ~std::uint64_t{15});
          if (bytes)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(d.packed + p0), "r"(bytes) : "memory");
        }
        unsigned claim = 0;
        if (lane == 0) claim = atomicAdd(&next_tile, 1u);
        const std::uint64_t next = seg + __shfl_sync(0xffffffffu, claim, 0);
        if (next < seg_end) load_warp_tile(d, next, log2T, lane, nxt);
        warp_tile<WIDE>(d, cur, log2T, len_off, ws, lane);
        tile = next;
      }
    } else {
#if ECF8_CLAIM_AHEAD
      // The tile after `tile` is claimed one tile early, so the claim's
      // shared atomic completes while a tile decodes; its sections go to L2
      // at the end of the tile before it (a tile of lead).  Claims are held
      // as 32-bit offsets from seg (one register).
      const std::uint32_t n_rel = static_cast<std::uint32_t>(seg_end - seg);
      if (tile < seg_end && lane < 5) prefetch_tile_l2(d, tile, log2T, lane);
      unsigned claim = 0;
      if (lane == 0) claim = atomicAdd(&next_tile, 1u);
      std::uint32_t next = __shfl_sync(0xffffffffu, claim, 0);
      if (next < n_rel && lane < 5) prefetch_tile_l2(d, seg + next, log2T, lane);
      while (tile < seg_end) {
        WarpIn cur;
        load_warp_tile<kLaneWin, true, false, !DIRECT>(d, tile, log2T, lane, cur);
        unsigned claim2 = 0;
        if (lane == 0 && next < n_rel) claim2 = atomicAdd(&next_tile, 1u);
        warp_tile<WIDE>(d, cur, log2T, len_off, ws, lane);
        const std::uint32_t next2 = next < n_rel ? __shfl_sync(0xffffffffu, claim2, 0) : n_rel;
        if (next2 < n_rel && lane < 5) prefetch_tile_l2(d, seg + next2, log2T, lane);
        tile = seg + next;
        next = next2;
      }
#else
#if ECF8_PF_GROUP > 1
      // The sections go to L2 in groups of G consecutive tiles, kPfAhead
      // tiles ahead of the claims: the claim of tile c prefetches group
      // [c + kPfAhead, c + kPfAhead + G) when that starts a group; the warps
      // prefetch the groups before the first claim between them.
      constexpr std::uint32_t G = ECF8_PF_GROUP, kPfAhead = ECF8_PF_AHEAD;
      const std::uint64_t n_rel = seg_end - seg;
      constexpr std::uint32_t kInit = (NW + kPfAhead + G - 1) / G;  // groups before the first claim's
      for (std::uint32_t g = warp; g < kInit && g * G < n_rel; g += NW)
        if (lane < 5) prefetch_tile_l2(d, seg + g * G, log2T, lane, static_cast<std::uint32_t>(min(std::uint64_t{G}, n_rel - g * G)));
#elif ECF8_PF_TAB
      if (tile < seg_end && lane < 5) prefetch_tile_l2_tab(d, g_f.pf, tile, log2T, lane);
#else
      if (tile < seg_end && lane < 5) prefetch_tile_l2(d, tile, log2T, lane);
#endif
      while (tile < seg_end) {
        WarpIn cur;
        load_warp_tile<kLaneWin, true, false, !DIRECT>(d, tile, log2T, lane, cur);
#if ECF8_STATIC_TILES  // A/B: round-robin tiles (no shared atomic)
        const std::uint64_t next = tile + NW;
        const unsigned claim = static_cast<unsigned>(next - seg);
#else
        unsigned claim = 0;
        if (lane == 0) claim = atomicAdd(&next_tile, 1u);
        claim = __shfl_sync(0xffffffffu, claim, 0);
        const std::uint64_t next = seg + claim;
#endif
#if ECF8_PF_GROUP > 1
        {
          const std::uint64_t pf = std::uint64_t{claim} + kPfAhead;
          if (pf % G == 0 && pf < n_rel && lane < 5)
            prefetch_tile_l2(d, seg + pf, log2T, lane, static_cast<std::uint32_t>(min(std::uint64_t{G}, n_rel - pf)));
        }
#elif ECF8_PF_TAB
        if (next < seg_end && lane < 5) prefetch_tile_l2_tab(d, g_f.pf, next, log2T, lane);
#else
        if (next < seg_end && lane < 5) prefetch_tile_l2(d, next, log2T, lane);
#if ECF8_WIN_L1
        if (next < seg_end) {  // A/B: the next tile's windows into this SM's L1 too
          const std::uint32_t m1 = 256u >> log2T;
          const std::uint64_t b0 = d.blk_begin + (next - d.tile_begin) * m1;
          const std::uint64_t nb = d.blk_end - b0 < m1 ? d.blk_end - b0 : m1;
          const std::uint64_t e0 = 8 * (b0 << log2T), e1 = e0 + 8 * (nb << log2T) + 8;
          for (std::uint64_t a = (e0 & ~std::uint64_t{127}) + 128u * lane; a < e1; a += 32u * 128u)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(d.encoded + a));
        }
#endif
#endif
        if (lane == 0) {  // this tile's sign/mantissa bytes -> L2 (direct tiles read them at write-back)
          const std::uint64_t p0 = (cur.A >> 1) & ~std::uint64_t{15};
          const std::uint32_t bytes = static_cast<std::uint32_t>((((cur.E + 1) >> 1) - p0 + 15) & ~std::uint64_t{15});
          if (bytes) prefetch_l2(d.packed + p0, bytes);
        }
#if ECF8_PK_L1
        {  // A/B: ... and into this SM's L1, one 128-byte line per lane
          const std::uint64_t l0 = (cur.A >> 1) & ~std::uint64_t{127}, l1 = (cur.E + 1) >> 1;
          for (std::uint64_t a = l0 + 128u * lane; a < l1; a += 32u * 128u)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(d.packed + a));
        }
#endif
        warp_tile<WIDE, TILED, DIRECT>(d, cur, log2T, len_off, ws, lane);
        tile = next;
      }
#endif
    }
    seg = seg_end;
  }
}

// ---- variant 6: codes with a 1-bit word by 64-bit byte steps (E5M2 bytes
// through the reference format, small-gamma E4M3).  Same structure as the
// byte-step loop above; every tile is direct (checked at upload), the
// packed bytes come from L2, the 32 KB table is staged per segment.
using Fsm64WarpSmem = WarpPipeSmem<1, 2 * 32 * kSlotWords + 8>;  // 16384 nibbles + alignment
__shared__ __align__(16) std::uint64_t g_fsm64[256 * kFsmStates];
__shared__ unsigned g6_next_tile;
__shared__ TensorDesc g6_desc;
__shared__ PfSec g6_pf[5];  // the segment's prefetch section table (ECF8_PF_TAB)

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) decode_fsm64_kernel(const LaunchArgs args) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Fsm64WarpSmem& ws = reinterpret_cast<Fsm64WarpSmem*>(smem_raw)[warp];
  asm volatile("griddepcontrol.launch_dependents;");
  const std::uint64_t total_tiles = args.total_tiles;
  const std::uint64_t t_lo = total_tiles * blockIdx.x / gridDim.x;
  const std::uint64_t t_hi = total_tiles * (blockIdx.x + 1) / gridDim.x;
  const Fsm64At ft{smem_addr(g_fsm64)};
  for (std::uint64_t seg = t_lo; seg < t_hi;) {
    std::uint64_t seg_end;
    int di = 0;
    if (args.descs) {
      if (args.n_desc <= 32) {
        const bool le = lane < args.n_desc && args.descs[lane].tile_begin <= seg;
        di = 31 - __clz(__ballot_sync(0xffffffffu, le) | 1u);
      } else {
        di = find_desc(args.descs, args.n_desc, seg);
      }
      seg_end = (di + 1 < args.n_desc) ? args.descs[di + 1].tile_begin : total_tiles;
    } else {
      seg_end = total_tiles;
    }
    if (seg_end > t_hi) seg_end = t_hi;
    __syncthreads();
    if (warp == 0) {
      const auto* src = reinterpret_cast<const unsigned long long*>(args.descs ? &args.descs[di] : &args.inline_desc);
      if (lane < static_cast<int>(sizeof(TensorDesc) / 8)) reinterpret_cast<unsigned long long*>(&g6_desc)[lane] = src[lane];
    }
    __syncthreads();
    const TensorDesc& d = g6_desc;
    const std::uint32_t log2T = 31 - __clz(d.T);
    {
      const uint4* f4 = reinterpret_cast<const uint4*>(d.fsm64);
      uint4* s4 = reinterpret_cast<uint4*>(g_fsm64);
      for (int i = threadIdx.x; i < 256 * kFsmStates / 2; i += NW * 32) s4[i] = __ldg(f4 + i);
    }
    if (threadIdx.x == 0) g6_next_tile = NW;
#if ECF8_PF_TAB
    if (threadIdx.x < 5) g6_pf[threadIdx.x] = pf_section(d, threadIdx.x, log2T);
#define PF6(t) prefetch_tile_l2_tab(d, g6_pf, t, log2T, lane)
#else
#define PF6(t) prefetch_tile_l2(d, t, log2T, lane)
#endif
    __syncthreads();
    std::uint64_t tile = seg + warp;
    if (tile < seg_end && lane < 5) PF6(tile);
    while (tile < seg_end) {
      WarpIn cur;
      load_warp_tile<kLaneWin, true, false, false>(d, tile, log2T, lane, cur);
      unsigned claim = 0;
      if (lane == 0) claim = atomicAdd(&g6_next_tile, 1u);
      const std::uint64_t next = seg + __shfl_sync(0xffffffffu, claim, 0);
      if (next < seg_end && lane < 5) PF6(next);
      if (lane == 0) {  // this tile's sign/mantissa bytes -> L2 (read at write-back)
        const std::uint64_t p0 = (cur.A >> 1) & ~std::uint64_t{15};
        const std::uint32_t bytes = static_cast<std::uint32_t>((((cur.E + 1) >> 1) - p0 + 15) & ~std::uint64_t{15});
        if (bytes) prefetch_l2(d.packed + p0, bytes);
      }
      direct_tile64<kWbUnroll>(
          d, cur, ws, lane, [&] { return GlobalOut{d.out + ((cur.A & ~std::uint64_t{15}) - d.out_offset)}; }, ft);
      tile = next;
    }
    seg = seg_end;
  }
}

#ifndef ECF8_DIRECT_WARPS
#define ECF8_DIRECT_WARPS 24
#endif

#ifndef ECF8_FSM64_WARPS
#define ECF8_FSM64_WARPS 22  // 22 x 8.2 KB of staging + the 32 KB table
#endif

template <int NW, bool WIDE = false, bool TILED = false, bool DIRECT = false>
cudaError_t launch_nw(const LaunchArgs& args, cudaStream_t s) {
  static int grid_cap = 0;
  const int smem = static_cast<int>(sizeof(KernelWarpSmem<WIDE, DIRECT>)) * NW;
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(decode_warp_kernel<NW, WIDE, TILED, DIRECT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_warp_kernel<NW, WIDE, TILED, DIRECT>, NW * 32, smem);
    if (e != cudaSuccess) return e;
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const std::uint64_t want = (args.total_tiles + NW - 1) / NW;
  const std::uint64_t grid = want < static_cast<std::uint64_t>(grid_cap) ? want : grid_cap;
  if (grid == 0) return cudaSuccess;
  // Programmatic dependent launch: consecutive decodes (layer after layer)
  // overlap the tail of one grid with the start of the next.
  static const bool pdl = std::getenv("ECF8_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = static_cast<std::size_t>(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, decode_warp_kernel<NW, WIDE, TILED, DIRECT>, args);
}

// One CTA iteration per 256-window tile, one thread per window: the
// reference walk of the window (window_end, codec.cpp:143-160) gives its end
// nibble (endgap) and its word count.  A window inside an 8-window group that
// does not end where the next window's gap says clears its tile's tile_ok
// bit.  The counts are summed per 4-window group and scanned per block
// (lane_start: one u16 per group; the two groups of an 8-window lane in one
// 32-bit word);
// a block that decodes to fewer words than its outpos range, or to more (but
// the tensor's last block), clears tile_direct.
__global__ void __launch_bounds__(256) verify_gaps_kernel(const TensorDesc d, std::uint64_t w_begin,
                                                          std::uint64_t n_win, std::uint64_t nb_total,
                                                          std::uint32_t* tile_ok, std::uint8_t* endgap,
                                                          std::uint16_t* lane_start, std::uint32_t* tile_direct) {
  __shared__ Tables tb;
  __shared__ std::uint32_t gsum[64];
  __shared__ unsigned over;
  stage_tables(d, tb, threadIdx.x, blockDim.x);
  __syncthreads();
  const std::uint32_t len_off = (d.n_luts - 1) << 8;
  const std::uint32_t log2T = 31 - __clz(d.T);
  const std::uint64_t n_tiles = (n_win - w_begin + 255) / 256;  // w_begin: a multiple of 256
  for (std::uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const std::uint64_t w_tile = w_begin + 256 * t, k = w_tile + threadIdx.x;
    bool bad = false;
    std::uint32_t eg = 0, cnt = 0;
    if (k < n_win) {
      const uint2 a = __ldg(reinterpret_cast<const uint2*>(d.encoded + 8 * k));
      const uint2 b = __ldg(reinterpret_cast<const uint2*>(d.encoded + 8 * k + 8));
      const std::uint32_t g0 = (d.gaps[k >> 1] >> ((k & 1) ? 0 : 4)) & 15u;
      eg = window_end(bswap32(a.x), bswap32(a.y), bswap32(b.x), bswap32(b.y), g0, SmemTables{tb}, len_off, &cnt) - 64;
      if ((k & 7) != 7 && k + 1 < n_win) {
        const std::uint32_t g1 = (d.gaps[(k + 1) >> 1] >> (((k + 1) & 1) ? 0 : 4)) & 15u;
        bad = eg != g1;
      }
    }
    // two windows per byte, the even one in the high nibble (gap layout)
    const std::uint32_t pair = __shfl_xor_sync(0xffffffffu, eg, 1);
    if (k < n_win && !(k & 1)) endgap[k >> 1] = static_cast<std::uint8_t>((eg << 4) | (k + 1 < n_win ? pair : 0u));
    if (__ballot_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) {
      const std::uint64_t v = k >> 8;
      atomicAnd(tile_ok + (v >> 5), ~(1u << (v & 31)));
    }
    if (lane_start) {
      std::uint32_t g = cnt;  // the 4-window group's words
      g += __shfl_xor_sync(0xffffffffu, g, 1);
      g += __shfl_xor_sync(0xffffffffu, g, 2);
      if ((threadIdx.x & 3) == 0) gsum[threadIdx.x >> 2] = g;
      if (threadIdx.x == 0) over = 0;
      __syncthreads();
      if (threadIdx.x < 32) {  // lane i: groups 2i, 2i + 1 (windows 8i .. 8i + 7)
        const std::uint32_t i = threadIdx.x, v0 = gsum[2 * i], v1 = gsum[2 * i + 1], v = v0 + v1;
        std::uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (i >= static_cast<std::uint32_t>(o)) incl += y;
        }
        const std::uint32_t lpb = log2T >= 8 ? 32u : (1u << (log2T - 3));  // lanes (8 windows) per block
        const std::uint32_t excl = incl - v - __shfl_sync(0xffffffffu, incl - v, i & ~(lpb - 1));
        const std::uint64_t wg = w_tile + 8 * i;
        if (wg < n_win) {
          reinterpret_cast<std::uint32_t*>(lane_start)[wg >> 3] = excl | ((excl + v0) << 16);
          if ((i & (lpb - 1)) == lpb - 1 || wg + 8 >= n_win) {  // the block's last lane
            const std::uint64_t blk = wg >> log2T;
            // direct placement needs every block to decode to exactly its
            // range (the tensor's last block may decode past it: padding)
            const std::uint64_t range = d.outpos[blk + 1] - d.outpos[blk];
            if (excl + v < range || (blk + 1 < nb_total && excl + v > range)) atomicOr(&over, 1u);
          }
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && over) {  // a block decodes past its range: no direct placement for this tile
        const std::uint64_t v = w_tile >> 8;
        atomicAnd(tile_direct + (v >> 5), ~(1u << (v & 31)));
      }
      __syncthreads();  // gsum / over are reused by the next tile
    }
  }
}

__global__ void stream_fence_kernel() {}

}  // namespace

// Warps per CTA: 24 (default; 24 x 8.2 KB of warp state + 29 KB of tables,
// <= 85 registers), 22 or 20 (ECF8_WARPS).  Measured (8 x 14336x4096, T 256):
// 24 warps 3532 GB/s, 22 warps 3448 GB/s, 20 warps 3206 GB/s.
cudaError_t launch_decode_warp(const LaunchArgs& args, cudaStream_t s) {
  static const int nw = [] {
    const char* e = std::getenv("ECF8_WARPS");
    return e ? std::atoi(e) : 24;
  }();
  if (!args.descs && args.inline_desc.out_tiled_k) return launch_nw<24, false, true>(args, s);  // rows of a fused weight
  return nw == 20 ? launch_nw<20>(args, s) : nw == 22 ? launch_nw<22>(args, s) : launch_nw<24>(args, s);
}

// Variant 7 (every tile direct): the staging tile alone per warp.  A/B
// (70B layers): 24-28 warps the same, +1.5-2 % over variant 4; 30 warps -3 %.
cudaError_t launch_decode_warp_direct(const LaunchArgs& args, cudaStream_t s) {
  if (!args.descs && args.inline_desc.out_tiled_k) return launch_nw<24, false, true>(args, s);  // rows of a fused weight
  return launch_nw<ECF8_DIRECT_WARPS, false, false, true>(args, s);
}

// Variant 5 (1-bit codes): 12 warps x 16.5 KB of warp state.
cudaError_t launch_decode_warp_wide(const LaunchArgs& args, cudaStream_t s) { return launch_nw<12, true>(args, s); }

// Variant 6 (1-bit codes, every tile direct): 64-bit byte steps.
cudaError_t launch_decode_fsm64(const LaunchArgs& args, cudaStream_t s) {
  constexpr int NW = ECF8_FSM64_WARPS;
  static int grid_cap = 0;
  const int smem = static_cast<int>(sizeof(Fsm64WarpSmem)) * NW;
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(decode_fsm64_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_fsm64_kernel<NW>, NW * 32, smem);
    if (e != cudaSuccess) return e;
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const std::uint64_t want = (args.total_tiles + NW - 1) / NW;
  const std::uint64_t grid = want < static_cast<std::uint64_t>(grid_cap) ? want : grid_cap;
  if (grid == 0) return cudaSuccess;
  static const bool pdl = std::getenv("ECF8_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = static_cast<std::size_t>(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, decode_fsm64_kernel<NW>, args);
}

cudaError_t launch_verify_gaps(const TensorDesc& d, std::uint64_t nb_total, std::uint32_t* tile_ok,
                               std::uint8_t* endgap, std::uint16_t* lane_start, std::uint32_t* tile_direct,
                               cudaStream_t s) {
  const std::uint64_t w_begin = d.blk_begin * d.T, n_win = d.blk_end * d.T;
  if (n_win <= w_begin) return cudaSuccess;
  const std::uint64_t blocks = (n_win - w_begin + 255) / 256;
  if (d.T < 8 || d.T > 256) lane_start = nullptr;  // groups of 8 windows inside one block
  verify_gaps_kernel<<<static_cast<unsigned>(blocks < 1184 ? blocks : 1184), 256, 0, s>>>(
      d, w_begin, n_win, nb_total, tile_ok, endgap, lane_start, tile_direct);
  // A plain launch after it: a decode launched next with programmatic
  // serialization may only overlap this empty grid, which starts after the
  // gap check has completed -- the tile bits are final before any decode reads them.
  stream_fence_kernel<<<1, 32, 0, s>>>();
  return cudaGetLastError();
}

}  // namespace ecf8::dev
