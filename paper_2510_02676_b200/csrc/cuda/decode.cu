// decode.cu -- ECF8 -> FP8 decode kernels for sm_100a (B200): tile-group
// kernel, count_phase kernel, launch dispatch.
//
// Replaces the reference's OpenMP block decoder
// (/root/reference/proj/src/codec.cpp:133-273: count_phase, Blelloch scan,
// emit_phase, staging copy).  The reference decodes every symbol twice
// (count, then emit); these kernels decode once.  Two kernel shapes:
//
//   decode_warp.cu  one warp owns a 256-window tile (T in [8, 256], shortest
//                   code >= 2 bits -- the common case); warp-synchronous.
//   this file       GROUPS independent 256-thread tile groups per CTA for
//                   the remaining geometries (T = 1, 2, 512, 1024 or 1-bit
//                   codes); the groups share one shared-memory copy of the
//                   tables and synchronise with their own named barrier.
//
// Per tile (a run of whole reference blocks): window bits -> registers
// (prefetched a tile ahead) -> table walk (decode_common.cuh) -> nibble
// slots -> scan of counts seeded by outpos[] and clamped to the block limits
// (codec.cpp:239-246) -> funnel-shift compaction into a nibble staging tile
// -> SWAR merge with the sign/mantissa nibbles -> 16-byte stores; tile edges
// byte-wise.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "decode.cuh"
#include "decode_common.cuh"

namespace ecf8::dev {

bool warp_variant_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("ECF8_NO_WARP_KERNEL");
    return !(e && e[0] == '1');
  }();
  return on;
}

cudaError_t launch_decode_warp(const LaunchArgs& args, cudaStream_t s);       // decode_warp.cu
cudaError_t launch_decode_fsm64(const LaunchArgs& args, cudaStream_t s);      // decode_warp.cu
cudaError_t launch_decode_warp_wide(const LaunchArgs& args, cudaStream_t s);  // decode_warp.cu (1-bit codes)
cudaError_t launch_decode_warp_direct(const LaunchArgs& args, cudaStream_t s);  // decode_warp.cu (every tile direct)

namespace {

constexpr int kWarps = kThreads / 32;  // warps per group

template <int SLOTW>
struct GroupSmem {
  static constexpr int kSlotStride = SLOTW + 1;             // words; odd => no bank conflicts
  static constexpr int kStageWords = kThreads * SLOTW + 8;  // tile nibbles + 16-nibble slack
  std::uint32_t slot[kThreads * kSlotStride];
  alignas(16) std::uint32_t stage[kStageWords];
  std::uint32_t rs[kThreads];
  std::uint32_t re[kThreads];
  std::uint32_t head[kThreads];
  std::uint64_t blk[2][kThreads + 1];  // outpos[b0 .. b0 + nblk], by tile parity
  std::uint32_t warp_sum[kWarps];
};

template <int SLOTW, int GROUPS>
struct Smem {
  Tables tb;
  GroupSmem<SLOTW> g[GROUPS];
};

__device__ __forceinline__ void group_sync(int group) {
  asm volatile("bar.sync %0, %1;" ::"r"(group + 1), "r"(kThreads) : "memory");
}

// Tile geometry (uniform across a group).
struct TileGeo {
  std::uint64_t b0;    // first reference block
  std::uint32_t nblk;  // blocks in the tile
  std::uint32_t nwin;  // windows in the tile
};

template <int KWIN>
__device__ __forceinline__ TileGeo tile_geo(const TensorDesc& d, std::uint64_t tile, std::uint32_t log2T) {
  constexpr std::uint32_t kTileWin = static_cast<std::uint32_t>(kThreads) * KWIN;
  const std::uint32_t m = d.T >= kTileWin ? 1u : (kTileWin >> log2T);
  TileGeo g;
  g.b0 = d.blk_begin + (tile - d.tile_begin) * m;
  g.nblk = static_cast<std::uint32_t>(d.blk_end - g.b0 < m ? d.blk_end - g.b0 : m);
  g.nwin = g.nblk << log2T;
  return g;
}

// Bitstream words and gaps of one thread's windows; loaded a tile ahead.
template <int KWIN>
struct TileIn {
  uint2 win[KWIN + 1];  // window bytes, little-endian words
  std::uint32_t gaps;   // raw gap byte(s) covering my windows
};

template <int KWIN>
__device__ __forceinline__ void load_tile(const TensorDesc& d, const TileGeo& g, std::uint32_t log2T,
                                          int tid, TileIn<KWIN>& in) {
  const std::uint32_t wl = static_cast<std::uint32_t>(tid) * KWIN;
  if (wl < g.nwin) {
    const std::uint64_t w0g = g.b0 << log2T;
    const uint2* src = reinterpret_cast<const uint2*>(d.encoded) + (w0g + wl);
#pragma unroll
    for (int i = 0; i <= KWIN; ++i) in.win[i] = __ldg(src + i);
    if (KWIN == 1) in.gaps = __ldg(d.gaps + ((w0g + wl) >> 1));
    else if (KWIN == 2) in.gaps = __ldg(d.gaps + (w0g >> 1) + tid);
    else in.gaps = __ldg(reinterpret_cast<const std::uint16_t*>(d.gaps + (w0g >> 1)) + tid);
  }
}

template <int KWIN>
__device__ __forceinline__ std::uint32_t gap_of(std::uint32_t gaps, int i, std::uint32_t wl) {
  if (KWIN == 1) return (gaps >> ((wl & 1) ? 0 : 4)) & 15u;
  // byte j holds windows 2j (high nibble) and 2j + 1 (low nibble)
  return (gaps >> (8 * (i >> 1) + ((i & 1) ? 0 : 4))) & 15u;
}

// One group decodes one tile: windows -> slots -> scan -> staging -> HBM.
template <int KWIN, int SLOTW>
__device__ __forceinline__ void decode_tile(const TensorDesc& d, const TileGeo& g, const TileIn<KWIN>& cur,
                                            const std::uint64_t* blk, const Tables& tb,
                                            GroupSmem<SLOTW>& gs, std::uint32_t log2T,
                                            std::uint32_t len_off, int group, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  std::uint32_t* const my_slot = gs.slot + tid * GroupSmem<SLOTW>::kSlotStride;
  const std::uint32_t wl0 = static_cast<std::uint32_t>(tid) * KWIN;
  const bool active = wl0 < g.nwin;

  // ---- decode my windows into my slot
  const std::uint32_t slot_base = smem_addr(my_slot);
  SlotSink sink{slot_base};
  if (active) {
#pragma unroll
    for (int i = 0; i < KWIN; ++i) {
      if (wl0 + i < g.nwin)
        decode_window(bswap32(cur.win[i].x), bswap32(cur.win[i].y), bswap32(cur.win[i + 1].x),
                      bswap32(cur.win[i + 1].y), gap_of<KWIN>(cur.gaps, i, wl0 + i), SmemTables{tb}, len_off, sink);
    }
  }
  const std::uint32_t cnt = sink.finish(slot_base);

  // ---- exclusive scan of the per-thread counts
  std::uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) gs.warp_sum[warp] = incl;
  group_sync(group);
  const std::uint32_t wsum = lane < kWarps ? gs.warp_sum[lane] : 0u;
  std::uint32_t wincl = wsum;
#pragma unroll
  for (int o = 1; o < kWarps; o <<= 1) {
    const std::uint32_t y = __shfl_up_sync(0xffffffffu, wincl, o);
    if (lane >= o) wincl += y;
  }
  const std::uint32_t wexcl = wincl - wsum;
  constexpr std::uint32_t kLogKwin = KWIN == 1 ? 0 : (KWIN == 2 ? 1 : 2);
  const std::uint32_t log2tpb = log2T - kLogKwin;  // threads per reference block
  const std::uint32_t first_tid = log2tpb >= 8 ? 0u : (static_cast<std::uint32_t>(tid) & ~((1u << log2tpb) - 1));
  const std::uint32_t lexcl = incl - cnt;
  const std::uint32_t excl = __shfl_sync(0xffffffffu, wexcl, warp) + lexcl;
  const std::uint32_t first_lex = __shfl_sync(0xffffffffu, lexcl, first_tid & 31);
  const std::uint32_t first_excl = __shfl_sync(0xffffffffu, wexcl, first_tid >> 5) +
                                   ((first_tid >> 5) == static_cast<std::uint32_t>(warp) ? first_lex : 0u);

  // ---- my output range, clamped to my reference block's outpos limit
  const std::uint64_t A = blk[0];
  const std::uint32_t bl = wl0 >> log2T;
  const std::uint32_t bl_c = bl < g.nblk ? bl : g.nblk - 1;
  const std::uint32_t start_rel = static_cast<std::uint32_t>(blk[bl_c] - A) + excl - first_excl;
  const std::uint32_t lim_rel = static_cast<std::uint32_t>(blk[bl_c + 1] - A);
  const std::uint32_t cc = (active && start_rel < lim_rel) ? min(cnt, lim_rel - start_rel) : 0u;
  const std::uint32_t off = static_cast<std::uint32_t>(A & 15);  // staging nibble of element A
  const std::uint32_t d0 = start_rel + off, dend = d0 + cc;
  const std::uint32_t data_end = off + static_cast<std::uint32_t>(blk[g.nblk] - A);
  gs.rs[tid] = d0;
  gs.re[tid] = dend;

  // ---- move my nibbles to their final place; publish partial words
  std::uint32_t headv = 0, tailv = 0;
  const std::uint32_t fw = d0 >> 3, lw = (dend - 1) >> 3;
  const std::uint32_t f4 = (d0 & 7) * 4, lastn = ((dend - 1) & 7) + 1;
  if (cc) {
    std::uint32_t prev = my_slot[0];
    const std::uint32_t v0 = prev << f4;
    if (fw == lw) {
      const std::uint32_t v = v0 & low_nibbles(lastn);
      if (f4 == 0 && lastn == 8) gs.stage[fw] = v;
      else headv = v;
    } else {
      if (f4 == 0) gs.stage[fw] = v0;
      else headv = v0;
      std::uint32_t j = 1;
      for (std::uint32_t k = fw + 1; k < lw; ++k, ++j) {
        const std::uint32_t c = my_slot[j];
        gs.stage[k] = __funnelshift_l(prev, c, f4);
        prev = c;
      }
      const std::uint32_t v = __funnelshift_l(prev, my_slot[j], f4) & low_nibbles(lastn);
      if (lastn == 8) gs.stage[lw] = v;
      else tailv = v;
    }
  }
  gs.head[tid] = headv;
  group_sync(group);

  // ---- owners assemble words shared between threads
  if (cc) {
    const bool start_owner = (f4 == 0 || d0 == off) && !(f4 == 0 && (fw < lw || lastn == 8));
    const bool tail_owner = fw != lw && lastn != 8;
    if (start_owner || tail_owner) {
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 0 ? !start_owner : !tail_owner) continue;
        const std::uint32_t k = pass == 0 ? fw : lw;
        std::uint32_t v = pass == 0 ? headv : tailv;
        const std::uint32_t wend = min(8 * k + 8, data_end);
        std::uint32_t covered = dend;
        for (int j = tid + 1; covered < wend && j < kThreads; ++j) {
          const std::uint32_t rj = gs.rs[j], ej = gs.re[j];
          if (ej > rj) {
            v |= gs.head[j];
            covered = ej;
          }
        }
        gs.stage[k] = v;
      }
    }
  }
  group_sync(group);

  // ---- write-back: exponent nibbles + sign/mantissa nibbles -> FP8 bytes
  const std::uint64_t S0 = A - off;
  std::uint8_t* const out = d.out + (S0 - d.out_offset);
  const std::uint8_t* const pk = d.packed + (S0 >> 1);
  const std::uint32_t nch = (data_end + 15) >> 4;
  const std::uint32_t full_lo = (off + 15) >> 4, full_hi = data_end >> 4;  // full chunks [lo, hi)
  const uint2* sp = reinterpret_cast<const uint2*>(gs.stage);
  const uint2* pp = reinterpret_cast<const uint2*>(pk);
  uint4* op = reinterpret_cast<uint4*>(out);
  for (std::uint32_t c0 = full_lo + tid; c0 < full_hi; c0 += 4 * kThreads) {
    uint2 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // all loads first: four L2 round trips overlap
      const std::uint32_t ci = c0 + u * kThreads;
      if (ci < full_hi) q[u] = __ldg(pp + ci);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const std::uint32_t ci = c0 + u * kThreads;
      if (ci < full_hi) {
        const uint2 s = sp[ci];
        uint4 r;
        merge8(s.x, q[u].x, r.x, r.y);
        merge8(s.y, q[u].y, r.z, r.w);
        op[ci] = r;
      }
    }
  }
  if (tid < 2) {  // partial edge chunks (at most two), byte-wise
    const std::uint32_t ci = tid == 0 ? 0u : nch - 1;
    const bool partial = tid == 0 ? (full_lo > 0 && nch > 0) : (full_hi < nch && !(nch == 1 && full_lo > 0));
    if (partial) {
      const std::uint32_t g16 = 16 * ci;
      write_edge(gs.stage, out, pk, g16 < off ? off : g16, g16 + 16 < data_end ? g16 + 16 : data_end);
    }
  }
}

template <int KWIN, int SLOTW, int GROUPS>
__global__ void __launch_bounds__(kThreads * GROUPS, 1) decode_kernel(const LaunchArgs args) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<SLOTW, GROUPS>& sm = *reinterpret_cast<Smem<SLOTW, GROUPS>*>(smem_raw);
  const int group = threadIdx.x / kThreads, tid = threadIdx.x % kThreads;
  GroupSmem<SLOTW>& gs = sm.g[group];
  const std::uint64_t total_tiles = args.total_tiles;
  const std::uint64_t t_lo = total_tiles * blockIdx.x / gridDim.x;
  const std::uint64_t t_hi = total_tiles * (blockIdx.x + 1) / gridDim.x;
  std::uint32_t parity = 0;

  // Segments of the CTA's tile range that lie in one tensor: tables are
  // (re)loaded CTA-wide between segments, groups take tiles round robin.
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
    __syncthreads();  // every group is done with the previous tables
    stage_tables(d, sm.tb, threadIdx.x, kThreads * GROUPS);
    const std::uint32_t len_off = (d.n_luts - 1) << 8;
    __syncthreads();

    TileIn<KWIN> nxt;
    std::uint64_t nA = 0, nE = 0;  // tid 0: outpos bounds of the prefetched tile
    std::uint64_t tile = seg + group;
    if (tile < seg_end) {
      const TileGeo g0 = tile_geo<KWIN>(d, tile, log2T);
      load_tile<KWIN>(d, g0, log2T, tid, nxt);
      if (tid == 0) {
        nA = __ldg(d.outpos + g0.b0);
        nE = __ldg(d.outpos + g0.b0 + g0.nblk);
      }
    }
    for (; tile < seg_end; tile += GROUPS, parity ^= 1) {
      const TileGeo g = tile_geo<KWIN>(d, tile, log2T);
      const TileIn<KWIN> cur = nxt;
      std::uint64_t* const blk = gs.blk[parity];
      for (std::uint32_t i = tid; i <= g.nblk; i += kThreads) blk[i] = __ldg(d.outpos + g.b0 + i);
      if (tid == 0) {  // sign/mantissa bytes of this tile -> L2 (one bulk TMA prefetch)
        const std::uint64_t p0 = (nA >> 1) & ~std::uint64_t{15};
        const std::uint32_t bytes = static_cast<std::uint32_t>((((nE + 1) >> 1) - p0 + 15) & ~std::uint64_t{15});
        if (bytes)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(d.packed + p0), "r"(bytes) : "memory");
      }
      if (tile + GROUPS < seg_end) {
        const TileGeo g1 = tile_geo<KWIN>(d, tile + GROUPS, log2T);
        load_tile<KWIN>(d, g1, log2T, tid, nxt);
        if (tid == 0) {
          nA = __ldg(d.outpos + g1.b0);
          nE = __ldg(d.outpos + g1.b0 + g1.nblk);
        }
      }
      decode_tile<KWIN, SLOTW>(d, g, cur, blk, sm.tb, gs, log2T, len_off, group, tid);
    }
    seg = seg_end;
  }
}

__global__ void count_window_kernel(const std::uint8_t* w16, unsigned gap, TensorDesc d, std::uint32_t* out) {
  __shared__ Tables tb;
  stage_tables(d, tb, threadIdx.x, blockDim.x);
  __syncthreads();
  if (threadIdx.x == 0) {
    std::uint32_t w[4];
    for (int k = 0; k < 4; ++k) {
      std::uint32_t v = 0;
      for (int j = 0; j < 4; ++j) {
        const int idx = 4 * k + j;
        v = (v << 8) | (idx < 10 ? w16[idx] : 0u);  // only the 10 window bytes exist
      }
      w[k] = v;
    }
    CountSink c;
    decode_window_exact(w[0], w[1], w[2], w[3], gap & 15u, SmemTables{tb}, (d.n_luts - 1) << 8, c);
    *out = c.n4 >> 2;
  }
}

template <int KWIN, int SLOTW, int G>
cudaError_t launch_k(const LaunchArgs& args, cudaStream_t s) {
  static int grid_cap = 0;
  const int smem = static_cast<int>(sizeof(Smem<SLOTW, G>));
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<KWIN, SLOTW, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<KWIN, SLOTW, G>, kThreads * G, smem);
    if (e != cudaSuccess) return e;
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const std::uint64_t want = (args.total_tiles + G - 1) / G;  // every group gets work
  const std::uint64_t grid = want < static_cast<std::uint64_t>(grid_cap) ? want : grid_cap;
  if (grid == 0) return cudaSuccess;
  decode_kernel<KWIN, SLOTW, G><<<static_cast<unsigned>(grid), kThreads * G, smem, s>>>(args);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_decode(const LaunchArgs& args, int variant, cudaStream_t stream) {
  // Three 256-thread groups per CTA keep <= 85 registers (no spills) at 24
  // warps/SM.
  switch (variant) {  // ids of variant_for() in decode.cuh
    case 0: return launch_k<1, 8, 3>(args, stream);
    case 1: return launch_k<2, 16, 3>(args, stream);
    case 2: return launch_k<4, 16, 3>(args, stream);
    case 3: return launch_k<4, 32, 2>(args, stream);
    case 4: return launch_decode_warp(args, stream);
    case 5: return launch_decode_warp_wide(args, stream);
    case 6: return launch_decode_fsm64(args, stream);
    case 7: return launch_decode_warp_direct(args, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_count_window(const std::uint8_t* d_window16, unsigned gap, const TensorDesc& d,
                                std::uint32_t* d_count, cudaStream_t stream) {
  count_window_kernel<<<1, 128, 0, stream>>>(d_window16, gap, d, d_count);
  return cudaGetLastError();
}

}  // namespace ecf8::dev
