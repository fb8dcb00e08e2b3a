// e5_decode.cu -- B200 decoder of the native E5M2 variant (include/ecf8_e5m2.h,
// SURVEY §8(f) row 3).
//
// The variant's stream is the reference's (64-bit windows, gaps, outpos,
// codec.cpp:49-98) over a 32-symbol code, so the decode follows the
// reference's block structure (codec.cpp:201-253) with one thread per window:
//
//   count   each thread walks its window: the code words that start in
//           [gap, 64), one 10-bit table probe per word (longer words: the
//           canonical first-code / count tables; no match: the lowest
//           present symbol with its own length);
//   scan    CTA-wide exclusive scan of the counts, segmented by reference
//           block (T threads each), clamped to the block's outpos range;
//   emit    the walk again, each symbol stored as one byte at its final
//           place in the CTA's staging tile in shared memory;
//   write   16 output bytes per thread-step: 16 exponent bytes + the 16
//           elements' sign / mantissa bits from the three raw bit planes
//           (one multiply spreads 4 plane bits to 4 bytes), coalesced
//           128-bit stores; the tile's ragged first / last chunk byte-wise.
//
// A CTA owns NT = max(256, T) consecutive windows (NT / T whole blocks) and
// loops over tiles; its staging tile holds NT * 64 symbols (a window holds at
// most 64).  Walking twice trades decode work for staging space: the variant
// is a secondary format, integer-bound, and memory-light (3 raw bits per
// element instead of 4).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ecf8_cuda.h"
#include "ecf8_e5m2.h"

extern "C" int ecf8_internal_set_error(int status, const char* msg);
extern "C" int ecf8_internal_require_device(void);

namespace ecf8::dev::e5 {

// Write-back chunks per lane unrolled: their raw-plane loads (L2) in flight together.
#ifndef ECF8_E5_WB_UNROLL
#define ECF8_E5_WB_UNROLL 1
#endif
constexpr int kE5WbUnroll = ECF8_E5_WB_UNROLL;

constexpr int kSyms = 32;
constexpr int kFastBits = 10;
constexpr std::uint64_t kPad = 64;

// Decode tables (built on the host from the code lengths).
struct Tables {
  std::uint16_t fast[1 << kFastBits];  // sym | len << 8 for a word of <= 10 bits at the index; 0: look further
  std::uint16_t base[17];              // first canonical code value of each length
  std::uint16_t count[17];             // words of each length
  std::uint8_t offset[17];             // index of the length's first symbol in syms[]
  std::uint8_t syms[kSyms];            // symbols in (length, symbol) order
  std::uint8_t fb_sym, fb_len;         // no word matches: lowest present symbol, its length
};

struct Desc {
  const std::uint8_t* encoded;
  const std::uint8_t* gaps;
  const std::uint64_t* outpos;
  const std::uint32_t* raw;  // 3 u32 per 32 elements
  const Tables* tables;
  std::uint8_t* out;
  std::uint64_t n_elem, n_blocks, n_windows;
  std::uint32_t T;
  std::uint32_t lmin;                // shortest code length
  const std::uint32_t* lane_start;   // per 8-window lane: its two 4-window groups' offsets in their block (u16 each)
  const uint2* fsm;                  // byte-step table (32 states x 256); set when every tile passed the upload check
};

__device__ __forceinline__ std::uint64_t be64(const std::uint8_t* p) {
  const uint2 v = *reinterpret_cast<const uint2*>(p);  // 8-byte aligned: windows start at 8 w
  return (static_cast<std::uint64_t>(__byte_perm(v.x, 0, 0x0123)) << 32) | __byte_perm(v.y, 0, 0x0123);
}

// One code word at bit p (< 64) of the window (hi:lo = its 128 bits).
__device__ __forceinline__ void word_at(const Tables& tb, std::uint64_t hi, std::uint64_t lo, std::uint32_t p,
                                        std::uint32_t& sym, std::uint32_t& len) {
  const std::uint32_t w16 = static_cast<std::uint32_t>((p ? (hi << p) | (lo >> (64 - p)) : hi) >> 48);
  const std::uint32_t e = tb.fast[w16 >> (16 - kFastBits)];
  if (e >> 8) {
    sym = e & 0xFFu;
    len = e >> 8;
    return;
  }
  for (std::uint32_t l = kFastBits + 1; l <= 16; ++l) {
    const std::uint32_t c = w16 >> (16 - l);
    if (c >= tb.base[l] && c - tb.base[l] < tb.count[l]) {
      sym = tb.syms[tb.offset[l] + (c - tb.base[l])];
      len = l;
      return;
    }
  }
  sym = tb.fb_sym;
  len = tb.fb_len;
}

__device__ __forceinline__ std::uint32_t spread4(std::uint32_t b) {  // bit k of b -> bit 8k
  return (b * 0x00204081u) & 0x01010101u;
}

template <int NT>
__global__ void __launch_bounds__(NT) e5_decode_kernel(const Desc d) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Tables tb;
  __shared__ std::uint32_t excl_s[NT];
  __shared__ std::uint32_t warp_sum[NT / 32];
  std::uint8_t* const stage = smem;  // NT * 64 + 32 bytes
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < static_cast<int>(sizeof(Tables) / 2); i += NT)
    reinterpret_cast<std::uint16_t*>(&tb)[i] = reinterpret_cast<const std::uint16_t*>(d.tables)[i];
  __syncthreads();

  const std::uint32_t T = d.T;
  const std::uint64_t n_tiles = (d.n_windows + NT - 1) / NT;
  for (std::uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const std::uint64_t w = tile * NT + tid;
    const bool active = w < d.n_windows;
    std::uint64_t hi = 0, lo = 0;
    std::uint32_t gap = 0, cnt = 0;
    if (active) {
      hi = be64(d.encoded + 8 * w);
      lo = be64(d.encoded + 8 * w + 8);  // the next window's bytes (padding past the last)
      gap = (d.gaps[w >> 1] >> ((w & 1) ? 0 : 4)) & 15u;
      for (std::uint32_t p = gap; p < 64;) {  // count_phase (codec.cpp:133-161)
        std::uint32_t s, l;
        word_at(tb, hi, lo, p, s, l);
        p += l;
        ++cnt;
      }
    }
    // CTA-wide exclusive scan of the counts
    std::uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      std::uint32_t v = lane < NT / 32 ? warp_sum[lane] : 0u, x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane < NT / 32) warp_sum[lane] = x - v;
    }
    __syncthreads();
    const std::uint32_t excl = warp_sum[warp] + incl - cnt;
    excl_s[tid] = excl;
    __syncthreads();
    // the tile's blocks and output range [A, E)
    const std::uint64_t b0 = tile * NT / T;
    const std::uint64_t nb = std::min<std::uint64_t>(NT / T, d.n_blocks - b0);
    const std::uint64_t A = d.outpos[b0], E = d.outpos[b0 + nb];
    const std::uint32_t off = static_cast<std::uint32_t>(A & 15);
    if (active) {  // emit_phase with the block clamp (codec.cpp:168-190, 239-251)
      const std::uint64_t b = w / T;
      const std::uint32_t first = static_cast<std::uint32_t>(tid) & ~(T - 1);
      const std::uint64_t o_start = d.outpos[b] + (excl - excl_s[first]), lim = d.outpos[b + 1];
      if (o_start < lim) {
        const std::uint32_t keep = static_cast<std::uint32_t>(std::min<std::uint64_t>(cnt, lim - o_start));
        std::uint8_t* dst = stage + (o_start - A) + off;
        std::uint32_t p = gap;
        for (std::uint32_t k = 0; k < keep; ++k) {
          std::uint32_t s, l;
          word_at(tb, hi, lo, p, s, l);
          p += l;
          dst[k] = static_cast<std::uint8_t>(s);
        }
      }
    }
    __syncthreads();
    // write-out: element S0 + i from stage[i] and the raw bit planes
    const std::uint64_t S0 = A - off;
    const std::uint32_t data_end = off + static_cast<std::uint32_t>(E - A);
    const std::uint32_t nch = (data_end + 15) >> 4;
    for (std::uint32_t c = tid; c < nch; c += NT) {
      const std::uint32_t i0 = 16 * c;
      const std::uint64_t g0 = S0 + i0;
      const std::uint32_t* rp = d.raw + 3 * (g0 >> 5);
      const std::uint32_t sh = static_cast<std::uint32_t>(g0 & 16);
      const std::uint32_t sg = __ldg(rp) >> sh, m1 = __ldg(rp + 1) >> sh, m0 = __ldg(rp + 2) >> sh;
      if (i0 >= off && i0 + 16 <= data_end) {
        const uint4 x = *reinterpret_cast<const uint4*>(stage + i0);
        const std::uint32_t xs[4] = {x.x, x.y, x.z, x.w};
        std::uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          o[q] = (xs[q] << 2) | (spread4((sg >> (4 * q)) & 15u) << 7) | (spread4((m1 >> (4 * q)) & 15u) << 1) |
                 spread4((m0 >> (4 * q)) & 15u);
        asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(d.out + g0), "r"(o[0]), "r"(o[1]), "r"(o[2]),
                     "r"(o[3]));
      } else {
        for (std::uint32_t j = 0; j < 16; ++j) {
          const std::uint32_t i = i0 + j;
          if (i < off || i >= data_end) continue;
          d.out[g0 + j] = static_cast<std::uint8_t>((stage[i] << 2) | (((sg >> j) & 1u) << 7) |
                                                    (((m1 >> j) & 1u) << 1) | ((m0 >> j) & 1u));
        }
      }
    }
    __syncthreads();  // the stage and excl_s are reused by the next tile
  }
}

// ---- byte-step path (every tile of the tensor passed the upload check)
//
// As the E4M3 kernel (decode_warp.cuh, direct tiles): a warp decodes a tile
// of 256 windows, 8 per lane as two 4-window chains, one table probe per
// input byte of a finite-state machine over the 32-symbol code tree (state =
// pending prefix, < 32; entry = the byte's completed words: low exponent
// nibbles in .x, 4 * count | state << 8 | high exponent bits << 16 in .y).
// Runs start at the upload check's group offsets and end at the next run's
// start (or the block end, clamped to outpos); the low nibbles go to a nibble
// staging tile, the high bits to a bit plane, both placed directly.

struct Sink4 {  // nibbles, 8 per 32-bit word
  std::uint32_t addr, lo = 0, q4 = 0;  // q4: bits 0..4 exact, bit 5 toggles per filled word
};
struct Sink1 {  // bits, 32 per word
  std::uint32_t addr, lo = 0, q = 0;   // q < 32
};

__device__ __forceinline__ void sts(std::uint32_t a, std::uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

template <bool BOUNDED>
__device__ __forceinline__ void put(Sink4& k, Sink1& b, uint2 e, std::uint32_t ew4, std::uint32_t ew1,
                                    std::uint32_t& t4, std::uint32_t& t1) {
  {  // low nibbles (up to 8)
    const std::uint32_t q = k.q4 + e.y;
    const std::uint32_t nl = k.lo | __funnelshift_l(0u, e.x, k.q4);
    const std::uint32_t nh = __funnelshift_l(e.x, 0u, k.q4);
    const bool full = ((q ^ k.q4) & 32u) != 0;
    if (full && (!BOUNDED || k.addr < ew4)) sts(k.addr, nl);
    if (BOUNDED && full && k.addr == ew4) t4 = nl;
    k.addr += full ? 4u : 0u;
    k.lo = full ? nh : nl;
    k.q4 = q;
  }
  {  // high bits (one per word)
    const std::uint32_t hb = (e.y >> 16) & 0xFFu, n = (e.y & 63u) >> 2;
    const std::uint32_t nl = b.lo | (hb << b.q);
    const std::uint32_t nh = __funnelshift_l(hb, 0u, b.q);
    const std::uint32_t q = b.q + n;
    const bool full = q >= 32;
    if (full && (!BOUNDED || b.addr < ew1)) sts(b.addr, nl);
    if (BOUNDED && full && b.addr == ew1) t1 = nl;
    b.addr += full ? 4u : 0u;
    b.lo = full ? nh : nl;
    b.q = full ? q - 32 : q;
  }
}

__device__ __forceinline__ std::uint32_t prmt(std::uint32_t a, std::uint32_t b, std::uint32_t sel) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ uint2 probe(std::uint32_t tab, std::uint32_t word, std::uint32_t prev_y, int j) {
  // index = state * 256 + byte j of the stream (state: byte 1 of the previous entry's .y)
  const std::uint32_t idx = prmt(word, prev_y, 0xDD50u | static_cast<std::uint32_t>(3 - (j & 3)));
  std::uint32_t a;
  uint2 v;
  asm("mad.lo.u32 %0, %1, 8, %2;" : "=r"(a) : "r"(idx), "r"(tab));
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

// Two 4-window chains of a lane, interleaved (two probe chains in flight).
__device__ __forceinline__ void decode_chains(const std::uint32_t (&w)[18], std::uint32_t ga, std::uint32_t gb,
                                              std::uint32_t tab, Sink4& a4, Sink1& a1, std::uint32_t ea, Sink4& b4,
                                              Sink1& b1, std::uint32_t eb, std::uint32_t st4, std::uint32_t st1,
                                              std::uint32_t (&tails)[4]) {
  std::uint32_t sa[9], sb[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    sa[i] = __funnelshift_l(w[i + 1], w[i], ga);
    sb[i] = __funnelshift_l(w[i + 9], w[i + 8], gb);
  }
  const std::uint32_t ea4 = st4 + 4 * (ea >> 3), ea1 = st1 + 4 * (ea >> 5);
  const std::uint32_t eb4 = st4 + 4 * (eb >> 3), eb1 = st1 + 4 * (eb >> 5);
  std::uint32_t ya = 0, yb = 0, ta4 = 0, ta1 = 0, tb4 = 0, tb1 = 0;
#pragma unroll
  for (int j = 0; j < 30; ++j) {  // every word these bytes complete belongs to the run
    const uint2 x = probe(tab, sa[j >> 2], ya, j);
    const uint2 y = probe(tab, sb[j >> 2], yb, j);
    put<false>(a4, a1, x, 0, 0, ta4, ta1);
    put<false>(b4, b1, y, 0, 0, tb4, tb1);
    ya = x.y;
    yb = y.y;
  }
#pragma unroll
  for (int j = 30; j < 34; ++j) {  // the run's end falls in these bytes: later words dropped by position
    const uint2 x = probe(tab, sa[j >> 2], ya, j);
    const uint2 y = probe(tab, sb[j >> 2], yb, j);
    put<true>(a4, a1, x, ea4, ea1, ta4, ta1);
    put<true>(b4, b1, y, eb4, eb1, tb4, tb1);
    ya = x.y;
    yb = y.y;
  }
  if (a4.addr == ea4) ta4 = a4.lo;
  if (a1.addr == ea1) ta1 = a1.lo;
  if (b4.addr == eb4) tb4 = b4.lo;
  if (b1.addr == eb1) tb1 = b1.lo;
  tails[0] = ta4 & ((1u << (4 * (ea & 7))) - 1);
  tails[1] = ta1 & ((ea & 31) ? (1u << (ea & 31)) - 1 : 0u);
  tails[2] = tb4 & ((1u << (4 * (eb & 7))) - 1);
  tails[3] = tb1 & ((eb & 31) ? (1u << (eb & 31)) - 1 : 0u);
}

// Bytes [lo, hi) (0 <= lo < hi <= 16) of a 16-byte output chunk at a
// 16-byte aligned dst: whole words as word stores, the rest byte-wise.
__device__ __forceinline__ void store_partial16(std::uint8_t* dst, const std::uint32_t (&o)[4], std::uint32_t lo,
                                                std::uint32_t hi) {
#pragma unroll
  for (std::uint32_t q = 0; q < 4; ++q) {
    const std::uint32_t a = 4 * q;
    if (a >= lo && a + 4 <= hi) {
      *reinterpret_cast<std::uint32_t*>(dst + a) = o[q];
    } else if (a + 4 > lo && a < hi) {
#pragma unroll
      for (std::uint32_t b = 0; b < 4; ++b)
        if (a + b >= lo && a + b < hi) dst[a + b] = static_cast<std::uint8_t>(o[q] >> (8 * b));
    }
  }
}

__device__ __forceinline__ std::uint32_t bswap(std::uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// 4 nibbles (bits 4j..4j+3 of x, j < 4) -> 4 bytes
__device__ __forceinline__ std::uint32_t nib_bytes(std::uint32_t x) {
  const std::uint32_t t = ((x & 0xFF00u) << 8) | (x & 0xFFu);
  return (t | (t << 4)) & 0x0F0F0F0Fu;
}

template <int NW, bool WIDE>
__global__ void __launch_bounds__(NW * 32, 1) e5_fsm_kernel(const Desc d) {
  asm volatile("griddepcontrol.launch_dependents;");  // the next decode may take SMs as ours free up
  // per warp: the nibble tile (WIDE: 64 symbols per window) and the bit plane
  constexpr std::uint32_t kSym = WIDE ? 16384 : 8192;
  constexpr std::uint32_t kW4 = kSym / 8 + 8, kW1 = kSym / 32 + 8;  // words (+ alignment and tail slack)
  extern __shared__ __align__(16) unsigned char smem_raw[];  // [table 64 KB][per warp: nibble tile, bit plane]
  uint2* const tab_s = reinterpret_cast<uint2*>(smem_raw);
  __shared__ unsigned next_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint32_t* const w4 = reinterpret_cast<std::uint32_t*>(smem_raw + 8 * 32 * 256) + warp * (kW4 + kW1);
  std::uint32_t* const w1 = w4 + kW4;
  for (int i = threadIdx.x; i < 32 * 256 / 2; i += NW * 32)
    reinterpret_cast<uint4*>(tab_s)[i] = __ldg(reinterpret_cast<const uint4*>(d.fsm) + i);
  if (threadIdx.x == 0) next_tile = NW;
  __syncthreads();
  const std::uint32_t tab = static_cast<std::uint32_t>(__cvta_generic_to_shared(tab_s));
  const std::uint32_t st4 = static_cast<std::uint32_t>(__cvta_generic_to_shared(w4));
  const std::uint32_t st1 = static_cast<std::uint32_t>(__cvta_generic_to_shared(w1));
  const std::uint32_t T = d.T, log2T = 31 - __clz(T), m = 256u >> log2T;
  const std::uint64_t n_tiles = (d.n_blocks + m - 1) / m;
  const std::uint64_t t_lo = n_tiles * blockIdx.x / gridDim.x, t_hi = n_tiles * (blockIdx.x + 1) / gridDim.x;
  // a tile's input sections -> L2 (lanes 0-3; the next tile's, one tile ahead)
  auto prefetch = [&](std::uint64_t t) {
    const std::uint64_t pb0 = t * m, pnb = min(static_cast<std::uint64_t>(m), d.n_blocks - pb0);
    const std::uint64_t pw0 = pb0 << log2T, pnw = pnb << log2T;
    const std::uint8_t* p = d.encoded + 8 * pw0;
    std::uint64_t n = 8 * pnw + 8;
    p = lane == 1 ? d.gaps + (pw0 >> 1) : p;
    p = lane == 2 ? reinterpret_cast<const std::uint8_t*>(d.lane_start + (pw0 >> 3)) : p;
    p = lane == 3 ? reinterpret_cast<const std::uint8_t*>(d.outpos + pb0) : p;
    n = lane == 1 ? pnw >> 1 : lane == 2 ? pnw >> 1 : lane == 3 ? 8 * (pnb + 1) : n;
    const std::uint64_t a = reinterpret_cast<std::uint64_t>(p) & ~std::uint64_t{15};
    const std::uint32_t bytes = static_cast<std::uint32_t>((reinterpret_cast<std::uint64_t>(p) + n - a + 15) & ~std::uint64_t{15});
    if (lane < 4 && n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
  };
  std::uint64_t tile = t_lo + warp;
  if (tile < t_hi) prefetch(tile);
  while (tile < t_hi) {
    unsigned claim = 0;
    if (lane == 0) claim = atomicAdd(&next_tile, 1u);
    const std::uint64_t next = t_lo + __shfl_sync(0xffffffffu, claim, 0);
    if (next < t_hi) prefetch(next);
    const std::uint64_t b0 = tile * m;
    const std::uint32_t nblk = static_cast<std::uint32_t>(min(static_cast<std::uint64_t>(m), d.n_blocks - b0));
    const std::uint32_t nwin = nblk << log2T, wl = static_cast<std::uint32_t>(lane) * 8;
    const std::uint64_t w0 = b0 << log2T;
    const bool active = wl < nwin;
    const std::uint64_t A = __ldg(d.outpos + b0), E = __ldg(d.outpos + b0 + nblk);
    const std::uint32_t bl = min(wl >> log2T, nblk - 1);
    const std::uint64_t o0 = __ldg(d.outpos + b0 + bl), o1 = __ldg(d.outpos + b0 + bl + 1);
    if (lane == 0) {  // the tile's raw plane words -> L2 (read at write-back)
      const std::uint64_t r0 = 12 * (A >> 5), r1 = 12 * ((E >> 5) + 1);
      const std::uint64_t a = reinterpret_cast<std::uint64_t>(d.raw) + r0;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a & ~std::uint64_t{15}),
                   "r"(static_cast<std::uint32_t>(((r1 - r0) + (a & 15) + 15) & ~std::uint64_t{15}))
                   : "memory");
    }
    std::uint32_t w[18] = {};
    std::uint32_t gaps = 0, ls = 0;
    if (active) {
      const uint4* src = reinterpret_cast<const uint4*>(d.encoded + 8 * (w0 + wl));
      const uint4 q0 = __ldg(src), q1 = __ldg(src + 1), q2 = __ldg(src + 2), q3 = __ldg(src + 3);
      const uint2 q4 = __ldg(reinterpret_cast<const uint2*>(src + 4));
      w[0] = bswap(q0.x), w[1] = bswap(q0.y), w[2] = bswap(q0.z), w[3] = bswap(q0.w);
      w[4] = bswap(q1.x), w[5] = bswap(q1.y), w[6] = bswap(q1.z), w[7] = bswap(q1.w);
      w[8] = bswap(q2.x), w[9] = bswap(q2.y), w[10] = bswap(q2.z), w[11] = bswap(q2.w);
      w[12] = bswap(q3.x), w[13] = bswap(q3.y), w[14] = bswap(q3.z), w[15] = bswap(q3.w);
      w[16] = bswap(q4.x), w[17] = bswap(q4.y);
      gaps = __ldg(reinterpret_cast<const std::uint32_t*>(d.gaps + ((w0 + wl) >> 1)));
      ls = __ldg(d.lane_start + ((w0 + wl) >> 3));
    }
    const std::uint32_t off = static_cast<std::uint32_t>(A & 15);
    const std::uint32_t data_end = off + static_cast<std::uint32_t>(E - A);
    const std::uint64_t S0 = A - off;
    const std::uint32_t base = static_cast<std::uint32_t>(o0 - A) + off, blk_end = static_cast<std::uint32_t>(o1 - A) + off;
    const std::uint32_t da = base + (ls & 0xFFFFu), db = base + (ls >> 16);
    const std::uint32_t next_da = __shfl_down_sync(0xffffffffu, da, 1);
    const std::uint32_t nl = static_cast<std::uint32_t>(lane) + 1;
    const bool next_same = nl < 32 && (nl & ((T >> 3) - 1)) != 0 && nl * 8 < nwin;
    const std::uint32_t ea = max(min(max(db, da), blk_end), min(da, blk_end));
    const std::uint32_t eb = max(min(max(next_same ? next_da : blk_end, db), blk_end), min(db, blk_end));
    __syncwarp();  // the previous tile's write-back is done with the tiles
    if (active) {  // only the runs' end words need zeroes (every other word is filled by one run)
      sts(st4 + 4 * (ea >> 3), 0u);
      sts(st4 + 4 * (eb >> 3), 0u);
      sts(st1 + 4 * (ea >> 5), 0u);
      sts(st1 + 4 * (eb >> 5), 0u);
    }
    __syncwarp();
    std::uint32_t tails[4] = {0, 0, 0, 0};
    if (active) {
      Sink4 a4{st4 + 4 * (da >> 3)}, b4{st4 + 4 * (db >> 3)};
      Sink1 a1{st1 + 4 * (da >> 5)}, b1{st1 + 4 * (db >> 5)};
      a4.q4 = 4 * (da & 7);
      b4.q4 = 4 * (db & 7);
      a1.q = da & 31;
      b1.q = db & 31;
      decode_chains(w, (gaps >> 4) & 15u, (gaps >> 20) & 15u, tab, a4, a1, ea, b4, b1, eb, st4, st1, tails);
    }
    __syncwarp();  // every run's plain stores are in place
    if (tails[0]) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(st4 + 4 * (ea >> 3)), "r"(tails[0]) : "memory");
    if (tails[1]) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(st1 + 4 * (ea >> 5)), "r"(tails[1]) : "memory");
    if (tails[2]) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(st4 + 4 * (eb >> 3)), "r"(tails[2]) : "memory");
    if (tails[3]) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(st1 + 4 * (eb >> 5)), "r"(tails[3]) : "memory");
    __syncwarp();
    // write-back: 16 elements per lane-step from the nibble tile, the bit
    // plane and the raw planes; 128-bit stores, the ragged edges byte-wise
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous grid (PDL) is done writing
    const std::uint32_t nch = (data_end + 15) >> 4;
#pragma unroll kE5WbUnroll
    for (std::uint32_t c = static_cast<std::uint32_t>(lane); c < nch; c += 32) {
      const uint2 nib = reinterpret_cast<const uint2*>(w4)[c];
      const std::uint32_t hb = (w1[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
      const std::uint64_t e = S0 + 16 * static_cast<std::uint64_t>(c);
      const std::uint32_t* rp = d.raw + 3 * (e >> 5);
      const std::uint32_t sh = static_cast<std::uint32_t>(e & 16);
      const std::uint32_t sg = __ldg(rp) >> sh, m1 = __ldg(rp + 1) >> sh, m0 = __ldg(rp + 2) >> sh;
      std::uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const std::uint32_t x = (q < 2 ? nib.x : nib.y) >> (16 * (q & 1));
        const std::uint32_t ex = nib_bytes(x) | (spread4((hb >> (4 * q)) & 15u) << 4);
        o[q] = (ex << 2) | (spread4((sg >> (4 * q)) & 15u) << 7) | (spread4((m1 >> (4 * q)) & 15u) << 1) |
               spread4((m0 >> (4 * q)) & 15u);
      }
      const std::uint32_t i0 = 16 * c;
      if (i0 >= off && i0 + 16 <= data_end) {
        asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(d.out + e), "r"(o[0]), "r"(o[1]), "r"(o[2]),
                     "r"(o[3]));
      } else {  // a ragged edge chunk: bytes [lo, hi) of it
        store_partial16(d.out + e, o, i0 < off ? off - i0 : 0u, min(16u, data_end - i0));
      }
    }
    tile = next;
  }
}

// Codes whose words are all >= 2 bits complete at most 4 words per byte: the
// symbols then fit one 32-bit entry word as bytes (.x = symbol bytes, first
// lowest; .y = 8 * count | state << 8), and the lanes append whole symbol
// bytes to a byte staging tile -- one sink instead of nibbles + a bit plane,
// and a write-back without nibble / bit spreading.
struct SinkB {
  std::uint32_t addr, lo = 0, q = 0;  // q: bits 0..4 exact (a multiple of 8), bit 5 toggles per filled word
};

template <bool BOUNDED>
__device__ __forceinline__ void putb(SinkB& k, uint2 e, std::uint32_t ew, std::uint32_t& tail) {
  const std::uint32_t q = k.q + e.y;
  const std::uint32_t nl = k.lo | __funnelshift_l(0u, e.x, k.q);
  const std::uint32_t nh = __funnelshift_l(e.x, 0u, k.q);
  const bool full = ((q ^ k.q) & 32u) != 0;
  if (full && (!BOUNDED || k.addr < ew)) sts(k.addr, nl);
  if (BOUNDED && full && k.addr == ew) tail = nl;
  k.addr += full ? 4u : 0u;
  k.lo = full ? nh : nl;
  k.q = q;
}

__device__ __forceinline__ void decode_chains_b(const std::uint32_t (&w)[18], std::uint32_t ga, std::uint32_t gb,
                                                std::uint32_t tab, SinkB& a, std::uint32_t ea, SinkB& b,
                                                std::uint32_t eb, std::uint32_t st, std::uint32_t& ta,
                                                std::uint32_t& tb) {
  std::uint32_t sa[9], sb[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    sa[i] = __funnelshift_l(w[i + 1], w[i], ga);
    sb[i] = __funnelshift_l(w[i + 9], w[i + 8], gb);
  }
  const std::uint32_t ewa = st + (ea & ~3u), ewb = st + (eb & ~3u);
  std::uint32_t ya = 0, yb = 0;
  ta = tb = 0;
#pragma unroll
  for (int j = 0; j < 30; ++j) {
    const uint2 x = probe(tab, sa[j >> 2], ya, j);
    const uint2 y = probe(tab, sb[j >> 2], yb, j);
    putb<false>(a, x, 0, ta);
    putb<false>(b, y, 0, tb);
    ya = x.y;
    yb = y.y;
  }
#pragma unroll
  for (int j = 30; j < 34; ++j) {
    const uint2 x = probe(tab, sa[j >> 2], ya, j);
    const uint2 y = probe(tab, sb[j >> 2], yb, j);
    putb<true>(a, x, ewa, ta);
    putb<true>(b, y, ewb, tb);
    ya = x.y;
    yb = y.y;
  }
  if (a.addr == ewa) ta = a.lo;
  if (b.addr == ewb) tb = b.lo;
  ta &= (ea & 3) ? (1u << (8 * (ea & 3))) - 1 : 0u;
  tb &= (eb & 3) ? (1u << (8 * (eb & 3))) - 1 : 0u;
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) e5_fsm_bytes_kernel(const Desc d) {
  asm volatile("griddepcontrol.launch_dependents;");  // the next decode may take SMs as ours free up
  constexpr std::uint32_t kBytes = 8192 + 32;  // a warp tile's symbols (<= 32 per window) + alignment / tail slack
  extern __shared__ __align__(16) unsigned char smem_raw[];  // [table 64 KB][per warp: symbol bytes]
  uint2* const tab_s = reinterpret_cast<uint2*>(smem_raw);
  __shared__ unsigned next_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint8_t* const sb_ = smem_raw + 8 * 32 * 256 + warp * kBytes;
  for (int i = threadIdx.x; i < 32 * 256 / 2; i += NW * 32)
    reinterpret_cast<uint4*>(tab_s)[i] = __ldg(reinterpret_cast<const uint4*>(d.fsm) + i);
  if (threadIdx.x == 0) next_tile = NW;
  __syncthreads();
  const std::uint32_t tab = static_cast<std::uint32_t>(__cvta_generic_to_shared(tab_s));
  const std::uint32_t st = static_cast<std::uint32_t>(__cvta_generic_to_shared(sb_));
  const std::uint32_t T = d.T, log2T = 31 - __clz(T), m = 256u >> log2T;
  const std::uint64_t n_tiles = (d.n_blocks + m - 1) / m;
  const std::uint64_t t_lo = n_tiles * blockIdx.x / gridDim.x, t_hi = n_tiles * (blockIdx.x + 1) / gridDim.x;
  auto prefetch = [&](std::uint64_t t) {
    const std::uint64_t pb0 = t * m, pnb = min(static_cast<std::uint64_t>(m), d.n_blocks - pb0);
    const std::uint64_t pw0 = pb0 << log2T, pnw = pnb << log2T;
    const std::uint8_t* p = d.encoded + 8 * pw0;
    std::uint64_t n = 8 * pnw + 8;
    p = lane == 1 ? d.gaps + (pw0 >> 1) : p;
    p = lane == 2 ? reinterpret_cast<const std::uint8_t*>(d.lane_start + (pw0 >> 3)) : p;
    p = lane == 3 ? reinterpret_cast<const std::uint8_t*>(d.outpos + pb0) : p;
    n = lane == 1 ? pnw >> 1 : lane == 2 ? pnw >> 1 : lane == 3 ? 8 * (pnb + 1) : n;
    const std::uint64_t a = reinterpret_cast<std::uint64_t>(p) & ~std::uint64_t{15};
    const std::uint32_t bytes = static_cast<std::uint32_t>((reinterpret_cast<std::uint64_t>(p) + n - a + 15) & ~std::uint64_t{15});
    if (lane < 4 && n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
  };
  std::uint64_t tile = t_lo + warp;
  if (tile < t_hi) prefetch(tile);
  while (tile < t_hi) {
    unsigned claim = 0;
    if (lane == 0) claim = atomicAdd(&next_tile, 1u);
    const std::uint64_t next = t_lo + __shfl_sync(0xffffffffu, claim, 0);
    if (next < t_hi) prefetch(next);
    const std::uint64_t b0 = tile * m;
    const std::uint32_t nblk = static_cast<std::uint32_t>(min(static_cast<std::uint64_t>(m), d.n_blocks - b0));
    const std::uint32_t nwin = nblk << log2T, wl = static_cast<std::uint32_t>(lane) * 8;
    const std::uint64_t w0 = b0 << log2T;
    const bool active = wl < nwin;
    const std::uint64_t A = __ldg(d.outpos + b0), E = __ldg(d.outpos + b0 + nblk);
    const std::uint32_t bl = min(wl >> log2T, nblk - 1);
    const std::uint64_t o0 = __ldg(d.outpos + b0 + bl), o1 = __ldg(d.outpos + b0 + bl + 1);
    if (lane == 0) {  // the tile's raw plane words -> L2 (read at write-back)
      const std::uint64_t r0 = 12 * (A >> 5), r1 = 12 * ((E >> 5) + 1);
      const std::uint64_t a = reinterpret_cast<std::uint64_t>(d.raw) + r0;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a & ~std::uint64_t{15}),
                   "r"(static_cast<std::uint32_t>(((r1 - r0) + (a & 15) + 15) & ~std::uint64_t{15}))
                   : "memory");
    }
    std::uint32_t w[18] = {};
    std::uint32_t gaps = 0, ls = 0;
    if (active) {
      const uint4* src = reinterpret_cast<const uint4*>(d.encoded + 8 * (w0 + wl));
      const uint4 q0 = __ldg(src), q1 = __ldg(src + 1), q2 = __ldg(src + 2), q3 = __ldg(src + 3);
      const uint2 q4 = __ldg(reinterpret_cast<const uint2*>(src + 4));
      w[0] = bswap(q0.x), w[1] = bswap(q0.y), w[2] = bswap(q0.z), w[3] = bswap(q0.w);
      w[4] = bswap(q1.x), w[5] = bswap(q1.y), w[6] = bswap(q1.z), w[7] = bswap(q1.w);
      w[8] = bswap(q2.x), w[9] = bswap(q2.y), w[10] = bswap(q2.z), w[11] = bswap(q2.w);
      w[12] = bswap(q3.x), w[13] = bswap(q3.y), w[14] = bswap(q3.z), w[15] = bswap(q3.w);
      w[16] = bswap(q4.x), w[17] = bswap(q4.y);
      gaps = __ldg(reinterpret_cast<const std::uint32_t*>(d.gaps + ((w0 + wl) >> 1)));
      ls = __ldg(d.lane_start + ((w0 + wl) >> 3));
    }
    const std::uint32_t off = static_cast<std::uint32_t>(A & 15);
    const std::uint32_t data_end = off + static_cast<std::uint32_t>(E - A);
    const std::uint64_t S0 = A - off;
    const std::uint32_t base = static_cast<std::uint32_t>(o0 - A) + off, blk_end = static_cast<std::uint32_t>(o1 - A) + off;
    const std::uint32_t da = base + (ls & 0xFFFFu), db = base + (ls >> 16);
    const std::uint32_t next_da = __shfl_down_sync(0xffffffffu, da, 1);
    const std::uint32_t nl = static_cast<std::uint32_t>(lane) + 1;
    const bool next_same = nl < 32 && (nl & ((T >> 3) - 1)) != 0 && nl * 8 < nwin;
    const std::uint32_t ea = max(min(max(db, da), blk_end), min(da, blk_end));
    const std::uint32_t eb = max(min(max(next_same ? next_da : blk_end, db), blk_end), min(db, blk_end));
    __syncwarp();  // the previous tile's write-back is done with the staging bytes
    if (active) {  // only the runs' end words need zeroes
      sts(st + (ea & ~3u), 0u);
      sts(st + (eb & ~3u), 0u);
    }
    __syncwarp();
    std::uint32_t ta = 0, tb = 0;
    if (active) {
      SinkB a{st + (da & ~3u)}, b{st + (db & ~3u)};
      a.q = 8 * (da & 3);
      b.q = 8 * (db & 3);
      decode_chains_b(w, (gaps >> 4) & 15u, (gaps >> 20) & 15u, tab, a, ea, b, eb, st, ta, tb);
    }
    __syncwarp();
    if (ta) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(st + (ea & ~3u)), "r"(ta) : "memory");
    if (tb) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(st + (eb & ~3u)), "r"(tb) : "memory");
    __syncwarp();
    // write-back: 16 symbol bytes + the raw planes' 16 bits each per lane-step
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous grid (PDL) is done writing
    const std::uint32_t nch = (data_end + 15) >> 4;
#pragma unroll kE5WbUnroll
    for (std::uint32_t c = static_cast<std::uint32_t>(lane); c < nch; c += 32) {
      const uint4 ex = reinterpret_cast<const uint4*>(sb_)[c];
      const std::uint64_t e = S0 + 16 * static_cast<std::uint64_t>(c);
      const std::uint32_t* rp = d.raw + 3 * (e >> 5);
      const std::uint32_t sh = static_cast<std::uint32_t>(e & 16);
      const std::uint32_t sg = __ldg(rp) >> sh, m1 = __ldg(rp + 1) >> sh, m0 = __ldg(rp + 2) >> sh;
      const std::uint32_t xs[4] = {ex.x, ex.y, ex.z, ex.w};
      std::uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // bit k of a 4-bit group -> bit 8k + 7 / 8k + 1 / 8k (one multiply each)
        const std::uint32_t s7 = (((sg >> (4 * q)) & 15u) * 0x10204080u) & 0x80808080u;
        const std::uint32_t m1b = (((m1 >> (4 * q)) & 15u) * 0x00408102u) & 0x02020202u;
        const std::uint32_t m0b = (((m0 >> (4 * q)) & 15u) * 0x00204081u) & 0x01010101u;
        o[q] = (xs[q] << 2) | s7 | m1b | m0b;
      }
      const std::uint32_t i0 = 16 * c;
      if (i0 >= off && i0 + 16 <= data_end) {
        asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(d.out + e), "r"(o[0]), "r"(o[1]), "r"(o[2]),
                     "r"(o[3]));
      } else {  // a ragged edge chunk: bytes [lo, hi) of it
        store_partial16(d.out + e, o, i0 < off ? off - i0 : 0u, min(16u, data_end - i0));
      }
    }
    tile = next;
  }
}

// Upload check (the E4M3 verify_gaps_kernel's job for this variant): per
// window the reference walk's count and end; a tile whose 8-window lanes
// run through (each inner window ends where the next one's gap says) and
// whose blocks decode to exactly their ranges keeps its bit in `ok`; the
// lanes' group offsets into lane_start.
__global__ void __launch_bounds__(256) e5_verify_kernel(const Desc d, std::uint32_t* ok, std::uint32_t* lane_start) {
  __shared__ Tables tb;
  __shared__ std::uint32_t gsum[64], lexcl[32];
  __shared__ unsigned bad_tile;
  for (int i = threadIdx.x; i < static_cast<int>(sizeof(Tables) / 2); i += 256)
    reinterpret_cast<std::uint16_t*>(&tb)[i] = reinterpret_cast<const std::uint16_t*>(d.tables)[i];
  __syncthreads();
  const std::uint32_t log2T = 31 - __clz(d.T);
  const std::uint32_t lpb = log2T >= 8 ? 32u : (1u << (log2T - 3));  // 8-window lanes per block
  const std::uint64_t n_tiles = (d.n_windows + 255) / 256;
  const std::uint64_t last_blk = d.n_blocks - 1;
  const std::uint64_t last_range = d.outpos[d.n_blocks] - d.outpos[last_blk];
  for (std::uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const std::uint64_t k = 256 * t + threadIdx.x;
    std::uint32_t cnt = 0, end = 0;
    bool mismatch = false;
    if (k < d.n_windows) {
      const std::uint64_t hi = be64(d.encoded + 8 * k), lo = be64(d.encoded + 8 * k + 8);
      std::uint32_t p = (d.gaps[k >> 1] >> ((k & 1) ? 0 : 4)) & 15u;
      while (p < 64) {
        std::uint32_t s, l;
        word_at(tb, hi, lo, p, s, l);
        p += l;
        ++cnt;
      }
      end = p - 64;
      if ((k & 7) != 7 && k + 1 < d.n_windows)
        mismatch = end != ((d.gaps[(k + 1) >> 1] >> (((k + 1) & 1) ? 0 : 4)) & 15u);
    }
    if (threadIdx.x == 0) bad_tile = 0;
    std::uint32_t g = cnt;
    g += __shfl_xor_sync(0xffffffffu, g, 1);
    g += __shfl_xor_sync(0xffffffffu, g, 2);
    if ((threadIdx.x & 3) == 0) gsum[threadIdx.x >> 2] = g;
    __syncthreads();
    if (threadIdx.x < 32) {
      const std::uint32_t i = threadIdx.x, v0 = gsum[2 * i], v1 = gsum[2 * i + 1], v = v0 + v1;
      std::uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (i >= static_cast<std::uint32_t>(o)) incl += y;
      }
      const std::uint32_t excl = incl - v - __shfl_sync(0xffffffffu, incl - v, i & ~(lpb - 1));
      lexcl[i] = excl;
      const std::uint64_t wg = 256 * t + 8 * i;
      if (wg < d.n_windows) {
        lane_start[wg >> 3] = excl | ((excl + v0) << 16);
        if ((i & (lpb - 1)) == lpb - 1 || wg + 8 >= d.n_windows) {  // the block's last lane
          const std::uint64_t blk = wg >> log2T;
          const std::uint64_t range = d.outpos[blk + 1] - d.outpos[blk];
          if (excl + v < range || (blk + 1 < d.n_blocks && excl + v > range)) atomicOr(&bad_tile, 1u);
        }
      }
    }
    __syncthreads();
    // A window whose walk does not end where the next window's gap says
    // breaks the lane's continuous parse -- unless the block's words already
    // ran out (the tensor's last block, past its final word: the zero padding
    // parses into words the block clamp drops, as the reference's does).
    std::uint32_t incl8 = cnt;  // the window's words and those of the windows before it in its 8-window lane
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl8, o, 8);
      if ((threadIdx.x & 7) >= static_cast<unsigned>(o)) incl8 += y;
    }
    const bool spent = (k >> log2T) == last_blk && lexcl[threadIdx.x >> 3] + incl8 >= last_range;
    if (__ballot_sync(0xffffffffu, mismatch && !spent) && (threadIdx.x & 31) == 0) atomicOr(&bad_tile, 1u);
    __syncthreads();
    if (threadIdx.x == 0 && bad_tile) atomicAnd(ok + (t >> 5), ~(1u << (t & 31)));
    __syncthreads();
  }
}

template <int NW, bool WIDE>
cudaError_t launch_fsm(const Desc& d, cudaStream_t s) {
  constexpr std::uint32_t kSym = WIDE ? 16384 : 8192;
  const int smem = 8 * 32 * 256 + static_cast<int>(4 * ((kSym / 8 + 8) + (kSym / 32 + 8))) * NW;
  static int grid_cap = 0;
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(e5_fsm_kernel<NW, WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid_cap = sms;
  }
  const std::uint32_t m = 256 / d.T;
  const std::uint64_t tiles = (d.n_blocks + m - 1) / m;
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>((tiles + NW - 1) / NW, grid_cap));
  if (grid == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = static_cast<std::size_t>(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = std::getenv("ECF8_NO_PDL") ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, e5_fsm_kernel<NW, WIDE>, d);
}

template <int NW>
cudaError_t launch_fsm_bytes(const Desc& d, cudaStream_t s) {
  const int smem = 8 * 32 * 256 + (8192 + 32) * NW;
  static int grid_cap = 0;
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(e5_fsm_bytes_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid_cap = sms;
  }
  const std::uint32_t m = 256 / d.T;
  const std::uint64_t tiles = (d.n_blocks + m - 1) / m;
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>((tiles + NW - 1) / NW, grid_cap));
  if (grid == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = static_cast<std::size_t>(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = std::getenv("ECF8_NO_PDL") ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, e5_fsm_bytes_kernel<NW>, d);
}

template <int NT>
cudaError_t launch(const Desc& d, cudaStream_t s) {
  const int smem = NT * 64 + 32;
  static int grid_cap = 0;
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(e5_decode_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, e5_decode_kernel<NT>, NT, smem);
    if (e != cudaSuccess) return e;
    grid_cap = sms * std::max(per_sm, 1);
  }
  const std::uint64_t tiles = (d.n_windows + NT - 1) / NT;
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(tiles, grid_cap));
  if (grid == 0) return cudaSuccess;
  e5_decode_kernel<NT><<<grid, NT, smem, s>>>(d);
  return cudaGetLastError();
}

#ifndef ECF8_E5_FSM_WARPS
#define ECF8_E5_FSM_WARPS 18  // 18 x 8 KB of symbol bytes + the 64 KB table
#endif
cudaError_t launch_e5(const Desc& d, cudaStream_t s) {
  if (d.fsm) return d.lmin >= 2 ? launch_fsm_bytes<ECF8_E5_FSM_WARPS>(d, s) : launch_fsm<14, true>(d, s);
  if (d.T <= 256) return launch<256>(d, s);
  if (d.T == 512) return launch<512>(d, s);
  return launch<1024>(d, s);
}

// Host: the byte-step state machine of a complete code (Kraft sum 1, >= 2
// words): states = internal nodes of the canonical code tree (the pending
// prefix; 0 = root), entry (state, byte) = the words the byte completes:
// .x low exponent nibbles (first lowest), .y = 4 * count | next state << 8 |
// high exponent bits << 16.  Empty when the code has none (incomplete, one
// word, > 32 states).
std::vector<uint2> build_fsm(const std::uint8_t lengths[kSyms]) {
  std::map<std::pair<int, std::uint32_t>, int> leaf, node;
  std::uint64_t kraft = 0;
  int present = 0;
  std::uint32_t code = 0, prev = 0;
  for (std::uint32_t l = 1; l <= 16; ++l)
    for (int s = 0; s < kSyms; ++s)
      if (lengths[s] == l) {
        if (prev) code <<= (l - prev);
        prev = l;
        leaf[{static_cast<int>(l), code++}] = s;
        kraft += std::uint64_t{1} << (16 - l);
        ++present;
      }
  if (present < 2 || kraft != (std::uint64_t{1} << 16)) return {};
  node[{0, 0}] = 0;
  for (int l = 1; l <= 16; ++l)
    for (const auto& [k, s] : leaf)
      if (k.first > l) {
        const std::pair<int, std::uint32_t> pre{l, k.second >> (k.first - l)};
        if (!node.count(pre)) node.emplace(pre, static_cast<int>(node.size()));
      }
  if (node.size() > 32) return {};
  int lmin = 16;
  for (const auto& [k, sym] : leaf) lmin = std::min(lmin, k.first);
  const bool bytes_form = lmin >= 2;  // <= 4 words per byte: symbols as bytes (e5_fsm_bytes_kernel)
  std::vector<uint2> t(32 * 256, uint2{0, 0});
  for (const auto& [pre, id] : node)
    for (std::uint32_t b = 0; b < 256; ++b) {
      int l = pre.first;
      std::uint32_t v = pre.second, lo = 0, hi = 0, n = 0, byte_syms = 0;
      for (int i = 0; i < 8; ++i) {
        ++l;
        v = (v << 1) | ((b >> (7 - i)) & 1u);
        auto f = leaf.find({l, v});
        if (f != leaf.end()) {
          lo |= static_cast<std::uint32_t>(f->second & 15) << (4 * n);
          if (n < 4) byte_syms |= static_cast<std::uint32_t>(f->second) << (8 * n);
          hi |= static_cast<std::uint32_t>((f->second >> 4) & 1) << n;
          ++n;
          l = 0;
          v = 0;
        } else if (!node.count({l, v})) {
          return {};  // not a prefix of any word (cannot happen for a complete code)
        }
      }
      t[id * 256 + b] = bytes_form ? uint2{byte_syms, (8 * n) | (static_cast<std::uint32_t>(node.at({l, v})) << 8)}
                                   : uint2{lo, (4 * n) | (static_cast<std::uint32_t>(node.at({l, v})) << 8) | (hi << 16)};
    }
  return t;
}

// Host: tables from the code lengths (validated: <= 16, Kraft <= 1, non-empty).
Tables build_tables(const std::uint8_t lengths[kSyms]) {
  std::uint64_t kraft = 0;
  bool any = false;
  for (int s = 0; s < kSyms; ++s) {
    if (lengths[s] > 16) throw std::invalid_argument("invalid length vector");
    if (lengths[s]) kraft += std::uint64_t{1} << (16 - lengths[s]), any = true;
  }
  if (!any || kraft > (std::uint64_t{1} << 16)) throw std::invalid_argument("invalid length vector");
  Tables t{};
  std::uint32_t code = 0, prev = 0, n = 0;
  std::uint16_t codes[kSyms] = {};
  for (std::uint32_t l = 1; l <= 16; ++l) {
    t.offset[l] = static_cast<std::uint8_t>(n);
    bool first = true;
    for (int s = 0; s < kSyms; ++s) {
      if (lengths[s] != l) continue;
      if (prev) code <<= (l - prev);
      prev = l;
      if (first) t.base[l] = static_cast<std::uint16_t>(code), first = false;
      codes[s] = static_cast<std::uint16_t>(code++);
      t.syms[n++] = static_cast<std::uint8_t>(s);
      ++t.count[l];
    }
  }
  for (int s = 0; s < kSyms; ++s)
    if (lengths[s]) {
      t.fb_sym = static_cast<std::uint8_t>(s), t.fb_len = lengths[s];
      break;
    }
  for (int s = 0; s < kSyms; ++s) {
    const std::uint32_t l = lengths[s];
    if (!l || l > static_cast<std::uint32_t>(kFastBits)) continue;
    const std::uint32_t lo = static_cast<std::uint32_t>(codes[s]) << (kFastBits - l), span = 1u << (kFastBits - l);
    for (std::uint32_t i = 0; i < span; ++i) t.fast[lo + i] = static_cast<std::uint16_t>(s | (l << 8));
  }
  return t;
}

}  // namespace ecf8::dev::e5

struct ecf8_e5_dev_tensor {
  void* arena = nullptr;
  void* aux = nullptr;  // byte-step table, group offsets, tile bits
  ecf8::dev::e5::Desc desc{};
};

namespace {

struct CudaFailure {
  cudaError_t err;
  const char* what;
};
inline void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure{e, what};
}
template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const CudaFailure& e) {
    cudaGetLastError();
    return ecf8_internal_set_error(ECF8_ECUDA, (std::string(e.what) + ": " + cudaGetErrorString(e.err)).c_str());
  } catch (const std::bad_alloc&) {
    return ecf8_internal_set_error(ECF8_ENOMEM, "host allocation failed");
  } catch (const std::invalid_argument& e) {
    return ecf8_internal_set_error(ECF8_EINVAL, e.what());
  } catch (const std::exception& e) {
    return ecf8_internal_set_error(ECF8_ECUDA, e.what());
  }
}

std::uint64_t up256(std::uint64_t x) { return (x + 255) & ~std::uint64_t{255}; }

// The decode-side checks of decode_parallel_into (codec.cpp:259-261) and
// parse_container (container.cpp:196-242) for the variant's sizes.
void validate(const ecf8_e5_sections& s) {
  const std::uint32_t T = s.threads_per_block;
  if (T < 1 || T > 1024 || (T & (T - 1)))
    throw std::invalid_argument("threads per block must be a power of two in [1, 1024]");
  if (s.encoded_len < 2 || (s.encoded_len - 2) % (std::uint64_t{8} * T))
    throw std::invalid_argument("encoded section length mismatch");
  const std::uint64_t nb = (s.encoded_len - 2) / (std::uint64_t{8} * T);
  if (s.n_outpos != nb + 1 || !s.outpos) throw std::invalid_argument("inconsistent block offsets");
  if (s.gaps_len != (nb * T + 1) / 2) throw std::invalid_argument("gap section length mismatch");
  if (s.raw_len != 12 * ((s.n_elem + 31) / 32)) throw std::invalid_argument("raw section length mismatch");
  if (s.outpos[0] != 0 || s.outpos[nb] != s.n_elem) throw std::invalid_argument("inconsistent block offsets");
  for (std::uint64_t b = 0; b < nb; ++b)
    if (s.outpos[b + 1] < s.outpos[b] || s.outpos[b + 1] - s.outpos[b] > std::uint64_t{64} * T)
      throw std::invalid_argument("inconsistent block offsets");
  if (s.n_elem && nb == 0) throw std::invalid_argument("encoded section length mismatch");
}

}  // namespace

extern "C" {

int ecf8_e5_upload(const ecf8_e5_sections* s, ecf8_e5_dev_tensor** out) {
  return guarded([&]() -> int {
    if (!s || !out) return ecf8_internal_set_error(ECF8_EINVAL, "null argument");
    *out = nullptr;
    if (int rc = ecf8_internal_require_device()) return rc;
    validate(*s);
    auto t = std::make_unique<ecf8_e5_dev_tensor>();
    ecf8::dev::e5::Tables tb{};
    if (s->n_elem) tb = ecf8::dev::e5::build_tables(s->lengths);
    const std::uint64_t nb = s->n_outpos - 1;
    const std::uint64_t o_enc = 0, o_gap = up256(s->encoded_len + 64), o_pos = o_gap + up256(s->gaps_len + 64),
                        o_raw = o_pos + up256(8 * s->n_outpos), o_tab = o_raw + up256(s->raw_len + 64),
                        total = o_tab + up256(sizeof(tb));
    cu(cudaMalloc(&t->arena, total), "cudaMalloc(e5 arena)");
    auto* base = static_cast<std::uint8_t*>(t->arena);
    cu(cudaMemset(base, 0, total), "memset(e5 arena)");
    cu(cudaMemcpy(base + o_enc, s->encoded, s->encoded_len, cudaMemcpyHostToDevice), "H2D encoded");
    if (s->gaps_len) cu(cudaMemcpy(base + o_gap, s->gaps, s->gaps_len, cudaMemcpyHostToDevice), "H2D gaps");
    cu(cudaMemcpy(base + o_pos, s->outpos, 8 * s->n_outpos, cudaMemcpyHostToDevice), "H2D outpos");
    if (s->raw_len) cu(cudaMemcpy(base + o_raw, s->raw, s->raw_len, cudaMemcpyHostToDevice), "H2D raw");
    cu(cudaMemcpy(base + o_tab, &tb, sizeof(tb), cudaMemcpyHostToDevice), "H2D tables");
    auto& d = t->desc;
    d.encoded = base + o_enc;
    d.gaps = base + o_gap;
    d.outpos = reinterpret_cast<const std::uint64_t*>(base + o_pos);
    d.raw = reinterpret_cast<const std::uint32_t*>(base + o_raw);
    d.tables = reinterpret_cast<const ecf8::dev::e5::Tables*>(base + o_tab);
    d.n_elem = s->n_elem;
    d.n_blocks = nb;
    d.n_windows = nb * s->threads_per_block;
    d.T = s->threads_per_block;
    d.lmin = 16;
    for (int i = 0; i < 32; ++i)
      if (s->lengths[i]) d.lmin = std::min<std::uint32_t>(d.lmin, s->lengths[i]);
    // byte steps when the code has a state machine and every tile passes the
    // upload check (encoder output); the window walk otherwise
    static const bool no_fsm = std::getenv("ECF8_E5_NO_FSM") != nullptr;  // A/B runs
    const std::uint32_t T = s->threads_per_block;
    const std::vector<uint2> fsm = (s->n_elem && T >= 8 && T <= 256 && !no_fsm)
                                       ? ecf8::dev::e5::build_fsm(s->lengths) : std::vector<uint2>{};
    if (!fsm.empty()) {
      const std::uint64_t n_tiles = (d.n_windows + 255) / 256, ok_words = (n_tiles + 31) / 32;
      void* aux = nullptr;
      const std::uint64_t o_ls = up256(8 * fsm.size()), o_ok = o_ls + up256(4 * (d.n_windows / 8 + 1));
      cu(cudaMalloc(&aux, o_ok + 4 * ok_words), "cudaMalloc(e5 aux)");
      t->aux = aux;
      auto* ab = static_cast<std::uint8_t*>(aux);
      cu(cudaMemcpy(ab, fsm.data(), 8 * fsm.size(), cudaMemcpyHostToDevice), "H2D e5 fsm");
      cu(cudaMemset(ab + o_ls, 0, 4 * (d.n_windows / 8 + 1)), "memset(lane_start)");
      cu(cudaMemset(ab + o_ok, 0xFF, 4 * ok_words), "memset(ok)");
      auto* ls = reinterpret_cast<std::uint32_t*>(ab + o_ls);
      auto* okb = reinterpret_cast<std::uint32_t*>(ab + o_ok);
      ecf8::dev::e5::e5_verify_kernel<<<static_cast<unsigned>(std::min<std::uint64_t>(n_tiles, 1184)), 256>>>(d, okb, ls);
      cu(cudaGetLastError(), "e5 verify launch");
      std::vector<std::uint32_t> bits(ok_words);
      cu(cudaMemcpy(bits.data(), okb, 4 * ok_words, cudaMemcpyDeviceToHost), "D2H ok");
      bool all = true;
      for (std::uint64_t v = 0; v < n_tiles; ++v) all &= ((bits[v >> 5] >> (v & 31)) & 1u) != 0;
      if (all) {
        d.fsm = reinterpret_cast<const uint2*>(ab);
        d.lane_start = ls;
      }
    }
    *out = t.release();
    return ECF8_OK;
  });
}

int ecf8_e5_decode_device(const ecf8_e5_dev_tensor* t, uint8_t* d_out, void* stream) {
  return guarded([&]() -> int {
    if (!t || (!d_out && t->desc.n_elem)) return ecf8_internal_set_error(ECF8_EINVAL, "null argument");
    if (reinterpret_cast<std::uintptr_t>(d_out) & 15)
      return ecf8_internal_set_error(ECF8_EINVAL, "device output must be 16-byte aligned");
    if (!t->desc.n_elem) return ECF8_OK;
    ecf8::dev::e5::Desc d = t->desc;
    d.out = d_out;
    cu(ecf8::dev::e5::launch_e5(d, static_cast<cudaStream_t>(stream)), "e5 decode launch");
    return ECF8_OK;
  });
}

uint64_t ecf8_e5_dev_n_elem(const ecf8_e5_dev_tensor* t) { return t ? t->desc.n_elem : 0; }

int ecf8_e5_dev_byte_steps(const ecf8_e5_dev_tensor* t) { return t && t->desc.fsm ? 1 : 0; }

void ecf8_e5_free(ecf8_e5_dev_tensor* t) {
  if (!t) return;
  if (t->arena) cudaFree(t->arena);
  if (t->aux) cudaFree(t->aux);
  delete t;
}

int ecf8_e5_decode_host(const ecf8_e5_sections* s, uint8_t* out, uint64_t out_len) {
  return guarded([&]() -> int {
    if (!s || (!out && s->n_elem)) return ecf8_internal_set_error(ECF8_EINVAL, "null argument");
    if (out_len != s->n_elem) return ecf8_internal_set_error(ECF8_EINVAL, "output size mismatch");
    ecf8_e5_dev_tensor* t = nullptr;
    if (int rc = ecf8_e5_upload(s, &t)) return rc;
    std::unique_ptr<ecf8_e5_dev_tensor, void (*)(ecf8_e5_dev_tensor*)> hold(t, ecf8_e5_free);
    if (!s->n_elem) return ECF8_OK;
    std::uint8_t* d_out = nullptr;
    cu(cudaMalloc(&d_out, (s->n_elem + 15) & ~std::uint64_t{15}), "cudaMalloc(e5 out)");
    std::unique_ptr<std::uint8_t, cudaError_t (*)(void*)> hold_out(d_out, cudaFree);
    if (int rc = ecf8_e5_decode_device(t, d_out, nullptr)) return rc;
    cu(cudaMemcpy(out, d_out, s->n_elem, cudaMemcpyDeviceToHost), "D2H e5 out");
    return ECF8_OK;
  });
}

}  // extern "C"
