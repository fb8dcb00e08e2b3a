// decode_common.cuh -- device building blocks shared by the ECF8 decode
// kernels (decode.cu: 256-thread tile groups; decode_warp.cu: warp tiles).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "decode.cuh"
#include "tables.hpp"

namespace ecf8::dev {

constexpr int kFastShift = 32 - kFastBits;

// Decode tables as staged in shared memory (see tables.hpp).  Entries of
// the fast table whose first word is not resolvable from kFastBits bits are
// rewritten on staging to the "flagged" form below.
struct Tables {
  std::uint32_t fast[kFastEntries];
  std::uint16_t smask[kFastEntries];
  std::uint8_t cascade[18 * 256];
};

// A fast entry with n == 0 is staged as: advance 1 bit, emit nothing, set
// kSlowFlag.  The fast walk then runs branch-free; a window that met such an
// entry is decoded again exactly by the slow walk (rare: code words longer
// than kFastBits bits, or garbage windows of incomplete codes).
constexpr std::uint32_t kSlowFlag = 1u << 11;
__host__ __device__ constexpr std::uint32_t stage_entry(std::uint32_t e) {
  return ((e >> 5) & 31) ? e : (kSlowFlag | 1u);
}

// Shared-memory accesses by 32-bit shared-window address: one register per
// address and no generic-to-shared conversion in the hot loops.
__device__ __forceinline__ std::uint32_t smem_addr(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ std::uint32_t lds32(std::uint32_t a) {
  std::uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ std::uint32_t lds16(std::uint32_t a) {
  std::uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(std::uint32_t a, std::uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Packs 4-bit symbols into consecutive 32-bit words (first symbol lowest)
// at shared address `addr`.
struct SlotSink {
  std::uint32_t addr;    // next word
  std::uint32_t lo = 0;  // partial word
  std::uint32_t q4 = 0;  // bits used in lo, < 32
  __device__ __forceinline__ void put(std::uint32_t syms, std::uint32_t n4) {
    const std::uint32_t nl = lo | (syms << q4);
    const std::uint32_t nh = __funnelshift_l(syms, 0u, q4);
    q4 += n4;
    if (q4 >= 32) {
      sts32(addr, nl);
      addr += 4;
      lo = nh;
      q4 -= 32;
    } else {
      lo = nl;
    }
  }
  // Flush the partial word; returns the symbol count since `base`.
  __device__ __forceinline__ std::uint32_t finish(std::uint32_t base) {
    if (q4) sts32(addr, lo);
    return (addr - base) * 2 + (q4 >> 2);
  }
};

struct CountSink {
  std::uint32_t n4 = 0;
  __device__ __forceinline__ void put(std::uint32_t, std::uint32_t k4) { n4 += k4; }
};

// The reference cascade (lut.hpp:43-49) on the 16-bit head of `hi`, as a
// fast-format entry: one symbol, its length as b.
__device__ __forceinline__ std::uint32_t slow_entry(std::uint32_t hi, const Tables& tb,
                                                    std::uint32_t len_off) {
  const std::uint32_t w16 = hi >> 16;
  std::uint32_t v = tb.cascade[w16 >> 8];
  if (v >= 240) v = tb.cascade[((256u - v) << 8) | (w16 & 255u)];
  return (v << 12) | (4u << 5) | tb.cascade[len_off + v];
}

// Exact walk of one 64-bit window: the code words that start in [gap, 64)
// (codec.cpp:133-190 semantics); w0..w3 = window bits 0..127, big-endian.
// Handles every entry kind; used for count_phase and for flagged windows.
template <class Sink>
__device__ __forceinline__ void decode_window_exact(std::uint32_t w0, std::uint32_t w1,
                                                    std::uint32_t w2, std::uint32_t w3,
                                                    std::uint32_t gap, const Tables& tb,
                                                    std::uint32_t len_off, Sink& sink) {
  std::uint32_t hi = __funnelshift_l(w1, w0, gap);
  std::uint32_t lo = __funnelshift_l(w2, w1, gap);
  std::uint32_t p = gap;
  while (p < 32) {
    std::uint32_t e = tb.fast[hi >> kFastShift];
    if (e & kSlowFlag) e = slow_entry(hi, tb, len_off);
    sink.put(e >> 12, (e >> 5) & 31);
    hi = __funnelshift_l(lo, hi, e);
    lo = __funnelshift_l(0u, lo, e);
    p += e & 31;
  }
  hi = __funnelshift_l(w2, w1, p - 32);
  lo = __funnelshift_l(w3, w2, p - 32);
  for (;;) {
    const std::uint32_t idx = hi >> kFastShift;
    std::uint32_t e = tb.fast[idx];
    const bool fast_hit = !(e & kSlowFlag);
    if (!fast_hit) e = slow_entry(hi, tb, len_off);
    const std::uint32_t b = e & 31, r = 64 - p;
    if (b >= r) {
      const std::uint32_t starts = fast_hit ? tb.smask[idx] : 1u;
      const std::uint32_t k4 = 4 * __popc(starts & ((1u << r) - 1));
      sink.put((e >> 12) & ((1u << k4) - 1), k4);
      return;
    }
    sink.put(e >> 12, (e >> 5) & 31);
    hi = __funnelshift_l(lo, hi, e);
    lo = __funnelshift_l(0u, lo, e);
    p += b;
  }
}

// Branch-free fast walk of one window; returns false (sink contents then
// garbage) if a flagged entry was met -- the caller rewinds and uses the
// exact walk.
//
// Phase A runs while at least 32 valid bits remain in the 64-bit register
// window (one entry never reaches the window boundary from there); one
// refill; phase B takes whole entries until the next one would cross bit 64
// and then exactly the symbols that start before it (start-bit mask +
// popcount, the codec.cpp:143-160 rule).
// fast = shared address of tb.fast, smask = shared address of tb.smask.
__device__ __forceinline__ bool decode_window_fast(std::uint32_t w0, std::uint32_t w1, std::uint32_t w2,
                                                   std::uint32_t w3, std::uint32_t gap, std::uint32_t fast,
                                                   std::uint32_t smask, SlotSink& sink) {
  std::uint32_t hi = __funnelshift_l(w1, w0, gap);
  std::uint32_t lo = __funnelshift_l(w2, w1, gap);
  std::uint32_t p = gap, flags = 0;
  while (p < 32) {
    const std::uint32_t e = lds32(fast + ((hi >> (kFastShift - 2)) & ~3u));
    flags |= e;
    sink.put(e >> 12, (e >> 5) & 31);
    hi = __funnelshift_l(lo, hi, e);  // shift amount = e & 31 = bits consumed
    lo = __funnelshift_l(0u, lo, e);
    p += e & 31;
  }
  hi = __funnelshift_l(w2, w1, p - 32);  // p in [32, 44): window = bits [p, p + 64)
  lo = __funnelshift_l(w3, w2, p - 32);
  for (;;) {
    const std::uint32_t idx = hi >> kFastShift;
    const std::uint32_t e = lds32(fast + 4 * idx);
    flags |= e;
    const std::uint32_t b = e & 31, r = 64 - p;
    if (b >= r) {
      const std::uint32_t k4 = 4 * __popc(lds16(smask + 2 * idx) & ((1u << r) - 1));
      sink.put((e >> 12) & ((1u << k4) - 1), k4);
      break;
    }
    sink.put(e >> 12, (e >> 5) & 31);
    hi = __funnelshift_l(lo, hi, e);
    lo = __funnelshift_l(0u, lo, e);
    p += b;
  }
  return !(flags & kSlowFlag);
}

// Two independent windows walked in lockstep (two dependency chains per
// thread).  Each chain is the branch-free fast walk above; a finished or
// absent chain is fed the null entry (b = n = 0), which is a no-op.
struct Walk {
  std::uint32_t hi, lo, p, flags;
  bool live;
};

__device__ __forceinline__ Walk walk_begin(std::uint32_t w0, std::uint32_t w1, std::uint32_t w2,
                                           std::uint32_t gap, bool live) {
  return Walk{__funnelshift_l(w1, w0, gap), __funnelshift_l(w2, w1, gap), gap, 0u, live};
}

__device__ __forceinline__ void walk_step_a(Walk& s, std::uint32_t fast, SlotSink& sink) {
  const std::uint32_t e0 = lds32(fast + ((s.hi >> (kFastShift - 2)) & ~3u));
  const std::uint32_t e = (s.live && s.p < 32) ? e0 : 0u;
  s.flags |= e;
  sink.put(e >> 12, (e >> 5) & 31);
  s.hi = __funnelshift_l(s.lo, s.hi, e);
  s.lo = __funnelshift_l(0u, s.lo, e);
  s.p += e & 31;
}

__device__ __forceinline__ void walk_refill(Walk& s, std::uint32_t w1, std::uint32_t w2, std::uint32_t w3) {
  const std::uint32_t sh = s.p - 32;  // p in [32, 44) for live walks
  s.hi = __funnelshift_l(w2, w1, sh);
  s.lo = __funnelshift_l(w3, w2, sh);
}

__device__ __forceinline__ void walk_step_b(Walk& s, std::uint32_t fast, std::uint32_t smask, SlotSink& sink) {
  const std::uint32_t idx = s.hi >> kFastShift;
  const std::uint32_t e0 = lds32(fast + 4 * idx);
  const std::uint32_t e = s.live ? e0 : 0u;
  s.flags |= e;
  const std::uint32_t b = e & 31, r = 64 - s.p;
  const bool tail = b >= r;  // never for a dead walk (b = 0 < r)
  std::uint32_t syms = e >> 12, k4 = (e >> 5) & 31;
  if (tail) {  // only the symbols that start before bit 64
    k4 = 4 * __popc(lds16(smask + 2 * idx) & ((1u << (r < 16 ? r : 16)) - 1));
    syms &= (1u << k4) - 1;
    s.live = false;
  }
  sink.put(syms, k4);
  s.hi = __funnelshift_l(s.lo, s.hi, e);
  s.lo = __funnelshift_l(0u, s.lo, e);
  s.p += b;
}

// Windows (a0..a3, ga) -> sink_a and (b0..b3, gb) -> sink_b, interleaved.
// Flagged windows are rewound and decoded by the exact walk.
__device__ __forceinline__ void decode_window_pair(const std::uint32_t* wa, std::uint32_t ga, bool la,
                                                   SlotSink& sa, const std::uint32_t* wb, std::uint32_t gb,
                                                   bool lb, SlotSink& sb, const Tables& tb,
                                                   std::uint32_t fast, std::uint32_t smask,
                                                   std::uint32_t len_off) {
  const SlotSink save_a = sa, save_b = sb;
  Walk A = walk_begin(wa[0], wa[1], wa[2], ga, la);
  Walk B = walk_begin(wb[0], wb[1], wb[2], gb, lb);
  while ((A.live && A.p < 32) || (B.live && B.p < 32)) {
    walk_step_a(A, fast, sa);
    walk_step_a(B, fast, sb);
  }
  walk_refill(A, wa[1], wa[2], wa[3]);
  walk_refill(B, wb[1], wb[2], wb[3]);
  while (A.live || B.live) {
    walk_step_b(A, fast, smask, sa);
    walk_step_b(B, fast, smask, sb);
  }
  if (la && (A.flags & kSlowFlag)) {
    sa = save_a;
    decode_window_exact(wa[0], wa[1], wa[2], wa[3], ga, tb, len_off, sa);
  }
  if (lb && (B.flags & kSlowFlag)) {
    sb = save_b;
    decode_window_exact(wb[0], wb[1], wb[2], wb[3], gb, tb, len_off, sb);
  }
}

// Appends the `nb` nibbles at slot words [src, ...) to the `na` nibbles at
// slot words [dst, ...) (shared addresses; dst + na/8 <= src, so every
// source word is read before it can be overwritten).
__device__ __forceinline__ void join_nibbles(std::uint32_t dst, std::uint32_t na, std::uint32_t src,
                                             std::uint32_t nb) {
  if (nb == 0) return;
  const std::uint32_t f4 = (na & 7) * 4;
  std::uint32_t at = dst + 4 * (na >> 3);
  const std::uint32_t nw = (nb + 7) >> 3;
  std::uint32_t prev = f4 ? (lds32(at) & ((1u << f4) - 1)) : 0u;  // head of the first piece
  std::uint32_t carry = prev;
  for (std::uint32_t k = 0; k < nw; ++k, at += 4) {
    const std::uint32_t cur = lds32(src + 4 * k);
    sts32(at, (cur << f4) | carry);
    carry = f4 ? (cur >> (32 - f4)) : 0u;
  }
  if (f4) sts32(at, carry);
  (void)prev;
}

__device__ __forceinline__ void decode_window(std::uint32_t w0, std::uint32_t w1, std::uint32_t w2,
                                              std::uint32_t w3, std::uint32_t gap, const Tables& tb,
                                              std::uint32_t len_off, SlotSink& sink) {
  const SlotSink saved = sink;
  if (!decode_window_fast(w0, w1, w2, w3, gap, smem_addr(tb.fast), smem_addr(tb.smask), sink)) {
    sink = saved;
    decode_window_exact(w0, w1, w2, w3, gap, tb, len_off, sink);
  }
}

__device__ __forceinline__ std::uint32_t bswap32(std::uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__device__ __forceinline__ std::uint32_t sel(std::uint32_t a, std::uint32_t b, std::uint32_t m) {
  return (a & m) | (b & ~m);
}

// Eight FP8 bytes from eight exponent nibbles S (element i at bits 4i..4i+3)
// and four packed sign/mantissa bytes P (element 2j in the high nibble of
// byte j): byte = sign << 7 | exponent << 3 | mantissa  (fp8.hpp assemble).
__device__ __forceinline__ void merge8(std::uint32_t S, std::uint32_t P, std::uint32_t& o0,
                                       std::uint32_t& o1) {
  const std::uint32_t even = sel(sel(S << 3, P, 0x78787878u), P >> 4, 0xF8F8F8F8u);
  const std::uint32_t odd = sel(sel(S >> 1, P << 4, 0x78787878u), P, 0xF8F8F8F8u);
  o0 = __byte_perm(even, odd, 0x5140);
  o1 = __byte_perm(even, odd, 0x7362);
}

__device__ __forceinline__ std::uint8_t merge1(std::uint32_t x, std::uint32_t qb, std::uint32_t odd) {
  const std::uint32_t qh = odd ? (qb << 4) : qb;
  return static_cast<std::uint8_t>((x << 3) | (qh & 0x80u) | ((qh >> 4) & 7u));
}

__device__ __forceinline__ std::uint32_t low_nibbles(std::uint32_t n) {  // n in 1..8
  return n >= 8 ? 0xFFFFFFFFu : ((1u << (4 * n)) - 1);
}

__device__ __forceinline__ int find_desc(const TensorDesc* descs, int n, std::uint64_t tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (descs[mid].tile_begin <= tile) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Stage a tensor's tables into shared memory (all threads of the CTA).
__device__ __forceinline__ void stage_tables(const TensorDesc& d, Tables& tb, int tid, int nthreads) {
  const uint4* f4 = reinterpret_cast<const uint4*>(d.fast);
  uint4* sf4 = reinterpret_cast<uint4*>(tb.fast);
  for (int i = tid; i < kFastEntries / 4; i += nthreads) {
    uint4 v = __ldg(f4 + i);
    v.x = stage_entry(v.x);
    v.y = stage_entry(v.y);
    v.z = stage_entry(v.z);
    v.w = stage_entry(v.w);
    sf4[i] = v;
  }
  const uint4* m4 = reinterpret_cast<const uint4*>(d.smask);
  uint4* sm4 = reinterpret_cast<uint4*>(tb.smask);
  for (int i = tid; i < kFastEntries / 8; i += nthreads) sm4[i] = __ldg(m4 + i);
  for (int i = tid; i < static_cast<int>(d.n_luts) * 256; i += nthreads) tb.cascade[i] = d.cascade[i];
}

// Byte-wise write of output elements [lo, hi) (staging nibble coordinates)
// for tile edges shared with neighbouring tiles.
__device__ __forceinline__ void write_edge(const std::uint32_t* stage, std::uint8_t* out,
                                           const std::uint8_t* pk, std::uint32_t lo, std::uint32_t hi) {
  for (std::uint32_t i = lo; i < hi; ++i) {
    const std::uint32_t x = (stage[i >> 3] >> (4 * (i & 7))) & 15u;
    out[i] = merge1(x, pk[i >> 1], i & 1);
  }
}

}  // namespace ecf8::dev
