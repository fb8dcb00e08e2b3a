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
struct alignas(16) Tables {
  std::uint16_t smask[kFastEntries];
  std::uint8_t cascade[18 * 256];
  std::uint32_t fast[kFastEntries];  // last: decode_warp.cu places it at a 16 KB-aligned shared address
};


// Staged (shared-memory) fast entries, rearranged from the host layout
// (tables.hpp: b 0..4, n4 5..9, symbols 12..31):
//   bits  0..4   b   bits consumed (the funnel-shift amount)
//   bit   5      0
//   bit   6      kSlowFlag: first code word not resolvable from kFastBits
//                bits (then b = 0, nothing emitted; the window is redone by
//                the exact walk -- rare: long code words, garbage windows)
//   bits  7..11  n4  4 x symbols
//   bits 12..31  up to five 4-bit symbols, first lowest
// Bits 0..6 of a walk position that adds whole entries are therefore exact
// (at most 43 + 64 < 128, no carry into bit 7); higher bits collect garbage
// that nothing reads -- one IADD per step instead of mask + add.
constexpr std::uint32_t kSlowFlag = 1u << 6;
constexpr std::uint32_t kPhaseDone = 0x60u;  // position bits 5..6: past bit 32 of the phase, or flagged
__host__ __device__ constexpr std::uint32_t stage_entry(std::uint32_t e) {
  return ((e >> 5) & 31) ? ((e & 0xFFFFF01Fu) | (((e >> 5) & 31u) << 7)) : kSlowFlag;
}
__host__ __device__ constexpr std::uint32_t entry_n4_ref(std::uint32_t e) { return (e >> 7) & 31u; }

// Integer multiplies the compiler must keep: IMAD runs on the FMA pipe, so a
// shift-left by multiply (plus the right shift or LEA.HI that follows)
// replaces a shift + LOP3 mask pair on the ALU pipe, which the walk keeps
// ~70 % busy.  ECF8_ALU_MASKS=1 restores the plain expressions (A/B).
#ifndef ECF8_ALU_MASKS
#define ECF8_ALU_MASKS 0
#endif
template <std::uint32_t M>
__device__ __forceinline__ std::uint32_t imul(std::uint32_t x) {
  std::uint32_t r;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "n"(M));
  return r;
}
__device__ __forceinline__ std::uint32_t entry_n4(std::uint32_t e) {
#if ECF8_ALU_MASKS
  return entry_n4_ref(e);
#else
  return imul<1u << 20>(e) >> 27;  // bits 7..11
#endif
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

// The fast-table entry for the next kFastBits bits of hi.
// FIXED: the kernel pins the table at shared address kFastAt (decode_warp.cu
// checks it), so the address is offset + constant -- the constant folds into
// the load's immediate and no base register has to live across the walk.
constexpr std::uint32_t kFastAt = 0x4000;
template <bool FIXED>
__device__ __forceinline__ std::uint32_t fast_entry(std::uint32_t fast, std::uint32_t hi) {
#if ECF8_ALU_MASKS
  const std::uint32_t off = (hi >> (kFastShift - 2)) & ~3u;
#else
  const std::uint32_t off = imul<4>(hi >> kFastShift);
#endif
  if constexpr (FIXED) {
    std::uint32_t v;  // constant in the load's immediate (ptxas would otherwise OR it in)
    asm volatile("ld.shared.u32 %0, [%1+16384];" : "=r"(v) : "r"(off));
    static_assert(kFastAt == 16384, "immediate above");
    return v;
  } else {
    return lds32(fast + off);
  }
}

// Packs 4-bit symbols into consecutive 32-bit slot words (first symbol
// lowest) starting at shared address `addr`; consecutive words are WS bytes
// apart (4: a lane's slot is contiguous; 128: the slots of a warp are
// interleaved word by word, so the 32 lanes' stores hit 32 different banks).
template <int WS>
struct SlotSinkT {
  std::uint32_t addr;    // next word
  std::uint32_t lo = 0;  // partial word
  std::uint32_t q4 = 0;  // bits used in lo, < 32
  __device__ __forceinline__ void put(std::uint32_t syms, std::uint32_t n4) {
    const std::uint32_t nl = lo | (syms << q4);
    const std::uint32_t nh = __funnelshift_l(syms, 0u, q4);
    q4 += n4;
    if (q4 >= 32) {
      sts32(addr, nl);
      addr += WS;
      lo = nh;
      q4 -= 32;
    } else {
      lo = nl;
    }
  }
  // Flush the partial word; returns the symbol count since `base`.
  __device__ __forceinline__ std::uint32_t finish(std::uint32_t base) {
    if (q4) sts32(addr, lo);
    return (addr - base) / WS * 8 + (q4 >> 2);
  }
};
using SlotSink = SlotSinkT<4>;

struct CountSink {
  std::uint32_t n4 = 0;
  __device__ __forceinline__ void put(std::uint32_t, std::uint32_t k4) { n4 += k4; }
};

// Table access for the walks (a view, so a kernel may keep the start masks
// and the cascade -- window ends and flagged entries only -- elsewhere than
// shared memory; the fast table is always addressed in shared memory).
struct SmemTables {
  static constexpr bool kGlobal = false;
  const Tables& tb;
  __device__ __forceinline__ std::uint32_t fast_addr() const { return smem_addr(tb.fast); }
  __device__ __forceinline__ std::uint32_t fast(std::uint32_t idx) const { return tb.fast[idx]; }
  __device__ __forceinline__ std::uint32_t smask(std::uint32_t idx) const { return tb.smask[idx]; }
  __device__ __forceinline__ std::uint32_t cascade(std::uint32_t i) const { return tb.cascade[i]; }
};


// The same tables read from global memory (L1-cached) -- for the kernels
// whose shared memory holds the byte-step decoder instead (decode_warp.cu);
// only windows off the verified fast path get here.
struct GlobalTables {
  static constexpr bool kGlobal = true;
  const TensorDesc& d;
  __device__ __forceinline__ std::uint32_t fast_addr() const { return 0; }
  __device__ __forceinline__ std::uint32_t fast(std::uint32_t idx) const { return stage_entry(__ldg(d.fast + idx)); }
  __device__ __forceinline__ std::uint32_t smask(std::uint32_t idx) const { return __ldg(d.smask + idx); }
  __device__ __forceinline__ std::uint32_t cascade(std::uint32_t i) const { return __ldg(d.cascade + i); }
};

// The staged fast-table entry for the next kFastBits bits of hi, from
// shared memory (address `fast`) or through the global view.
template <bool OR_BASE, class TV>
__device__ __forceinline__ std::uint32_t tv_fast(const TV& tv, std::uint32_t fast, std::uint32_t hi) {
  if constexpr (TV::kGlobal) return tv.fast(hi >> kFastShift);
  else return fast_entry<OR_BASE>(fast, hi);
}

// The reference cascade (lut.hpp:43-49) on the 16-bit head of `hi`, as a
// fast-format entry: one symbol, its length as b.
template <class TV>
__device__ __forceinline__ std::uint32_t slow_entry(std::uint32_t hi, const TV& tv, std::uint32_t len_off) {
  const std::uint32_t w16 = hi >> 16;
  std::uint32_t v = tv.cascade(w16 >> 8);
  if (v >= 240) v = tv.cascade(((256u - v) << 8) | (w16 & 255u));
  return (v << 12) | (4u << 7) | tv.cascade(len_off + v);
}

// Exact walk of one 64-bit window: the code words that start in [gap, 64)
// (codec.cpp:133-190 semantics); w0..w3 = window bits 0..127, big-endian.
// Handles every entry kind; used for count_phase and for flagged windows.
template <class Sink, class TV>
__device__ __forceinline__ void decode_window_exact(std::uint32_t w0, std::uint32_t w1,
                                                    std::uint32_t w2, std::uint32_t w3,
                                                    std::uint32_t gap, const TV& tb,
                                                    std::uint32_t len_off, Sink& sink) {
  std::uint32_t hi = __funnelshift_l(w1, w0, gap);
  std::uint32_t lo = __funnelshift_l(w2, w1, gap);
  std::uint32_t p = gap;
  while (p < 32) {
    std::uint32_t e = tb.fast(hi >> kFastShift);
    if (e & kSlowFlag) e = slow_entry(hi, tb, len_off);
    sink.put(e >> 12, entry_n4(e));
    hi = __funnelshift_l(lo, hi, e);
    lo = __funnelshift_l(0u, lo, e);
    p += e & 31;
  }
  hi = __funnelshift_l(w2, w1, p - 32);
  lo = __funnelshift_l(w3, w2, p - 32);
  for (;;) {
    const std::uint32_t idx = hi >> kFastShift;
    std::uint32_t e = tb.fast(idx);
    const bool fast_hit = !(e & kSlowFlag);
    if (!fast_hit) e = slow_entry(hi, tb, len_off);
    const std::uint32_t b = e & 31, r = 64 - p;
    if (b >= r) {
      const std::uint32_t starts = fast_hit ? tb.smask(idx) : 1u;
      const std::uint32_t k4 = 4 * __popc(starts & ((1u << r) - 1));
      sink.put((e >> 12) & ((1u << k4) - 1), k4);
      return;
    }
    sink.put(e >> 12, entry_n4(e));
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
template <class Sink, bool OR_BASE, class TV>
__device__ __forceinline__ bool decode_window_fast(std::uint32_t w0, std::uint32_t w1, std::uint32_t w2,
                                                   std::uint32_t w3, std::uint32_t gap, std::uint32_t fast,
                                                   const TV& tv, Sink& sink) {
  std::uint32_t hi = __funnelshift_l(w1, w0, gap);
  std::uint32_t lo = __funnelshift_l(w2, w1, gap);
  std::uint32_t p = gap;  // adds whole staged entries: bits 0..6 exact, kSlowFlag ends the loop
  while (!(p & kPhaseDone)) {
    const std::uint32_t e = tv_fast<OR_BASE>(tv, fast, hi);
    sink.put(e >> 12, entry_n4(e));
    hi = __funnelshift_l(lo, hi, e);  // shift amount = e & 31 = bits consumed
    lo = __funnelshift_l(0u, lo, e);
    p += e;
  }
  if (p & kSlowFlag) return false;
  p &= 63;
  hi = __funnelshift_l(w2, w1, p - 32);  // p in [32, 44): window = bits [p, p + 64)
  lo = __funnelshift_l(w3, w2, p - 32);
  for (;;) {
    const std::uint32_t idx = hi >> kFastShift;
    const std::uint32_t e = tv_fast<OR_BASE>(tv, fast, hi);
    if (e & kSlowFlag) return false;
    const std::uint32_t b = e & 31, r = 64 - p;
    if (b >= r) {
      const std::uint32_t k4 = 4 * __popc(tv.smask(idx) & ((1u << r) - 1));
      sink.put((e >> 12) & ((1u << k4) - 1), k4);
      return true;
    }
    sink.put(e >> 12, entry_n4(e));
    hi = __funnelshift_l(lo, hi, e);
    lo = __funnelshift_l(0u, lo, e);
    p += b;
  }
}

// Continuous fast walk over a lane's n consecutive windows (n <= 8; w holds
// their 2n big-endian words plus 2 lookahead words): starts at the first
// window's gap and runs through the window boundaries without restarting,
// taking every code word that starts before bit 64n.  Equals the per-window
// walks of decode_window_fast (codec.cpp:133-190) exactly when each window's
// gap is the start of the first code word the stream places in it -- true
// for every encoder-produced stream; the upload-time gap check
// (verify_gaps_kernel) establishes it per 256-window tile.  Returns false if
// a flagged entry was met (the caller redoes the windows exactly).
template <int NW, class Sink, bool OR_BASE, class TV, bool FULL = false>
__device__ __forceinline__ bool decode_lane_continuous(const std::uint32_t (&w)[2 * NW + 2], std::uint32_t n,
                                                       std::uint32_t gap, std::uint32_t fast, const TV& tv,
                                                       Sink& sink) {
  std::uint32_t hi = __funnelshift_l(w[1], w[0], gap);
  std::uint32_t lo = __funnelshift_l(w[2], w[1], gap);
  // p: bit position of hi's MSB within the current 32-bit phase (bits 0..6,
  // the walk adds whole staged entries).  A flagged entry sets kSlowFlag,
  // which ends this and -- kept through the phase steps -- every later phase
  // loop: no separate flag accumulator in the hot loop.
  std::uint32_t p = gap;
  const std::uint32_t last = FULL ? 2 * NW - 1 : 2 * n - 1;  // FULL: n == NW known at compile time
#pragma unroll
  for (std::uint32_t k = 0; k < 2 * NW; ++k) {
    if (k == last) {
      // final half window: whole entries while they end before bit 32, then
      // the symbols that start before it (start mask + popcount)
      if (!(p & kPhaseDone)) {
        p &= 31;
        for (;;) {
          const std::uint32_t idx = hi >> kFastShift;
          const std::uint32_t e = fast_entry<OR_BASE>(fast, hi);
          if (e & kSlowFlag) {
            p = kSlowFlag;
            break;
          }
          const std::uint32_t b = e & 31, r = 32 - p;
          if (b >= r) {
            const std::uint32_t k4 = 4 * __popc(tv.smask(idx) & ((1u << r) - 1));
            sink.put((e >> 12) & ((1u << k4) - 1), k4);
            break;
          }
          sink.put(e >> 12, entry_n4(e));
          hi = __funnelshift_l(lo, hi, e);
          lo = __funnelshift_l(0u, lo, e);
          p += b;
        }
      }
      break;
    }
    while (!(p & kPhaseDone)) {
      const std::uint32_t e = fast_entry<OR_BASE>(fast, hi);
      sink.put(e >> 12, entry_n4(e));
      hi = __funnelshift_l(lo, hi, e);
      lo = __funnelshift_l(0u, lo, e);
      p += e;
    }
    p = (p & kSlowFlag) ? kSlowFlag : (p & 63) - 32;  // next phase: hi:lo = bits [32(k+1) + p, +64)
    if (k + 3 < 2 * NW + 2) {
      hi = __funnelshift_l(w[k + 2], w[k + 1], p);
      lo = __funnelshift_l(w[k + 3], w[k + 2], p);
    }
  }
  return !(p & kSlowFlag);
}

// ---- byte-step decoder (tables.hpp fsm / fsm_cm) --------------------------

__device__ __forceinline__ std::uint32_t prmt(std::uint32_t a, std::uint32_t b, std::uint32_t sel) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Shared address of the staged byte-step table: the kernels that use it pin
// it there, so a probe is [index * 4 + constant] (decode_warp.cu checks).
constexpr std::uint32_t kFsmAt = 0x800;
constexpr std::uint32_t kFsmCmAt = kFsmAt + 4 * 256 * kFsmStates;

// One byte step: the entry for (state of `prev`, byte j of the pre-shifted
// lane stream s[]).  The index is state * 256 + byte, built by one byte
// permute: byte 0 from the stream word (big-endian: byte j is byte 3 - j % 4
// of s[j / 4]), byte 1 = prev's state byte, bytes 2-3 = that byte's sign
// (0: states are < 16).
__device__ __forceinline__ std::uint32_t fsm_index(std::uint32_t word, std::uint32_t prev, int j) {
  return prmt(word, prev, 0xDD50u | static_cast<std::uint32_t>(3 - (j & 3)));
}
__device__ __forceinline__ std::uint32_t fsm_entry(std::uint32_t idx) {
  std::uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1+2048];" : "=r"(v) : "r"(imul<4>(idx)));
  static_assert(kFsmAt == 2048, "immediate above");
  return v;
}
__device__ __forceinline__ std::uint32_t fsm_cm(std::uint32_t idx) {
  std::uint16_t v;
  asm volatile("ld.shared.u8 %0, [%1+18432];" : "=h"(v) : "r"(idx));
  static_assert(kFsmCmAt == 18432, "immediate above");
  return v;
}

// Where the byte-step tables are: pinned at kFsmAt (FsmPinned, the probe
// address in the load's immediate), or at shared addresses held in registers
// (FsmAt: the kernels whose static shared layout is not pinned; index * 4 +
// base is one IMAD, like index * 4).
struct FsmPinned {
  __device__ __forceinline__ std::uint32_t entry(std::uint32_t idx) const { return fsm_entry(idx); }
  __device__ __forceinline__ std::uint32_t cm(std::uint32_t idx) const { return fsm_cm(idx); }
};
struct FsmAt {
  std::uint32_t tab, cmb;  // shared addresses of the entries and the completion masks
  __device__ __forceinline__ std::uint32_t entry(std::uint32_t idx) const {
    std::uint32_t a, v;
    asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a) : "r"(idx), "r"(tab));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
  }
  __device__ __forceinline__ std::uint32_t cm(std::uint32_t idx) const {
    std::uint16_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(idx + cmb));
    return v;
  }
};

// Nibble sink for two byte steps at once: their symbol fields (<= 4 + 4
// symbols) are joined into one 32-bit run c, then appended at nibble q4 of
// the partial word lo; a full word goes to the slot.  q4 adds the whole
// entries (n4 in bits 0..4, bit 5 clear): bits 0..4 stay exact, bit 5
// toggles when a word fills (the pair adds <= 32 bits: at most one word),
// the state / symbol bits above collect garbage nothing reads.
#ifndef ECF8_PUT2_PRED
#define ECF8_PUT2_PRED 1
#endif
// The symbol fields of two consecutive byte-step entries joined into one run:
// (e1 >> 16) | ((e2 >> 16) << n4(e1)).  The two right shifts run as IMAD.HI
// (x * 2^16, high word) on the FMA pipe and the OR folds into the second one's
// addend (the fields are disjoint), leaving one funnel shift on the ALU pipe,
// which the byte steps keep ~73 % busy.  ECF8_JOIN_ALU=1: the plain shifts.
#ifndef ECF8_JOIN_ALU
#define ECF8_JOIN_ALU 0
#endif
#if ECF8_JOIN_CONST
__constant__ std::uint32_t c_65536 = 65536;
#endif
__device__ __forceinline__ std::uint32_t join_pair(std::uint32_t e1, std::uint32_t e2) {
#if ECF8_JOIN_ALU
  return (e1 >> 16) | __funnelshift_l(0u, e2 >> 16, e1);
#else
  std::uint32_t t, c;
  asm("mul.hi.u32 %0, %1, 65536;" : "=r"(t) : "r"(e2));
  t = __funnelshift_l(0u, t, e1);  // << n4(e1) (bits 0..4 of e1)
#if ECF8_JOIN_CONST
  c = __umulhi(e1, c_65536) + t;  // IMAD.HI by a constant-bank 2^16 (ptxas keeps it on the FMA pipe)
#else
  asm("mad.hi.u32 %0, %1, 65536, %2;" : "=r"(c) : "r"(e1), "r"(t));  // (ptxas: LEA.HI)
#endif
  return c;
#endif
}

// The sink's adds as IMADs by a constant-bank 1 the compiler cannot fold
// (x * c_one + y), moving two more ALU-pipe operations per byte pair to the
// FMA pipe: q4 + e1 + e2, and the OR of the disjoint partial word and shifted
// run.  A/B (r3j): decode +0.1-0.9 %, fused -0.3-0.6 % time; 0 restores them.
#ifndef ECF8_SINK_FMA
#define ECF8_SINK_FMA 1
#endif
#if ECF8_SINK_FMA
__constant__ std::uint32_t c_one = 1;
__device__ __forceinline__ std::uint32_t add3_fma(std::uint32_t a, std::uint32_t b, std::uint32_t c) {
  return b * c_one + (c * c_one + a);
}
__device__ __forceinline__ std::uint32_t or_disjoint(std::uint32_t a, std::uint32_t b) { return b * c_one + a; }
#else
__device__ __forceinline__ std::uint32_t add3_fma(std::uint32_t a, std::uint32_t b, std::uint32_t c) {
  return a + b + c;
}
__device__ __forceinline__ std::uint32_t or_disjoint(std::uint32_t a, std::uint32_t b) { return a | b; }
#endif

template <int WS>
struct PairSink {
  std::uint32_t addr;  // next slot word
  std::uint32_t lo = 0, q4 = 0;
  __device__ __forceinline__ void put2(std::uint32_t e1, std::uint32_t e2) {
    const std::uint32_t c = join_pair(e1, e2);  // f2 << n4(e1)
    const std::uint32_t q = add3_fma(q4, e1, e2);
    const std::uint32_t nl = or_disjoint(lo, __funnelshift_l(0u, c, q4));  // c << (q4 % 32)
    const std::uint32_t nh = __funnelshift_l(c, 0u, q4);       // c >> (32 - q4 % 32)
#if ECF8_PUT2_PRED
    // one predicate for the store, the address step and the select (no
    // 0 / WS materialisation)
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
        "xor.b32 t, %3, %4;\n\t"
        "and.b32 t, t, 32;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "@p st.shared.u32 [%0], %5;\n\t"
        "@p add.u32 %0, %0, %6;\n\t"
        "selp.b32 %1, %2, %5, p;\n\t}"
        : "+r"(addr), "=r"(lo)
        : "r"(nh), "r"(q), "r"(q4), "r"(nl), "n"(WS)
        : "memory");
#else
    const bool full = ((q ^ q4) & 32u) != 0;
    if (full) sts32(addr, nl);
    addr += full ? WS : 0u;
    lo = full ? nh : nl;
#endif
    q4 = q;
  }
  __device__ __forceinline__ std::uint32_t finish(std::uint32_t base) {
    if (q4 & 31u) sts32(addr, lo);
    return (addr - base) / WS * 8 + ((q4 & 31u) >> 2);
  }
  // put2 for a run that ends at a known place: words before `ew` (the word
  // holding the run's end nibble) are stored, the end word's bits go to
  // `tail` (OR-ed in by the caller, masked to the run), words after it are
  // dropped -- the symbols a parse produces past the run's end.
  __device__ __forceinline__ void put2_bounded(std::uint32_t e1, std::uint32_t e2, std::uint32_t ew,
                                               std::uint32_t& tail) {
    const std::uint32_t c = join_pair(e1, e2);
    const std::uint32_t q = add3_fma(q4, e1, e2);
    const std::uint32_t nl = or_disjoint(lo, __funnelshift_l(0u, c, q4));
    const std::uint32_t nh = __funnelshift_l(c, 0u, q4);
    const bool full = ((q ^ q4) & 32u) != 0;
    if (full && addr < ew) sts32(addr, nl);
    if (full && addr == ew) tail = nl;
    addr += full ? WS : 0u;
    lo = full ? nh : nl;
    q4 = q;
  }
};

// The code words of n consecutive windows (w: their 2n big-endian words + 2
// lookahead words) from bit gap0 of the first up to bit 64 n + end, decoded
// by byte steps and appended to the sink.  With end = the last window's
// endgap (its reference walk stops at bit 64 + end: the first word starting
// at or after the window boundary, codec.cpp:143-160) this is exactly the
// words the reference's walks of the n windows take -- for n = 1 always,
// for n > 1 when every inner window ends where the next one's gap says
// (the upload check).  A complete code parses every bit string the way the
// reference's decode_one chain does, so no fallback is needed.
template <int NWIN, int WS, class FT = FsmPinned>
__device__ __forceinline__ void decode_windows_fsm(const std::uint32_t* w, std::uint32_t gap0, std::uint32_t end,
                                                   PairSink<WS>& sink, const FT& ft = FT{}) {
  constexpr int NB = 8 * NWIN;      // bytes of the windows
  constexpr int NS = 2 * NWIN + 1;  // stream words from bit gap0: bytes 0 .. 4 NS - 1 >= NB + 2
  std::uint32_t st[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) st[i] = __funnelshift_l(w[i + 1], w[i], gap0);
  // end of the words, relative to gap0: byte Bp, bit r of it
  const std::uint32_t Lp = 64u * NWIN + end - gap0;  // in [64 n - 15, 64 n + 15]
  const std::uint32_t Bp = Lp >> 3, rmask = (1u << (Lp & 7)) - 1;
  std::uint32_t e = 0;  // root
#pragma unroll
  for (int j = 0; j < NB - 2; j += 2) {  // bytes before NB - 2 <= Bp: every word they complete is taken
    const std::uint32_t e1 = ft.entry(fsm_index(st[j >> 2], e, j));
    const std::uint32_t e2 = ft.entry(fsm_index(st[(j + 1) >> 2], e1, j + 1));
    sink.put2(e1, e2);
    e = e2;
  }
  // bytes NB - 2 .. NB + 1: whole before Bp; at Bp the words completing in
  // its first r bits (they end by Lp); after Bp none
  auto clip = [&](std::uint32_t ej, std::uint32_t idx, int j) -> std::uint32_t {
    const std::uint32_t lm = static_cast<std::uint32_t>(j) == Bp ? rmask : 0u;
    const std::uint32_t kept4 = 4u * __popc(ft.cm(idx) & lm);
    const std::uint32_t clipped = (ej & ((0x10000u << kept4) - 0x10000u)) | kept4;
    return static_cast<std::uint32_t>(j) < Bp ? ej : clipped;
  };
#pragma unroll
  for (int j = NB - 2; j < NB + 2; j += 2) {
    const std::uint32_t i1 = fsm_index(st[j >> 2], e, j);
    const std::uint32_t e1 = clip(ft.entry(i1), i1, j);
    const std::uint32_t i2 = fsm_index(st[(j + 1) >> 2], e1, j + 1);
    const std::uint32_t e2 = clip(ft.entry(i2), i2, j + 1);
    sink.put2(e1, e2);
    e = e2;
  }
}

// Two independent runs of decode_windows_fsm (NWIN windows each: words wa /
// wb, start gaps, recorded ends, sinks), their byte steps interleaved so
// both table-probe chains are in flight at once.
template <int NWIN = 4, int WS = 4, class FT = FsmPinned>
__device__ __forceinline__ void decode_two_fsm(const std::uint32_t* wa, std::uint32_t ga, std::uint32_t ea,
                                               PairSink<WS>& sa, const std::uint32_t* wb, std::uint32_t gb,
                                               std::uint32_t eb, PairSink<WS>& sb, const FT& ft = FT{}) {
  constexpr int NB = 8 * NWIN, NS = 2 * NWIN + 1;
  std::uint32_t sta[NS], stb[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    sta[i] = __funnelshift_l(wa[i + 1], wa[i], ga);
    stb[i] = __funnelshift_l(wb[i + 1], wb[i], gb);
  }
  const std::uint32_t LA = 64u * NWIN + ea - ga, LB = 64u * NWIN + eb - gb;
  const std::uint32_t BA = LA >> 3, rA = (1u << (LA & 7)) - 1, BB = LB >> 3, rB = (1u << (LB & 7)) - 1;
  std::uint32_t xa = 0, xb = 0;
#pragma unroll
  for (int j = 0; j < NB - 2; j += 2) {
    const std::uint32_t a1 = ft.entry(fsm_index(sta[j >> 2], xa, j));
    const std::uint32_t b1 = ft.entry(fsm_index(stb[j >> 2], xb, j));
    const std::uint32_t a2 = ft.entry(fsm_index(sta[(j + 1) >> 2], a1, j + 1));
    const std::uint32_t b2 = ft.entry(fsm_index(stb[(j + 1) >> 2], b1, j + 1));
    sa.put2(a1, a2);
    sb.put2(b1, b2);
    xa = a2;
    xb = b2;
  }
  auto clip = [&](std::uint32_t ej, std::uint32_t idx, int j, std::uint32_t Bp, std::uint32_t rmask) {
    const std::uint32_t lm = static_cast<std::uint32_t>(j) == Bp ? rmask : 0u;
    const std::uint32_t kept4 = 4u * __popc(ft.cm(idx) & lm);
    const std::uint32_t clipped = (ej & ((0x10000u << kept4) - 0x10000u)) | kept4;
    return static_cast<std::uint32_t>(j) < Bp ? ej : clipped;
  };
#pragma unroll
  for (int j = NB - 2; j < NB + 2; j += 2) {
    const std::uint32_t ia1 = fsm_index(sta[j >> 2], xa, j), ib1 = fsm_index(stb[j >> 2], xb, j);
    const std::uint32_t a1 = clip(ft.entry(ia1), ia1, j, BA, rA), b1 = clip(ft.entry(ib1), ib1, j, BB, rB);
    const std::uint32_t ia2 = fsm_index(sta[(j + 1) >> 2], a1, j + 1), ib2 = fsm_index(stb[(j + 1) >> 2], b1, j + 1);
    const std::uint32_t a2 = clip(ft.entry(ia2), ia2, j + 1, BA, rA), b2 = clip(ft.entry(ib2), ib2, j + 1, BB, rB);
    sa.put2(a1, a2);
    sb.put2(b1, b2);
    xa = a2;
    xb = b2;
  }
}

// One byte step of the 64-bit table (1-bit codes): up to 8 symbols (32
// bits) per byte; h = the entry's high word, n4 in bits 0..5 (<= 32), the
// state in bits 8..11.  q4 adds h whole: bits 0..4 stay exact and bit 5
// toggles when a word fills (n4 = 32 fills exactly one).
template <int WS>
__device__ __forceinline__ void put1(PairSink<WS>& k, std::uint32_t c, std::uint32_t h) {
  const std::uint32_t q = k.q4 + h;
  const std::uint32_t nl = k.lo | __funnelshift_l(0u, c, k.q4);
  const std::uint32_t nh = __funnelshift_l(c, 0u, k.q4);
  const bool full = ((q ^ k.q4) & 32u) != 0;
  if (full) sts32(k.addr, nl);
  k.addr += full ? WS : 0u;
  k.lo = full ? nh : nl;
  k.q4 = q;
}
template <int WS>
__device__ __forceinline__ void put1_bounded(PairSink<WS>& k, std::uint32_t c, std::uint32_t h, std::uint32_t ew,
                                             std::uint32_t& tail) {
  const std::uint32_t q = k.q4 + h;
  const std::uint32_t nl = k.lo | __funnelshift_l(0u, c, k.q4);
  const std::uint32_t nh = __funnelshift_l(c, 0u, k.q4);
  const bool full = ((q ^ k.q4) & 32u) != 0;
  if (full && k.addr < ew) sts32(k.addr, nl);
  if (full && k.addr == ew) tail = nl;
  k.addr += full ? WS : 0u;
  k.lo = full ? nh : nl;
  k.q4 = q;
}

// The 64-bit table staged in shared memory (address in a register).
struct Fsm64At {
  std::uint32_t tab;
  __device__ __forceinline__ uint2 entry(std::uint32_t idx) const {
    std::uint32_t a;
    uint2 v;
    asm("mad.lo.u32 %0, %1, 8, %2;" : "=r"(a) : "r"(idx), "r"(tab));
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
  }
};

// decode_two_fsm_counted with the 64-bit table: one byte per step (a byte
// can complete 8 one-bit words, 32 bits of symbols).
template <int NWIN = 4, int WS = 4>
__device__ __forceinline__ void decode_two_fsm64_counted(const std::uint32_t* wa, std::uint32_t ga, std::uint32_t ea,
                                                         PairSink<WS>& sa, std::uint32_t& ta, const std::uint32_t* wb,
                                                         std::uint32_t gb, std::uint32_t eb, PairSink<WS>& sb,
                                                         std::uint32_t& tb, std::uint32_t stage, const Fsm64At& ft) {
  constexpr int NB = 8 * NWIN, NS = 2 * NWIN + 1;
  std::uint32_t sta[NS], stb[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    sta[i] = __funnelshift_l(wa[i + 1], wa[i], ga);
    stb[i] = __funnelshift_l(wb[i + 1], wb[i], gb);
  }
  std::uint32_t ha = 0, hb = 0;  // previous entries' high words (state in byte 1; root = 0)
#pragma unroll
  for (int j = 0; j < NB - 2; ++j) {
    const uint2 a = ft.entry(fsm_index(sta[j >> 2], ha, j));
    const uint2 b = ft.entry(fsm_index(stb[j >> 2], hb, j));
    put1(sa, a.x, a.y);
    put1(sb, b.x, b.y);
    ha = a.y;
    hb = b.y;
  }
  const std::uint32_t ewa = stage + 4 * (ea >> 3), ewb = stage + 4 * (eb >> 3);
  ta = tb = 0;
#pragma unroll
  for (int j = NB - 2; j < NB + 2; ++j) {
    const uint2 a = ft.entry(fsm_index(sta[j >> 2], ha, j));
    const uint2 b = ft.entry(fsm_index(stb[j >> 2], hb, j));
    put1_bounded(sa, a.x, a.y, ewa, ta);
    put1_bounded(sb, b.x, b.y, ewb, tb);
    ha = a.y;
    hb = b.y;
  }
  if (sa.addr == ewa) ta = sa.lo;
  if (sb.addr == ewb) tb = sb.lo;
  ta &= (1u << (4 * (ea & 7))) - 1;
  tb &= (1u << (4 * (eb & 7))) - 1;
}

// decode_two_fsm for two runs whose symbol counts are known (the upload
// check's lane_start offsets): each run's stage nibbles [start, end) with
// end = ea / eb (absolute nibble positions, start = the sink's).  The byte
// steps run through all NWIN windows + the 2 lookahead bytes; the symbols
// the last 4 bytes complete past a run's end are dropped by position instead
// of by the completion masks (no fsm_cm probes, no popcounts).  Returns the
// end words' contents in ta / tb (the caller ORs them in, masked to the run).
template <int NWIN = 4, int WS = 4, class FT = FsmPinned>
__device__ __forceinline__ void decode_two_fsm_counted(const std::uint32_t* wa, std::uint32_t ga, std::uint32_t ea,
                                                       PairSink<WS>& sa, std::uint32_t& ta, const std::uint32_t* wb,
                                                       std::uint32_t gb, std::uint32_t eb, PairSink<WS>& sb,
                                                       std::uint32_t& tb, std::uint32_t stage, const FT& ft = FT{}) {
  constexpr int NB = 8 * NWIN, NS = 2 * NWIN + 1;
  std::uint32_t sta[NS], stb[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    sta[i] = __funnelshift_l(wa[i + 1], wa[i], ga);
    stb[i] = __funnelshift_l(wb[i + 1], wb[i], gb);
  }
  std::uint32_t xa = 0, xb = 0;
#pragma unroll
  for (int j = 0; j < NB - 2; j += 2) {  // every word these bytes complete belongs to the run
    const std::uint32_t a1 = ft.entry(fsm_index(sta[j >> 2], xa, j));
    const std::uint32_t b1 = ft.entry(fsm_index(stb[j >> 2], xb, j));
    const std::uint32_t a2 = ft.entry(fsm_index(sta[(j + 1) >> 2], a1, j + 1));
    const std::uint32_t b2 = ft.entry(fsm_index(stb[(j + 1) >> 2], b1, j + 1));
    sa.put2(a1, a2);
    sb.put2(b1, b2);
    xa = a2;
    xb = b2;
  }
  const std::uint32_t ewa = stage + 4 * (ea >> 3), ewb = stage + 4 * (eb >> 3);
  ta = tb = 0;
#pragma unroll
  for (int j = NB - 2; j < NB + 2; j += 2) {
    const std::uint32_t a1 = ft.entry(fsm_index(sta[j >> 2], xa, j));
    const std::uint32_t b1 = ft.entry(fsm_index(stb[j >> 2], xb, j));
    const std::uint32_t a2 = ft.entry(fsm_index(sta[(j + 1) >> 2], a1, j + 1));
    const std::uint32_t b2 = ft.entry(fsm_index(stb[(j + 1) >> 2], b1, j + 1));
    sa.put2_bounded(a1, a2, ewa, ta);
    sb.put2_bounded(b1, b2, ewb, tb);
    xa = a2;
    xb = b2;
  }
  if (sa.addr == ewa) ta = sa.lo;
  if (sb.addr == ewb) tb = sb.lo;
  ta &= (1u << (4 * (ea & 7))) - 1;  // the run's nibbles of its end word (none when it ends on a boundary)
  tb &= (1u << (4 * (eb & 7))) - 1;
}

// Where window (w0..w3, gap)'s reference walk stops: the start of the first
// code word at or after bit 64, relative to the window (codec.cpp:143-160 --
// the walk takes the words that start in [gap, 64)).  For a stream written
// by the encoder this is 64 + the next window's gap (codec.cpp:49-98).
// *count (optional): the words the walk takes (count_phase, codec.cpp:133-161).
template <class TV>
__device__ __forceinline__ std::uint32_t window_end(std::uint32_t w0, std::uint32_t w1, std::uint32_t w2,
                                                    std::uint32_t w3, std::uint32_t gap, const TV& tb,
                                                    std::uint32_t len_off, std::uint32_t* count = nullptr) {
  std::uint32_t hi = __funnelshift_l(w1, w0, gap);
  std::uint32_t lo = __funnelshift_l(w2, w1, gap);
  std::uint32_t p = gap, n4 = 0;
  while (p < 32) {
    std::uint32_t e = tb.fast(hi >> kFastShift);
    if (e & kSlowFlag) e = slow_entry(hi, tb, len_off);
    n4 += entry_n4(e);
    hi = __funnelshift_l(lo, hi, e);
    lo = __funnelshift_l(0u, lo, e);
    p += e & 31;
  }
  hi = __funnelshift_l(w2, w1, p - 32);
  lo = __funnelshift_l(w3, w2, p - 32);
  for (;;) {
    const std::uint32_t idx = hi >> kFastShift;
    std::uint32_t e = tb.fast(idx);
    const bool fast_hit = !(e & kSlowFlag);
    if (!fast_hit) e = slow_entry(hi, tb, len_off);
    const std::uint32_t b = e & 31, r = 64 - p;
    if (b >= r) {  // r <= 16 here
      const std::uint32_t st = fast_hit ? tb.smask(idx) : 1u;
      if (count) *count = (n4 >> 2) + __popc(st & ((1u << r) - 1));
      const std::uint32_t m = st >> r;
      return m ? 64 + __ffs(m) - 1 : p + b;
    }
    n4 += entry_n4(e);
    hi = __funnelshift_l(lo, hi, e);
    lo = __funnelshift_l(0u, lo, e);
    p += b;
  }
}

template <bool OR_BASE = false, class Sink, class TV>
__device__ __forceinline__ void decode_window(std::uint32_t w0, std::uint32_t w1, std::uint32_t w2,
                                              std::uint32_t w3, std::uint32_t gap, const TV& tb,
                                              std::uint32_t len_off, Sink& sink) {
  const Sink saved = sink;
  if (!decode_window_fast<Sink, OR_BASE>(w0, w1, w2, w3, gap, tb.fast_addr(), tb, sink)) {
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
#ifdef ECF8_MERGE_C
  const std::uint32_t even = sel(sel(S << 3, P, 0x78787878u), P >> 4, 0xF8F8F8F8u);
  const std::uint32_t odd = sel(sel(S >> 1, P << 4, 0x78787878u), P, 0xF8F8F8F8u);
#else
  // lop3 0xE4: (a & c) | (b & ~c) -- one select per mask, 10 instructions per 8 bytes
  std::uint32_t even, odd;
  asm("{\n\t.reg .b32 t, u;\n\t"
      "shl.b32 t, %2, 3;\n\t"
      "shr.b32 u, %3, 4;\n\t"
      "lop3.b32 t, t, u, 0x78787878, 0xE4;\n\t"
      "lop3.b32 %0, t, %3, 0x7F7F7F7F, 0xE4;\n\t"
      "shr.b32 t, %2, 1;\n\t"
      "shl.b32 u, %3, 4;\n\t"
      "lop3.b32 t, t, %3, 0x78787878, 0xE4;\n\t"
      "lop3.b32 %1, t, u, 0x7F7F7F7F, 0xE4;\n\t}"
      : "=r"(even), "=r"(odd)
      : "r"(S), "r"(P));
#endif
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
  const uint4* c4 = reinterpret_cast<const uint4*>(d.cascade);  // n_luts x 256 bytes, 16-byte aligned
  uint4* sc4 = reinterpret_cast<uint4*>(tb.cascade);
  for (int i = tid; i < static_cast<int>(d.n_luts) * 16; i += nthreads) sc4[i] = __ldg(c4 + i);
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
