// decode.cu -- ECF8 -> FP8 decode kernels for sm_100a (B200).
//
// Replaces the reference's OpenMP block decoder
// (/root/reference/proj/src/codec.cpp:133-273: count_phase, Blelloch scan,
// emit_phase, staging copy).  The reference decodes every symbol twice
// (count, then emit); this kernel decodes once:
//
//   * persistent CTAs, each owning a contiguous run of "tiles"; a tile is
//     whole reference blocks covering 256 * KWIN windows (T <= 256: 256/T
//     blocks, one window per thread; T = 512/1024: one block, 2/4 windows per
//     thread), so a tile starts at an outpos[] boundary;
//   * decode tables (tables.hpp) live in shared memory per tensor;
//   * each thread pulls its window bits straight into registers (two 8-byte
//     loads, coalesced across the warp) and walks them with a 64-bit register
//     window, up to five symbols per table load; the symbols that start
//     before the window's 64-bit boundary are taken exactly, the last entry
//     partially via a start-bit mask + popcount (codec.cpp:143-160 rule);
//     symbols are packed as nibbles into a private shared-memory slot;
//   * a warp-shuffle + cross-warp scan of the per-thread counts, seeded by
//     outpos[] per reference block, gives every thread its output offset;
//     counts past a block's outpos limit are clamped (codec.cpp:239-246);
//   * each thread copies its nibbles to their final place in a nibble
//     staging tile (funnel shifts, whole words); words shared by
//     neighbouring threads are assembled by one owner from published
//     partial words -- no atomics;
//   * write-back merges exponent nibbles with the sign/mantissa nibbles in
//     SWAR form and stores 16 bytes per thread-step; tile edges are written
//     byte-wise so neighbouring tiles never touch the same byte.
#include <cuda_runtime.h>

#include <cstdint>

#include "decode.cuh"
#include "tables.hpp"

namespace ecf8::dev {

namespace {

constexpr int kWarps = kThreads / 32;
constexpr int kFastShift = 32 - kFastBits;

struct Tables {
  std::uint32_t fast[kFastEntries];
  std::uint16_t smask[kFastEntries];
  std::uint8_t cascade[18 * 256];
};

template <int KWIN>
struct Smem {
  static constexpr int kSlotStride = KWIN * 8 + 1;             // words; odd => no bank conflicts
  static constexpr int kStageWords = KWIN * kThreads * 8 + 8;  // tile nibbles + 16-nibble slack
  Tables tb;
  std::uint32_t slot[kThreads * kSlotStride];
  alignas(16) std::uint32_t stage[kStageWords];
  std::uint32_t rs[kThreads];
  std::uint32_t re[kThreads];
  std::uint32_t head[kThreads];
  std::uint32_t excl[kThreads];
  std::uint32_t blk[kThreads + 1];
  std::uint32_t warp_sum[kWarps];
};

// ---------------------------------------------------------------- sinks

// Packs 4-bit symbols into consecutive 32-bit words (first symbol lowest).
struct SlotSink {
  std::uint32_t* ptr;
  std::uint32_t lo = 0;  // partial word
  std::uint32_t q4 = 0;  // bits used in lo, < 32
  __device__ __forceinline__ void put(std::uint32_t syms, std::uint32_t n4) {
    const std::uint32_t nl = lo | (syms << q4);
    const std::uint32_t nh = __funnelshift_l(syms, 0u, q4);
    q4 += n4;
    if (q4 >= 32) {
      *ptr++ = nl;
      lo = nh;
      q4 -= 32;
    } else {
      lo = nl;
    }
  }
};

struct CountSink {
  std::uint32_t n4 = 0;
  __device__ __forceinline__ void put(std::uint32_t, std::uint32_t k4) { n4 += k4; }
};

// The reference cascade (lut.hpp:43-49) on a 16-bit window: symbol.
__device__ __forceinline__ std::uint32_t cascade_symbol(std::uint32_t w16, const Tables& tb) {
  std::uint32_t v = tb.cascade[w16 >> 8];
  if (v >= 240) v = tb.cascade[((256u - v) << 8) | (w16 & 255u)];
  return v;
}

// Decodes the words that start in [gap, 64) of one 64-bit window
// (codec.cpp:133-190 semantics); w0..w3 = window bits 0..127, big-endian.
template <class Sink>
__device__ __forceinline__ void decode_window(std::uint32_t w0, std::uint32_t w1, std::uint32_t w2,
                                              std::uint32_t w3, std::uint32_t gap,
                                              const Tables& tb, std::uint32_t len_off,
                                              Sink& sink) {
  std::uint32_t hi = __funnelshift_l(w1, w0, gap);
  std::uint32_t lo = __funnelshift_l(w2, w1, gap);
  std::uint32_t p = gap;
  // Phase A: at least 32 valid bits remain in the register window.
  while (p < 32) {
    const std::uint32_t e = tb.fast[hi >> kFastShift];
    const std::uint32_t n4 = (e >> 5) & 31;
    std::uint32_t adv;
    if (n4) {
      sink.put(e >> 12, n4);
      adv = e & 31;
    } else {
      const std::uint32_t v = cascade_symbol(hi >> 16, tb);
      sink.put(v, 4);
      adv = tb.cascade[len_off + v];
    }
    hi = __funnelshift_l(lo, hi, adv);
    lo = __funnelshift_l(0u, lo, adv);
    p += adv;
  }
  // Refill once: p in [32, 48); window = bits [p, p + 64).
  hi = __funnelshift_l(w2, w1, p - 32);
  lo = __funnelshift_l(w3, w2, p - 32);
  for (;;) {
    const std::uint32_t idx = hi >> kFastShift;
    const std::uint32_t e = tb.fast[idx];
    const std::uint32_t n4 = (e >> 5) & 31;
    const std::uint32_t r = 64 - p;  // bits left before the window boundary
    if (n4 == 0) {
      const std::uint32_t v = cascade_symbol(hi >> 16, tb);
      sink.put(v, 4);
      const std::uint32_t len = tb.cascade[len_off + v];
      p += len;
      if (p >= 64) break;
      hi = __funnelshift_l(lo, hi, len);
      lo = __funnelshift_l(0u, lo, len);
      continue;
    }
    const std::uint32_t b = e & 31;
    if (b >= r) {  // last entry: only the symbols that start before bit 64
      const std::uint32_t k4 = 4 * __popc(tb.smask[idx] & ((1u << r) - 1));
      sink.put((e >> 12) & ((1u << k4) - 1), k4);
      break;
    }
    sink.put(e >> 12, n4);
    hi = __funnelshift_l(lo, hi, e);  // shift amount = e & 31 = b
    lo = __funnelshift_l(0u, lo, e);
    p += b;
  }
}

__device__ __forceinline__ std::uint32_t bswap32(std::uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__device__ __forceinline__ std::uint32_t sel(std::uint32_t a, std::uint32_t b, std::uint32_t m) {
  return (a & m) | (b & ~m);
}

// Eight FP8 bytes from eight exponent nibbles S (element i at bits 4i..4i+3)
// and four packed sign/mantissa bytes P (element 2j in the high nibble of
// byte j): byte = sign << 7 | exponent << 3 | mantissa.
__device__ __forceinline__ void merge8(std::uint32_t S, std::uint32_t P, std::uint32_t& o0,
                                       std::uint32_t& o1) {
  const std::uint32_t even = sel(sel(S << 3, P, 0x78787878u), P >> 4, 0xF8F8F8F8u);
  const std::uint32_t odd = sel(sel(S >> 1, P << 4, 0x78787878u), P, 0xF8F8F8F8u);
  o0 = __byte_perm(even, odd, 0x5140);
  o1 = __byte_perm(even, odd, 0x7362);
}

__device__ __forceinline__ std::uint8_t merge1(std::uint32_t x, std::uint32_t qb, std::uint64_t i) {
  const std::uint32_t qh = (i & 1) ? (qb << 4) : qb;
  return static_cast<std::uint8_t>((x << 3) | (qh & 0x80u) | ((qh >> 4) & 7u));
}

__device__ __forceinline__ std::uint32_t nib_mask(std::uint32_t lo_n, std::uint32_t hi_n) {
  const std::uint32_t top = hi_n >= 8 ? 0xFFFFFFFFu : ((1u << (4 * hi_n)) - 1);
  return top & ~((1u << (4 * lo_n)) - 1);
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

template <int KWIN>
__global__ void __launch_bounds__(kThreads) decode_kernel(const LaunchArgs args) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<KWIN>& sm = *reinterpret_cast<Smem<KWIN>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const std::uint64_t total_tiles = args.total_tiles;

  const std::uint64_t t_lo = total_tiles * blockIdx.x / gridDim.x;
  const std::uint64_t t_hi = total_tiles * (blockIdx.x + 1) / gridDim.x;
  int di = -1;
  std::uint64_t next_begin = 0;
  TensorDesc d;
  std::uint32_t len_off = 0;

  for (std::uint64_t tile = t_lo; tile < t_hi; ++tile) {
    if (di < 0 || tile >= next_begin) {
      if (args.descs) {
        di = find_desc(args.descs, args.n_desc, tile);
        d = args.descs[di];
        next_begin = (di + 1 < args.n_desc) ? args.descs[di + 1].tile_begin : total_tiles;
      } else {
        di = 0;
        d = args.inline_desc;
        next_begin = total_tiles;
      }
      __syncthreads();  // everyone is past the previous tile's decode
      const uint4* f4 = reinterpret_cast<const uint4*>(d.fast);
      uint4* sf4 = reinterpret_cast<uint4*>(sm.tb.fast);
      for (int i = tid; i < kFastEntries / 4; i += kThreads) sf4[i] = __ldg(f4 + i);
      const uint4* m4 = reinterpret_cast<const uint4*>(d.smask);
      uint4* sm4 = reinterpret_cast<uint4*>(sm.tb.smask);
      for (int i = tid; i < kFastEntries / 8; i += kThreads) sm4[i] = __ldg(m4 + i);
      for (int i = tid; i < static_cast<int>(d.n_luts) * 256; i += kThreads) sm.tb.cascade[i] = d.cascade[i];
      len_off = (d.n_luts - 1) << 8;
      __syncthreads();
    }
    const std::uint32_t T = d.T;
    const std::uint32_t m = T >= 256 ? 1u : 256u / T;
    const std::uint64_t b0 = d.blk_begin + (tile - d.tile_begin) * m;
    const std::uint32_t nblk = static_cast<std::uint32_t>(d.blk_end - b0 < m ? d.blk_end - b0 : m);
    const std::uint32_t nwin = nblk * T;
    const std::uint64_t w0g = b0 * T;
    const std::uint64_t A = __ldg(d.outpos + b0);
    const std::uint64_t E = __ldg(d.outpos + b0 + nblk);
    for (std::uint32_t i = tid; i <= nblk; i += kThreads)
      sm.blk[i] = static_cast<std::uint32_t>(__ldg(d.outpos + b0 + i) - A);

    // ---- decode my windows into my slot
    std::uint32_t* const my_slot = sm.slot + tid * Smem<KWIN>::kSlotStride;
    SlotSink sink{my_slot};
#pragma unroll
    for (int i = 0; i < KWIN; ++i) {
      const std::uint32_t wl = tid * KWIN + i;
      if (wl < nwin) {
        const std::uint64_t wg = w0g + wl;
        const uint2 a = __ldg(reinterpret_cast<const uint2*>(d.encoded + 8 * wg));
        const uint2 b = __ldg(reinterpret_cast<const uint2*>(d.encoded + 8 * wg + 8));
        const std::uint32_t gap = (__ldg(d.gaps + (wg >> 1)) >> ((wg & 1) ? 0 : 4)) & 15u;
        decode_window(bswap32(a.x), bswap32(a.y), bswap32(b.x), bswap32(b.y), gap, sm.tb, len_off, sink);
      }
    }
    if (sink.q4) *sink.ptr = sink.lo;
    const std::uint32_t cnt = static_cast<std::uint32_t>(sink.ptr - my_slot) * 8 + (sink.q4 >> 2);

    // ---- exclusive scan of the per-thread counts
    std::uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) sm.warp_sum[warp] = incl;
    __syncthreads();
    std::uint32_t excl = incl - cnt;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) excl += (w < warp) ? sm.warp_sum[w] : 0u;
    sm.excl[tid] = excl;
    __syncthreads();

    // ---- my output range, clamped to my reference block's outpos limit
    const std::uint32_t bl = (T < 256) ? static_cast<std::uint32_t>(tid) / T : 0u;
    const std::uint32_t first = (T < 256) ? sm.excl[bl * T] : 0u;
    const std::uint32_t start_rel = sm.blk[bl] + excl - first;
    const std::uint32_t lim_rel = sm.blk[bl + 1];
    std::uint32_t cc = 0;
    if (static_cast<std::uint32_t>(tid) * KWIN < nwin && start_rel < lim_rel)
      cc = min(cnt, lim_rel - start_rel);
    const std::uint32_t off = static_cast<std::uint32_t>(A & 15);  // staging nibble of element A
    const std::uint32_t d0 = start_rel + off, dend = d0 + cc;
    const std::uint32_t data_end = off + static_cast<std::uint32_t>(E - A);
    sm.rs[tid] = d0;
    sm.re[tid] = dend;

    // ---- copy my nibbles to their final place; publish partial words
    std::uint32_t headv = 0, tailv = 0;
    const std::uint32_t fw = d0 >> 3, lw = (dend - 1) >> 3;
    if (cc) {
      const std::uint32_t f4 = (d0 & 7) * 4;
      std::uint32_t prev = 0;
      for (std::uint32_t k = fw; k <= lw; ++k) {
        const std::uint32_t cur = my_slot[k - fw];
        std::uint32_t v = __funnelshift_l(prev, cur, f4);
        prev = cur;
        const std::uint32_t lo_n = (k == fw) ? (d0 & 7) : 0u;
        const std::uint32_t hi_n = (k == lw) ? ((dend - 1) & 7) + 1 : 8u;
        v &= nib_mask(lo_n, hi_n);
        if (lo_n == 0 && hi_n == 8) sm.stage[k] = v;
        else if (k == fw) headv = v;
        else tailv = v;
      }
    }
    sm.head[tid] = headv;
    __syncthreads();

    // ---- owners assemble words shared between threads
    if (cc) {
      const bool starts_fw = ((d0 & 7) == 0) || (d0 == off);
      const bool fw_full = ((d0 & 7) == 0) && (dend >= 8 * fw + 8);
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        std::uint32_t k, v;
        if (pass == 0) {
          if (!starts_fw || fw_full) continue;
          k = fw;
          v = headv;
        } else {
          if (lw == fw || (dend & 7) == 0) continue;
          k = lw;
          v = tailv;
        }
        const std::uint32_t wend = min(8 * k + 8, data_end);
        std::uint32_t covered = dend;
        for (int j = tid + 1; covered < wend && j < kThreads; ++j) {
          if (sm.re[j] > sm.rs[j]) {
            v |= sm.head[j];
            covered = sm.re[j];
          }
        }
        sm.stage[k] = v;
      }
    }
    __syncthreads();

    // ---- write-back: exponent nibbles + sign/mantissa nibbles -> FP8 bytes
    {
      const std::uint64_t S0 = A - off;
      const std::uint32_t nchunk = (data_end + 15) >> 4;
      std::uint8_t* out = d.out;
      for (std::uint32_t ci = tid; ci < nchunk; ci += kThreads) {
        const std::uint64_t g = S0 + 16ull * ci;
        if (g >= A && g + 16 <= E) {
          const uint2 s = *reinterpret_cast<const uint2*>(sm.stage + 2 * ci);
          const uint2 q = __ldg(reinterpret_cast<const uint2*>(d.packed + (g >> 1)));
          uint4 r;
          merge8(s.x, q.x, r.x, r.y);
          merge8(s.y, q.y, r.z, r.w);
          *reinterpret_cast<uint4*>(out + (g - d.out_offset)) = r;
        } else {
          const std::uint64_t lo = g < A ? A : g;
          const std::uint64_t hi = g + 16 < E ? g + 16 : E;
          for (std::uint64_t i = lo; i < hi; ++i) {
            const std::uint32_t nidx = static_cast<std::uint32_t>(i - S0);
            const std::uint32_t x = (sm.stage[nidx >> 3] >> (4 * (nidx & 7))) & 15u;
            out[i - d.out_offset] = merge1(x, d.packed[i >> 1], i);
          }
        }
      }
    }
  }
}

__global__ void count_window_kernel(const std::uint8_t* w16, unsigned gap, const std::uint32_t* fast,
                                    const std::uint16_t* smask, const std::uint8_t* casc,
                                    std::uint32_t n_luts, std::uint32_t* out) {
  __shared__ Tables tb;
  for (int i = threadIdx.x; i < kFastEntries; i += blockDim.x) {
    tb.fast[i] = fast[i];
    tb.smask[i] = smask[i];
  }
  for (int i = threadIdx.x; i < static_cast<int>(n_luts) * 256; i += blockDim.x) tb.cascade[i] = casc[i];
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
    decode_window(w[0], w[1], w[2], w[3], gap & 15u, tb, (n_luts - 1) << 8, c);
    *out = c.n4 >> 2;
  }
}

template <int KWIN>
cudaError_t launch_k(const LaunchArgs& args, cudaStream_t s) {
  static int grid_cap = 0;
  const int smem = static_cast<int>(sizeof(Smem<KWIN>));
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<KWIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<KWIN>, kThreads, smem);
    if (e != cudaSuccess) return e;
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const std::uint64_t total = args.total_tiles;
  const std::uint64_t grid = total < static_cast<std::uint64_t>(grid_cap) ? total : grid_cap;
  if (grid == 0) return cudaSuccess;
  decode_kernel<KWIN><<<static_cast<unsigned>(grid), kThreads, smem, s>>>(args);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_decode(const LaunchArgs& args, int kwin, cudaStream_t stream) {
  switch (kwin) {
    case 1: return launch_k<1>(args, stream);
    case 2: return launch_k<2>(args, stream);
    case 4: return launch_k<4>(args, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_count_window(const std::uint8_t* d_window16, unsigned gap, const std::uint32_t* d_fast,
                                const std::uint16_t* d_smask, const std::uint8_t* d_cascade,
                                std::uint32_t n_luts, std::uint32_t* d_count, cudaStream_t stream) {
  count_window_kernel<<<1, 128, 0, stream>>>(d_window16, gap, d_fast, d_smask, d_cascade, n_luts, d_count);
  return cudaGetLastError();
}

}  // namespace ecf8::dev
