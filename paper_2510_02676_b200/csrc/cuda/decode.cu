// decode.cu -- ECF8 -> FP8 decode kernels for sm_100a (B200).
//
// Replaces the reference's OpenMP block decoder
// (/root/reference/proj/src/codec.cpp:133-273: count_phase, Blelloch scan,
// emit_phase, staging copy) with a persistent CTA-per-SM kernel:
//
//   * a CTA owns a contiguous range of "tiles"; a tile is whole reference
//     blocks covering 256 * kwin windows (T <= 256: 256/T blocks, one window
//     per thread; T = 512/1024: one block, 2/4 windows per thread), so every
//     tile starts at an outpos[] boundary and needs nothing from neighbours;
//   * the tile's bitstream is staged to shared memory as big-endian 32-bit
//     words (16-byte vector loads), the decode tables once per tensor;
//   * pass 1 counts the words starting in each 64-bit window with the
//     multi-symbol table (tables.hpp), several symbols per shared load;
//   * a warp-shuffle + cross-warp scan of the counts, seeded by outpos[] per
//     reference block, gives each window its output offset; counts past a
//     block's outpos limit are clamped exactly as codec.cpp:239-246 does;
//   * pass 2 re-decodes and drops exponent bytes (x << 3) into a shared
//     staging tile;
//   * write-back merges staging with the sign/mantissa nibbles in SWAR form
//     and stores 16 output bytes per thread-iteration (edges byte-wise, so
//     neighbouring tiles never touch the same byte).
#include <cuda_runtime.h>

#include <cstdint>

#include "decode.cuh"
#include "tables.hpp"

namespace ecf8::dev {

namespace {

constexpr int kWarps = kThreads / 32;
constexpr int kFastShift = 32 - kFastBits;

template <int KWIN>
struct Smem {
  static constexpr int kWindows = kThreads * KWIN;
  static constexpr int kStreamWords = kWindows * 2 + 8;     // + lookahead / overread
  static constexpr int kStagingBytes = kWindows * 64 + 32;  // <= T*64 per block, +align
  std::uint32_t fast[kFastEntries];
  std::uint32_t stream[kStreamWords];
  std::uint64_t outpos[kThreads + 1];
  std::uint32_t prefix[kThreads];
  std::uint32_t warp_sum[kWarps];
  std::uint8_t cascade[18 * 256];
  alignas(16) std::uint8_t staging[kStagingBytes];
};

__device__ __forceinline__ std::uint32_t peek32(const std::uint32_t* sw, std::uint32_t p) {
  const std::uint32_t j = p >> 5;
  return __funnelshift_l(sw[j + 1], sw[j], p & 31);
}

struct Step {
  std::uint32_t sym, len;
};

// One reference decode_one at the head of x (top 16 bits), or the first
// symbol of a fast entry.
__device__ __forceinline__ Step single_step(std::uint32_t e, std::uint32_t n, std::uint32_t x,
                                            const std::uint8_t* casc, std::uint32_t n_luts,
                                            std::uint64_t lenpack) {
  Step s;
  if (n != 0) {
    s.sym = (e >> 8) & 15;
    const std::uint32_t l = static_cast<std::uint32_t>(lenpack >> (4 * s.sym)) & 15;
    s.len = l ? l : 16;
  } else {
    const std::uint32_t w = x >> 16;
    std::uint32_t v = casc[w >> 8];
    if (v >= 240) v = casc[((256u - v) << 8) | (w & 255u)];
    s.sym = v;
    s.len = casc[((n_luts - 1) << 8) + v];
  }
  return s;
}

// Words starting in [p, end): codec.cpp:133-161 semantics.
__device__ __forceinline__ std::uint32_t count_window(const std::uint32_t* sw, std::uint32_t p,
                                                      std::uint32_t end, const std::uint32_t* fast,
                                                      const std::uint8_t* casc,
                                                      std::uint32_t n_luts, std::uint64_t lenpack) {
  std::uint32_t c = 0;
  do {
    const std::uint32_t x = peek32(sw, p);
    const std::uint32_t e = fast[x >> kFastShift];
    const std::uint32_t b = e & 31, n = (e >> 5) & 7;
    if (n != 0 && p + b <= end) {
      c += n;
      p += b;
    } else {
      c += 1;
      p += single_step(e, n, x, casc, n_luts, lenpack).len;
    }
  } while (p < end);
  return c;
}

// codec.cpp:168-190: emit staging[q .. q_end) from bit p.
__device__ __forceinline__ void emit_window(const std::uint32_t* sw, std::uint32_t p,
                                            std::uint32_t q, std::uint32_t q_end,
                                            std::uint8_t* stage, const std::uint32_t* fast,
                                            const std::uint8_t* casc, std::uint32_t n_luts,
                                            std::uint64_t lenpack) {
  while (q < q_end) {
    const std::uint32_t x = peek32(sw, p);
    const std::uint32_t e = fast[x >> kFastShift];
    const std::uint32_t b = e & 31, n = (e >> 5) & 7;
    if (n != 0 && q + n <= q_end) {
      std::uint32_t syms = e >> 8;
      for (std::uint32_t i = 0; i < n; ++i, syms >>= 4) stage[q + i] = static_cast<std::uint8_t>((syms & 15) << 3);
      q += n;
      p += b;
    } else {
      const Step s = single_step(e, n, x, casc, n_luts, lenpack);
      stage[q++] = static_cast<std::uint8_t>(s.sym << 3);
      p += s.len;
    }
  }
}

// Exponent bytes (x << 3) merged with four sign/mantissa nibbles taken from
// two packed bytes (element 2i in the high half).  v = [q0, q0, q1, q1].
__device__ __forceinline__ std::uint32_t merge4(std::uint32_t xbytes, std::uint32_t v) {
  return xbytes | (v & 0x00800080u) | ((v >> 4) & 0x00070007u) | ((v << 4) & 0x80008000u) |
         (v & 0x07000700u);
}

__device__ __forceinline__ std::uint8_t merge1(std::uint8_t xbyte, std::uint8_t qb, std::uint64_t i) {
  const std::uint32_t qh = (i & 1) ? (static_cast<std::uint32_t>(qb) << 4) : qb;
  return static_cast<std::uint8_t>(xbyte | (qh & 0x80u) | ((qh >> 4) & 7u));
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
  const TensorDesc* __restrict__ descs = args.descs;
  const int n_desc = args.n_desc;
  const std::uint64_t total_tiles = args.total_tiles;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<KWIN>& sm = *reinterpret_cast<Smem<KWIN>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // Contiguous tile range per CTA: few tensor switches, tables reused.
  const std::uint64_t t_lo = total_tiles * blockIdx.x / gridDim.x;
  const std::uint64_t t_hi = total_tiles * (blockIdx.x + 1) / gridDim.x;
  int di = -1;
  std::uint64_t next_begin = 0;
  TensorDesc d;

  for (std::uint64_t tile = t_lo; tile < t_hi; ++tile) {
    if (di < 0 || tile >= next_begin) {
      if (descs) {
        di = find_desc(descs, n_desc, tile);
        d = descs[di];
        next_begin = (di + 1 < n_desc) ? descs[di + 1].tile_begin : total_tiles;
      } else {
        di = 0;
        d = args.inline_desc;
        next_begin = total_tiles;
      }
      __syncthreads();  // previous tile done with the old tables
      for (int i = tid; i < kFastEntries; i += kThreads) sm.fast[i] = d.fast[i];
      for (int i = tid; i < static_cast<int>(d.n_luts) * 256; i += kThreads) sm.cascade[i] = d.cascade[i];
    }
    const std::uint32_t T = d.T;
    const std::uint32_t m = T >= 256 ? 1u : 256u / T;
    const std::uint64_t b0 = d.blk_begin + (tile - d.tile_begin) * m;
    const std::uint32_t nblk = static_cast<std::uint32_t>(d.blk_end - b0 < m ? d.blk_end - b0 : m);
    const std::uint32_t nwin = nblk * T;
    const std::uint64_t w0 = b0 * T;

    // ---- stage bitstream words and block offsets
    {
      const uint4* src = reinterpret_cast<const uint4*>(d.encoded + w0 * 8);
      const std::uint32_t nvec = (nwin * 8 + 16 + 15) / 16;
      for (std::uint32_t v = tid; v < nvec; v += kThreads) {
        const uint4 q = __ldg(src + v);
        sm.stream[4 * v + 0] = __byte_perm(q.x, 0, 0x0123);
        sm.stream[4 * v + 1] = __byte_perm(q.y, 0, 0x0123);
        sm.stream[4 * v + 2] = __byte_perm(q.z, 0, 0x0123);
        sm.stream[4 * v + 3] = __byte_perm(q.w, 0, 0x0123);
      }
      for (std::uint32_t i = tid; i <= nblk; i += kThreads) sm.outpos[i] = d.outpos[b0 + i];
    }
    __syncthreads();

    // ---- pass 1: per-window counts
    std::uint32_t cnt[KWIN];
    std::uint32_t total = 0;
#pragma unroll
    for (int i = 0; i < KWIN; ++i) {
      const std::uint32_t wl = tid * KWIN + i;
      cnt[i] = 0;
      if (wl < nwin) {
        const std::uint64_t wg = w0 + wl;
        const std::uint32_t gap = (d.gaps[wg >> 1] >> ((wg & 1) ? 0 : 4)) & 15;
        cnt[i] = count_window(sm.stream, wl * 64 + gap, wl * 64 + 64, sm.fast, sm.cascade,
                              d.n_luts, d.lenpack);
      }
      total += cnt[i];
    }

    // ---- exclusive scan of per-thread totals (warp shuffles + warp sums)
    std::uint32_t incl = total;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) sm.warp_sum[warp] = incl;
    __syncthreads();
    std::uint32_t warp_base = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) warp_base += (w < warp) ? sm.warp_sum[w] : 0u;
    const std::uint32_t excl = warp_base + incl - total;
    sm.prefix[tid] = excl;
    __syncthreads();

    // ---- pass 2: emit exponent bytes into staging
    const std::uint64_t A = sm.outpos[0];
    const std::uint64_t S0 = A & ~std::uint64_t{15};
    {
      std::uint32_t run = excl;
#pragma unroll
      for (int i = 0; i < KWIN; ++i) {
        const std::uint32_t wl = tid * KWIN + i;
        if (wl < nwin && cnt[i] != 0) {
          const std::uint32_t bl = wl / T;
          const std::uint64_t base = sm.outpos[bl];
          const std::uint64_t lim = sm.outpos[bl + 1];
          const std::uint64_t o_start = base + run - sm.prefix[(bl * T) / KWIN];
          if (o_start < lim) {
            const std::uint64_t o_end = o_start + cnt[i] < lim ? o_start + cnt[i] : lim;
            const std::uint64_t wg = w0 + wl;
            const std::uint32_t gap = (d.gaps[wg >> 1] >> ((wg & 1) ? 0 : 4)) & 15;
            emit_window(sm.stream, wl * 64 + gap, static_cast<std::uint32_t>(o_start - S0),
                        static_cast<std::uint32_t>(o_end - S0), sm.staging, sm.fast, sm.cascade,
                        d.n_luts, d.lenpack);
          }
        }
        run += cnt[i];
      }
    }
    __syncthreads();

    // ---- write-back: staging + nibbles -> FP8 bytes, 16 per step
    {
      const std::uint64_t E = sm.outpos[nblk];
      const std::uint64_t nchunk = (E - S0 + 15) / 16;
      std::uint8_t* out = d.out;
      for (std::uint64_t ci = tid; ci < nchunk; ci += kThreads) {
        const std::uint64_t g = S0 + 16 * ci;
        if (g >= A && g + 16 <= E) {
          const uint4 xs = *reinterpret_cast<const uint4*>(sm.staging + (g - S0));
          const uint2 q = __ldg(reinterpret_cast<const uint2*>(d.packed + g / 2));
          uint4 r;
          r.x = merge4(xs.x, __byte_perm(q.x, 0, 0x1100));
          r.y = merge4(xs.y, __byte_perm(q.x, 0, 0x3322));
          r.z = merge4(xs.z, __byte_perm(q.y, 0, 0x1100));
          r.w = merge4(xs.w, __byte_perm(q.y, 0, 0x3322));
          *reinterpret_cast<uint4*>(out + (g - d.out_offset)) = r;
        } else {
          const std::uint64_t lo = g < A ? A : g;
          const std::uint64_t hi = g + 16 < E ? g + 16 : E;
          for (std::uint64_t i = lo; i < hi; ++i)
            out[i - d.out_offset] = merge1(sm.staging[i - S0], d.packed[i >> 1], i);
        }
      }
    }
    __syncthreads();
  }
}

__global__ void count_window_kernel(const std::uint8_t* w16, unsigned gap, const std::uint32_t* fast,
                                    const std::uint8_t* casc, std::uint32_t n_luts,
                                    std::uint64_t lenpack, std::uint32_t* out) {
  __shared__ std::uint32_t sw[8];
  __shared__ std::uint32_t sfast[kFastEntries];
  __shared__ std::uint8_t scasc[18 * 256];
  for (int i = threadIdx.x; i < kFastEntries; i += blockDim.x) sfast[i] = fast[i];
  for (int i = threadIdx.x; i < static_cast<int>(n_luts) * 256; i += blockDim.x) scasc[i] = casc[i];
  if (threadIdx.x < 8) {
    std::uint32_t v = 0;
    for (int k = 0; k < 4; ++k) {
      const int idx = 4 * threadIdx.x + k;
      v = (v << 8) | (idx < 10 ? w16[idx] : 0u);  // only the 10 window bytes exist
    }
    sw[threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) *out = count_window(sw, gap, 64, sfast, scasc, n_luts, lenpack);
}

template <int KWIN>
cudaError_t launch_k(const LaunchArgs& args, cudaStream_t s) {
  const std::uint64_t total_tiles = args.total_tiles;
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
  const std::uint64_t grid = total_tiles < static_cast<std::uint64_t>(grid_cap) ? total_tiles : grid_cap;
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
                                const std::uint8_t* d_cascade, std::uint32_t n_luts,
                                std::uint64_t lenpack, std::uint32_t* d_count, cudaStream_t stream) {
  count_window_kernel<<<1, 128, 0, stream>>>(d_window16, gap, d_fast, d_cascade, n_luts, lenpack, d_count);
  return cudaGetLastError();
}

}  // namespace ecf8::dev
