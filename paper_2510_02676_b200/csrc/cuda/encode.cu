// encode.cu -- the ECF8 encoder and the exponent histogram on the device
// (SURVEY §8f row 4).  Byte-identical to the host encoder
// (csrc/host/codec.cpp: encode, restating codec.cpp:49-98):
//   * codes concatenated MSB-first from bit 0, tail zero-padded;
//   * gap of window w = in-window start bit of the first code that starts
//     in w (0 when none does), even window in the high nibble;
//   * outpos[b+1] = number of codes that start in windows of blocks <= b;
//   * packed = sign/mantissa nibbles, element 2i in the high half.
// Three passes: per-chunk code bits, one scan of the chunk sizes (the host
// reads the total to size the arena), then the emit pass, where each CTA
// builds its chunk's bit run in shared memory and writes it out with plain
// stores (interior words) and atomicOr (the two words it may share with
// the neighbouring chunks).
#include "encode.cuh"

#include <algorithm>

namespace ecf8::dev {
namespace {

constexpr int kEncThreads = 256;
constexpr int kPerThread = kEncChunkElems / kEncThreads;  // 16
static_assert(kPerThread == 16, "one uint4 of input per thread");

__device__ __forceinline__ std::uint32_t exp_of(std::uint32_t b) { return (b >> 3) & 15u; }
__device__ __forceinline__ std::uint32_t nib_of(std::uint32_t b) { return (b & 7u) | ((b & 0x80u) >> 4); }

// Up to 16 bytes of fp8 from element e0 (cnt valid, the rest 0).
__device__ __forceinline__ void load16(const std::uint8_t* fp8, std::uint64_t e0, std::uint32_t cnt,
                                       std::uint8_t (&x)[16]) {
  if (cnt == 16 && ((reinterpret_cast<std::uintptr_t>(fp8 + e0) & 15) == 0)) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(fp8 + e0));
    const std::uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = static_cast<std::uint8_t>(w[j >> 2] >> (8 * (j & 3)));
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = j < static_cast<int>(cnt) ? fp8[e0 + j] : 0;
  }
}

// Block-wide exclusive scan of one u32 per thread; *total = block sum.
__device__ __forceinline__ std::uint32_t block_excl_scan(std::uint32_t v, std::uint32_t* wsum,
                                                         std::uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint32_t inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const std::uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  std::uint32_t base = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kEncThreads / 32; ++w) {
    const std::uint32_t s = wsum[w];
    base += w < warp ? s : 0;
    all += s;
  }
  *total = all;
  return base + inc - v;
}

__global__ void __launch_bounds__(256) histogram_kernel(const std::uint8_t* __restrict__ fp8, std::uint64_t n,
                                                        unsigned long long* __restrict__ counts) {
  __shared__ std::uint32_t cnt[16 * 256];  // thread t's bin e at [e*256 + t]: conflict-free
  const std::uint32_t t = threadIdx.x;
#pragma unroll
  for (int e = 0; e < 16; ++e) cnt[e * 256 + t] = 0;
  const std::uint64_t n16 = (n + 15) / 16;
  for (std::uint64_t i = blockIdx.x * 256ull + t; i < n16; i += gridDim.x * 256ull) {
    const std::uint64_t e0 = i * 16;
    const std::uint32_t c = static_cast<std::uint32_t>(n - e0 < 16 ? n - e0 : 16);
    std::uint8_t x[16];
    load16(fp8, e0, c, x);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < static_cast<int>(c)) ++cnt[exp_of(x[j]) * 256 + t];
  }
  __syncthreads();
  // 16 bins x 256 partials: warp w sums bins 2w, 2w+1
  const int lane = t & 31, warp = t >> 5;
  for (int e = 2 * warp; e < 2 * warp + 2; ++e) {
    std::uint32_t s = 0;
    for (int k = lane; k < 256; k += 32) s += cnt[e * 256 + k];
#pragma unroll
    for (int d = 16; d; d >>= 1) s += __shfl_down_sync(0xffffffffu, s, d);
    if (lane == 0 && s) atomicAdd(&counts[e], static_cast<unsigned long long>(s));
  }
}

__global__ void __launch_bounds__(256) chunk_bits_kernel(const std::uint8_t* __restrict__ fp8, std::uint64_t n,
                                                         const std::uint8_t* __restrict__ lengths16,
                                                         std::uint32_t* __restrict__ chunk_bits,
                                                         std::uint32_t* __restrict__ bad) {
  __shared__ std::uint32_t s_len[16];
  __shared__ std::uint32_t wsum[8];
  if (threadIdx.x < 16) s_len[threadIdx.x] = lengths16[threadIdx.x];
  __syncthreads();
  const std::uint64_t e_begin = blockIdx.x * static_cast<std::uint64_t>(kEncChunkElems);
  const std::uint64_t e0 = e_begin + kPerThread * threadIdx.x;
  const std::uint32_t cnt = e0 < n ? static_cast<std::uint32_t>(n - e0 < 16 ? n - e0 : 16) : 0;
  std::uint8_t x[16];
  load16(fp8, e0, cnt, x);
  std::uint32_t bits = 0, missing = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < static_cast<int>(cnt)) {
      const std::uint32_t l = s_len[exp_of(x[j])];
      bits += l;
      missing |= l == 0;
    }
  }
  if (missing) atomicOr(bad, 1u);
  std::uint32_t total;
  (void)block_excl_scan(bits, wsum, &total);
  if (threadIdx.x == 0) chunk_bits[blockIdx.x] = total;
}

// One CTA: exclusive scan of the chunk sizes (u64 running carry).
__global__ void __launch_bounds__(1024) chunk_scan_kernel(const std::uint32_t* __restrict__ chunk_bits,
                                                          std::uint64_t n_chunks,
                                                          std::uint64_t* __restrict__ chunk_start,
                                                          unsigned long long* __restrict__ total) {
  __shared__ std::uint64_t wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint64_t carry = 0;
  for (std::uint64_t base = 0; base < n_chunks; base += 1024) {
    const std::uint64_t i = base + threadIdx.x;
    const std::uint64_t v = i < n_chunks ? chunk_bits[i] : 0;
    std::uint64_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const std::uint64_t o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += o;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    std::uint64_t before = 0, all = 0;
    for (int w = 0; w < 32; ++w) {
      before += w < warp ? wsum[w] : 0;
      all += wsum[w];
    }
    if (i < n_chunks) chunk_start[i] = carry + before + inc - v;
    carry += all;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(256) encode_emit_kernel(const EncodeArgs a) {
  constexpr int kWords = (kEncChunkElems * 16 + 31) / 32 + 2;  // the chunk's bit run + misalignment
  __shared__ std::uint32_t run[kWords];
  __shared__ std::uint32_t s_lc[16];  // code MSB-aligned | length (low 5 bits: the code is <= 16 bits)
  __shared__ std::uint32_t wsum[8];
  const std::uint32_t t = threadIdx.x;
  if (t < 16) {
    std::uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i)  // static indices: the parameter array stays in param space
      if (static_cast<int>(t) == i) v = a.lc[i];
    s_lc[t] = v;
  }
  for (int i = t; i < kWords; i += kEncThreads) run[i] = 0;
  const std::uint64_t e_begin = blockIdx.x * static_cast<std::uint64_t>(kEncChunkElems);
  const std::uint64_t e0 = e_begin + kPerThread * t;
  const std::uint32_t cnt = e0 < a.n ? static_cast<std::uint32_t>(a.n - e0 < 16 ? a.n - e0 : 16) : 0;
  std::uint8_t x[16];
  load16(a.fp8, e0, cnt, x);
  // the chunk's first bit and the previous element (its code length: window
  // and block ownership of my first code), loaded up front with x
  const std::uint64_t cs = a.chunk_start[blockIdx.x];
  const std::uint32_t x_prev = (cnt && e0) ? a.fp8[e0 - 1] : 0;
  __syncthreads();

  // sign/mantissa nibbles: 16 elements -> 8 packed bytes
  if (cnt) {
    std::uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const std::uint32_t b = (nib_of(x[2 * k]) << 4) | (2 * k + 1 < static_cast<int>(cnt) ? nib_of(x[2 * k + 1]) : 0);
      if (k < 4) lo |= b << (8 * k);
      else hi |= b << (8 * (k - 4));
    }
    std::uint8_t* const dst = a.packed + e0 / 2;
    if (cnt == 16) {
      *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
    } else {
      for (std::uint32_t k = 0; k < (cnt + 1) / 2; ++k) dst[k] = static_cast<std::uint8_t>((k < 4 ? lo : hi) >> (8 * (k & 3)));
    }
  }

  std::uint32_t my_bits = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < static_cast<int>(cnt)) my_bits += s_lc[exp_of(x[j])] & 31u;
  std::uint32_t chunk_total;
  const std::uint32_t excl = block_excl_scan(my_bits, wsum, &chunk_total);
  const std::uint64_t gw0 = cs >> 5;  // first global word of the chunk's run

  if (cnt) {
    // 32-bit positions relative to B = the chunk start rounded down to a
    // window: window and block changes are bit changes of lp ^ prev.
    const std::uint64_t B = cs & ~std::uint64_t{63};
    const std::uint32_t blk_shift = 6 + a.log2T;
    const std::uint32_t boff = static_cast<std::uint32_t>(B & ((std::uint64_t{1} << blk_shift) - 1));
    std::uint32_t lp = static_cast<std::uint32_t>(cs - B) + excl;  // my first code's start
    // previous code's length (element 0: a fake 64 marks its window as new)
    std::uint32_t len_prev = e0 ? (s_lc[exp_of(x_prev)] & 31u) : 64u;
    const std::uint32_t lb = static_cast<std::uint32_t>(cs & 31) + excl;  // bit offset in run[]
    std::uint32_t word = lb >> 5, fill = lb & 31, cur = 0;
    std::uint32_t lp_last = lp;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j < static_cast<int>(cnt)) {
        const std::uint32_t lc = s_lc[exp_of(x[j])];
        const std::uint32_t len = lc & 31u, val = lc & ~31u;  // code MSB-aligned
        const std::uint32_t prev = lp - len_prev;             // previous code's start (mod 2^32)
        if ((lp ^ prev) >> 6) {
          // first code starting in window B/64 + lp/64: its gap nibble
          const std::uint64_t w = (B >> 6) + (lp >> 6);
          const std::uint64_t gb = w >> 1;
          const std::uint32_t v = (lp & 63) << ((w & 1) ? 0 : 4);
          if (v) atomicOr(a.gaps + (gb >> 2), v << (8 * (gb & 3)));
        }
        if (((lp + boff) ^ (prev + boff)) >> blk_shift) a.outpos[(B + lp) >> blk_shift] = e0 + j;
        cur |= val >> fill;
        const std::uint32_t spill = fill ? val << (32 - fill) : 0u;
        fill += len;
        if (fill >= 32) {
          atomicOr(&run[word], cur);
          cur = spill;
          fill -= 32;
          ++word;
        }
        lp_last = lp;
        lp += len;
        len_prev = len;
      }
    }
    if (fill) atomicOr(&run[word], cur);
    if (e0 + cnt == a.n) {
      // blocks after the last code's: no code starts there
      for (std::uint64_t b = ((B + lp_last) >> blk_shift) + 1; b <= a.n_blocks; ++b) a.outpos[b] = a.n;
    }
  }
  __syncthreads();

  const std::uint64_t ce = cs + chunk_total;
  if (ce > cs) {
    const std::uint32_t nw = static_cast<std::uint32_t>(((ce - 1) >> 5) - gw0 + 1);
    for (std::uint32_t i = t; i < nw; i += kEncThreads) {
      const std::uint32_t v = __byte_perm(run[i], 0, 0x0123);  // MSB-first bytes
      if (i == 0 || i == nw - 1) {
        if (v) atomicOr(a.encoded + gw0 + i, v);
      } else {
        a.encoded[gw0 + i] = v;
      }
    }
  }
}

}  // namespace

cudaError_t launch_exponent_histogram(const std::uint8_t* fp8, std::uint64_t n, unsigned long long* counts,
                                      cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const std::uint64_t want = (n + 16 * 256 - 1) / (16 * 256);
  const unsigned grid = static_cast<unsigned>(want < static_cast<std::uint64_t>(4 * sms) ? want : 4 * sms);
  histogram_kernel<<<grid, 256, 0, s>>>(fp8, n, counts);
  return cudaGetLastError();
}

cudaError_t launch_encode_sizes(const std::uint8_t* fp8, std::uint64_t n, const std::uint8_t* lengths16,
                                std::uint32_t* chunk_bits, std::uint64_t* chunk_start, unsigned long long* total,
                                std::uint32_t* bad, cudaStream_t s) {
  const std::uint64_t n_chunks = (n + kEncChunkElems - 1) / kEncChunkElems;
  if (n_chunks == 0) return cudaSuccess;
  chunk_bits_kernel<<<static_cast<unsigned>(n_chunks), kEncThreads, 0, s>>>(fp8, n, lengths16, chunk_bits, bad);
  chunk_scan_kernel<<<1, 1024, 0, s>>>(chunk_bits, n_chunks, chunk_start, total);
  return cudaGetLastError();
}

cudaError_t launch_encode_emit(const EncodeArgs& a, cudaStream_t s) {
  const std::uint64_t n_chunks = (a.n + kEncChunkElems - 1) / kEncChunkElems;
  if (n_chunks == 0) return cudaSuccess;
  encode_emit_kernel<<<static_cast<unsigned>(n_chunks), kEncThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// One thread per 16-byte chunk: tile (nt, kt) in row-major tile order, each
// tile the 128B-swizzled K-major image (chunk c of row r at r * 128 +
// ((c ^ (r & 7)) << 4)) -- the host layout of ecf8_host_fused_layout.
__global__ void fused_layout_kernel(const uint4* __restrict__ in, std::uint64_t n, std::uint64_t k,
                                    uint4* __restrict__ out, bool inverse) {
  const std::uint64_t KT = k / 128, chunks = n * k / 16;
  for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < chunks;
       i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
    // i: chunk of the row-major matrix (coalesced on that side)
    const std::uint64_t row = i / (k / 16), cc = i % (k / 16);
    const std::uint64_t nt = row / 128, r = row % 128, kt = cc / 8, c = cc % 8;
    const std::uint64_t t = (nt * KT + kt) * 1024 + r * 8 + (c ^ (r & 7));
    if (inverse) out[i] = in[t];
    else out[t] = in[i];
  }
}

cudaError_t launch_fused_layout(const std::uint8_t* in, std::uint64_t n, std::uint64_t k, std::uint8_t* out,
                                bool inverse, cudaStream_t s) {
  const std::uint64_t chunks = n * k / 16;
  if (!chunks) return cudaSuccess;
  const std::uint64_t blocks = std::min<std::uint64_t>((chunks + 255) / 256, 148 * 16);
  fused_layout_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(reinterpret_cast<const uint4*>(in), n, k,
                                                                    reinterpret_cast<uint4*>(out), inverse);
  return cudaGetLastError();
}

}  // namespace ecf8::dev
