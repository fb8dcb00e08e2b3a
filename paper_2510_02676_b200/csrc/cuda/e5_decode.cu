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
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ecf8_cuda.h"
#include "ecf8_e5m2.h"

extern "C" int ecf8_internal_set_error(int status, const char* msg);
extern "C" int ecf8_internal_require_device(void);

namespace ecf8::dev::e5 {

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

cudaError_t launch_e5(const Desc& d, cudaStream_t s) {
  if (d.T <= 256) return launch<256>(d, s);
  if (d.T == 512) return launch<512>(d, s);
  return launch<1024>(d, s);
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

void ecf8_e5_free(ecf8_e5_dev_tensor* t) {
  if (!t) return;
  if (t->arena) cudaFree(t->arena);
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
