// capi.cu -- implementation of the C ABI in include/ecf8_cuda.h.
//
// Host orchestration only: validation with the reference's messages, HBM
// layout of a device tensor, descriptor setup, launches.  The decode itself
// is decode.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "decode.cuh"
#include "encode.cuh"
#include "ecf8/entropy.hpp"
#include "ecf8/huffman.hpp"
#include "fused_gemm.cuh"
#include "ecf8_cuda.h"
#include "tables.hpp"

using ecf8::dev::TensorDesc;

namespace {

thread_local std::string g_last_error;

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

struct CudaFailure {
  cudaError_t err;
  const char* what;
};

inline void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure{e, what};
}

// Runs f, mapping C++ / CUDA failures onto status codes.
template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const CudaFailure& e) {
    cudaGetLastError();  // clear sticky-free errors
    return fail(ECF8_ECUDA, std::string(e.what) + ": " + cudaGetErrorString(e.err));
  } catch (const std::bad_alloc&) {
    return fail(ECF8_ENOMEM, "host allocation failed");
  } catch (const std::invalid_argument& e) {
    return fail(ECF8_EINVAL, e.what());
  } catch (const std::exception& e) {
    return fail(ECF8_ECUDA, e.what());
  }
}

int require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(ECF8_ECUDA, "no CUDA device: the ECF8 decoder runs on the B200 only (no CPU fallback)");
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return fail(ECF8_ECUDA, "device is not sm_100 (kernels are built for sm_100a only)");
  return ECF8_OK;
}

// Reference checks (codec.cpp:259-261, container.cpp:196-242) plus the
// bounds the kernel relies on.
int validate(const ecf8_sections* s, std::uint64_t* n_blocks_out) {
  if (!s) return fail(ECF8_EINVAL, "null sections");
  const std::uint32_t T = s->threads_per_block;
  if (T < 1 || T > 1024 || (T & (T - 1)))
    return fail(ECF8_EINVAL, "threads per block must be a power of two in [1, 1024]");
  const std::uint64_t bb = std::uint64_t{T} * 8;
  if (s->encoded_len < 2 || (s->encoded_len - 2) % bb != 0)
    return fail(ECF8_EINVAL, "encoded section length mismatch");
  const std::uint64_t nb = (s->encoded_len - 2) / bb;
  if (s->n_outpos != nb + 1 || !s->outpos || s->outpos[nb] != s->n_elem || s->outpos[0] != 0)
    return fail(ECF8_EINVAL, "inconsistent block offsets");
  // The reference allows a block up to T * 64 elements (container.cpp:231-239),
  // but a block's windows can hold at most T * ceil(64 / Lmin) code words
  // (every code word, garbage fallbacks included, is >= Lmin bits): elements
  // past that are never emitted, and the reference copies stale scratch for
  // them (codec.cpp:242-253).  Such a container is not encoder output; it is
  // rejected, since the kernels size their slots and staging tiles by Lmin.
  std::uint32_t lmin = 16;
  for (int i = 0; i < 16; ++i)
    if (s->lengths[i] && s->lengths[i] < lmin) lmin = s->lengths[i];
  const std::uint64_t cap = std::uint64_t{T} * ((64 + lmin - 1) / lmin);
  for (std::uint64_t b = 0; b < nb; ++b)
    if (s->outpos[b + 1] < s->outpos[b] || s->outpos[b + 1] - s->outpos[b] > cap)
      return fail(ECF8_EINVAL, "inconsistent block offsets");
  if (s->gaps_len < (nb * T + 1) / 2) return fail(ECF8_EINVAL, "gap section length mismatch");
  if (s->packed_len < (s->n_elem + 1) / 2) return fail(ECF8_EINVAL, "packed section length mismatch");
  if (s->n_elem > 0 && (nb == 0 || !s->encoded || !s->gaps || !s->packed))
    return fail(ECF8_EINVAL, "encoded section length mismatch");
  if (s->n_elem > 0) {
    try {
      (void)ecf8::dev::tables_for(s->lengths);
    } catch (const std::invalid_argument&) {
      return fail(ECF8_EINVAL, "invalid length vector");
    }
  }
  *n_blocks_out = nb;
  return ECF8_OK;
}

std::uint64_t align_up(std::uint64_t x, std::uint64_t a) { return (x + a - 1) / a * a; }

std::uint32_t lmin_of(const std::uint8_t lengths[16]) {
  std::uint32_t m = 16;
  for (int s = 0; s < 16; ++s)
    if (lengths[s] && lengths[s] < m) m = lengths[s];
  return m;
}

// Device copies of the decode tables, shared by every tensor with the same
// code lengths (per device).
struct DevTables {
  std::uint32_t* fast = nullptr;
  std::uint16_t* smask = nullptr;
  std::uint8_t* cascade = nullptr;
  std::uint32_t n_luts = 0;
  std::uint64_t lenpack = 0;
  std::uint32_t* fsm = nullptr;  // byte-step decoder (tables.hpp), nullptr when the code has none
  std::uint8_t* fsm_cm = nullptr;
  std::uint64_t* fsm64 = nullptr;  // its 64-bit form for codes with a 1-bit word
};

const DevTables& device_tables(const std::uint8_t lengths[16]) {
  static std::mutex mu;
  static std::map<std::pair<int, std::array<std::uint8_t, 16>>, DevTables> cache;
  int dev = 0;
  cu(cudaGetDevice(&dev), "cudaGetDevice");
  std::array<std::uint8_t, 16> key{};
  std::memcpy(key.data(), lengths, 16);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, key});
  if (it != cache.end()) return it->second;
  const auto t = ecf8::dev::tables_for(lengths);
  DevTables d;
  d.n_luts = t->n_luts;
  d.lenpack = t->lenpack;
  void* p = nullptr;
  cu(cudaMalloc(&p, t->fast.size() * 4 + t->smask.size() * 2 + t->cascade.size()), "cudaMalloc(tables)");
  d.fast = static_cast<std::uint32_t*>(p);
  d.smask = reinterpret_cast<std::uint16_t*>(static_cast<std::uint8_t*>(p) + t->fast.size() * 4);
  d.cascade = static_cast<std::uint8_t*>(p) + t->fast.size() * 4 + t->smask.size() * 2;
  cu(cudaMemcpy(d.fast, t->fast.data(), t->fast.size() * 4, cudaMemcpyHostToDevice), "upload tables");
  cu(cudaMemcpy(d.smask, t->smask.data(), t->smask.size() * 2, cudaMemcpyHostToDevice), "upload tables");
  cu(cudaMemcpy(d.cascade, t->cascade.data(), t->cascade.size(), cudaMemcpyHostToDevice), "upload tables");
  if (t->fsm_ok) {
    void* q = nullptr;
    cu(cudaMalloc(&q, t->fsm.size() * 4 + t->fsm_cm.size()), "cudaMalloc(tables)");
    d.fsm = static_cast<std::uint32_t*>(q);
    d.fsm_cm = static_cast<std::uint8_t*>(q) + t->fsm.size() * 4;
    cu(cudaMemcpy(d.fsm, t->fsm.data(), t->fsm.size() * 4, cudaMemcpyHostToDevice), "upload tables");
    cu(cudaMemcpy(d.fsm_cm, t->fsm_cm.data(), t->fsm_cm.size(), cudaMemcpyHostToDevice), "upload tables");
  }
  if (t->fsm64_ok) {
    void* q = nullptr;
    cu(cudaMalloc(&q, t->fsm64.size() * 8), "cudaMalloc(tables)");
    d.fsm64 = static_cast<std::uint64_t*>(q);
    cu(cudaMemcpy(d.fsm64, t->fsm64.data(), t->fsm64.size() * 8, cudaMemcpyHostToDevice), "upload tables");
  }
  return cache.emplace(std::make_pair(dev, key), d).first->second;
}

}  // namespace

// One HBM allocation per tensor, sections at 256-byte aligned offsets, each
// followed by zero padding (kernels over-read whole 16-byte vectors).
struct ecf8_dev_tensor {
  void* arena = nullptr;
  std::uint64_t arena_bytes = 0;
  std::uint64_t n_elem = 0, n_blocks = 0;
  std::uint64_t algo_bytes = 0;
  std::uint32_t T = 0;
  std::uint64_t n_vtiles = 0;      // 256-window verification tiles (tile_ok bits)
  std::uint32_t* ok_bits = nullptr;  // their bitmap in the arena
  std::uint8_t* endgap = nullptr;    // per-window end nibbles (verify_gaps_kernel)
  std::uint32_t* direct_bits = nullptr;  // tile_direct bitmap
  std::uint16_t* lane_start = nullptr;   // per 4-window group output offsets
  TensorDesc desc{};     // out / tile fields filled per launch
  std::uint64_t encoded_len = 0, gaps_len = 0, n_outpos = 0, packed_len = 0;
  std::uint8_t lengths[16] = {};
  bool pooled = false;  // arena from the stream-ordered pool (device encoder)
  cudaStream_t home = nullptr;      // pooled: the stream it was allocated (and is freed) on
  cudaEvent_t last_use = nullptr;   // pooled: recorded after every launch that reads it
};

// A launch on `st` reads t: a pooled arena is freed stream-ordered after it.
void note_use(const ecf8_dev_tensor* t, cudaStream_t st) {
  if (!t || !t->pooled) return;
  auto* m = const_cast<ecf8_dev_tensor*>(t);
  if (!m->last_use) cu(cudaEventCreateWithFlags(&m->last_use, cudaEventDisableTiming), "event");
  cu(cudaEventRecord(m->last_use, st), "record");
}

void free_arena(ecf8_dev_tensor* t) {
  if (!t->arena) return;
  if (t->pooled) {
    // stream-ordered: back to the pool once the last launch reading it (on
    // any stream) and the work on its own stream are done -- no device-wide
    // sync (which would also break a CUDA graph capture elsewhere)
    if (t->last_use) cudaStreamWaitEvent(t->home, t->last_use, 0);
    cudaFreeAsync(t->arena, t->home);
    if (t->last_use) cudaEventDestroy(t->last_use);
    t->last_use = nullptr;
  } else {
    cudaFree(t->arena);
  }
  t->arena = nullptr;
}

struct ecf8_fused {
  const ecf8_dev_tensor* w = nullptr;
  // CTA plans for m > 128 ([0]) and m <= 128 ([1]): both one wave of the
  // SMs (the accumulators are reused round-robin, so any segment count per
  // CTA fits); they differ only under the ECF8_FUSED_SEG_CAP A/B switch.
  ecf8::dev::FusedCta* d_plan[2] = {nullptr, nullptr};
  std::uint32_t n_cta[2] = {0, 0}, max_seg[2] = {0, 0};
  std::uint32_t split_k = 1;
  std::uint64_t n = 0, k = 0;
  std::uint32_t w_fmt = 0;
  bool fsm = false;  // byte-step direct decode: the code has a byte-step decoder and every tile is direct
  std::vector<std::uint64_t> outpos;  // host copy of the weight's block offsets (row ranges -> blocks)
};

struct ecf8_batch {
  std::vector<const ecf8_dev_tensor*> pooled;  // members whose arenas are freed stream-ordered
  std::vector<TensorDesc*> d_descs;  // one device array per kwin group
  std::vector<int> counts;
  std::vector<int> kwins;
  std::vector<std::uint64_t> tiles;
};

namespace {

// The tensor's HBM arena for sections of the sizes in *s (pointers unused):
// allocated, zeroed on `st`, descriptor filled.  The caller fills the
// sections (H2D copies, or the device encoder).
void alloc_arena(ecf8_dev_tensor* t, const ecf8_sections* s, std::uint64_t nb, cudaStream_t st,
                 bool pooled = false) {
  const std::uint64_t P = ecf8::dev::kPad;
  const std::uint64_t off_enc = 0;
  const std::uint64_t off_gap = align_up(off_enc + s->encoded_len + P, 256);
  const std::uint64_t off_pos = align_up(off_gap + s->gaps_len + P, 256);
  const std::uint64_t off_pak = align_up(off_pos + 8 * s->n_outpos, 256);
  const std::uint64_t n_vtiles = (nb * s->threads_per_block + 255) / 256;
  const std::uint64_t off_ok = align_up(off_pak + s->packed_len + P, 256);
  const std::uint64_t n_win = nb * s->threads_per_block;
  const std::uint64_t off_dir = align_up(off_ok + 4 * ((n_vtiles + 31) / 32), 256);
  const std::uint64_t off_eg = align_up(off_dir + 4 * ((n_vtiles + 31) / 32), 256);
  const std::uint64_t off_ls = align_up(off_eg + (n_win + 1) / 2 + P, 256);
  const std::uint64_t total = align_up(off_ls + 2 * ((n_win + 3) / 4) + P, 256);
  if (pooled) {
    // stream-ordered pool (the device encoder: many tensors created and
    // dropped in a row; cudaMalloc/cudaFree cost ~1 ms each at 50 MB)
    static const bool keep = [] {
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        std::uint64_t thr = ~std::uint64_t{0};
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      cudaGetLastError();
      return true;
    }();
    (void)keep;
    cu(cudaMallocAsync(&t->arena, total, st), "cudaMallocAsync(tensor)");
    t->pooled = true;
    t->home = st;
  } else {
    cu(cudaMalloc(&t->arena, total), "cudaMalloc(tensor)");
  }
  t->arena_bytes = total;
  auto* base = static_cast<std::uint8_t*>(t->arena);
  cu(cudaMemsetAsync(base, 0, total, st), "cudaMemset");
  t->n_vtiles = n_vtiles;
  t->ok_bits = reinterpret_cast<std::uint32_t*>(base + off_ok);
  t->endgap = base + off_eg;
  t->direct_bits = reinterpret_cast<std::uint32_t*>(base + off_dir);
  t->lane_start = reinterpret_cast<std::uint16_t*>(base + off_ls);
  t->encoded_len = s->encoded_len;
  t->gaps_len = s->gaps_len;
  t->n_outpos = s->n_outpos;
  t->packed_len = s->packed_len;
  std::memcpy(t->lengths, s->lengths, 16);

  t->n_elem = s->n_elem;
  t->n_blocks = nb;
  t->T = s->threads_per_block;
  t->algo_bytes = s->encoded_len + s->gaps_len + 8 * s->n_outpos + s->packed_len + s->n_elem;
  TensorDesc& d = t->desc;
  d.encoded = base + off_enc;
  d.gaps = base + off_gap;
  d.outpos = reinterpret_cast<const std::uint64_t*>(base + off_pos);
  d.packed = base + off_pak;
  d.n_elem = s->n_elem;
  d.blk_begin = 0;
  d.blk_end = nb;
  d.T = s->threads_per_block;
  d.lmin = lmin_of(s->lengths);
  if (s->n_elem) {
    const DevTables& tb = device_tables(s->lengths);
    d.fast = tb.fast;
    d.smask = tb.smask;
    d.cascade = tb.cascade;
    d.n_luts = tb.n_luts;
    d.lenpack = tb.lenpack;
    d.fsm = tb.fsm;
    d.fsm_cm = tb.fsm_cm;
  }
}

void upload_into(ecf8_dev_tensor* t, const ecf8_sections* s, std::uint64_t nb, cudaStream_t st) {
  alloc_arena(t, s, nb, st);
  const TensorDesc& d = t->desc;
  cu(cudaMemcpyAsync(const_cast<std::uint8_t*>(d.encoded), s->encoded, s->encoded_len, cudaMemcpyHostToDevice, st),
     "H2D encoded");
  if (s->gaps_len)
    cu(cudaMemcpyAsync(const_cast<std::uint8_t*>(d.gaps), s->gaps, s->gaps_len, cudaMemcpyHostToDevice, st),
       "H2D gaps");
  cu(cudaMemcpyAsync(const_cast<std::uint64_t*>(d.outpos), s->outpos, 8 * s->n_outpos, cudaMemcpyHostToDevice, st),
     "H2D outpos");
  if (s->packed_len)
    cu(cudaMemcpyAsync(const_cast<std::uint8_t*>(d.packed), s->packed, s->packed_len, cudaMemcpyHostToDevice, st),
       "H2D packed");
}

// Gap check at upload (verify_gaps_kernel): every window's end (endgap) is
// recorded; tiles whose 8-window lanes are internally consistent (each window
// ends where the next one's gap says) take the continuous walk, the rest
// keep the reference's window-by-window semantics.
void verify_into(ecf8_dev_tensor* t, cudaStream_t st) {
  static const bool off = std::getenv("ECF8_NO_CONT_WALK") != nullptr;  // A/B runs
  const int vid = t->n_elem ? ecf8::dev::variant_of(t->desc).id : -1;
  if (off || (vid != 4 && vid != 5)) return;
  std::uint32_t* const ok = t->ok_bits;
  cu(cudaMemsetAsync(ok, 0xFF, 4 * ((t->n_vtiles + 31) / 32), st), "memset(tile_ok)");
  cu(cudaMemsetAsync(t->direct_bits, 0xFF, 4 * ((t->n_vtiles + 31) / 32), st), "memset(tile_direct)");
  cu(ecf8::dev::launch_verify_gaps(t->desc, t->n_blocks, ok, t->endgap, t->lane_start, t->direct_bits, st),
     "verify launch");
  t->desc.tile_ok = ok;
  t->desc.endgap = t->endgap;
  if (vid == 4) {
    t->desc.lane_start = t->lane_start;
    t->desc.tile_direct = t->direct_bits;
    // every tile placed directly: variant 7 (no fallback path; one read-back
    // of the tile bitmap)
    static const bool no_direct = std::getenv("ECF8_NO_DIRECT_KERNEL") != nullptr;  // A/B runs
    if (!no_direct) {
      const std::size_t words = (t->n_vtiles + 31) / 32;
      std::vector<std::uint32_t> dirb(words);
      cu(cudaMemcpyAsync(dirb.data(), t->direct_bits, 4 * words, cudaMemcpyDeviceToHost, st), "D2H tile_direct");
      cu(cudaStreamSynchronize(st), "sync");
      bool all = true;
      for (std::uint64_t v = 0; v < t->n_vtiles; ++v) all &= (dirb[v >> 5] >> (v & 31)) & 1u;
      t->desc.all_direct = all ? 1u : 0u;
    }
  }
  // Variant 6 (1-bit codes by byte steps) places every tile directly and has
  // no per-window fallback: it is chosen only when every tile passed (one
  // read-back of the two tile bitmaps; tensors of crafted streams keep
  // variant 5).
  static const bool no64 = std::getenv("ECF8_NO_FSM64") != nullptr;  // A/B runs
  const DevTables& tb = device_tables(t->lengths);
  if (vid == 5 && tb.fsm64 && !no64 && t->T >= 8 && t->T <= 256) {
    const std::size_t words = (t->n_vtiles + 31) / 32;
    std::vector<std::uint32_t> okb(words), dirb(words);
    cu(cudaMemcpyAsync(okb.data(), ok, 4 * words, cudaMemcpyDeviceToHost, st), "D2H tile_ok");
    cu(cudaMemcpyAsync(dirb.data(), t->direct_bits, 4 * words, cudaMemcpyDeviceToHost, st), "D2H tile_direct");
    cu(cudaStreamSynchronize(st), "sync");
    bool all = true;
    for (std::uint64_t v = 0; v < t->n_vtiles; ++v) all &= ((okb[v >> 5] & dirb[v >> 5]) >> (v & 31)) & 1u;
    if (all) {
      t->desc.lane_start = t->lane_start;
      t->desc.tile_direct = t->direct_bits;
      t->desc.fsm64 = tb.fsm64;
    }
  }
}

// Single-descriptor launch: the descriptor rides in the kernel parameters.
int launch_one(const TensorDesc& d, cudaStream_t st, int variant_override = -1) {
  if (d.blk_end <= d.blk_begin) return ECF8_OK;
  ecf8::dev::Variant v = ecf8::dev::variant_of(d);
  if (variant_override >= 0) v.id = variant_override;
  ecf8::dev::LaunchArgs a{};
  a.descs = nullptr;
  a.n_desc = 1;
  a.total_tiles = ecf8::dev::tiles_of(d.T, v.tile_win, d.blk_end - d.blk_begin);
  a.inline_desc = d;
  a.inline_desc.tile_begin = 0;
  cu(ecf8::dev::launch_decode(a, v.id, st), "decode launch");
  return ECF8_OK;
}

// Launch variant for a device tensor.
int tensor_variant(const ecf8_dev_tensor* t) {
  return ecf8::dev::variant_of(t->desc).id;
}

// Per-thread state of the host-span path: three streams (copy-in, decode,
// copy-out) and a ring of chunk slots in HBM.  Deliberately never freed:
// CUDA may already be torn down when thread_local destructors run at exit.
struct HostCtx {
  // Chunk slots in flight (ECF8_SLOTS, 2..kMaxSlots): the H2D of chunk k
  // waits for the D2H of chunk k - nslots.
  static constexpr int kMaxSlots = 16;
  int nslots = 4;
  // Chunk limits.  PCIe copies pay ~15 us each, so chunks are large (32 M
  // elements = 32 MB D2H) in the steady state and ramp from 4 M at the start
  // and towards the end of a call (short pipeline fill and drain).  Measured
  // on one Llama-8B layer (tools/e2e_probe.py): 2/16 M 62 GB/s, 4/16 M 70,
  // 4/32 M 73, 4/64 M 71.
  static constexpr std::uint64_t kEncChunk = std::uint64_t{8} << 20;    // encoded bytes per chunk (min)
  static constexpr std::uint64_t kElemChunk = std::uint64_t{32} << 20;  // elements per chunk
  static constexpr std::uint64_t kElemMin = std::uint64_t{4} << 20;
  std::uint64_t elem_chunk = kElemChunk, elem_min = kElemMin, enc_chunk = kEncChunk;  // ECF8_CHUNK_M / ECF8_CHUNK_MIN_M (M elements)
  static constexpr std::uint64_t kSlack = 4096;
  int dev = -1;
  cudaStream_t s_in = nullptr, s_run = nullptr, s_out = nullptr;
  struct Slot {
    std::uint8_t *enc, *pak, *out;
    std::uint8_t* eg;     // the chunk's window ends (verify_gaps_kernel)
    std::uint32_t* ok;    // and its tile_ok words
    std::uint32_t* dir;   // tile_direct words
    std::uint16_t* ls;    // 4-window group offsets
    cudaEvent_t in, run, out_done;
    bool used;
    // Pageable host spans: pinned staging (allocated on first need).  The
    // inputs are copied in by the host threads before the slot's H2D, the
    // output copied out after its D2H completed (when the slot is reused,
    // or at the end of the call).
    std::uint8_t *h_in = nullptr, *h_out = nullptr;
    std::uint8_t* pend_dst = nullptr;  // pageable destination of the slot's last D2H
    std::uint64_t pend_bytes = 0;
  } slot[kMaxSlots]{};
  std::uint64_t h_in_bytes = 0, h_out_bytes = 0;
  // Per-tensor gaps + outpos (one copy each per tensor, not per chunk),
  // double-buffered by tensor parity.
  struct Meta {
    std::uint8_t* buf = nullptr;
    std::uint64_t cap = 0;
    cudaEvent_t done = nullptr;
    bool used = false;
  } meta[2];
};

HostCtx& host_ctx() {
  thread_local HostCtx c;
  int dev = 0;
  cu(cudaGetDevice(&dev), "cudaGetDevice");
  if (c.dev != dev) {
    c = HostCtx{};
    cu(cudaStreamCreateWithFlags(&c.s_in, cudaStreamNonBlocking), "stream");
    cu(cudaStreamCreateWithFlags(&c.s_run, cudaStreamNonBlocking), "stream");
    cu(cudaStreamCreateWithFlags(&c.s_out, cudaStreamNonBlocking), "stream");
    if (const char* e = std::getenv("ECF8_CHUNK_M")) c.elem_chunk = std::min<std::uint64_t>(std::atoi(e), 128) << 20;
    if (const char* e = std::getenv("ECF8_CHUNK_MIN_M")) c.elem_min = std::min<std::uint64_t>(std::atoi(e), 16) << 20;
    if (const char* e = std::getenv("ECF8_SLOTS")) c.nslots = std::clamp(std::atoi(e), 2, HostCtx::kMaxSlots);
    // a chunk is >= one tile and the ramp never exceeds the slot size
    c.elem_chunk = std::max<std::uint64_t>(c.elem_chunk, ecf8::dev::kTileElemsMax);
    c.elem_min = std::clamp<std::uint64_t>(c.elem_min, ecf8::dev::kTileElemsMax, c.elem_chunk);
    const std::uint64_t S = HostCtx::kSlack;
    c.enc_chunk = std::max(HostCtx::kEncChunk, c.elem_chunk / 2);
    const std::uint64_t b_enc = align_up(c.enc_chunk + ecf8::dev::kTileBytesMax + S, 256);
    const std::uint64_t b_pak = align_up(c.elem_chunk / 2 + ecf8::dev::kTileElemsMax + S, 256);
    const std::uint64_t b_out = align_up(c.elem_chunk + 2 * ecf8::dev::kTileElemsMax + S, 256);
    const std::uint64_t b_eg = align_up(b_enc / 16 + S, 256);              // a nibble per 8-byte window
    const std::uint64_t b_ok = align_up(4 * (b_enc / 8 / 8192 + 2), 256);  // a bit per 256 windows (+ a straddled word)
    const std::uint64_t b_ls = align_up(2 * (b_enc / 32 + 1) + S, 256);    // a u16 per 4 windows
    for (int si = 0; si < c.nslots; ++si) {
      HostCtx::Slot& sl = c.slot[si];
      void* p = nullptr;
      const std::uint64_t all = b_enc + b_pak + b_out + b_eg + 2 * b_ok + b_ls;
      cu(cudaMalloc(&p, all), "cudaMalloc(staging)");
      cu(cudaMemset(p, 0, all), "cudaMemset(staging)");
      auto* base = static_cast<std::uint8_t*>(p);
      sl.enc = base;
      sl.pak = base + b_enc;
      sl.out = base + b_enc + b_pak;
      sl.eg = base + b_enc + b_pak + b_out;
      sl.ok = reinterpret_cast<std::uint32_t*>(base + b_enc + b_pak + b_out + b_eg);
      sl.dir = reinterpret_cast<std::uint32_t*>(base + b_enc + b_pak + b_out + b_eg + b_ok);
      sl.ls = reinterpret_cast<std::uint16_t*>(base + b_enc + b_pak + b_out + b_eg + 2 * b_ok);
      cu(cudaEventCreateWithFlags(&sl.in, cudaEventDisableTiming), "event");
      cu(cudaEventCreateWithFlags(&sl.run, cudaEventDisableTiming), "event");
      cu(cudaEventCreateWithFlags(&sl.out_done, cudaEventDisableTiming), "event");
      sl.used = false;
    }
    for (auto& mt : c.meta) cu(cudaEventCreateWithFlags(&mt.done, cudaEventDisableTiming), "event");
    c.h_in_bytes = b_enc + b_pak;
    c.h_out_bytes = b_out;
    c.dev = dev;
  }
  return c;
}

// Host memory the DMA engines can read / write directly (cudaMallocHost,
// cudaHostRegister); anything else is pageable and goes through staging.
bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// memcpy by all host threads (pinned staging <-> pageable spans).
void par_copy(void* dst, const void* src, std::uint64_t n) {
  constexpr std::uint64_t kPiece = std::uint64_t{1} << 20;
  const std::int64_t pieces = static_cast<std::int64_t>((n + kPiece - 1) / kPiece);
  if (pieces <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < pieces; ++i) {
    const std::uint64_t o = static_cast<std::uint64_t>(i) * kPiece;
    std::memcpy(static_cast<std::uint8_t*>(dst) + o, static_cast<const std::uint8_t*>(src) + o, std::min(kPiece, n - o));
  }
}

// The slot's staged output, once its D2H has completed, to its pageable destination.
void drain_out(HostCtx::Slot& sl) {
  if (!sl.pend_bytes) return;
  cu(cudaEventSynchronize(sl.out_done), "sync");
  par_copy(sl.pend_dst, sl.h_out, sl.pend_bytes);
  sl.pend_bytes = 0;
}

// Pointer whose element `lo` is `slot` (the kernels index sections with
// global block / window / element numbers; only [lo, hi) is dereferenced).
template <class P>
P rebase(P slot, std::uint64_t lo_bytes) {
  return reinterpret_cast<P>(reinterpret_cast<std::uintptr_t>(slot) - lo_bytes);
}

// decode_parallel_into on host spans, for one or many tensors: every tensor
// is cut into chunks of whole tiles (<= 2 MB encoded, <= 8 M elements);
// chunk k's sections go H2D on s_in into slot k%4 while chunk k-1 decodes
// on s_run and chunk k-2's bytes come back on s_out, across tensor
// boundaries.  With pinned host memory both PCIe directions and the
// decode overlap; the call returns when every byte is in `outs`.
//
// blk_lo / blk_hi (optional): decode only blocks [blk_lo[i], blk_hi[i]) of
// tensor i -- its elements [outpos[lo], outpos[hi]) land at the same offsets
// of outs[i] (decode_block); only those blocks' sections cross PCIe.
// Streaming delivery (ecf8_decode_host_stream): every tensor decodes into the
// same pinned buffer; chunk (tensor i, [o0, o1)) is handed to `fn` once its
// D2H completed, in order, and a D2H into the buffer waits until the earlier
// tensors' bytes it overwrites were handed over.
struct StreamSink {
  ecf8_chunk_fn fn = nullptr;
  void* ctx = nullptr;
  struct Pending {
    int slot, tensor;
    std::uint64_t o0, o1;
  };
  std::deque<Pending> q;
  int rc = 0;
};

int host_pipeline(const ecf8_sections* const* ss, const std::uint64_t* nbs, std::uint8_t* const* outs, int count,
                  const std::uint64_t* blk_lo = nullptr, const std::uint64_t* blk_hi = nullptr,
                  StreamSink* sink = nullptr) {
  HostCtx& c = host_ctx();
  auto deliver_front = [&]() {  // the oldest pending chunk, once its D2H completed
    const StreamSink::Pending p = sink->q.front();
    sink->q.pop_front();
    cu(cudaEventSynchronize(c.slot[p.slot].out_done), "sync");
    if (sink->rc == 0 && p.o1 > p.o0) sink->rc = sink->fn(sink->ctx, p.tensor, p.o0, p.o1 - p.o0);
  };
  std::uint64_t k = 0, remaining = 0;
  for (int i = 0; i < count; ++i)
    remaining += blk_lo ? ss[i]->outpos[blk_hi[i]] - ss[i]->outpos[blk_lo[i]] : ss[i]->n_elem;
  std::uint64_t target = c.elem_min;
  int parity = 0;
  static const bool skip_kernel = std::getenv("ECF8_DIAG_NO_KERNEL") != nullptr;  // PCIe-only diagnostics
  for (int i = 0; i < count; ++i) {
    const ecf8_sections* s = ss[i];
    const std::uint64_t b_begin = blk_lo ? blk_lo[i] : 0, nb = blk_lo ? blk_hi[i] : nbs[i];
    if (s->n_elem == 0 || s->outpos[nb] == s->outpos[b_begin]) continue;
    std::uint8_t* const out = outs[i];
    const bool in_pinned = is_pinned(s->encoded) && is_pinned(s->packed), out_pinned = is_pinned(out);
    const std::uint32_t T = s->threads_per_block;
    const DevTables& tb = device_tables(s->lengths);
    const ecf8::dev::Variant v = ecf8::dev::variant_for(T, lmin_of(s->lengths), tb.fsm != nullptr);
    const std::uint64_t m = ecf8::dev::blocks_per_tile(T, v.tile_win);
    const std::uint64_t tile_enc = m * T * 8;
    TensorDesc d{};
    d.n_elem = s->n_elem;
    d.T = T;
    d.fast = tb.fast;
    d.smask = tb.smask;
    d.cascade = tb.cascade;
    d.n_luts = tb.n_luts;
    d.lenpack = tb.lenpack;
    d.fsm = tb.fsm;
    d.fsm_cm = tb.fsm_cm;
    d.lmin = lmin_of(s->lengths);

    HostCtx::Meta& mt = c.meta[parity];
    parity ^= 1;
    // the blocks' gaps (window nibbles [b_begin T, nb T)) and outpos [b_begin, nb]
    const std::uint64_t g0 = (b_begin * T) >> 1, g1 = std::min(s->gaps_len, (nb * T + 1) / 2 + 1);
    const std::uint64_t off_pos = align_up(g1 - g0 + ecf8::dev::kPad, 256);
    const std::uint64_t need = off_pos + 8 * (nb - b_begin + 1);
    if (need > mt.cap) {
      if (mt.used) cu(cudaEventSynchronize(mt.done), "sync");
      if (mt.buf) cudaFree(mt.buf);
      mt.buf = nullptr;
      mt.cap = 0;
      cu(cudaMalloc(&mt.buf, need + (need >> 2)), "cudaMalloc(staging)");
      mt.cap = need + (need >> 2);
    } else if (mt.used) {
      cu(cudaStreamWaitEvent(c.s_in, mt.done, 0), "wait");
    }
    mt.used = true;
    if (g1 > g0) cu(cudaMemcpyAsync(mt.buf, s->gaps + g0, g1 - g0, cudaMemcpyHostToDevice, c.s_in), "H2D gaps");
    cu(cudaMemcpyAsync(mt.buf + off_pos, s->outpos + b_begin, 8 * (nb - b_begin + 1), cudaMemcpyHostToDevice, c.s_in),
       "H2D outpos");
    d.gaps = rebase(static_cast<const std::uint8_t*>(mt.buf), g0);
    d.outpos = rebase(reinterpret_cast<const std::uint64_t*>(mt.buf + off_pos), 8 * b_begin);
    for (std::uint64_t lo = b_begin; lo < nb; ++k) {
      // grow the chunk tile by tile up to the ramped target and slot limits
      const std::uint64_t want =
          std::max(c.elem_min, std::min({target, c.elem_chunk, remaining / 3}));
      std::uint64_t hi = std::min(nb, lo + m);
      while (hi < nb) {
        const std::uint64_t nh = std::min(nb, hi + m);
        if ((nh - lo) * T * 8 > c.enc_chunk || s->outpos[nh] - s->outpos[lo] > want) break;
        hi = nh;
      }
      (void)tile_enc;
      target = std::min(2 * target, c.elem_chunk);  // ramp up (saturating)
      remaining -= s->outpos[hi] - s->outpos[lo];
      HostCtx::Slot& sl = c.slot[k % c.nslots];
      if (sl.used) cu(cudaStreamWaitEvent(c.s_in, sl.out_done, 0), "wait");
      const std::uint64_t e0 = lo * T * 8, e1 = hi * T * 8 + 2;
      const std::uint64_t o0 = s->outpos[lo], o1 = s->outpos[hi];
      const std::uint64_t p0 = (o0 / 2) & ~std::uint64_t{15}, p1 = std::min(s->packed_len, (o1 + 1) / 2);
      if (in_pinned) {
        cu(cudaMemcpyAsync(sl.enc, s->encoded + e0, e1 - e0, cudaMemcpyHostToDevice, c.s_in), "H2D encoded");
        if (p1 > p0)
          cu(cudaMemcpyAsync(sl.pak, s->packed + p0, p1 - p0, cudaMemcpyHostToDevice, c.s_in), "H2D packed");
      } else {
        // pageable sections: the host threads copy the chunk into the slot's
        // pinned staging (free once its previous H2D completed), the DMA
        // engine takes it from there
        if (!sl.h_in) {
          void* h = nullptr;
          cu(cudaMallocHost(&h, c.h_in_bytes), "cudaMallocHost(staging)");
          sl.h_in = static_cast<std::uint8_t*>(h);
        }
        if (sl.used) cu(cudaEventSynchronize(sl.in), "sync");
        const std::uint64_t enc_bytes = align_up(e1 - e0, 256);
        par_copy(sl.h_in, s->encoded + e0, e1 - e0);
        if (p1 > p0) par_copy(sl.h_in + enc_bytes, s->packed + p0, p1 - p0);
        cu(cudaMemcpyAsync(sl.enc, sl.h_in, e1 - e0, cudaMemcpyHostToDevice, c.s_in), "H2D encoded");
        if (p1 > p0)
          cu(cudaMemcpyAsync(sl.pak, sl.h_in + enc_bytes, p1 - p0, cudaMemcpyHostToDevice, c.s_in), "H2D packed");
      }
      sl.used = true;
      cu(cudaEventRecord(sl.in, c.s_in), "record");

      cu(cudaStreamWaitEvent(c.s_run, sl.in, 0), "wait");
      TensorDesc dk = d;
      dk.encoded = rebase(static_cast<const std::uint8_t*>(sl.enc), e0);
      dk.packed = rebase(static_cast<const std::uint8_t*>(sl.pak), p0);
      dk.out = sl.out;
      dk.out_offset = o0 & ~std::uint64_t{15};
      dk.blk_begin = lo;
      dk.blk_end = hi;
      if (v.id == 4 && dk.fsm && !skip_kernel) {
        // the byte-step decoder needs every window's end: the upload check on
        // this chunk (its windows only) into the slot's scratch
        const std::uint64_t w0 = lo * T;
        dk.endgap = rebase(sl.eg, w0 >> 1);
        dk.tile_ok = rebase(sl.ok, 4 * (w0 >> 13));
        dk.tile_direct = rebase(sl.dir, 4 * (w0 >> 13));
        dk.lane_start = rebase(sl.ls, 2 * (w0 >> 2));
        const std::uint64_t words = ((hi * T) >> 13) - (w0 >> 13) + 1;
        cu(cudaMemsetAsync(sl.ok, 0xFF, 4 * words, c.s_run), "memset(tile_ok)");
        cu(cudaMemsetAsync(sl.dir, 0xFF, 4 * words, c.s_run), "memset(tile_direct)");
        cu(ecf8::dev::launch_verify_gaps(dk, nbs[i], const_cast<std::uint32_t*>(dk.tile_ok),
                                         const_cast<std::uint8_t*>(dk.endgap), const_cast<std::uint16_t*>(dk.lane_start),
                                         const_cast<std::uint32_t*>(dk.tile_direct), c.s_run),
           "verify launch");
      }
      if (!skip_kernel)
        if (int rc = launch_one(dk, c.s_run)) return rc;
      cu(cudaEventRecord(sl.run, c.s_run), "record");

      cu(cudaStreamWaitEvent(c.s_out, sl.run, 0), "wait");
      if (sink) {
        // the slot's previous chunk, and earlier tensors' chunks this D2H
        // overwrites in the shared buffer, are handed over first (in order)
        while (!sink->q.empty() && (sink->q.front().slot == static_cast<int>(k % c.nslots) ||
                                    (sink->q.front().tensor < i && sink->q.front().o0 < o1))) {
          deliver_front();
        }
        // ... and the ones already complete (keeps the host writer busy)
        while (!sink->q.empty() && cudaEventQuery(c.slot[sink->q.front().slot].out_done) == cudaSuccess)
          deliver_front();
        cudaGetLastError();
      }
      if (out_pinned) {
        if (o1 > o0)
          cu(cudaMemcpyAsync(out + o0, sl.out + (o0 - dk.out_offset), o1 - o0, cudaMemcpyDeviceToHost, c.s_out),
             "D2H out");
      } else {
        // pageable destination: D2H into the slot's pinned staging, copied out
        // by the host threads once it completed (slot reuse or call end)
        if (!sl.h_out) {
          void* h = nullptr;
          cu(cudaMallocHost(&h, c.h_out_bytes), "cudaMallocHost(staging)");
          sl.h_out = static_cast<std::uint8_t*>(h);
        }
        drain_out(sl);
        if (o1 > o0) {
          cu(cudaMemcpyAsync(sl.h_out, sl.out + (o0 - dk.out_offset), o1 - o0, cudaMemcpyDeviceToHost, c.s_out),
             "D2H out");
          sl.pend_dst = out + o0;
          sl.pend_bytes = o1 - o0;
        }
      }
      cu(cudaEventRecord(sl.out_done, c.s_out), "record");
      if (sink) sink->q.push_back({static_cast<int>(k % c.nslots), i, o0, o1});
      lo = hi;
    }
    cu(cudaEventRecord(mt.done, c.s_run), "record");
  }
  if (sink)
    while (!sink->q.empty()) deliver_front();
  cu(cudaStreamSynchronize(c.s_out), "sync");
  for (int si = 0; si < c.nslots; ++si) drain_out(c.slot[si]);
  return ECF8_OK;
}

}  // namespace

extern "C" {

const char* ecf8_last_error(void) { return g_last_error.c_str(); }

int ecf8_internal_set_error(int status, const char* msg) { return fail(status, msg ? msg : ""); }

int ecf8_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

const char* ecf8_build_info(void) {
  return "ecf8-b200: sm_100a decode kernels (persistent tiles, multi-symbol tables)";
}

int ecf8_tensor_upload(const ecf8_sections* s, void* stream, ecf8_dev_tensor** out) {
  return guarded([&]() -> int {
    if (!out) return fail(ECF8_EINVAL, "null output handle");
    *out = nullptr;
    std::uint64_t nb = 0;
    if (int rc = validate(s, &nb)) return rc;
    if (int rc = require_device()) return rc;
    auto t = std::make_unique<ecf8_dev_tensor>();
    try {
      upload_into(t.get(), s, nb, static_cast<cudaStream_t>(stream));
      verify_into(t.get(), static_cast<cudaStream_t>(stream));
    } catch (...) {
      free_arena(t.get());
      throw;
    }
    *out = t.release();
    return ECF8_OK;
  });
}

namespace {
// Per-thread device scratch of the encoder (grow-only, never freed: see
// HostCtx) and a pinned readback word block.
struct EncScratch {
  int dev = -1;
  std::uint8_t* buf = nullptr;
  std::uint64_t cap = 0;
  unsigned long long* host = nullptr;  // pinned, 32 words
  cudaEvent_t free_at = nullptr;       // recorded after the last reader of buf
};
// `st` waits until the previous user of the scratch (any stream) is done.
EncScratch& enc_scratch(std::uint64_t need, cudaStream_t st) {
  thread_local EncScratch e;
  int dev = 0;
  cu(cudaGetDevice(&dev), "cudaGetDevice");
  if (e.dev != dev) {
    e = EncScratch{};
    cu(cudaMallocHost(reinterpret_cast<void**>(&e.host), 32 * sizeof(unsigned long long)), "cudaMallocHost");
    cu(cudaEventCreateWithFlags(&e.free_at, cudaEventDisableTiming), "event");
    cu(cudaEventRecord(e.free_at, st), "record");
    e.dev = dev;
  }
  cu(cudaStreamWaitEvent(st, e.free_at, 0), "wait");
  if (need > e.cap) {
    if (e.buf) {
      cu(cudaEventSynchronize(e.free_at), "sync");  // the scratch's last user (any stream), not the whole device
      cudaFree(e.buf);
      e.buf = nullptr;
      e.cap = 0;
    }
    const std::uint64_t cap = std::max<std::uint64_t>(need + (need >> 1), 1 << 20);
    cu(cudaMalloc(&e.buf, cap), "cudaMalloc(encode scratch)");
    e.cap = cap;
  }
  return e;
}
}  // namespace

int ecf8_exponent_histogram(const uint8_t* d_fp8, uint64_t n, uint64_t counts[16], void* stream) {
  return guarded([&]() -> int {
    if (!counts || (n && !d_fp8)) return fail(ECF8_EINVAL, "null argument");
    if (int rc = require_device()) return rc;
    const auto st = static_cast<cudaStream_t>(stream);
    EncScratch& sc = enc_scratch(256, st);
    auto* d_counts = reinterpret_cast<unsigned long long*>(sc.buf);
    cu(cudaMemsetAsync(d_counts, 0, 16 * sizeof(unsigned long long), st), "cudaMemset");
    cu(ecf8::dev::launch_exponent_histogram(d_fp8, n, d_counts, st), "histogram launch");
    cu(cudaMemcpyAsync(sc.host, d_counts, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st), "D2H");
    cu(cudaEventRecord(sc.free_at, st), "record");
    cu(cudaStreamSynchronize(st), "sync");
    for (int i = 0; i < 16; ++i) counts[i] = sc.host[i];
    return ECF8_OK;
  });
}

int ecf8_encode_device(const uint8_t* d_fp8, uint64_t n, uint32_t T, const uint8_t lengths[16], void* stream,
                       ecf8_dev_tensor** out) {
  return guarded([&]() -> int {
    if (!out || !lengths || (n && !d_fp8)) return fail(ECF8_EINVAL, "null argument");
    *out = nullptr;
    if (T < 1 || T > 1024 || (T & (T - 1)))
      return fail(ECF8_EINVAL, "threads per block must be a power of two in [1, 1024]");
    std::array<std::uint8_t, 16> lv{};
    std::memcpy(lv.data(), lengths, 16);
    const ecf8::CodeTable code = ecf8::canonical_codes(lv);  // "invalid length vector" (huffman.cpp:137-142)
    if (int rc = require_device()) return rc;
    const auto st = static_cast<cudaStream_t>(stream);
    const std::uint64_t n_chunks = (n + ecf8::dev::kEncChunkElems - 1) / ecf8::dev::kEncChunkElems;

    // passes 1-2: code bits per chunk, their scan, the total (one sync: it sizes the arena)
    const std::uint64_t off_start = align_up(4 * n_chunks, 256), off_tot = off_start + align_up(8 * n_chunks, 256);
    EncScratch& sc = enc_scratch(off_tot + 256, st);
    std::uint8_t* const work = sc.buf;
    auto* chunk_bits = reinterpret_cast<std::uint32_t*>(work);
    auto* chunk_start = reinterpret_cast<std::uint64_t*>(work + off_start);
    auto* d_total = reinterpret_cast<unsigned long long*>(work + off_tot);
    auto* d_bad = reinterpret_cast<std::uint32_t*>(work + off_tot + 8);
    std::uint8_t* d_len = work + off_tot + 16;
    cu(cudaMemsetAsync(work + off_tot, 0, 16, st), "cudaMemset");
    cu(cudaMemcpyAsync(d_len, lengths, 16, cudaMemcpyHostToDevice, st), "H2D lengths");
    cu(ecf8::dev::launch_encode_sizes(d_fp8, n, d_len, chunk_bits, chunk_start, d_total, d_bad, st), "encode sizes");
    cu(cudaMemcpyAsync(sc.host, d_total, 16, cudaMemcpyDeviceToHost, st), "D2H total");
    cu(cudaStreamSynchronize(st), "sync");
    const unsigned long long tot_bad[2] = {sc.host[0], sc.host[1]};
    if (tot_bad[1] & 0xFFFFFFFFu) {
      cu(cudaEventRecord(sc.free_at, st), "record");
      return fail(ECF8_EINVAL, "symbol absent from code table");  // codec.cpp:53
    }

    // geometry (make_geometry, codec.cpp:39-47) and the arena
    const std::uint64_t bits = tot_bad[0];
    const std::uint64_t bytes = (bits + 7) / 8, bb = std::uint64_t{T} * 8;
    const std::uint64_t nb = bytes / bb + (bytes % bb != 0);
    ecf8_sections sz{};
    sz.n_elem = n;
    sz.threads_per_block = T;
    std::memcpy(sz.lengths, lengths, 16);
    sz.encoded_len = nb * bb + 2;
    sz.gaps_len = (nb * T + 1) / 2;
    sz.n_outpos = nb + 1;
    sz.packed_len = (n + 1) / 2;
    auto t = std::make_unique<ecf8_dev_tensor>();
    try {
      alloc_arena(t.get(), &sz, nb, st, true);
      t->n_elem = n;
      t->n_blocks = nb;
      t->T = T;
      t->algo_bytes = sz.encoded_len + sz.gaps_len + 8 * sz.n_outpos + sz.packed_len + n;
      if (n) {
        ecf8::dev::EncodeArgs a{};
        a.fp8 = d_fp8;
        a.n = n;
        a.chunk_start = chunk_start;
        a.encoded = reinterpret_cast<std::uint32_t*>(const_cast<std::uint8_t*>(t->desc.encoded));
        a.gaps = reinterpret_cast<std::uint32_t*>(const_cast<std::uint8_t*>(t->desc.gaps));
        a.outpos = const_cast<std::uint64_t*>(t->desc.outpos);
        a.packed = const_cast<std::uint8_t*>(t->desc.packed);
        a.n_blocks = nb;
        a.log2T = static_cast<std::uint32_t>(31 - __builtin_clz(T));
        for (int i = 0; i < 16; ++i)
          a.lc[i] = lengths[i] ? (static_cast<std::uint32_t>(code.codes[i]) << (32 - lengths[i])) | lengths[i] : 0u;
        cu(ecf8::dev::launch_encode_emit(a, st), "encode emit");
      }
      cu(cudaEventRecord(sc.free_at, st), "record");  // chunk_start read
      verify_into(t.get(), st);
    } catch (...) {
      free_arena(t.get());
      throw;
    }
    *out = t.release();
    return ECF8_OK;
  });
}

int ecf8_make_stats_device(const uint8_t* d_fp8, uint64_t n, uint32_t T, uint32_t name_len, uint32_t rank,
                           void* stream, ecf8_entropy_report* out) {
  return guarded([&]() -> int {
    if (!out || (n && !d_fp8) || rank == 0) return fail(ECF8_EINVAL, "null argument");
    // container.cpp:386-413 (make_stats), the histogram and the encode on the GPU
    const ecf8::EntropyBounds gauss = ecf8::entropy_bounds(2.0);
    ecf8_entropy_report r{};
    r.n_elem = n;
    r.bound_lower = gauss.lower;
    r.bound_upper = gauss.upper;
    if (n) {
      ecf8::ExponentHistogram h;
      if (int rc = ecf8_exponent_histogram(d_fp8, n, h.counts.data(), stream)) return rc;
      const ecf8::CodeTable code = ecf8::build_code(h);
      r.entropy_bits = ecf8::shannon_entropy(h);
      r.bits_per_symbol = ecf8::expected_length(code, h);
      r.bits_per_weight = 4.0 + r.bits_per_symbol;
      r.projected_savings = (4.0 - r.bits_per_symbol) / 8.0;
      ecf8_dev_tensor* t = nullptr;
      if (int rc = ecf8_encode_device(d_fp8, n, T, code.lengths.data(), stream, &t)) return rc;
      // tensor_section_bytes (container.cpp): shape, fixed fields, sections
      const std::uint64_t bytes = 2 + std::uint64_t{name_len} + 1 + 8 * std::uint64_t{rank} + (8 + 4 + 16 + 8 + 8 + 8) +
                                  t->encoded_len + t->gaps_len + 8 * t->n_outpos + t->packed_len;
      ecf8_tensor_free(t);
      r.actual_savings = 1.0 - static_cast<double>(bytes) / static_cast<double>(n);
    }
    *out = r;
    return ECF8_OK;
  });
}

int ecf8_tensor_sections(const ecf8_dev_tensor* t, ecf8_sections* out) {
  if (!t || !out) return fail(ECF8_EINVAL, "null argument");
  ecf8_sections s{};
  s.n_elem = t->n_elem;
  s.threads_per_block = t->T;
  std::memcpy(s.lengths, t->lengths, 16);
  s.encoded = t->desc.encoded;
  s.encoded_len = t->encoded_len;
  s.gaps = t->desc.gaps;
  s.gaps_len = t->gaps_len;
  s.outpos = t->desc.outpos;
  s.n_outpos = t->n_outpos;
  s.packed = t->desc.packed;
  s.packed_len = t->packed_len;
  *out = s;
  return ECF8_OK;
}

int ecf8_tensor_download(const ecf8_dev_tensor* t, uint8_t* encoded, uint8_t* gaps, uint64_t* outpos,
                         uint8_t* packed) {
  return guarded([&]() -> int {
    if (!t) return fail(ECF8_EINVAL, "null tensor");
    const TensorDesc& d = t->desc;
    if (encoded) cu(cudaMemcpy(encoded, d.encoded, t->encoded_len, cudaMemcpyDeviceToHost), "D2H encoded");
    if (gaps && t->gaps_len) cu(cudaMemcpy(gaps, d.gaps, t->gaps_len, cudaMemcpyDeviceToHost), "D2H gaps");
    if (outpos) cu(cudaMemcpy(outpos, d.outpos, 8 * t->n_outpos, cudaMemcpyDeviceToHost), "D2H outpos");
    if (packed && t->packed_len) cu(cudaMemcpy(packed, d.packed, t->packed_len, cudaMemcpyDeviceToHost), "D2H packed");
    return ECF8_OK;
  });
}

void ecf8_tensor_free(ecf8_dev_tensor* t) {
  if (!t) return;
  free_arena(t);
  delete t;
}

uint64_t ecf8_tensor_n_elem(const ecf8_dev_tensor* t) { return t ? t->n_elem : 0; }
int ecf8_tensor_kernel_variant(const ecf8_dev_tensor* t) { return t && t->n_elem ? tensor_variant(t) : -1; }

uint64_t ecf8_tensor_verified_tiles(const ecf8_dev_tensor* t, uint64_t* total) {
  if (total) *total = t ? t->n_vtiles : 0;
  if (!t || !t->desc.tile_ok || t->n_vtiles == 0) return 0;
  std::vector<std::uint32_t> bits((t->n_vtiles + 31) / 32);
  if (cudaMemcpy(bits.data(), t->desc.tile_ok, 4 * bits.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  std::uint64_t n = 0;
  for (std::uint64_t v = 0; v < t->n_vtiles; ++v) n += (bits[v >> 5] >> (v & 31)) & 1u;
  return n;
}
uint64_t ecf8_tensor_algorithmic_bytes(const ecf8_dev_tensor* t) { return t ? t->algo_bytes : 0; }
uint64_t ecf8_tensor_device_bytes(const ecf8_dev_tensor* t) { return t ? t->arena_bytes : 0; }

int ecf8_decode_device(const ecf8_dev_tensor* t, uint8_t* d_out, void* stream) {
  return guarded([&]() -> int {
    if (!t) return fail(ECF8_EINVAL, "null tensor");
    if (t->n_elem == 0) return ECF8_OK;
    if (!d_out || (reinterpret_cast<std::uintptr_t>(d_out) & 15))
      return fail(ECF8_EINVAL, "device output must be 16-byte aligned");
    TensorDesc d = t->desc;
    d.out = d_out;
    d.out_offset = 0;
    d.tile_begin = 0;
    const int rc = launch_one(d, static_cast<cudaStream_t>(stream), tensor_variant(t));
    note_use(t, static_cast<cudaStream_t>(stream));
    return rc;
  });
}

int ecf8_batch_create(const ecf8_dev_tensor* const* ts, uint8_t* const* d_outs, int count,
                      ecf8_batch** out) {
  return guarded([&]() -> int {
    if (!out || (count > 0 && (!ts || !d_outs))) return fail(ECF8_EINVAL, "null argument");
    *out = nullptr;
    auto b = std::make_unique<ecf8_batch>();
    for (int i = 0; i < count; ++i)
      if (ts[i] && ts[i]->pooled) b->pooled.push_back(ts[i]);
    for (int kw = 0; kw < 8; ++kw) {  // one launch per kernel variant present (ids 0..7)
      std::vector<TensorDesc> group;
      std::uint64_t tiles = 0;
      int kwin_tile = 1;
      for (int i = 0; i < count; ++i) {
        const ecf8_dev_tensor* t = ts[i];
        if (!t) return fail(ECF8_EINVAL, "null tensor");
        const ecf8::dev::Variant v = ecf8::dev::variant_of(t->desc);
        if (t->n_elem == 0 || tensor_variant(t) != kw) continue;
        kwin_tile = v.tile_win;
        if (!d_outs[i] || (reinterpret_cast<std::uintptr_t>(d_outs[i]) & 15))
          return fail(ECF8_EINVAL, "device output must be 16-byte aligned");
        TensorDesc d = t->desc;
        d.out = d_outs[i];
        d.out_offset = 0;
        d.tile_begin = tiles;
        tiles += ecf8::dev::tiles_of(d.T, kwin_tile, t->n_blocks);
        group.push_back(d);
      }
      if (group.empty()) continue;
      TensorDesc* dd = nullptr;
      cu(cudaMalloc(&dd, sizeof(TensorDesc) * group.size()), "cudaMalloc(batch)");
      cu(cudaMemcpy(dd, group.data(), sizeof(TensorDesc) * group.size(), cudaMemcpyHostToDevice), "H2D batch");
      b->d_descs.push_back(dd);
      b->counts.push_back(static_cast<int>(group.size()));
      b->kwins.push_back(kw);
      b->tiles.push_back(tiles);
    }
    *out = b.release();
    return ECF8_OK;
  });
}

int ecf8_batch_decode(const ecf8_batch* b, void* stream) {
  return guarded([&]() -> int {
    if (!b) return fail(ECF8_EINVAL, "null batch");
    for (std::size_t g = 0; g < b->d_descs.size(); ++g) {
      ecf8::dev::LaunchArgs a{};
      a.descs = b->d_descs[g];
      a.n_desc = b->counts[g];
      a.total_tiles = b->tiles[g];
      cu(ecf8::dev::launch_decode(a, b->kwins[g], static_cast<cudaStream_t>(stream)), "decode launch");
    }
    for (const ecf8_dev_tensor* t : b->pooled) note_use(t, static_cast<cudaStream_t>(stream));
    return ECF8_OK;
  });
}

int ecf8_batch_launches(const ecf8_batch* b) { return b ? static_cast<int>(b->d_descs.size()) : 0; }

void ecf8_batch_free(ecf8_batch* b) {
  if (!b) return;
  for (TensorDesc* p : b->d_descs) cudaFree(p);
  delete b;
}

int ecf8_decode_host(const ecf8_sections* s, uint8_t* out, uint64_t out_len) {
  return guarded([&]() -> int {
    if (!s) return fail(ECF8_EINVAL, "null sections");
    if (out_len != s->n_elem) return fail(ECF8_EINVAL, "output size mismatch");
    std::uint64_t nb = 0;
    if (int rc = validate(s, &nb)) return rc;
    if (s->n_elem == 0) return ECF8_OK;
    if (int rc = require_device()) return rc;
    return host_pipeline(&s, &nb, &out, 1);
  });
}

int ecf8_decode_host_many(const ecf8_sections* const* ss, uint8_t* const* outs, const uint64_t* out_lens,
                          int count) {
  return guarded([&]() -> int {
    if (count < 0 || (count > 0 && (!ss || !outs || !out_lens))) return fail(ECF8_EINVAL, "null argument");
    std::vector<std::uint64_t> nbs(static_cast<std::size_t>(count));
    bool any = false;
    for (int i = 0; i < count; ++i) {
      if (!ss[i]) return fail(ECF8_EINVAL, "null sections");
      if (out_lens[i] != ss[i]->n_elem) return fail(ECF8_EINVAL, "output size mismatch");
      if (int rc = validate(ss[i], &nbs[i])) return rc;
      if (ss[i]->n_elem && !outs[i]) return fail(ECF8_EINVAL, "null argument");
      any |= ss[i]->n_elem > 0;
    }
    if (!any) return ECF8_OK;
    if (int rc = require_device()) return rc;
    return host_pipeline(ss, nbs.data(), outs, count);
  });
}

int ecf8_decode_host_stream(const ecf8_sections* const* ss, int count, uint8_t* buf, uint64_t buf_len,
                            ecf8_chunk_fn fn, void* ctx) {
  return guarded([&]() -> int {
    if (count < 0 || (count > 0 && (!ss || !fn))) return fail(ECF8_EINVAL, "null argument");
    std::vector<std::uint64_t> nbs(static_cast<std::size_t>(count));
    bool any = false;
    for (int i = 0; i < count; ++i) {
      if (!ss[i]) return fail(ECF8_EINVAL, "null sections");
      if (ss[i]->n_elem > buf_len) return fail(ECF8_EINVAL, "output size mismatch");
      if (int rc = validate(ss[i], &nbs[i])) return rc;
      any |= ss[i]->n_elem > 0;
    }
    if (!any) return ECF8_OK;
    if (!buf) return fail(ECF8_EINVAL, "null argument");
    if (!is_pinned(buf)) return fail(ECF8_EINVAL, "stream buffer must be page-locked");
    if (int rc = require_device()) return rc;
    std::vector<std::uint8_t*> outs(static_cast<std::size_t>(count), buf);
    StreamSink sink;
    sink.fn = fn;
    sink.ctx = ctx;
    if (int rc = host_pipeline(ss, nbs.data(), outs.data(), count, nullptr, nullptr, &sink)) return rc;
    if (sink.rc) return fail(ECF8_EIO, "chunk sink failed");
    return ECF8_OK;
  });
}

int ecf8_decode_block_host(const ecf8_sections* s, uint64_t block, uint8_t* out, uint64_t out_len) {
  return guarded([&]() -> int {
    std::uint64_t nb = 0;
    if (int rc = validate(s, &nb)) return rc;
    if (block >= nb) return fail(ECF8_EINVAL, "block index out of range");
    if (out_len < s->outpos[block + 1]) return fail(ECF8_EINVAL, "output size mismatch");
    if (s->outpos[block + 1] == s->outpos[block]) return ECF8_OK;
    if (int rc = require_device()) return rc;
    // only this block's sections go to the device (decode_block, codec.cpp:201-254)
    const std::uint64_t hi = block + 1;
    return host_pipeline(&s, &nb, &out, 1, &block, &hi);
  });
}

int ecf8_count_window(const uint8_t window10[10], unsigned gap, const uint8_t lengths[16],
                      uint32_t* count) {
  return guarded([&]() -> int {
    if (!window10 || !lengths || !count) return fail(ECF8_EINVAL, "null argument");
    try {
      (void)ecf8::dev::tables_for(lengths);
    } catch (const std::invalid_argument&) {
      return fail(ECF8_EINVAL, "invalid length vector");
    }
    if (int rc = require_device()) return rc;
    const DevTables& tb = device_tables(lengths);
    struct Scratch {
      std::uint8_t* win = nullptr;
      std::uint32_t* cnt = nullptr;
    };
    thread_local Scratch sc;
    if (!sc.win) {
      cu(cudaMalloc(&sc.win, 16), "cudaMalloc");
      cu(cudaMalloc(&sc.cnt, 4), "cudaMalloc");
    }
    std::uint8_t w16[16] = {0};
    std::memcpy(w16, window10, 10);
    cu(cudaMemcpy(sc.win, w16, 16, cudaMemcpyHostToDevice), "H2D window");
    TensorDesc td{};
    td.fast = tb.fast;
    td.smask = tb.smask;
    td.cascade = tb.cascade;
    td.n_luts = tb.n_luts;
    cu(ecf8::dev::launch_count_window(sc.win, gap & 15, td, sc.cnt, nullptr), "count launch");
    cu(cudaMemcpy(count, sc.cnt, 4, cudaMemcpyDeviceToHost), "D2H count");
    return ECF8_OK;
  });
}


// ---- decode-fused FP8 GEMM (fused_gemm.cu) -------------------------------

int ecf8_fused_create(const ecf8_dev_tensor* t, uint64_t n, uint64_t k, int w_fmt, ecf8_fused** out) {
  return guarded([&]() -> int {
    if (!t || !out) return fail(ECF8_EINVAL, "null argument");
    *out = nullptr;
    if (n == 0 || k == 0 || n % 128 || k % 128) return fail(ECF8_EINVAL, "fused GEMM needs n, k multiples of 128");
    if (t->n_elem != n * k) return fail(ECF8_EINVAL, "output size mismatch");
    if (w_fmt != 0 && w_fmt != 1) return fail(ECF8_EINVAL, "weight format must be 0 (E4M3) or 1 (E5M2)");
    if (ecf8::dev::fused_lane_windows(t->T, t->desc.lmin) == 0)
      return fail(ECF8_EINVAL, "fused GEMM needs T in [4, 128], or T = 256 (T <= 128 when a code word is 1 bit)");
    if (int rc = require_device()) return rc;
    std::vector<std::uint64_t> outpos(t->n_blocks + 1);
    cu(cudaMemcpy(outpos.data(), t->desc.outpos, 8 * outpos.size(), cudaMemcpyDeviceToHost), "D2H outpos");
    const std::vector<std::uint64_t>& outpos_ref = outpos;
    // whole waves of the SMs (one CTA per SM); as few waves as keep every
    // CTA's run of tiles within max_seg n-tiles (one TMEM accumulator each)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const std::uint64_t KT = k / 128, total = (n / 128) * KT;
    auto f = std::make_unique<ecf8_fused>();
    f->w = t;
    f->n = n;
    f->k = k;
    f->w_fmt = static_cast<std::uint32_t>(w_fmt);
    auto make_plan = [&](std::uint64_t ctas) {
      std::vector<ecf8::dev::FusedCta> plan;
      for (std::uint64_t c = 0; c < ctas; ++c) {
        ecf8::dev::FusedCta p{};
        p.tile0 = static_cast<std::uint32_t>(total * c / ctas);
        p.tile1 = static_cast<std::uint32_t>(total * (c + 1) / ctas);
        p.e0 = std::uint64_t{p.tile0} * 16384;
        p.e1 = std::uint64_t{p.tile1} * 16384;
        // blocks overlapping [e0, e1): the block holding element e0 .. first block starting >= e1
        auto ub = std::upper_bound(outpos.begin(), outpos.end() - 1, p.e0);
        p.blk_begin = static_cast<std::uint64_t>(ub - outpos.begin()) - 1;
        auto lb = std::lower_bound(outpos.begin(), outpos.end(), p.e1);
        p.blk_end = std::min<std::uint64_t>(static_cast<std::uint64_t>(lb - outpos.begin()), t->n_blocks);
        plan.push_back(p);
      }
      return plan;
    };
    auto segs = [&](const std::vector<ecf8::dev::FusedCta>& plan) {
      std::uint32_t m = 1;
      for (const auto& p : plan)
        if (p.tile1 > p.tile0) m = std::max<std::uint32_t>(m, static_cast<std::uint32_t>((p.tile1 - 1) / KT - p.tile0 / KT + 1));
      return m;
    };
    // accumulators are reused round-robin within a CTA, so every plan is one
    // wave (ECF8_FUSED_SEG_CAP: A/B runs with a segment cap instead)
    static const std::uint32_t seg_cap = [] {
      const char* e = std::getenv("ECF8_FUSED_SEG_CAP");
      return e ? static_cast<std::uint32_t>(std::strtoul(e, nullptr, 10)) : 0u;
    }();
    const std::uint32_t caps[2] = {seg_cap ? seg_cap : ~0u, seg_cap ? seg_cap : ~0u};
    for (int i = 0; i < 2; ++i) {
      std::vector<ecf8::dev::FusedCta> plan;
      static const std::uint64_t min_waves = [] {  // A/B runs only
        const char* e = std::getenv("ECF8_FUSED_MIN_WAVES");
        return e ? std::max<std::uint64_t>(1, std::strtoull(e, nullptr, 10)) : std::uint64_t{1};
      }();
      for (std::uint64_t waves = min_waves;; ++waves) {
        plan = make_plan(std::min<std::uint64_t>(total, waves * static_cast<std::uint64_t>(sms)));
        if (segs(plan) <= caps[i] || plan.size() == total) break;
      }
      f->n_cta[i] = static_cast<std::uint32_t>(plan.size());
      f->max_seg[i] = segs(plan);
      cu(cudaMalloc(&f->d_plan[i], sizeof(ecf8::dev::FusedCta) * plan.size()), "cudaMalloc(plan)");
      cu(cudaMemcpy(f->d_plan[i], plan.data(), sizeof(ecf8::dev::FusedCta) * plan.size(), cudaMemcpyHostToDevice),
         "H2D plan");
    }
    f->split_k = static_cast<std::uint32_t>((f->n_cta[1] + n / 128 - 1) / (n / 128));
    // byte-step direct decode when every verification tile is direct (the
    // upload check's tile_direct bits) -- always, for encoder-written weights
    static const bool no_fsm = std::getenv("ECF8_FUSED_NO_FSM") != nullptr;  // A/B runs
    if (!no_fsm && t->desc.fsm && t->desc.lane_start && t->T >= 8 && t->T <= 256) {
      std::vector<std::uint32_t> bits((t->n_vtiles + 31) / 32);
      cu(cudaMemcpy(bits.data(), t->desc.tile_direct, 4 * bits.size(), cudaMemcpyDeviceToHost), "D2H tile_direct");
      bool all = true;
      for (std::uint64_t v = 0; v < t->n_vtiles; ++v) all &= ((bits[v >> 5] >> (v & 31)) & 1u) != 0;
      f->fsm = all;
    }
    f->outpos = outpos_ref;
    *out = f.release();
    return ECF8_OK;
  });
}

int ecf8_fused_decode_rows(const ecf8_fused* f, uint64_t row0, uint64_t row1, uint8_t* d_rows, void* stream) {
  return guarded([&]() -> int {
    if (!f || !d_rows) return fail(ECF8_EINVAL, "null argument");
    if (row0 >= row1 || row1 > f->n || row0 % 128 || row1 % 128)
      return fail(ECF8_EINVAL, "rows must be a non-empty range of whole 128-row tiles");
    if (reinterpret_cast<std::uintptr_t>(d_rows) & 15) return fail(ECF8_EINVAL, "device output must be 16-byte aligned");
    if (!f->fsm) return fail(ECF8_EINVAL, "row decode needs a byte-step weight with every tile direct");
    const std::uint64_t KT = f->k / 128;
    const std::uint64_t e0 = row0 / 128 * KT * 16384, e1 = row1 / 128 * KT * 16384;
    TensorDesc d = f->w->desc;
    const std::uint64_t T = d.T, m = std::max<std::uint64_t>(1, 256 / T);  // blocks per warp tile
    // blocks holding [e0, e1), widened to whole warp tiles of the tensor
    const auto& op = f->outpos;
    std::uint64_t b0 = static_cast<std::uint64_t>(std::upper_bound(op.begin(), op.end() - 1, e0) - op.begin()) - 1;
    std::uint64_t b1 = static_cast<std::uint64_t>(std::lower_bound(op.begin(), op.end(), e1) - op.begin());
    b1 = std::min<std::uint64_t>(b1, f->w->n_blocks);
    b0 = b0 / m * m;
    b1 = std::min<std::uint64_t>((b1 + m - 1) / m * m, f->w->n_blocks);
    d.blk_begin = b0;
    d.blk_end = b1;
    d.out = d_rows - row0 * f->k;  // row-major W[0][0] (only rows [row0, row1) are written)
    d.out_offset = 0;
    d.out_tiled_k = static_cast<std::uint32_t>(f->k);
    d.out_lo = e0;
    d.out_hi = e1;
    if (int rc = launch_one(d, static_cast<cudaStream_t>(stream))) return rc;
    note_use(f->w, static_cast<cudaStream_t>(stream));
    return ECF8_OK;
  });
}

int ecf8_fused_byte_steps(const ecf8_fused* f) { return f && f->fsm ? 1 : 0; }

int ecf8_fused_split_k(const ecf8_fused* f) { return f ? static_cast<int>(f->split_k) : 0; }

// Workspace of the fused GEMM calls on one stream, shared by every weight:
// the swizzled X tiles (x_tiles_kernel, grow-only) and the L2-ring variant's
// per-CTA rings (kRingSlots K tiles for each of up to one wave of CTAs,
// allocated once at full size).  Calls on one stream may share it: the next
// call's x_tiles_kernel writes X only after griddepcontrol.wait (the previous
// fused grid complete), and its decode warps write the rings only after the
// same wait (GRingOut::wait).  Calls on different streams may run at once,
// so every stream has its own.  Never freed (a process-lifetime cache, like
// the decode tables); growing X waits for the stream.
struct FusedWorkspace {
  std::mutex mu;  // held by a call from the X growth to its launches (host threads sharing a stream)
  std::uint8_t* xt = nullptr;
  std::uint64_t xt_cap = 0;
  std::uint8_t* ring = nullptr;
  std::uint32_t ring_ctas = 0;
};

FusedWorkspace& fused_workspace(cudaStream_t st) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, FusedWorkspace> all;
  int dev = 0;
  cu(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  FusedWorkspace& w = all[{dev, st}];
  if (!w.ring) {
    int sms = 0;
    cu(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    cu(cudaMalloc(&w.ring, static_cast<std::uint64_t>(sms) * ecf8::dev::kRingSlots * 16384), "cudaMalloc(fused rings)");
    w.ring_ctas = static_cast<std::uint32_t>(sms);
  }
  return w;
}

// (caller holds w.mu)
void grow_x_tiles(FusedWorkspace& w, std::uint64_t need, cudaStream_t st) {
  if (need <= w.xt_cap) return;
  if (w.xt) {
    cu(cudaStreamSynchronize(st), "sync");  // the stream's earlier calls are done with it
    cudaFree(w.xt);
    w.xt = nullptr;
    w.xt_cap = 0;
  }
  cu(cudaMalloc(&w.xt, need), "cudaMalloc(x tiles)");
  w.xt_cap = need;
}

int ecf8_fused_gemm(const ecf8_fused* f, const uint8_t* d_x, uint32_t m, float scale, float* d_y, void* stream) {
  return guarded([&]() -> int {
    if (!f || !d_x || !d_y) return fail(ECF8_EINVAL, "null argument");
    if (m == 0 || m > 256) return fail(ECF8_EINVAL, "fused GEMM supports 1 <= m <= 256 tokens");
    if ((reinterpret_cast<std::uintptr_t>(d_x) & 15) || (reinterpret_cast<std::uintptr_t>(d_y) & 15))
      return fail(ECF8_EINVAL, "x and y must be 16-byte aligned");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    ecf8::dev::FusedArgs a{};
    a.w = f->w->desc;
    const int pi = m <= 128 ? 1 : 0;  // accumulator columns <= 128: up to four n-tile segments per CTA
    a.plan = f->d_plan[pi];
    a.x = d_x;
    a.y = d_y;
    FusedWorkspace& ws = fused_workspace(st);
    std::lock_guard<std::mutex> ws_lock(ws.mu);
    grow_x_tiles(ws, f->k * ((m + 15) / 16 * 16), st);
    a.xt = ws.xt;
    a.m = m;
    a.m_pad = (m + 15) / 16 * 16;
    a.n = static_cast<std::uint32_t>(f->n);
    a.k = static_cast<std::uint32_t>(f->k);
    a.split_k = f->split_k;
    a.fsm = f->fsm ? 1u : 0u;
    a.stages_a = ecf8::dev::fused_stages_a(
        a.m_pad, ecf8::dev::fused_warp_smem(f->w->T, f->w->desc.lmin, a.m_pad, f->fsm), f->fsm);
    a.stages_b = ecf8::dev::fused_stages_b(a.m_pad, f->fsm);
    // byte-step weights: the L2-ring variant (decode warps as the standalone
    // decoder, decoded K tiles through a per-CTA ring in L2); ECF8_FUSED_L2=0: the shared-memory ring
    static const bool l2 = [] {
      const char* e = std::getenv("ECF8_FUSED_L2");
      return !e || std::atoi(e) != 0;
    }();
    a.scratch = nullptr;
    // (plans of more than one wave -- the ECF8_FUSED_MIN_WAVES / SEG_CAP A/B switches -- use the shared-memory ring)
    if (l2 && f->fsm && ecf8::dev::fused_l2_stages(a.m_pad) >= 2 && f->n_cta[pi] <= ws.ring_ctas) {
      a.scratch = ws.ring;
      a.stages_a = ecf8::dev::fused_l2_stages(a.m_pad);
      a.stages_b = a.stages_a;
    }
    if (a.stages_a < 2) return fail(ECF8_EINVAL, "fused GEMM: shared memory too small for this m");
    a.acc_cols = 32;
    while (a.acc_cols < a.m_pad) a.acc_cols <<= 1;
    // one accumulator per n-tile segment of a CTA while they fit the 512
    // TMEM columns; beyond that they are reused round-robin (flushed first)
    a.tmem_cols = 32;
    while (a.tmem_cols < f->max_seg[pi] * a.acc_cols && a.tmem_cols < 512) a.tmem_cols <<= 1;
    a.acc_bufs = std::min<std::uint32_t>(a.tmem_cols / a.acc_cols, ecf8::dev::kMaxAccBufs);
    a.w_fmt = f->w_fmt;
    a.scale = scale;
    cu(ecf8::dev::launch_fused_gemm(a, f->n_cta[pi], st), "fused GEMM launch");
    note_use(f->w, st);
    return ECF8_OK;
  });
}

void ecf8_fused_free(ecf8_fused* f) {
  if (!f) return;
  for (auto* p : f->d_plan)
    if (p) cudaFree(p);
  delete f;
}

int ecf8_fused_layout_device(const uint8_t* d_in, uint64_t n, uint64_t k, uint8_t* d_out, int inverse, void* stream) {
  return guarded([&]() -> int {
    if (!d_in || !d_out) return fail(ECF8_EINVAL, "null argument");
    if (n % 128 || k % 128) return fail(ECF8_EINVAL, "fused layout needs n, k multiples of 128");
    if ((reinterpret_cast<std::uintptr_t>(d_in) | reinterpret_cast<std::uintptr_t>(d_out)) & 15)
      return fail(ECF8_EINVAL, "device buffers must be 16-byte aligned");
    if (int rc = require_device()) return rc;
    cu(ecf8::dev::launch_fused_layout(d_in, n, k, d_out, inverse != 0, static_cast<cudaStream_t>(stream)),
       "fused layout launch");
    return ECF8_OK;
  });
}

int ecf8_host_pin(void* p, uint64_t bytes) {
  return guarded([&]() -> int {
    if (!p || !bytes) return ECF8_OK;
    if (int rc = require_device()) return rc;
    const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
      cudaGetLastError();
      return ECF8_OK;
    }
    cu(e, "cudaHostRegister");
    return ECF8_OK;
  });
}

int ecf8_host_alloc_pinned(uint64_t bytes, void** out) {
  return guarded([&]() -> int {
    if (!out) return fail(ECF8_EINVAL, "null argument");
    *out = nullptr;
    if (!bytes) return ECF8_OK;
    if (int rc = require_device()) return rc;
    if (cudaMallocHost(out, bytes) != cudaSuccess) {
      cudaGetLastError();
      *out = nullptr;
      return fail(ECF8_ENOMEM, "cudaMallocHost failed");
    }
    return ECF8_OK;
  });
}

int ecf8_host_free_pinned(void* p) {
  return guarded([&]() -> int {
    if (p) cu(cudaFreeHost(p), "cudaFreeHost");
    return ECF8_OK;
  });
}

int ecf8_host_unpin(void* p) {
  return guarded([&]() -> int {
    if (!p) return ECF8_OK;
    const cudaError_t e = cudaHostUnregister(p);
    if (e == cudaErrorHostMemoryNotRegistered) {
      cudaGetLastError();
      return ECF8_OK;
    }
    cu(e, "cudaHostUnregister");
    return ECF8_OK;
  });
}

}  // extern "C"

extern "C" int ecf8_internal_require_device(void) { return require_device(); }
