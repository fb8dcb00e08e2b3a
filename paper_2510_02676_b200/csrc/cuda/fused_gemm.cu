// fused_gemm.cu -- decode-fused tcgen05 FP8 GEMM.
//
//   Y[M, N] (fp32) = scale * X[M, K] (E4M3) . W[N, K]^T (E4M3 / E5M2)
//
// W stays ECF8-compressed in HBM and is decoded straight into shared memory;
// the decoded weights never touch HBM.  There is no reference counterpart:
// the paper decodes a layer into a buffer and then runs the GEMM
// (PAPER.md:170-173); this kernel fuses the two.
//
// Fused weight layout ("tiled" ECF8 tensor, ecf8_host_fused_layout): W is cut
// into 128 x 128 tiles, tile (nt, kt) in row-major tile order, and each
// tile's 16384 bytes are stored in the exact shared-memory image the tensor
// core reads: K-major, 128-byte rows, 128B swizzle (16-byte chunk c of row r
// at r*128 + ((c ^ (r & 7)) << 4)).  The tiled byte sequence is an ordinary
// 1-D tensor for the (unchanged) ECF8 encoder.  A decoded element's tile-
// major index therefore IS its shared-memory offset within its tile.
//
// CTA = a contiguous run of weight tiles in tile-major order, balanced over
// the launch (a whole number of waves of the 148 SMs, one CTA per SM); a run
// spans at most two n-tiles, each accumulated in its own TMEM block, and the
// partial rows are added into y with red.global.add.f32.  Warp roles:
//   decode warps (20; 12 for 1-bit codes)  claim ECF8 warp tiles (decode_warp.cuh)
//       covering the CTA's element range in order, decode them into their
//       nibble slots, then merge exponent + sign/mantissa nibbles and store
//       the FP8 bytes straight into the A ring stage of their K tile; each
//       warp arrives on the stage's "full" mbarrier with the number of bytes
//       it wrote (a stage completes at 16384 bytes).
//   control warp   allocates TMEM, streams X K-tiles (pre-swizzled by
//       x_tiles_kernel) into a B ring (2 stages; 1 when m > 128 so the A ring
//       keeps 5 stages) by bulk async copy, and one lane
//       issues
//       tcgen05.mma.cta_group::1.kind::f8f6f4 (M = 128 W rows, N = padded
//       token count, K = 32 per instruction, 4 per K tile) with the fp32
//       accumulator in TMEM; tcgen05.commit frees A / B stages.
//   epilogue       decode warps 0-3 (TMEM lane quadrants) read the
//       accumulator with tcgen05.ld.32x32b and write Y^T rows coalesced.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "decode.cuh"
#include "decode_common.cuh"
#include "decode_warp.cuh"
#include "fused_gemm.cuh"

namespace ecf8::dev {

namespace {

#ifndef ECF8_FUSED_WARPS
#define ECF8_FUSED_WARPS 24
#endif
// Decode warps per CTA.  Half-size warp tiles (LW 4, 17 slot rows): 24
// (measured on a 28672x8192 weight at m = 1: 16 -> 211, 20 -> 196, 22 -> 190,
// 24 -> 184, 26 -> 197 us).  For m > 128 (WIDE) one 32 KB X stage keeps room
// for three A stages: 24 warps / 1 X stage 236 us, 16 / 2 264 us, 22 / 2 287
// us (two A stages) at m = 256.  Lanes holding 256 symbols (LW 8, or
// 64-symbol windows): 12.
#ifndef ECF8_FUSED_WIDE_WARPS
#define ECF8_FUSED_WIDE_WARPS 24
#endif
#ifndef ECF8_FUSED_WIDE_XSTAGES
#define ECF8_FUSED_WIDE_XSTAGES 1
#endif
#ifndef ECF8_FUSED_FSM_WIDE_WARPS
#define ECF8_FUSED_FSM_WIDE_WARPS 12  // m > 128
#endif
#ifndef ECF8_FUSED_FSM_WIDE_XSTAGES
#define ECF8_FUSED_FSM_WIDE_XSTAGES 1
#endif
#ifndef ECF8_FUSED_FSM_WARPS
#define ECF8_FUSED_FSM_WARPS 12
#endif
#ifndef ECF8_FUSED_GPK
#define ECF8_FUSED_GPK 0  // 1: packed bytes read from L2 at write-back instead of staged (A/B: slower)
#endif
#ifndef ECF8_FUSED_CHAIN
#define ECF8_FUSED_CHAIN 1  // consecutive fused GEMMs overlap (x_tiles_kernel as a programmatic dependent)
#endif
#ifndef ECF8_FUSED_XPROBE
#define ECF8_FUSED_XPROBE 0
#endif
#ifndef ECF8_FUSED_MMAPROBE
#define ECF8_FUSED_MMAPROBE 0
#endif
#ifndef ECF8_FUSED_EPI
#define ECF8_FUSED_EPI 1  // 0: timing experiment without the epilogue's y updates (wrong results)
#endif
// Byte-step variant: 8-window lanes, two chains each (direct_tile), 4.2 KB of
// warp state (the staging tile): ECF8_FUSED_FSM_WARPS decode warps.
template <int LW, int ROWS, bool WIDE, bool FSM = false>
constexpr int decode_warps() {
  return FSM ? (WIDE ? ECF8_FUSED_FSM_WIDE_WARPS : ECF8_FUSED_FSM_WARPS)
             : ROWS > 17 ? 12 : (WIDE ? ECF8_FUSED_WIDE_WARPS : ECF8_FUSED_WARPS);
}
constexpr std::uint32_t kTileElems = 128 * 128;  // one K tile of A (bytes)


__shared__ Tables g_tbf;
__shared__ alignas(16) std::uint32_t g_fsmf[256 * kFsmStates];  // byte-step variant: its tables
__shared__ alignas(16) std::uint8_t g_cmf[256 * kFsmStates];
__shared__ TensorDesc g_wdesc;  // this CTA's weight descriptor (read where used: frees ~30 registers)
__shared__ unsigned g_qnext;
__shared__ alignas(8) unsigned long long g_full[kMaxStagesA];
__shared__ alignas(8) unsigned long long g_empty[kMaxStagesA];  // arrived by tcgen05.commit (MMAs done)
__shared__ alignas(8) unsigned long long g_free[kMaxStagesA];   // arrived by the MMA lane once it saw g_empty
__shared__ alignas(8) unsigned long long g_bfull[2];
__shared__ alignas(8) unsigned long long g_segdone[kMaxAccBufs];  // arrived by tcgen05.commit after a segment's last MMA
__shared__ alignas(8) unsigned long long g_accfree[kMaxAccBufs];  // arrived by the 4 flushing warps once they read it
__shared__ std::uint32_t g_nflush[16];  // per flushing warp: the next segment it flushes
__shared__ std::uint32_t g_tmem;
__shared__ std::uint32_t g_consumed;  // K tiles whose MMAs have completed (stage reusable)

// ---- PTX helpers ---------------------------------------------------------

__device__ __forceinline__ void mbar_init(std::uint32_t bar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(std::uint32_t bar, std::uint32_t count) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(bar),
               "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(std::uint32_t bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Waits that back off: a spinning try_wait loop steals issue slots from the
// decode warps sharing the scheduler.
__device__ __forceinline__ void mbar_wait_sleep(std::uint32_t bar, std::uint32_t parity, unsigned ns) {
  for (;;) {
    std::uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(ns);
  }
}

__device__ __forceinline__ std::uint32_t mbar_try(std::uint32_t bar, std::uint32_t parity) {
  std::uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok;
}

// Non-blocking probe (test_wait; try_wait may suspend the thread for a while).
__device__ __forceinline__ std::uint32_t mbar_test(std::uint32_t bar, std::uint32_t parity) {
  std::uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok;
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(std::uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

// K-major, 128-byte rows, 128B swizzle, 8-row groups 1024 bytes apart.
__device__ __forceinline__ std::uint64_t smem_desc(std::uint32_t saddr) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((saddr >> 4) & 0x3FFF);  // start address
  d |= static_cast<std::uint64_t>(1) << 16;                 // leading byte offset (unused for SW128 K-major)
  d |= static_cast<std::uint64_t>(1024 >> 4) << 32;         // stride byte offset
  d |= static_cast<std::uint64_t>(1) << 46;                 // descriptor version (sm_100)
  d |= static_cast<std::uint64_t>(2) << 61;                 // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_f8(std::uint32_t tmem_d, std::uint64_t adesc, std::uint64_t bdesc,
                                       std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(std::uint32_t taddr, float (&v)[8]) {
  std::uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- decode warps: one ECF8 tile -> FP8 bytes in the A ring ---------------

struct Flush;
struct Ring {
  std::uint32_t a_base;  // shared address of A stage 0 (1024-aligned)
  std::uint32_t stages;  // A stages
  std::uint64_t e0, e1;  // CTA element range (tile-major), multiples of 16384
  const Flush* fl;       // this warp's accumulator flushes (polled while waiting)
};

// Writers of K tile t need stage t % S back from the MMAs of tile t - S
// (completion u - 1 of that stage's "free" barrier, u = t / S).  The MMA
// lane arrives on "free" after it has waited for the stage's "empty"
// barrier (tcgen05.commit): a thread-to-thread release/acquire chain
// (writer -> full -> MMA lane -> free -> next writer) that compute-sanitizer
// racecheck can follow, which a hardware-arrived barrier is not.  Decode
// warps run up to ~8 K tiles ahead of the MMA, so a bare parity wait could
// alias a completion two phases back; the control warp's monotonic count of
// consumed K tiles first guarantees the barrier is at most one phase behind
// (tile t - 2S consumed), then the parity wait does the rest.
// ---- accumulator flushes: partial rows of finished n-tile segments -> y
//
// A CTA's run covers segments s = 0 .. nseg-1 (n-tiles), accumulated in
// TMEM buffer s % nb (nb = accumulator buffers that fit the 512 columns).
// The MMA lane commits g_segdone[b] after a segment's last MMA; warps 0-3
// (one TMEM lane quadrant each) read the buffer with tcgen05.ld, add the
// partial rows into y, and arrive on g_accfree[b], which the MMA lane waits
// for before it starts segment s + nb in the same buffer.  Warps 0-3 flush
// between their decode tiles and while they wait for ring stages, so a
// segment's epilogue overlaps the decode of the next ones; only the last
// segment is flushed after the CTA's decode work.
struct Flush {
  const FusedArgs* a;  // the kernel's parameters (__grid_constant__: read in place)
  std::uint32_t tmem_d, nt0, nseg;
  std::uint32_t nfw = 4;  // mid-run flushing warps 0 .. nfw-1 (4, 8, 12, 16): warp w flushes quadrant w % 4, column
                          // groups w / 4, w / 4 + nfw / 4, ...; g_accfree counts nfw arrivals

  __device__ __forceinline__ void segment(std::uint32_t sg) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const std::uint32_t b = sg % a->acc_bufs;
    const std::uint32_t row = static_cast<std::uint32_t>(warp) * 32 + static_cast<std::uint32_t>(lane);
    const std::uint64_t col = static_cast<std::uint64_t>(nt0 + sg) * 128 + row;
    const std::uint32_t tq = tmem_d + b * a->acc_cols + (static_cast<std::uint32_t>(warp * 32) << 16);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // y zeroed by x_tiles_kernel (returns at once after)
    const std::uint32_t m = a->m;
    for (std::uint32_t c0 = 0; c0 < m; c0 += 8) {
      float v[8];
      tmem_ld8(tq + c0, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const std::uint32_t mcol = c0 + j;
#if ECF8_FUSED_EPI
        if (mcol < m) atomicAdd(a->y + static_cast<std::uint64_t>(mcol) * a->n + col, v[j] * a->scale);
#else
        if (mcol < m && v[j] == 12345.f) a->y[0] = 0.f;  // timing experiment only: no y updates
#endif
      }
    }
  }
  // Columns [c_begin, m) step c_step of segment sg's TMEM lane quadrant q.
  __device__ __forceinline__ void segment_cols(std::uint32_t sg, std::uint32_t q, std::uint32_t c_begin,
                                               std::uint32_t c_step) const {
    const int lane = threadIdx.x & 31;
    const std::uint32_t b = sg % a->acc_bufs;
    const std::uint64_t col = static_cast<std::uint64_t>(nt0 + sg) * 128 + q * 32 + static_cast<std::uint32_t>(lane);
    const std::uint32_t tq = tmem_d + b * a->acc_cols + ((q * 32) << 16);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const std::uint32_t m = a->m;
    for (std::uint32_t c0 = c_begin; c0 < m; c0 += c_step) {
      float v[8];
      tmem_ld8(tq + c0, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const std::uint32_t mcol = c0 + j;
        if (mcol < m) atomicAdd(a->y + static_cast<std::uint64_t>(mcol) * a->n + col, v[j] * a->scale);
      }
    }
  }
  // After the decode: the segments not flushed yet, by all nw decode warps
  // (warp w reads TMEM lane quadrant w % 4; the warps of a quadrant split its
  // columns 8 at a time).  Named barrier 1 over the decode warps: before
  // (every mid-run flush is done, g_nflush final) and after each segment
  // (its buffer's columns all read before the quadrant's arrival frees it).
  __device__ __forceinline__ void run_final(int nw) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const std::uint32_t q = static_cast<std::uint32_t>(warp) & 3u, part = static_cast<std::uint32_t>(warp) >> 2;
    const std::uint32_t parts = (static_cast<std::uint32_t>(nw) - q + 3) / 4;
    const std::uint32_t nb = a->acc_bufs, nh = nfw / 4;
    asm volatile("bar.sync 1, %0;" ::"r"(nw * 32) : "memory");
    std::uint32_t f0 = g_nflush[0];
    for (std::uint32_t w = 1; w < nfw; ++w) f0 = min(f0, g_nflush[w]);
    for (std::uint32_t f = f0; f < nseg; ++f) {
      // the column groups of quadrant q whose mid-run flusher has not done f,
      // split over the quadrant's warps
      bool waited = false;
      for (std::uint32_t h = 0; h < nh; ++h) {
        if (f < g_nflush[q + 4 * h]) continue;
        if (!waited) {
          mbar_wait(smem_addr(&g_segdone[f % nb]), (f / nb) & 1u);
          tc_fence_after();
          waited = true;
        }
        segment_cols(f, q, 8 * h + 8 * nh * part, 8 * nh * parts);
      }
      if (waited) tc_fence_before();
      asm volatile("bar.sync 1, %0;" ::"r"(nw * 32) : "memory");
      if (static_cast<std::uint32_t>(warp) < nfw && f >= g_nflush[warp] && lane == 0)
        mbar_arrive(smem_addr(&g_accfree[f % nb]), 1);
    }
  }
  // Flush every finished segment (block: wait for each until all are done).
  __device__ __forceinline__ void run(bool block) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (static_cast<std::uint32_t>(warp) >= nfw) return;
    const std::uint32_t nh = nfw / 4;
    const std::uint32_t nb = a->acc_bufs;
    for (;;) {
      const std::uint32_t f = g_nflush[warp];
      if (f >= nseg) return;
      const std::uint32_t bar = smem_addr(&g_segdone[f % nb]), par = (f / nb) & 1u;
      if (block) mbar_wait(bar, par);
      else if (!__all_sync(0xffffffffu, mbar_test(bar, par))) return;
      tc_fence_after();
      if (nh == 1) segment(f);
      else segment_cols(f, static_cast<std::uint32_t>(warp) & 3u, 8 * (static_cast<std::uint32_t>(warp) >> 2), 8 * nh);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(smem_addr(&g_accfree[f % nb]), 1);
        g_nflush[warp] = f + 1;
      }
      __syncwarp();
    }
  }
  __device__ __forceinline__ void operator()() const { run(false); }
};

#ifndef ECF8_FUSED_MIDFLUSH
#define ECF8_FUSED_MIDFLUSH 1
#endif
#ifndef ECF8_FUSED_POLL
#define ECF8_FUSED_POLL 1  // 0: A/B only (no flushes while waiting: deadlocks when accumulators are reused)
#endif
template <class Poll>
__device__ __forceinline__ void wait_stage_free(const Ring& R, std::uint32_t t, const Poll& poll) {
  if (t < R.stages) return;
#if !ECF8_FUSED_POLL
  if (t >= 2 * R.stages) {
    const std::uint32_t need = t - 2 * R.stages + 1;
    const std::uint32_t addr = smem_addr(&g_consumed);
    while (true) {
      std::uint32_t v;
      asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
      if (v >= need) break;
      __nanosleep(128);
    }
  }
  mbar_wait_sleep(smem_addr(&g_free[t % R.stages]), ((t / R.stages) - 1) & 1u, 128);
  return;
#endif
  if (t >= 2 * R.stages) {
    const std::uint32_t need = t - 2 * R.stages + 1;
    const std::uint32_t addr = smem_addr(&g_consumed);
    while (true) {
      std::uint32_t v;
      asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
      if (__all_sync(0xffffffffu, v >= need)) break;
      poll();
      __nanosleep(128);
    }
  }
  const std::uint32_t bar = smem_addr(&g_free[t % R.stages]), par = ((t / R.stages) - 1) & 1u;
  while (!__all_sync(0xffffffffu, mbar_try(bar, par))) {
    poll();
    __nanosleep(128);
  }
}

// Output into the A ring: element g of the CTA range [e0, e1) lands in ring
// tile (g - e0) >> 14 at offset g & 16383 (the tiled layout is the swizzled
// shared-memory image).  A warp tile spans at most two ring tiles, tf and
// tf + 1; elements outside [e0, e1) belong to the neighbouring CTA.
struct RingOut {
  std::uint64_t S0;              // element of chunk 0
  std::uint64_t e0, e1;          // CTA range
  std::uint32_t c_lo, c_hi;      // chunks inside [e0, e1) (chunks never straddle e0 / e1: multiples of 16384)
  std::uint32_t c_split;         // first chunk in ring tile tf + 1
  std::uint32_t base_f, base_l;  // shared address of chunk 0 if it were in ring tile tf / tf + 1
  std::uint32_t tf;              // first ring tile of the warp tile
  std::uint32_t bf, bl;          // bytes this warp writes into ring tiles tf, tf + 1
  std::uint32_t bar_f, bar_l;    // their "full" barriers
  const Ring* R;
  int lane;

  __device__ __forceinline__ void wait() const {
    wait_stage_free(*R, tf, *R->fl);
    if (bl) wait_stage_free(*R, tf + 1, *R->fl);
  }
  __device__ __forceinline__ void chunk(std::uint32_t c, const uint4& r) const {
    if (c < c_lo || c >= c_hi) return;
    const std::uint32_t a = (c < c_split ? base_f : base_l) + 16 * c;
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w)
                 : "memory");
  }
  __device__ __forceinline__ void byte(std::uint32_t i, std::uint8_t b) const {
    const std::uint64_t g = S0 + i;
    if (g < e0 || g >= e1) return;
    const std::uint32_t a = ((i >> 4) < c_split ? base_f : base_l) + i;
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(static_cast<std::uint32_t>(b)) : "memory");
  }
  // every writer fences its generic-proxy stores for the tensor core's async
  // proxy, then lane 0 arrives with the warp's byte counts
  __device__ __forceinline__ void done() const {
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (bf) mbar_arrive(bar_f, bf);
      if (bl) mbar_arrive(bar_l, bl);
    }
  }
};

// The ring output of an ECF8 tile whose elements [tA, tE) meet the CTA range
// (A < E after clipping).
__device__ __forceinline__ RingOut ring_out(std::uint64_t tA, std::uint64_t A, std::uint64_t E, const Ring& R, int lane) {
  RingOut out;
  out.S0 = tA & ~std::uint64_t{15};
  out.e0 = R.e0;
  out.e1 = R.e1;
  out.tf = static_cast<std::uint32_t>((A - R.e0) >> 14);
  const std::uint32_t tl = static_cast<std::uint32_t>((E - 1 - R.e0) >> 14);
  const std::uint64_t bnd = R.e0 + (static_cast<std::uint64_t>(out.tf + 1) << 14);
  out.bf = static_cast<std::uint32_t>((E < bnd ? E : bnd) - A);
  out.bl = tl != out.tf ? static_cast<std::uint32_t>(E - bnd) : 0u;
  // chunk c holds elements S0 + 16c ..; CTA-relative element g - e0 of ring
  // tile t lives at a_base + (t % stages) * 16384 + (g - e0 - 16384 t)
  const std::int64_t s_rel = static_cast<std::int64_t>(out.S0) - static_cast<std::int64_t>(R.e0);
  out.c_lo = s_rel >= 0 ? 0u : static_cast<std::uint32_t>((-s_rel) >> 4);
  out.c_hi = static_cast<std::uint32_t>((static_cast<std::int64_t>(R.e1) - static_cast<std::int64_t>(out.S0)) >> 4);
  out.c_split = static_cast<std::uint32_t>((static_cast<std::int64_t>(bnd) - static_cast<std::int64_t>(out.S0)) >> 4);
  const std::int32_t s_rel32 = static_cast<std::int32_t>(s_rel);  // a CTA run is < 2^31 elements
  out.base_f = static_cast<std::uint32_t>(static_cast<std::int32_t>(R.a_base + (out.tf % R.stages) * kTileElems) -
                                          static_cast<std::int32_t>(out.tf << 14) + s_rel32);
  out.base_l = static_cast<std::uint32_t>(static_cast<std::int32_t>(R.a_base + ((out.tf + 1) % R.stages) * kTileElems) -
                                          static_cast<std::int32_t>((out.tf + 1) << 14) + s_rel32);
  out.bar_f = smem_addr(&g_full[out.tf % R.stages]);
  out.bar_l = smem_addr(&g_full[(out.tf + 1) % R.stages]);
  out.R = &R;
  out.lane = lane;
  return out;
}

template <int LW, class WSm>
__device__ __forceinline__ void ring_tile(const TensorDesc& d, const WarpInT<LW>& in, std::uint32_t log2T,
                                          std::uint32_t len_off, WSm& ws, const Ring& R, int lane) {
  const LaneRun run = warp_decode_scan<LW, 128>(in, log2T, len_off, SmemTables{g_tbf}, smem_addr(ws.slot + lane), lane,
                                                tile_verified(d, in, log2T));
  // this ECF8 tile's part of the CTA range, in ring tiles tf (and tf + 1)
  const std::uint64_t A = in.A > R.e0 ? in.A : R.e0;
  const std::uint64_t E = in.E < R.e1 ? in.E : R.e1;
  if (A >= E) {
    __syncwarp();
    return;
  }
  RingOut out = ring_out(in.A, A, E, R, lane);
  compact_write<2>(d, in.A, in.E, run, ws, lane, out);
}

// Byte-step variant: every lane's output offset is known (lane_start), the
// lanes decode straight into the warp's staging tile (direct_tile) and the
// merged FP8 bytes go to the A ring.
template <int LW, class WSm>
__device__ __forceinline__ void ring_tile_fsm(const TensorDesc& d, const WarpInT<LW>& in, std::uint32_t log2T, WSm& ws,
                                              const Ring& R, int lane, const FsmAt& ft) {
  const std::uint64_t A = in.A > R.e0 ? in.A : R.e0;
  const std::uint64_t E = in.E < R.e1 ? in.E : R.e1;
  if (A >= E) return;
  direct_tile<2, LW, ECF8_FUSED_GPK != 0>(
      d, in, ws, lane, [&] { return ring_out(in.A, A, E, R, lane); }, tile_verified(d, in, log2T), ft);
}

// Per decode warp: slots of SLOT_ROWS words per lane (a lane's run of LW
// windows), the staging tile (32 LW windows x <= 32 or 64 symbols).
template <int LW, int SLOT_ROWS>
using FusedWarpSmem = WarpPipeSmem<SLOT_ROWS, 32 * LW * (SLOT_ROWS > 17 && LW == 4 ? 64 : 32) / 8 + 8>;
// Byte-step variant: the staging tile only (the packed bytes are read from
// L2 at write-back): SLOT_ROWS = 1.
template <int LW, int SLOT_ROWS, bool FSM>
using FusedWarpSmemF =
    std::conditional_t<FSM && ECF8_FUSED_GPK, WarpPipeSmem<1, 32 * LW * 32 / 8 + 8>, FusedWarpSmem<LW, SLOT_ROWS>>;

// Warps after the decode warps: the MMA (control) warp.
template <bool FSM>
constexpr int extra_warps() { return 1; }

template <int LW, int SLOT_ROWS, bool WIDE, bool FSM = false>
__global__ void __launch_bounds__((decode_warps<LW, SLOT_ROWS, WIDE, FSM>() + extra_warps<FSM>()) * 32, 1)
    fused_gemm_kernel(const __grid_constant__ FusedArgs args) {
  using WSm = FusedWarpSmemF<LW, SLOT_ROWS, FSM>;
  constexpr int kDecodeWarps = decode_warps<LW, SLOT_ROWS, WIDE, FSM>();
  constexpr int kThreadsF = (kDecodeWarps + extra_warps<FSM>()) * 32;
  constexpr int kCtrlWarp = kDecodeWarps;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#if ECF8_FUSED_CHAIN
  asm volatile("griddepcontrol.launch_dependents;");  // the next call's x_tiles_kernel may queue now
#endif
  const FusedCta cta = args.plan[blockIdx.x];
  const std::uint32_t n_kt = cta.tile1 - cta.tile0;
  const std::uint32_t KT = args.k / 128;
  const std::uint32_t nt0 = cta.tile0 / KT;  // first n-tile (segment 0)

  // dynamic smem: [pad to 1024][A ring][B ring x2][decode slots]
  const std::uint32_t raw = smem_addr(smem_raw);
  const std::uint32_t a_base = (raw + 1023u) & ~1023u;
  const std::uint32_t b_base = a_base + args.stages_a * kTileElems;
  const std::uint32_t b_bytes = args.m_pad * 128u;
  WSm* const wsm = reinterpret_cast<WSm*>(smem_raw + (b_base + args.stages_b * b_bytes - raw));

  if (threadIdx.x == 0) {
    g_wdesc = args.w;
    g_wdesc.blk_begin = cta.blk_begin;
    g_wdesc.blk_end = cta.blk_end;
    g_wdesc.tile_begin = 0;
  }
  __syncthreads();
  const TensorDesc& d = g_wdesc;
  const std::uint32_t log2T = 31 - __clz(d.T);
  const std::uint32_t m_blk = (32u * LW) >> log2T;
  const std::uint64_t n_tiles = (cta.blk_end - cta.blk_begin + m_blk - 1) / m_blk;

  if (warp == kCtrlWarp) {
    // TMEM accumulator: 128 lanes x m_pad fp32 columns (power of two >= 32)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&g_tmem)),
                 "r"(args.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    if (lane == 0) {
      for (std::uint32_t s = 0; s < args.stages_a; ++s) {
        mbar_init(smem_addr(&g_full[s]), kTileElems);
        mbar_init(smem_addr(&g_empty[s]), 1);
        mbar_init(smem_addr(&g_free[s]), 1);
      }
      mbar_init(smem_addr(&g_bfull[0]), 1);
      mbar_init(smem_addr(&g_bfull[1]), 1);
      for (std::uint32_t b = 0; b < args.acc_bufs; ++b) {
        mbar_init(smem_addr(&g_segdone[b]), 1);
        mbar_init(smem_addr(&g_accfree[b]), 4);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      g_qnext = kDecodeWarps;
      g_consumed = 0;
      for (int w = 0; w < 4; ++w) g_nflush[w] = 0;
    }
  }
  if constexpr (FSM) {
    const uint4* f4 = reinterpret_cast<const uint4*>(d.fsm);
    const uint4* c4 = reinterpret_cast<const uint4*>(d.fsm_cm);
    for (int i = threadIdx.x; i < 256 * kFsmStates / 4; i += kThreadsF) reinterpret_cast<uint4*>(g_fsmf)[i] = __ldg(f4 + i);
    for (int i = threadIdx.x; i < 256 * kFsmStates / 16; i += kThreadsF) reinterpret_cast<uint4*>(g_cmf)[i] = __ldg(c4 + i);
  } else {
    stage_tables(d, g_tbf, threadIdx.x, kThreadsF);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem_d = g_tmem;

  const std::uint32_t nseg = n_kt ? (cta.tile1 - 1) / KT - nt0 + 1 : 0;
  const Flush fl{&args, tmem_d, nt0, nseg};

  if (warp < kDecodeWarps) {
    // ---- decode warps: dynamic queue over the CTA's ECF8 tiles, in order
    const Ring R{a_base, args.stages_a, cta.e0, cta.e1, &fl};
    const std::uint32_t len_off = (d.n_luts - 1) << 8;
    WSm& ws = wsm[warp];
    WarpInT<LW> nxt;
    std::uint64_t tile = warp;
    if (tile < n_tiles) load_warp_tile<LW, FSM, LW == 4, false>(d, tile, log2T, lane, nxt);
    while (tile < n_tiles) {
      const WarpInT<LW> cur = nxt;
      unsigned claim = 0;
      if (lane == 0) {
        claim = atomicAdd(&g_qnext, 1u);
        // sign/mantissa bytes of this tile -> L2 while it decodes
        const std::uint64_t p0 = (cur.A >> 1) & ~std::uint64_t{15};
        const std::uint32_t bytes = static_cast<std::uint32_t>((((cur.E + 1) >> 1) - p0 + 15) & ~std::uint64_t{15});
        if (bytes)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(d.packed + p0), "r"(bytes) : "memory");
      }
      const std::uint64_t next = __shfl_sync(0xffffffffu, claim, 0);
      if (next < n_tiles) load_warp_tile<LW, FSM, LW == 4, false>(d, next, log2T, lane, nxt);
      if constexpr (FSM) ring_tile_fsm(d, cur, log2T, ws, R, lane, FsmAt{smem_addr(g_fsmf), smem_addr(g_cmf)});
      else ring_tile(d, cur, log2T, len_off, ws, R, lane);
#if ECF8_FUSED_MIDFLUSH
      fl.run(false);  // warps 0-3: flush the segments the MMAs have finished
#endif
      tile = next;
    }
    fl.run(true);  // warps 0-3: the remaining segments
  } else {
    // ---- control warp: X tiles -> B ring, one lane issues the MMAs
    const std::uint32_t idesc = (1u << 4)                       // D = f32
                                | (args.w_fmt << 7)             // A = W (E4M3 0 / E5M2 1)
                                | (0u << 10)                    // B = X E4M3
                                | ((args.m_pad >> 3) << 17)     // N
                                | ((128u >> 4) << 24);          // M
    // X K-tiles arrive by bulk async copy (TMA engine) from the pre-swizzled
    // xt (x_tiles_kernel): one contiguous m_pad x 128-byte image per K tile
    auto issue_x = [&](std::uint32_t t) {
      const std::uint32_t bsl = t % args.stages_b;
      const std::uint32_t kt = (cta.tile0 + t) % KT;
      const std::uint32_t bar = smem_addr(&g_bfull[bsl]);
#if ECF8_FUSED_XPROBE  // timing experiment: X tiles not loaded (wrong results)
      (void)kt;
      mbar_arrive(bar, 1);
#else
      asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(bar),
                   "r"(b_bytes)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       b_base + bsl * b_bytes),
                   "l"(args.xt + static_cast<std::uint64_t>(kt) * b_bytes), "r"(b_bytes), "r"(bar)
                   : "memory");
#endif
    };
    asm volatile("griddepcontrol.wait;" ::: "memory");  // x_tiles_kernel: X tiles written, y zeroed
    if (lane == 0 && n_kt) issue_x(0);
    for (std::uint32_t t = 0; t < n_kt; ++t) {
      const std::uint32_t bs = t % args.stages_b;
      const std::uint32_t bdst = b_base + bs * b_bytes;
      const std::uint32_t g = cta.tile0 + t;
      const std::uint32_t seg = g / KT - nt0;
      const std::uint32_t buf = seg % args.acc_bufs;
      const bool first_of_seg = t == 0 || g % KT == 0;
      const bool last_of_seg = t + 1 == n_kt || (g + 1) % KT == 0;
      // two B stages: next K tile's X into the other stage now (its previous
      // reader, the MMAs of tile t-1, completed: waited on at the end of
      // iteration t-1); one stage (m_pad > 128): after this tile's MMAs
      if (lane == 0 && args.stages_b == 2 && t + 1 < n_kt) issue_x(t + 1);
      // segment seg reuses the accumulator of segment seg - acc_bufs: wait
      // until warps 0-3 have read it out
      if (first_of_seg && seg >= args.acc_bufs)
        mbar_wait_sleep(smem_addr(&g_accfree[buf]), ((seg / args.acc_bufs) - 1) & 1u, 32);
      mbar_wait_sleep(smem_addr(&g_bfull[bs]), (t / args.stages_b) & 1u, 32);
      const std::uint32_t s = t % args.stages_a;
      mbar_wait_sleep(smem_addr(&g_full[s]), (t / args.stages_a) & 1u, 32);
      tc_fence_after();
      if (lane == 0) {
        const std::uint32_t a_st = a_base + s * kTileElems;
#pragma unroll
        for (std::uint32_t k = 0; k < 4; ++k)
#if ECF8_FUSED_MMAPROBE  // timing experiment: one K = 32 MMA per tile (wrong results)
          if (k == 0)
#endif
          mma_f8(tmem_d + buf * args.acc_cols, smem_desc(a_st + 32 * k), smem_desc(bdst + 32 * k), idesc,
                 !(first_of_seg && k == 0));
        tc_commit(smem_addr(&g_empty[s]));
        if (last_of_seg) tc_commit(smem_addr(&g_segdone[buf]));
        // the MMAs of tile t have read stage s: publish it to the decode warps
        mbar_wait(smem_addr(&g_empty[s]), (t / args.stages_a) & 1u);
        mbar_arrive(smem_addr(&g_free[s]), 1);
        asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(&g_consumed)), "r"(t + 1)
                     : "memory");
        if (args.stages_b == 1 && t + 1 < n_kt) issue_x(t + 1);
      }
      __syncwarp();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kCtrlWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(args.tmem_cols)
                 : "memory");
  }
}

// ---- L2-ring variant (byte-step weights) ---------------------------------
//
// The shared-memory A ring caps the decode warps in flight (a warp tile is
// ~0.4 K tiles of ring; 12 warps fill a 5-stage ring).  Here the decode warps
// run exactly as the standalone decoder (23 warps, direct tiles, packed bytes
// from L2) and store merged FP8 bytes to a per-CTA ring of kRingSlots K tiles
// in global memory, small enough to stay in L2; a loader warp moves each
// completed K tile (and its X tile) into a shared-memory stage by bulk async
// copy, an MMA warp multiplies.  Per K tile t, slot t % R:
//   decode warps  wait until the loader copied slot t - R (g2_loaded), store,
//                 fence.proxy.async.global, arrive on g2_full[slot] with their bytes
//   loader        wait g2_full (16384 bytes), wait the stage's MMAs (g2_empty),
//                 bulk-copy A (16 KB) + X into stage t % S (g2_sfull)
//   MMA warp      wait g2_sfull, publish g2_loaded = t + 1, tcgen05.mma, commit g2_empty

#ifndef ECF8_FUSED_L2_WARPS
#define ECF8_FUSED_L2_WARPS 23
#endif
constexpr int kL2DecodeWarps = ECF8_FUSED_L2_WARPS;
constexpr int kL2MaxStages = 6;
__shared__ alignas(8) unsigned long long g2_full[kRingSlots];
__shared__ alignas(8) unsigned long long g2_sfull[kL2MaxStages];
__shared__ alignas(8) unsigned long long g2_empty[kL2MaxStages];
__shared__ std::uint32_t g2_loaded;
__shared__ unsigned g2_qnext;

#ifndef ECF8_L2_PROBE
#define ECF8_L2_PROBE 0  // timing experiments only (wrong results): 1 no MMAs, 2 no ring stores
#endif

// L2-ring kernel: decode warps that flush finished segments mid-run (4, 8,
// 12 or 16).  A/B (one Llama-3-70B layer): 4 -> 8 takes M = 256 from 0.631 to
// 0.595-0.600 ms (the flushes no longer hold back the four warps whose K tiles
// the ring waits for), M <= 64 the same; 12 / 16 the same as 8; choosing 4 at
// M <= 64 at run time measured slower than the constant.
#ifndef ECF8_FLUSH_WARPS
#define ECF8_FLUSH_WARPS 8
#endif

#ifndef ECF8_FUSED_FINAL_ALL
#define ECF8_FUSED_FINAL_ALL 1  // the segments left after the decode: flushed by all decode warps (0: warps 0-3)
#endif

#ifndef ECF8_FUSED_WB_UNROLL
#define ECF8_FUSED_WB_UNROLL 4  // write-back chunks per lane in flight (the ring sink)
#endif

#ifndef ECF8_SLOT_SLEEP
#define ECF8_SLOT_SLEEP 64  // ns between a waiting ring writer's polls
#endif

struct GRingOut {
  // element g of the CTA's K tile t sits in ring slot t % R at g - e0 - 16384 t,
  // i.e. at ring + ((g - e0) mod 16384 R): R is a power of two and e0 a
  // multiple of 16384
  std::uint8_t* ring;
  std::uint32_t s0r;             // (S0 - e0) mod 2^32, S0 = element of chunk 0
  std::uint32_t c_lo, c_n;       // chunks [c_lo, c_lo + c_n) are inside the CTA range
  std::uint32_t tf, bf, bl, bar_f, bar_l;  // first K tile of the write-back, bytes in tf / tf + 1, their full barriers
  const Flush* fl;
  int lane;
  static constexpr std::uint32_t kMask = kRingSlots * kTileElems - 1;
  static_assert((kRingSlots & (kRingSlots - 1)) == 0, "ring slots: a power of two");
  __device__ __forceinline__ void wait_slot(std::uint32_t t) const {
    if (t < kRingSlots) return;
    const std::uint32_t need = t - kRingSlots + 1, addr = smem_addr(&g2_loaded);
    for (;;) {
      std::uint32_t v;
      asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
      if (__all_sync(0xffffffffu, v >= need)) return;
      (*fl)();
      __nanosleep(ECF8_SLOT_SLEEP);
    }
  }
  __device__ __forceinline__ void wait() const {
    // the rings are shared by the calls on a stream: write only once the
    // previous call's grid is complete (x_tiles_kernel waited for it)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    wait_slot(tf);
    if (bl) wait_slot(tf + 1);
  }
  __device__ __forceinline__ void chunk(std::uint32_t c, const uint4& r) const {
    if (c - c_lo >= c_n || ECF8_L2_PROBE == 2) return;  // probe 2: no ring stores (timing only)
    std::uint8_t* p = ring + ((s0r + 16 * c) & kMask);
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w) : "memory");
  }
  __device__ __forceinline__ void byte(std::uint32_t i, std::uint8_t b) const {
    if ((i >> 4) - c_lo >= c_n) return;
    ring[(s0r + i) & kMask] = b;
  }
  // (A/B: deferring the fence and arrivals to after the warp's next decode
  // phase made a 70B layer 4 % slower)
  __device__ __forceinline__ void done() const {
    // the generic-proxy stores must be visible to the loader's bulk copies
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      if (bf) mbar_arrive(bar_f, bf);
      if (bl) mbar_arrive(bar_l, bl);
    }
  }
};

// The decode warps' L2 prefetches of their next tile: addresses from the
// section table (decode_warp.cuh: prefetch_tile_l2_tab) or computed per tile.
#ifndef ECF8_FUSED_PF_TAB
#define ECF8_FUSED_PF_TAB 1  // A/B r3p: -1.5 % per layer at every M (M = 1: 0.455 -> 0.448 ms)
#endif
#if ECF8_FUSED_PF_TAB
__shared__ PfSec g_wpf[5];
#define PF_TILE(d, t, l2t, ln) prefetch_tile_l2_tab(d, g_wpf, t, l2t, ln)
#else
#define PF_TILE(d, t, l2t, ln) prefetch_tile_l2(d, t, l2t, ln)
#endif

__global__ void __launch_bounds__((kL2DecodeWarps + 2) * 32, 1) fused_l2_kernel(const __grid_constant__ FusedArgs args) {
  constexpr int kWarps = kL2DecodeWarps + 2, kLoader = kL2DecodeWarps, kMma = kL2DecodeWarps + 1;
  using WSm = WarpPipeSmem<1, 32 * 8 * 32 / 8 + 8>;  // the staging tile (packed bytes come from L2)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  asm volatile("griddepcontrol.launch_dependents;");
  const FusedCta cta = args.plan[blockIdx.x];
  const std::uint32_t n_kt = cta.tile1 - cta.tile0, KT = args.k / 128, nt0 = cta.tile0 / KT;
  const std::uint32_t S = args.stages_a;
  const std::uint32_t raw = smem_addr(smem_raw);
  const std::uint32_t a_base = (raw + 1023u) & ~1023u;
  const std::uint32_t b_base = a_base + S * kTileElems, b_bytes = args.m_pad * 128u;
  WSm* const wsm = reinterpret_cast<WSm*>(smem_raw + (b_base + S * b_bytes - raw));
  std::uint8_t* const ring = args.scratch + static_cast<std::uint64_t>(blockIdx.x) * kRingSlots * kTileElems;

#if ECF8_FUSED_PF_TAB
  if (threadIdx.x < 5) g_wpf[threadIdx.x] = pf_section(args.w, threadIdx.x, 31 - __clz(args.w.T));
#endif
  if (threadIdx.x == 0) {
    g_wdesc = args.w;
    g_wdesc.blk_begin = cta.blk_begin;
    g_wdesc.blk_end = cta.blk_end;
    g_wdesc.tile_begin = 0;
  }
  if (warp == kMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&g_tmem)),
                 "r"(args.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == kLoader && lane == 0) {
    for (std::uint32_t r = 0; r < kRingSlots; ++r) mbar_init(smem_addr(&g2_full[r]), kTileElems);
    for (std::uint32_t s = 0; s < S; ++s) {
      mbar_init(smem_addr(&g2_sfull[s]), 1);
      mbar_init(smem_addr(&g2_empty[s]), 1);
    }
    for (std::uint32_t b = 0; b < args.acc_bufs; ++b) {
      mbar_init(smem_addr(&g_segdone[b]), 1);
      mbar_init(smem_addr(&g_accfree[b]), ECF8_FLUSH_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    g2_loaded = 0;
    g2_qnext = kL2DecodeWarps;
    for (int w = 0; w < 16; ++w) g_nflush[w] = 0;
  }
  {
    const uint4* f4 = reinterpret_cast<const uint4*>(args.w.fsm);
    const uint4* c4 = reinterpret_cast<const uint4*>(args.w.fsm_cm);
    for (int i = threadIdx.x; i < 256 * kFsmStates / 4; i += kWarps * 32) reinterpret_cast<uint4*>(g_fsmf)[i] = __ldg(f4 + i);
    for (int i = threadIdx.x; i < 256 * kFsmStates / 16; i += kWarps * 32) reinterpret_cast<uint4*>(g_cmf)[i] = __ldg(c4 + i);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const TensorDesc& d = g_wdesc;
  const std::uint32_t tmem_d = g_tmem;
  const std::uint32_t nseg = n_kt ? (cta.tile1 - 1) / KT - nt0 + 1 : 0;
  const Flush fl{&args, tmem_d, nt0, nseg, ECF8_FLUSH_WARPS};
  const std::uint32_t log2T = 31 - __clz(d.T);

  if (warp < kL2DecodeWarps) {
    // ---- decode warps: the standalone kernel's loop over the CTA's ECF8 tiles
    const std::uint32_t m_blk = 256u >> log2T;
    const std::uint64_t n_tiles = (cta.blk_end - cta.blk_begin + m_blk - 1) / m_blk;
    WSm& ws = wsm[warp];
    const FsmAt ft{smem_addr(g_fsmf), smem_addr(g_cmf)};
    std::uint64_t tile = warp;
    if (tile < n_tiles && lane < 5) PF_TILE(d, tile, log2T, lane);
    while (tile < n_tiles) {
      WarpInT<8> cur;
      load_warp_tile<8, true, false, false>(d, tile, log2T, lane, cur);
      unsigned claim = 0;
      if (lane == 0) claim = atomicAdd(&g2_qnext, 1u);
      const std::uint64_t next = __shfl_sync(0xffffffffu, claim, 0);
      if (next < n_tiles && lane < 5) PF_TILE(d, next, log2T, lane);
      if (lane == 0) {  // this tile's sign/mantissa bytes -> L2 (read at write-back)
        const std::uint64_t p0 = (cur.A >> 1) & ~std::uint64_t{15};
        const std::uint32_t bytes = static_cast<std::uint32_t>((((cur.E + 1) >> 1) - p0 + 15) & ~std::uint64_t{15});
        if (bytes) prefetch_l2(d.packed + p0, bytes);
      }
      const std::uint64_t A = cur.A > cta.e0 ? cur.A : cta.e0, E = cur.E < cta.e1 ? cur.E : cta.e1;
      if (A < E) {
        const std::uint32_t tf = static_cast<std::uint32_t>((A - cta.e0) >> 14);
        const std::uint32_t tl = static_cast<std::uint32_t>((E - 1 - cta.e0) >> 14);
        const std::uint64_t bnd = cta.e0 + (static_cast<std::uint64_t>(tf + 1) << 14);
        const std::uint32_t bf = static_cast<std::uint32_t>((E < bnd ? E : bnd) - A);
        const std::uint32_t bl = tl != tf ? static_cast<std::uint32_t>(E - bnd) : 0u;
        direct_tile<ECF8_FUSED_WB_UNROLL, 8, true>(
            d, cur, ws, lane,
            [&] {
              GRingOut o;
              const std::uint64_t S0 = cur.A & ~std::uint64_t{15};
              const std::int64_t s_rel = static_cast<std::int64_t>(S0) - static_cast<std::int64_t>(cta.e0);
              o.tf = tf;
              o.bf = bf;
              o.bl = bl;
              o.bar_f = smem_addr(&g2_full[tf % kRingSlots]);
              o.bar_l = smem_addr(&g2_full[(tf + 1) % kRingSlots]);
              o.lane = lane;
              o.ring = ring;
              o.s0r = static_cast<std::uint32_t>(s_rel);
              o.c_lo = s_rel >= 0 ? 0u : static_cast<std::uint32_t>((-s_rel) >> 4);
              o.c_n = static_cast<std::uint32_t>((static_cast<std::int64_t>(cta.e1) - static_cast<std::int64_t>(S0)) >> 4) - o.c_lo;
              o.fl = &fl;
              return o;
            },
            tile_verified(d, cur, log2T), ft);
      }
      fl.run(false);  // warps 0-3: flush the segments the MMAs have finished
      tile = next;
    }
#if ECF8_FUSED_FINAL_ALL
    fl.run_final(kL2DecodeWarps);  // the last segments, by every decode warp
#else
    fl.run(true);
#endif
  } else if (warp == kLoader) {
    // ---- loader: completed K tiles of the ring + their X tiles -> shared-memory stages
    asm volatile("griddepcontrol.wait;" ::: "memory");  // x_tiles_kernel: X tiles written, y zeroed
    if (lane == 0) {
      for (std::uint32_t t = 0; t < n_kt; ++t) {
        const std::uint32_t r = t % kRingSlots, s = t % S;
        mbar_wait_sleep(smem_addr(&g2_full[r]), (t / kRingSlots) & 1u, 32);
        if (t >= S) mbar_wait_sleep(smem_addr(&g2_empty[s]), ((t / S) - 1) & 1u, 32);
        const std::uint32_t bar = smem_addr(&g2_sfull[s]);
        const std::uint32_t kt = (cta.tile0 + t) % KT;
        asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(bar),
                     "r"(kTileElems + b_bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         a_base + s * kTileElems),
                     "l"(ring + static_cast<std::uint64_t>(r) * kTileElems), "r"(kTileElems), "r"(bar)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         b_base + s * b_bytes),
                     "l"(args.xt + static_cast<std::uint64_t>(kt) * b_bytes), "r"(b_bytes), "r"(bar)
                     : "memory");
      }
    }
    __syncwarp();
  } else {
    // ---- MMA warp
    const std::uint32_t idesc = (1u << 4) | (args.w_fmt << 7) | (0u << 10) | ((args.m_pad >> 3) << 17) | ((128u >> 4) << 24);
    for (std::uint32_t t = 0; t < n_kt; ++t) {
      const std::uint32_t s = t % S;
      const std::uint32_t g = cta.tile0 + t;
      const std::uint32_t seg = g / KT - nt0, buf = seg % args.acc_bufs;
      const bool first_of_seg = t == 0 || g % KT == 0, last_of_seg = t + 1 == n_kt || (g + 1) % KT == 0;
      if (first_of_seg && seg >= args.acc_bufs)
        mbar_wait_sleep(smem_addr(&g_accfree[buf]), ((seg / args.acc_bufs) - 1) & 1u, 32);
      mbar_wait_sleep(smem_addr(&g2_sfull[s]), (t / S) & 1u, 32);
      tc_fence_after();
      if (lane == 0) {
        // the ring slot's bytes are in shared memory: writers may reuse it
        asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(&g2_loaded)), "r"(t + 1) : "memory");
        const std::uint32_t a_st = a_base + s * kTileElems, bdst = b_base + s * b_bytes;
#pragma unroll
        for (std::uint32_t k = 0; k < (ECF8_L2_PROBE == 1 ? 0u : 4u); ++k)
          mma_f8(tmem_d + buf * args.acc_cols, smem_desc(a_st + 32 * k), smem_desc(bdst + 32 * k), idesc,
                 !(first_of_seg && k == 0));
        tc_commit(smem_addr(&g2_empty[s]));
        if (last_of_seg) tc_commit(smem_addr(&g_segdone[buf]));
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(args.tmem_cols)
                 : "memory");
  }
}

// x [m, k] row-major -> xt [k/128][m_pad][128 B] in the 128B-swizzled
// K-major image (rows >= m zero), so every B tile is one contiguous copy.
// Also zeroes y (the split-K partial sums are added into it).  The fused
// kernel is launched as its programmatic dependent: its decode warps start
// while this runs; its X loads and y updates wait for it (griddepcontrol).
__global__ void x_tiles_kernel(const std::uint8_t* __restrict__ x, std::uint8_t* __restrict__ xt, std::uint32_t m,
                               std::uint32_t m_pad, std::uint32_t k, float* __restrict__ y, std::uint64_t y_elems) {
  asm volatile("griddepcontrol.launch_dependents;");
  // Launched as a programmatic dependent of whatever precedes it (typically
  // the previous fused GEMM, whose tail -- last flushes, pipeline drain --
  // then overlaps this call's start and the next GEMM's decode warps): x and
  // y may be the previous kernel's output / input, so wait for it first.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  const std::uint64_t tid = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if ((reinterpret_cast<std::uintptr_t>(y) & 15) == 0) {
    for (std::uint64_t i = tid; i < y_elems / 4; i += stride)
      reinterpret_cast<float4*>(y)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid < (y_elems & 3)) y[(y_elems & ~std::uint64_t{3}) + tid] = 0.f;
  } else {
    for (std::uint64_t i = tid; i < y_elems; i += stride) y[i] = 0.f;
  }
  const std::uint64_t chunks = static_cast<std::uint64_t>(k / 128) * m_pad * 8;
  for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < chunks;
       i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
    const std::uint32_t ch = static_cast<std::uint32_t>(i & 7);
    const std::uint64_t rr = i >> 3;
    const std::uint32_t r = static_cast<std::uint32_t>(rr % m_pad);
    const std::uint32_t kt = static_cast<std::uint32_t>(rr / m_pad);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < m) v = __ldg(reinterpret_cast<const uint4*>(x + static_cast<std::uint64_t>(r) * k + kt * 128u) + ch);
    const std::uint64_t dst = (static_cast<std::uint64_t>(kt) * m_pad + r) * 128 + ((ch ^ (r & 7u)) << 4);
    *reinterpret_cast<uint4*>(xt + dst) = v;
  }
}

}  // namespace

// X ring stages: two, except m > 128 with the round-1 decode warps (their
// shared memory leaves room for one 32 KB X stage beside 3+ A stages)
std::uint32_t fused_stages_b(std::uint32_t m_pad, bool fsm) {
  if (m_pad <= 128) return 2u;
  return fsm ? ECF8_FUSED_FSM_WIDE_XSTAGES : ECF8_FUSED_WIDE_XSTAGES;
}

// Decode-warp geometry for a tiled weight:
//   Lmin >= 2, T <= 128: 4 windows per lane, 17 slot rows -- half-size warp
//       tiles keep the decode warps within ~4 K tiles of the MMA;
//   Lmin >= 2, T == 256: 8 windows per lane, 33 slot rows;
//   Lmin == 1, T <= 128: 4 windows of up to 64 symbols, 33 slot rows.
int fused_lane_windows(std::uint32_t T, std::uint32_t lmin) {
  if (lmin >= 2 && T >= 4 && T <= 128) return 4;
  if (lmin >= 2 && T == 256) return 8;
  if (lmin >= 1 && T >= 4 && T <= 128) return 4;
  return 0;
}

template <int LW, int ROWS, bool WIDE, bool FSM = false>
constexpr std::uint32_t warps_smem() {
  return static_cast<std::uint32_t>(decode_warps<LW, ROWS, WIDE, FSM>() * sizeof(FusedWarpSmemF<LW, ROWS, FSM>));
}

// All decode warps' pipeline state.
std::uint32_t fused_warp_smem(std::uint32_t T, std::uint32_t lmin, std::uint32_t m_pad, bool fsm) {
  const bool wide = m_pad > 128;
  if (fsm) return wide ? warps_smem<8, 33, true, true>() : warps_smem<8, 33, false, true>();
  if (fused_lane_windows(T, lmin) == 8) return wide ? warps_smem<8, 33, true>() : warps_smem<8, 33, false>();
  if (lmin >= 2) return wide ? warps_smem<4, 17, true>() : warps_smem<4, 17, false>();
  return wide ? warps_smem<4, 33, true>() : warps_smem<4, 33, false>();
}

std::uint32_t fused_stages_a(std::uint32_t m_pad, std::uint32_t warp_smem, bool fsm) {
  // 227 KB per CTA: tables 29 KB static (byte-step tables: 20 KB), the
  // decode warps' pipeline state, B ring 2 x m_pad x 128 B, A ring stages x
  // 16 KB, 1 KB alignment slack
  const std::uint32_t budget = 232448 - (fsm ? 21 : 30) * 1024;
  const std::uint32_t fixed = warp_smem + fused_stages_b(m_pad, fsm) * m_pad * 128 + 1024;
  const std::uint32_t s = fixed < budget ? (budget - fixed) / kTileElems : 0;
  return s > kMaxStagesA ? kMaxStagesA : s;
}

std::uint32_t fused_smem_bytes(std::uint32_t m_pad, std::uint32_t stages_a, std::uint32_t warp_smem, bool fsm) {
  return 1024 + stages_a * kTileElems + fused_stages_b(m_pad, fsm) * m_pad * 128 + warp_smem;
}

template <int LW, int ROWS, bool WIDE, bool FSM = false>
cudaError_t launch_lw(const FusedArgs& args, std::uint32_t n_cta, cudaStream_t s) {
  const std::uint32_t smem = fused_smem_bytes(args.m_pad, args.stages_a, warps_smem<LW, ROWS, WIDE, FSM>(), FSM);
  cudaError_t e = cudaFuncSetAttribute(fused_gemm_kernel<LW, ROWS, WIDE, FSM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  static const bool pdl = std::getenv("ECF8_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_cta);
  cfg.blockDim = dim3((decode_warps<LW, ROWS, WIDE, FSM>() + extra_warps<FSM>()) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fused_gemm_kernel<LW, ROWS, WIDE, FSM>, args);
}

template <bool WIDE>
cudaError_t launch_geometry(const FusedArgs& args, std::uint32_t n_cta, cudaStream_t s) {
  if (args.fsm) return launch_lw<8, 33, WIDE, true>(args, n_cta, s);
  if (fused_lane_windows(args.w.T, args.w.lmin) == 8) return launch_lw<8, 33, WIDE>(args, n_cta, s);
  return args.w.lmin >= 2 ? launch_lw<4, 17, WIDE>(args, n_cta, s) : launch_lw<4, 33, WIDE>(args, n_cta, s);
}

std::uint32_t fused_l2_stages(std::uint32_t m_pad) {
  // 227 KB: static ~21 KB, the decode warps' staging tiles, S x (A 16 KB + X m_pad x 128 B), 1 KB alignment
  const std::uint32_t warps = kL2DecodeWarps * static_cast<std::uint32_t>(sizeof(WarpPipeSmem<1, 32 * 8 * 32 / 8 + 8>));
  const std::uint32_t budget = 232448 - 22 * 1024 - warps - 1024;
  const std::uint32_t s = budget / (kTileElems + m_pad * 128);
  return s < 2 ? 0u : (s > static_cast<std::uint32_t>(kL2MaxStages) ? kL2MaxStages : s);
}

cudaError_t launch_fused_gemm(const FusedArgs& args, std::uint32_t n_cta, cudaStream_t s) {
  const std::uint64_t chunks = static_cast<std::uint64_t>(args.k / 128) * args.m_pad * 8;
  const unsigned blocks = static_cast<unsigned>(std::min<std::uint64_t>((chunks + 255) / 256, 4 * 148));
  {
    static const bool pdl = std::getenv("ECF8_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl && ECF8_FUSED_CHAIN ? 1 : 0;
    if (cudaError_t e = cudaLaunchKernelEx(&cfg, x_tiles_kernel, args.x, const_cast<std::uint8_t*>(args.xt), args.m,
                                           args.m_pad, args.k, args.y, static_cast<std::uint64_t>(args.m) * args.n);
        e != cudaSuccess)
      return e;
  }
  if (args.scratch) {
    const std::uint32_t smem = 1024 + args.stages_a * (kTileElems + args.m_pad * 128) +
                               kL2DecodeWarps * static_cast<std::uint32_t>(sizeof(WarpPipeSmem<1, 32 * 8 * 32 / 8 + 8>));
    cudaError_t e = cudaFuncSetAttribute(fused_l2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    static const bool pdl = std::getenv("ECF8_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_cta);
    cfg.blockDim = dim3((kL2DecodeWarps + 2) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fused_l2_kernel, args);
  }
  return args.m_pad > 128 ? launch_geometry<true>(args, n_cta, s) : launch_geometry<false>(args, n_cta, s);
}

}  // namespace ecf8::dev
