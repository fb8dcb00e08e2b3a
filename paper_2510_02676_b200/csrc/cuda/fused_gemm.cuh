// fused_gemm.cuh -- descriptors for the decode-fused tcgen05 FP8 GEMM.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "decode.cuh"

namespace ecf8::dev {

constexpr std::uint32_t kMaxStagesA = 8;
constexpr std::uint32_t kMaxAccBufs = 16;  // TMEM accumulator buffers (512 columns / 32)

// One CTA's work: the contiguous run of 128x128 weight tiles [tile0, tile1)
// in tile-major (nt, kt) order; each n-tile of it (a "segment") is
// accumulated in TMEM buffer (segment % acc_bufs).  Its elements [e0, e1) of the
// tiled tensor live in ECF8 blocks [blk_begin, blk_end).
struct FusedCta {
  std::uint64_t blk_begin, blk_end;
  std::uint64_t e0, e1;
  std::uint32_t tile0, tile1;
};

struct FusedArgs {
  TensorDesc w;              // the tiled ECF8 weight tensor (blk range set per CTA)
  const FusedCta* plan;      // one entry per CTA
  const std::uint8_t* x;     // [m, k] E4M3, row-major
  const std::uint8_t* xt;    // workspace: k * m_pad bytes (swizzled X tiles)
  float* y;                  // [m, n] fp32, row-major, zeroed before the launch
  std::uint32_t m, m_pad;    // tokens; padded to a multiple of 16 (MMA N)
  std::uint32_t n, k;
  std::uint32_t split_k;
  std::uint32_t stages_a;
  std::uint32_t stages_b;   // X ring stages (2)
  std::uint32_t tmem_cols;  // allocation: acc_bufs x acc_cols (power of two <= 512)
  std::uint32_t acc_cols;   // power of two >= max(32, m_pad)
  std::uint32_t acc_bufs;   // accumulator buffers, reused round-robin by the CTA's segments
  std::uint32_t w_fmt;       // 0 E4M3, 1 E5M2
  std::uint32_t fsm;         // 1: byte-step direct decode (lane offsets known for every tile; 8-window lanes)
  float scale;
  std::uint8_t* scratch;     // L2-ring variant: kRingSlots x 16 KB per CTA (nullptr: the shared-memory ring kernel)
};

#ifndef ECF8_FUSED_RING
#define ECF8_FUSED_RING 16
#endif
constexpr std::uint32_t kRingSlots = ECF8_FUSED_RING;  // decoded K tiles per CTA between the decode warps and the MMA (L2-resident)

// Windows per decode lane for a tiled weight (4 or 8; 0 = unsupported) and
// the shared memory of one decode warp's pipeline (fused_gemm.cu).
int fused_lane_windows(std::uint32_t T, std::uint32_t lmin);
std::uint32_t fused_warp_smem(std::uint32_t T, std::uint32_t lmin, std::uint32_t m_pad, bool fsm);
std::uint32_t fused_stages_b(std::uint32_t m_pad, bool fsm);
std::uint32_t fused_stages_a(std::uint32_t m_pad, std::uint32_t warp_smem, bool fsm);
std::uint32_t fused_smem_bytes(std::uint32_t m_pad, std::uint32_t stages_a, std::uint32_t warp_smem, bool fsm);
cudaError_t launch_fused_gemm(const FusedArgs& args, std::uint32_t n_cta, cudaStream_t s);
// Stages of the L2-ring variant for this m (0: it does not fit).
std::uint32_t fused_l2_stages(std::uint32_t m_pad);

}  // namespace ecf8::dev
