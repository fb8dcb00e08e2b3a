/*
 * ecf8_cuda.h -- the drop-in boundary: a C ABI over the B200 ECF8 decoder.
 *
 * Plain pointers, sizes and int status codes; no C++ or torch types.  The C++
 * API in include/ecf8/ headers (the reference's own interface) is implemented on
 * top of these calls, and Python/ctypes binds them directly
 * (paper_2510_02676_b200/_lib.py).  Each entry point names the reference
 * function it replaces (/root/reference/proj/...).
 *
 * Threading: every call is reentrant.  Device calls are stream-ordered and
 * asynchronous unless stated; host-span calls are synchronous.
 * Errors: a non-zero ecf8_status plus a thread-local message from
 * ecf8_last_error() carrying the reference's exception text.
 */
#ifndef ECF8_CUDA_H
#define ECF8_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ecf8_status {
  ECF8_OK = 0,
  ECF8_EINVAL = 1,  /* std::invalid_argument in the C++ API            */
  ECF8_EFORMAT = 2, /* ecf8::FormatError                               */
  ECF8_ECUDA = 3,   /* CUDA runtime failure or no sm_100 device        */
  ECF8_ENOMEM = 4,  /* device / pinned allocation failed               */
  ECF8_EIO = 5      /* ecf8::IoError                                   */
} ecf8_status;

/* One tensor's container sections (container.hpp:18-30 layout).  Whether
 * the pointers are host or device memory is stated per call. */
typedef struct ecf8_sections {
  uint64_t n_elem;
  uint32_t threads_per_block; /* T, power of two in [1, 1024]            */
  uint8_t lengths[16];        /* canonical code lengths, 0 = absent       */
  const uint8_t *encoded;
  uint64_t encoded_len; /* n_blocks * T * 8 + 2                          */
  const uint8_t *gaps;
  uint64_t gaps_len; /* (n_blocks * T + 1) / 2                              */
  const uint64_t *outpos;
  uint64_t n_outpos; /* n_blocks + 1                                        */
  const uint8_t *packed;
  uint64_t packed_len; /* (n_elem + 1) / 2                                  */
} ecf8_sections;

/* Device-resident tensor: sections copied to HBM (zero-padded for 16-byte
 * vector access) plus the device decode tables built from `lengths`. */
typedef struct ecf8_dev_tensor ecf8_dev_tensor;

/* A prepared multi-tensor decode (one launch for many tensors). */
typedef struct ecf8_batch ecf8_batch;

/* A weight prepared for the decode-fused FP8 GEMM. */
typedef struct ecf8_fused ecf8_fused;

const char *ecf8_last_error(void);
/* 0 when no usable device; never falls back to the CPU. */
int ecf8_device_count(void);
/* Kernel build info ("sm_100a ..."), for logs. */
const char *ecf8_build_info(void);

/* ---- host-span entry points (synchronous) ------------------------------ */

/* Replaces ecf8::decode_parallel_into (codec.cpp:256-273): validates like
 * the reference ("output size mismatch", "inconsistent block offsets"),
 * stages the sections to the device, decodes on the B200, copies `out` back. */
int ecf8_decode_host(const ecf8_sections *host, uint8_t *out, uint64_t out_len);

/* decode_parallel_into for many tensors in one call (a layer, or a whole
 * container as in decompress_streaming, container.cpp:324-352): the chunked
 * H2D / decode / D2H pipeline runs across tensor boundaries instead of
 * draining after each tensor.  Same validation and messages per tensor. */
int ecf8_decode_host_many(const ecf8_sections *const *host, uint8_t *const *outs, const uint64_t *out_lens,
                          int count);

/* decode_parallel_into for a sequence of tensors through ONE page-locked
 * buffer (buf_len >= the largest n_elem; decompress_streaming's reusable
 * buffer, container.cpp:324-352): tensor i decodes into buf[0, n_elem), and
 * fn(ctx, i, offset, n) is called -- in tensor order, offsets ascending --
 * once bytes [offset, offset + n) of tensor i are in buf; the pipeline
 * overwrites them only after fn returned.  The next tensor's sections cross
 * PCIe and decode while the current one is still being handed over.  A
 * non-zero return from fn stops the delivery (ECF8_EIO). */
typedef int (*ecf8_chunk_fn)(void *ctx, int tensor, uint64_t offset, uint64_t n);
int ecf8_decode_host_stream(const ecf8_sections *const *host, int count, uint8_t *buf, uint64_t buf_len,
                            ecf8_chunk_fn fn, void *ctx);

/* Page-lock / unlock a host buffer the host-span calls write into (the
 * ReusableBuffer of decompress_streaming): device-to-host copies into it run
 * at full PCIe rate instead of through a pageable bounce buffer.  Returns
 * ECF8_OK also when the memory was already registered. */
int ecf8_host_pin(void *p, uint64_t bytes);
int ecf8_host_unpin(void *p);
/* Page-locked host allocation (cudaMallocHost) / its release: the
 * process-lifetime buffer decompress_streaming streams through. */
int ecf8_host_alloc_pinned(uint64_t bytes, void **out);
int ecf8_host_free_pinned(void *p);

/* Replaces ecf8::decode_block (codec.cpp:201-254): decodes block `block`
 * into out[outpos[block], outpos[block+1]). out_len must be n_elem. */
int ecf8_decode_block_host(const ecf8_sections *host, uint64_t block, uint8_t *out,
                           uint64_t out_len);

/* Replaces ecf8::count_phase (codec.cpp:133-161) on one window. */
int ecf8_count_window(const uint8_t window10[10], unsigned gap, const uint8_t lengths[16],
                      uint32_t *count);

/* ---- device-resident path --------------------------------------------- */

/* Device load path (container.cpp:324-352 per-tensor setup + lut.cpp:47-97):
 * validates the sections, copies them to HBM on `stream` (cudaStream_t or
 * NULL), builds the device tables. */
int ecf8_tensor_upload(const ecf8_sections *host, void *stream, ecf8_dev_tensor **out);
void ecf8_tensor_free(ecf8_dev_tensor *t);
uint64_t ecf8_tensor_n_elem(const ecf8_dev_tensor *t);
/* Decode kernel variant the tensor launches with (decode.cuh ids: 4 = the
 * warp-tile kernel, 7 = the same for tensors whose every tile is placed
 * directly (encoder output), 5 / 6 = codes with a 1-bit word, 0-3 = T
 * outside [8, 256]; -1 for an empty tensor). */
int ecf8_tensor_kernel_variant(const ecf8_dev_tensor *t);
/* Upload-time gap check (verify_gaps_kernel): how many of the tensor's
 * 256-window tiles (*total) have every window ending where the next
 * window's gap says -- those decode by the continuous group walk, the rest
 * window by window with the reference's semantics (codec.cpp:201-253).
 * Synchronises with the device. */
uint64_t ecf8_tensor_verified_tiles(const ecf8_dev_tensor *t, uint64_t *total);
/* Container bytes the decoder reads + n_elem written (roofline numerator). */
uint64_t ecf8_tensor_algorithmic_bytes(const ecf8_dev_tensor *t);
uint64_t ecf8_tensor_device_bytes(const ecf8_dev_tensor *t);

/* ---- device encoder -------------------------------- */

/* make_stats' exponent histogram (container.cpp:386-413, ExponentHistogram::
 * of_bytes) of n FP8 bytes in device memory; counts[16] on the host.
 * Synchronises `stream`. */
int ecf8_exponent_histogram(const uint8_t *d_fp8, uint64_t n, uint64_t counts[16], void *stream);
/* encode_tensor (codec.cpp:49-98 + the nibble split, fp8.hpp:24-57) of n FP8
 * bytes in device memory with the canonical code of `lengths`, straight into
 * a device-resident tensor (same sections, byte for byte, as the host
 * encoder + ecf8_tensor_upload).  Errors as the reference: "invalid length
 * vector", "symbol absent from code table", bad T (ECF8_EINVAL).
 * Synchronises `stream` (the code-bit total sizes the arena). */
int ecf8_encode_device(const uint8_t *d_fp8, uint64_t n, uint32_t T, const uint8_t lengths[16], void *stream,
                       ecf8_dev_tensor **out);
/* One tensor's make_stats report (EntropyReport, entropy.hpp; the name is
 * the caller's). */
typedef struct ecf8_entropy_report {
  uint64_t n_elem;
  double entropy_bits, bits_per_symbol, bits_per_weight;
  double bound_lower, bound_upper; /* entropy_bounds(2.0) */
  double projected_savings, actual_savings;
} ecf8_entropy_report;
/* make_stats (container.cpp:386-413) for one tensor whose FP8 bytes are in
 * device memory: histogram and encode on the GPU, the code and the entropy
 * arithmetic on the host.  name_len and rank (>= 1) give the container
 * overhead that actual_savings counts (tensor_section_bytes).  Same numbers
 * as ecf8_host_make_stats.  Synchronises `stream`. */
int ecf8_make_stats_device(const uint8_t *d_fp8, uint64_t n, uint32_t T, uint32_t name_len, uint32_t rank,
                           void *stream, ecf8_entropy_report *out);
/* The tensor's sections: sizes, T, lengths, and DEVICE pointers. */
int ecf8_tensor_sections(const ecf8_dev_tensor *t, ecf8_sections *out);
/* Copy sections to host buffers sized by ecf8_tensor_sections (NULL skips). */
int ecf8_tensor_download(const ecf8_dev_tensor *t, uint8_t *encoded, uint8_t *gaps, uint64_t *outpos,
                         uint8_t *packed);

/* Decode into device memory d_out (n_elem bytes, 16-byte aligned). */
int ecf8_decode_device(const ecf8_dev_tensor *t, uint8_t *d_out, void *stream);

/* Many tensors, one launch.  The batch copies its descriptors to the device
 * once; ecf8_batch_decode may then be called repeatedly (and captured in a
 * CUDA graph). */
int ecf8_batch_create(const ecf8_dev_tensor *const *ts, uint8_t *const *d_outs, int count,
                      ecf8_batch **out);
int ecf8_batch_decode(const ecf8_batch *b, void *stream);
void ecf8_batch_free(ecf8_batch *b);
/* Launches of the decode kernel issued by one ecf8_batch_decode call. */
int ecf8_batch_launches(const ecf8_batch *b);

/* ---- decode-fused tcgen05 FP8 GEMM (no reference counterpart; the paper's
 * decode-then-use, fused into one kernel) --------------
 *
 * `t` holds an n x k FP8 weight W in the tiled layout of
 * ecf8_host_fused_layout (128 x 128 tiles, each in the swizzled shared-memory
 * image the tensor core reads), ECF8-encoded with T in [8, 256].  The GEMM
 *   y[m, n] = scale * sum_k x[m, k] * W[n, k]     (fp32 accumulate / out)
 * decodes W tile by tile into shared memory; decoded weights never reach
 * HBM.  x: m x k E4M3 row-major on the device (16-byte aligned), 1 <= m <=
 * 256; y: m x n fp32 row-major (16-byte aligned).  w_fmt: 0 = E4M3, 1 = E5M2 weights.  The
 * fused handle keeps a pointer to `t`, which must outlive it. */
int ecf8_fused_create(const ecf8_dev_tensor *t, uint64_t n, uint64_t k, int w_fmt, ecf8_fused **out);
int ecf8_fused_gemm(const ecf8_fused *f, const uint8_t *d_x, uint32_t m, float scale, float *d_y, void *stream);
/* CTAs sharing one 128-row tile of W (rounded up): the launch is cut into
 * balanced runs of weight tiles, one per SM; partial sums are added into y. */
int ecf8_fused_split_k(const ecf8_fused *f);
/* Rows [row0, row1) (whole 128-row tiles) of the fused weight decoded back to
 * row-major FP8 bytes at d_rows ((row1 - row0) x k, 16-byte aligned),
 * stream-ordered: the large-m path of the fused linear (decode a chunk of W
 * into an L2-resident buffer, then a dense FP8 GEMM on it).  Needs a
 * byte-step weight whose tiles all decode directly (encoder output). */
int ecf8_fused_decode_rows(const ecf8_fused *f, uint64_t row0, uint64_t row1, uint8_t *d_rows, void *stream);
/* 1 when the weight decodes by byte steps with every tile direct (the
 * fused kernel's byte-step variant; ecf8_fused_decode_rows available). */
int ecf8_fused_byte_steps(const ecf8_fused *f);
void ecf8_fused_free(ecf8_fused *f);
/* ecf8_host_fused_layout on device memory, stream-ordered: row-major n x k
 * FP8 bytes <-> the tiled, swizzled sequence (inverse != 0: back).  With the
 * device decoder and encoder this re-tiles a weight from a reference-format
 * container (row-major, any T) for the fused GEMM without a host round trip:
 * decode -> ecf8_fused_layout_device -> ecf8_encode_device (T = 128). */
int ecf8_fused_layout_device(const uint8_t *d_in, uint64_t n, uint64_t k, uint8_t *d_out, int inverse, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ECF8_CUDA_H */
