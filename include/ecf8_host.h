/*
 * ecf8_host.h -- C ABI over the host half of the library (encoder, container
 * I/O, table inspection, synthetic data), for language bindings.
 *
 * The decode path is ecf8_cuda.h; these calls never touch the GPU except
 * ecf8_host_decompress, which is decompress_streaming (container.cpp:324-352)
 * and decodes on the B200.  Status codes are ecf8_status from ecf8_cuda.h;
 * messages via ecf8_last_error().
 */
#ifndef ECF8_HOST_H
#define ECF8_HOST_H

#include <stddef.h>
#include <stdint.h>

#include "ecf8_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ecf8_host_tensor ecf8_host_tensor; /* an EncodedTensor */
typedef struct ecf8_host_file ecf8_host_file;     /* an Ecf8File      */

void ecf8_host_free(void *p);

/* build_code (huffman.cpp:111-129) on a 16-bin histogram. */
int ecf8_host_build_code(const uint64_t counts[16], uint8_t lengths[16]);
/* build_lut (lut.cpp:47-97): entries needs 18*256 bytes. */
int ecf8_host_build_lut(const uint8_t lengths[16], uint8_t *entries, uint32_t *n_luts);
/* The device tables for `lengths` (tables.hpp): fast needs 1 << 16 u32,
 * smask 1 << 16 u16, cascade 18*256 bytes (first 1 << fast_bits used). */
int ecf8_host_device_tables(const uint8_t lengths[16], uint32_t *fast, uint16_t *smask,
                            uint8_t *cascade, uint32_t *n_luts, uint32_t *fast_bits);
/* The byte-step decoder for `lengths` (tables.hpp fsm / fsm_cm): fsm needs
 * 16*256 u32, cm 16*256 bytes; *ok = 0 when the code has none (incomplete
 * code, or a 1-bit word). */
int ecf8_host_fsm_tables(const uint8_t lengths[16], uint32_t *fsm, uint8_t *cm, int *ok);

/* encode_tensor (codec.cpp:100-109) with the tensor's own build_code;
 * lengths may be NULL (histogram code) or a caller-chosen code. */
int ecf8_host_encode(const uint8_t *fp8, uint64_t n, uint32_t T, const uint8_t *lengths,
                     ecf8_host_tensor **out);
/* Many tensors, all host threads (nthreads <= 0: all). */
int ecf8_host_encode_many(const uint8_t *const *fp8, const uint64_t *n, int count, uint32_t T,
                          ecf8_host_tensor **out, int nthreads);
int ecf8_host_tensor_sections(const ecf8_host_tensor *t, ecf8_sections *out);
void ecf8_host_tensor_free(ecf8_host_tensor *t);

/* decode_reference (codec.cpp:125-131), host sequential oracle API. */
int ecf8_host_decode_reference(const ecf8_sections *s, uint8_t *out, uint64_t out_len);

/* parse_raw + compress_tensors + serialize (container.cpp:291-322). */
int ecf8_host_compress_raw(const uint8_t *raw, size_t len, uint32_t T, uint8_t **out,
                           size_t *out_len);
/* parse_container (container.cpp:182-250). */
int ecf8_host_parse(const uint8_t *bytes, size_t len, ecf8_host_file **out);
int ecf8_host_file_count(const ecf8_host_file *f);
int ecf8_host_file_tensor(const ecf8_host_file *f, int i, ecf8_sections *out, const char **name);
/* Tensor i's shape (container.hpp TensorShape): rank, then up to max_rank dims. */
int ecf8_host_file_shape(const ecf8_host_file *f, int i, uint64_t *dims, int max_rank, int *rank);
void ecf8_host_file_free(ecf8_host_file *f);
/* decompress_streaming: container bytes -> raw file bytes (B200 decode). */
int ecf8_host_decompress(const uint8_t *bytes, size_t len, uint8_t **out, size_t *out_len,
                         uint64_t *allocations, uint64_t *capacity);
/* decompress_streaming into a caller sink: write(ctx, data, n) receives the
 * raw file in order (a file descriptor, a socket, a counter).  Returns the
 * first nonzero write() result as ECF8_EIO. */
typedef int (*ecf8_write_fn)(void *ctx, const uint8_t *data, size_t n);
int ecf8_host_decompress_to(const uint8_t *bytes, size_t len, ecf8_write_fn write, void *ctx,
                            uint64_t *allocations, uint64_t *capacity);

/* synth_raw data (container.cpp:482-495), bit-identical, on nthreads host
 * threads (SplitMix64 jump-ahead). fmt 0 = E4M3, 1 = E5M2. */
int ecf8_host_synth(double alpha, double gamma, uint64_t n, uint64_t seed, int fmt, uint8_t *out,
                    int nthreads);

int ecf8_host_max_threads(void);
/* make_stats (container.cpp:386-413) of one raw tensor with a name of
 * name_len bytes and `rank` dims (the container overhead in actual_savings). */
int ecf8_host_make_stats(const uint8_t *fp8, uint64_t n, uint32_t T, uint32_t name_len, uint32_t rank,
                         ecf8_entropy_report *out);

/* Weight layout for the decode-fused GEMM (ecf8_cuda.h ecf8_fused_*): an
 * n x k row-major FP8 matrix -> 128 x 128 tiles in row-major tile order,
 * each tile as its 16384-byte shared-memory image (K-major, 128-byte rows,
 * 16-byte chunk c of row r at r*128 + ((c ^ (r & 7)) << 4)).  inverse != 0
 * maps the tiled sequence back to row-major.  n, k multiples of 128.  (New:
 * the reference has no GEMM; the tiled bytes are an ordinary tensor for the
 * unchanged encoder and container.) */
int ecf8_host_fused_layout(const uint8_t *w, uint64_t n, uint64_t k, uint8_t *out, int inverse);

#ifdef __cplusplus
}
#endif
#endif /* ECF8_HOST_H */
