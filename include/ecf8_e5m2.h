/*
 * ecf8_e5m2.h -- C ABI of the native E5M2 variant of ECF8 (SURVEY.md §8(f)
 * row 3).  The reference is E4M3-only ("E5M2 is
 * not supported"), so these entry points extend the format rather than
 * replace a reference function; every rule not listed here is the
 * reference's (codec.cpp:49-273, huffman.cpp:43-157, container.cpp:142-250).
 *
 * Format of one tensor (ecf8_e5_sections):
 *   symbol   the 5-bit exponent field (b >> 2) & 31 of each E5M2 byte b,
 *            Huffman-coded with a 32-symbol length-limited (16) code built
 *            by package-merge with the reference's tie rules; canonical
 *            codes in (length, symbol) order
 *   encoded  MSB-first code stream in 64-bit windows, T windows per block,
 *            n_blocks * T * 8 + 2 bytes (2 lookahead bytes)
 *   gaps     per window the start bit of the first code word starting in
 *            it (4 bits, even window in the high nibble)
 *   outpos   n_blocks + 1 exclusive symbol offsets by starting window
 *   raw      sign and the two mantissa bits as three bit planes: per 32
 *            elements three little-endian u32 words (signs, mantissa bit 1,
 *            mantissa bit 0), element i of the group at bit i;
 *            12 * ceil(n_elem / 32) bytes
 * Decoding takes, per window, the code words that start in [gap, 64); per
 * block the counts are scanned and clamped to the block's outpos range; a
 * window position no code word matches decodes as the lowest present symbol
 * with its own length (the reference table's fallback rule).
 *
 * Container ("EC5M"): magic, u32 version 1, u32 count; per tensor u16
 * name_len + name, u8 rank + u64 dims, u64 n_elem, u32 T, 32 code lengths,
 * u64 encoded_len + encoded, u64 gaps_len + gaps, (n_blocks + 1) u64 outpos,
 * u64 raw_len + raw.  Little-endian; validated like parse_container
 * (container.cpp:182-250) with the variant's sizes.
 *
 * Status codes and ecf8_last_error() are those of ecf8_cuda.h.
 */
#ifndef ECF8_E5M2_H
#define ECF8_E5M2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ecf8_e5_sections {
  uint64_t n_elem;
  uint32_t threads_per_block; /* T, power of two in [1, 1024] */
  uint8_t lengths[32];        /* code length per 5-bit exponent, 0 = absent, <= 16 */
  const uint8_t *encoded;
  uint64_t encoded_len;
  const uint8_t *gaps;
  uint64_t gaps_len;
  const uint64_t *outpos;
  uint64_t n_outpos;
  const uint8_t *raw;
  uint64_t raw_len;
} ecf8_e5_sections;

typedef struct ecf8_e5_host_tensor ecf8_e5_host_tensor;
typedef struct ecf8_e5_host_file ecf8_e5_host_file;
typedef struct ecf8_e5_dev_tensor ecf8_e5_dev_tensor;

/* ---- host: code, encoder, container (csrc/host/e5m2.cpp) -------------- */
int ecf8_e5_build_code(const uint64_t counts[32], uint8_t lengths[32]);
/* Histogram -> code -> stream + raw planes of n E5M2 bytes. */
int ecf8_e5_encode(const uint8_t *e5m2, uint64_t n, uint32_t T, ecf8_e5_host_tensor **out);
int ecf8_e5_tensor_sections(const ecf8_e5_host_tensor *t, ecf8_e5_sections *out);
void ecf8_e5_tensor_free(ecf8_e5_host_tensor *t);
/* A raw FP8R file (container.cpp:128-140) of E5M2 tensors -> EC5M container
 * (free *out with ecf8_host_free). */
int ecf8_e5_compress_raw(const uint8_t *raw_file, size_t len, uint32_t T, uint8_t **out, size_t *out_len);
int ecf8_e5_parse(const uint8_t *bytes, size_t len, ecf8_e5_host_file **out);
int ecf8_e5_file_count(const ecf8_e5_host_file *f);
int ecf8_e5_file_tensor(const ecf8_e5_host_file *f, int i, ecf8_e5_sections *out, const char **name);
int ecf8_e5_file_shape(const ecf8_e5_host_file *f, int i, uint64_t *dims, int max_rank, int *rank);
void ecf8_e5_file_free(ecf8_e5_host_file *f);
/* EC5M container -> FP8R raw file, every tensor decoded on the B200. */
int ecf8_e5_decompress(const uint8_t *bytes, size_t len, uint8_t **out, size_t *out_len);

/* ---- device decode (csrc/cuda/e5_decode.cu) --------------------------- */
/* Sections -> HBM (one arena, 64 zero bytes after each section) + tables. */
int ecf8_e5_upload(const ecf8_e5_sections *host, ecf8_e5_dev_tensor **out);
/* Decode into device memory d_out (n_elem bytes, 16-byte aligned), stream-ordered. */
int ecf8_e5_decode_device(const ecf8_e5_dev_tensor *t, uint8_t *d_out, void *stream);
uint64_t ecf8_e5_dev_n_elem(const ecf8_e5_dev_tensor *t);
/* 1 when the tensor decodes by byte steps (a complete code, T in [8, 256],
 * every tile passed the upload check), 0 for the per-window walk. */
int ecf8_e5_dev_byte_steps(const ecf8_e5_dev_tensor *t);
void ecf8_e5_free(ecf8_e5_dev_tensor *t);
/* Host spans: upload, decode, copy back (synchronous). */
int ecf8_e5_decode_host(const ecf8_e5_sections *host, uint8_t *out, uint64_t out_len);

#ifdef __cplusplus
}
#endif

#endif /* ECF8_E5M2_H */
