/*
 * ecf8_oracle.h -- CPU restatement of the reference ECF8 codec, plain C.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 decode
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker or the timed CPU
 * baseline.  The product library (paper_2510_02676_b200/) never links it.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/...).  Pinned against the reference's own golden
 * vectors (tests/test_oracle.py) and, where /root/reference is present,
 * against the reference library itself built by oracle/Makefile into
 * oracle/_ref/ (tests/test_oracle_vs_ref.py).
 */
#ifndef ECF8_ORACLE_H
#define ECF8_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = -1, ORC_ETRUNC = -2, ORC_EFORMAT = -3 };

/* huffman.cpp:131-157 -- canonical words in (length, symbol) order. */
int orc_canonical_codes(const uint8_t lengths[16], uint16_t codes[16]);

/* huffman.cpp:43-129 -- package-merge lengths (packages win ties),
 * single present symbol gets length 1. */
int orc_build_code(const uint64_t counts[16], uint8_t lengths[16]);

/* lut.cpp:47-97 -- cascaded byte LUT.  entries must hold 18*256 bytes. */
int orc_build_lut(const uint8_t lengths[16], uint8_t *entries, uint32_t *n_luts);

/* lut.hpp:43-49 */
void orc_decode_one(const uint8_t *entries, uint32_t n_luts, uint16_t window,
                    uint8_t *symbol, uint8_t *bits);

/* codec.cpp:39-47 -- returns n_blocks; -1 on bad T. */
int64_t orc_n_blocks(uint64_t bitstream_bytes, uint32_t T);

/* codec.cpp:49-98 sizes of the encoded sections for a tensor. */
int orc_encoded_sizes(const uint8_t *fp8, uint64_t n, const uint8_t lengths[16],
                      uint32_t T, uint64_t *n_blocks, uint64_t *encoded_len,
                      uint64_t *gaps_len, uint64_t *packed_len);

/* codec.cpp:49-109 + fp8.cpp:8-37 -- encoder. Buffers sized by
 * orc_encoded_sizes (outpos holds n_blocks+1 entries). */
int orc_encode(const uint8_t *fp8, uint64_t n, const uint8_t lengths[16], uint32_t T,
               uint8_t *encoded, uint8_t *gaps, uint64_t *outpos, uint8_t *packed);

/* codec.cpp:111-131 -- single-cursor decode + nibble reassembly.
 * Returns ORC_ETRUNC when the cursor runs off the stream. */
int orc_decode_reference(const uint8_t *encoded, uint64_t encoded_len,
                         const uint8_t *packed, uint64_t n_elem,
                         const uint8_t lengths[16], uint8_t *out);

/* codec.cpp:133-161 */
uint32_t orc_count_phase(const uint8_t window10[10], unsigned gap,
                         const uint8_t *entries, uint32_t n_luts);

/* codec.cpp:168-273 -- the block-parallel algorithm (count, Blelloch scan,
 * clamp, emit, copy) restated with plain sequential loops over blocks. */
int orc_decode_parallel(const uint8_t *encoded, uint64_t encoded_len,
                        const uint8_t *gaps, uint64_t gaps_len,
                        const uint64_t *outpos, uint64_t n_blocks, uint32_t T,
                        const uint8_t *packed, uint64_t n_elem,
                        const uint8_t lengths[16], uint8_t *out);

/* Same, OpenMP over blocks when compiled with -fopenmp (timed CPU baseline
 * "port"); nthreads <= 0 means all available. */
int orc_decode_parallel_mt(const uint8_t *encoded, uint64_t encoded_len,
                           const uint8_t *gaps, uint64_t gaps_len,
                           const uint64_t *outpos, uint64_t n_blocks, uint32_t T,
                           const uint8_t *packed, uint64_t n_elem,
                           const uint8_t lengths[16], uint8_t *out, int nthreads);

int orc_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
