/*
 * ecf8_oracle.c -- CPU restatement of the reference ECF8 codec (plain C99).
 *
 * TEST INFRASTRUCTURE ONLY (see ecf8_oracle.h).  Written from the reference
 * algorithm description; each function cites the reference lines it follows.
 * Nothing here is tuned: it is the checker, not the product.
 */
#include "ecf8_oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NSYM 16
#define MAXLEN 16

/* ---------------------------------------------------------------- codes */

/* huffman.cpp:131-157: validate cap + Kraft, then hand out words in
 * (length, symbol) order, MSB-first. */
int orc_canonical_codes(const uint8_t lengths[16], uint16_t codes[16]) {
  uint64_t kraft = 0;
  int present = 0;
  for (int s = 0; s < NSYM; ++s) {
    codes[s] = 0;
    if (!lengths[s]) continue;
    if (lengths[s] > MAXLEN) return ORC_EINVAL;
    kraft += 1ull << (MAXLEN - lengths[s]);
    ++present;
  }
  if (!present || kraft > (1ull << MAXLEN)) return ORC_EINVAL;
  uint32_t code = 0;
  int prev = -1, first = 1;
  for (int len = 1; len <= MAXLEN; ++len) {
    for (int s = 0; s < NSYM; ++s) {
      if (lengths[s] != len) continue;
      if (first) {
        code = 0;
        first = 0;
      } else {
        code = (code + 1) << (len - prev);
      }
      codes[s] = (uint16_t)code;
      prev = len;
    }
  }
  return ORC_OK;
}

/* huffman.cpp:30-107: package-merge.  Items carry a weight and per-symbol
 * leaf multiplicities; packages win weight ties in the merge. */
typedef struct {
  uint64_t w;
  uint8_t leaf[NSYM];
} pm_item;

int orc_build_code(const uint64_t counts[16], uint8_t lengths[16]) {
  int order[NSYM], n = 0;
  memset(lengths, 0, NSYM);
  for (int s = 0; s < NSYM; ++s)
    if (counts[s]) order[n++] = s;
  if (n == 0) return ORC_EINVAL;
  if (n == 1) { /* huffman.cpp:122-124 */
    lengths[order[0]] = 1;
    return ORC_OK;
  }
  /* singletons sorted by (count, symbol): huffman.cpp:67-71 */
  for (int i = 1; i < n; ++i)
    for (int j = i; j > 0; --j) {
      int a = order[j - 1], b = order[j];
      if (counts[a] > counts[b] || (counts[a] == counts[b] && a > b)) {
        order[j - 1] = b;
        order[j] = a;
      } else
        break;
    }
  pm_item singles[NSYM];
  for (int i = 0; i < n; ++i) {
    memset(&singles[i], 0, sizeof(pm_item));
    singles[i].w = counts[order[i]];
    singles[i].leaf[order[i]] = 1;
  }
  pm_item cur[4 * NSYM], packs[4 * NSYM], next[4 * NSYM];
  int ncur = n;
  memcpy(cur, singles, sizeof(pm_item) * n);
  for (int level = MAXLEN - 1; level >= 1; --level) { /* huffman.cpp:85-91 */
    int np = 0;
    for (int i = 0; i + 1 < ncur; i += 2) {
      packs[np].w = cur[i].w + cur[i + 1].w;
      for (int s = 0; s < NSYM; ++s) packs[np].leaf[s] = cur[i].leaf[s] + cur[i + 1].leaf[s];
      ++np;
    }
    int i = 0, j = 0, k = 0;
    while (i < n || j < np) { /* merge_lists, huffman.cpp:46-63 */
      if (i == n) next[k++] = packs[j++];
      else if (j == np) next[k++] = singles[i++];
      else if (packs[j].w <= singles[i].w) next[k++] = packs[j++];
      else next[k++] = singles[i++];
    }
    memcpy(cur, next, sizeof(pm_item) * k);
    ncur = k;
  }
  int take = 2 * (n - 1); /* huffman.cpp:96-106 */
  if (take > ncur) return ORC_EINVAL;
  uint32_t tally[NSYM] = {0};
  for (int i = 0; i < take; ++i)
    for (int s = 0; s < NSYM; ++s) tally[s] += cur[i].leaf[s];
  for (int s = 0; s < NSYM; ++s) {
    if (tally[s] > MAXLEN) return ORC_EINVAL;
    lengths[s] = (uint8_t)tally[s];
  }
  return ORC_OK;
}

/* ----------------------------------------------------------------- LUT */

/* lut.cpp:47-97 */
int orc_build_lut(const uint8_t lengths[16], uint8_t *entries, uint32_t *n_luts) {
  uint16_t codes[NSYM];
  int fb = -1;
  uint64_t kraft = 0;
  for (int s = 0; s < NSYM; ++s) {
    if (!lengths[s]) continue;
    if (lengths[s] > MAXLEN) return ORC_EINVAL;
    kraft += 1ull << (MAXLEN - lengths[s]);
    if (fb < 0) fb = s;
  }
  if (fb < 0 || kraft > (1ull << MAXLEN)) return ORC_EINVAL;
  if (orc_canonical_codes(lengths, codes) != ORC_OK) return ORC_EINVAL;

  uint8_t root[256];
  unsigned prefixes[NSYM + 1];
  int nprefix = 0;
  for (unsigned b = 0; b < 256; ++b) {
    int hit = -1; /* lut.cpp:25-31 short_match: first symbol in index order */
    for (int s = 0; s < NSYM && hit < 0; ++s) {
      int len = lengths[s];
      if (len >= 1 && len <= 8 && (b >> (8 - len)) == codes[s]) hit = s;
    }
    if (hit >= 0) {
      root[b] = (uint8_t)hit;
      continue;
    }
    int longp = 0; /* lut.cpp:16-22 */
    for (int s = 0; s < NSYM; ++s) {
      int len = lengths[s];
      if (len > 8 && (unsigned)(codes[s] >> (len - 8)) == b) longp = 1;
    }
    if (longp) {
      int idx = 0;
      while (idx < nprefix && prefixes[idx] != b) ++idx;
      if (idx == nprefix) prefixes[nprefix++] = b;
      if (nprefix > 16) return ORC_EINVAL;
      root[b] = (uint8_t)(255 - idx);
    } else {
      root[b] = (uint8_t)fb;
    }
  }
  uint32_t nl = 2 + (uint32_t)nprefix;
  memset(entries, 0, 256 * nl);
  memcpy(entries, root, 256);
  for (int i = 0; i < nprefix; ++i) { /* lut.cpp:34-44, 85-91 */
    uint8_t *sub = entries + 256 * (i + 1);
    for (unsigned b2 = 0; b2 < 256; ++b2) {
      int hit = -1;
      for (int s = 0; s < NSYM && hit < 0; ++s) {
        int len = lengths[s];
        if (len <= 8) continue;
        if ((unsigned)(codes[s] >> (len - 8)) != prefixes[i]) continue;
        unsigned rest = codes[s] & ((1u << (len - 8)) - 1);
        if ((b2 >> (16 - len)) == rest) hit = s;
      }
      sub[b2] = (uint8_t)(hit >= 0 ? hit : fb);
    }
  }
  for (int s = 0; s < NSYM; ++s) entries[256 * (nl - 1) + s] = lengths[s];
  *n_luts = nl;
  return ORC_OK;
}

/* lut.hpp:43-49 */
void orc_decode_one(const uint8_t *e, uint32_t n_luts, uint16_t window, uint8_t *symbol,
                    uint8_t *bits) {
  uint32_t x = e[window >> 8];
  if (x >= 240) x = e[256u * (256u - x) + (window & 0xffu)];
  *symbol = (uint8_t)x;
  *bits = e[256u * (n_luts - 1) + x];
}

/* -------------------------------------------------------------- encoder */

/* codec.cpp:39-47 */
int64_t orc_n_blocks(uint64_t bitstream_bytes, uint32_t T) {
  if (T == 0 || T > 1024 || (T & (T - 1))) return -1;
  uint64_t bb = (uint64_t)T * 8;
  return (int64_t)((bitstream_bytes + bb - 1) / bb);
}

int orc_encoded_sizes(const uint8_t *fp8, uint64_t n, const uint8_t lengths[16], uint32_t T,
                      uint64_t *n_blocks, uint64_t *encoded_len, uint64_t *gaps_len,
                      uint64_t *packed_len) {
  uint64_t bits = 0;
  for (uint64_t i = 0; i < n; ++i) {
    unsigned s = (fp8[i] >> 3) & 15;
    if (!lengths[s]) return ORC_EINVAL; /* codec.cpp:53 */
    bits += lengths[s];
  }
  int64_t nb = orc_n_blocks((bits + 7) / 8, T);
  if (nb < 0) return ORC_EINVAL;
  *n_blocks = (uint64_t)nb;
  *encoded_len = (uint64_t)nb * T * 8 + 2;
  *gaps_len = ((uint64_t)nb * T + 1) / 2;
  *packed_len = (n + 1) / 2;
  return ORC_OK;
}

/* codec.cpp:49-98 (bitstream, gaps, outpos) + fp8.cpp:8-18 (nibbles). */
int orc_encode(const uint8_t *fp8, uint64_t n, const uint8_t lengths[16], uint32_t T,
               uint8_t *encoded, uint8_t *gaps, uint64_t *outpos, uint8_t *packed) {
  uint64_t nb, el, gl, pl;
  int rc = orc_encoded_sizes(fp8, n, lengths, T, &nb, &el, &gl, &pl);
  if (rc) return rc;
  uint16_t codes[NSYM];
  if (n && orc_canonical_codes(lengths, codes)) return ORC_EINVAL;
  memset(encoded, 0, el);
  memset(gaps, 0, gl);
  memset(outpos, 0, (nb + 1) * sizeof(uint64_t));
  memset(packed, 0, pl);
  uint64_t pos = 0, last_window = ~0ull;
  for (uint64_t i = 0; i < n; ++i) {
    unsigned s = (fp8[i] >> 3) & 15;
    uint64_t w = pos >> 6;
    if (w != last_window) {
      unsigned gap = (unsigned)(pos & 63);
      gaps[w / 2] |= (uint8_t)(gap << (4 - (w % 2) * 4));
      last_window = w;
    }
    outpos[w / T + 1] += 1;
    for (int k = lengths[s] - 1; k >= 0; --k, ++pos) /* MSB-first bit writer */
      if ((codes[s] >> k) & 1) encoded[pos >> 3] |= (uint8_t)(0x80u >> (pos & 7));
    uint8_t nib = (uint8_t)(((fp8[i] >> 4) & 8) | (fp8[i] & 7)); /* fp8.hpp:28-30 */
    if (i % 2 == 0) packed[i / 2] = (uint8_t)(nib << 4);
    else packed[i / 2] |= nib;
  }
  for (uint64_t b = 1; b <= nb; ++b) outpos[b] += outpos[b - 1];
  return ORC_OK;
}

/* -------------------------------------------------------------- decoders */

static uint16_t window16(const uint8_t *buf, uint64_t len, uint64_t bit) { /* codec.cpp:28-35 */
  uint64_t byte = bit >> 3;
  unsigned sh = (unsigned)(bit & 7);
  uint32_t w = 0;
  for (int i = 0; i < 3; ++i) w = (w << 8) | (byte + i < len ? buf[byte + i] : 0);
  return (uint16_t)(w >> (8 - sh));
}

static uint8_t assemble(uint8_t x, uint8_t q) { /* fp8.hpp:42-44 */
  return (uint8_t)((x << 3) | (q & 0x80) | ((q >> 4) & 7));
}

static uint8_t nibble_high(const uint8_t *packed, uint64_t i) { /* fp8.hpp:55-57 */
  return (uint8_t)(packed[i / 2] << ((i % 2) * 4));
}

int orc_decode_reference(const uint8_t *encoded, uint64_t encoded_len, const uint8_t *packed,
                         uint64_t n_elem, const uint8_t lengths[16], uint8_t *out) {
  if (!n_elem) return ORC_OK;
  uint8_t lut[18 * 256];
  uint32_t nl;
  if (orc_build_lut(lengths, lut, &nl)) return ORC_EINVAL;
  uint64_t cap = encoded_len * 8, pos = 0;
  for (uint64_t i = 0; i < n_elem; ++i) {
    if (pos >= cap) return ORC_ETRUNC; /* codec.cpp:117 */
    uint8_t s, b;
    orc_decode_one(lut, nl, window16(encoded, encoded_len, pos), &s, &b);
    out[i] = assemble(s, nibble_high(packed, i));
    pos += b;
  }
  return ORC_OK;
}

static uint64_t be64(const uint8_t *p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v = (v << 8) | p[i];
  return v;
}

/* codec.cpp:133-161 */
uint32_t orc_count_phase(const uint8_t w10[10], unsigned gap, const uint8_t *e, uint32_t nl) {
  uint64_t L = be64(w10) << gap;
  uint16_t S = (uint16_t)((w10[8] << 8) | w10[9]);
  unsigned f = gap;
  uint32_t c = 0;
  uint8_t s, b;
  while (f < 16) {
    orc_decode_one(e, nl, (uint16_t)(L >> 48), &s, &b);
    L <<= b;
    f += b;
    ++c;
  }
  L |= (uint64_t)S << (f - 16);
  f -= 16;
  while (f < 48) {
    orc_decode_one(e, nl, (uint16_t)(L >> 48), &s, &b);
    L <<= b;
    f += b;
    ++c;
  }
  return c;
}

/* codec.cpp:168-190 */
static void emit_phase(const uint8_t *w10, unsigned gap, const uint8_t *e, uint32_t nl,
                       const uint8_t *packed, uint64_t o, uint64_t o_end, uint64_t o_base,
                       uint8_t *staging) {
  if (o >= o_end) return;
  uint64_t L = be64(w10) << gap;
  uint16_t S = (uint16_t)((w10[8] << 8) | w10[9]);
  unsigned f = gap;
  uint8_t s, b;
  while (f < 16) {
    orc_decode_one(e, nl, (uint16_t)(L >> 48), &s, &b);
    staging[o - o_base] = assemble(s, nibble_high(packed, o));
    if (++o == o_end) return;
    L <<= b;
    f += b;
  }
  L |= (uint64_t)S << (f - 16);
  for (;;) {
    orc_decode_one(e, nl, (uint16_t)(L >> 48), &s, &b);
    staging[o - o_base] = assemble(s, nibble_high(packed, o));
    if (++o == o_end) return;
    L <<= b;
  }
}

static unsigned gap_at(const uint8_t *gaps, uint64_t t) { /* codec.hpp:50-52 */
  return (gaps[t / 2] >> (4 - (t % 2) * 4)) & 15;
}

/* codec.cpp:201-254 for one block, scratch supplied by the caller. */
static void decode_block(const uint8_t *encoded, const uint8_t *gaps, const uint64_t *outpos,
                         uint32_t T, const uint8_t *packed, const uint8_t *e, uint32_t nl,
                         uint64_t block, uint8_t *out, uint32_t *counts, uint64_t *acc,
                         uint8_t *staging) {
  uint64_t o_base = outpos[block], o_limit = outpos[block + 1];
  if (o_limit == o_base) return;
  for (uint32_t t = 0; t < T; ++t) {
    uint64_t tg = block * T + t;
    counts[t] = orc_count_phase(encoded + tg * 8, gap_at(gaps, tg), e, nl);
  }
  /* Blelloch up-sweep / down-sweep (codec.cpp:227-237) */
  for (uint32_t i = 0; i < T; ++i) acc[i] = counts[i];
  for (uint32_t d = 1; d < T; d <<= 1)
    for (uint32_t i = 2 * d - 1; i < T; i += 2 * d) acc[i] += acc[i - d];
  acc[T - 1] = 0;
  for (uint32_t d = T >> 1; d >= 1; d >>= 1)
    for (uint32_t i = 2 * d - 1; i < T; i += 2 * d) {
      uint64_t l = acc[i - d];
      acc[i - d] = acc[i];
      acc[i] += l;
    }
  for (uint32_t t = 0; t < T; ++t) { /* codec.cpp:242-251 */
    uint64_t o_start = o_base + acc[t];
    if (o_start >= o_limit) continue;
    uint64_t o_end = o_start + counts[t];
    if (o_end > o_limit) o_end = o_limit;
    uint64_t tg = block * T + t;
    emit_phase(encoded + tg * 8, gap_at(gaps, tg), e, nl, packed, o_start, o_end, o_base,
               staging);
  }
  memcpy(out + o_base, staging, o_limit - o_base); /* codec.cpp:253 */
}

static int check_sections(uint64_t encoded_len, uint64_t gaps_len, uint64_t n_blocks, uint32_t T,
                          const uint64_t *outpos, uint64_t n_elem) {
  if (orc_n_blocks(0, T) < 0) return ORC_EINVAL;
  if (encoded_len != n_blocks * T * 8 + 2) return ORC_EINVAL;
  if (gaps_len != (n_blocks * T + 1) / 2) return ORC_EINVAL;
  if (outpos[n_blocks] != n_elem) return ORC_EINVAL; /* codec.cpp:260-261 */
  return ORC_OK;
}

int orc_decode_parallel_mt(const uint8_t *encoded, uint64_t encoded_len, const uint8_t *gaps,
                           uint64_t gaps_len, const uint64_t *outpos, uint64_t n_blocks,
                           uint32_t T, const uint8_t *packed, uint64_t n_elem,
                           const uint8_t lengths[16], uint8_t *out, int nthreads) {
  int rc = check_sections(encoded_len, gaps_len, n_blocks, T, outpos, n_elem);
  if (rc || !n_elem) return rc;
  uint8_t lut[18 * 256];
  uint32_t nl;
  if (orc_build_lut(lengths, lut, &nl)) return ORC_EINVAL;
  int64_t nb = (int64_t)n_blocks;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#else
  (void)nthreads;
#endif
  {
    uint32_t *counts = (uint32_t *)malloc(sizeof(uint32_t) * T);
    uint64_t *acc = (uint64_t *)malloc(sizeof(uint64_t) * T);
    uint8_t *staging = (uint8_t *)malloc((size_t)T * 64);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t b = 0; b < nb; ++b)
      decode_block(encoded, gaps, outpos, T, packed, lut, nl, (uint64_t)b, out, counts, acc,
                   staging);
    free(counts);
    free(acc);
    free(staging);
  }
  return ORC_OK;
}

int orc_decode_parallel(const uint8_t *encoded, uint64_t encoded_len, const uint8_t *gaps,
                        uint64_t gaps_len, const uint64_t *outpos, uint64_t n_blocks, uint32_t T,
                        const uint8_t *packed, uint64_t n_elem, const uint8_t lengths[16],
                        uint8_t *out) {
  return orc_decode_parallel_mt(encoded, encoded_len, gaps, gaps_len, outpos, n_blocks, T, packed,
                                n_elem, lengths, out, 1);
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
