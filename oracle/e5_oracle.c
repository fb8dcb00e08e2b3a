/*
 * e5_oracle.c -- TEST INFRASTRUCTURE ONLY: a plain-C statement of the native
 * E5M2 variant of ECF8, used by tests/ as the checker
 * of the product encoder (csrc/host/e5m2.cpp) and the GPU decoder
 * (csrc/cuda/e5_decode.cu).  Nothing in the product links or calls it.
 *
 * There is no reference implementation of this variant: the reference is
 * E4M3-only ("E5M2 is not supported").  The
 * variant keeps every rule of the reference's E4M3 format and changes only
 * the symbol alphabet and the raw field:
 *   symbol  = the 5-bit exponent field, (b >> 2) & 31   (32 symbols)
 *   raw     = sign (bit 7) and the two mantissa bits (bits 1, 0), stored as
 *             three bit planes: per 32 elements three little-endian u32
 *             words -- signs, mantissa bit 1, mantissa bit 0 -- element i of
 *             the group at bit i (raw_len = 12 * ceil(n / 32), tail zero)
 * and, unchanged from the reference:
 *   code    = length-limited (16) Huffman by package-merge with the
 *             reference's tie rules (huffman.cpp:43-107) over 32 symbols,
 *             canonical codes in (length, symbol) order (huffman.cpp:131-157)
 *   stream  = MSB-first codes, 64-bit windows, gap = start of the first word
 *             starting in the window, outpos by starting window, T-window
 *             blocks, 2 lookahead bytes (codec.cpp:49-98)
 *   decode  = per window, the words that start in [gap, 64); per block,
 *             counts -> exclusive scan -> clamp to the block's outpos range
 *             (codec.cpp:133-253); a window position no code word matches
 *             decodes as the lowest present symbol with its own length (the
 *             reference table's fallback, lut.cpp:47-97).
 * Parity of this variant is therefore pinned by round trips (decode(encode(x))
 * == x) and by agreement of three independent implementations, not by
 * reference golden vectors.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NS 32
#define MAXL 16
#define OK 0
#define EINVAL 1

typedef struct {
  uint64_t w;
  uint8_t leaf[NS];
} item5;

/* huffman.cpp:43-107 (package-merge, coin-collector form) over 32 symbols */
int orc5_build_code(const uint64_t counts[NS], uint8_t lengths[NS]) {
  int order[NS], n = 0;
  memset(lengths, 0, NS);
  for (int s = 0; s < NS; ++s)
    if (counts[s]) order[n++] = s;
  if (n == 0) return EINVAL;
  if (n == 1) {
    lengths[order[0]] = 1;
    return OK;
  }
  for (int i = 1; i < n; ++i)
    for (int j = i; j > 0; --j) {
      int a = order[j - 1], b = order[j];
      if (counts[a] > counts[b] || (counts[a] == counts[b] && a > b)) {
        order[j - 1] = b;
        order[j] = a;
      } else
        break;
    }
  item5 *singles = calloc(NS, sizeof(item5)), *cur = calloc(4 * NS, sizeof(item5)),
        *packs = calloc(4 * NS, sizeof(item5)), *next = calloc(4 * NS, sizeof(item5));
  for (int i = 0; i < n; ++i) {
    singles[i].w = counts[order[i]];
    singles[i].leaf[order[i]] = 1;
  }
  int ncur = n;
  memcpy(cur, singles, sizeof(item5) * n);
  for (int level = MAXL - 1; level >= 1; --level) {
    int np = 0;
    for (int i = 0; i + 1 < ncur; i += 2) {
      packs[np].w = cur[i].w + cur[i + 1].w;
      for (int s = 0; s < NS; ++s) packs[np].leaf[s] = cur[i].leaf[s] + cur[i + 1].leaf[s];
      ++np;
    }
    int i = 0, j = 0, k = 0;
    while (i < n || j < np) {
      if (i == n) next[k++] = packs[j++];
      else if (j == np) next[k++] = singles[i++];
      else if (packs[j].w <= singles[i].w) next[k++] = packs[j++];
      else next[k++] = singles[i++];
    }
    memcpy(cur, next, sizeof(item5) * k);
    ncur = k;
  }
  int rc = OK, take = 2 * (n - 1);
  if (take > ncur) rc = EINVAL;
  uint32_t tally[NS] = {0};
  for (int i = 0; rc == OK && i < take; ++i)
    for (int s = 0; s < NS; ++s) tally[s] += cur[i].leaf[s];
  for (int s = 0; rc == OK && s < NS; ++s) {
    if (tally[s] > MAXL) rc = EINVAL;
    lengths[s] = (uint8_t)tally[s];
  }
  free(singles), free(cur), free(packs), free(next);
  return rc;
}

/* huffman.cpp:131-157: codes in (length, symbol) order; Kraft sum <= 1 */
int orc5_canonical_codes(const uint8_t lengths[NS], uint16_t codes[NS]) {
  uint64_t kraft = 0;
  int any = 0;
  for (int s = 0; s < NS; ++s) {
    if (lengths[s] > MAXL) return EINVAL;
    if (lengths[s]) kraft += 1ull << (MAXL - lengths[s]), any = 1;
  }
  if (!any || kraft > (1ull << MAXL)) return EINVAL;
  uint32_t code = 0;
  int prev = 0;
  for (int l = 1; l <= MAXL; ++l)
    for (int s = 0; s < NS; ++s)
      if (lengths[s] == l) {
        code <<= (l - prev);
        prev = l;
        codes[s] = (uint16_t)code++;
      }
  return OK;
}

uint64_t orc5_raw_len(uint64_t n) { return 12 * ((n + 31) / 32); }

int orc5_sizes(const uint8_t *e5, uint64_t n, const uint8_t lengths[NS], uint32_t T, uint64_t *n_blocks,
               uint64_t *encoded_len, uint64_t *gaps_len, uint64_t *raw_len) {
  if (T == 0 || T > 1024 || (T & (T - 1))) return EINVAL;
  uint64_t bits = 0;
  for (uint64_t i = 0; i < n; ++i) {
    unsigned s = (e5[i] >> 2) & 31;
    if (!lengths[s]) return EINVAL;
    bits += lengths[s];
  }
  uint64_t bb = (uint64_t)T * 8, nb = ((bits + 7) / 8 + bb - 1) / bb;
  *n_blocks = nb;
  *encoded_len = nb * T * 8 + 2;
  *gaps_len = (nb * T + 1) / 2;
  *raw_len = orc5_raw_len(n);
  return OK;
}

/* codec.cpp:49-98 with 5-bit symbols, plus the raw bit planes */
int orc5_encode(const uint8_t *e5, uint64_t n, const uint8_t lengths[NS], uint32_t T, uint8_t *encoded,
                uint8_t *gaps, uint64_t *outpos, uint8_t *raw) {
  uint64_t nb, el, gl, rl;
  int rc = orc5_sizes(e5, n, lengths, T, &nb, &el, &gl, &rl);
  if (rc) return rc;
  uint16_t codes[NS];
  if (n && orc5_canonical_codes(lengths, codes)) return EINVAL;
  memset(encoded, 0, el);
  memset(gaps, 0, gl);
  memset(outpos, 0, (nb + 1) * sizeof(uint64_t));
  memset(raw, 0, rl);
  uint64_t pos = 0, last_window = ~0ull;
  for (uint64_t i = 0; i < n; ++i) {
    const uint8_t b = e5[i];
    unsigned s = (b >> 2) & 31;
    uint64_t w = pos >> 6;
    if (w != last_window) {
      gaps[w / 2] |= (uint8_t)((pos & 63) << (4 - (w % 2) * 4));
      last_window = w;
    }
    outpos[w / T + 1] += 1;
    for (int k = lengths[s] - 1; k >= 0; --k, ++pos)
      if ((codes[s] >> k) & 1) encoded[pos >> 3] |= (uint8_t)(0x80u >> (pos & 7));
    const uint64_t g = i / 32, bit = i % 32;
    const unsigned plane[3] = {(unsigned)(b >> 7) & 1u, (unsigned)(b >> 1) & 1u, (unsigned)b & 1u};
    for (int p = 0; p < 3; ++p)
      if (plane[p]) raw[12 * g + 4 * p + bit / 8] |= (uint8_t)(1u << (bit % 8));
  }
  for (uint64_t b = 1; b <= nb; ++b) outpos[b] += outpos[b - 1];
  return OK;
}

/* one code word from the 16-bit MSB-aligned window w (canonical decode; no
 * match: the lowest present symbol with its own length) */
static void decode_one5(const uint8_t lengths[NS], const uint16_t codes[NS], uint16_t w, unsigned *sym,
                        unsigned *bits) {
  for (int l = 1; l <= MAXL; ++l)
    for (int s = 0; s < NS; ++s)
      if (lengths[s] == l && codes[s] == (w >> (16 - l))) {
        *sym = (unsigned)s, *bits = (unsigned)l;
        return;
      }
  for (int s = 0; s < NS; ++s)
    if (lengths[s]) {
      *sym = (unsigned)s, *bits = lengths[s];
      return;
    }
  *sym = 0, *bits = 1;
}

static uint16_t win16(const uint8_t *buf, uint64_t len, uint64_t bit) {
  uint64_t byte = bit >> 3;
  uint32_t w = 0;
  for (int i = 0; i < 3; ++i) w = (w << 8) | (byte + i < len ? buf[byte + i] : 0);
  return (uint16_t)(w >> (8 - (bit & 7)));
}

static uint8_t assemble5(unsigned sym, const uint8_t *raw, uint64_t i) {
  const uint64_t g = i / 32, bit = i % 32;
  const unsigned s = (raw[12 * g + bit / 8] >> (bit % 8)) & 1u, m1 = (raw[12 * g + 4 + bit / 8] >> (bit % 8)) & 1u,
                 m0 = (raw[12 * g + 8 + bit / 8] >> (bit % 8)) & 1u;
  return (uint8_t)((s << 7) | (sym << 2) | (m1 << 1) | m0);
}

/* codec.cpp:201-273 restated for the variant: per block, per window the
 * words that start in [gap, 64); exclusive scan of the counts; clamp */
int orc5_decode(const uint8_t lengths[NS], uint32_t T, const uint8_t *encoded, uint64_t encoded_len,
                const uint8_t *gaps, uint64_t gaps_len, const uint64_t *outpos, uint64_t n_blocks, const uint8_t *raw,
                uint64_t raw_len, uint8_t *out, uint64_t n) {
  if (T == 0 || T > 1024 || (T & (T - 1))) return EINVAL;
  if (n == 0) return OK;
  if (encoded_len != n_blocks * T * 8 + 2 || gaps_len != (n_blocks * T + 1) / 2 || raw_len != orc5_raw_len(n))
    return EINVAL;
  if (outpos[0] != 0 || outpos[n_blocks] != n) return EINVAL;
  uint16_t codes[NS];
  if (orc5_canonical_codes(lengths, codes)) return EINVAL;
  uint32_t *cnt = malloc(sizeof(uint32_t) * T);
  for (uint64_t b = 0; b < n_blocks; ++b) {
    if (outpos[b + 1] < outpos[b]) {
      free(cnt);
      return EINVAL;
    }
    for (uint32_t t = 0; t < T; ++t) {
      const uint64_t w = b * T + t;
      const unsigned gap = (gaps[w / 2] >> (4 - (w % 2) * 4)) & 15;
      uint64_t p = 64 * w + gap;
      uint32_t c = 0;
      while (p < 64 * w + 64) {
        unsigned sym, bits;
        decode_one5(lengths, codes, win16(encoded, encoded_len, p), &sym, &bits);
        p += bits;
        ++c;
      }
      cnt[t] = c;
    }
    uint64_t o = outpos[b];
    for (uint32_t t = 0; t < T; ++t) {
      const uint64_t w = b * T + t;
      const unsigned gap = (gaps[w / 2] >> (4 - (w % 2) * 4)) & 15;
      uint64_t p = 64 * w + gap;
      const uint64_t o_start = o, o_end = o + cnt[t] < outpos[b + 1] ? o + cnt[t] : outpos[b + 1];
      o += cnt[t];
      for (uint64_t k = o_start; k < o_end; ++k) {
        unsigned sym, bits;
        decode_one5(lengths, codes, win16(encoded, encoded_len, p), &sym, &bits);
        p += bits;
        out[k] = assemble5(sym, raw, k);
      }
    }
  }
  free(cnt);
  return OK;
}
