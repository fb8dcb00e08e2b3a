// e5m2.cpp -- host side of the native E5M2 variant (include/ecf8_e5m2.h):
// 32-symbol code, encoder (stream + raw bit planes), EC5M container.
//
// The variant keeps the reference's stream rules (codec.cpp:49-98: MSB-first
// codes, 64-bit windows, gap = start of the first word starting in a window,
// outpos by starting window, 2 lookahead bytes) and code construction
// (huffman.cpp:43-157, package-merge with the reference's tie rules,
// canonical codes); only the alphabet (5-bit exponents) and the raw field
// (sign + 2 mantissa bits as bit planes) differ.  The reference has no E5M2
// support.  Decoding runs on the B200 (csrc/cuda/e5_decode.cu).
#include <algorithm>
#include <array>
#include <bit>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "ecf8/container.hpp"
#include "ecf8/errors.hpp"
#include "ecf8_cuda.h"
#include "ecf8_e5m2.h"
#include "package_merge.hpp"

extern "C" int ecf8_internal_set_error(int status, const char* msg);

namespace ecf8::e5 {

constexpr int kSyms = 32;
constexpr int kMaxLen = 16;
constexpr char kMagic[4] = {'E', 'C', '5', 'M'};
constexpr std::uint32_t kVersion = 1;

struct Code {
  std::array<std::uint8_t, kSyms> lengths{};
  std::array<std::uint16_t, kSyms> codes{};
};

// huffman.cpp:131-157 over 32 symbols (validates the length vector).
Code canonical(const std::array<std::uint8_t, kSyms>& lengths) {
  std::uint64_t kraft = 0;
  bool any = false;
  for (std::uint8_t l : lengths) {
    if (l > kMaxLen) throw std::invalid_argument("invalid length vector");
    if (l) kraft += std::uint64_t{1} << (kMaxLen - l), any = true;
  }
  if (!any || kraft > (std::uint64_t{1} << kMaxLen)) throw std::invalid_argument("invalid length vector");
  Code c;
  c.lengths = lengths;
  std::uint32_t next = 0;
  int cur = 0;
  for (int l = 1; l <= kMaxLen; ++l)
    for (int s = 0; s < kSyms; ++s)
      if (lengths[s] == l) {
        if (cur) next <<= (l - cur);
        cur = l;
        c.codes[s] = static_cast<std::uint16_t>(next++);
      }
  return c;
}

Code build_code(const std::array<std::uint64_t, kSyms>& counts) {
  int present = 0, last = -1;
  for (int s = 0; s < kSyms; ++s)
    if (counts[s]) ++present, last = s;
  if (present == 0) throw std::invalid_argument("empty input");
  std::array<std::uint8_t, kSyms> len{};
  if (present == 1) len[last] = 1;  // a zero-length word would never advance a decoder
  else len = host::package_merge_lengths<kSyms, kMaxLen>(counts);
  return canonical(len);
}

struct Tensor {
  std::uint64_t n_elem = 0;
  std::uint32_t T = 256;
  std::array<std::uint8_t, kSyms> lengths{};
  std::vector<std::uint8_t> encoded, gaps, raw;
  std::vector<std::uint64_t> outpos;
};

std::uint64_t raw_len(std::uint64_t n) { return 12 * ((n + 31) / 32); }

Tensor encode(std::span<const std::uint8_t> x, std::uint32_t T) {
  if (T < 1 || T > 1024 || !std::has_single_bit(T))
    throw std::invalid_argument("threads per block must be a power of two in [1, 1024]");
  Tensor t;
  t.n_elem = x.size();
  t.T = T;
  if (x.empty()) {  // an empty tensor: no blocks, a 2-byte lookahead stream
    t.encoded.assign(2, 0);
    t.outpos.assign(1, 0);
    return t;
  }
  std::array<std::uint64_t, kSyms> counts{};
  for (std::uint8_t b : x) ++counts[(b >> 2) & 31];
  const Code code = build_code(counts);
  t.lengths = code.lengths;
  std::uint64_t bits = 0;
  for (int s = 0; s < kSyms; ++s) bits += counts[s] * code.lengths[s];
  const std::uint64_t bb = std::uint64_t{8} * T, bytes = (bits + 7) / 8, nb = (bytes + bb - 1) / bb;
  t.encoded.assign(nb * bb + 2, 0);
  t.gaps.assign((nb * T + 1) / 2, 0);
  t.outpos.assign(nb + 1, 0);
  t.raw.assign(raw_len(x.size()), 0);

  // 64-bit MSB-first accumulator, flushed a byte at a time (as codec.cpp)
  std::uint64_t acc = 0, pos = 0, owner = ~std::uint64_t{0};
  unsigned fill = 0;
  std::uint8_t* dst = t.encoded.data();
  std::uint32_t planes[3] = {0, 0, 0};
  for (std::uint64_t i = 0; i < x.size(); ++i) {
    const std::uint8_t b = x[i];
    const unsigned s = (b >> 2) & 31;
    const std::uint64_t w = pos >> 6;
    if (w != owner) {
      owner = w;
      t.gaps[w >> 1] |= static_cast<std::uint8_t>((pos & 63) << ((w & 1) ? 0 : 4));
    }
    t.outpos[w / T + 1] += 1;
    const unsigned len = code.lengths[s];
    acc = (acc << len) | code.codes[s];
    fill += len;
    pos += len;
    while (fill >= 8) {
      fill -= 8;
      *dst++ = static_cast<std::uint8_t>(acc >> fill);
    }
    const unsigned bit = i & 31;
    planes[0] |= static_cast<std::uint32_t>(b >> 7) << bit;
    planes[1] |= static_cast<std::uint32_t>((b >> 1) & 1) << bit;
    planes[2] |= static_cast<std::uint32_t>(b & 1) << bit;
    if (bit == 31 || i + 1 == x.size()) {
      std::uint8_t* g = t.raw.data() + 12 * (i >> 5);
      for (int p = 0; p < 3; ++p)
        for (int k = 0; k < 4; ++k) g[4 * p + k] = static_cast<std::uint8_t>(planes[p] >> (8 * k));
      planes[0] = planes[1] = planes[2] = 0;
    }
  }
  if (fill) *dst = static_cast<std::uint8_t>(acc << (8 - fill));
  for (std::size_t k = 1; k < t.outpos.size(); ++k) t.outpos[k] += t.outpos[k - 1];
  return t;
}

ecf8_e5_sections sections_of(const Tensor& t) {
  ecf8_e5_sections s{};
  s.n_elem = t.n_elem;
  s.threads_per_block = t.T;
  std::memcpy(s.lengths, t.lengths.data(), kSyms);
  s.encoded = t.encoded.data();
  s.encoded_len = t.encoded.size();
  s.gaps = t.gaps.data();
  s.gaps_len = t.gaps.size();
  s.outpos = t.outpos.data();
  s.n_outpos = t.outpos.size();
  s.raw = t.raw.data();
  s.raw_len = t.raw.size();
  return s;
}

// ---- EC5M container (layout: include/ecf8_e5m2.h)

class Cursor {
 public:
  explicit Cursor(std::span<const std::uint8_t> b) : b_(b) {}
  std::span<const std::uint8_t> take(std::uint64_t n) {
    if (b_.size() - at_ < n) throw FormatError("truncated file");
    const auto s = b_.subspan(at_, n);
    at_ += n;
    return s;
  }
  template <class U>
  U le() {
    const auto s = take(sizeof(U));
    U v = 0;
    for (std::size_t i = sizeof(U); i-- > 0;) v = static_cast<U>((v << 8) | s[i]);
    return v;
  }
  void finish() const {
    if (at_ != b_.size()) throw FormatError("trailing bytes after last tensor");
  }

 private:
  std::span<const std::uint8_t> b_;
  std::size_t at_ = 0;
};

struct Writer {
  std::vector<std::uint8_t> bytes;
  template <class U>
  void le(U v) {
    for (std::size_t i = 0; i < sizeof(U); ++i) bytes.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
  }
  void put(const void* p, std::size_t n) {
    const auto* c = static_cast<const std::uint8_t*>(p);
    bytes.insert(bytes.end(), c, c + n);
  }
};

struct Entry {
  TensorShape shape;
  Tensor t;
};

std::vector<std::uint8_t> serialize(const std::vector<Entry>& es) {
  Writer w;
  w.put(kMagic, 4);
  w.le<std::uint32_t>(kVersion);
  w.le<std::uint32_t>(static_cast<std::uint32_t>(es.size()));
  for (const Entry& e : es) {
    if (e.shape.name.size() > 0xFFFF) throw std::invalid_argument("tensor name too long");
    if (e.shape.dims.size() > 0xFF) throw std::invalid_argument("tensor rank too large");
    w.le<std::uint16_t>(static_cast<std::uint16_t>(e.shape.name.size()));
    w.put(e.shape.name.data(), e.shape.name.size());
    w.le<std::uint8_t>(static_cast<std::uint8_t>(e.shape.dims.size()));
    for (std::uint64_t d : e.shape.dims) w.le<std::uint64_t>(d);
    w.le<std::uint64_t>(e.t.n_elem);
    w.le<std::uint32_t>(e.t.T);
    w.put(e.t.lengths.data(), kSyms);
    w.le<std::uint64_t>(e.t.encoded.size());
    w.put(e.t.encoded.data(), e.t.encoded.size());
    w.le<std::uint64_t>(e.t.gaps.size());
    w.put(e.t.gaps.data(), e.t.gaps.size());
    for (std::uint64_t o : e.t.outpos) w.le<std::uint64_t>(o);
    w.le<std::uint64_t>(e.t.raw.size());
    w.put(e.t.raw.data(), e.t.raw.size());
  }
  return std::move(w.bytes);
}

// Validation order and messages follow parse_container (container.cpp:182-250).
std::vector<Entry> parse(std::span<const std::uint8_t> bytes) {
  Cursor r(bytes);
  if (std::memcmp(r.take(4).data(), kMagic, 4) != 0) throw FormatError("bad magic");
  if (r.le<std::uint32_t>() != kVersion) throw FormatError("unsupported version");
  const std::uint32_t count = r.le<std::uint32_t>();
  std::vector<Entry> out;
  for (std::uint32_t i = 0; i < count; ++i) {
    Entry e;
    const std::uint16_t nl = r.le<std::uint16_t>();
    const auto name = r.take(nl);
    e.shape.name.assign(name.begin(), name.end());
    const std::uint8_t rank = r.le<std::uint8_t>();
    std::uint64_t prod = 1;
    for (int k = 0; k < rank; ++k) {
      e.shape.dims.push_back(r.le<std::uint64_t>());
      prod *= e.shape.dims.back();
    }
    Tensor& t = e.t;
    t.n_elem = r.le<std::uint64_t>();
    if (t.n_elem != prod) throw FormatError("element count does not match dims");
    t.T = r.le<std::uint32_t>();
    if (t.T < 1 || t.T > 1024 || (t.T & (t.T - 1))) throw FormatError("invalid thread count");
    const auto len = r.take(kSyms);
    std::copy(len.begin(), len.end(), t.lengths.begin());
    std::uint64_t kraft = 0;
    bool any = false;
    for (std::uint8_t l : t.lengths) {
      if (l > kMaxLen) throw FormatError("invalid length vector in container");
      if (l) kraft += std::uint64_t{1} << (kMaxLen - l), any = true;
    }
    if (kraft > (std::uint64_t{1} << kMaxLen) || (t.n_elem > 0 && !any))
      throw FormatError("invalid length vector in container");
    const std::uint64_t el = r.le<std::uint64_t>();
    const std::uint64_t bb = std::uint64_t{8} * t.T;
    if (el < 2 || (el - 2) % bb != 0) throw FormatError("encoded section length mismatch");
    const std::uint64_t nb = (el - 2) / bb;
    if (t.n_elem > 0 && nb == 0) throw FormatError("encoded section length mismatch");
    const auto enc = r.take(el);
    t.encoded.assign(enc.begin(), enc.end());
    const std::uint64_t gl = r.le<std::uint64_t>();
    if (gl != (nb * t.T + 1) / 2) throw FormatError("gap section length mismatch");
    const auto g = r.take(gl);
    t.gaps.assign(g.begin(), g.end());
    t.outpos.resize(nb + 1);
    for (auto& o : t.outpos) o = r.le<std::uint64_t>();
    if (t.outpos[0] != 0 || t.outpos[nb] != t.n_elem) throw FormatError("block offsets do not cover the tensor");
    for (std::uint64_t b = 0; b < nb; ++b)
      if (t.outpos[b + 1] < t.outpos[b] || t.outpos[b + 1] - t.outpos[b] > std::uint64_t{64} * t.T)
        throw FormatError("block offsets out of range");
    const std::uint64_t rl = r.le<std::uint64_t>();
    if (rl != raw_len(t.n_elem)) throw FormatError("raw section length mismatch");
    const auto rw = r.take(rl);
    t.raw.assign(rw.begin(), rw.end());
    out.push_back(std::move(e));
  }
  r.finish();
  return out;
}

}  // namespace ecf8::e5

// ---- C ABI (host part)

struct ecf8_e5_host_tensor {
  ecf8::e5::Tensor t;
};
struct ecf8_e5_host_file {
  std::vector<ecf8::e5::Entry> entries;
};

namespace {
struct Status {  // a C-ABI status whose message is already set
  int rc;
};
template <class F>
int guarded5(F&& f) {
  try {
    f();
    return ECF8_OK;
  } catch (const Status& s) {
    return s.rc;
  } catch (const ecf8::FormatError& e) {
    return ecf8_internal_set_error(ECF8_EFORMAT, e.what());
  } catch (const ecf8::IoError& e) {
    return ecf8_internal_set_error(ECF8_EIO, e.what());
  } catch (const std::invalid_argument& e) {
    return ecf8_internal_set_error(ECF8_EINVAL, e.what());
  } catch (const std::bad_alloc&) {
    return ecf8_internal_set_error(ECF8_ENOMEM, "out of host memory");
  } catch (const std::exception& e) {
    return ecf8_internal_set_error(ECF8_EINVAL, e.what());
  }
}

std::uint8_t* copy_out(const std::vector<std::uint8_t>& v) {
  auto* p = static_cast<std::uint8_t*>(std::malloc(v.size() ? v.size() : 1));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), v.size());
  return p;
}
}  // namespace

extern "C" {

int ecf8_e5_build_code(const uint64_t counts[32], uint8_t lengths[32]) {
  return guarded5([&] {
    if (!counts || !lengths) throw std::invalid_argument("null argument");
    std::array<std::uint64_t, 32> c{};
    std::copy(counts, counts + 32, c.begin());
    const auto code = ecf8::e5::build_code(c);
    std::copy(code.lengths.begin(), code.lengths.end(), lengths);
  });
}

int ecf8_e5_encode(const uint8_t* e5m2, uint64_t n, uint32_t T, ecf8_e5_host_tensor** out) {
  return guarded5([&] {
    if (!out || (n && !e5m2)) throw std::invalid_argument("null argument");
    auto h = std::make_unique<ecf8_e5_host_tensor>();
    h->t = ecf8::e5::encode({e5m2, static_cast<std::size_t>(n)}, T);
    *out = h.release();
  });
}

int ecf8_e5_tensor_sections(const ecf8_e5_host_tensor* t, ecf8_e5_sections* out) {
  return guarded5([&] {
    if (!t || !out) throw std::invalid_argument("null argument");
    *out = ecf8::e5::sections_of(t->t);
  });
}

void ecf8_e5_tensor_free(ecf8_e5_host_tensor* t) { delete t; }

int ecf8_e5_compress_raw(const uint8_t* raw_file, size_t len, uint32_t T, uint8_t** out, size_t* out_len) {
  return guarded5([&] {
    if (!raw_file || !out || !out_len) throw std::invalid_argument("null argument");
    const ecf8::RawTensorFile rf = ecf8::parse_raw({raw_file, len});
    std::vector<ecf8::e5::Entry> es(rf.tensors.size());
#pragma omp parallel for schedule(dynamic, 1)
    for (std::size_t i = 0; i < rf.tensors.size(); ++i) {
      es[i].shape = rf.tensors[i].shape;
      es[i].t = ecf8::e5::encode(rf.tensors[i].data, T);
    }
    const std::vector<std::uint8_t> bytes = ecf8::e5::serialize(es);
    *out = copy_out(bytes);
    *out_len = bytes.size();
  });
}

int ecf8_e5_parse(const uint8_t* bytes, size_t len, ecf8_e5_host_file** out) {
  return guarded5([&] {
    if (!bytes || !out) throw std::invalid_argument("null argument");
    auto f = std::make_unique<ecf8_e5_host_file>();
    f->entries = ecf8::e5::parse({bytes, len});
    *out = f.release();
  });
}

int ecf8_e5_file_count(const ecf8_e5_host_file* f) { return f ? static_cast<int>(f->entries.size()) : -1; }

int ecf8_e5_file_tensor(const ecf8_e5_host_file* f, int i, ecf8_e5_sections* out, const char** name) {
  return guarded5([&] {
    if (!f || !out || i < 0 || static_cast<std::size_t>(i) >= f->entries.size())
      throw std::invalid_argument("tensor index out of range");
    *out = ecf8::e5::sections_of(f->entries[i].t);
    if (name) *name = f->entries[i].shape.name.c_str();
  });
}

int ecf8_e5_file_shape(const ecf8_e5_host_file* f, int i, uint64_t* dims, int max_rank, int* rank) {
  return guarded5([&] {
    if (!f || !rank || i < 0 || static_cast<std::size_t>(i) >= f->entries.size())
      throw std::invalid_argument("tensor index out of range");
    const auto& d = f->entries[i].shape.dims;
    *rank = static_cast<int>(d.size());
    for (int k = 0; k < std::min<int>(max_rank, *rank); ++k) dims[k] = d[k];
  });
}

void ecf8_e5_file_free(ecf8_e5_host_file* f) { delete f; }

int ecf8_e5_decompress(const uint8_t* bytes, size_t len, uint8_t** out, size_t* out_len) {
  return guarded5([&] {
    if (!bytes || !out || !out_len) throw std::invalid_argument("null argument");
    const auto es = ecf8::e5::parse({bytes, len});
    std::vector<std::uint8_t> raw;
    auto le = [&](std::uint64_t v, int width) {
      for (int k = 0; k < width; ++k) raw.push_back(static_cast<std::uint8_t>(v >> (8 * k)));
    };
    raw.insert(raw.end(), {'F', 'P', '8', 'R'});
    le(1, 4);
    le(es.size(), 4);
    std::vector<std::uint8_t> buf;
    for (const auto& e : es) {
      le(e.shape.name.size(), 2);
      raw.insert(raw.end(), e.shape.name.begin(), e.shape.name.end());
      raw.push_back(static_cast<std::uint8_t>(e.shape.dims.size()));
      for (std::uint64_t d : e.shape.dims) le(d, 8);
      if (e.t.n_elem) {
        buf.resize(e.t.n_elem);
        const ecf8_e5_sections s = ecf8::e5::sections_of(e.t);
        const int rc = ecf8_e5_decode_host(&s, buf.data(), buf.size());
        if (rc != ECF8_OK) throw Status{rc};
        raw.insert(raw.end(), buf.begin(), buf.end());
      }
    }
    *out = copy_out(raw);
    *out_len = raw.size();
  });
}

}  // extern "C"
