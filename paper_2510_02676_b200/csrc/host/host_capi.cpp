// host_capi.cpp -- implementation of include/ecf8_host.h.
#include <omp.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <numbers>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>

#include "../cuda/tables.hpp"
#include "ecf8/container.hpp"
#include "ecf8_host.h"
#include "host_util.hpp"

struct ecf8_host_tensor {
  ecf8::EncodedTensor t;
};
struct ecf8_host_file {
  ecf8::Ecf8File f;
};

// The C ABI's thread-local message lives in capi.cu.
extern "C" int ecf8_internal_set_error(int status, const char* msg);

namespace {

int set_error(int st, const char* msg) { return ecf8_internal_set_error(st, msg); }

template <class F>
int guarded(F&& f) {
  try {
    f();
    return ECF8_OK;
  } catch (const ecf8::FormatError& e) {
    return set_error(ECF8_EFORMAT, e.what());
  } catch (const ecf8::IoError& e) {
    return set_error(ECF8_EIO, e.what());
  } catch (const std::invalid_argument& e) {
    return set_error(ECF8_EINVAL, e.what());
  } catch (const std::bad_alloc&) {
    return set_error(ECF8_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return set_error(ECF8_ECUDA, e.what());
  }
}

void give(const void* p, std::size_t n, std::uint8_t** out, std::size_t* out_len) {
  *out = static_cast<std::uint8_t*>(std::malloc(n ? n : 1));
  if (!*out) throw std::bad_alloc();
  if (n) std::memcpy(*out, p, n);
  *out_len = n;
}

std::array<std::uint8_t, 16> arr16(const std::uint8_t* l) {
  std::array<std::uint8_t, 16> a{};
  std::memcpy(a.data(), l, 16);
  return a;
}

ecf8::EncodedTensor from_sections(const ecf8_sections* s) {
  ecf8::EncodedTensor t;
  auto& st = t.stream;
  st.n_elem = s->n_elem;
  st.geometry.threads_per_block = s->threads_per_block;
  st.geometry.n_blocks = s->n_outpos ? s->n_outpos - 1 : 0;
  st.lengths = arr16(s->lengths);
  st.encoded.assign(s->encoded, s->encoded + s->encoded_len);
  st.gaps.assign(s->gaps, s->gaps + s->gaps_len);
  st.outpos.assign(s->outpos, s->outpos + s->n_outpos);
  t.packed.assign(s->packed, s->packed + s->packed_len);
  return t;
}

}  // namespace

extern "C" {

void ecf8_host_free(void* p) { std::free(p); }

int ecf8_host_max_threads(void) { return omp_get_max_threads(); }

int ecf8_host_make_stats(const uint8_t* fp8, uint64_t n, uint32_t T, uint32_t name_len, uint32_t rank,
                         ecf8_entropy_report* out) {
  return guarded([&] {
    if (!out || (n && !fp8) || rank == 0) throw std::invalid_argument("invalid argument");
    ecf8::RawTensorFile raw;
    ecf8::RawTensor rt;
    rt.shape.name.assign(name_len, 't');
    rt.shape.dims.assign(rank, 1);
    rt.shape.dims[0] = n;
    rt.data.assign(fp8, fp8 + n);
    raw.tensors.push_back(std::move(rt));
    const ecf8::EntropyReport r = ecf8::make_stats(raw, T).at(0);
    *out = ecf8_entropy_report{r.n_elem,      r.entropy_bits, r.bits_per_symbol,   r.bits_per_weight,
                               r.bound_lower, r.bound_upper,  r.projected_savings, r.actual_savings};
  });
}

int ecf8_host_build_code(const uint64_t counts[16], uint8_t lengths[16]) {
  return guarded([&] {
    ecf8::ExponentHistogram h;
    for (int s = 0; s < 16; ++s) h.counts[s] = counts[s];
    const ecf8::CodeTable t = ecf8::build_code(h);
    std::memcpy(lengths, t.lengths.data(), 16);
  });
}

int ecf8_host_build_lut(const uint8_t lengths[16], uint8_t* entries, uint32_t* n_luts) {
  return guarded([&] {
    const ecf8::CascadedLut lut = ecf8::build_lut(ecf8::canonical_codes(arr16(lengths)));
    std::memcpy(entries, lut.entries.data(), lut.entries.size());
    *n_luts = lut.n_luts;
  });
}

int ecf8_host_device_tables(const uint8_t lengths[16], uint32_t* fast, uint16_t* smask,
                            uint8_t* cascade, uint32_t* n_luts, uint32_t* fast_bits) {
  return guarded([&] {
    const ecf8::dev::DecodeTables t = ecf8::dev::build_tables(lengths);
    std::memcpy(fast, t.fast.data(), t.fast.size() * 4);
    std::memcpy(smask, t.smask.data(), t.smask.size() * 2);
    std::memcpy(cascade, t.cascade.data(), t.cascade.size());
    *n_luts = t.n_luts;
    *fast_bits = ecf8::dev::kFastBits;
  });
}

int ecf8_host_fsm_tables(const uint8_t lengths[16], uint32_t* fsm, uint8_t* cm, int* ok) {
  return guarded([&] {
    const ecf8::dev::DecodeTables t = ecf8::dev::build_tables(lengths);
    std::memcpy(fsm, t.fsm.data(), t.fsm.size() * 4);
    std::memcpy(cm, t.fsm_cm.data(), t.fsm_cm.size());
    *ok = t.fsm_ok ? 1 : 0;
  });
}

int ecf8_host_encode(const uint8_t* fp8, uint64_t n, uint32_t T, const uint8_t* lengths,
                     ecf8_host_tensor** out) {
  return guarded([&] {
    *out = nullptr;
    auto h = std::make_unique<ecf8_host_tensor>();
    const std::span<const std::uint8_t> data(fp8, n);
    if (lengths) {
      h->t = ecf8::encode_tensor(data, ecf8::canonical_codes(arr16(lengths)), T);
    } else if (n == 0) {
      h->t.stream.geometry = ecf8::make_geometry(0, T);
      h->t.stream.encoded.assign(2, 0);
      h->t.stream.outpos.assign(1, 0);
    } else {
      h->t = ecf8::encode_tensor(data, ecf8::build_code(ecf8::ExponentHistogram::of_bytes(data)), T);
    }
    *out = h.release();
  });
}

int ecf8_host_encode_many(const uint8_t* const* fp8, const uint64_t* n, int count, uint32_t T,
                          ecf8_host_tensor** out, int nthreads) {
  for (int i = 0; i < count; ++i) out[i] = nullptr;
  int status = ECF8_OK;
  std::string msg;
#pragma omp parallel for schedule(dynamic) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())
  for (int i = 0; i < count; ++i) {
    const int rc = ecf8_host_encode(fp8[i], n[i], T, nullptr, &out[i]);
    if (rc != ECF8_OK) {
#pragma omp critical
      if (status == ECF8_OK) {
        status = rc;
        msg = ecf8_last_error();
      }
    }
  }
  if (status != ECF8_OK) {
    for (int i = 0; i < count; ++i) {
      delete out[i];
      out[i] = nullptr;
    }
    return set_error(status, msg.c_str());
  }
  return ECF8_OK;
}

int ecf8_host_tensor_sections(const ecf8_host_tensor* t, ecf8_sections* out) {
  if (!t || !out) return set_error(ECF8_EINVAL, "null argument");
  *out = ecf8::host::sections_of(t->t);
  return ECF8_OK;
}

void ecf8_host_tensor_free(ecf8_host_tensor* t) { delete t; }

int ecf8_host_decode_reference(const ecf8_sections* s, uint8_t* out, uint64_t out_len) {
  return guarded([&] {
    if (out_len != s->n_elem) throw std::invalid_argument("output size mismatch");
    if (s->n_elem == 0) return;
    const ecf8::EncodedTensor t = from_sections(s);
    const auto v = ecf8::decode_reference(t, ecf8::build_lut(ecf8::canonical_codes(t.stream.lengths)));
    std::memcpy(out, v.data(), v.size());
  });
}

int ecf8_host_compress_raw(const uint8_t* raw, size_t len, uint32_t T, uint8_t** out, size_t* out_len) {
  return guarded([&] {
    const auto bytes = ecf8::serialize(ecf8::compress_tensors(ecf8::parse_raw({raw, len}), T));
    give(bytes.data(), bytes.size(), out, out_len);
  });
}

int ecf8_host_parse(const uint8_t* bytes, size_t len, ecf8_host_file** out) {
  return guarded([&] {
    *out = nullptr;
    auto f = std::make_unique<ecf8_host_file>();
    f->f = ecf8::parse_container({bytes, len});
    *out = f.release();
  });
}

int ecf8_host_file_count(const ecf8_host_file* f) { return f ? static_cast<int>(f->f.tensors.size()) : 0; }

int ecf8_host_file_tensor(const ecf8_host_file* f, int i, ecf8_sections* out, const char** name) {
  if (!f || i < 0 || static_cast<std::size_t>(i) >= f->f.tensors.size())
    return set_error(ECF8_EINVAL, "tensor index out of range");
  *out = ecf8::host::sections_of(f->f.tensors[i].tensor);
  if (name) *name = f->f.tensors[i].shape.name.c_str();
  return ECF8_OK;
}

int ecf8_host_file_shape(const ecf8_host_file* f, int i, uint64_t* dims, int max_rank, int* rank) {
  if (!f || i < 0 || static_cast<std::size_t>(i) >= f->f.tensors.size() || !rank)
    return set_error(ECF8_EINVAL, "tensor index out of range");
  const auto& d = f->f.tensors[i].shape.dims;
  *rank = static_cast<int>(d.size());
  for (int j = 0; j < *rank && j < max_rank; ++j) dims[j] = d[j];
  return ECF8_OK;
}

void ecf8_host_file_free(ecf8_host_file* f) { delete f; }

int ecf8_host_decompress(const uint8_t* bytes, size_t len, uint8_t** out, size_t* out_len,
                         uint64_t* allocations, uint64_t* capacity) {
  return guarded([&] {
    std::ostringstream os;
    const ecf8::DecompressStats st = ecf8::host::decompress_bytes({bytes, len}, os);
    const std::string s = os.str();
    give(s.data(), s.size(), out, out_len);
    if (allocations) *allocations = st.buffer_allocations;
    if (capacity) *capacity = st.buffer_capacity_bytes;
  });
}

int ecf8_host_fused_layout(const uint8_t* w, uint64_t n, uint64_t k, uint8_t* out, int inverse) {
  return guarded([&] {
    if (!w || !out) throw std::invalid_argument("null argument");
    if (n % 128 || k % 128) throw std::invalid_argument("fused layout needs n, k multiples of 128");
    const std::uint64_t KT = k / 128, NT = n / 128;
#pragma omp parallel for schedule(static)
    for (std::int64_t t = 0; t < static_cast<std::int64_t>(NT * KT); ++t) {
      const std::uint64_t nt = static_cast<std::uint64_t>(t) / KT, kt = static_cast<std::uint64_t>(t) % KT;
      std::uint8_t* tile = out + static_cast<std::uint64_t>(t) * 16384;
      const std::uint8_t* itile = w + static_cast<std::uint64_t>(t) * 16384;
      for (std::uint64_t r = 0; r < 128; ++r) {
        const std::uint64_t row = (nt * 128 + r) * k + kt * 128;
        for (std::uint64_t c = 0; c < 8; ++c) {  // 16-byte chunks, 128B swizzle
          const std::uint64_t img = r * 128 + ((c ^ (r & 7)) << 4);
          if (inverse)
            std::memcpy(out + row + 16 * c, itile + img, 16);
          else
            std::memcpy(tile + img, w + row + 16 * c, 16);
        }
      }
    }
  });
}

namespace {
// std::streambuf forwarding to an ecf8_write_fn (decompress_streaming's ostream)
class SinkBuf : public std::streambuf {
 public:
  SinkBuf(ecf8_write_fn w, void* ctx) : w_(w), ctx_(ctx) {}
  int status() const { return rc_; }

 protected:
  std::streamsize xsputn(const char* s, std::streamsize n) override {
    if (rc_ == 0 && n > 0) rc_ = w_(ctx_, reinterpret_cast<const uint8_t*>(s), static_cast<size_t>(n));
    return rc_ == 0 ? n : 0;
  }
  int_type overflow(int_type c) override {
    if (c == traits_type::eof()) return traits_type::not_eof(c);
    const char ch = static_cast<char>(c);
    return xsputn(&ch, 1) == 1 ? c : traits_type::eof();
  }

 private:
  ecf8_write_fn w_;
  void* ctx_;
  int rc_ = 0;
};
}  // namespace

int ecf8_host_decompress_to(const uint8_t* bytes, size_t len, ecf8_write_fn write, void* ctx, uint64_t* allocations,
                            uint64_t* capacity) {
  if (!write) return set_error(ECF8_EINVAL, "null sink");
  SinkBuf buf(write, ctx);
  int rc = guarded([&] {
    std::ostream os(&buf);
    const ecf8::DecompressStats st = ecf8::host::decompress_bytes({bytes, len}, os);
    if (allocations) *allocations = st.buffer_allocations;
    if (capacity) *capacity = st.buffer_capacity_bytes;
  });
  // a failed sink makes the stream throw IoError("write failed"): report the sink
  if (buf.status() != 0) return set_error(ECF8_EIO, "sink write failed");
  return rc;
}

int ecf8_host_synth(double alpha, double gamma, uint64_t n, uint64_t seed, int fmt, uint8_t* out,
                    int nthreads) {
  return guarded([&] {
    if (!(alpha > 0.0 && alpha <= 2.0)) throw std::invalid_argument("alpha must be in (0, 2]");
    if (!(gamma > 0.0)) throw std::invalid_argument("gamma must be positive");
    if (fmt != 0 && fmt != 1) throw std::invalid_argument("fmt must be 0 (E4M3) or 1 (E5M2)");
    const int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
    const double ia = 1.0 / alpha;
    // Same arithmetic as sample_stable(): draw i consumes SplitMix64 calls
    // 2i and 2i+1, so chunks start from jump(2 * first).
#pragma omp parallel num_threads(nt)
    {
      const int k = omp_get_thread_num(), nk = omp_get_num_threads();
      const std::uint64_t lo = n * k / nk, hi = n * (k + 1) / nk;
      ecf8::SplitMix64 rng(seed);
      rng.jump(2 * lo);
      for (std::uint64_t i = lo; i < hi; ++i) {
        const double v = std::numbers::pi * (rng.next_unit() - 0.5);
        const double w = -std::log(rng.next_unit());
        double x;
        if (alpha == 1.0)
          x = std::tan(v);
        else
          x = std::sin(alpha * v) / std::pow(std::cos(v), ia) *
              std::pow(std::cos((1.0 - alpha) * v) / w, (1.0 - alpha) * ia);
        const double y = gamma * x;
        out[i] = fmt == 0 ? ecf8::e4m3_from_double(y) : ecf8::e5m2_from_double(y);
      }
    }
  });
}

}  // extern "C"
