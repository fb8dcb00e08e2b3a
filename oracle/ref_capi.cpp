// ref_capi.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with /root/reference/proj/src/*.cpp (namespace renamed to
// ecf8_ref via -Decf8=ecf8_ref) into oracle/_ref/libecf8_ref.so.  Python
// tests use it to pin the C oracle and the product encoder against the real
// reference; bench.py --impl reference times ecf8_ref::decode_parallel_into
// through it.  Nothing in the product links it.
#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ecf8/codec.hpp"
#include "ecf8/container.hpp"
#include "ecf8/errors.hpp"
#include "ecf8/huffman.hpp"
#include "ecf8/lut.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ecf8::FormatError& e) {
    g_err = e.what();
    return -3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -4;
  }
}

void give(const std::vector<std::uint8_t>& v, std::uint8_t** out, std::size_t* out_len) {
  *out = static_cast<std::uint8_t*>(std::malloc(v.size() ? v.size() : 1));
  if (!v.empty()) std::memcpy(*out, v.data(), v.size());
  *out_len = v.size();
}

struct RefTensor {
  ecf8::EncodedTensor t;
  ecf8::CascadedLut lut;
};
}  // namespace

extern "C" {

const char* ecf8ref_last_error() { return g_err.c_str(); }
void ecf8ref_free(void* p) { std::free(p); }

int ecf8ref_compress_raw(const std::uint8_t* raw, std::size_t len, std::uint32_t T,
                         std::uint8_t** out, std::size_t* out_len) {
  return guarded([&] {
    const auto f = ecf8::parse_raw({raw, len});
    give(ecf8::serialize(ecf8::compress_tensors(f, T)), out, out_len);
  });
}

int ecf8ref_decompress(const std::uint8_t* c, std::size_t len, std::uint8_t** out,
                       std::size_t* out_len, std::uint64_t* allocations) {
  return guarded([&] {
    const auto f = ecf8::parse_container({c, len});
    std::ostringstream os;
    const auto st = ecf8::decompress_streaming(f, os);
    const std::string s = os.str();
    give(std::vector<std::uint8_t>(s.begin(), s.end()), out, out_len);
    if (allocations) *allocations = st.buffer_allocations;
  });
}

// mode 0: decode_parallel_into, 1: decode_reference
int ecf8ref_decode_tensor(const std::uint8_t* c, std::size_t len, std::uint32_t index, int mode,
                          std::uint8_t* out, std::size_t out_len) {
  return guarded([&] {
    const auto f = ecf8::parse_container({c, len});
    if (index >= f.tensors.size()) throw std::invalid_argument("tensor index out of range");
    const auto& t = f.tensors[index].tensor;
    if (out_len != t.stream.n_elem) throw std::invalid_argument("output size mismatch");
    if (t.stream.n_elem == 0) return;
    const auto lut = ecf8::build_lut(ecf8::canonical_codes(t.stream.lengths));
    if (mode == 0) {
      ecf8::decode_parallel_into(t, lut, {out, out_len});
    } else {
      const auto v = ecf8::decode_reference(t, lut);
      std::memcpy(out, v.data(), v.size());
    }
  });
}

int ecf8ref_synth_raw(double alpha, double gamma, std::uint64_t n, std::uint64_t seed,
                      std::uint8_t* out) {
  return guarded([&] {
    const auto f = ecf8::synth_raw(alpha, gamma, n, seed);
    std::memcpy(out, f.tensors[0].data.data(), n);
  });
}

int ecf8ref_build_code(const std::uint64_t counts[16], std::uint8_t lengths[16]) {
  return guarded([&] {
    ecf8::ExponentHistogram h;
    for (int i = 0; i < 16; ++i) h.counts[i] = counts[i];
    const auto t = ecf8::build_code(h);
    for (int i = 0; i < 16; ++i) lengths[i] = t.lengths[i];
  });
}

int ecf8ref_build_lut(const std::uint8_t lengths[16], std::uint8_t* entries,
                      std::uint32_t* n_luts) {
  return guarded([&] {
    std::array<std::uint8_t, 16> l{};
    for (int i = 0; i < 16; ++i) l[i] = lengths[i];
    const auto lut = ecf8::build_lut(ecf8::canonical_codes(l));
    std::memcpy(entries, lut.entries.data(), lut.entries.size());
    *n_luts = lut.n_luts;
  });
}

int ecf8ref_count_phase(const std::uint8_t w10[10], unsigned gap, const std::uint8_t lengths[16],
                        std::uint32_t* count) {
  return guarded([&] {
    std::array<std::uint8_t, 16> l{};
    for (int i = 0; i < 16; ++i) l[i] = lengths[i];
    const auto lut = ecf8::build_lut(ecf8::canonical_codes(l));
    *count = ecf8::count_phase(std::span<const std::uint8_t, 10>(w10, 10), gap, lut);
  });
}

// A parsed tensor kept across timed calls (bench reference arm).
void* ecf8ref_tensor_new(std::uint64_t n_elem, std::uint32_t T, const std::uint8_t lengths[16],
                         const std::uint8_t* encoded, std::uint64_t encoded_len,
                         const std::uint8_t* gaps, std::uint64_t gaps_len,
                         const std::uint64_t* outpos, std::uint64_t n_outpos,
                         const std::uint8_t* packed, std::uint64_t packed_len) {
  RefTensor* r = nullptr;
  const int rc = guarded([&] {
    auto* x = new RefTensor;
    auto& s = x->t.stream;
    s.n_elem = n_elem;
    s.geometry.threads_per_block = T;
    s.geometry.n_blocks = n_outpos - 1;
    for (int i = 0; i < 16; ++i) s.lengths[i] = lengths[i];
    s.encoded.assign(encoded, encoded + encoded_len);
    s.gaps.assign(gaps, gaps + gaps_len);
    s.outpos.assign(outpos, outpos + n_outpos);
    x->t.packed.assign(packed, packed + packed_len);
    if (n_elem) x->lut = ecf8::build_lut(ecf8::canonical_codes(s.lengths));
    r = x;
  });
  return rc == 0 ? r : nullptr;
}

void ecf8ref_tensor_free(void* h) { delete static_cast<RefTensor*>(h); }

// Every tensor of a container parsed once by the reference's parse_container
// (container.cpp:182-250), each with its LUT built (the per-tensor work of
// decompress_streaming, container.cpp:334-339), as handles for
// ecf8ref_tensor_decode.  The bench reference arm builds its inputs with
// ecf8ref_synth_raw + ecf8ref_compress_raw and this, never with the product.
int ecf8ref_container_tensors(const std::uint8_t* c, std::size_t len, void** handles,
                              std::uint32_t cap, std::uint32_t* count) {
  return guarded([&] {
    auto f = ecf8::parse_container({c, len});
    if (f.tensors.size() > cap) throw std::invalid_argument("too many tensors for the handle array");
    *count = static_cast<std::uint32_t>(f.tensors.size());
    for (std::size_t i = 0; i < f.tensors.size(); ++i) {
      auto* x = new RefTensor;
      x->t = std::move(f.tensors[i].tensor);
      if (x->t.stream.n_elem) x->lut = ecf8::build_lut(ecf8::canonical_codes(x->t.stream.lengths));
      handles[i] = x;
    }
  });
}

std::uint64_t ecf8ref_tensor_n_elem(void* h) { return static_cast<RefTensor*>(h)->t.stream.n_elem; }

// Algorithmic bytes of one decode: container sections read
// (encoded + gaps + 8 (n_blocks + 1) + packed) + n_elem FP8 bytes written.
std::uint64_t ecf8ref_tensor_algorithmic_bytes(void* h) {
  const auto& t = static_cast<RefTensor*>(h)->t;
  return t.stream.encoded.size() + t.stream.gaps.size() + 8 * t.stream.outpos.size() + t.packed.size() +
         t.stream.n_elem;
}

// Decode with `nthreads` OpenMP threads (<= 0: all); returns seconds.
double ecf8ref_tensor_decode(void* h, std::uint8_t* out, int nthreads) {
  auto* r = static_cast<RefTensor*>(h);
  if (nthreads > 0) omp_set_num_threads(nthreads);
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = guarded(
      [&] { ecf8::decode_parallel_into(r->t, r->lut, {out, r->t.stream.n_elem}); });
  const double dt =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return rc == 0 ? dt : -1.0;
}

// The reference's sequential decoder (codec.cpp:125-131) on a kept tensor;
// returns seconds (the returned vector's allocation included: that is the API).
double ecf8ref_tensor_decode_reference(void* h, std::uint8_t* out) {
  auto* r = static_cast<RefTensor*>(h);
  double dt = -1.0;
  guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    const auto v = ecf8::decode_reference(r->t, r->lut);
    dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(out, v.data(), v.size());
  });
  return dt;
}

int ecf8ref_max_threads() { return omp_get_max_threads(); }

}  // extern "C"
