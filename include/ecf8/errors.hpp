// ecf8/errors.hpp -- exception types of the ECF8 host API (B200 build).
//
// Same two categories as /root/reference/proj/include/ecf8/errors.hpp so
// callers keep their catch clauses and CLI exit-code mapping:
//   FormatError  malformed / inconsistent serialized data   (exit 2)
//   IoError      open / read / write failures               (exit 3)
// The C ABI (include/ecf8_cuda.h) reports these as ECF8_EFORMAT / ECF8_EIO
// status codes; the C++ layer rethrows them with the original message.
#pragma once

#include <stdexcept>
#include <string>

namespace ecf8 {

struct FormatError : std::runtime_error {
  explicit FormatError(const std::string& msg) : std::runtime_error(msg) {}
};

struct IoError : std::runtime_error {
  explicit IoError(const std::string& msg) : std::runtime_error(msg) {}
};

}  // namespace ecf8
