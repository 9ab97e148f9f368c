// spmk/error.hpp — drop-in for /root/reference/proj/include/spmk/error.hpp:10-13.
//
// Same error convention: every contract violation throws spmk::Error (a
// std::runtime_error) carrying the message.  On this device path the message
// comes from the C ABI (spmk_last_error(), include/spmk_capi.h).
#pragma once

#include <stdexcept>
#include <string>

#include "spmk_capi.h"

namespace spmk {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};

namespace detail {

// Map a C-ABI status to the reference's exception type.
inline void check_status(spmk_status st, const char* where) {
  if (st == SPMK_OK) return;
  std::string msg = spmk_last_error();
  if (msg.empty()) msg = "spmk status " + std::to_string((int)st);
  throw Error(std::string(where) + ": " + msg);
}

}  // namespace detail
}  // namespace spmk
