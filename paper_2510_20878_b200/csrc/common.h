// Shared host-side helpers of libharag: status exceptions and CUDA checks.
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "harag.h"

namespace harag {

// Internal error carrying an hr_status; converted to a return code at the ABI.
struct Error : std::runtime_error {
  hr_status code;
  Error(hr_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(hr_status c, const std::string& m) { throw Error(c, m); }

inline void require(bool ok, hr_status c, const std::string& m) {
  if (!ok) fail(c, m);
}
// literal messages bind here: no std::string is built unless the check fails (hr_assemble_kv runs a few
// dozen checks per call)
inline void require(bool ok, hr_status c, const char* m) {
  if (!ok) fail(c, m);
}

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

}  // namespace harag

#define HR_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      ::harag::fail(HR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));         \
  } while (0)
