// Shared host-side plumbing: error type mirroring semrank::Error
// (include/semrank/error.hpp:13-42) and the C-ABI status bridge.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "semrank_b200.h"

namespace srh {

// Thrown inside the library; converted to an sr_status at the C boundary.
class Error : public std::runtime_error {
 public:
  Error(sr_status code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
  sr_status code() const { return code_; }

 private:
  sr_status code_;
};

[[noreturn]] inline void fail(sr_status code, const std::string& msg) { throw Error(code, msg); }

void set_last_error(const std::string& msg);

// Runs f(); maps exceptions to status codes and records the message.
template <typename F>
int32_t guard(F&& f) {
  try {
    f();
    set_last_error("");
    return SR_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code();
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return SR_CUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SR_SPEC_VIOLATION;
  }
}

}  // namespace srh

#define SR_CUDA_CHECK(expr)                                                               \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      cudaGetLastError(); /* a non-sticky error must not fail the next launch check */    \
      ::srh::fail(SR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e) + " at " + \
                               __FILE__ + ":" + std::to_string(__LINE__));                \
    }                                                                                     \
  } while (0)
