// Shared helpers for the SLIDE B200 library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <stdexcept>

namespace slide {

// Error carried across the C-ABI: every extern "C" entry point catches these
// and turns them into a status code plus slide_last_error() text.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

enum Status : int {
  kOk = 0,
  kValueError = 1,   // maps to Python ValueError
  kIndexError = 2,   // maps to Python IndexError
  kCudaError = 3,    // maps to Python RuntimeError
  kNotSupported = 4, // maps to Python NotImplementedError
  kInternal = 5,
};

#define SLIDE_CUDA(expr)                                                              \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      throw ::slide::Error(::slide::kCudaError, std::string(#expr) + " (" + __FILE__ + ":" +   \
                                                    std::to_string(__LINE__) + "): " +               \
                                                    cudaGetErrorString(_e));         \
  } while (0)

#define SLIDE_CHECK(cond, code, msg)                          \
  do {                                                        \
    if (!(cond)) throw ::slide::Error((code), (msg));         \
  } while (0)

// every hand-written kernel launch goes through this check; it also counts
// the launches (slide_launch_count) so the bench can report its kernels
extern unsigned long long g_slide_launches;
#define SLIDE_LAUNCH_CHECK()            \
  do {                                  \
    ++::slide::g_slide_launches;        \
    SLIDE_CUDA(cudaGetLastError());     \
  } while (0)

constexpr int kSms = 148;  // B200

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace slide
