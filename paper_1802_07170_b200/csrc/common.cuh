// Common definitions for the CytonMT B200 engine (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <stdexcept>

#define CMT_HD __host__ __device__ __forceinline__
#define CMT_D __device__ __forceinline__

namespace cmt {

typedef __nv_bfloat16 bf16;

// Error carried from the engine to the C-ABI boundary.
struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

enum Status {
  CMT_OK = 0,
  CMT_ERR_CONFIG = 1,     // ConfigError (bad token id, bad config)
  CMT_ERR_MASK = 2,       // MaskError (fully masked source column)
  CMT_ERR_SHAPE = 3,      // ShapeError
  CMT_ERR_NUM_SCORES = 4, // NumericError: non-finite attention scores (tensor.py:139-140)
  CMT_ERR_NUM_LOGITS = 5, // NumericError: non-finite logits (tensor.py:148-149)
  CMT_ERR_NUM_LOSS = 6,   // NumericError: non-finite loss (training.py:154-155)
  CMT_ERR_NUM_NORM = 7,   // NumericError: non-finite grad norm (training.py:133-134)
  CMT_ERR_CUDA = 8,
  CMT_ERR_INTERNAL = 9,
};

// device status bits (set by kernels, read once per step)
// ST_HANG: a recurrent scan's flag wait exceeded its budget (lstm_common.cuh SpinGuard)
enum StatusBits { ST_SCORES = 1, ST_LOGITS = 2, ST_LOSS = 4, ST_NORM = 8, ST_HANG = 16 };

#define CMT_CUDA(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      throw ::cmt::Error(::cmt::CMT_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + \
                         " at " + __FILE__ + ":" + std::to_string(__LINE__));         \
  } while (0)

// Every kernel launch of the engine goes through this counter so bench.py can
// report how many of OUR kernels ran inside the timed region.
extern unsigned long long g_launches;
#define CMT_LAUNCHED() (++::cmt::g_launches)

template <typename T> CMT_HD float to_f(T v);
template <> CMT_HD float to_f<float>(float v) { return v; }
template <> CMT_HD float to_f<bf16>(bf16 v) { return __bfloat162float(v); }
template <typename T> CMT_HD T from_f(float v);
template <> CMT_HD float from_f<float>(float v) { return v; }
template <> CMT_HD bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

CMT_D float sigmoidf_(float x) {
  // branch-split stable sigmoid (reference tensor.py:165-172)
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  float e = expf(x);
  return e / (1.f + e);
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace cmt
