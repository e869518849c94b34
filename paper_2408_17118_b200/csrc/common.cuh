// Internal helpers shared by the liboica kernels and host runtime (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/oica.h"

namespace oica {

// Internal error carrying an ABI status; converted at the extern "C" boundary.
struct Error : std::runtime_error {
  oica_status status;
  Error(oica_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define OICA_CUDA(call)                                                                    \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      throw ::oica::Error(e_ == cudaErrorMemoryAllocation ? OICA_ERR_OUT_OF_MEMORY          \
                                                          : OICA_ERR_CUDA,                 \
                          std::string(#call) + ": " + cudaGetErrorString(e_));             \
  } while (0)

#define OICA_REQUIRE(cond, status, msg)                \
  do {                                                 \
    if (!(cond)) throw ::oica::Error((status), (msg)); \
  } while (0)

// Candidate state codes (per candidate, this rank).
enum : uint8_t { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_DEGENERATE = 2 };

constexpr double kDegenerateNorm = 1e-12;   // A18
constexpr double kClusterDelta = 1e-6;      // A6
constexpr double kNearTieRel = 1e-6;        // A6
constexpr double kAlphaFloor = -2.0 + 1e-12;  // A13
constexpr int kMaxClusters = 8;             // refined clusters per component

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Upsilon of eq. (1), natural log (A14); -inf outside the domain (A13).
__host__ __device__ inline double upsilon_of(double a) {
  return a > kAlphaFloor ? a - 2.0 * log(a * 0.5 + 1.0) : -INFINITY;
}

}  // namespace oica
