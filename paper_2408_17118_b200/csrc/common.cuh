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

// Candidate generator (reading A7): coordinate n of the N(0,1) vector of component
// i (1-based), global candidate id l: counter c = ((i 2^24 + l) 2^9 + n/2) 2 + h, SplitMix64
// finaliser (Steele, Lea, Flood 2014) of seed + (c+1) phi64, u = ((z >> 11) + 1/2) 2^-53,
// Box-Muller in fp64 (even n: cos, odd n: sin).
__device__ __forceinline__ uint64_t splitmix64_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform01(uint64_t seed, uint64_t c) {
  uint64_t z = splitmix64_mix(seed + (c + 1ull) * 0x9E3779B97F4A7C15ull);
  return ((double)(z >> 11) + 0.5) * 0x1.0p-53;
}
__device__ __forceinline__ double candidate_normal(uint64_t seed, int i, uint64_t l, int n) {
  uint64_t p = (uint64_t)(n >> 1);
  uint64_t c0 = ((((uint64_t)i << 24) + l) * 512ull + p) * 2ull;
  double u0 = uniform01(seed, c0), u1 = uniform01(seed, c0 + 1ull);
  double rad = sqrt(-2.0 * log(u0));
  double ang = 2.0 * 3.141592653589793 * u1;
  return (n & 1) ? rad * sin(ang) : rad * cos(ang);
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Split-slot parts (DESIGN.md §5 "few active rows"): when the active row tiles x slots cannot
// fill the GPU, the chunks of every slot are divided among P CTAs, each with its own fp32 partial
// (summed in fp64, slot-major).  P depends only on the GLOBAL active count and the slot count, so
// a row's arithmetic is the same for any GPU count.
constexpr int kSplitTarget = 296;   // work units wanted per launch (2 per SM)
constexpr int kSplitMax = 8;
__host__ __device__ inline int split_parts(int L_global, int S) {
  const int64_t tiles = round_up(ceil_div(L_global > 0 ? L_global : 1, 128), 2);
  const int64_t P = kSplitTarget / (tiles * (int64_t)(S > 0 ? S : 1));
  return (int)(P < 1 ? 1 : (P > kSplitMax ? kSplitMax : P));
}

// Upsilon of eq. (1), natural log (A14); -inf outside the domain (A13).
__host__ __device__ inline double upsilon_of(double a) {
  return a > kAlphaFloor ? a - 2.0 * log(a * 0.5 + 1.0) : -INFINITY;
}

}  // namespace oica
