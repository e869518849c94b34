// §3.3 "Reduction of Signals under Orthonormality Constraints" (Alg. 2
// lines 4-12): the iteration for component i runs on X~ = G X, where the
// d = N-i+1 rows of G are an orthonormal basis of the complement of the accepted rows.
//   K6a k_reduce_apply : X~ = G X (fp32 out, optional fp16 tensor-core plane, zero padded)
//   K6b k_cand_basis   : b0 = G r / ||G r|| for the counter-generated r (A7, A9)
// The basis itself (Householder, fp64) lives on the host (runtime.cu).
#include <cuda_fp16.h>

#include "kernels.cuh"

namespace oica {
namespace {

constexpr int kMaxV = 8;   // 256 / 32 coordinates per lane

// X~[r][m] = sum_n G[r][n] X[n][m].  CTA tile 64 rows x 128 samples, 256 threads, 4 x 8 outputs
// per thread, K (= n) staged through shared memory 32 at a time.  fp32 FMA over N <= 256 terms.
constexpr int RT = 64, MTL = 128, KT = 32;
__global__ void __launch_bounds__(256) k_reduce_apply(const float* __restrict__ Gf, int d, int N,
                                                       const float* __restrict__ X, int64_t ld, int64_t M,
                                                       float* __restrict__ Xr, int64_t ldr, __half* __restrict__ Xh,
                                                       int NPd, int64_t ldx) {
  __shared__ float Gs[KT][RT + 1];
  __shared__ __align__(16) float Xs[KT][MTL];
  const int r0 = blockIdx.y * RT;
  const int64_t m0 = (int64_t)blockIdx.x * MTL;
  const int tr = threadIdx.x / 16, tm = threadIdx.x % 16;   // 16 x 16 threads: rows tr*4.., cols tm*8..
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  for (int n0 = 0; n0 < N; n0 += KT) {
    for (int idx = threadIdx.x; idx < KT * RT; idx += 256) {
      int kk = idx % KT, rr = idx / KT;
      int r = r0 + rr, n = n0 + kk;
      Gs[kk][rr] = (r < d && n < N) ? Gf[(int64_t)r * N + n] : 0.f;
    }
    for (int idx = threadIdx.x; idx < KT * MTL; idx += 256) {
      int kk = idx / MTL, mm = idx % MTL;
      int n = n0 + kk;
      int64_t m = m0 + mm;
      Xs[kk][mm] = (n < N && m < M) ? __ldg(X + (int64_t)n * ld + m) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < KT; ++kk) {
      float g[4], x[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) g[i] = Gs[kk][tr * 4 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = Xs[kk][tm * 8 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(g[i], x[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = r0 + tr * 4 + i;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int64_t m = m0 + tm * 8 + j;
      if (r < d && m < M) Xr[(int64_t)r * ldr + m] = acc[i][j];
      if (Xh && r < NPd && m < ldx)
        Xh[(int64_t)r * ldx + m] = __float2half_rn((r < d && m < M) ? acc[i][j] * kXScale : 0.f);
    }
  }
}

// b0 = G r / ||G r|| with r the counter-generated N(0,1) vector of (seed, i, global id) (A7): the
// reduced-space start of Alg. 2 line 13-15 in the form that reproduces the projection form's
// trajectory (reading A9: G^T G = P, ||G r|| = ||P r||).  One warp per candidate.
__global__ void k_cand_basis(uint64_t seed, int i, int64_t id_base, int64_t L_local, int N,
                             const double* __restrict__ G, int d, double* __restrict__ W64,
                             uint8_t* __restrict__ state, uint8_t* __restrict__ keep, uint8_t* __restrict__ fine,
                             uint8_t fine_init, double* __restrict__ dprev) {
  int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (j >= L_local) return;
  uint64_t l = (uint64_t)(id_base + j);
  double r[kMaxV];
#pragma unroll
  for (int u = 0; u < kMaxV; ++u) {
    int n = lane + 32 * u;
    r[u] = 0.0;
    if (n < N) r[u] = candidate_normal(seed, i, l, n);   // A7
  }
  double b[kMaxV];   // b[u] holds coordinate lane + 32u of G r
#pragma unroll
  for (int u = 0; u < kMaxV; ++u) b[u] = 0.0;
  for (int q = 0; q < d; ++q) {
    const double* g = G + (int64_t)q * N;
    double part = 0.0;
#pragma unroll
    for (int u = 0; u < kMaxV; ++u) {
      int n = lane + 32 * u;
      if (n < N) part += g[n] * r[u];
    }
    part = warp_sum(part);
    if ((q & 31) == lane) b[q >> 5] = part;
  }
  double ss = 0.0;
#pragma unroll
  for (int u = 0; u < kMaxV; ++u) ss += b[u] * b[u];
  double nrm = sqrt(warp_sum(ss));
  bool deg = nrm < kDegenerateNorm;                       // A18
#pragma unroll
  for (int u = 0; u < kMaxV; ++u) {
    int q = lane + 32 * u;
    if (q < d) W64[j * d + q] = deg ? 0.0 : b[u] / nrm;   // PAPER.md:239 normalise
  }
  if (lane == 0) {
    state[j] = deg ? ST_DEGENERATE : ST_ACTIVE;
    keep[j] = deg ? 0 : 1;
    if (fine) fine[j] = fine_init;
    if (dprev) dprev[j] = INFINITY;
  }
}

}  // namespace

int launch_reduce_apply(cudaStream_t st, const float* Gf, int d, int N, const float* X, int64_t ld, int64_t M,
                        float* Xr, int64_t ldr, __half* Xh, int NPd, int64_t ldx) {
  int64_t mcols = Xh ? ldx : M;
  int rows = Xh ? NPd : d;
  dim3 grid((unsigned)ceil_div(mcols, MTL), (unsigned)ceil_div(rows, RT));
  k_reduce_apply<<<grid, 256, 0, st>>>(Gf, d, N, X, ld, M, Xr, ldr, Xh, NPd, ldx);
  return 1;
}

int launch_cand_basis(cudaStream_t st, uint64_t seed, int i, int64_t id_base, int64_t L_local, int N,
                      const double* G, int d, double* W64, uint8_t* state, uint8_t* keep, uint8_t* fine,
                      uint8_t fine_init, double* dprev) {
  int64_t threads = L_local * 32;
  k_cand_basis<<<(unsigned)ceil_div(threads, 256), 256, 0, st>>>(seed, i, id_base, L_local, N, G, d, W64, state, keep,
                                                                 fine, fine_init, dprev);
  return 1;
}

}  // namespace oica
