// Boundary: PCA whitening "in advance" (readings A11/A12), fp64 arithmetic.
//   row means -> covariance C = Xc Xc^T / M (64x64 tiles, fixed-order split-M reduction)
//   -> (host Jacobi eigensolver in abi.cpp) -> Xw = V (X - mean) in fp32.
#include "kernels.cuh"

namespace oica {
namespace {

__global__ void __launch_bounds__(256) k_row_mean(const float* __restrict__ X, int64_t ld, int64_t M,
                                                  double* __restrict__ mean) {
  __shared__ double red[8];
  const float* x = X + (int64_t)blockIdx.x * ld;
  double s = 0.0;
  for (int64_t m = threadIdx.x; m < M; m += 256) s += (double)x[m];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    mean[blockIdx.x] = t / (double)M;
  }
}

constexpr int T = 64, KC = 32;

// part[split][i][j] = sum over the split's samples of (x_i - mu_i)(x_j - mu_j)
__global__ void __launch_bounds__(256) k_cov_tile(const float* __restrict__ X, int64_t ld, int N, int64_t M,
                                                  const double* __restrict__ mean, int nsplit, double* __restrict__ part) {
  __shared__ double A[KC][T + 1], B[KC][T + 1];
  int bi = blockIdx.x * T, bj = blockIdx.y * T, sp = blockIdx.z;
  int64_t chunk = round_up(ceil_div(M, nsplit), KC);
  int64_t mb = (int64_t)sp * chunk, me = min(M, mb + chunk);
  int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int64_t m0 = mb; m0 < me; m0 += KC) {
    for (int idx = threadIdx.x; idx < T * KC; idx += 256) {
      int r = idx / KC, c = idx % KC;
      int64_t m = m0 + c;
      int gi = bi + r, gj = bj + r;
      A[c][r] = (gi < N && m < me) ? (double)X[(int64_t)gi * ld + m] - mean[gi] : 0.0;
      B[c][r] = (gj < N && m < me) ? (double)X[(int64_t)gj * ld + m] - mean[gj] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int c = 0; c < KC; ++c) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { a[u] = A[c][ty + 16 * u]; b[u] = B[c][tx + 16 * u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      int gi = bi + ty + 16 * u, gj = bj + tx + 16 * v;
      if (gi < N && gj < N) part[((int64_t)sp * N + gi) * N + gj] = acc[u][v];
    }
}

__global__ void k_cov_reduce(const double* __restrict__ part, int nsplit, int N, int64_t M, double* __restrict__ C) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N * N) return;
  double s = 0.0;
  for (int sp = 0; sp < nsplit; ++sp) s += part[(int64_t)sp * N * N + idx];
  C[idx] = s / (double)M;
}

// Xw[i][m] = sum_j V[i][j] (x_jm - mu_j), fp64 accumulate, fp32 store.
__global__ void __launch_bounds__(256) k_apply(const float* __restrict__ X, int64_t ld, int N, int64_t M,
                                               const double* __restrict__ mean, const double* __restrict__ V,
                                               float* __restrict__ Xw, int64_t ldo) {
  __shared__ double Vs[T][KC + 1], Xs[KC][T + 1];
  int bi = blockIdx.y * T;
  int64_t bm = (int64_t)blockIdx.x * T;
  int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int j0 = 0; j0 < N; j0 += KC) {
    for (int idx = threadIdx.x; idx < T * KC; idx += 256) {
      int r = idx / KC, c = idx % KC;
      int gi = bi + r, gj = j0 + c;
      Vs[r][c] = (gi < N && gj < N) ? V[(int64_t)gi * N + gj] : 0.0;
      int cj = idx / T, cm = idx % T;
      int gjj = j0 + cj;
      int64_t m = bm + cm;
      Xs[cj][cm] = (gjj < N && m < M) ? (double)X[(int64_t)gjj * ld + m] - mean[gjj] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int c = 0; c < KC; ++c) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { a[u] = Vs[ty + 16 * u][c]; b[u] = Xs[c][tx + 16 * u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      int gi = bi + ty + 16 * u;
      int64_t m = bm + tx + 16 * v;
      if (gi < N && m < M) Xw[(int64_t)gi * ldo + m] = (float)acc[u][v];
    }
}

}  // namespace

int launch_row_mean(cudaStream_t st, const float* X, int64_t ld, int N, int64_t M, double* mean) {
  k_row_mean<<<N, 256, 0, st>>>(X, ld, M, mean);
  return 1;
}

int launch_covariance(cudaStream_t st, const float* X, int64_t ld, int N, int64_t M, const double* mean, double* part,
                      int nsplit, double* C) {
  dim3 grid((unsigned)ceil_div(N, T), (unsigned)ceil_div(N, T), (unsigned)nsplit);
  k_cov_tile<<<grid, 256, 0, st>>>(X, ld, N, M, mean, nsplit, part);
  k_cov_reduce<<<(unsigned)ceil_div((int64_t)N * N, 256), 256, 0, st>>>(part, nsplit, N, M, C);
  return 2;
}

int launch_apply_whitening(cudaStream_t st, const float* X, int64_t ld, int N, int64_t M, const double* mean,
                           const double* V, float* Xw, int64_t ldo) {
  dim3 grid((unsigned)ceil_div(M, T), (unsigned)ceil_div(N, T));
  k_apply<<<grid, 256, 0, st>>>(X, ld, N, M, mean, V, Xw, ldo);
  return 1;
}

}  // namespace oica
