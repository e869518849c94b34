// Hybrid L -> M tail: once few candidate runs remain active
// across the ranks of an L-sharded job, their state is all-gathered (C4), iterated M-sharded by
// every rank, and written back to the owning rank for the selection.
//   k_tail_pack    : active rows of this rank -> records [w (d) | alpha_old | dprev | fine | global id]
//   k_tail_unpack  : gathered records (rank order) -> the tail's row arrays
//   k_tail_scatter : tail rows owned by this rank -> its candidate arrays (by global id)
// Plain data movement: no arithmetic of the method happens here.
#include <algorithm>

#include "kernels.cuh"

namespace oica {
namespace {

__global__ void k_tail_pack(const int* __restrict__ act, const int* __restrict__ cnt, int L_ub,
                            const double* __restrict__ W64, const double* __restrict__ alpha_old,
                            const double* __restrict__ dprev, const uint8_t* __restrict__ fine, int64_t id_base, int d,
                            double* __restrict__ out) {
  const int R = d + 4;
  const int L = min(L_ub, cnt[0]);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)L * R;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(idx / R), c = (int)(idx % R);
    const int l = act[a];
    double v;
    if (c < d)
      v = W64[(int64_t)l * d + c];
    else if (c == d)
      v = alpha_old[l];
    else if (c == d + 1)
      v = dprev ? dprev[l] : 0.0;
    else if (c == d + 2)
      v = (fine && fine[l]) ? 1.0 : 0.0;
    else
      v = (double)(id_base + l);   // < 2^24: exact
    out[idx] = v;
  }
}

__global__ void k_tail_unpack(const double* __restrict__ in, int T, int d, double* __restrict__ W64,
                              double* __restrict__ alpha_old, double* __restrict__ dprev, uint8_t* __restrict__ fine,
                              uint8_t* __restrict__ state, uint8_t* __restrict__ keep, int64_t* __restrict__ ids) {
  const int R = d + 4;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)T * R;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(idx / R), c = (int)(idx % R);
    const double v = in[idx];
    if (c < d) {
      W64[(int64_t)a * d + c] = v;
    } else if (c == d) {
      alpha_old[a] = v;
    } else if (c == d + 1) {
      dprev[a] = v;
    } else if (c == d + 2) {
      fine[a] = v != 0.0 ? 1 : 0;
    } else {
      ids[a] = (int64_t)v;
      state[a] = ST_ACTIVE;
      keep[a] = 1;
    }
  }
}

__global__ void k_tail_scatter(int T, const int64_t* __restrict__ ids, const double* __restrict__ tW64,
                               const double* __restrict__ t_alpha, const int* __restrict__ t_iters,
                               const uint8_t* __restrict__ t_state, int64_t id_base, int64_t L_local, int d,
                               double* __restrict__ W64, double* __restrict__ alpha_old, int* __restrict__ iters,
                               uint8_t* __restrict__ state) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)T * d;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(idx / d), c = (int)(idx % d);
    const int64_t l = ids[a] - id_base;
    if (l < 0 || l >= L_local) continue;   // another rank's candidate
    W64[l * d + c] = tW64[idx];
    if (c == 0) {
      alpha_old[l] = t_alpha[a];
      iters[l] = t_iters[a];
      state[l] = t_state[a];
    }
  }
}

unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 4096)); }

}  // namespace

int launch_tail_pack(cudaStream_t st, const int* act, const int* cnt, int L_ub, const double* W64,
                     const double* alpha_old, const double* dprev, const uint8_t* fine, int64_t id_base, int d,
                     double* out) {
  if (L_ub <= 0) return 0;
  k_tail_pack<<<grid_for((int64_t)L_ub * (d + 4)), 256, 0, st>>>(act, cnt, L_ub, W64, alpha_old, dprev, fine, id_base,
                                                                  d, out);
  return 1;
}

int launch_tail_unpack(cudaStream_t st, const double* in, int T, int d, double* W64, double* alpha_old,
                       double* dprev, uint8_t* fine, uint8_t* state, uint8_t* keep, int64_t* ids) {
  if (T <= 0) return 0;
  k_tail_unpack<<<grid_for((int64_t)T * (d + 4)), 256, 0, st>>>(in, T, d, W64, alpha_old, dprev, fine, state, keep,
                                                                 ids);
  return 1;
}

int launch_tail_scatter(cudaStream_t st, int T, const int64_t* ids, const double* tW64, const double* t_alpha,
                        const int* t_iters, const uint8_t* t_state, int64_t id_base, int64_t L_local, int d,
                        double* W64, double* alpha_old, int* iters, uint8_t* state) {
  if (T <= 0) return 0;
  k_tail_scatter<<<grid_for((int64_t)T * d), 256, 0, st>>>(T, ids, tW64, t_alpha, t_iters, t_state, id_base, L_local,
                                                            d, W64, alpha_old, iters, state);
  return 1;
}

}  // namespace oica
