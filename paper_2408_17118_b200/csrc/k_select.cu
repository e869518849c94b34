// K5: device-side selection and accept (eqs. (1)-(2); reading A6).
//
//   census      counts of converged / unconverged / degenerate candidates on this rank
//   argmax(c)   p_c = argmax Upsilon(alpha_old) over eligible, unassigned candidates (ties ->
//               lowest id); for c > 0 only candidates within a margin of the first maximum
//   assign(c)   cluster c = unassigned eligible l with 1 - |w_l . w_pc| <= 1e-6; q_c = min id
//   alpha_exact alpha at the FINAL w of each q_c, y in fp64 (A15)
//   finish      per-rank cluster records (q, alpha, Upsilon, size, iters) + rows
//   merge_accept  all ranks' records -> winner (merge.hpp), canonical sign (A17), append to
//               W_acc, Gaussianity flag
#include "kernels.cuh"
#include "merge.hpp"

namespace oica {
namespace {

constexpr double kRefineMarginRel = 1e-2;   // clusters refined: Upsilon~ >= max - 1%
constexpr double kRefineMarginAbs = 1e-7;

// w_l . w_p as one warp computes it: lane j sums coordinates j, j + 32, ... (fma chain from 0),
// then the xor butterfly of warp_sum.  The cluster test of every selection path uses exactly this
// arithmetic, so membership never depends on which kernel (and so on the L-shard split) decides it.
__device__ __forceinline__ double dot_warp(const double* __restrict__ a, const double* __restrict__ b, int N,
                                           int lane) {
  double d = 0.0;
  for (int n = lane; n < N; n += 32) d = fma(a[n], b[n], d);
  return warp_sum(d);
}
__device__ __forceinline__ bool eligible(uint8_t st, bool include_unconv, int n_conv) {
  return st == ST_CONVERGED || (st == ST_ACTIVE && (include_unconv || n_conv == 0));
}

// counts: [0] converged, [1] unconverged (active), [2] degenerate, [3] domain-excluded eligible
// nconv_g (device, may be null): the converged count over ALL ranks (L-shard): reading A4's
// "no run converged" fallback must be decided globally, or a rank whose runs all missed the cap
// would submit unconverged records that a single GPU would have excluded (GPU-count invariance)
__global__ void __launch_bounds__(1024) k_census(const uint8_t* __restrict__ state, const double* __restrict__ alpha,
                                                 int L, uint32_t flags, int* counts, int* cluster,
                                                 const int* __restrict__ nconv_g) {
  __shared__ int c[4];
  if (threadIdx.x < 4) c[threadIdx.x] = 0;
  __syncthreads();
  int nc = 0, na = 0, nd = 0;
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    uint8_t s = state[l];
    nc += s == ST_CONVERGED;
    na += s == ST_ACTIVE;
    nd += s == ST_DEGENERATE;
    cluster[l] = -1;
  }
  atomicAdd(&c[0], nc);
  atomicAdd(&c[1], na);
  atomicAdd(&c[2], nd);
  __syncthreads();
  bool inc = flags & OICA_INCLUDE_UNCONVERGED;
  const int n_conv = nconv_g ? *nconv_g : c[0];
  int ndom = 0;
  for (int l = threadIdx.x; l < L; l += blockDim.x)
    if (eligible(state[l], inc, n_conv) && !(alpha[l] > kAlphaFloor)) ++ndom;
  atomicAdd(&c[3], ndom);
  __syncthreads();
  if (threadIdx.x < 4) counts[threadIdx.x] = c[threadIdx.x];
}

__global__ void __launch_bounds__(1024) k_argmax(const double* __restrict__ alpha, const uint8_t* __restrict__ state,
                                                 const int* __restrict__ cluster, const int* __restrict__ counts, int L,
                                                 int64_t id_base, uint32_t flags, int c, double* ups_max, int* pc,
                                                 int* qc, int* csize, const int* __restrict__ nconv_g) {
  __shared__ double su[32];
  __shared__ int sl[32];
  bool inc = flags & OICA_INCLUDE_UNCONVERGED;
  int n_conv = nconv_g ? *nconv_g : counts[0];
  double thr = -INFINITY;
  if (c > 0) {
    double um = *ups_max;
    if (pc[c - 1] < 0) {   // previous round found nothing
      if (threadIdx.x == 0) { pc[c] = -1; qc[c] = INT32_MAX; csize[c] = 0; }
      return;
    }
    thr = um - fmax(kRefineMarginRel * fabs(um), kRefineMarginAbs);
  }
  double bu = -INFINITY;
  int bl = INT32_MAX;
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    if (!eligible(state[l], inc, n_conv) || cluster[l] >= 0) continue;
    double u = upsilon_of(alpha[l]);
    if (!(u > -INFINITY) || u < thr) continue;
    if (u > bu || (u == bu && l < bl)) { bu = u; bl = l; }
  }
  // warp then block reduce: max u, ties -> lowest index (ids are id_base + l, monotone)
  for (int o = 16; o > 0; o >>= 1) {
    double u2 = __shfl_xor_sync(0xffffffffu, bu, o);
    int l2 = __shfl_xor_sync(0xffffffffu, bl, o);
    if (u2 > bu || (u2 == bu && l2 < bl)) { bu = u2; bl = l2; }
  }
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { su[w] = bu; sl[w] = bl; }
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    bu = lane < nw ? su[lane] : -INFINITY;
    bl = lane < nw ? sl[lane] : INT32_MAX;
    for (int o = 16; o > 0; o >>= 1) {
      double u2 = __shfl_xor_sync(0xffffffffu, bu, o);
      int l2 = __shfl_xor_sync(0xffffffffu, bl, o);
      if (u2 > bu || (u2 == bu && l2 < bl)) { bu = u2; bl = l2; }
    }
    if (lane == 0) {
      bool found = bu > -INFINITY && bl != INT32_MAX;
      pc[c] = found ? bl : -1;
      qc[c] = INT32_MAX;
      csize[c] = 0;
      if (c == 0) *ups_max = found ? bu : -INFINITY;
    }
  }
  (void)id_base;
}

__global__ void k_assign(const double* __restrict__ W64, const double* __restrict__ alpha,
                         const uint8_t* __restrict__ state, int* __restrict__ cluster, const int* __restrict__ counts,
                         int L, int N, uint32_t flags, int c, const int* __restrict__ pc, int* qc, int* csize,
                         const int* __restrict__ nconv_g) {
  int l = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int lane = threadIdx.x & 31;
  int p = pc[c];
  if (p < 0 || l >= L) return;
  bool inc = flags & OICA_INCLUDE_UNCONVERGED;
  if (!eligible(state[l], inc, nconv_g ? *nconv_g : counts[0]) || cluster[l] >= 0 || !(alpha[l] > kAlphaFloor)) return;
  if ((flags & OICA_RAW_ARGMAX) && l != p) return;   // raw argmax: singleton records
  const double d = dot_warp(W64 + (int64_t)l * N, W64 + (int64_t)p * N, N, lane);
  if (1.0 - fabs(d) <= kClusterDelta && lane == 0) {
    cluster[l] = c;
    atomicMin(&qc[c], l);
    atomicAdd(&csize[c], 1);
  }
}

// census + all argmax / assign rounds in one single-block launch for small L (the multi-kernel
// sequence is ~17 launches of a few microseconds each there).  Same decisions as k_census,
// k_argmax and k_assign: block reductions with the same tie rule, the same refine margin, the same
// cluster test; q_c = min id and the sizes are order-independent (atomics).
constexpr int kSelectSmallL = 2048;   // above: the multi-block assign is faster (cfg 2, L = 4096: 250 vs 350 us)
constexpr int kSelectThreadN = 64;    // up to this N the single block takes ...
// (cluster tests: one warp per candidate row, coalesced 8-byte lanes; one thread per row read 32
// rows per load instruction -- ~225 us per selection at cfg 2 under ncu)
constexpr int kSelectSmallLThread = 4096;   // ... and takes up to this many candidates
__global__ void __launch_bounds__(1024) k_select_small(const double* __restrict__ W64,
                                                       const double* __restrict__ alpha,
                                                       const uint8_t* __restrict__ state, int L, int N,
                                                       uint32_t flags, int* counts, int* cluster, double* ups_max,
                                                       int* pc, int* qc, int* csize, const int* __restrict__ nconv_g) {
  __shared__ int cnt[4];
  __shared__ double su[32];
  __shared__ int sl[32];
  __shared__ int s_p;
  __shared__ double s_um;
  __shared__ double s_wp[256];   // N <= 256 (oica_set_data)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const bool inc = flags & OICA_INCLUDE_UNCONVERGED;
  const bool raw = flags & OICA_RAW_ARGMAX;
  if (tid < 4) cnt[tid] = 0;
  __syncthreads();
  int nc = 0, na = 0, nd = 0;
  for (int l = tid; l < L; l += blockDim.x) {
    const uint8_t st = state[l];
    nc += st == ST_CONVERGED;
    na += st == ST_ACTIVE;
    nd += st == ST_DEGENERATE;
    cluster[l] = -1;
  }
  atomicAdd(&cnt[0], nc);
  atomicAdd(&cnt[1], na);
  atomicAdd(&cnt[2], nd);
  __syncthreads();
  const int n_conv = nconv_g ? *nconv_g : cnt[0];
  int ndom = 0;
  for (int l = tid; l < L; l += blockDim.x)
    if (eligible(state[l], inc, n_conv) && !(alpha[l] > kAlphaFloor)) ++ndom;
  atomicAdd(&cnt[3], ndom);
  __syncthreads();
  if (tid < 4) counts[tid] = cnt[tid];
  bool done = false;
  for (int c = 0; c < kMaxClusters; ++c) {
    if (done) {   // an earlier round found nothing: the remaining records are empty
      if (tid == 0) { pc[c] = -1; qc[c] = INT32_MAX; csize[c] = 0; }
      continue;
    }
    double thr = -INFINITY;
    if (c > 0) thr = s_um - fmax(kRefineMarginRel * fabs(s_um), kRefineMarginAbs);
    double bu = -INFINITY;
    int bl = INT32_MAX;
    for (int l = tid; l < L; l += blockDim.x) {
      if (!eligible(state[l], inc, n_conv) || cluster[l] >= 0) continue;
      const double u = upsilon_of(alpha[l]);
      if (!(u > -INFINITY) || u < thr) continue;
      if (u > bu || (u == bu && l < bl)) { bu = u; bl = l; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double u2 = __shfl_xor_sync(0xffffffffu, bu, o);
      const int l2 = __shfl_xor_sync(0xffffffffu, bl, o);
      if (u2 > bu || (u2 == bu && l2 < bl)) { bu = u2; bl = l2; }
    }
    if (lane == 0) { su[w] = bu; sl[w] = bl; }
    __syncthreads();
    if (w == 0) {
      bu = su[lane];
      bl = sl[lane];
      for (int o = 16; o > 0; o >>= 1) {
        const double u2 = __shfl_xor_sync(0xffffffffu, bu, o);
        const int l2 = __shfl_xor_sync(0xffffffffu, bl, o);
        if (u2 > bu || (u2 == bu && l2 < bl)) { bu = u2; bl = l2; }
      }
      if (lane == 0) {
        const bool found = bu > -INFINITY && bl != INT32_MAX;
        s_p = found ? bl : -1;
        pc[c] = s_p;
        qc[c] = INT32_MAX;
        csize[c] = 0;
        if (c == 0) {
          s_um = found ? bu : -INFINITY;
          *ups_max = s_um;
        }
      }
    }
    __syncthreads();
    const int p = s_p;
    if (p < 0) {
      done = true;
      continue;
    }
    // cluster test, one warp per candidate row (coalesced lanes, dot_warp's arithmetic: lane j
    // sums coordinates j, j + 32, ... by an fma chain from 0, then the butterfly), up to kB rows
    // of a warp's 32 in flight together (latency-bound otherwise)
    for (int n = tid; n < N; n += blockDim.x) s_wp[n] = W64[(int64_t)p * N + n];
    __syncthreads();
    constexpr int kB = 8;
    for (int base = w * 32; base < L; base += blockDim.x) {   // a warp takes 32 consecutive rows
      const int l = base + lane;
      const bool e = l < L && eligible(state[l], inc, n_conv) && cluster[l] < 0 && alpha[l] > kAlphaFloor &&
                     !(raw && l != p);
      unsigned mask = __ballot_sync(0xffffffffu, e);
      while (mask) {
        int rr[kB];
        int nr = 0;
#pragma unroll
        for (int i = 0; i < kB; ++i) {
          rr[i] = mask ? base + __ffs(mask) - 1 : -1;
          if (mask) {
            mask &= mask - 1;
            ++nr;
          }
        }
        double d[kB];
#pragma unroll
        for (int i = 0; i < kB; ++i) d[i] = 0.0;
        for (int n = lane; n < N; n += 32) {
          const double b = s_wp[n];
#pragma unroll
          for (int i = 0; i < kB; ++i)
            if (i < nr) d[i] = fma(W64[(int64_t)rr[i] * N + n], b, d[i]);
        }
#pragma unroll
        for (int i = 0; i < kB; ++i) {
          if (i >= nr) break;
          const double di = warp_sum(d[i]);
          if (1.0 - fabs(di) <= kClusterDelta && lane == 0) {
            cluster[rr[i]] = c;
            atomicMin(&qc[c], rr[i]);
            atomicAdd(&csize[c], 1);
          }
        }
      }
    }
    __syncthreads();
  }
}

// acc[c] += sum over this thread's samples of (w_c . x_m)^4 for the first CC rows, y in fp64.
template <int CC>
__device__ __forceinline__ void alpha_accumulate(const double (*ws)[256], const float* __restrict__ X, int64_t ld,
                                                 int N, int64_t mb, int64_t me, double (&acc)[kMaxClusters]) {
  for (int64_t m = mb + threadIdx.x; m < me; m += blockDim.x) {
    double y[CC];
#pragma unroll
    for (int c = 0; c < CC; ++c) y[c] = 0.0;
    int n = 0;
    for (; n + 8 <= N; n += 8) {   // 8 independent loads in flight per thread (latency-bound otherwise)
      float xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = __ldg(X + (int64_t)(n + u) * ld + m);
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int c = 0; c < CC; ++c) y[c] = fma(ws[c][n + u], (double)xv[u], y[c]);
    }
    for (; n < N; ++n) {
      double x = (double)__ldg(X + (int64_t)n * ld + m);
#pragma unroll
      for (int c = 0; c < CC; ++c) y[c] = fma(ws[c][n], x, y[c]);
    }
#pragma unroll
    for (int c = 0; c < CC; ++c) {
      double y2 = y[c] * y[c];
      acc[c] = fma(y2, y2, acc[c]);
    }
  }
}

// part[c][b] = sum over block b's samples of (w_c . x_m)^4, y in fp64 (fixed order).
__global__ void __launch_bounds__(256) k_alpha_exact(const double* __restrict__ W64, const float* __restrict__ X,
                                                     int64_t ld, int64_t M, int N, const int* __restrict__ pc,
                                                     const int* __restrict__ qc, uint32_t flags, double* part,
                                                     int nblk) {
  __shared__ double ws[kMaxClusters][256];
  __shared__ int rows[kMaxClusters];
  __shared__ int nv;
  __shared__ double red[kMaxClusters][8];
  bool raw = flags & OICA_RAW_ARGMAX;
  if (threadIdx.x == 0) {
    int k = 0;
    for (int c = 0; c < kMaxClusters; ++c) {
      int r = raw ? pc[c] : (pc[c] >= 0 ? qc[c] : -1);
      rows[c] = r;
      if (r >= 0) k = c + 1;
    }
    nv = k;
  }
  __syncthreads();
  int C = nv;
  for (int idx = threadIdx.x; idx < C * N; idx += blockDim.x) {
    int c = idx / N, n = idx % N;
    ws[c][n] = rows[c] >= 0 ? W64[(int64_t)rows[c] * N + n] : 0.0;
  }
  __syncthreads();
  int64_t chunk = ceil_div(M, nblk);
  int64_t mb = (int64_t)blockIdx.x * chunk, me = min(M, mb + chunk);
  double acc[kMaxClusters];
#pragma unroll
  for (int c = 0; c < kMaxClusters; ++c) acc[c] = 0.0;
  // usually one or two clusters are refined: the row count is a block-uniform template choice
  if (C <= 1)
    alpha_accumulate<1>(ws, X, ld, N, mb, me, acc);
  else if (C <= 2)
    alpha_accumulate<2>(ws, X, ld, N, mb, me, acc);
  else if (C <= 4)
    alpha_accumulate<4>(ws, X, ld, N, mb, me, acc);
  else
    alpha_accumulate<kMaxClusters>(ws, X, ld, N, mb, me, acc);
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < kMaxClusters; ++c) {
    double v = warp_sum(acc[c]);
    if (lane == 0) red[c][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < kMaxClusters) {
    double v = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) v += red[threadIdx.x][k];
    part[(int64_t)threadIdx.x * nblk + blockIdx.x] = v;
  }
}

// one warp per cluster row: lane j sums blocks j, j + 32, ... in order, then the xor butterfly
// (a fixed order; one thread per row was a ~1200-long chain of dependent adds, ~20 us)
__global__ void __launch_bounds__(32 * kMaxClusters) k_alpha_reduce(const double* __restrict__ part, int nblk,
                                                                    double* s4c) {
  const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* p = part + (int64_t)c * nblk;
  double v = 0.0;
  for (int b = lane; b < nblk; b += 32) v += p[b];
  v = warp_sum(v);
  if (lane == 0) s4c[c] = v;
}

__global__ void k_finish(const double* __restrict__ W64, const int* __restrict__ iters, const int* __restrict__ counts,
                         const int* __restrict__ pc, const int* __restrict__ qc, const int* __restrict__ csize,
                         const double* __restrict__ s4c, int64_t id_base, int N, double M, uint32_t flags,
                         int64_t sum_active, int n_iter, const int* __restrict__ nonfinite,
                         const IterCtl* __restrict__ ctl, RankSummary* sum, double* wsum) {
  bool raw = flags & OICA_RAW_ARGMAX;
  for (int idx = threadIdx.x; idx < kMaxClusters * N; idx += blockDim.x) {
    int c = idx / N, n = idx % N;
    int r = raw ? pc[c] : (pc[c] >= 0 ? qc[c] : -1);
    wsum[idx] = r >= 0 ? W64[(int64_t)r * N + n] : 0.0;
  }
  if (threadIdx.x < kMaxClusters) {
    int c = threadIdx.x;
    int r = raw ? pc[c] : (pc[c] >= 0 ? qc[c] : -1);
    oica_cluster_record rec{};
    if (r >= 0) {
      const double obj = s4c[c] / M;                    // sum y^4 / M at the final w
      double a = obj - 3.0;                             // eq. (2)
      rec.alpha = a;
      rec.objective = obj;
      rec.upsilon = upsilon_of(a);                      // eq. (1)
      rec.q = id_base + r;
      rec.size = raw ? 1 : csize[c];
      rec.iters = iters[r];
      rec.valid = rec.upsilon > -INFINITY ? 1 : 0;
    }
    sum->rec[c] = rec;
  }
  if (threadIdx.x == 0) {
    sum->n_conv = counts[0];
    sum->n_unconv = counts[1];
    sum->n_deg = counts[2];
    sum->n_domain = counts[3];
    sum->sum_active = sum_active >= 0 ? sum_active : ctl->sum_active;
    sum->n_iter = sum_active >= 0 ? n_iter : ctl->t - 1;
    sum->n_nonfinite = nonfinite ? *nonfinite : 0;
  }
}

__global__ void k_merge_accept(const RankSummary* __restrict__ all, const double* __restrict__ wall, int world, int N,
                               int i, double M, uint32_t flags, double* Wacc, int k, ComponentRecord* out,
                               double* w_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  oica_cluster_record recs[64 * kMaxClusters];
  int32_t group[64 * kMaxClusters];
  int n = 0;
  ComponentRecord r{};
  for (int rk = 0; rk < world; ++rk) {
    for (int c = 0; c < kMaxClusters; ++c) recs[n++] = all[rk].rec[c];
    r.n_conv += all[rk].n_conv;
    r.n_unconv += all[rk].n_unconv;
    r.n_deg += all[rk].n_deg;
    r.n_domain += all[rk].n_domain;
    r.sum_active += all[rk].sum_active;
    r.n_nonfinite += all[rk].n_nonfinite;
    r.n_iter = max(r.n_iter, all[rk].n_iter);
  }
  MergeOut m = merge_records(recs, wall, n, N, group, flags & OICA_RAW_ARGMAX, kClusterDelta, kNearTieRel);
  if (m.winner < 0) {
    int64_t L = r.n_conv + r.n_unconv + r.n_deg;
    r.status = (r.n_deg == L) ? OICA_ERR_ALL_CANDIDATES_DEGENERATE : OICA_ERR_DOMAIN;
    *out = r;
    return;
  }
  const oica_cluster_record& win = recs[m.winner];
  const double* w = wall + (int64_t)m.winner * N;
  int jm = 0;
  double am = -1.0;
  for (int j = 0; j < N; ++j)
    if (fabs(w[j]) > am) { am = fabs(w[j]); jm = j; }
  double sg = w[jm] < 0.0 ? -1.0 : 1.0;                  // canonical sign (A17)
  for (int j = 0; j < N; ++j) {
    Wacc[(int64_t)k * N + j] = sg * w[j];
    w_out[j] = sg * w[j];
  }
  r.w_alpha = win.alpha;
  r.w_upsilon = win.upsilon;
  r.w_objective = win.objective;
  r.q = win.q;
  r.iters = win.iters;
  r.cluster_size = m.merged_size;
  r.near_tie = m.near_tie;
  r.gaussian = win.upsilon < 2.0 * (N - i + 2) * (N - i + 1) / M ? 1 : 0;
  r.status = OICA_OK;
  *out = r;
}

// out[0] = number of converged candidates on this rank (summed over ranks by the caller)
__global__ void __launch_bounds__(1024) k_count_converged(const uint8_t* __restrict__ state, int L, int* out) {
  __shared__ int c;
  if (threadIdx.x == 0) c = 0;
  __syncthreads();
  int n = 0;
  for (int l = threadIdx.x; l < L; l += blockDim.x) n += state[l] == ST_CONVERGED;
  n = __reduce_add_sync(0xffffffffu, n);
  if ((threadIdx.x & 31) == 0) atomicAdd(&c, n);
  __syncthreads();
  if (threadIdx.x == 0) *out = c;
}

}  // namespace

int launch_count_converged(cudaStream_t st, const uint8_t* state, int L, int* out) {
  k_count_converged<<<1, 1024, 0, st>>>(state, L, out);
  return 1;
}

int launch_select_local(cudaStream_t st, const double* W64, const double* alpha_old, const uint8_t* state,
                        const int* iters, int L_local, int64_t id_base, int N, uint32_t flags, const float* X,
                        int64_t ld, int64_t M_local, int* cluster, int* pc, int* qc, int* csize, double* ups_max,
                        int* counts, double* part, int nblk, double* s4c, const int* nconv_g) {
  (void)iters;
  int launches = 0;
  if (L_local <= kSelectSmallL || (N <= kSelectThreadN && L_local <= kSelectSmallLThread)) {
    k_select_small<<<1, 1024, 0, st>>>(W64, alpha_old, state, L_local, N, flags, counts, cluster, ups_max, pc, qc,
                                       csize, nconv_g);
    ++launches;
  } else {
    k_census<<<1, 1024, 0, st>>>(state, alpha_old, L_local, flags, counts, cluster, nconv_g);
    ++launches;
    unsigned ablocks = (unsigned)ceil_div((int64_t)L_local * 32, 256);
    for (int c = 0; c < kMaxClusters; ++c) {
      k_argmax<<<1, 1024, 0, st>>>(alpha_old, state, cluster, counts, L_local, id_base, flags, c, ups_max, pc, qc,
                                   csize, nconv_g);
      k_assign<<<ablocks, 256, 0, st>>>(W64, alpha_old, state, cluster, counts, L_local, N, flags, c, pc, qc, csize,
                                        nconv_g);
      launches += 2;
    }
  }
  k_alpha_exact<<<nblk, 256, 0, st>>>(W64, X, ld, M_local, N, pc, qc, flags, part, nblk);
  k_alpha_reduce<<<1, 32 * kMaxClusters, 0, st>>>(part, nblk, s4c);
  return launches + 2;
}

int launch_select_finish(cudaStream_t st, const double* W64, const int* iters, const int* counts, const int* pc,
                         const int* qc, const int* csize, const double* s4c, int64_t id_base, int N, double M_global,
                         uint32_t flags, int64_t sum_active, int n_iter, const int* nonfinite, const IterCtl* ctl,
                         RankSummary* summary, double* wsum) {
  k_finish<<<1, 256, 0, st>>>(W64, iters, counts, pc, qc, csize, s4c, id_base, N, M_global, flags, sum_active, n_iter,
                              nonfinite, ctl, summary, wsum);
  return 1;
}

int launch_merge_accept(cudaStream_t st, const RankSummary* all, const double* wall, int world, int N, int i,
                        double M_global, uint32_t flags, double* Wacc, int k, ComponentRecord* rec, double* w_out) {
  k_merge_accept<<<1, 32, 0, st>>>(all, wall, world, N, i, M_global, flags, Wacc, k, rec, w_out);
  return 1;
}

}  // namespace oica
