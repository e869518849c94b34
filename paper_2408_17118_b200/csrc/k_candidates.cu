// K1 candidate init, K3 fp64 epilogue, K4 compaction and operand gathers.
// One warp per candidate row for the fp64 row work (N <= 256 -> <= 8 values per lane).
#include <cuda_fp16.h>

#include "kernels.cuh"

namespace oica {
namespace {

constexpr int kMaxV = 8;  // 256 / 32 coordinates per lane


// v <- v - E v with E = Wacc^T Wacc: all coefficients w_k . v are
// taken from the incoming v (one projection, as written in the paper).
template <int V>
__device__ __forceinline__ void project_warp(double (&v)[V], const double* __restrict__ Wacc, int k,
                                             int N, int lane) {
  double h[V];
#pragma unroll
  for (int u = 0; u < V; ++u) h[u] = 0.0;
  // rows in blocks of RB: their loads and warp reductions are independent (latency-bound
  // otherwise when few rows run); same operations in the same order per row.  RB x V bounded
  // (registers: 8 coordinates per lane already fill them)
  constexpr int RB = V >= 8 ? 1 : 8 / V;
  for (int r0 = 0; r0 < k; r0 += RB) {
    const int nb = min(RB, k - r0);
    double c[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      c[b] = 0.0;
      if (b < nb) {
        const double* wr = Wacc + (int64_t)(r0 + b) * N;
#pragma unroll
        for (int u = 0; u < V; ++u) {
          int n = lane + 32 * u;
          if (n < N) c[b] += __ldg(wr + n) * v[u];
        }
      }
    }
#pragma unroll
    for (int b = 0; b < RB; ++b) c[b] = warp_sum(c[b]);
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      if (b < nb) {
        const double* wr = Wacc + (int64_t)(r0 + b) * N;
#pragma unroll
        for (int u = 0; u < V; ++u) {
          int n = lane + 32 * u;
          if (n < N) h[u] += c[b] * __ldg(wr + n);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < V; ++u) v[u] -= h[u];
}

__global__ void k_cand_init(uint64_t seed, int i, int64_t id_base, int64_t L_local, int N,
                            const double* __restrict__ Wacc, int k, double* __restrict__ W64,
                            uint8_t* __restrict__ state, uint8_t* __restrict__ keep, uint8_t* __restrict__ fine,
                            uint8_t fine_init, double* __restrict__ dprev) {
  int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (j >= L_local) return;
  uint64_t l = (uint64_t)(id_base + j);
  double v[kMaxV];
#pragma unroll
  for (int u = 0; u < kMaxV; ++u) {
    int n = lane + 32 * u;
    v[u] = 0.0;
    if (n < N) v[u] = candidate_normal(seed, i, l, n);   // A7
  }
  project_warp<kMaxV>(v, Wacc, k, N, lane);
  double ss = 0.0;
#pragma unroll
  for (int u = 0; u < kMaxV; ++u) ss += v[u] * v[u];
  double nrm = sqrt(warp_sum(ss));
  bool deg = nrm < kDegenerateNorm;                       // A18
#pragma unroll
  for (int u = 0; u < kMaxV; ++u) {
    int n = lane + 32 * u;
    if (n < N) W64[j * N + n] = deg ? 0.0 : v[u] / nrm;
  }
  if (lane == 0) {
    state[j] = deg ? ST_DEGENERATE : ST_ACTIVE;
    keep[j] = deg ? 0 : 1;
    if (fine) fine[j] = fine_init;
    if (dprev) dprev[j] = INFINITY;
  }
}

// sum_{j < n} v(j) in order j = 0, 1, ... (fp64), loads issued 8 at a time: with few active
// rows the epilogue is a chain of dependent adds over S (x P) partials, latency-bound otherwise
template <int D = 8, class F>
__device__ __forceinline__ double ordered_sum(int n, F&& v) {
  double acc = 0.0;
  int j = 0;
  for (; j + D <= n; j += D) {
    double t[D];
#pragma unroll
    for (int u = 0; u < D; ++u) t[u] = v(j + u);
#pragma unroll
    for (int u = 0; u < D; ++u) acc += t[u];
  }
  for (; j < n; ++j) acc += v(j);
  return acc;
}

// Partial sum of slot s for element (a, n): the slot's fp32 value, or with split parts (P > 1,
// common.cuh split_parts) the fp64 sum of its P parts in part order.
__device__ __forceinline__ double slot_part(const SlotPartials& Gp, int P, int s, int64_t cap, int ldg, int a, int n) {
  if (P > 1) {
    const float* g = Gp.sub + (((int64_t)s * kSplitMax) * Gp.sub_cap + a) * ldg + n;
    const int64_t qs = Gp.sub_cap * ldg;
    float t[kSplitMax];
#pragma unroll
    for (int q = 0; q < kSplitMax; ++q) t[q] = q < P ? __ldg(g + q * qs) : 0.f;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < kSplitMax; ++q)
      if (q < P) acc += (double)t[q];
    return acc;
  }
  if (Gp.f32) return (double)__ldg((const float*)Gp.p + ((int64_t)s * cap + a) * ldg + n);
  return __ldg((const double*)Gp.p + ((int64_t)s * cap + a) * ldg + n);
}

__device__ __forceinline__ int parts_of(const SlotPartials& Gp, int S) {
  return (Gp.f32 && Gp.sub) ? split_parts(Gp.cnt_g ? Gp.cnt_g[0] : Gp.L_g_host, S) : 1;
}

// sum over slots (fixed slot order) of the slot partial sums: the definition every consumer of
// the slot partials shares (epilogue, k_slot_reduce), so a row's G is the same whichever runs it
template <int D = 8>   // loads in flight per call (callers with many coordinates per lane: fewer)
__device__ __forceinline__ double slot_sum(SlotPartials Gp, int S, int64_t cap, int ldg, int a, int n) {
  const int P = parts_of(Gp, S);
  if (P > 1) return ordered_sum<D>(S, [&](int s) { return slot_part(Gp, P, s, cap, ldg, a, n); });
  // one partial per slot (the common case; the loop the whole-L epilogue streams at HBM rate)
  if (Gp.f32) {
    const float* g = (const float*)Gp.p + (int64_t)a * ldg + n;
    const int64_t st = cap * ldg;
    return ordered_sum<D>(S, [&](int s) { return (double)g[s * st]; });
  }
  const double* g = (const double*)Gp.p + (int64_t)a * ldg + n;
  const int64_t st = cap * ldg;
  return ordered_sum<D>(S, [&](int s) { return g[s * st]; });
}

// coordinate n of the point the contraction used for active row a (master value w64 if none)
__device__ __forceinline__ double eval_coord(EvalPoint ev, int a, int n, double w64) {
  int64_t i = (int64_t)a * ev.ld + n;
  if (ev.hi) return ((double)__half2float(ev.hi[i]) + (ev.lo ? (double)__half2float(ev.lo[i]) : 0.0)) * 0.0625;
  if (ev.f32) return (double)ev.f32[i];
  return w64;
}

// K3: g = sum_s Gp / M - 3 w_e; g <- g - E g; w = g / ||g||;
// d = 1 - |w . w_old| as 0.5 ||w - s w_old||^2 (A1/A2); converged iff d <= tol.
// w_e is the operand the contraction was evaluated at (the whole of eq. (5) at
// one point, so the map keeps its vanishing tangent Jacobian at the fixed points); w_old is
// the fp64 master row.
template <int V>
__device__ __forceinline__ void epilogue_row(int a, int lane, const SlotPartials& Gp, const double* __restrict__ s4p,
                                             int S, int64_t cap, int ldg, const EvalPoint& ev,
                                             const int* __restrict__ act, const double* __restrict__ Wacc, int k,
                                             int N, double M, double tol, int t, double* __restrict__ W64,
                                             double* __restrict__ alpha_old, int* __restrict__ iters,
                                             uint8_t* __restrict__ state, uint8_t* __restrict__ keep,
                                             const Promotion& pr) {
  int l = act[a];
  double g[V], wo[V];
  double s4g = 0.0;
#pragma unroll
  for (int u = 0; u < V; ++u) {
    int n = lane + 32 * u;
    double acc = 0.0, w = 0.0, we = 0.0;
    if (n < N) {
      acc = slot_sum<(V >= 8 ? 2 : 8 / V)>(Gp, S, cap, ldg, a, n);
      w = W64[(int64_t)l * N + n];
      we = eval_coord(ev, a, n, w);
    }
    wo[u] = w;
    s4g += we * acc;
    g[u] = (n < N) ? acc / M - 3.0 * we : 0.0;           // PAPER.md:244-245 (eq. (5), A3)
  }
  double s4 = 0.0;
  if (s4p) {
    if (lane == 0)
      s4 = ordered_sum(S, [&](int s) { return __ldg(s4p + (int64_t)s * cap + a); });
  } else {
    s4 = warp_sum(s4g);   // identity w . sum_m y^3 x = sum_m y^4 (tensor-core path: approximate alpha)
  }
  project_warp<V>(g, Wacc, k, N, lane);
  double ss = 0.0;
#pragma unroll
  for (int u = 0; u < V; ++u) ss += g[u] * g[u];
  double nrm = sqrt(warp_sum(ss));
  // a non-finite update (fp16 range failure, non-finite data) retires the row and is reported
  // (Promotion::nonfinite): it must neither keep iterating to the cap nor enter the argmax
  const bool bad = !isfinite(nrm);
  bool deg = bad || nrm < kDegenerateNorm;
  double dot = 0.0;
#pragma unroll
  for (int u = 0; u < V; ++u) {
    g[u] = deg ? 0.0 : g[u] / nrm;
    dot += g[u] * wo[u];
  }
  dot = warp_sum(dot);
  double sg = dot < 0.0 ? -1.0 : 1.0;
  double dd = 0.0;
#pragma unroll
  for (int u = 0; u < V; ++u) {
    double e = g[u] - sg * wo[u];
    dd += e * e;
  }
  dd = 0.5 * warp_sum(dd);
  bool conv = !deg && dd <= tol;                          // PAPER.md:249-250 (A2)
  if (!deg) {
#pragma unroll
    for (int u = 0; u < V; ++u) {
      int n = lane + 32 * u;
      if (n < N) W64[(int64_t)l * N + n] = g[u];
    }
  }
  if (lane == 0) {
    if (bad && pr.nonfinite) atomicAdd(pr.nonfinite, 1);
    iters[l] = t;
    alpha_old[l] = s4 / M - 3.0;                          // eq. (2) at w_old (A15)
    state[l] = deg ? ST_DEGENERATE : (conv ? ST_CONVERGED : ST_ACTIVE);
    keep[a] = (deg || conv) ? 0 : 1;
    if (pr.fine && !deg && !conv) {                       // DESIGN.md §5 precision promotion
      if (!pr.fine[l] && ((dd <= pr.d_promote && dd > pr.ratio * pr.dprev[l]) || t >= pr.t_force)) pr.fine[l] = 1;
      pr.dprev[l] = dd;
    }
  }
}

template <int V>
__global__ void k_epilogue(SlotPartials Gp, const double* __restrict__ s4p, int S, int64_t cap, int ldg,
                           EvalPoint ev, const int* __restrict__ act, int L_act, const double* __restrict__ Wacc,
                           int k, int N, double M, double tol, int t, double* __restrict__ W64,
                           double* __restrict__ alpha_old, int* __restrict__ iters, uint8_t* __restrict__ state,
                           uint8_t* __restrict__ keep, Promotion pr, const int* __restrict__ cnt) {
  int a = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int lane = threadIdx.x & 31;
  if (cnt) L_act = min(L_act, cnt[0]);   // device count when the grid is an upper bound
  if (a >= L_act) return;
  epilogue_row<V>(a, lane, Gp, s4p, S, cap, ldg, ev, act, Wacc, k, N, M, tol, t, W64, alpha_old, iters, state, keep,
                  pr);
}

// Single-block, order-preserving compaction (deterministic), stably partitioned into coarse
// rows followed by fine rows.  Each thread takes a contiguous run of positions; per-thread counts
// are scanned with warp shuffles and one warp over the 32 warp totals (3 barriers).
__global__ void __launch_bounds__(1024) k_compact(const int* __restrict__ act_in, const uint8_t* __restrict__ keep,
                                                  const uint8_t* __restrict__ fine, int L_in, int* __restrict__ act_out,
                                                  int* out_dev, int* host_mapped, const int* cnt_in, int* hist) {
  __shared__ int wc[32], wf[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (cnt_in) L_in = min(L_in, cnt_in[0]);   // may alias out_dev: read before the barrier below
  __syncthreads();
  const int per = (L_in + 1023) / 1024;
  const int b = t * per, e = min(L_in, b + per);
  int cc = 0, cf = 0;
  for (int a = b; a < e; ++a) {
    if (!keep[a]) continue;
    int id = act_in ? act_in[a] : a;
    if (fine && fine[id]) ++cf; else ++cc;
  }
  // inclusive warp scans of (cc, cf)
  int ic = cc, jf = cf;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int vc = __shfl_up_sync(0xffffffffu, ic, o), vf = __shfl_up_sync(0xffffffffu, jf, o);
    if (lane >= o) {
      ic += vc;
      jf += vf;
    }
  }
  if (lane == 31) {
    wc[w] = ic;
    wf[w] = jf;
  }
  __syncthreads();
  if (w == 0) {   // exclusive scan of the warp totals
    int xc = wc[lane], xf = wf[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int vc = __shfl_up_sync(0xffffffffu, xc, o), vf = __shfl_up_sync(0xffffffffu, xf, o);
      if (lane >= o) {
        xc += vc;
        xf += vf;
      }
    }
    wc[lane] = xc;   // inclusive totals through warp `lane`
    wf[lane] = xf;
  }
  __syncthreads();
  const int n_coarse = wc[31], n_fine = wf[31];
  const int base_c = (w ? wc[w - 1] : 0) + ic - cc, base_f = (w ? wf[w - 1] : 0) + jf - cf;
  int pc = base_c, pf = n_coarse + base_f;
  for (int a = b; a < e; ++a) {
    if (!keep[a]) continue;
    int id = act_in ? act_in[a] : a;
    if (fine && fine[id]) act_out[pf++] = id; else act_out[pc++] = id;
  }
  if (t == 0) {
    out_dev[0] = n_coarse + n_fine;
    out_dev[1] = n_coarse;
    if (host_mapped) {
      ((volatile int*)host_mapped)[0] = n_coarse + n_fine;
      ((volatile int*)host_mapped)[1] = n_coarse;
    }
    if (hist) {
      hist[0] = n_coarse + n_fine;
      hist[1] = n_coarse;
    }
  }
}

__device__ __forceinline__ void operand_f32_elem(int64_t idx, int a, int n, const int* __restrict__ act,
                                                 const double* __restrict__ W64, int N, float* __restrict__ W32) {
  W32[idx] = n < N ? (float)W64[(int64_t)act[a] * N + n] : 0.f;
}

__global__ void k_operand_f32(const int* __restrict__ act, const int* __restrict__ Lact, int cap,
                              const double* __restrict__ W64, int N, int NP, float* __restrict__ W32) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int a = (int)(idx / NP), n = (int)(idx % NP);
  if (a >= cap || a >= *Lact) return;
  operand_f32_elem(idx, a, n, act, W64, N, W32);
}

// Split fp16 operand: w is scaled by 2^4 (|w| <= 1 -> <= 16) so most w_lo stay normal fp16;
// hi = fp16(2^4 w), lo = fp16(2^4 w - hi).  hi + lo = 2^4 w to ~2^-22 relative (absolute error
// <= 3e-8 / 16 per coordinate from lo subnormals); both GEMM1 passes share one accumulator.
// Coarse rows (fine[l] == 0) get lo = 0 (their contraction is the one-pass w_h product).
__device__ __forceinline__ void operand_f16x2_elem(int64_t idx, int a, int n, const int* __restrict__ act,
                                                   const double* __restrict__ W64, int N,
                                                   const uint8_t* __restrict__ fine, __half* __restrict__ Whi,
                                                   __half* __restrict__ Wlo) {
  int l = act[a];
  double w = n < N ? W64[(int64_t)l * N + n] * 16.0 : 0.0;
  __half hi = __double2half(w);
  __half lo = (fine && !fine[l]) ? __double2half(0.0) : __double2half(w - (double)__half2float(hi));
  Whi[idx] = hi;
  if (Wlo) Wlo[idx] = lo;
}

__global__ void k_operand_f16x2(const int* __restrict__ act, const int* __restrict__ Lact, int cap,
                                const double* __restrict__ W64, int N, int NP, const uint8_t* __restrict__ fine,
                                __half* __restrict__ Whi, __half* __restrict__ Wlo) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int a = (int)(idx / NP), n = (int)(idx % NP);
  if (a >= cap || a >= *Lact) return;
  operand_f16x2_elem(idx, a, n, act, W64, N, fine, Whi, Wlo);
}

// Few active rows (<= 32): K3 epilogue (one warp per row), K4 compaction (warp ballots, the
// same stable coarse-then-fine order as k_compact) and the next iteration's operand gather in
// one single-block launch instead of three (each of those kernels is a few microseconds of pure
// latency at this size).  Same per-row arithmetic as k_epilogue.
template <int V>
__global__ void __launch_bounds__(1024) k_iter_small(SlotPartials Gp, const double* __restrict__ s4p, int S,
                                                     int64_t cap, int ldg, EvalPoint ev, const int* __restrict__ act,
                                                     int L_ub, const double* __restrict__ Wacc, int k, int N,
                                                     double M, double tol, int t, double* __restrict__ W64,
                                                     double* __restrict__ alpha_old, int* __restrict__ iters,
                                                     uint8_t* __restrict__ state, uint8_t* __restrict__ keep,
                                                     Promotion pr, int* cnt, const uint8_t* __restrict__ fine,
                                                     int* __restrict__ act_out, int* host_mapped, int* hist,
                                                     int build, int NP, __half* __restrict__ Whi,
                                                     __half* __restrict__ Wlo, float* __restrict__ W32) {
  __shared__ int s_new;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L_in = min(L_ub, cnt[0]);
  if (warp < L_in)
    epilogue_row<V>(warp, lane, Gp, s4p, S, cap, ldg, ev, act, Wacc, k, N, M, tol, t, W64, alpha_old, iters, state,
                    keep, pr);
  __syncthreads();
  if (warp == 0) {   // stable partition: kept coarse rows, then kept fine rows (k_compact order)
    const bool in = lane < L_in && keep[lane];
    const int id = lane < L_in ? act[lane] : 0;
    const bool isf = in && fine && fine[id];
    const unsigned mc = __ballot_sync(0xffffffffu, in && !isf), mf = __ballot_sync(0xffffffffu, isf);
    const unsigned lt = (1u << lane) - 1u;
    const int n_coarse = __popc(mc), n_new = n_coarse + __popc(mf);
    if (in) act_out[isf ? n_coarse + __popc(mf & lt) : __popc(mc & lt)] = id;
    if (lane == 0) {
      cnt[0] = n_new;
      cnt[1] = n_coarse;
      if (host_mapped) {
        ((volatile int*)host_mapped)[0] = n_new;
        ((volatile int*)host_mapped)[1] = n_coarse;
      }
      if (hist) {
        hist[0] = n_new;
        hist[1] = n_coarse;
      }
      s_new = n_new;
    }
  }
  __syncthreads();
  if (!build) return;
  const int tot = s_new * NP;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int a = idx / NP, n = idx - a * NP;
    if (Whi)
      operand_f16x2_elem(idx, a, n, act_out, W64, N, fine, Whi, Wlo);
    else
      operand_f32_elem(idx, a, n, act_out, W64, N, W32);
  }
}

// G_out[a][n] = slot_sum(...) and s4_out[a] (fixed slot order), one block per (row, 32
// coordinates): 8 slot lanes load and part-sum the slots in parallel into shared memory, then
// one thread per coordinate adds them in slot order (few active rows: the serial chain over
// S x P partials of one thread was latency-bound)
constexpr int kRedSlots = 128;
__global__ void __launch_bounds__(256) k_slot_reduce(SlotPartials Gp, const double* __restrict__ s4p, int S,
                                                     int64_t cap, int ldg, int L, int N, double* __restrict__ G_out,
                                                     int ldo, double* __restrict__ s4_out, const int* __restrict__ cnt) {
  __shared__ double T[kRedSlots][33];
  const int a = blockIdx.x;
  // rows beyond the device count hold no partials (and split-part buffers have only sub_cap rows)
  if (cnt && a >= cnt[0]) return;   // block-uniform
  const int nl = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int n = blockIdx.y * 32 + nl;
  const bool g_col = n < N, s4_col = n == N && s4p && s4_out;
  const int P = parts_of(Gp, S);
  double acc = 0.0;
  for (int s0 = 0; s0 < S; s0 += kRedSlots) {
    const int ns = min(kRedSlots, S - s0);
    for (int j = sl; j < ns; j += 8) {
      double v = 0.0;
      if (g_col)
        v = slot_part(Gp, P, s0 + j, cap, ldg, a, n);
      else if (s4_col)
        v = __ldg(s4p + (int64_t)(s0 + j) * cap + a);
      T[j][nl] = v;
    }
    __syncthreads();
    if (sl == 0)
      for (int j = 0; j < ns; ++j) acc += T[j][nl];
    __syncthreads();
  }
  if (sl == 0) {
    if (g_col) G_out[(int64_t)a * ldo + n] = acc;
    if (s4_col) s4_out[a] = acc;
  }
}

// s4 = w_e . G_raw (identity sum_m y^3 (w_e.x) = sum_m y^4), rows by position; one warp per row.
__global__ void k_s4_from_g(EvalPoint ev, const double* __restrict__ W, const double* __restrict__ G, int ldg, int L,
                            int N, double* __restrict__ s4) {
  int a = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int lane = threadIdx.x & 31;
  if (a >= L) return;
  double v = 0.0;
  for (int n = lane; n < N; n += 32) v += eval_coord(ev, a, n, W[(int64_t)a * N + n]) * G[(int64_t)a * ldg + n];
  v = warp_sum(v);
  if (lane == 0) s4[a] = v;
}

}  // namespace

int launch_cand_init(cudaStream_t st, uint64_t seed, int i, int64_t id_base, int64_t L_local, int N,
                     const double* Wacc, int k, double* W64, uint8_t* state, uint8_t* keep, uint8_t* fine,
                     uint8_t fine_init, double* dprev) {
  int64_t threads = L_local * 32;
  k_cand_init<<<(unsigned)ceil_div(threads, 256), 256, 0, st>>>(seed, i, id_base, L_local, N, Wacc, k, W64, state, keep,
                                                                fine, fine_init, dprev);
  return 1;
}

int launch_epilogue(cudaStream_t st, SlotPartials Gp, const double* s4p, int S, int64_t cap, int ldg, EvalPoint ev,
                    const int* act, int L_act, const double* Wacc, int k, int N, double M, double tol, int t,
                    double* W64, double* alpha_old, int* iters, uint8_t* state, uint8_t* keep, Promotion pr,
                    const int* cnt) {
  if (L_act <= 0) return 0;
  int64_t threads = (int64_t)L_act * 32;
  // coordinates per lane: only as many as N needs (bitwise the same as the 8-wide loop)
  auto kern = N <= 32 ? k_epilogue<1> : N <= 64 ? k_epilogue<2> : N <= 128 ? k_epilogue<4> : k_epilogue<kMaxV>;
  kern<<<(unsigned)ceil_div(threads, 256), 256, 0, st>>>(Gp, s4p, S, cap, ldg, ev, act, L_act, Wacc, k, N, M, tol, t,
                                                         W64, alpha_old, iters, state, keep, pr, cnt);
  return 1;
}

int launch_iter_small(cudaStream_t st, SlotPartials Gp, const double* s4p, int S, int64_t cap, int ldg, EvalPoint ev,
                      const int* act, int L_ub, const double* Wacc, int k, int N, double M, double tol, int t,
                      double* W64, double* alpha_old, int* iters, uint8_t* state, uint8_t* keep, Promotion pr,
                      int* cnt, const uint8_t* fine, int* act_out, int* host_mapped, int* hist, bool build, int NP,
                      __half* Whi, __half* Wlo, float* W32) {
  if (L_ub <= 0) return 0;
  auto kern = N <= 32 ? k_iter_small<1> : N <= 64 ? k_iter_small<2> : N <= 128 ? k_iter_small<4> : k_iter_small<kMaxV>;
  kern<<<1, 1024, 0, st>>>(Gp, s4p, S, cap, ldg, ev, act, L_ub, Wacc, k, N, M, tol, t, W64, alpha_old, iters, state,
                           keep, pr, cnt, fine, act_out, host_mapped, hist, build ? 1 : 0, NP, Whi, Wlo, W32);
  return 1;
}

int launch_compact(cudaStream_t st, const int* act_in, const uint8_t* keep, const uint8_t* fine, int L_in,
                   int* act_out, int* out_dev, int* host_mapped, const int* cnt_in, int* hist) {
  k_compact<<<1, 1024, 0, st>>>(act_in, keep, fine, L_in, act_out, out_dev, host_mapped, cnt_in, hist);
  return 1;
}

int launch_operand_f32(cudaStream_t st, const int* act, const int* Lact, int cap, const double* W64, int N, int NP,
                       float* W32) {
  if (cap <= 0) return 0;
  int64_t tot = (int64_t)cap * NP;
  k_operand_f32<<<(unsigned)ceil_div(tot, 256), 256, 0, st>>>(act, Lact, cap, W64, N, NP, W32);
  return 1;
}

int launch_operand_f16x2(cudaStream_t st, const int* act, const int* Lact, int cap, const double* W64, int N, int NP,
                         const uint8_t* fine, __half* Whi, __half* Wlo) {
  if (cap <= 0) return 0;
  int64_t tot = (int64_t)cap * NP;
  k_operand_f16x2<<<(unsigned)ceil_div(tot, 256), 256, 0, st>>>(act, Lact, cap, W64, N, NP, fine, Whi, Wlo);
  return 1;
}

int launch_slot_reduce(cudaStream_t st, SlotPartials Gp, const double* s4p, int S, int64_t cap, int ldg, int L,
                       int N, double* G_out, int ldo, double* s4_out, const int* cnt) {
  if (L <= 0) return 0;
  const int cols = N + (s4p && s4_out ? 1 : 0);   // coordinates (+ the s4 column when there is one)
  k_slot_reduce<<<dim3((unsigned)L, (unsigned)ceil_div(cols, 32)), 256, 0, st>>>(Gp, s4p, S, cap, ldg, L, N, G_out,
                                                                                ldo, s4_out, cnt);
  return 1;
}

// alpha_old[act[a]] = s4[a] / M - 3 for the runs still active at the cap (rows by position)
__global__ void k_alpha_refresh(const int* __restrict__ act, const int* __restrict__ cnt, int L_ub,
                                const double* __restrict__ s4, double M, double* __restrict__ alpha_old) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= min(L_ub, cnt[0])) return;
  alpha_old[act[a]] = s4[a] / M - 3.0;   // eq. (2) at the final w
}

int launch_alpha_refresh(cudaStream_t st, const int* act, const int* cnt, int L_ub, const double* s4, double M,
                         double* alpha_old) {
  if (L_ub <= 0) return 0;
  k_alpha_refresh<<<(unsigned)ceil_div(L_ub, 256), 256, 0, st>>>(act, cnt, L_ub, s4, M, alpha_old);
  return 1;
}

int launch_s4_from_g(cudaStream_t st, EvalPoint ev, const double* W, const double* G, int ldg, int L, int N,
                     double* s4) {
  if (L <= 0) return 0;
  k_s4_from_g<<<(unsigned)ceil_div((int64_t)L * 32, 256), 256, 0, st>>>(ev, W, G, ldg, L, N, s4);
  return 1;
}

}  // namespace oica
