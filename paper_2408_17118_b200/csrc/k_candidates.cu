// K1 candidate init, K3 fp64 epilogue, K4 compaction and operand gathers.
// One warp per candidate row for the fp64 row work (N <= 256 -> <= 8 values per lane).
#include <cuda_fp16.h>

#include <algorithm>

#include <atomic>

#include "kernels.cuh"
#include "update_core.cuh"

namespace oica {
namespace {

using namespace upd;


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

// K3 + K4 fused (see launch_update).  Block = 16 warps = RPB rows x NG warps: the NG warps of a
// row sum its slot partials, 32 coordinates each, in fixed slot order (the association of every
// consumer of the slot partials: a row's G is bitwise the same whatever path or GPU count reduces
// it), then the row's first warp runs epilogue_core.  Few rows (L_in <= RPB, the tail of every
// component): block 0 alone, compacting in shared memory; otherwise the block that finishes last
// (ticket) compacts.
template <int NG, bool F32>
__global__ void __launch_bounds__(512, 1) k_update(UpdateArgs u) {
  constexpr int RPB = 16 / NG;
  __shared__ double gsh[RPB][NG * 32];
  __shared__ double s4sh[RPB];
  __shared__ int s_keep[RPB];
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (u.gate_in && u.gate_in[0] == 0) return;   // grid-uniform (the writer is this kernel's last block)
  const int t = u.ctl->t, k = u.ctl->k;
  const int L_in = u.cnt_in ? min(u.L_ub, u.cnt_in[0]) : u.L_ub;
  const bool single = L_in <= RPB && u.compact;   // grid-uniform
  if (L_in <= RPB && blockIdx.x != 0) return;
#ifdef OICA_EXPERIMENTS
  long long stamp[8];
  stamp[3] = clock64();
  update_pass<NG, F32, RPB>(u, blockIdx.x * RPB, L_in, t, k, gsh, s4sh, s_keep, !single || !u.compact, stamp);
  stamp[4] = clock64();
#else
  update_pass<NG, F32, RPB>(u, blockIdx.x * RPB, L_in, t, k, gsh, s4sh, s_keep, !single || !u.compact);
#endif
  if (!u.compact) return;   // (k_compact follows)
  int2 r;
  if (single) {   // K4 by one warp: kept coarse rows, then kept fine rows (k_compact's order)
    __syncthreads();
    if (warp == 0) {
      const bool in = lane < L_in && s_keep[lane];
      const int id = lane < L_in ? u.act_in[lane] : 0;
      const bool isf = in && u.pr.fine && u.pr.fine[id];
      const unsigned mc = __ballot_sync(0xffffffffu, in && !isf), mf = __ballot_sync(0xffffffffu, isf);
      const unsigned lt = (1u << lane) - 1u;
      const int n_coarse = __popc(mc);
      const int pos = isf ? n_coarse + __popc(mf & lt) : __popc(mc & lt);
      __syncwarp();
      if (in) {
        u.act_out[pos] = id;
        if (u.copy_back) const_cast<int*>(u.act_in)[pos] = id;   // (all lanes read act_in above)
      }
      r = make_int2(n_coarse + __popc(mf), n_coarse);
    }
  } else {
    // completion ticket: the block that finishes last sees every row's keep / fine / state
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned tk = atomicAdd(&u.ctl->done, 1u);
      s_last = tk == gridDim.x - 1 ? 1 : 0;
    }
    __syncthreads();
    if (!s_last) return;
#ifdef OICA_EXPERIMENTS
    stamp[5] = clock64();
#endif
    __threadfence();
    r = compact_block(u.act_in, u.keep, u.pr.fine, L_in, u.act_out,
                      u.copy_back ? const_cast<int*>(u.act_in) : nullptr);   // K4
  }
#ifdef OICA_EXPERIMENTS
  if (threadIdx.x == 0 && !single) stamp[6] = clock64();
#endif
  if (threadIdx.x == 0) finish_iteration(u, r, L_in, t);
#ifdef OICA_EXPERIMENTS
  // phase cycles of the block that finished last (its own SM clock): entry -> row loads landed ->
  // slot sums stored -> barrier -> epilogue done -> ticket known -> compaction done -> finish
  if (threadIdx.x == 0 && !single && t <= 3 && (k & 7) == 1)
    printf("oica exp: k_update<%d> k %d t %d L_in %d grid %d block %d: rows %lld slots %lld barrier %lld epilogue %lld "
           "ticket %lld compact %lld finish %lld cycles\n", NG, k, t, L_in, (int)gridDim.x, (int)blockIdx.x,
           stamp[0] - stamp[3], stamp[1] - stamp[0], stamp[2] - stamp[1], stamp[4] - stamp[2], stamp[5] - stamp[4],
           stamp[6] - stamp[5], clock64() - stamp[6]);
#endif
}

// K3 + K4 for few rows (L_ub <= kUpdateCoopRows, the tail of a component): one block of 16 warps
// per row, the row's slot values loaded by all warps at once into shared memory and summed in slot
// order (update_row_coop: bitwise k_update's G -- in k_update the row's NG warps walk the S
// slots x P split parts themselves, a chain of S/2 dependent L2 round trips per row), then the
// block that finishes last compacts.
template <int NG>
__global__ void __launch_bounds__(512) k_update_coop(UpdateArgs u) {
  extern __shared__ double T[];   // [S][NG * 32]
  __shared__ double gsh[1][NG * 32];
  __shared__ double s4sh[1];
  __shared__ int s_last;
  if (u.gate_in && u.gate_in[0] == 0) return;   // grid-uniform (the writer is this kernel's last block)
  const int t = u.ctl->t, k = u.ctl->k;
  const int L_in = u.cnt_in ? min(u.L_ub, u.cnt_in[0]) : u.L_ub;
  upd::update_row_coop<NG>(u, blockIdx.x, L_in, t, k, T, gsh, s4sh);
  if (threadIdx.x == 0) {   // completion ticket: the last block sees every row's keep / fine / state
    __threadfence();
    const unsigned tk = atomicAdd(&u.ctl->done, 1u);
    s_last = tk == gridDim.x - 1 ? 1 : 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int2 r = compact_block(u.act_in, u.keep, u.pr.fine, L_in, u.act_out);   // K4
  if (u.copy_back) {
    int* dst = const_cast<int*>(u.act_in);
    for (int j = threadIdx.x; j < r.x; j += blockDim.x) dst[j] = u.act_out[j];
  }
  if (threadIdx.x == 0) finish_iteration(u, r, L_in, t);
}

// K3 for many rows (L_ub > kUpdateCompactRows: the HBM-bound regime, where occupancy and not the
// latency of one row matters): one warp per row with V coordinates per lane (slot sums in the same
// sequential order as k_update), 8 rows per block; keep[] for k_compact_iter.
template <int V, bool F32>
__global__ void __launch_bounds__(256) k_update_rows(UpdateArgs u) {
  const int a = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (u.gate_in && u.gate_in[0] == 0) return;
  const int t = u.ctl->t, k = u.ctl->k;
  const int L_in = u.cnt_in ? min(u.L_ub, u.cnt_in[0]) : u.L_ub;
  if (a >= L_in) return;
  const int l = u.act_in[a];
  double wo[V], we[V], acc[V];
  load_row<V>(u, l, lane, wo, we);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int n = lane + 32 * v;
    acc[v] = n < u.N ? slot_sum<(V >= 8 ? 2 : 8 / V), (F32 ? 2 : 1)>(u.G, u.S, u.cap, u.ldg, a, n) : 0.0;
  }
  double s4 = 0.0;
  if (u.s4p && lane == 0) s4 = ordered_sum(u.S, [&](int s) { return __ldg(u.s4p + (int64_t)s * u.cap + a); });
  const bool kp = epilogue_core<V>(l, lane, acc, s4, wo, we, u, k, t);
  if (lane == 0) u.keep[a] = kp ? 1 : 0;
}

// K4 for many rows after launch_update with compact = 0: one 1024-thread block scans the list
// (k_compact's arithmetic) and ends the iteration like the update's last block would.
__global__ void __launch_bounds__(1024) k_compact_iter(UpdateArgs u) {
  if (u.gate_in && u.gate_in[0] == 0) return;   // (read by every thread before the barrier below)
  const int t = u.ctl->t;
  const int L_in = u.cnt_in ? min(u.L_ub, u.cnt_in[0]) : u.L_ub;
  __syncthreads();   // every thread read cnt_in (may alias cnt_out) before thread 0 writes it
  const int2 r = compact_block(u.act_in, u.keep, u.pr.fine, L_in, u.act_out);
  if (u.copy_back) {
    int* dst = const_cast<int*>(u.act_in);
    for (int j = threadIdx.x; j < r.x; j += blockDim.x) dst[j] = u.act_out[j];
  }
  if (threadIdx.x == 0) finish_iteration(u, r, L_in, t);
}

// First node of the device-side loop graph: the first WHILE node starts only if runs are active
// and t <= K (a pipelined upload may have run iteration 1 already: with K = 1 nothing is left)
__global__ void k_loop_gate(cudaGraphConditionalHandle h, const int* __restrict__ cnt, const IterCtl* __restrict__ ctl,
                            int K) {
  cudaGraphSetConditional(h, (cnt[0] > 0 && ctl->t <= K) ? 1u : 0u);
}

__global__ void k_ctl_set(IterCtl* ctl, int t, int k) {
  ctl->t = t;
  ctl->k = k;
  ctl->done = 0u;
  ctl->sum_active = 0;
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

// operand rows 0..L-1 by candidate id from the fp64 master
__global__ void k_operand_f32(int L, const double* __restrict__ W64, int N, int NP, float* __restrict__ W32) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)L * NP) return;
  int l = (int)(idx / NP), n = (int)(idx % NP);
  W32[idx] = n < N ? (float)W64[(int64_t)l * N + n] : 0.f;
}

__global__ void k_operand_f16x2(int L, const double* __restrict__ W64, int N, int NP, const uint8_t* __restrict__ fine,
                                __half* __restrict__ Whi, __half* __restrict__ Wlo) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)L * NP) return;
  int l = (int)(idx / NP), n = (int)(idx % NP);
  operand_f16x2_coord(n < N ? W64[(int64_t)l * N + n] : 0.0, !fine || fine[l], Whi + idx, Wlo ? Wlo + idx : nullptr);
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

// s4 = w_e . G_raw (identity sum_m y^3 (w_e.x) = sum_m y^4), G rows by position; the evaluation
// point of position a is candidate act[a] (identity if act is null); one warp per row.
__global__ void k_s4_from_g(EvalPoint ev, const int* __restrict__ act, const double* __restrict__ G, int ldg, int L,
                            int N, double* __restrict__ s4, const int* __restrict__ cnt) {
  int a = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int lane = threadIdx.x & 31;
  if (a >= L || (cnt && a >= cnt[0])) return;
  const int l = act ? act[a] : a;
  double v = 0.0;
  for (int n = lane; n < N; n += 32) v += eval_coord(ev, l, n, 0.0) * G[(int64_t)a * ldg + n];
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

int update_blocks(int L_ub, int NP) {
  const int NG = (NP + 31) / 32, RPB = 16 / NG;
  return (int)ceil_div(std::max(L_ub, 1), RPB);
}

int launch_update(cudaStream_t st, const UpdateArgs& u, int NP) {
  if (u.L_ub <= 0) return 0;
  const int NG = (NP + 31) / 32;
  if (!u.compact) {   // many rows: warp per row (k_compact_iter compacts)
    const unsigned nbr = (unsigned)ceil_div((int64_t)u.L_ub * 32, 256);
    const bool f = u.G.f32;
    if (NG <= 1)
      f ? k_update_rows<1, true><<<nbr, 256, 0, st>>>(u) : k_update_rows<1, false><<<nbr, 256, 0, st>>>(u);
    else if (NG <= 2)
      f ? k_update_rows<2, true><<<nbr, 256, 0, st>>>(u) : k_update_rows<2, false><<<nbr, 256, 0, st>>>(u);
    else if (NG <= 4)
      f ? k_update_rows<4, true><<<nbr, 256, 0, st>>>(u) : k_update_rows<4, false><<<nbr, 256, 0, st>>>(u);
    else
      f ? k_update_rows<8, true><<<nbr, 256, 0, st>>>(u) : k_update_rows<8, false><<<nbr, 256, 0, st>>>(u);
    return 1;
  }
  const size_t coop_smem = sizeof(double) * (size_t)u.S * (size_t)NG * 32;
  if (u.L_ub <= kUpdateCoopRows && coop_smem <= kUpdateCoopSmem) {   // few rows: one block per row
    // the shared-memory opt-in is a per-device function attribute: set once per (device, NG)
    static std::atomic<uint64_t> attr_set[9];
    int dev = 0;
    OICA_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
#define OICA_UPDC(g)                                                                             \
  case g:                                                                                        \
    if (!(attr_set[g].load() & bit)) {                                                           \
      OICA_CUDA(cudaFuncSetAttribute(k_update_coop<g>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     (int)kUpdateCoopSmem));                                     \
      attr_set[g].fetch_or(bit);                                                                 \
    }                                                                                            \
    k_update_coop<g><<<(unsigned)u.L_ub, 512, coop_smem, st>>>(u);                              \
    break;
    switch (NG) {
      OICA_UPDC(1)
      OICA_UPDC(2)
      OICA_UPDC(3)
      OICA_UPDC(4)
      OICA_UPDC(5)
      OICA_UPDC(6)
      OICA_UPDC(7)
      OICA_UPDC(8)
      default: throw Error(OICA_ERR_INVALID_ARGUMENT, "unsupported padded N for the update");
    }
#undef OICA_UPDC
    return 1;
  }
  const unsigned nb = (unsigned)update_blocks(u.L_ub, NP);
  // fp32 slot partials (tensor-core step, split parts possible) or fp64 (FP32 step, reduced sums)
  const bool f32 = u.G.f32;
#define OICA_UPD(g)                                                          \
  case g:                                                                    \
    if (f32)                                                                 \
      k_update<g, true><<<nb, 512, 0, st>>>(u);                              \
    else                                                                     \
      k_update<g, false><<<nb, 512, 0, st>>>(u);                             \
    break;
  switch (NG) {
    OICA_UPD(1)
    OICA_UPD(2)
    OICA_UPD(3)
    OICA_UPD(4)
    OICA_UPD(5)
    OICA_UPD(6)
    OICA_UPD(7)
    OICA_UPD(8)
    default: throw Error(OICA_ERR_INVALID_ARGUMENT, "unsupported padded N for the update");
  }
#undef OICA_UPD
  return 1;
}

int launch_compact_iter(cudaStream_t st, const UpdateArgs& u) {
  if (u.L_ub <= 0) return 0;
  k_compact_iter<<<1, 1024, 0, st>>>(u);
  return 1;
}

void add_loop_gate_node(cudaGraph_t g, cudaGraphNode_t* node, cudaGraphConditionalHandle h, const int* cnt,
                        const IterCtl* ctl, int K) {
  void* args[] = {(void*)&h, (void*)&cnt, (void*)&ctl, (void*)&K};
  cudaKernelNodeParams kp{};
  kp.func = (void*)k_loop_gate;
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(1);
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  OICA_CUDA(cudaGraphAddKernelNode(node, g, nullptr, 0, &kp));
}

int launch_ctl_set(cudaStream_t st, IterCtl* ctl, int t, int k) {
  k_ctl_set<<<1, 1, 0, st>>>(ctl, t, k);
  return 1;
}

int launch_compact(cudaStream_t st, const int* act_in, const uint8_t* keep, const uint8_t* fine, int L_in,
                   int* act_out, int* out_dev, int* host_mapped, const int* cnt_in, int* hist) {
  k_compact<<<1, 1024, 0, st>>>(act_in, keep, fine, L_in, act_out, out_dev, host_mapped, cnt_in, hist);
  return 1;
}

int launch_operand_f32(cudaStream_t st, int L, const double* W64, int N, int NP, float* W32) {
  if (L <= 0) return 0;
  int64_t tot = (int64_t)L * NP;
  k_operand_f32<<<(unsigned)ceil_div(tot, 256), 256, 0, st>>>(L, W64, N, NP, W32);
  return 1;
}

int launch_operand_f16x2(cudaStream_t st, int L, const double* W64, int N, int NP, const uint8_t* fine, __half* Whi,
                         __half* Wlo) {
  if (L <= 0) return 0;
  int64_t tot = (int64_t)L * NP;
  k_operand_f16x2<<<(unsigned)ceil_div(tot, 256), 256, 0, st>>>(L, W64, N, NP, fine, Whi, Wlo);
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

int launch_s4_from_g(cudaStream_t st, EvalPoint ev, const int* act, const double* G, int ldg, int L, int N,
                     double* s4, const int* cnt) {
  if (L <= 0) return 0;
  k_s4_from_g<<<(unsigned)ceil_div((int64_t)L * 32, 256), 256, 0, st>>>(ev, act, G, ldg, L, N, s4, cnt);
  return 1;
}

}  // namespace oica
