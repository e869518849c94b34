// Persistent do-while for tiny FP32 problems (DESIGN.md §5 "iteration"): the paper's own experiment
// sizes (N = 20-30, M = 1e4, L <= 100, K = 30) do a few MFLOP per iteration, so an
// iteration costs what its launches and dependent memory round trips cost.  Here the whole loop of
// PAPER.md:241-256 for one component is ONE cooperative launch: per iteration
//   the FP32 step's (row tile, slot) units spread over the blocks   (K2b, simt_unit.cuh)
//   grid barrier
//   the few-row update of every active row (K3, update_core.cuh update_pass)
//   grid barrier
//   compaction + end of the iteration by block 0 (K4, compact_block / finish_iteration)
//   grid barrier
// until no run is active or t > K.  The device functions are the ones k_step_simt and k_update run,
// so the result is bitwise that of the other loops (tests/test_gpu_parity.py::test_device_loop_bitwise).
#include <cooperative_groups.h>

#include <algorithm>
#include <type_traits>

#include "kernels.cuh"
#include "simt_unit.cuh"
#include "update_core.cuh"

namespace oica {
namespace {

namespace cg = cooperative_groups;

struct LoopSimtArgs {
  const float* X;
  int64_t ld;
  int64_t M;
  int64_t slot_len;
  int S;
  int flush;
  int K;
  int coop_update;   // block-per-row updates through shared memory (S * (NP + 1) doubles <= 96 KB)
  UpdateArgs u;      // G = the fp64 slot partials (S x cap x NP), s4p, act_in (kept in place), ctl, ...
};

template <int NP, int NG>
__global__ void __launch_bounds__(256, 2) k_loop_simt(LoopSimtArgs a) {
  constexpr int RPB = 8 / NG;
  __shared__ double gsh[RPB][NG * 32];
  __shared__ double s4sh[RPB];
  __shared__ int s_keep[RPB];
  extern __shared__ float smem[];   // the step unit's tiles
  cg::grid_group grid = cg::this_grid();
  const UpdateArgs& u = a.u;
  double* Gp = (double*)u.G.p;
  double* s4p = const_cast<double*>(u.s4p);
#ifdef OICA_DEBUG_CHECKS
  unsigned long long ph[4] = {0, 0, 0, 0}, tp;
  auto tick = [&](int i) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (i >= 0) ph[i] += now - tp;
    tp = now;
  };
  tick(-1);
  int iters = 0;
#define OICA_TICK(i) tick(i)
#else
#define OICA_TICK(i)
#endif
  for (;;) {
    const int L_act = min(u.L_ub, u.cnt_in[0]);
    const int t = u.ctl->t, k = u.ctl->k;
    if (L_act <= 0 || t > a.K) break;   // the same values in every block (read after a barrier)
#ifdef OICA_DEBUG_CHECKS
    ++iters;
#endif
    // K2b: G, s4 slot partials of the active rows (operand rows by candidate id through act_in);
    // row tiles of 16 / 32 / 64 rows as few rows remain (a row's arithmetic is the same for any)
    auto step_units = [&](auto RTc) {
      constexpr int RT = decltype(RTc)::value;
      const int tiles = (L_act + RT - 1) / RT;
      for (int unit = blockIdx.x; unit < tiles * a.S; unit += gridDim.x)
        simt::simt_step_unit<NP, RT>(a.X, a.ld, a.M, u.N, u.ev.f32, u.act_in, L_act, a.slot_len, a.flush, Gp, s4p,
                                     u.cap, unit % tiles, unit / tiles, smem);
    };
    if (L_act <= 16)
      step_units(std::integral_constant<int, 16>{});
    else if (L_act <= 32)
      step_units(std::integral_constant<int, 32>{});
    else
      step_units(std::integral_constant<int, 64>{});
    OICA_TICK(0);
    grid.sync();
    OICA_TICK(3);
    // K3: every active row (fixed-order slot sums, eq. (5), projection, convergence, operand row):
    // one row per block while there are blocks to spare (the block's warps load its slot partials
    // in parallel into the step's shared memory), else the warp-group passes of k_update
    if (a.coop_update && L_act <= (int)gridDim.x) {
      if ((int)blockIdx.x < L_act)
        upd::update_row_coop<NG, true>(u, blockIdx.x, L_act, t, k, (double*)smem, gsh, s4sh);
    } else {
      for (int a0 = blockIdx.x * RPB; a0 < L_act; a0 += gridDim.x * RPB) {
        upd::update_pass<NG, false, RPB>(u, a0, L_act, t, k, gsh, s4sh, s_keep, true);
        __syncthreads();   // gsh / s_keep are rewritten by the block's next pass
      }
    }
    OICA_TICK(1);
    grid.sync();
    OICA_TICK(3);
    // K4 + end of the iteration (counts, history, t)
    if (blockIdx.x == 0) {
      const int2 r = upd::compact_block(u.act_in, u.keep, u.pr.fine, L_act, u.act_out);
      int* dst = const_cast<int*>(u.act_in);
      for (int j = threadIdx.x; j < r.x; j += blockDim.x) dst[j] = u.act_out[j];
      if (threadIdx.x == 0) upd::finish_iteration(u, r, L_act, t);
    }
    OICA_TICK(2);
    grid.sync();
    OICA_TICK(3);
  }
#ifdef OICA_DEBUG_CHECKS
  if (blockIdx.x == 0 && threadIdx.x == 0 && iters > 0)
    printf("oica debug: persistent loop %d iterations, per iteration: step %.2f us, update %.2f us, compact %.2f us, "
           "barriers %.2f us (block 0, grid %d)\n", iters, ph[0] * 1e-3 / iters, ph[1] * 1e-3 / iters,
           ph[2] * 1e-3 / iters, ph[3] * 1e-3 / iters, gridDim.x);
#endif
#undef OICA_TICK
}

template <int NP, int NG>
int launch_np(cudaStream_t st, const LoopSimtArgs& a, int num_sms) {
  auto kern = k_loop_simt<NP, NG>;
  // the step unit's tiles, reused by the block-per-row update for the S x NP slot partials of a row
  // (+ S doubles: the row's sum-y^4 slot partials, update_row_coop<NG, true>)
  const size_t smem =
      std::max(simt::unit_smem_bytes<NP>(), a.coop_update ? (size_t)a.S * (NP + 1) * sizeof(double) : 0);
  static size_t attr = 0;
  if (smem > attr) {
    OICA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  int per_sm = 0;
  OICA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
  OICA_REQUIRE(per_sm >= 1, OICA_ERR_CUDA, "persistent loop kernel does not fit on an SM");
  // as many blocks as there is work at the first iteration, all co-resident (cooperative launch)
  const int tiles = (int)ceil_div(a.u.L_ub, simt::R);
  const int work = std::max(tiles * a.S, (int)ceil_div(a.u.L_ub, 8 / NG));
  const int grid = std::max(1, std::min(work, per_sm * num_sms));
  LoopSimtArgs args = a;
  void* params[] = {&args};
  OICA_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(256), params, smem, st));
  return 1;
}

}  // namespace

int launch_loop_simt(cudaStream_t st, const float* X, int64_t ld, int64_t M, int64_t slot_len, int S, int flush,
                     int K, const UpdateArgs& u, int NP, int num_sms) {
  LoopSimtArgs a{X, ld, M, slot_len, S, flush, K, 0, u};
  switch (NP) {
    case 32:
      a.coop_update = (size_t)S * (32 + 1) * sizeof(double) <= 96 * 1024 ? 1 : 0;
      return launch_np<32, 1>(st, a, num_sms);
    case 64:
      a.coop_update = (size_t)S * (64 + 1) * sizeof(double) <= 96 * 1024 ? 1 : 0;
      return launch_np<64, 2>(st, a, num_sms);
    default: throw Error(OICA_ERR_INVALID_ARGUMENT, "persistent FP32 loop: padded N must be 32 or 64");
  }
}

}  // namespace oica
