// K2b: fused GEMM-cube-GEMM on CUDA cores (FP32 FFMA).
//
// For the active rows w_a (fp32 operand, a < L_act) and one split-M slot s, computes
//   Gp[s][a][n] = sum_{m in slot s} y_am^3 x_nm,   s4p[s][a] = sum_{m in slot s} y_am^4,
//   y_am = sum_n w_an x_nm                                  (eq. (4)-(5))
// without materialising Y: each CTA keeps a 64-row W tile on chip, streams X through shared
// memory in 64-sample chunks, and accumulates G in fp32 registers for `flush` samples before
// adding the partial into its private fp64 slot (no atomics: bitwise deterministic, and the
// result for a row does not depend on which other rows share its tile).
#include "kernels.cuh"
#include "simt_unit.cuh"

namespace oica {
namespace {

using namespace simt;

template <int NP>
__global__ void __launch_bounds__(256, 1)
k_step_simt(const float* __restrict__ X, int64_t ld, int64_t M, int N, const float* __restrict__ W32,
            const int* __restrict__ act, int L_ub,
            int64_t slot_len, int flush, double* __restrict__ Gp, double* __restrict__ s4p, int64_t cap,
            const int* __restrict__ cnt) {
  const int L_act = cnt ? min(L_ub, cnt[0]) : L_ub;   // device count when the grid is an upper bound
  if ((int)(blockIdx.x * R) >= L_act) return;
  extern __shared__ float smem[];
  simt_step_unit<NP>(X, ld, M, N, W32, act, L_act, slot_len, flush, Gp, s4p, cap, blockIdx.x, blockIdx.y, smem);
}

template <int NP>
void launch_np(cudaStream_t st, const float* X, int64_t ld, int64_t M, int N, const float* W32, const int* act, int L_act,
               int64_t slot_len, int S, int flush, double* Gp, double* s4p, int64_t cap, const int* cnt) {
  const size_t smem = unit_smem_bytes<NP>();
  static bool attr = false;
  if (!attr) {
    OICA_CUDA(cudaFuncSetAttribute(k_step_simt<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  dim3 grid((unsigned)ceil_div(L_act, R), (unsigned)S);
  k_step_simt<NP><<<grid, 256, smem, st>>>(X, ld, M, N, W32, act, L_act, slot_len, flush, Gp, s4p, cap, cnt);
}

}  // namespace

int launch_step_simt(cudaStream_t st, const float* X, int64_t ld, int64_t M, int N, int NP, const float* W32,
                     const int* act, int L_act, int64_t slot_len, int S, int flush, double* Gp, double* s4p, int64_t cap,
                     const int* cnt) {
  if (L_act <= 0) return 0;
  switch (NP) {
    case 32: launch_np<32>(st, X, ld, M, N, W32, act, L_act, slot_len, S, flush, Gp, s4p, cap, cnt); break;
    case 64: launch_np<64>(st, X, ld, M, N, W32, act, L_act, slot_len, S, flush, Gp, s4p, cap, cnt); break;
    case 128: launch_np<128>(st, X, ld, M, N, W32, act, L_act, slot_len, S, flush, Gp, s4p, cap, cnt); break;
    case 256: launch_np<256>(st, X, ld, M, N, W32, act, L_act, slot_len, S, flush, Gp, s4p, cap, cnt); break;
    default: throw Error(OICA_ERR_INVALID_ARGUMENT, "unsupported padded N for the SIMT step");
  }
  return 1;
}

}  // namespace oica
