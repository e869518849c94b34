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

namespace oica {
namespace {

constexpr int R = 64;        // rows per CTA
constexpr int MC = 64;       // samples per chunk
constexpr int XS = MC + 1;   // padded X row stride (conflict-free column reads)
constexpr int YS = R + 1;    // padded Y^3 row stride

template <int NP>
__global__ void __launch_bounds__(256, 1)
k_step_simt(const float* __restrict__ X, int64_t ld, int64_t M, int N, const float* __restrict__ W32,
            const int* __restrict__ act, int L_ub,
            int64_t slot_len, int flush, double* __restrict__ Gp, double* __restrict__ s4p, int64_t cap,
            const int* __restrict__ cnt) {
  const int L_act = cnt ? min(L_ub, cnt[0]) : L_ub;   // device count when the grid is an upper bound
  if ((int)(blockIdx.x * R) >= L_act) return;
  constexpr int TN = NP / 32;
  extern __shared__ float smem[];
  float* WT = smem;                 // [NP][R]   W tile, transposed
  float* Xs = WT + NP * R;          // [NP][XS]  X chunk
  float* Y3 = Xs + NP * XS;         // [MC][YS]  y^3 chunk
  float* S4 = Y3 + MC * YS;         // [16][R]   s4 partials for the fixed-order reduction

  const int tid = threadIdx.x;
  const int row0 = blockIdx.x * R;
  const int s = blockIdx.y;
  const int64_t m_begin = (int64_t)s * slot_len;
  const int64_t m_end = min(M, m_begin + slot_len);

  for (int idx = tid; idx < R * NP; idx += 256) {
    int r = idx / NP, n = idx % NP;
    WT[n * R + r] = (row0 + r < L_act) ? W32[(int64_t)act[row0 + r] * NP + n] : 0.f;   // operand row by id
  }

  const int rg = tid >> 4, cg = tid & 15;     // phase 1: rows rg*4+i, cols cg+16j
  const int rg2 = tid >> 5, ng = tid & 31;    // phase 2: rows rg2*8+i, n = ng+32k
  float acc[8][TN];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int k = 0; k < TN; ++k) acc[i][k] = 0.f;
  float s4a[4] = {0.f, 0.f, 0.f, 0.f};
  bool first = true;
  int since = 0;

  for (int64_t m0 = m_begin; m0 < m_end; m0 += MC) {
    __syncthreads();
    for (int idx = tid; idx < NP * MC; idx += 256) {
      int n = idx / MC, j = idx % MC;
      int64_t m = m0 + j;
      Xs[n * XS + j] = (n < N && m < m_end) ? __ldg(X + (int64_t)n * ld + m) : 0.f;
    }
    __syncthreads();
    // phase 1: y = W x (fixed n order per output)
    float y[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) y[i][j] = 0.f;
#pragma unroll 4
    for (int n = 0; n < NP; ++n) {
      float4 w4 = *reinterpret_cast<const float4*>(&WT[n * R + rg * 4]);
      float xv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) xv[j] = Xs[n * XS + cg + 16 * j];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        y[0][j] = fmaf(w4.x, xv[j], y[0][j]);
        y[1][j] = fmaf(w4.y, xv[j], y[1][j]);
        y[2][j] = fmaf(w4.z, xv[j], y[2][j]);
        y[3][j] = fmaf(w4.w, xv[j], y[3][j]);
      }
    }
    // cube and fourth power (eq. (2))
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float y2 = y[i][j] * y[i][j];
        s4a[i] = fmaf(y2, y2, s4a[i]);
        Y3[(cg + 16 * j) * YS + rg * 4 + i] = y2 * y[i][j];
      }
    __syncthreads();
    // phase 2: G += y^3 x^T (fixed m order per output)
#pragma unroll 2
    for (int j = 0; j < MC; ++j) {
      float a[8], xv[TN];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = Y3[j * YS + rg2 * 8 + i];
#pragma unroll
      for (int k = 0; k < TN; ++k) xv[k] = Xs[(ng + 32 * k) * XS + j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int k = 0; k < TN; ++k) acc[i][k] = fmaf(a[i], xv[k], acc[i][k]);
    }
    since += MC;
    if (since >= flush || m0 + MC >= m_end) {
      // flush fp32 partials into this CTA's private fp64 slot, fixed order
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int a = row0 + rg2 * 8 + i;
        if (a < L_act) {
#pragma unroll
          for (int k = 0; k < TN; ++k) {
            int n = ng + 32 * k;
            if (n < N) {
              double* p = Gp + ((int64_t)s * cap + a) * NP + n;
              *p = (first ? 0.0 : *p) + (double)acc[i][k];
            }
          }
        }
#pragma unroll
        for (int k = 0; k < TN; ++k) acc[i][k] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        S4[cg * R + rg * 4 + i] = s4a[i];
        s4a[i] = 0.f;
      }
      __syncthreads();
      if (tid < R && row0 + tid < L_act) {
        double v = 0.0;
        for (int c = 0; c < 16; ++c) v += (double)S4[c * R + tid];
        double* p = s4p + (int64_t)s * cap + row0 + tid;
        *p = (first ? 0.0 : *p) + v;
      }
      first = false;
      since = 0;
    }
  }
}

template <int NP>
void launch_np(cudaStream_t st, const float* X, int64_t ld, int64_t M, int N, const float* W32, const int* act, int L_act,
               int64_t slot_len, int S, int flush, double* Gp, double* s4p, int64_t cap, const int* cnt) {
  size_t smem = sizeof(float) * ((size_t)NP * R + (size_t)NP * XS + (size_t)MC * YS + 16 * R);
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
