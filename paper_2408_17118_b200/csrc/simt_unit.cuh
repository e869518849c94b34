// The FP32 step's work unit (K2b), shared by k_step_simt and the persistent
// small-problem loop (k_loop_simt.cu): ONE definition of the FP32 contraction's arithmetic.
// Internal.
#pragma once
#include "kernels.cuh"

namespace oica {
namespace simt {

constexpr int R = 64;        // rows per CTA
constexpr int MC = 64;       // samples per chunk
constexpr int XS = MC + 1;   // padded X row stride (conflict-free column reads)
constexpr int YS = R + 1;    // padded Y^3 row stride

// dynamic shared memory of one unit with RT-row tiles
template <int NP, int RT = R>
constexpr size_t unit_smem_bytes() {
  return sizeof(float) * ((size_t)NP * RT + (size_t)NP * XS + (size_t)MC * (RT + 1) + 16 * RT);
}

// One work unit of the FP32 step: row tile `tile` (RT active positions: 64, or 32 / 16 for the few
// rows of a persistent loop) x slot s, 256 threads, shared memory unit_smem_bytes<NP, RT>().  A row's
// arithmetic does not depend on RT: y over n, y^3 x over the chunk's samples, the s4 partials over
// the 16 column groups are summed in the same order for every tile height.  The ONE definition of the FP32 contraction's arithmetic:
// k_step_simt and the persistent loop kernel (k_loop_simt.cu) both run it, so a row's slot partial
// is bitwise the same whichever launches it.
template <int NP, int RT = R>
__device__ __forceinline__ void simt_step_unit(const float* __restrict__ X, int64_t ld, int64_t M, int N,
                                               const float* __restrict__ W32, const int* __restrict__ act,
                                               int L_act, int64_t slot_len, int flush, double* __restrict__ Gp,
                                               double* __restrict__ s4p, int64_t cap, int tile, int s, float* smem) {
  constexpr int TN = NP / 32;
  constexpr int P1 = RT / 16;       // phase-1 rows per thread
  constexpr int P2 = RT / 8;        // phase-2 rows per thread
  constexpr int YT = RT + 1;        // padded Y^3 row stride
  float* WT = smem;                 // [NP][RT]  W tile, transposed
  float* Xs = WT + NP * RT;         // [NP][XS]  X chunk
  float* Y3 = Xs + NP * XS;         // [MC][YT]  y^3 chunk
  float* S4 = Y3 + MC * YT;         // [16][RT]  s4 partials for the fixed-order reduction

  const int tid = threadIdx.x;
  const int row0 = tile * RT;
  const int64_t m_begin = (int64_t)s * slot_len;
  const int64_t m_end = min(M, m_begin + slot_len);

  // X chunks are staged through registers one chunk ahead (their loads overlap the W tile load and
  // the previous chunk's arithmetic; the values and every sum are the same as loading in place)
  constexpr int XPT = NP * MC / 256;   // X elements per thread per chunk
  float xr[XPT];
  auto load_x = [&](int64_t m0) {
#pragma unroll
    for (int q = 0; q < XPT; ++q) {
      const int idx = tid + 256 * q;
      const int n = idx / MC, j = idx % MC;
      const int64_t m = m0 + j;
      xr[q] = (n < N && m < m_end) ? __ldg(X + (int64_t)n * ld + m) : 0.f;
    }
  };
  load_x(m_begin);
  for (int idx = tid; idx < RT * NP; idx += 256) {
    int r = idx / NP, n = idx % NP;
    WT[n * RT + r] = (row0 + r < L_act) ? W32[(int64_t)act[row0 + r] * NP + n] : 0.f;   // operand row by id
  }

  const int rg = tid >> 4, cg = tid & 15;     // phase 1: rows rg*P1+i, cols cg+16j
  const int rg2 = tid >> 5, ng = tid & 31;    // phase 2: rows rg2*P2+i, n = ng+32k
  float acc[P2][TN];
#pragma unroll
  for (int i = 0; i < P2; ++i)
#pragma unroll
    for (int k = 0; k < TN; ++k) acc[i][k] = 0.f;
  float s4a[P1];
#pragma unroll
  for (int i = 0; i < P1; ++i) s4a[i] = 0.f;
  bool first = true;
  int since = 0;

  for (int64_t m0 = m_begin; m0 < m_end; m0 += MC) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < XPT; ++q) {
      const int idx = tid + 256 * q;
      Xs[(idx / MC) * XS + idx % MC] = xr[q];
    }
    if (m0 + MC < m_end) load_x(m0 + MC);   // next chunk in flight during this one
    __syncthreads();
    // phase 1: y = W x (fixed n order per output)
    float y[P1][4];
#pragma unroll
    for (int i = 0; i < P1; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) y[i][j] = 0.f;
#pragma unroll 4
    for (int n = 0; n < NP; ++n) {
      float wv[P1];
      if constexpr (P1 == 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(&WT[n * RT + rg * 4]);
        wv[0] = w4.x;
        wv[1] = w4.y;
        wv[2] = w4.z;
        wv[3] = w4.w;
      } else {
#pragma unroll
        for (int i = 0; i < P1; ++i) wv[i] = WT[n * RT + rg * P1 + i];
      }
      float xv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) xv[j] = Xs[n * XS + cg + 16 * j];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < P1; ++i) y[i][j] = fmaf(wv[i], xv[j], y[i][j]);
    }
    // cube and fourth power (eq. (2))
#pragma unroll
    for (int i = 0; i < P1; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float y2 = y[i][j] * y[i][j];
        s4a[i] = fmaf(y2, y2, s4a[i]);
        Y3[(cg + 16 * j) * YT + rg * P1 + i] = y2 * y[i][j];
      }
    __syncthreads();
    // phase 2: G += y^3 x^T (fixed m order per output)
#pragma unroll 2
    for (int j = 0; j < MC; ++j) {
      float a[P2], xv[TN];
#pragma unroll
      for (int i = 0; i < P2; ++i) a[i] = Y3[j * YT + rg2 * P2 + i];
#pragma unroll
      for (int k = 0; k < TN; ++k) xv[k] = Xs[(ng + 32 * k) * XS + j];
#pragma unroll
      for (int i = 0; i < P2; ++i)
#pragma unroll
        for (int k = 0; k < TN; ++k) acc[i][k] = fmaf(a[i], xv[k], acc[i][k]);
    }
    since += MC;
    if (since >= flush || m0 + MC >= m_end) {
      // flush fp32 partials into this CTA's private fp64 slot, fixed order
#pragma unroll
      for (int i = 0; i < P2; ++i) {
        int a = row0 + rg2 * P2 + i;
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
      for (int i = 0; i < P1; ++i) {
        S4[cg * RT + rg * P1 + i] = s4a[i];
        s4a[i] = 0.f;
      }
      __syncthreads();
      if (tid < RT && row0 + tid < L_act) {
        double v = 0.0;
        for (int c = 0; c < 16; ++c) v += (double)S4[c * RT + tid];
        double* p = s4p + (int64_t)s * cap + row0 + tid;
        *p = (first ? 0.0 : *p) + v;
      }
      first = false;
      since = 0;
    }
  }
  __syncthreads();   // the unit's shared memory may be reused by the caller's next unit
}

}  // namespace simt
}  // namespace oica
