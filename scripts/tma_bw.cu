// Microbenchmark (dev aid, not part of the library): TMA ingest rate of the step kernel's X
// stream, per SM and chip-wide, for an L2-resident fp16 plane set [NP rows][M samples] read in
// [NP][64]-sample 128B-swizzled boxes (the step kernel's layout) or from a sample-major copy
// [M][NP] (one contiguous box per chunk).  A producer thread keeps STAGES chunks in flight; a
// consumer warp only waits for each chunk and releases its stage.  DESIGN.md §9 (narrow N).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_bw scripts/tma_bw.cu -lcuda && /tmp/tma_bw
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)), "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}

// LAYOUT 0: [NP][M] planes, MT/64 boxes of [NP rows][64 samples] per chunk; 1: [M][NP] sample-major,
// boxes of [64 samples][NP] (NP * 2 = 128 B rows), MT/64 per chunk; 2: sample-major, one box of
// [MT samples][NP] per chunk (MT <= 256)
// PROD: producer threads (1: thread 0; 2: threads 0 and 64 take alternate chunks, each waiting
// only for its own stages; 3: lanes 0..MT/64-1 of warp 0 each issue one box of every chunk)
template <int NP, int MT, int STAGES, int LAYOUT, int PROD = 1>
__global__ void __launch_bounds__(128, 1) k_tma_bw(const __grid_constant__ CUtensorMap tm, int64_t M, int nchunk,
                                                   unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* s = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int STAGE = NP * MT * 2;
  uint64_t* full = (uint64_t*)(s + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nblk = M / MT;
  const int64_t c0 = ((int64_t)blockIdx.x * 977) % nblk;   // scattered start, wraps around M
  unsigned long long t0 = clock64();
  const bool prod = PROD == 2 ? (threadIdx.x == 0 || threadIdx.x == 64) : PROD == 3 ? (threadIdx.x < MT / 64) : threadIdx.x == 0;
  if (prod) {
    const int j0 = PROD == 2 ? (threadIdx.x == 64) : 0, dj = PROD == 2 ? 2 : 1;
    for (int j = j0; j < nchunk; j += dj) {
      const int st = j % STAGES;
      if (j >= STAGES) mbar_wait(&empty[st], ((j / STAGES) - 1) & 1);
      const int m0 = (int)(((c0 + j) % nblk) * MT);
      if (PROD != 3 || threadIdx.x == 0) mbar_expect_tx(&full[st], STAGE);
      if (PROD == 3) __syncwarp((1u << (MT / 64)) - 1u);
      for (int h = 0; h < MT / 64; ++h) {
        if (PROD == 3 && h != (int)threadIdx.x) continue;
        if (LAYOUT == 0)
          tma2d(s + st * STAGE + h * NP * 128, &tm, &full[st], m0 + 64 * h, 0);
        else if (LAYOUT == 1)
          tma2d(s + st * STAGE + h * NP * 128, &tm, &full[st], 0, m0 + 64 * h);
        else if (h == 0)
          tma2d(s + st * STAGE, &tm, &full[st], 0, m0);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int j = 0; j < nchunk; ++j) {
      const int st = j % STAGES;
      mbar_wait(&full[st], (j / STAGES) & 1);
      mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int NP, int MT, int STAGES, int LAYOUT, int PROD = 1>
void run(EncodeFn enc, __half* X, int64_t M, int grid) {
  CUtensorMap m;
  cuuint32_t es[2] = {1, 1};
  if (LAYOUT == 0) {
    cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)NP}, str[1] = {(cuuint64_t)M * 2};
    cuuint32_t box[2] = {64, NP};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[2] = {(cuuint64_t)NP, (cuuint64_t)M}, str[1] = {(cuuint64_t)NP * 2};
    cuuint32_t box[2] = {NP, LAYOUT == 1 ? 64u : (cuuint32_t)MT};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  constexpr int SMEM = STAGES * NP * MT * 2 + 2048;
  auto k = k_tma_bw<NP, MT, STAGES, LAYOUT, PROD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  unsigned long long* cyc;
  cudaMalloc(&cyc, grid * 8);
  const int nchunk = 2000;
  k<<<grid, 128, SMEM>>>(m, M, 64, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 128, SMEM>>>(m, M, nchunk, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < grid; ++i) c += h[i];
  c /= grid;
  const double bytes = (double)nchunk * NP * MT * 2;
  printf("{\"prod\": %d, \"NP\": %d, \"MT\": %d, \"stages\": %d, \"layout\": %d, \"grid\": %d, \"B_per_clk_per_cta\": %.1f, "
         "\"TBps_chip\": %.2f, \"err\": \"%s\"}\n",
         PROD, NP, MT, STAGES, LAYOUT, grid, bytes / c, bytes * grid / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
  cudaFree(cyc);
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  const int64_t M = 250000 / 192 * 192;
  __half* X;
  cudaMalloc(&X, (size_t)64 * M * 2);
  cudaMemset(X, 0, (size_t)64 * M * 2);
  // per-CTA rate vs stage depth, box size, grid (CTAs per SM) and issuing warps
  for (int g : {148, 296}) {
    run<64, 192, 8, 0, 1>(enc, X, M, g);   // the step kernel's NP = 64 stream (3 boxes per chunk)
    run<64, 192, 2, 0, 1>(enc, X, M, g);
    run<64, 64, 8, 0, 1>(enc, X, M, g);
    run<64, 192, 8, 2, 1>(enc, X, M, g);   // one box per chunk (sample-major copy)
    run<64, 256, 6, 2, 1>(enc, X, M, g);
    run<64, 192, 8, 0, 2>(enc, X, M, g);   // two issuing warps
    run<64, 192, 8, 0, 3>(enc, X, M, g);   // three lanes of one warp
    run<64, 192, 8, 2, 2>(enc, X, M, g);
  }
  return 0;
}
