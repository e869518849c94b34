// Microbenchmark (dev aid, not part of the library): tcgen05.mma kind::f16 issue/throughput for
// the step kernel's shapes (M = 128, K = 16 per instruction, N = 64 ... 256), A from TMEM (the
// step's form) or from shared memory, B K-major or MN-major, one issuing thread, operands resident
// (no data movement).  Prints flop/clk/SM against the 8192 flop/clk dense rate.  DESIGN.md §9.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_rate scripts/mma_rate.cu && /tmp/mma_rate
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_f16(int N, int b_mn_major) {
  return (1u << 4) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc),
               "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc),
               "r"(acc) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P1;\n\tW:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}

// TS: A from TMEM; BMN: B MN-major; ND: accumulators rotated over ND regions; per round KB
// instructions (K = 16 each) into one accumulator
template <int N, bool TS, int BMN, int ND, int KB, int ISS = 1>
__global__ void __launch_bounds__(128, 1) k_mma(int rounds) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* s = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    mbar_init(&bar, ISS);   // one commit per issuer
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot;
  if (warp >= 1 && warp <= ISS) {   // ISS issuing warps, each into its own accumulators
    constexpr uint32_t id = idesc_f16(N, BMN);
    const uint64_t da = sdesc(smem_u32(s), 16, 1024);
    const uint64_t db = sdesc(smem_u32(s + 32768), BMN ? 8192 : 16, 1024);
    // TMEM: A at columns [0, 8 KB) (K = 16 fp16 = 8 columns per instruction), accumulators after
    const uint32_t d0 = tm + 64 + (uint32_t)((warp - 1) * ND * N);
    constexpr int DSTRIDE = N;   // accumulator columns
    static_assert(64 + ISS * ND * DSTRIDE <= 512, "TMEM");
    for (int r = 0; r < rounds; ++r) {
      const uint32_t d = d0 + (uint32_t)((r % ND) * DSTRIDE);
      if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
          const uint64_t b = db + (uint64_t)((BMN ? ((kb % 4) * 2048) : ((kb % 4) * 32)) >> 4);
          if (TS)
            mma_ts(d, tm + (kb % 8) * 8, b, id, kb > 0 ? 1u : 0u);
          else
            mma_ss(d, da + (uint64_t)((kb * 32) >> 4), b, id, kb > 0 ? 1u : 0u);
        }
      }
      __syncwarp();
    }
    if ((threadIdx.x & 31) == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int N, bool TS, int BMN, int ND, int KB, int ISS = 1>
void run() {
  const int blocks = 148, rounds = 2000;
  auto k = k_mma<N, TS, BMN, ND, KB, ISS>;
  const int SMEM = 100 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  k<<<blocks, 128, SMEM>>>(10);
  cudaError_t err = cudaGetLastError();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, 128, SMEM>>>(rounds);
  cudaEventRecord(e1);
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err == cudaSuccess) err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 128 * N * 16 * (double)KB * rounds * ISS;
  const double tf = flops * blocks / (ms * 1e-3) / 1e12;
  printf("{\"issuers\": %d, \"N\": %d, \"A\": \"%s\", \"B\": \"%s\", \"instr_per_round\": %d, \"ms\": %.3f, "
         "\"TFLOPs_chip\": %.1f, \"ns_per_instr_per_issuer\": %.2f, \"err\": \"%s\"}\n",
         ISS, N, TS ? "tmem" : "smem", BMN ? "mn" : "k", KB, ms, tf, ms * 1e6 / ((double)KB * rounds), cudaGetErrorString(err));
}

int main() {
  // the step's GEMM2 at NP = 64 / 32 (N = NP, B K-major, A = Y3 in TMEM), one to three issuers
  run<64, true, 0, 1, 12, 1>();
  run<64, true, 0, 1, 12, 2>();
  run<64, false, 0, 1, 12, 1>();
  run<32, true, 0, 1, 16, 1>();
  run<32, true, 0, 1, 16, 2>();
  run<32, true, 0, 1, 16, 3>();
  run<96, true, 0, 1, 12, 1>();
  // the step's GEMM1 (N = MT samples, B MN-major, A = W in TMEM) and wide N
  run<192, true, 1, 1, 4, 1>();
  run<128, true, 1, 1, 4, 1>();
  run<128, true, 0, 1, 8, 1>();
  run<256, true, 0, 1, 4, 1>();
  run<256, false, 0, 1, 4, 1>();
  return 0;
}
