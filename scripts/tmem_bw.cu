// Microbenchmark (dev aid, not part of the library): tcgen05.ld throughput per SM for the load
// shapes an epilogue can use, with 4 / 8 / 16 warps reading TMEM concurrently.  Answers whether
// the step kernel's epilogue (32x32b.x32, 4 warps) is at the SM's TMEM read limit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bw scripts/tmem_bw.cu && /tmp/tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define R8(i) "=r"(v[i + 0]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])
#define REGS32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"

template <int SHAPE>
__device__ __forceinline__ void ld32(uint32_t a, uint32_t (&v)[32]) {
  if (SHAPE == 0)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " REGS32 ", [%32];"
                 : R8(0), R8(8), R8(16), R8(24) : "r"(a));
  else if (SHAPE == 1)
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 " REGS32 ", [%32];"
                 : R8(0), R8(8), R8(16), R8(24) : "r"(a));
  else if (SHAPE == 2)
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 " REGS32 ", [%32];"
                 : R8(0), R8(8), R8(16), R8(24) : "r"(a));
  else
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 " REGS32 ", [%32];"
                 : R8(0), R8(8), R8(16), R8(24) : "r"(a));
}

// every warp: ITER rounds of DEPTH loads of 4 KB (32 regs/thread) then one wait::ld
template <int SHAPE, int DEPTH>
__global__ void k_tmem_bw(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot;
  // warp w reaches lane quadrant w % 4; the column window rotates per warp
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int colw = SHAPE == 0 ? 32 : SHAPE == 1 ? 64 : SHAPE == 2 ? 64 : 64;   // columns per load
  uint32_t acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t v[DEPTH][32];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      const uint32_t col = (uint32_t)(((it * DEPTH + d) * colw + (warp >> 2) * 64) % (512 - colw + 1)) & ~31u;
      ld32<SHAPE>(tm + lane_off + col, v[d]);
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int d = 0; d < DEPTH; ++d)
#pragma unroll
      for (int k = 0; k < 32; ++k) acc ^= v[d][k];
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int SHAPE, int DEPTH>
void run(const char* name, int warps) {
  const int iters = 4096, blocks = 148;
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, blocks * 8);
  cudaMalloc(&sink, 4096);
  k_tmem_bw<SHAPE, DEPTH><<<blocks, 32 * warps>>>(16, cyc, sink);   // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_tmem_bw<SHAPE, DEPTH><<<blocks, 32 * warps>>>(iters, cyc, sink);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < blocks; ++i) c += h[i];
  c /= blocks;
  const double bytes_per_sm = (double)iters * DEPTH * warps * 4096.0;
  printf("{\"shape\": \"%s\", \"warps\": %d, \"depth\": %d, \"bytes_per_clk_per_sm\": %.1f, \"ms\": %.3f, \"TBps_chip\": %.1f, \"err\": \"%s\"}\n",
         name, warps, DEPTH, bytes_per_sm / c, ms, bytes_per_sm * blocks / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0, 1>("32x32b.x32", w);
    run<0, 2>("32x32b.x32", w);
    run<0, 4>("32x32b.x32", w);
    run<1, 1>("16x256b.x8", w);
    run<1, 2>("16x256b.x8", w);
    run<2, 2>("16x128b.x16", w);
    run<3, 2>("16x64b.x32", w);
  }
  return 0;
}
