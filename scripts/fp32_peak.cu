// Microbenchmark (dev aid, not part of the library): FP32 FFMA throughput of the whole GPU -- the
// "alu" roofline of the FP32 step (K2b) measured instead of computed from 148 x 128 x 2 x clock.
// Each thread runs 16 independent FFMA chains in registers; the result is compared with the nominal
// 148 x 128 lanes x 2 flop x the maximum SM clock (run uncapped: the FP32 step is far below the
// power cap).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_peak scripts/fp32_peak.cu && /tmp/fp32_peak
#include <cuda_runtime.h>

#include <cstdio>

__global__ void __launch_bounds__(256) k_ffma(float* out, int iters, long long* cycles) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  const float b = 0.999999f, c = 1e-7f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;   // keep the chains live
  if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 8);
  const int iters = 1 << 16;
  for (int bps : {4, 8}) {   // resident 256-thread blocks per SM
    const int blocks = sms * bps;
    k_ffma<<<blocks, 256>>>(out, 1024, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_ffma<<<blocks, 256>>>(out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double flop = 2.0 * 16.0 * iters * (double)blocks * 256.0;
    const double tf = flop / (ms * 1e-3) / 1e12;
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double nominal = (double)sms * 128.0 * 2.0 * khz * 1e3 / 1e12;
    (void)c;
    printf("{\"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.1f, \"nominal_tflops_at_max_clock\": %.1f, "
           "\"max_sm_mhz\": %.0f, \"frac\": %.3f, \"err\": \"%s\"}\n",
           bps, ms, tf, nominal, khz / 1e3, tf / nominal, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
