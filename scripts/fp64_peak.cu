// FP64 pipe peak on this GPU: independent DFMA chains, 8 per thread, enough
// warps to fill every SM; reports TFLOP/s (2 flops per DFMA) and DFMA
// lane-ops per clock per SM.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak scripts/fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = threadIdx.x * 1e-3 + u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = fma(x[u], a, b);
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += x[u];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 512, blocks = sms * 4, iters = 1 << 16;
  k_dfma<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double dfma = (double)blocks * threads * iters * 8;
  const double tflops = 2.0 * dfma / (best * 1e-3) / 1e12;
  std::printf("{\"fp64_dfma_tflops\": %.3f, \"dfma_per_s\": %.4e, \"ms\": %.4f, \"sms\": %d, \"clock_mhz_attr\": %.0f, "
              "\"dfma_lanes_per_clk_per_sm_at_attr_clock\": %.2f}\n",
              tflops, dfma / (best * 1e-3), best, sms, clk_khz / 1e3, dfma / (best * 1e-3) / sms / (clk_khz * 1e3));
  return 0;
}
