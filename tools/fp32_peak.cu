// fp32_peak.cu — measured FP32 FFMA peak of this B200 (SURVEY §8(d) "FP32 peak":
// MEASURED_PEAKS.json has no FP32-SIMT figure). 8 independent FMA chains per thread,
// every SM full, CUDA-event timed, best of several runs. Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) fma_chains(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
        x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1234.5f) out[blockIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaSetDevice(dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 1 << 20);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_chains<<<blocks, threads>>>(out, 64, 0.999f, 1e-3f);
  cudaDeviceSynchronize();
  double best = 0;
  int runs = 0;
  cudaEvent_t t0;
  cudaEventCreate(&t0);
  cudaEventRecord(t0);
  float spent = 0.f;
  // repeat for ~3 s so that an NVML sampler sees the clock under this load
  for (int r = 0; r < 10 || spent < 3000.f; ++r, ++runs) {
    cudaEventRecord(e0);
    fma_chains<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
    cudaEventElapsedTime(&spent, t0, e1);
  }
  double nominal = 2.0 * 128 * sms * (clk * 1e3) / 1e12;
  printf("{\"fp32_tflops\": %.2f, \"sms\": %d, \"attr_clock_mhz\": %.0f, \"nominal_at_attr_clock\": %.2f, \"runs\": %d}\n",
         best, sms, clk / 1e3, nominal, runs);
  return 0;
}
