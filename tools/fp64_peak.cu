// fp64_peak.cu — DFMA throughput microbenchmark (the FP64 roofline denominator;
// MEASURED_PEAKS.json carries HBM and bf16 only).  8 independent FMA chains per
// thread, 148 SMs x 8 blocks x 256 threads, CUDA events, best of 5.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

int main(int argc, char** argv) {
  const double sustain_s = argc > 1 ? atof(argv[1]) : 0.0;  // > 0: also back to back for this long
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, threads>>>(d, 16, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  double sustained = 0.0;
  int reps = 0;
  float total = 0.f;
  if (sustain_s > 0.0) {  // back-to-back launches for sustain_s seconds (power / clock steady state)
    cudaEventRecord(e0);
    reps = (int)(sustain_s * 1e3 / best) + 1;
    for (int r = 0; r < reps; ++r) k_dfma<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&total, e0, e1);
    sustained = flops * reps / (total * 1e-3) / 1e12;
  }
  printf("{\"fp64_tflops\": %.3f, \"fp64_tflops_sustained\": %.3f, \"ms\": %.3f, \"sustained_s\": %.3f, "
         "\"sms\": %d, \"how\": \"DFMA microbenchmark tools/fp64_peak.cu, 8 chains x 256 thr x %d blocks: best of 5 "
         "(burst) and %d launches back to back (sustained)\"}\n",
         flops / (best * 1e-3) / 1e12, sustained, best, total * 1e-3, sms, blocks, reps);
  return 0;
}
