// fp64_peak.cu — measures the B200's dense FP64 (DFMA) throughput, the roofline
// denominator MEASURED_PEAKS.json lacks.  Standalone binary:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu -o fp64_peak
// Prints one JSON line: {"dfma_tflops": burst, "dfma_tflops_sustained": ..}.
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void dfma_loop(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5678) out[0] = s;  // keep the work alive
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 512, blocks = sms * 4;
  const double flops = 2.0 * kChains * (double)kIters * threads * blocks;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  // sustained: back to back for ~3 s
  const int reps = 400;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms_all;
  cudaEventElapsedTime(&ms_all, e0, e1);
  printf("{\"dfma_tflops\": %.2f, \"dfma_tflops_sustained\": %.2f, \"sms\": %d, \"burst_ms\": %.3f}\n",
         flops / (best * 1e-3) / 1e12, flops * reps / (ms_all * 1e-3) / 1e12, sms, best);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
