// fp64_lat.cu — DFMA dependent-issue latency and the FP64 throughput reached with
// W warps per SM each running C independent dependency chains: how much
// instruction-level parallelism the stage kernels need per scheduler.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_lat.cu -o fp64_lat
#include <cuda_runtime.h>

#include <cstdio>

template <int C>
__global__ void chains(double* out, long long* cyc, double a, double b, int iters) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  if (s == 1234.5678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int C>
void run(int sms, double* out, long long* cyc) {
  const int iters = 8192;
  // latency: one warp on one SM
  chains<C><<<1, 32>>>(out, cyc, 0.999999, 1e-7, iters);
  cudaDeviceSynchronize();
  long long c1;
  cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"chains\": %d, \"cycles_per_dfma_1warp\": %.2f", C, (double)c1 / iters / C);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w : {4, 8, 12, 16, 24, 32}) {
    const int threads = 32 * w, blocks = sms;
    chains<C><<<blocks, threads>>>(out, cyc, 0.999999, 1e-7, iters);
    cudaEventRecord(e0);
    chains<C><<<blocks, threads>>>(out, cyc, 0.999999, 1e-7, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * C * (double)iters * threads * blocks;
    printf(", \"tf_w%d\": %.2f", w, fl / (ms * 1e-3) / 1e12);
  }
  printf("}\n");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  run<1>(sms, out, cyc);
  run<2>(sms, out, cyc);
  run<4>(sms, out, cyc);
  run<8>(sms, out, cyc);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
