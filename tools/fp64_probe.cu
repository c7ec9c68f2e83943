// fp64_probe.cu — measured fp64 FMA throughput on the CUDA cores of the local B200 (the ALU
// roofline of the sort-free kernels).  8 independent DFMA chains per thread,
// 148 x 8 CTAs of 256 threads, best of 5 CUDA-event timings; prints one JSON object
// (committed as profiles/fp64_peak.json).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_loop(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = threadIdx.x * 1e-3 + q;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += x[q];
  if (s == 1.2345) out[0] = s;
}

// DMMA (fp64 tensor-core mma.sync m8n8k4): 4 independent accumulator chains per warp.
__global__ void __launch_bounds__(256) dmma_loop(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5 + threadIdx.x * 1e-4;
  double d[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[q][0]), "+d"(d[q][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) s += d[q][0] + d[q][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double *out;
  cudaMalloc(&out, 8);
  const int iters = 1 << 16, blocks = sms * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  dfma_loop<<<blocks, 256>>>(out, 1024, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    dfma_loop<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * (double)iters * blocks * 256;
  float best_mma = 1e30f;
  const int mma_iters = 1 << 14;
  dmma_loop<<<blocks, 256>>>(out, 64);
  cudaDeviceSynchronize();
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    dmma_loop<<<blocks, 256>>>(out, mma_iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best_mma) best_mma = ms;
  }
  const double mma_flops = 2.0 * 8 * 8 * 4 * 4 * (double)mma_iters * blocks * (256 / 32);
  printf("{\"dmma_m8n8k4_tflops\": %.3f, ", mma_flops / (best_mma * 1e-3) / 1e12);
  printf("\"fp64_fma_tflops\": %.3f, \"sms\": %d, \"sm_clock_khz\": %d, \"status\": \"%s\", "
         "\"how\": \"tools/fp64_probe.cu: 8 independent DFMA chains x 2^16 iterations per thread, "
         "%d CTAs x 256 threads, best of 5 CUDA-event timings\"}\n",
         flops / (best * 1e-3) / 1e12, sms, clk, cudaGetErrorString(cudaGetLastError()), blocks);
  return 0;
}
