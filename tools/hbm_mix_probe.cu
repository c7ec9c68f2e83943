// hbm_mix_probe.cu — HBM bandwidth by read:write mix on the local B200 (the
// gather-mode scan writes two bytes of U per byte it reads).  Streaming float4 kernels over
// multi-GB buffers, CUDA-event timed, best of 5; prints one JSON object.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// each thread: R float4 reads and W float4 writes per step (write index space = W/R x read's)
template <int R, int W>
__global__ void __launch_bounds__(256) mix(const float4 *__restrict__ a, float4 *__restrict__ b,
                                           int64_t steps) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t s = tid; s < steps; s += nt) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float4 v = __ldcs(a + s * R + r);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
#pragma unroll
    for (int w = 0; w < W; ++w) __stcs(b + s * W + w, acc);
  }
  if (W == 0 && acc.x == 1.2345f) b[tid] = acc;  // keeps the read-only variant's loads
}
template <typename F>
static float best_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int i = 0; i < 5; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t bytes = 8ll << 30;  // 8 GiB per buffer
  float4 *a, *b;
  if (cudaMalloc(&a, bytes) || cudaMalloc(&b, bytes)) {
    printf("{\"error\": \"alloc\"}\n");
    return 1;
  }
  cudaMemset(a, 0, bytes);
  cudaMemset(b, 0, bytes);
  const int grid = sms * 8;
  const int64_t n4 = bytes / 16;
  printf("{");
  {  // 1:1 copy
    const int64_t steps = n4;
    const float t = best_ms([&] { mix<1, 1><<<grid, 256>>>(a, b, steps); });
    printf("\"copy_1r1w_GBps\": %.1f, ", 2.0 * bytes / (t * 1e-3) / 1e9);
  }
  {  // 1:2
    const int64_t steps = n4 / 2;
    const float t = best_ms([&] { mix<1, 2><<<grid, 256>>>(a, b, steps); });
    printf("\"mix_1r2w_GBps\": %.1f, ", (steps * 16.0 * 3) / (t * 1e-3) / 1e9);
  }
  {  // 2:1
    const int64_t steps = n4 / 2;
    const float t = best_ms([&] { mix<2, 1><<<grid, 256>>>(a, b, steps); });
    printf("\"mix_2r1w_GBps\": %.1f, ", (steps * 16.0 * 3) / (t * 1e-3) / 1e9);
  }
  {  // read only (writes predicated away)
    const int64_t steps = n4;
    const float t = best_ms([&] { mix<1, 0><<<grid, 256>>>(a, b, steps); });
    printf("\"read_GBps\": %.1f, ", bytes / (t * 1e-3) / 1e9);
  }
  {  // write only
    const int64_t steps = n4;
    const float t = best_ms([&] { mix<0, 1><<<grid, 256>>>(a, b, steps); });
    printf("\"write_GBps\": %.1f, ", bytes / (t * 1e-3) / 1e9);
  }
  printf("\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
