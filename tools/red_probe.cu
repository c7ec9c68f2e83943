// red_probe.cu — L2 reduction throughput by element type and row width: random
// rows of an L2-resident 64 MiB buffer, W consecutive elements per row (one lane each).  Prints
// adds/s per (type, W).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void fill_idx(uint32_t *idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    idx[i] = (uint32_t)x;
  }
}
template <typename T, int W>
__global__ void __launch_bounds__(256) red_rows(const uint32_t *idx, int64_t rows, T *y,
                                                uint32_t yrows) {
  constexpr int G = 32 / W;  // rows per warp step
  const int lane = threadIdx.x & 31, c = lane % W, g = lane / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * 4 * G; base < rows; base += nw * 4 * G) {
    uint32_t p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) p[u] = __ldcs(idx + base + u * G + g);
#pragma unroll
    for (int u = 0; u < 4; ++u) atomicAdd(y + (int64_t)(p[u] % yrows) * W + c, (T)1);
  }
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
template <typename T, int W>
static void run(const char *name, const uint32_t *idx, int64_t rows, void *y, int grid) {
  const uint32_t yrows = (uint32_t)((64ll << 20) / (sizeof(T) * W));
  const float t = best_ms([&] { red_rows<T, W><<<grid, 256>>>(idx, rows, (T *)y, yrows); });
  printf("\"%s_w%d\": %.4g, ", name, W, rows * (double)W / (t * 1e-3));
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t rows = 1ll << 26;
  uint32_t *idx;
  void *y;
  cudaMalloc(&idx, rows * 4);
  cudaMalloc(&y, 64ll << 20);
  cudaMemset(y, 0, 64ll << 20);
  fill_idx<<<sms * 8, 256>>>(idx, rows);
  const int grid = sms * 8;
  printf("{");
  run<double, 1>("f64", idx, rows, y, grid);
  run<double, 2>("f64", idx, rows, y, grid);
  run<double, 4>("f64", idx, rows, y, grid);
  run<double, 8>("f64", idx, rows, y, grid);
  run<double, 16>("f64", idx, rows, y, grid);
  run<unsigned long long, 4>("u64", idx, rows, y, grid);
  run<unsigned long long, 8>("u64", idx, rows, y, grid);
  run<unsigned long long, 16>("u64", idx, rows, y, grid);
  run<float, 8>("f32", idx, rows, y, grid);
  run<float, 16>("f32", idx, rows, y, grid);
  run<unsigned, 8>("u32", idx, rows, y, grid);
  printf("\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
