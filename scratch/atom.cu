#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_red(double *y, size_t ny, size_t nops, int vec) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = tid; i < nops; i += stride) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull; x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    size_t a = (x % (ny / 4)) * 4;
    if (vec == 1) atomicAdd(y + a, 1.0);
    else if (vec == 2) { atomicAdd(y + a, 1.0); atomicAdd(y + a + 1, 2.0); }
    else { atomicAdd(y + a, 1.0); atomicAdd(y + a + 1, 2.0); atomicAdd(y + a + 2, 1.0); atomicAdd(y + a + 3, 2.0); }
  }
}
int main() {
  for (size_t mb : {8, 64}) {
    size_t ny = mb << 17;  // mb MiB of doubles
    double *y; cudaMalloc(&y, ny * 8); cudaMemset(y, 0, ny * 8);
    for (int vec : {1, 2, 4}) {
      size_t nops = 1ull << 28;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      k_red<<<148 * 8, 256>>>(y, ny, 1 << 20, vec); cudaDeviceSynchronize();
      cudaEventRecord(a); k_red<<<148 * 8, 256>>>(y, ny, nops, vec); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("array %zu MiB vec %d: %.3g red-ops/s = %.3g f64-adds/s (%s)\n", mb, vec, nops / (ms * 1e-3), nops * vec / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(y);
  }
}
