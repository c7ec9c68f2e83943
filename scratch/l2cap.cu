// L2 residency probe: per row, stream perm (evict_first), gather a 32-B Zt row from a ZS-MB
// buffer (evict_last) and add 8 doubles into a YS-MB buffer with hinted fp64 reductions.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t pf() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pl() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pn() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p)); return p; }
__global__ void __launch_bounds__(256) k(const uint32_t *idx, int64_t rows, const float *zt, uint32_t zrows,
                                         double *y, uint32_t yrows, int hint) {
  const uint64_t a = hint ? pf() : pn(), b = hint ? pl() : pn();
  const int lane = threadIdx.x & 31, c = lane & 7, g = lane >> 3;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * 16; base < rows; base += nw * 16) {
    uint32_t p[4]; float z[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t *ip = idx + base + u * 4 + g;
      asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(p[u]) : "l"(ip), "l"(a));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (zrows) { const float *zp = zt + (int64_t)(p[u] % zrows) * 8 + c;
        asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(z[u]) : "l"(zp), "l"(b)); }
      else z[u] = 1.0f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double *yp = y + (int64_t)((p[u] * 2654435761u) % yrows) * 8 + c;
      asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(yp), "d"((double)z[u]), "l"(b) : "memory");
    }
  }
}
__global__ void fill(uint32_t *idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull; x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32; idx[i] = (uint32_t)x; }
}
int main() {
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0); printf("L2 attr %d bytes\n", l2);
  int persist; cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, 0); printf("max persisting L2 %d bytes\n", persist);
  const int64_t rows = 1ll << 27;  // 134M rows (one c3 launch)
  uint32_t *idx; float *zt; double *y;
  cudaMalloc(&idx, rows * 4); cudaMalloc(&zt, 256ll << 20); cudaMalloc(&y, 256ll << 20);
  cudaMemset(zt, 0, 256ll << 20); cudaMemset(y, 0, 256ll << 20);
  fill<<<1184, 256>>>(idx, rows);
  int cfg[][2] = {{16, 8}, {32, 0}, {32, 16}, {48, 0}, {48, 24}, {64, 0}, {64, 16}, {64, 32}, {96, 0}, {128, 0}};
  for (int hint = 0; hint < 2; ++hint)
    for (auto &c : cfg) {
      const uint32_t yrows = (uint32_t)((int64_t)c[0] << 20) / 64, zrows = (uint32_t)((int64_t)c[1] << 20) / 32;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      k<<<1184, 256>>>(idx, rows / 8, zt, zrows, y, yrows, hint);
      cudaEventRecord(e0);
      k<<<1184, 256>>>(idx, rows, zt, zrows, y, yrows, hint);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("hint=%d Y %3d MB Zt %3d MB: %.3f ms  %.3g row-adds/s  %.3g f64-adds/s\n", hint, c[0], c[1], ms, rows / (ms * 1e-3), rows * 8 / (ms * 1e-3));
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
