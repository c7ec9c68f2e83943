// Memory micro-benchmarks on B200: write-only, copy, random row gathers of various widths.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_write(double *p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n / 2; i += (size_t)gridDim.x * blockDim.x)
    __stcs(reinterpret_cast<double2 *>(p) + i, make_double2(1.0, 2.0));
}
__global__ void k_read(const double *p, size_t n, double *out) {
  double a = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n / 2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(reinterpret_cast<const double2 *>(p) + i); a += v.x + v.y; }
  if (a == 12345.0) out[0] = a;
}
__global__ void k_copy(const double *a, double *b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n / 2; i += (size_t)gridDim.x * blockDim.x)
    __stcs(reinterpret_cast<double2 *>(b) + i, __ldcs(reinterpret_cast<const double2 *>(a) + i));
}
// gather rows of W bytes (W/16 lanes per row, 16 B each) from table (rows x W), random idx
template <int W>
__global__ void k_gather(const float4 *tab, const uint32_t *idx, size_t nidx, float *out) {
  constexpr int L = W / 16;
  float acc = 0;
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t e = tid; e < nidx * L; e += stride) {
    uint32_t r = idx[e / L];
    float4 v = __ldg(tab + (size_t)r * L + (e % L));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1.2345f) out[0] = acc;
}
// gather + write sequential (K5-like without scan): rows of W bytes, out writes 2*W bytes per row
template <int W>
__global__ void k_gather_write(const float4 *tab, const uint32_t *idx, size_t nidx, double2 *out) {
  constexpr int L = W / 16;
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t e = tid; e < nidx * L; e += stride) {
    uint32_t r = __ldcs(idx + e / L);
    float4 v = __ldg(tab + (size_t)r * L + (e % L));
    __stcs(out + 2 * e, make_double2(v.x, v.y));
    __stcs(out + 2 * e + 1, make_double2(v.z, v.w));
  }
}
__global__ void k_iota_rand(uint32_t *idx, size_t n, uint32_t rows) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull; x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    idx[i] = (uint32_t)(x % rows);
  }
}
template <typename F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}
int main() {
  const size_t N = (size_t)1 << 30;  // doubles = 8 GB
  double *A, *B, *o; CK(cudaMalloc(&A, N * 8)); CK(cudaMalloc(&B, N * 8)); CK(cudaMalloc(&o, 64));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  dim3 g(sms * 8), bl(256);
  float t = timeit([&] { k_write<<<g, bl>>>(A, N); });
  printf("write      %.0f GB/s\n", N * 8 / t / 1e6);
  t = timeit([&] { k_read<<<g, bl>>>(A, N, o); });
  printf("read       %.0f GB/s\n", N * 8 / t / 1e6);
  t = timeit([&] { k_copy<<<g, bl>>>(A, B, N / 2); });
  printf("copy(r+w)  %.0f GB/s\n", N * 8 / t / 1e6);
  // table: 2^20 rows (c3 Z) of 256 B = 256 MB; and 2^24 rows x 128 B (c4 Z) = 2 GB
  const size_t nidx = (size_t)1 << 26;
  uint32_t *idx; CK(cudaMalloc(&idx, nidx * 4));
  for (uint32_t rows : {1u << 20, 1u << 24}) {
    k_iota_rand<<<g, bl>>>(idx, nidx, rows);
    const float4 *tab = reinterpret_cast<const float4 *>(A);
#define G(W) t = timeit([&] { k_gather<W><<<g, bl>>>(tab, idx, nidx, (float *)o); }); \
    printf("rows=%u gather %4d B rows: %.0f GB/s useful\n", rows, W, nidx * (double)W / t / 1e6);
    G(16) G(32) G(64) G(128) G(256)
#define GW(W) t = timeit([&] { k_gather_write<W><<<g, bl>>>(tab, idx, nidx / (W / 16), (double2 *)B); }); \
    printf("rows=%u gather %4d B + write 2x: %.0f GB/s (read+write)\n", rows, W, (nidx / (W / 16)) * (double)W * 3 / t / 1e6);
    GW(32) GW(64) GW(256)
  }
  return 0;
}
