// Micro-benchmark: K5-like traffic (perm + sval stream, Z row gather, U row write) with
//   A) full 64-column Z rows gathered from a 256 MB row-major Z (current design)
//   B) column blocks of MB columns from a block-major Zt[cb][n][MB] copy, one launch per
//      block, gathers with an L2 evict_last policy and U stores evict-first
// n = 2^20, K coordinates, m = 64.  Reports time per (i,k) pair and HBM-equivalent rates.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ float4 ldg_hint(const float4 *p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(double2 *p, double2 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

// L lanes per row (16 B of Z each), UNR rows per lane-group in flight.
// Z row length ldz floats; column offset c0; U row length ldu doubles.
template <int L, int UNR, bool HINT>
__global__ void __launch_bounds__(256) k_scanlike(const uint32_t *perm, const float *sval, int64_t n,
                                                  const float *Z, int64_t ldz, int64_t c0, double *U,
                                                  int64_t ldu, int K) {
  const uint64_t pl = pol_last(), pf = pol_first();
  const int gpw = 32 / L;  // row groups per warp
  const int64_t lane = threadIdx.x & 31, sub = lane % L, g = lane / L;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t rows_total = (int64_t)K * n;
  for (int64_t base = warp * gpw * UNR; base < rows_total; base += nwarps * gpw * UNR) {
    uint32_t p[UNR]; float v[UNR]; float4 z[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t e = base + u * gpw + g;
      p[u] = e < rows_total ? __ldcs(perm + e) : 0; v[u] = e < rows_total ? __ldcs(sval + e) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const float4 *src = reinterpret_cast<const float4 *>(Z + (int64_t)p[u] * ldz + c0) + sub;
      z[u] = HINT ? ldg_hint(src, pl) : __ldg(src);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t e = base + u * gpw + g;
      if (e >= rows_total) continue;
      double2 *dst = reinterpret_cast<double2 *>(U + e * ldu + c0 + 4 * sub);
      const double2 a = make_double2(v[u] * (double)z[u].x, v[u] * (double)z[u].y);
      const double2 b = make_double2(v[u] * (double)z[u].z, v[u] * (double)z[u].w);
      if (HINT) { st_hint(dst, a, pf); st_hint(dst + 1, b, pf); }
      else { __stcs(dst, a); __stcs(dst + 1, b); }
    }
  }
}
__global__ void k_transpose(const float *Z, int64_t n, int64_t m, int MB, float *Zt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * m; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / m, c = e % m;
    Zt[(c / MB) * n * MB + i * MB + (c % MB)] = Z[e];
  }
}

// C: warp-coalesced fp64 reductions into an L2-resident Y block: rows of MB doubles at random
// row indices (perm), MB lanes per row.
template <int MB, bool VEC>
__global__ void __launch_bounds__(256) k_red(const uint32_t *perm, int64_t nrows_total, int64_t n, double *Y) {
  const int64_t lane = threadIdx.x & 31, sub = lane % (VEC ? MB / 2 : MB), g = lane / (VEC ? MB / 2 : MB);
  constexpr int GPW = 32 / (VEC ? MB / 2 : MB);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * GPW * 4; base < nrows_total; base += nwarps * GPW * 4) {
    uint32_t p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { const int64_t e = base + u * GPW + g; p[u] = e < nrows_total ? __ldcs(perm + e) : 0; }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double *y = Y + (int64_t)p[u] * MB;
      if constexpr (VEC) {
        atomicAdd(y + 2 * sub, 1.0); atomicAdd(y + 2 * sub + 1, 2.0);
      } else {
        atomicAdd(y + sub, 1.0);
      }
    }
  }
}
template <typename F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}
int main() {
  const int64_t n = 1 << 20, m = 64; const int K = 32;
  std::vector<uint32_t> hp((size_t)K * n);
  std::mt19937 rng(1);
  std::vector<uint32_t> base(n); for (int64_t i = 0; i < n; ++i) base[i] = (uint32_t)i;
  for (int k = 0; k < K; ++k) { std::shuffle(base.begin(), base.end(), rng); std::copy(base.begin(), base.end(), hp.begin() + (size_t)k * n); }
  uint32_t *perm; float *sval, *Z, *Zt; double *U;
  CK(cudaMalloc(&perm, hp.size() * 4)); CK(cudaMemcpy(perm, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&sval, hp.size() * 4)); CK(cudaMemset(sval, 0, hp.size() * 4));
  CK(cudaMalloc(&Z, n * m * 4)); CK(cudaMemset(Z, 0, n * m * 4));
  CK(cudaMalloc(&Zt, n * m * 4));
  CK(cudaMalloc(&U, (size_t)K * n * m * 8));
  const double pairs = (double)K * n;
  const int grid = 148 * 8;
  // A: full rows, 16 lanes x 16 B = 256 B
  for (int hint = 0; hint < 2; ++hint) {
    float ms = timeit([&] {
      if (hint) k_scanlike<16, 4, true><<<grid, 256>>>(perm, sval, n, Z, m, 0, U, m, K);
      else k_scanlike<16, 4, false><<<grid, 256>>>(perm, sval, n, Z, m, 0, U, m, K);
    });
    printf("A full-row hint=%d: %.3f ms  %.3f ns/pair  alg(8+12m)=%.0f GB/s\n", hint, ms, ms * 1e6 / pairs,
           pairs * (8 + 12 * m) / (ms * 1e-3) / 1e9);
  }
  for (int MB : {8, 16, 32}) {
    float tt = timeit([&] { k_transpose<<<grid, 256>>>(Z, n, m, MB, Zt); });
    for (int hint = 0; hint < 2; ++hint) {
      float ms = timeit([&] {
        for (int cb = 0; cb < m / MB; ++cb) {
          const float *zb = Zt + (int64_t)cb * n * MB;
          // U for block cb: column offset cb*MB within ldu = m rows
          double *ub = U + cb * MB;
#define GO(L) if (hint) k_scanlike<L, 4, true><<<grid, 256>>>(perm, sval, n, zb, MB, 0, ub, m, K); \
              else k_scanlike<L, 4, false><<<grid, 256>>>(perm, sval, n, zb, MB, 0, ub, m, K);
          if (MB == 8) { GO(2) } else if (MB == 16) { GO(4) } else { GO(8) }
#undef GO
        }
      });
      // note: the kernel writes U at column offset 0..MB of ub (c0 = 0 in zb): fine for timing
      const double hbm = pairs * (8.0 * (m / MB) + 8 * m);
      printf("B MB=%d hint=%d: %.3f ms (+transpose %.3f)  %.3f ns/pair  alg(8+12m)=%.0f GB/s  hbm-model=%.0f GB/s\n",
             MB, hint, ms, tt, ms * 1e6 / pairs, pairs * (8 + 12 * m) / (ms * 1e-3) / 1e9, hbm / (ms * 1e-3) / 1e9);
    }
  }

  {
    double *Y; CK(cudaMalloc(&Y, (size_t)n * 32 * 8)); CK(cudaMemset(Y, 0, (size_t)n * 32 * 8));
    const int64_t rows = (int64_t)K * n;
#define RT(MB, V) { float ms = timeit([&] { k_red<MB, V><<<grid, 256>>>(perm, rows, n, Y); }); \
      printf("C red MB=%d vec=%d: %.3f ms  %.3g f64-adds/s  (Y block %d MB)\n", MB, (int)V, ms, rows * (double)MB / (ms * 1e-3), (int)(n * MB * 8 >> 20)); }
    RT(1, false) RT(4, false) RT(8, false) RT(16, false) RT(32, false)
    RT(4, true) RT(8, true) RT(16, true)
    CK(cudaGetLastError());
  }
  // write-only reference: U stream
  float ws = timeit([&] { cudaMemsetAsync(U, 0, (size_t)K * n * m * 8); });
  printf("memset U: %.3f ms = %.0f GB/s\n", ws, (double)K * n * m * 8 / (ws * 1e-3) / 1e9);
  CK(cudaGetLastError());
  return 0;
}
