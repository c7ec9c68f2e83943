// l1dm_sortfree.cu — the sort-free products: even-p l_p^p (p = 2 is
// the squared Euclidean matrix), Alg. "query_p_even" (Thm. even_p) with
// the binomial coefficients and y_j the garbled text drops (R19):
//
//   (x_i - x_j)^p = sum_t C(p,t) (-1)^t x_i^(p-t) x_j^t            (p even: no sign/abs)
//   y_ic = sum_k sum_t c_t x_ik^(p-t) W_t[k][c],   W_t[k][c] = sum_j x_jk^t z_jc,  c_t = C(p,t)(-1)^t
//        = S_c hp_i + sum_{t=1}^{p-1} c_t (X^(p-t) W_t)_ic + G_c,
//   S_c = sum_j z_jc,  hp_i = sum_k x_ik^p,  G_c = sum_k W_p[k][c]  (c_0 = c_p = 1 for even p).
//
// Two dense contractions on the fp64 tensor cores (DMMA, mma.sync m8n8k4 f64: fp32 inputs,
// fp64 products and sums; the tcgen05 kinds below fp64 cannot hold the 1e-9 bar):
//   K12 moment reduce  W_t = (X^t)^T Z for t = 1..p, split over point chunks; each CTA owns a
//                      64 x 64 (coordinate, column) tile of one power and a chunk of points,
//                      staging X and Z sub-tiles in shared memory; partials per chunk
//   K13 moment fold    partials summed over chunks in fixed order (deterministic); S_c, G_c
//   K14 expand         per 64-point x 64-column tile: sum over k of the powers of x times the
//                      folded W (staged in shared memory), plus S_c hp_i + G_c
// Memory: X is read p+1 times, Z p times, Y written once; FLOPs ~2 n d m (2p - 1).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "l1dm_device.cuh"
#include "l1dm_internal.h"

namespace l1dm {

namespace {

constexpr int kTile = 64;    // output tile (rows x columns) of K12 and K14
constexpr int kStepK = 16;   // coordinates per shared-memory step of K14
#ifndef L1DM_EVEN_CTAS_PER_SM
#define L1DM_EVEN_CTAS_PER_SM 2  // K12 split-K: point chunks for ~this many CTAs per SM (one wave; 2 measured best)
#endif
#ifndef L1DM_K14_P2_G
#define L1DM_K14_P2_G 4
#endif
#ifndef L1DM_K14_P2_KS
#define L1DM_K14_P2_KS 16
#endif

__device__ __forceinline__ double powi(double x, int t) {
  double r = 1.0;
  for (int q = 0; q < t; ++q) r *= x;
  return r;
}

// ---- fp64 tensor-core (DMMA, mma.sync m8n8k4 f64) versions of K12 / K14 -----------------
// mma.sync.aligned.m8n8k4.row.col.f64: lane l holds A[l/4][l%4], B[l%4][l/4] and
// D[l/4][2(l%4) + {0,1}].  One DMMA = 256 fp64 FMAs; measured 37.2 TFLOP/s on this B200
// (tools/fp64_probe.cu) vs 34.2 for CUDA-core DFMA, and 8x fewer issue slots per FMA.
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int kDmmaKs = 32;          // points per shared-memory stage of K12
constexpr int kDmmaPad = kTile + 8;  // padded row length (doubles): two wavefronts per fragment

// K12 on DMMA: grid (k tiles, c tiles, p * chunks), 8 warps; a CTA owns 32 G coordinates x 64
// columns, warp w the coordinate rows 8 G (w % 4) .. +8 G (G 8-row groups) x columns
// 32 (w / 4) .. +32 (four 8-column tiles): G = 4 gives 16 DMMAs per 8 fragment loads (the
// d >= 128 tile), G = 2 the narrow one.  colpart (t = 1, first coordinate tile only): the
// chunk's column sums of Z, S_c's partials (folded by k13_colsum in fixed order).
template <int G>
__global__ void __launch_bounds__(256)
    k12_moment_reduce_dmma(const float *__restrict__ X, int64_t ldx, const float *__restrict__ Z,
                           int64_t ldz, int64_t n, int64_t d, int64_t m, int p, int64_t chunk,
                           double *__restrict__ part, double *__restrict__ colpart,
                           double *__restrict__ gpart, int pg) {
  constexpr int TK = 32 * G, XPAD = TK + 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *xs = reinterpret_cast<double *>(smem_raw);  // [kDmmaKs][XPAD]  x^t
  double *zs = xs + kDmmaKs * XPAD;                    // [kDmmaKs][kDmmaPad]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t k0 = (int64_t)blockIdx.x * TK, c0 = (int64_t)blockIdx.y * kTile;
  const int t = 1 + (int)(blockIdx.z % p);
  const int64_t ch = blockIdx.z / p;
  const int64_t i0 = ch * chunk, i1 = (i0 + chunk < n) ? i0 + chunk : n;
  const int rw = 8 * G * (w % 4), cw = 32 * (w / 4);
  const bool colsum = colpart && t == 1 && blockIdx.x == 0;
  // G_c's partial sum_j hp_j z_jc (hp_j = sum_k x_jk^pg) when the tile holds every coordinate
  const bool gsum = colsum && gpart && gridDim.x == 1;
  __shared__ double s_hp[kDmmaKs];
  double csum = 0.0, gsumc = 0.0;  // threads 0..63: column c0 + tid
  double acc[G][4][2];
#pragma unroll
  for (int a = 0; a < G; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // register double buffering: stage s+1's global loads are in flight while stage s computes
  constexpr int PX = kDmmaKs * TK / 256, PZ = kDmmaKs * kTile / 256;
  float xr[PX], zr[PZ];
  auto load = [&](int64_t base) {
#pragma unroll
    for (int u = 0; u < PX; ++u) {
      const int e = tid + 256 * u;
      const int r = e / TK, q = e - (e / TK) * TK;
      const int64_t i = base + r;
      xr[u] = (i < i1 && k0 + q < d) ? __ldcs(X + i * ldx + k0 + q) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < PZ; ++u) {
      const int e = tid + 256 * u;
      const int r = e / kTile, q = e - (e / kTile) * kTile;
      const int64_t i = base + r;
      zr[u] = (i < i1 && c0 + q < m) ? __ldcs(Z + i * ldz + c0 + q) : 0.0f;
    }
  };
  if (i0 < i1) load(i0);
  for (int64_t base = i0; base < i1; base += kDmmaKs) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PX; ++u) {
      const int e = tid + 256 * u;
      const int r = e / TK, q = e - (e / TK) * TK;
      xs[r * XPAD + q] = powi((double)xr[u], t);
    }
#pragma unroll
    for (int u = 0; u < PZ; ++u) {
      const int e = tid + 256 * u;
      const int r = e / kTile, q = e - (e / kTile) * kTile;
      zs[r * kDmmaPad + q] = (double)zr[u];
    }
    __syncthreads();
    if (base + kDmmaKs < i1) load(base + kDmmaKs);
    if (gsum) {  // hp of the stage's 32 points: 8 threads per point, 4 G coordinates each
      const int r = tid >> 3, q0 = (tid & 7) * (TK / 8);
      double h = 0.0;
#pragma unroll
      for (int q = 0; q < TK / 8; ++q) {
        const double x = xs[r * XPAD + q0 + q];  // x^1 (t == 1); zero past d and past i1
        h += powi(x, pg);
      }
#pragma unroll
      for (int off = 4; off; off >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, off);
      if ((tid & 7) == 0) s_hp[r] = h;
      __syncthreads();
    }
    if (colsum && tid < kTile) {
#pragma unroll 8
      for (int r = 0; r < kDmmaKs; ++r) csum += zs[r * kDmmaPad + tid];  // rows past i1 are 0
      if (gsum) {
#pragma unroll 8
        for (int r = 0; r < kDmmaKs; ++r) gsumc = fma(s_hp[r], zs[r * kDmmaPad + tid], gsumc);
      }
    }
#pragma unroll
    for (int kk = 0; kk < kDmmaKs / 4; ++kk) {
      const int pt = 4 * kk + (lane & 3);
      double a[G], b[4];
#pragma unroll
      for (int g = 0; g < G; ++g) a[g] = xs[pt * XPAD + rw + 8 * g + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = zs[pt * kDmmaPad + cw + 8 * j + (lane >> 2)];
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[g][j][0], acc[g][j][1], a[g], b[j]);
    }
  }
  if (colsum && tid < kTile && c0 + tid < m) colpart[ch * m + c0 + tid] = csum;
  if (gsum && tid < kTile && c0 + tid < m) gpart[ch * m + c0 + tid] = gsumc;
  double *out = part + ((ch * p + (t - 1)) * d) * m;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int64_t k = k0 + rw + 8 * g + (lane >> 2);
    if (k >= d) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t c = c0 + cw + 8 * j + 2 * (lane & 3) + h;
        if (c < m) out[k * m + c] = acc[g][j][h];
      }
  }
}

// the k12 variant for d coordinates, its CTA coordinate tile and dynamic shared memory
static int k12_g(int64_t d) { return d > 64 ? 4 : 2; }
static size_t k12_smem(int G) {
  return ((size_t)kDmmaKs * (32 * G + 8) + (size_t)kDmmaKs * kDmmaPad) * sizeof(double);
}
// K12 with fp32 operand tiles streamed by cp.async through a 3-stage shared-memory ring (one
// barrier per 32-point stage, no register staging), converted to fp64 (and raised to t) at
// fragment load.  Needs 16-byte aligned rows and full 128-coordinate tiles (d % 128 == 0) and
// 64-column tiles (m % 64 == 0 or the last tile zero-filled by chunk); K12<G> covers the rest.
constexpr int kRing = 3;
constexpr int kXs = 128 + 4, kZs = 64 + 4;  // padded fp32 row lengths (bank spread)
__global__ void __launch_bounds__(256)
    k12_moment_reduce_ring(const float *__restrict__ X, int64_t ldx, const float *__restrict__ Z,
                           int64_t ldz, int64_t n, int64_t d, int64_t m, int p, int64_t chunk,
                           double *__restrict__ part, double *__restrict__ colpart,
                           double *__restrict__ gpart, int pg) {
  constexpr int G = 4, TK = 128;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *xs = reinterpret_cast<float *>(smem_raw);  // [kRing][kDmmaKs][kXs]
  float *zs = xs + kRing * kDmmaKs * kXs;            // [kRing][kDmmaKs][kZs]
  __shared__ double s_hp[kDmmaKs];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t k0 = (int64_t)blockIdx.x * TK, c0 = (int64_t)blockIdx.y * kTile;
  const int t = 1 + (int)(blockIdx.z % p);
  const int64_t ch = blockIdx.z / p;
  const int64_t i0 = ch * chunk, i1 = (i0 + chunk < n) ? i0 + chunk : n;
  const int rw = 8 * G * (w % 4), cw = 32 * (w / 4);
  const bool colsum = colpart && t == 1 && blockIdx.x == 0;
  const bool gsum = colsum && gpart && gridDim.x == 1;
  double csum = 0.0, gsumc = 0.0;
  double acc[G][4][2];
#pragma unroll
  for (int a = 0; a < G; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int64_t nst = (i1 - i0 + kDmmaKs - 1) / kDmmaKs;
  auto issue = [&](int64_t st) {
    if (st < nst) {
      const int64_t base = i0 + st * kDmmaKs;
      float *xb = xs + (st % kRing) * kDmmaKs * kXs, *zb = zs + (st % kRing) * kDmmaKs * kZs;
      // X: 32 rows x 32 chunks of 16 B; Z: 32 rows x 16 chunks
      for (int e = tid; e < kDmmaKs * 32; e += 256) {
        const int r = e >> 5, q = e & 31;
        const bool ok = base + r < i1;
        cp_async<16>(xb + r * kXs + 4 * q, ok ? (const void *)(X + (base + r) * ldx + k0 + 4 * q)
                                              : (const void *)X, ok);
      }
      for (int e = tid; e < kDmmaKs * 16; e += 256) {
        const int r = e >> 4, q = e & 15;
        const bool ok = base + r < i1 && c0 + 4 * q < m;
        cp_async<16>(zb + r * kZs + 4 * q, ok ? (const void *)(Z + (base + r) * ldz + c0 + 4 * q)
                                              : (const void *)Z, ok);
      }
    }
    cp_async_commit();
  };
  for (int st = 0; st < kRing - 1; ++st) issue(st);
  for (int64_t st = 0; st < nst; ++st) {
    cp_async_wait_group<kRing - 2>();
    __syncthreads();  // stage st landed for every thread; stage st-1's buffer is free
    issue(st + kRing - 1);
    const float *xb = xs + (st % kRing) * kDmmaKs * kXs, *zb = zs + (st % kRing) * kDmmaKs * kZs;
    if (gsum) {
      const int r = tid >> 3, q0 = (tid & 7) * (TK / 8);
      double h = 0.0;
#pragma unroll
      for (int q = 0; q < TK / 8; ++q) h += powi((double)xb[r * kXs + q0 + q], pg);
#pragma unroll
      for (int off = 4; off; off >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, off);
      if ((tid & 7) == 0) s_hp[r] = h;
      __syncthreads();
    }
    if (colsum && tid < kTile) {
#pragma unroll 8
      for (int r = 0; r < kDmmaKs; ++r) csum += (double)zb[r * kZs + tid];  // zero-filled rows
      if (gsum) {
#pragma unroll 8
        for (int r = 0; r < kDmmaKs; ++r) gsumc = fma(s_hp[r], (double)zb[r * kZs + tid], gsumc);
      }
    }
#pragma unroll
    for (int kk = 0; kk < kDmmaKs / 4; ++kk) {
      const int pt = 4 * kk + (lane & 3);
      double a[G], b[4];
#pragma unroll
      for (int g = 0; g < G; ++g) a[g] = powi((double)xb[pt * kXs + rw + 8 * g + (lane >> 2)], t);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = (double)zb[pt * kZs + cw + 8 * j + (lane >> 2)];
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[g][j][0], acc[g][j][1], a[g], b[j]);
    }
    if (gsum) __syncthreads();  // s_hp is rewritten by the next stage
  }
  cp_async_wait_all();
  if (colsum && tid < kTile && c0 + tid < m) colpart[ch * m + c0 + tid] = csum;
  if (gsum && tid < kTile && c0 + tid < m) gpart[ch * m + c0 + tid] = gsumc;
  double *out = part + ((ch * p + (t - 1)) * d) * m;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int64_t k = k0 + rw + 8 * g + (lane >> 2);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t c = c0 + cw + 8 * j + 2 * (lane & 3) + h;
        if (c < m) out[k * m + c] = acc[g][j][h];
      }
  }
}

static void launch_k12(const float *X, int64_t ldx, const float *Z, int64_t ldz, int64_t n,
                       int64_t d, int64_t m, int p, int64_t chunk, int64_t nchunks, double *part,
                       double *colpart, double *gpart, int pg, cudaStream_t s) {
  static const bool ring_env = [] {
    const char *e = getenv("L1DM_K12_RING");
    return e ? atoi(e) != 0 : true;
  }();
  // (only for the first moment: higher powers would be recomputed at every fragment load,
  // which the staged kernel does once per element — measured slower at p = 4, 6)
  if (ring_env && p == 1 && d % 128 == 0 && m % 4 == 0 && ldx % 4 == 0 && ldz % 4 == 0 &&
      (uintptr_t)X % 16 == 0 && (uintptr_t)Z % 16 == 0) {
    const size_t sm = (size_t)kRing * kDmmaKs * (kXs + kZs) * sizeof(float);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k12_moment_reduce_ring, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sm);
      attr = true;
    }
    dim3 g((unsigned)(d / 128), (unsigned)((m + kTile - 1) / kTile), (unsigned)(p * nchunks));
    k12_moment_reduce_ring<<<g, 256, sm, s>>>(X, ldx, Z, ldz, n, d, m, p, chunk, part, colpart,
                                              gpart, pg);
    return;
  }
  const int G = k12_g(d);
  const size_t sm = k12_smem(G);
  dim3 g((unsigned)((d + 32 * G - 1) / (32 * G)), (unsigned)((m + kTile - 1) / kTile),
         (unsigned)(p * nchunks));
  if (G == 4) {
    cudaFuncSetAttribute(k12_moment_reduce_dmma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    k12_moment_reduce_dmma<4><<<g, 256, sm, s>>>(X, ldx, Z, ldz, n, d, m, p, chunk, part, colpart,
                                                  gpart, pg);
  } else {
    cudaFuncSetAttribute(k12_moment_reduce_dmma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    k12_moment_reduce_dmma<2><<<g, 256, sm, s>>>(X, ldx, Z, ldz, n, d, m, p, chunk, part, colpart,
                                                  gpart, pg);
  }
}

// K14 on DMMA: grid (point tiles, column tiles), 8 warps; warp w owns points 16 (w % 4) .. +16
// x columns 32 (w / 4) .. +32.  K = (P-1) d: for t = 1..P-1 the A operand is x^(P-t) (staged in
// shared memory as fp64), B = c_t W_t.  hp_i = sum_k x_ik^P accumulates while staging.
// SUB (odd p's totals term, launch_lp_totals_expand): Y -= the same expansion.
template <int P, int G, int KS, bool SUB = false>
__global__ void __launch_bounds__(256)
    k14_moment_expand_dmma(const float *__restrict__ X, int64_t ldx, int64_t n, int64_t d,
                           int64_t m, const double *__restrict__ Wc,
                           const double *__restrict__ S, const double *__restrict__ G_,
                           double *__restrict__ Y, int64_t ldy) {
  constexpr int TR = 32 * G;  // points per CTA (warp w: rows 8 G (w % 4) .. +8 G)
  constexpr int XP = KS + 2, WP = kDmmaPad;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *xp = reinterpret_cast<double *>(smem_raw);  // [P-1][TR][XP]  slot t: x^(P-1-t)...
  double *ws = xp + (P - 1) * TR * XP;                  // [P-1][KS][WP]  c_t W_t
  __shared__ double s_hp[TR];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * TR, c0 = (int64_t)blockIdx.y * kTile;
  const int rw = 8 * G * (w % 4), cw = 32 * (w / 4);
  double acc[G][4][2];
#pragma unroll
  for (int a = 0; a < G; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  double hp = 0.0;  // threads 0..TR-1: point i0 + tid
  // register double buffering of the next k step's X and c_t W_t
  constexpr int PX = TR * KS / 256, PW = (P - 1) * KS * kTile / 256;
  float xr[PX];
  double wr[PW];
  auto load = [&](int64_t kb) {
#pragma unroll
    for (int u = 0; u < PX; ++u) {
      const int e = tid + 256 * u;
      const int r = e / KS, q = e - (e / KS) * KS;
      const int64_t i = i0 + r, k = kb + q;
      xr[u] = (i < n && k < d) ? X[i * ldx + k] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < PW; ++u) {
      const int e = tid + 256 * u;
      const int tt = e / (KS * kTile), rem = e - tt * (KS * kTile);
      const int q = rem / kTile, cc = rem - (rem / kTile) * kTile;
      const int64_t k = kb + q, c = c0 + cc;
      wr[u] = (k < d && c < m) ? Wc[((int64_t)tt * d + k) * m + c] : 0.0;
    }
  };
  load(0);
  for (int64_t kb = 0; kb < d; kb += KS) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PX; ++u) {
      const int e = tid + 256 * u;
      const int r = e / KS, q = e - (e / KS) * KS;
      const double x = (double)xr[u];
      double pw = x;  // slot tt (t = tt + 1) holds x^(P-t) = x^(P-1-tt)
#pragma unroll
      for (int e2 = 1; e2 < P; ++e2) {
        xp[((P - 1 - e2) * TR + r) * XP + q] = pw;
        pw *= x;
      }
    }
#pragma unroll
    for (int u = 0; u < PW; ++u) {
      const int e = tid + 256 * u;
      const int tt = e / (KS * kTile), rem = e - tt * (KS * kTile);
      const int q = rem / kTile, cc = rem - (rem / kTile) * kTile;
      ws[(tt * KS + q) * WP + cc] = wr[u];
    }
    __syncthreads();
    if (kb + KS < d) load(kb + KS);
    if (tid < TR) {  // x^P = x^(P-1) (slot 0) * x (slot P-2)
#pragma unroll 4
      for (int q = 0; q < KS; ++q)
        hp = fma(xp[tid * XP + q], xp[((P - 2) * TR + tid) * XP + q], hp);
    }
#pragma unroll
    for (int tt = 0; tt < P - 1; ++tt) {
#pragma unroll
      for (int kk = 0; kk < KS / 4; ++kk) {
        const int kq = 4 * kk + (lane & 3);
        double a[G], b[4];
#pragma unroll
        for (int g = 0; g < G; ++g)
          a[g] = xp[(tt * TR + rw + 8 * g + (lane >> 2)) * XP + kq];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = ws[(tt * KS + kq) * WP + cw + 8 * j + (lane >> 2)];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[g][j][0], acc[g][j][1], a[g], b[j]);
      }
    }
  }
  if (tid < TR) s_hp[tid] = hp;
  __syncthreads();
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int r = rw + 8 * g + (lane >> 2);
    const int64_t i = i0 + r;
    if (i >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t c = c0 + cw + 8 * j + 2 * (lane & 3) + h;
        if (c < m) {
          const double e = fma(S[c], s_hp[r], acc[g][j][h] + G_[c]);
          if constexpr (SUB)
            Y[i * ldy + c] -= e;
          else
            Y[i * ldy + c] = e;
        }
      }
  }
}

// launch K14 for P with (G, KS): 32 G points x 64 columns per CTA, KS coordinates per stage
template <int P, int G, int KS, bool SUB = false>
static void launch_k14(const float *X, int64_t ldx, int64_t n, int64_t d, int64_t m,
                       const double *Wc, const double *S, const double *Gc, double *Y,
                       int64_t ldy, cudaStream_t s) {
  constexpr int TR = 32 * G;
  const size_t sm = ((size_t)(P - 1) * TR * (KS + 2) + (size_t)(P - 1) * KS * kDmmaPad) *
                    sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k14_moment_expand_dmma<P, G, KS, SUB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  dim3 g((unsigned)((n + TR - 1) / TR), (unsigned)((m + kTile - 1) / kTile));
  k14_moment_expand_dmma<P, G, KS, SUB><<<g, 256, sm, s>>>(X, ldx, n, d, m, Wc, S, Gc, Y, ldy);
}

// W[t][k][c] = c_t * sum_ch part[ch][t][k][c]  (t = 1..p-1, scaled for the expand), plus
// S_c = sum_i z_ic (fixed-order two-level sum over point blocks) and G_c = sum_k W_p[k][c].
__global__ void __launch_bounds__(256)
    k13_moment_fold(const double *__restrict__ part, int64_t nchunks, int64_t d, int64_t m,
                    int T, int p, double *__restrict__ W) {
  const int64_t total = (int64_t)T * d * m;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    double s = 0.0;
    for (int64_t ch = 0; ch < nchunks; ++ch) s += part[ch * total + e];
    const int t = 1 + (int)(e / (d * m));
    if (t < p) {
      double coef = 1.0;  // C(p, t) (-1)^t
      for (int q = 0; q < t; ++q) coef = coef * (double)(p - q) / (double)(q + 1);
      W[e] = (t & 1) ? -coef * s : coef * s;
    } else {
      W[e] = s;  // raw (bilinear: W = X^T Z)
    }
  }
}

// G_c = sum_k W_p[k][c] = sum_j hp_j z_jc with hp_j = sum_k x_jk^p: a GEMV over the points, not
// a d x m moment (K12 skips t = p).  Per point chunk (one CTA): warp per point, lanes over
// coordinates for hp (fixed shuffle tree) and over columns for the products; the CTA's partial
// goes to gpart[ch][c] (folded in fixed order by k13_colsum).
__global__ void __launch_bounds__(256)
    k13_gpart(const float *__restrict__ X, int64_t ldx, const float *__restrict__ Z, int64_t ldz,
              int64_t n, int64_t d, int64_t m, int p, int64_t chunk, double *__restrict__ gpart) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *acc = reinterpret_cast<double *>(smem_raw);  // [8][m]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t e = threadIdx.x; e < 8 * m; e += 256) acc[e] = 0.0;
  __syncthreads();
  const int64_t ch = blockIdx.x;
  const int64_t i0 = ch * chunk, i1 = (i0 + chunk < n) ? i0 + chunk : n;
  double *aw = acc + w * m;
  for (int64_t ib = i0 + w; ib < i1; ib += 32) {  // 4 points per warp step (independent loads)
    double hp[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = ib + 8 * u;
      hp[u] = 0.0;
      if (i < i1)
        for (int64_t k = lane; k < d; k += 32) hp[u] += powi((double)__ldg(X + i * ldx + k), p);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int off = 16; off; off >>= 1) hp[u] += __shfl_xor_sync(0xFFFFFFFFu, hp[u], off);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = ib + 8 * u;
      if (i >= i1) break;
      for (int64_t c = lane; c < m; c += 32)
        aw[c] = fma(hp[u], (double)__ldg(Z + i * ldz + c), aw[c]);
    }
  }
  __syncthreads();
  for (int64_t c = threadIdx.x; c < m; c += 256) {
    double g = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) g += acc[ww * m + c];
    gpart[ch * m + c] = g;
  }
}

__global__ void __launch_bounds__(256)
    k13_colsum(const double *__restrict__ gpart, const double *__restrict__ colpart,
               int64_t nchunks, int64_t m, double *__restrict__ S, double *__restrict__ G) {
  // one CTA per column: S_c and G_c from the chunks' partials (K12's column sums, k13_gpart)
  // in fixed order per thread, then a fixed-shape tree
  __shared__ double rs[256], rg[256];
  const int64_t c = blockIdx.x;
  double s = 0.0, g = 0.0;
  for (int64_t ch = threadIdx.x; ch < nchunks; ch += 256) {
    s += colpart[ch * m + c];
    g += gpart[ch * m + c];
  }
  rs[threadIdx.x] = s;
  rg[threadIdx.x] = g;
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if ((int)threadIdx.x < w) {
      rs[threadIdx.x] += rs[threadIdx.x + w];
      rg[threadIdx.x] += rg[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    S[c] = rs[0];
    G[c] = rg[0];
  }
}

// V[k][c] = sum_l M[k][l] W[l][c] (d x d times d x m; tiny next to the two contractions).
__global__ void __launch_bounds__(256)
    k15_small_gemm(const double *__restrict__ M, const double *__restrict__ W, int64_t d,
                   int64_t m, double *__restrict__ V) {
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < d * m;
       e += (int64_t)gridDim.x * 256) {
    const int64_t k = e / m, c = e - (e / m) * m;
    double s = 0.0;
    for (int64_t l = 0; l < d; ++l) s = fma(M[k * d + l], W[l * m + c], s);
    V[e] = s;
  }
}

__global__ void k15_zero(double *__restrict__ a, int64_t count) {
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * 256)
    a[e] = 0.0;
}

// Thm. l2embed: X'[i][r] = (1 / (beta k)) sum_j G[r][j] x_ij, beta = sqrt(2/pi),
// fp64 accumulation rounded once to fp32 (the l1 engine's input type).  grid: (point tiles,
// embedding-row tiles); block 16 x 16 threads, outputs (ty + 16u, tx + 16v).
__global__ void __launch_bounds__(256)
    k16_embed(const float *__restrict__ X, int64_t ldx, int64_t n, int64_t d,
              const float *__restrict__ G, int64_t ldg, int64_t k, double scale,
              float *__restrict__ Xp, int64_t ldp) {
  __shared__ double xs[kStepK][kTile + 1];  // [coordinate][point]
  __shared__ double gs[kStepK][kTile + 1];  // [coordinate][embedding row]
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = (int64_t)blockIdx.x * kTile, r0 = (int64_t)blockIdx.y * kTile;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t jb = 0; jb < d; jb += kStepK) {
    __syncthreads();
    for (int e = threadIdx.x; e < kTile * kStepK; e += 256) {
      const int row = e / kStepK, q = e - (e / kStepK) * kStepK;
      const int64_t j = jb + q;
      xs[q][row] = (i0 + row < n && j < d) ? (double)X[(i0 + row) * ldx + j] : 0.0;
      gs[q][row] = (r0 + row < k && j < d) ? (double)G[(r0 + row) * ldg + j] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kStepK; ++q) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = xs[q][ty + 16 * u];
        b[u] = gs[q][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = i0 + ty + 16 * u;
    if (i >= n) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t r = r0 + tx + 16 * v;
      if (r < k) Xp[i * ldp + r] = (float)(acc[u][v] * scale);
    }
  }
}

}  // namespace

int launch_embed(const float *X, int64_t ldx, int64_t n, int64_t d, const float *G, int64_t ldg,
                 int64_t k, float *Xp, int64_t ldp, cudaStream_t s) {
  const double beta = 0.79788456080286535588;  // sqrt(2 / pi)
  dim3 grid((unsigned)((n + kTile - 1) / kTile), (unsigned)((k + kTile - 1) / kTile));
  k16_embed<<<grid, 256, 0, s>>>(X, ldx, n, d, G, ldg, k, 1.0 / (beta * (double)k), Xp, ldp);
  return 1;
}

size_t bilinear_workspace(int64_t n, int64_t d, int64_t m, int sms) {
  // lpp_even's layout at p = 1 (partials | W | S | G) + V (d x m)
  return lpp_even_workspace(n, d, m, 1, nullptr, nullptr, sms) + (size_t)d * m * sizeof(double);
}

// Thm. maha: f(x, y) = x^T M y, A = X M X^T, Y = X (M (X^T Z)): Alg. 7's S = M X^T
// is never formed; W = X^T Z (k12 at p = 1), V = M W (k15), Y = X V (k14 with S = G = 0).
int launch_bilinear(const float *X, int64_t ldx, const double *M, const float *Z, int64_t ldz,
                    int64_t n, int64_t d, int64_t m, double *Y, int64_t ldy, double *ws, int sms,
                    cudaStream_t s) {
  int64_t nchunks = 1, chunk = n;
  lpp_even_workspace(n, d, m, 1, &nchunks, &chunk, sms);
  double *part = ws;
  double *W = part + (size_t)nchunks * d * m;
  double *S = W + (size_t)d * m;
  double *G = S + m;
  double *V = G + m;
  launch_k12(X, ldx, Z, ldz, n, d, m, 1, chunk, nchunks, part, nullptr, nullptr, 0, s);
  int64_t b13 = (d * m + 255) / 256;
  if (b13 > 148 * 8) b13 = 148 * 8;
  k13_moment_fold<<<(unsigned)b13, 256, 0, s>>>(part, nchunks, d, m, 1, 1, W);
  k15_small_gemm<<<(unsigned)b13, 256, 0, s>>>(M, W, d, m, V);
  k15_zero<<<1, 256, 0, s>>>(S, 2 * m);  // S and G (adjacent): no h S or G term
  launch_k14<2, 4, 32>(X, ldx, n, d, m, V, S, G, Y, ldy, s);
  return 5;  // k12, k13 fold, k15 gemm, k15 zero, k14
}

size_t lpp_even_workspace(int64_t n, int64_t d, int64_t m, int p, int64_t *nchunks_out,
                          int64_t *chunk_out, int sms) {
  const int64_t tk = 32 * k12_g(d);
  const int T = p > 1 ? p - 1 : 1;  // moments through DMMA: t = 1 .. p-1 (bilinear: 1)
  const int64_t tiles = ((d + tk - 1) / tk) * ((m + kTile - 1) / kTile) * T;
  // point chunks for ~2 CTAs per SM (one wave) with a single moment, ~4 with several (measured:
  // p = 2 1.73 vs 1.78 ms; p = 4 5.07 vs 5.96 ms)
  const int64_t per_sm = T == 1 ? L1DM_EVEN_CTAS_PER_SM : 2 * L1DM_EVEN_CTAS_PER_SM;
  int64_t nchunks = (per_sm * (int64_t)sms + tiles - 1) / tiles;
  const int64_t min_pts = 1024;
  if (nchunks * min_pts > n) nchunks = (n + min_pts - 1) / min_pts;
  if (nchunks < 1) nchunks = 1;
  const int64_t chunk = (n + nchunks - 1) / nchunks;
  nchunks = (n + chunk - 1) / chunk;
  if (nchunks_out) *nchunks_out = nchunks;
  if (chunk_out) *chunk_out = chunk;
  // partials (nchunks x T x d x m) | W (T x d x m) | S (m) | G (m) | column partials |
  // G partials (nchunks x m each)
  return ((size_t)nchunks * T * d * m + (size_t)T * d * m + 2 * (size_t)m +
          2 * (size_t)nchunks * m) * sizeof(double);
}

int launch_lpp_even(const float *X, int64_t ldx, const float *Z, int64_t ldz, int64_t n,
                    int64_t d, int64_t m, int p, double *Y, int64_t ldy, double *ws, int sms,
                    cudaStream_t s) {
  int64_t nchunks = 1, chunk = n;
  lpp_even_workspace(n, d, m, p, &nchunks, &chunk, sms);
  const int T = p - 1;  // even p >= 2: W_1 .. W_{p-1} on DMMA; W_p enters only through G
  double *part = ws;
  double *W = part + (size_t)nchunks * T * d * m;
  double *S = W + (size_t)T * d * m;
  double *G = S + m;
  double *colpart = G + m;
  double *gpart = colpart + (size_t)nchunks * m;
  launch_k12(X, ldx, Z, ldz, n, d, m, T, chunk, nchunks, part, colpart, gpart, p, s);
  const bool fused_g = d <= 32 * k12_g(d);  // one coordinate tile: K12 summed hp z itself
  if (!fused_g) {
    const size_t smg = (size_t)8 * m * sizeof(double);
    static bool gattr = false;
    if (!gattr) {
      cudaFuncSetAttribute(k13_gpart, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      gattr = true;
    }
    k13_gpart<<<(unsigned)nchunks, 256, smg, s>>>(X, ldx, Z, ldz, n, d, m, p, chunk, gpart);
  }
  int64_t b13 = ((int64_t)T * d * m + 255) / 256;
  if (b13 > 148 * 8) b13 = 148 * 8;
  k13_moment_fold<<<(unsigned)b13, 256, 0, s>>>(part, nchunks, d, m, T, p, W);
  k13_colsum<<<(unsigned)m, 256, 0, s>>>(gpart, colpart, nchunks, m, S, G);
  switch (p) {
    case 2: launch_k14<2, L1DM_K14_P2_G, L1DM_K14_P2_KS>(X, ldx, n, d, m, W, S, G, Y, ldy, s); break;
    case 4: launch_k14<4, 4, 16>(X, ldx, n, d, m, W, S, G, Y, ldy, s); break;
    case 6: launch_k14<6, 2, kStepK>(X, ldx, n, d, m, W, S, G, Y, ldy, s); break;
    default: return 3;
  }
  return fused_g ? 4 : 5;  // k12, (k13 G partials), k13 fold, k13 colsum, k14
}

// ---- odd p in one pass (DESIGN.md §2b / §6): the coordinate totals' part of each point's value,
//   E_ic = sum_k sum_t c_t x_ik^(P-t) T_ktc,   c_t = C(P, t) (-1)^t,
// with T_ktc = sum_j z_jc x_jk^t the segment totals the single-pass apply leaves in segtot (rows of
// ld_seg: (P+1) moments per column).  t = 0 is S_c hp_i (T_k0c = S_c for every k, hp_i = sum_k
// x_ik^P), t = P is the constant c_P sum_k T_kPc, 1 <= t < P is the DMMA expansion of K14 with
// W_t = c_t T_t.  Y -= E.
__global__ void __launch_bounds__(256)
    k14b_lp_totals(const double *__restrict__ segtot, int64_t ld_seg, int64_t dl, int64_t m, int P,
                   double *__restrict__ W, double *__restrict__ S, double *__restrict__ Gc) {
  const int K = P + 1;
  const int64_t total = (int64_t)(P - 1) * dl * m;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total + m;
       e += (int64_t)gridDim.x * 256) {
    if (e < total) {  // W[t-1][k][c] = c_t T_ktc
      const int64_t tt = e / (dl * m), rem = e - tt * dl * m, k = rem / m, c = rem - k * m;
      const int t = (int)tt + 1;
      double b = 1.0;  // C(P, t)
      for (int q = 0; q < t; ++q) b = b * (double)(P - q) / (double)(q + 1);
      W[e] = ((t & 1) ? -b : b) * segtot[k * ld_seg + K * c + t];
    } else {  // column c: S_c and c_P sum_k T_kPc (fixed order)
      const int64_t c = e - total;
      double g = 0.0;
      for (int64_t k = 0; k < dl; ++k) g += segtot[k * ld_seg + K * c + P];
      S[c] = segtot[K * c];
      Gc[c] = (P & 1) ? -g : g;
    }
  }
}

size_t lp_totals_workspace(int64_t dl, int64_t m, int p) {
  return ((size_t)(p - 1) * dl * m + 2 * (size_t)m) * sizeof(double);
}

int launch_lp_totals_expand(const float *X, int64_t ldx, int64_t n, int64_t dl, int64_t m,
                            const double *segtot, int64_t ld_seg, int p, double *work, double *Y,
                            int64_t ldy, cudaStream_t s) {
  double *W = work, *S = W + (size_t)(p - 1) * dl * m, *G = S + m;
  int64_t b = ((int64_t)(p - 1) * dl * m + m + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  k14b_lp_totals<<<(unsigned)b, 256, 0, s>>>(segtot, ld_seg, dl, m, p, W, S, G);
  switch (p) {
    case 3: launch_k14<3, 4, 16, true>(X, ldx, n, dl, m, W, S, G, Y, ldy, s); break;
    case 5: launch_k14<5, 4, 16, true>(X, ldx, n, dl, m, W, S, G, Y, ldy, s); break;
    case 7: launch_k14<7, 2, 16, true>(X, ldx, n, dl, m, W, S, G, Y, ldy, s); break;
    default: return 1;
  }
  return 2;
}

}  // namespace l1dm
