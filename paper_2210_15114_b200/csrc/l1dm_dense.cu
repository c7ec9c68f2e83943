// l1dm_dense.cu — the dense fp64 steps of the matrix-free consumers (
// Thm. musco, Thm. bakshi22, Thm. linear_system).
//
// The consumers touch A only through the block product (Lemma matrixmult); between
// products they need a handful of dense fp64 operations on tall n x b blocks and on small
// (q b) x (q b) matrices.  All of them run here, on the device, in stream order:
//
//   k40_gemm<TA, WM, WN>  C = alpha op(A) B + beta C on the fp64 tensor cores (DMMA,
//                         mma.sync m8n8k4 f64): TA = 1 is the tall-skinny reduction A^T B
//                         (Gram matrices, Gram-Schmidt coefficients, the Rayleigh quotient),
//                         split over K with a fixed-order fold (deterministic); TA = 0 is the
//                         tall update A W (projections, basis rotations).
//   k42_jacobi_*          symmetric eigen-decomposition by cyclic two-sided Jacobi with the
//                         round-robin ("circle") pair ordering: every step rotates N/2 disjoint
//                         pairs at once, so each 2 x 2 block of A and each row pair of V is
//                         updated by exactly one thread.  N <= 96: one CTA, A and V in shared
//                         memory; larger N: a cooperative grid (grid-wide barrier per phase),
//                         A and V in global memory (L2-resident at the sizes used).
//   k44_select ...        ordering of eigenvalues by |lambda|, column scalings, the hi/lo split
//                         of an fp64 block into the fp32 query type and the recombination, and
//                         the dot products / updates of conjugate gradients with device scalars.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "l1dm_device.cuh"
#include "l1dm_internal.h"

namespace cg = cooperative_groups;

namespace l1dm {
namespace {

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------------------------------- GEMM
// op(A)(m, k) = TA ? A[k lda + m] : A[m lda + k];  B(k, n) = B[k ldb + n].
// CTA tile (16 WM) x (32 WN), K stage 16; warp tile 16 x 32 = 2 x 4 DMMA 8x8 tiles.
// Shared layouts (padded so every fragment load is the minimum two wavefronts):
//   TA = 1: As[k][m] (row stride BM + 8)   TA = 0: As[m][k] (row stride 16 + 4)
//   Bs[k][n] (row stride BN + 8)
constexpr int GK = 16;

template <int TA, int WM, int WN, int KS = 1, int MI = 2>
struct GemmCfg {
  static_assert(WM * WN * KS == 8, "8 warps per CTA");
  // warp tile (8 MI) x 32: MI x 4 DMMA 8x8 tiles
  static constexpr int BM = 8 * MI * WM, BN = 32 * WN, SK = GK * KS;  // SK: rows per stage
  static constexpr int ALD = TA ? BM + 8 : SK + 4;   // As row stride (doubles)
  static constexpr int AROWS = TA ? SK : BM;
  static constexpr int BLD = BN + 8;
  static constexpr int A_ELEMS = BM * SK, B_ELEMS = SK * BN;
  static constexpr int AL = A_ELEMS / 256, BL = B_ELEMS / 256;  // per-thread loads per stage
  static constexpr size_t SMEM = 2 * ((size_t)AROWS * ALD + (size_t)SK * BLD) * sizeof(double);
  static_assert(KS == 1 || (size_t)(KS - 1) * BM * BN * sizeof(double) <= SMEM, "k-slice fold");
};

// KS > 1 (small M x N, long K): the 8 warps split each stage's rows into KS slices of 16 and
// their partial tiles are summed through shared memory at the end (fixed order).
template <int TA, int WM, int WN, int KS, int MI>
__global__ void __launch_bounds__(256)
    k40_gemm(int64_t M, int64_t N, int64_t K, const double *__restrict__ A, int64_t lda,
             const double *__restrict__ B, int64_t ldb, int64_t kchunk, double *__restrict__ C,
             int64_t ldc, double alpha, double beta, int direct) {
  using Cf = GemmCfg<TA, WM, WN, KS, MI>;
  constexpr int BM = Cf::BM, BN = Cf::BN, ALD = Cf::ALD, BLD = Cf::BLD, AROWS = Cf::AROWS;
  constexpr int AL = Cf::AL, BL = Cf::BL, SK = Cf::SK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *As = reinterpret_cast<double *>(smem_raw);  // [2][AROWS][ALD]
  double *Bs = As + 2 * AROWS * ALD;                  // [2][SK][BLD]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w % WM, wn = (w / WM) % WN, wk = w / (WM * WN);
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t kb = (int64_t)blockIdx.z * kchunk;
  const int64_t ke = (kb + kchunk < K) ? kb + kchunk : K;

  double ra[AL], rb[BL];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < AL; ++i) {
      const int e = tid + 256 * i;
      int mm, kk;
      if (TA) { kk = e / BM; mm = e % BM; } else { mm = e / SK; kk = e % SK; }
      const int64_t gm = m0 + mm, gk = k0 + kk;
      ra[i] = (gm < M && gk < ke) ? (TA ? __ldg(A + gk * lda + gm) : __ldg(A + gm * lda + gk)) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < BL; ++i) {
      const int e = tid + 256 * i;
      const int kk = e / BN, nn = e % BN;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      rb[i] = (gn < N && gk < ke) ? __ldg(B + gk * ldb + gn) : 0.0;
    }
  };
  auto store = [&](int buf) {
    double *as = As + buf * AROWS * ALD;
    double *bs = Bs + buf * SK * BLD;
#pragma unroll
    for (int i = 0; i < AL; ++i) {
      const int e = tid + 256 * i;
      if (TA) as[(e / BM) * ALD + (e % BM)] = ra[i];
      else as[(e / SK) * ALD + (e % SK)] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < BL; ++i) {
      const int e = tid + 256 * i;
      bs[(e / BN) * BLD + (e % BN)] = rb[i];
    }
  };
  double acc[MI][4][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  int buf = 0;
  if (kb < ke) {
    load(kb);
    store(0);
  }
  __syncthreads();
  for (int64_t k0 = kb; k0 < ke; k0 += SK) {
    const bool more = k0 + SK < ke;
    if (more) load(k0 + SK);  // next stage in flight during this stage's DMMAs
    const double *as = As + buf * AROWS * ALD;
    const double *bs = Bs + buf * SK * BLD;
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      const int kk = wk * GK + ks * 4 + (lane & 3);
      double a[MI], b[4];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int mm = wm * 8 * MI + i * 8 + (lane >> 2);
        a[i] = TA ? as[kk * ALD + mm] : as[mm * ALD + kk];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[kk * BLD + wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  if constexpr (KS > 1) {  // k-slice partials: slices 1.. park theirs, slice 0 adds them in order
    __syncthreads();
    double *red = As;  // [KS-1][BM][BN]
    if (wk > 0) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = wm * 8 * MI + i * 8 + (lane >> 2), c = wn * 32 + j * 8 + (lane & 3) * 2 + h;
            red[((size_t)(wk - 1) * BM + r) * BN + c] = acc[i][j][h];
          }
    }
    __syncthreads();
    if (wk > 0) return;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm * 8 * MI + i * 8 + (lane >> 2), c = wn * 32 + j * 8 + (lane & 3) * 2 + h;
          for (int q = 0; q < KS - 1; ++q) acc[i][j][h] += red[((size_t)q * BM + r) * BN + c];
        }
  }
  // epilogue: lane holds C[row][col], C[row][col + 1] of each 8x8 tile
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = m0 + wm * 8 * MI + i * 8 + (lane >> 2);
        const int64_t c = n0 + wn * 32 + j * 8 + (lane & 3) * 2 + h;
        if (r >= M || c >= N) continue;
        if (direct) {
          double *p = C + r * ldc + c;
          const double v = alpha * acc[i][j][h];
          *p = (beta != 0.0) ? fma(beta, *p, v) : v;
        } else {
          C[((int64_t)blockIdx.z * M + r) * N + c] = acc[i][j][h];  // partial of split z
        }
      }
}

// C = alpha sum_s P[s] + beta C, the splits summed in index order (deterministic).
__global__ void __launch_bounds__(256)
    k41_gemm_fold(int64_t M, int64_t N, int64_t S, const double *__restrict__ P, double *C,
                  int64_t ldc, double alpha, double beta) {
  const int64_t total = M * N;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    double s = 0.0;
    int64_t z = 0;
    for (; z + 8 <= S; z += 8) {  // eight loads in flight, added in index order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = P[(z + u) * total + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; z < S; ++z) s += P[z * total + e];
    const int64_t r = e / N, c = e - (e / N) * N;
    double *p = C + r * ldc + c;
    const double v = alpha * s;
    *p = (beta != 0.0) ? fma(beta, *p, v) : v;
  }
}

// ---- skinny GEMMs of the Krylov block steps (one dimension = the n points, the others <= 96)
// Bandwidth-bound shapes, so no shared-memory staging: DMMA fragments are loaded straight from
// global memory (lane l: rows k0 + l % 4, columns 8 t + l / 4 — four 64-byte row pieces per load
// instruction), several k-steps of loads in flight per warp.
//
// k44_skinny_tn<MT, NT>: partial C (M x N, M <= 8 MT, N <= 8 NT) = A^T B over a contiguous row
// range per warp; the 8 warps' tiles are summed in a fixed order through shared memory and each
// CTA writes its partial to P[blockIdx.x][M][N] (folded by k41_gemm_fold in CTA order).
// SYM (a Gram matrix: B = A, M = N): only the tiles i <= j are computed and the rest mirrored.
template <int MT, int NT, bool SYM = false>
__global__ void __launch_bounds__(256)
    k44_skinny_tn(int64_t M, int64_t N, int64_t K, const double *__restrict__ A, int64_t lda,
                  const double *__restrict__ B, int64_t ldb, int64_t rows_per_warp,
                  double *__restrict__ P) {
  static_assert(!SYM || MT == NT, "a Gram matrix is square");
  constexpr int U = MT * NT > 16 ? 2 : 4;  // k-steps (of 4 rows) in flight per warp
  __shared__ double red[MT * 8][NT * 8 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * 8 + w;
  const int64_t r0 = gw * rows_per_warp;
  const int64_t r1 = (r0 + rows_per_warp < K) ? r0 + rows_per_warp : K;
  const int kr = lane & 3, cl = lane >> 2;
  bool mok[MT], nok[NT];
#pragma unroll
  for (int t = 0; t < MT; ++t) mok[t] = 8 * t + cl < M;
#pragma unroll
  for (int t = 0; t < NT; ++t) nok[t] = 8 * t + cl < N;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int64_t k0 = r0; k0 < r1; k0 += 4 * U) {
    double a[U][MT], b[U][NT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + 4 * u + kr;
      const bool ok = k < r1;
#pragma unroll
      for (int t = 0; t < MT; ++t) a[u][t] = (ok && mok[t]) ? __ldg(A + k * lda + 8 * t + cl) : 0.0;
#pragma unroll
      for (int t = 0; t < NT; ++t)
        b[u][t] = SYM ? a[u][t < MT ? t : 0] : ((ok && nok[t]) ? __ldg(B + k * ldb + 8 * t + cl) : 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
          if (!SYM || i <= j) dmma884(acc[i][j][0], acc[i][j][1], a[u][i], b[u][j]);
  }
  // lane holds C[8 i + l / 4][8 j + 2 (l % 4) + h]; the warps add theirs in index order
  for (int q = 0; q < 8; ++q) {
    if (w == q) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (SYM && i > j) continue;
            double &r = red[8 * i + cl][8 * j + 2 * kr + h];
            r = (q == 0) ? acc[i][j][h] : r + acc[i][j][h];
          }
    }
    __syncthreads();
  }
  const int64_t tot = M * N;
  for (int64_t e = threadIdx.x; e < tot; e += 256) {
    const int r = (int)(e / N), c = (int)(e - (e / N) * N);
    P[(int64_t)blockIdx.x * tot + e] = (SYM && r / 8 > c / 8) ? red[c][r] : red[r][c];
  }
}

// k45_skinny_nn<NT, KQ, TU>: C (M x N, N <= 8 NT) = alpha A (M x K) B (K x N) + beta C with
// K <= 4 KQ and M the n points: B staged in shared memory once per CTA; each warp computes TU
// 8-row tiles of C per step (grid-stride), all their A fragments loaded straight from global
// memory before any DMMA (TU x KQ loads in flight per lane).
template <int NT, int KQ, int TU>
__global__ void __launch_bounds__(256)
    k45_skinny_nn(int64_t M, int64_t N, int64_t K, const double *__restrict__ A, int64_t lda,
                  const double *__restrict__ B, int64_t ldb, double alpha, double beta,
                  double *__restrict__ C, int64_t ldc) {
  __shared__ double bs[4 * KQ][NT * 8 + 1];
  for (int e = threadIdx.x; e < 4 * KQ * NT * 8; e += 256) {
    const int kk = e / (NT * 8), nn = e - (e / (NT * 8)) * (NT * 8);
    bs[kk][nn] = (kk < K && nn < N) ? B[(int64_t)kk * ldb + nn] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int kr = lane & 3, cl = lane >> 2;
  const int ksteps = (int)((K + 3) / 4);
  const bool vec2 = (ldc % 2 == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
  const int64_t tiles = (M + 7) / 8;
  const int64_t stride = (int64_t)gridDim.x * 8;
  for (int64_t t0 = (int64_t)blockIdx.x * 8 + w; t0 < tiles; t0 += stride * TU) {
    double a[TU][KQ];
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      const int64_t row = 8 * (t0 + u * stride) + cl;
      const bool rok = row < M;
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const int kk = 4 * q + kr;
        a[u][q] = (rok && kk < K) ? __ldg(A + row * lda + kk) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      const int64_t row = 8 * (t0 + u * stride) + cl;
      double acc[NT][2];
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        if (q >= ksteps) break;
#pragma unroll
        for (int j = 0; j < NT; ++j)
          dmma884(acc[j][0], acc[j][1], a[u][q], bs[4 * q + kr][8 * j + cl]);
      }
      if (row >= M) continue;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int64_t c = 8 * j + 2 * kr;
        double *p = C + row * ldc + c;
        if (vec2 && c + 1 < N) {  // whole 16-byte pairs: every warp store fills 32-byte sectors
          double2 v = make_double2(alpha * acc[j][0], alpha * acc[j][1]);
          if (beta != 0.0) {
            const double2 o = *reinterpret_cast<const double2 *>(p);
            v.x = fma(beta, o.x, v.x);
            v.y = fma(beta, o.y, v.y);
          }
          *reinterpret_cast<double2 *>(p) = v;
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (c + h >= N) continue;
            const double v = alpha * acc[j][h];
            p[h] = (beta != 0.0) ? fma(beta, p[h], v) : v;
          }
        }
      }
    }
  }
}

// The same fold for many partials (the skinny TN's one per CTA): a warp per element, lane l
// summing partials l, l + 32, ... in order, then a fixed butterfly (deterministic).
__global__ void __launch_bounds__(256)
    k41b_gemm_fold_warp(int64_t M, int64_t N, int64_t S, const double *__restrict__ P, double *C,
                        int64_t ldc, double alpha, double beta) {
  const int lane = threadIdx.x & 31;
  const int64_t e = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5), total = M * N;
  if (e >= total) return;
  double s = 0.0;
  for (int64_t z = lane; z < S; z += 32) s += P[z * total + e];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  if (lane == 0) {
    const int64_t r = e / N, c = e - (e / N) * N;
    double *p = C + r * ldc + c;
    const double v = alpha * s;
    *p = (beta != 0.0) ? fma(beta, *p, v) : v;
  }
}

template <int TA, int WM, int WN, int KS, int MI = 2>
int gemm_t(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda,
           const double *B, int64_t ldb, double beta, double *C, int64_t ldc, double *ws,
           int64_t splits, cudaStream_t s) {
  using Cf = GemmCfg<TA, WM, WN, KS, MI>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k40_gemm<TA, WM, WN, KS, MI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cf::SMEM);
    attr = true;
  }
  const int64_t mt = (M + Cf::BM - 1) / Cf::BM, nt = (N + Cf::BN - 1) / Cf::BN;
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = (kchunk + Cf::SK - 1) / Cf::SK * Cf::SK;
  splits = (K + kchunk - 1) / kchunk;
  if (splits < 1) splits = 1;
  dim3 g((unsigned)mt, (unsigned)nt, (unsigned)splits);
  if (splits == 1) {
    k40_gemm<TA, WM, WN, KS, MI><<<g, 256, Cf::SMEM, s>>>(M, N, K, A, lda, B, ldb, kchunk, C, ldc,
                                                      alpha, beta, 1);
    return 1;
  }
  k40_gemm<TA, WM, WN, KS, MI><<<g, 256, Cf::SMEM, s>>>(M, N, K, A, lda, B, ldb, kchunk, ws, N, 1.0,
                                                    0.0, 0);
  const int64_t tot = M * N;
  if (splits >= 64 && tot <= 148 * 64) {  // many partials of a small C: a warp per element
    k41b_gemm_fold_warp<<<(unsigned)((tot + 7) / 8), 256, 0, s>>>(M, N, splits, ws, C, ldc,
                                                                  alpha, beta);
    return 2;
  }
  int64_t fb = (tot + 255) / 256;
  if (fb > 148 * 8) fb = 148 * 8;
  k41_gemm_fold<<<(unsigned)(fb < 1 ? 1 : fb), 256, 0, s>>>(M, N, splits, ws, C, ldc, alpha,
                                                            beta);
  return 2;
}

// Split-K factor of the TN reduction (A^T B over the n points): enough CTAs to hide the
// operand loads' latency — measured on B200, the tall basis products (M > 64, N = 32) run best
// with ~8 CTAs per SM (2.13 ms vs 3.48 ms at 2 per SM for 608 x 32 x 2^20), the Gram-sized
// ones with ~2.
int64_t gemm_splits(int ta, int64_t M, int64_t N, int64_t K, int sms) {
  if (!ta) return 1;  // A W: K is a basis width (small); M (points) gives the parallelism
  const bool narrow = N <= 32;
  const int64_t bm = (M <= 32 && narrow) ? 32 : (M <= 64 && narrow) ? 64 : narrow ? 128 : 64;
  const int64_t bn = narrow ? 32 : 64;
  const int64_t per_sm = (narrow && M > 64) ? 8 : 2;
  const int64_t tiles = ((M + bm - 1) / bm) * ((N + bn - 1) / bn);
  int64_t sp = (per_sm * (int64_t)sms + tiles - 1) / tiles;
  const int64_t kmax = (K + 255) / 256;  // at least 256 rows per split
  if (sp > kmax) sp = kmax;
  return sp < 1 ? 1 : sp;
}

// ------------------------------------------------------------------------------------ Jacobi
// Round-robin pairing of N2 (even) indices at step s in [0, N2 - 1): position 0 holds index 0,
// positions 1..N2-1 rotate; pair i joins positions i and N2-1-i.  Over N2-1 steps every pair of
// indices meets exactly once (one cyclic sweep).
__device__ __forceinline__ void rr_pair(int i, int step, int N2, int &p, int &q) {
  const int L = N2 - 1;
  p = (i == 0) ? 0 : ((i - 1 + step) % L) + 1;
  q = ((N2 - 2 - i + step) % L) + 1;
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

constexpr double c_jac_rel = 1e-16;  // relative threshold (measured: 8-12 sweeps up to N = 640)
constexpr double c_jac_abs = 1e-30;  // absolute floor, relative to ||A||_F (zero diagonals)
// Rotation annihilating a_pq (Rutishauser): theta = (a_qq - a_pp) / (2 a_pq),
// t = sign(theta) / (|theta| + sqrt(theta^2 + 1)), c = 1/sqrt(1 + t^2), s = t c, applied as
// A' = J^T A J with J_pp = J_qq = c, J_pq = s, J_qp = -s.  Skipped (t = 0) when |a_pq| is below
// 1e-16 sqrt(|a_pp a_qq|) (relative accuracy reached) or below an absolute floor.
__device__ __forceinline__ bool jacobi_rot(double app, double aqq, double apq, double floor_abs,
                                           double &c, double &s, double &t) {
  const double aa = fabs(apq);
  if (!(aa > floor_abs) || aa <= c_jac_rel * sqrt(fabs(app) * fabs(aqq))) {
    c = 1.0;
    s = 0.0;
    t = 0.0;
    return false;
  }
  const double theta = (aqq - app) / (2.0 * apq);
  t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
  c = 1.0 / sqrt(fma(t, t, 1.0));
  s = t * c;
  return true;
}

// One Jacobi step's element updates for pair blocks [e0, e1) (stride es) of A and row pairs
// of V; rot[i] = (c, s, t) of pair i (t = 0: identity).  Exactly one thread owns each 2 x 2
// block of A and each (row, pair) of V, so the updates are in place.
__device__ __forceinline__ void jacobi_apply(double *a, int64_t lda, double *v, int64_t ldv,
                                             int N, int N2, int step, const double *rot,
                                             int64_t tid, int64_t nth) {
  const int H = N2 / 2;
  const int64_t nblk = (int64_t)H * H;
  for (int64_t e = tid; e < nblk; e += nth) {
    const int i = (int)(e / H), j = (int)(e - (e / H) * H);
    const double ti = rot[3 * i + 2], tj = rot[3 * j + 2];
    if (ti == 0.0 && tj == 0.0) continue;
    int pi, qi, pj, qj;
    rr_pair(i, step, N2, pi, qi);
    rr_pair(j, step, N2, pj, qj);
    const double ci = rot[3 * i], si = rot[3 * i + 1], cj = rot[3 * j], sj = rot[3 * j + 1];
    if (i == j) {
      // diagonal block: the stable forms a_pp - t a_pq, a_qq + t a_pq, a_pq = 0
      if (qi >= N) continue;
      const double apq = a[(int64_t)pi * lda + qi];
      a[(int64_t)pi * lda + pi] -= ti * apq;
      a[(int64_t)qi * lda + qi] += ti * apq;
      a[(int64_t)pi * lda + qi] = 0.0;
      a[(int64_t)qi * lda + pi] = 0.0;
      continue;
    }
    const bool qiv = qi < N, qjv = qj < N;  // index N (odd N's pad) does not exist
    double b00 = a[(int64_t)pi * lda + pj];
    double b01 = qjv ? a[(int64_t)pi * lda + qj] : 0.0;
    double b10 = qiv ? a[(int64_t)qi * lda + pj] : 0.0;
    double b11 = (qiv && qjv) ? a[(int64_t)qi * lda + qj] : 0.0;
    // rows: J_i^T B
    const double r00 = ci * b00 - si * b10, r01 = ci * b01 - si * b11;
    const double r10 = si * b00 + ci * b10, r11 = si * b01 + ci * b11;
    // columns: (J_i^T B) J_j
    a[(int64_t)pi * lda + pj] = cj * r00 - sj * r01;
    if (qjv) a[(int64_t)pi * lda + qj] = sj * r00 + cj * r01;
    if (qiv) a[(int64_t)qi * lda + pj] = cj * r10 - sj * r11;
    if (qiv && qjv) a[(int64_t)qi * lda + qj] = sj * r10 + cj * r11;
  }
  const int64_t nv = (int64_t)N * H;
  for (int64_t e = tid; e < nv; e += nth) {
    const int r = (int)(e / H), j = (int)(e - (e / H) * H);
    if (rot[3 * j + 2] == 0.0) continue;
    int pj, qj;
    rr_pair(j, step, N2, pj, qj);
    if (qj >= N) continue;
    const double c = rot[3 * j], s = rot[3 * j + 1];
    const double vp = v[(int64_t)r * ldv + pj], vq = v[(int64_t)r * ldv + qj];
    v[(int64_t)r * ldv + pj] = c * vp - s * vq;
    v[(int64_t)r * ldv + qj] = s * vp + c * vq;
  }
}

__device__ __forceinline__ void jacobi_rotations(const double *a, int64_t lda, int N, int N2,
                                                 int step, double floor_abs, double *rot,
                                                 unsigned *count, int64_t tid, int64_t nth) {
  for (int64_t i = tid; i < N2 / 2; i += nth) {
    int p, q;
    rr_pair((int)i, step, N2, p, q);
    double c = 1.0, s = 0.0, t = 0.0;
    if (q < N && jacobi_rot(a[(int64_t)p * lda + p], a[(int64_t)q * lda + q],
                            a[(int64_t)p * lda + q], floor_abs, c, s, t))
      atomicAdd(count, 1u);
    rot[3 * i] = c;
    rot[3 * i + 1] = s;
    rot[3 * i + 2] = t;
  }
}

constexpr int kJacobiSweeps = 60;
constexpr int kSmallN = 96;

// N <= kSmallN: one CTA, A and V in shared memory.  A (lda) is read, diagonalised in shared
// memory; W = diag, V = eigenvectors (columns), both written back (A is left unchanged).
__global__ void __launch_bounds__(1024)
    k42_jacobi_small(int N, const double *__restrict__ A, int64_t lda, double *__restrict__ W,
                     double *__restrict__ V, int64_t ldv, int *stats) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N2 = N + (N & 1);
  const int ld = N2 + 1;
  double *a = reinterpret_cast<double *>(smem_raw);  // [N2][ld]
  double *v = a + (size_t)N2 * ld;                   // [N2][ld]
  double *rot = v + (size_t)N2 * ld;                 // [N2/2][3]
  __shared__ unsigned cnt;
  __shared__ double s_fro;
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int e = tid; e < N2 * N2; e += nth) {
    const int r = e / N2, c = e % N2;
    a[r * ld + c] = (r < N && c < N) ? A[(int64_t)r * lda + c] : 0.0;
    v[r * ld + c] = (r == c) ? 1.0 : 0.0;
  }
  if (tid == 0) s_fro = 0.0;
  __syncthreads();
  if (tid < 32) {  // ||A||_F (fixed order: lane-strided partials, then a shuffle tree)
    double f = 0.0;
    for (int e = tid; e < N * N; e += 32) f += a[(e / N) * ld + (e % N)] * a[(e / N) * ld + (e % N)];
    for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xFFFFFFFFu, f, o);
    if (tid == 0) s_fro = sqrt(f);
  }
  __syncthreads();
  const double floor_abs = fmax(1e-300, c_jac_abs * s_fro);
  int sweep = 0;
  for (; sweep < kJacobiSweeps && N2 > 1; ++sweep) {
    if (tid == 0) cnt = 0;
    __syncthreads();
    for (int step = 0; step < N2 - 1; ++step) {
      jacobi_rotations(a, ld, N, N2, step, floor_abs, rot, &cnt, tid, nth);
      __syncthreads();
      jacobi_apply(a, ld, v, ld, N, N2, step, rot, tid, nth);
      __syncthreads();
    }
    if (cnt == 0) break;
    __syncthreads();
  }
  if (stats && tid == 0) stats[0] = sweep;
  for (int e = tid; e < N * N; e += nth) {
    const int r = e / N, c = e % N;
    V[(int64_t)r * ldv + c] = v[r * ld + c];
  }
  for (int i = tid; i < N; i += nth) W[i] = a[i * ld + i];
}

// Any N: a cooperative grid; A (lda) is read, then diagonalised in two ping-pong copies A0/A1
// (ld N, in ws) so that each step needs ONE grid-wide barrier: every thread computes the
// rotations it needs (pairs i and j of its 2 x 2 block) from the step's input copy and writes
// the output copy; V (ldv, initialised here) applies each step's rotations one step later, from
// the table the diagonal-block owners wrote (double-buffered by step parity).
// ws: A0, A1 (N x N each), rot [2][N2/2 x 3], the Frobenius norm, kJacobiSweeps counters.
__device__ __forceinline__ void jacobi_rot_of(const double *a, int64_t lda, int N, int N2, int i,
                                              int step, double floor_abs, int &p, int &q,
                                              double &c, double &s, double &t) {
  rr_pair(i, step, N2, p, q);
  c = 1.0;
  s = 0.0;
  t = 0.0;
  if (q < N) jacobi_rot(a[(int64_t)p * lda + p], a[(int64_t)q * lda + q], a[(int64_t)p * lda + q],
                        floor_abs, c, s, t);
}

__global__ void __launch_bounds__(512)
    k42_jacobi_grid(int N, const double *__restrict__ A, int64_t lda, double *__restrict__ W,
                    double *__restrict__ V, int64_t ldv, double *__restrict__ ws, int *stats) {
  cg::grid_group grid = cg::this_grid();
  const int N2 = N + (N & 1), H = N2 / 2;
  double *buf0 = ws, *buf1 = ws + (size_t)N * N;
  double *rot = buf1 + (size_t)N * N;  // [2][H][3]
  double *fro = rot + 6 * (size_t)H;
  unsigned *cnt = reinterpret_cast<unsigned *>(fro + 1);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = tid; e < (int64_t)N * N; e += nth) {
    const int64_t r = e / N, c = e - (e / N) * N;
    V[r * ldv + c] = (r == c) ? 1.0 : 0.0;
    buf0[e] = A[r * lda + c];
  }
  if (tid < kJacobiSweeps) cnt[tid] = 0;
  if (blockIdx.x == 0) {  // ||A||_F by one CTA (fixed order)
    __shared__ double sp[512];
    double f = 0.0;
    for (int64_t e = threadIdx.x; e < (int64_t)N * N; e += blockDim.x) {
      const double x = A[(e / N) * lda + (e % N)];
      f += x * x;
    }
    sp[threadIdx.x] = f;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
      if ((int)threadIdx.x < o) sp[threadIdx.x] += sp[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) *fro = sqrt(sp[0]);
  }
  grid.sync();
  const double floor_abs = fmax(1e-300, c_jac_abs * *fro);
  const double *cur = buf0;
  double *nxt = buf1;
  int sweep = 0, gstep = 0;  // gstep: steps done so far (parity selects the rotation table)
  bool pending = false;      // rotations of step gstep - 1 not yet applied to V
  const uint32_t nblk = (uint32_t)H * (uint32_t)H;
  for (; sweep < kJacobiSweeps && N2 > 1; ++sweep) {
    for (int step = 0; step < N2 - 1; ++step, ++gstep) {
      double *rt = rot + 3 * (size_t)H * (gstep & 1);
      const double *rp = rot + 3 * (size_t)H * ((gstep + 1) & 1);  // previous step's table
      for (uint32_t e = (uint32_t)tid; e < nblk; e += (uint32_t)nth) {
        const int i = (int)(e / (uint32_t)H), j = (int)(e % (uint32_t)H);
        int pi, qi, pj, qj;
        double ci, si, ti, cj, sj, tj;
        jacobi_rot_of(cur, N, N, N2, i, step, floor_abs, pi, qi, ci, si, ti);
        if (i == j) {
          if (ti != 0.0) atomicAdd(cnt + sweep, 1u);
          rt[3 * i] = ci;
          rt[3 * i + 1] = si;
          rt[3 * i + 2] = ti;
          if (qi >= N) {
            nxt[(int64_t)pi * N + pi] = cur[(int64_t)pi * N + pi];
            continue;
          }
          // diagonal block: the stable forms a_pp - t a_pq, a_qq + t a_pq, a_pq = 0
          const double app = cur[(int64_t)pi * N + pi], aqq = cur[(int64_t)qi * N + qi];
          const double apq = cur[(int64_t)pi * N + qi];
          nxt[(int64_t)pi * N + pi] = app - ti * apq;
          nxt[(int64_t)qi * N + qi] = aqq + ti * apq;
          nxt[(int64_t)pi * N + qi] = ti != 0.0 ? 0.0 : apq;
          nxt[(int64_t)qi * N + pi] = ti != 0.0 ? 0.0 : apq;
          continue;
        }
        jacobi_rot_of(cur, N, N, N2, j, step, floor_abs, pj, qj, cj, sj, tj);
        const bool qiv = qi < N, qjv = qj < N;  // index N (odd N's pad) does not exist
        const double b00 = cur[(int64_t)pi * N + pj];
        const double b01 = qjv ? cur[(int64_t)pi * N + qj] : 0.0;
        const double b10 = qiv ? cur[(int64_t)qi * N + pj] : 0.0;
        const double b11 = (qiv && qjv) ? cur[(int64_t)qi * N + qj] : 0.0;
        const double r00 = ci * b00 - si * b10, r01 = ci * b01 - si * b11;
        const double r10 = si * b00 + ci * b10, r11 = si * b01 + ci * b11;
        nxt[(int64_t)pi * N + pj] = cj * r00 - sj * r01;
        if (qjv) nxt[(int64_t)pi * N + qj] = sj * r00 + cj * r01;
        if (qiv) nxt[(int64_t)qi * N + pj] = cj * r10 - sj * r11;
        if (qiv && qjv) nxt[(int64_t)qi * N + qj] = sj * r10 + cj * r11;
      }
      if (pending) {  // V <- V J of the previous step (its table is complete: barrier passed)
        const uint32_t nv = (uint32_t)N * (uint32_t)H;
        for (uint32_t e = (uint32_t)tid; e < nv; e += (uint32_t)nth) {
          const int r = (int)(e / (uint32_t)H), j = (int)(e % (uint32_t)H);
          if (rp[3 * j + 2] == 0.0) continue;
          int pj, qj;
          rr_pair(j, step == 0 ? N2 - 2 : step - 1, N2, pj, qj);
          if (qj >= N) continue;
          const double c = rp[3 * j], s = rp[3 * j + 1];
          const double vp = V[(int64_t)r * ldv + pj], vq = V[(int64_t)r * ldv + qj];
          V[(int64_t)r * ldv + pj] = c * vp - s * vq;
          V[(int64_t)r * ldv + qj] = s * vp + c * vq;
        }
      }
      pending = true;
      grid.sync();
      const double *t_ = cur;
      cur = nxt;
      nxt = const_cast<double *>(t_);
    }
    if (*(volatile unsigned *)(cnt + sweep) == 0) {
      ++sweep;
      break;
    }
  }
  if (pending) {  // the last step's rotations
    const double *rp = rot + 3 * (size_t)H * ((gstep + 1) & 1);
    const int last = (gstep - 1) % (N2 - 1);
    const uint32_t nv = (uint32_t)N * (uint32_t)H;
    for (uint32_t e = (uint32_t)tid; e < nv; e += (uint32_t)nth) {
      const int r = (int)(e / (uint32_t)H), j = (int)(e % (uint32_t)H);
      if (rp[3 * j + 2] == 0.0) continue;
      int pj, qj;
      rr_pair(j, last, N2, pj, qj);
      if (qj >= N) continue;
      const double c = rp[3 * j], s = rp[3 * j + 1];
      const double vp = V[(int64_t)r * ldv + pj], vq = V[(int64_t)r * ldv + qj];
      V[(int64_t)r * ldv + pj] = c * vp - s * vq;
      V[(int64_t)r * ldv + qj] = s * vp + c * vq;
    }
  }
  if (stats && tid == 0) stats[0] = sweep;
  for (int64_t i = tid; i < N; i += nth) W[i] = cur[i * N + i];
}

// CholeskyQR with column dropping (one CTA, b <= 96): G = V^T V (b x b, ldg) -> S (b x b) with
// V S orthonormal: G = L L^T (left-looking, column by column), S = L^{-T}.  A column whose
// remaining squared norm d_j = G_jj - sum_k L_jk^2 is <= floor (floor = rtol^2 max_c G0_cc when
// G0 is given, else floor_abs) is dependent on the earlier ones: it is dropped (S column 0).
__global__ void __launch_bounds__(256)
    k43_chol_orth(int b, const double *__restrict__ G, int64_t ldg, const double *__restrict__ G0,
                  int64_t ldg0, double rtol, double floor_abs, double *__restrict__ S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ld = b + 1;
  double *L = reinterpret_cast<double *>(smem_raw);  // [b][ld]
  double *X = L + (size_t)b * ld;                    // [b][ld]: L^{-1}
  __shared__ double s_floor;
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int e = tid; e < b * b; e += nth) {
    L[(e / b) * ld + (e % b)] = G[(int64_t)(e / b) * ldg + (e % b)];
    X[(e / b) * ld + (e % b)] = 0.0;
  }
  if (tid == 0) {
    double fl = floor_abs;
    if (G0) {
      double mx = 0.0;
      for (int c = 0; c < b; ++c) mx = fmax(mx, G0[(int64_t)c * ldg0 + c]);
      fl = rtol * rtol * mx;
    }
    s_floor = fl;
  }
  __syncthreads();
  // right-looking Cholesky on the lower triangle (column j scaled, trailing update)
  for (int j = 0; j < b; ++j) {
    const double d = L[j * ld + j];
    const bool keep = d > s_floor;
    const double piv = keep ? sqrt(d) : 0.0;
    __syncthreads();
    for (int i = j + tid; i < b; i += nth) L[i * ld + j] = keep ? (i == j ? piv : L[i * ld + j] / piv) : 0.0;
    __syncthreads();
    for (int e = tid; e < (b - j - 1) * (b - j - 1); e += nth) {
      const int i = j + 1 + e / (b - j - 1), k = j + 1 + e % (b - j - 1);
      if (k <= i) L[i * ld + k] -= L[i * ld + j] * L[k * ld + j];
    }
    __syncthreads();
  }
  // X = L^{-1} (lower triangular; dropped rows/columns stay 0): thread per column
  for (int c = tid; c < b; c += nth) {
    if (L[c * ld + c] == 0.0) continue;
    X[c * ld + c] = 1.0 / L[c * ld + c];
    for (int i = c + 1; i < b; ++i) {
      if (L[i * ld + i] == 0.0) continue;
      double acc = 0.0;
      for (int k = c; k < i; ++k) acc = fma(L[i * ld + k], X[k * ld + c], acc);
      X[i * ld + c] = -acc / L[i * ld + i];
    }
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += nth) {
    const int r = e / b, c = e % b;
    S[(int64_t)r * b + c] = X[c * ld + r];  // S = X^T
  }
}

// ------------------------------------------------------------------------ top-k eigenpairs
// The Rayleigh-Ritz step needs only the k eigenpairs of largest |lambda| of the (q b)^2 matrix T:
//   k55_tridiag     Householder reduction T = H^T Tri H on a cooperative grid (two grid barriers
//                   per column: p = tau A22 v, then the rank-2 update A22 -= v w^T + w v^T),
//   k56_tri_topk    one CTA: Sturm-count bisection for the k smallest and k largest eigenvalues
//                   of the tridiagonal, the k of largest |lambda|, inverse iteration (tridiagonal
//                   LU with partial pivoting) with modified Gram-Schmidt inside eigenvalue
//                   clusters (|dl| <= 1e-3 ||Tri||_1, LAPACK dstein's grouping),
//   k57_back        one CTA per vector: y <- H_0 ... H_{N-3} y (reflectors in reverse order).
// ws layout (doubles): A copy N*N | p N | reflectors N*N | tau N | d N | e N
__global__ void __launch_bounds__(512)
    k55_tridiag(int N, double *__restrict__ A, double *__restrict__ p, double *__restrict__ H,
                double *__restrict__ tau, double *__restrict__ d, double *__restrict__ e) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[32];
  const int tid = threadIdx.x;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int lane = tid & 31;
  const int64_t gwarp = gtid >> 5, nwarps = nth >> 5;
  auto block_sum = [&](double v) -> double {  // fixed order: lanes (butterfly), then warps
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (lane == 0) red[tid >> 5] = v;
    __syncthreads();
    double r = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) r += red[q];
    __syncthreads();
    return r;
  };
  for (int j = 0; j < N - 2; ++j) {
    const int m = N - j - 1;           // length of x = A[j][j+1 .. N-1] (row j = column j)
    const double *x = A + (int64_t)j * N + j + 1;
    // every CTA computes the reflector's scalars from row j (unchanged during this step)
    double part = 0.0;
    for (int i = 1 + tid; i < m; i += blockDim.x) part += x[i] * x[i];
    const double sigma = block_sum(part);
    const double x0 = x[0];
    double alpha, t, v0;
    if (sigma == 0.0) {  // already tridiagonal in this column
      alpha = x0;
      t = 0.0;
      v0 = 0.0;
    } else {
      const double nrm = sqrt(fma(x0, x0, sigma));
      alpha = x0 >= 0.0 ? -nrm : nrm;
      v0 = x0 - alpha;
      t = 2.0 / fma(v0, v0, sigma);   // H = I - t v v^T, v = (v0, x_1, ..., x_{m-1})
    }
    if (blockIdx.x == 0 && tid == 0) {
      d[j] = A[(int64_t)j * N + j];
      e[j] = alpha;
      tau[j] = t;
    }
    for (int i = gtid; i < m; i += nth) H[(int64_t)j * N + i] = (i == 0) ? v0 : x[i];
    if (t != 0.0) {
      // p = t A22 v: one warp per row of the trailing block
      for (int64_t r = gwarp; r < m; r += nwarps) {
        const double *ar = A + (int64_t)(j + 1 + r) * N + j + 1;
        double acc = 0.0;
        for (int c = lane; c < m; c += 32) acc = fma(ar[c], c == 0 ? v0 : x[c], acc);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
        if (lane == 0) p[r] = t * acc;
      }
    }
    grid.sync();
    if (t != 0.0) {
      // K = t/2 v^T p; w = p - K v; A22 -= v w^T + w v^T
      double kp = 0.0;
      for (int i = tid; i < m; i += blockDim.x) kp = fma(i == 0 ? v0 : x[i], p[i], kp);
      const double K = 0.5 * t * block_sum(kp);
      const uint32_t mm = (uint32_t)m * (uint32_t)m;  // N <= 4096: fits 32 bits
      for (uint32_t q = (uint32_t)gtid; q < mm; q += (uint32_t)nth) {
        const uint32_t r = q / (uint32_t)m, c = q - r * (uint32_t)m;
        const double vr = r == 0 ? v0 : x[r], vc = c == 0 ? v0 : x[c];
        const double wr = p[r] - K * vr, wc = p[c] - K * vc;
        double *a = A + (int64_t)(j + 1 + r) * N + j + 1 + c;
        *a -= fma(vr, wc, wr * vc);
      }
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && tid == 0) {
    if (N >= 2) {
      d[N - 2] = A[(int64_t)(N - 2) * N + N - 2];
      e[N - 2] = A[(int64_t)(N - 1) * N + N - 2];
    }
    d[N - 1] = A[(int64_t)(N - 1) * N + N - 1];
  }
}

// number of eigenvalues of the tridiagonal (d, e) below x (Sturm count via the LDL^T pivots)
__device__ __forceinline__ int sturm_count(const double *d, const double *e2, int N, double x,
                                           double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < N; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// One CTA of 1024 threads.  Y (N x k, ldy = k): the tridiagonal's eigenvectors of the k eigenvalues
// of largest |lambda| (ties by index), in that order; lam[k], sigma[k] = |lam|.
// Eigenvalues: multisection — one warp per candidate index, its 32 lanes take Sturm counts at 32
// interior points of the bracket each round, so a round shrinks it 33-fold (12 rounds to full
// precision instead of ~60 bisection steps).
// Eigenvectors: inverse iteration (tridiagonal LU with partial pivoting, reciprocal pivots):
// three iterations of every vector concurrently (thread per vector; LU factors in lw, interleaved
// [i][r] so the k threads read adjacent words), then, in ascending eigenvalue order, two more with
// modified Gram-Schmidt against the earlier vectors of the same cluster (|dl| <= 1e-3 ||Tri||_1,
// LAPACK dstein's grouping) — the concurrent phase takes the long serial chains off the one-vector-
// at-a-time path.
// smem: d, e, e2 (later one vector's LU factors, 4.5 N), y (N) + candidates.  lw: 4 N k
// doubles + N k ints.
__global__ void __launch_bounds__(1024)
    k56_tri_topk(int N, int k, const double *__restrict__ dg, const double *__restrict__ eg,
                 double *__restrict__ lam, double *__restrict__ sigma, double *__restrict__ Y,
                 double *__restrict__ lw) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *d = reinterpret_cast<double *>(smem_raw);
  double *e = d + N, *e2 = e + N;
  double *y = d + (9 * (int64_t)N + 1) / 2;               // after 4.5 N: d, e, e2 | one LU
  double *cand = y + N;                                   // [2k] candidate eigenvalues
  int *cidx = reinterpret_cast<int *>(cand + 2 * k);      // [2k] their eigenvalue indices
  int *sel = cidx + 2 * k;                                // [k] chosen candidates, |lambda| desc
  int *ord = sel + k;                                     // [k] slots in ascending (lambda, index)
  __shared__ double s_lo, s_hi, s_norm, s_red[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nth = blockDim.x, nw = nth >> 5;
  for (int i = tid; i < N; i += nth) {
    d[i] = dg[i];
    e[i] = i < N - 1 ? eg[i] : 0.0;
    e2[i] = e[i] * e[i];
  }
  __syncthreads();
  if (tid == 0) {  // Gershgorin interval and ||Tri||_1
    double lo = d[0], hi = d[0], nrm = 0.0;
    for (int i = 0; i < N; ++i) {
      const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < N - 1 ? fabs(e[i]) : 0.0);
      lo = fmin(lo, d[i] - r);
      hi = fmax(hi, d[i] + r);
      nrm = fmax(nrm, fabs(d[i]) + r);
    }
    s_lo = lo;
    s_hi = hi;
    s_norm = nrm;
  }
  __syncthreads();
  const double tnorm = s_norm > 0.0 ? s_norm : 1.0;
  const double pivmin = fmax(1e-300, 1e-300 * tnorm);
  // eigenvalue indices 0..k-1 and N-k..N-1 (2k candidates, duplicates when 2k > N)
  const int nc = 2 * k;
  for (int c = w; c < nc; c += nw) {
    int idx = c < k ? c : N - nc + c;
    if (idx < 0) idx = 0;
    if (idx >= N) idx = N - 1;
    double lo = s_lo - 2.2e-16 * tnorm - pivmin, hi = s_hi + 2.2e-16 * tnorm + pivmin;
    for (int round = 0; round < 64; ++round) {
      if (hi - lo <= 2.2e-16 * fmax(fabs(lo), fabs(hi)) + pivmin) break;
      const double x = lo + (hi - lo) * ((double)(lane + 1) / 33.0);
      const bool above = x > lo && x < hi && sturm_count(d, e2, N, x, pivmin) > idx;
      // lanes whose point lies above eigenvalue idx; points are nondecreasing in the lane
      const unsigned b = __ballot_sync(0xFFFFFFFFu, above);
      const unsigned inside = __ballot_sync(0xFFFFFFFFu, x > lo && x < hi);
      if (!inside) break;  // no representable interior point left
      const int f = b ? __ffs(b) - 1 : 32;  // first lane above
      // the bracket becomes (x_{f-1}, x_f]: the largest interior point below, the first above
      const unsigned below = inside & ~b & ((f == 32) ? 0xFFFFFFFFu : ((1u << f) - 1u));
      const int g = below ? 31 - __clz(below) : -1;
      const double xf = __shfl_sync(0xFFFFFFFFu, x, f & 31);
      const double xg = __shfl_sync(0xFFFFFFFFu, x, g < 0 ? 0 : g);
      const double nlo = g >= 0 ? xg : lo, nhi = f < 32 ? xf : hi;
      if (nlo == lo && nhi == hi) break;
      lo = nlo;
      hi = nhi;
    }
    if (lane == 0) {
      cand[c] = 0.5 * (lo + hi);
      cidx[c] = idx;
    }
  }
  __syncthreads();
  if (tid == 0) {  // the k distinct eigenvalue indices of largest |lambda| (ties: smaller index)
    int nsel = 0;
    bool used[2 * 96 + 2];  // k <= 96
    for (int c = 0; c < nc; ++c) used[c] = false;
    for (int c = 0; c < nc; ++c)  // candidates with the same index are one eigenvalue
      for (int c2 = 0; c2 < c; ++c2)
        if (cidx[c2] == cidx[c]) used[c] = true;
    while (nsel < k) {
      int best = -1;
      for (int c = 0; c < nc; ++c) {
        if (used[c]) continue;
        if (best < 0 || fabs(cand[c]) > fabs(cand[best]) ||
            (fabs(cand[c]) == fabs(cand[best]) && cidx[c] < cidx[best]))
          best = c;
      }
      if (best < 0) break;
      used[best] = true;
      sel[nsel++] = best;
    }
    for (int r = nsel; r < k; ++r) sel[r] = sel[0];
    for (int a = 0; a < k; ++a) {  // ascending (lambda, index, slot) order of the selection
      int rank = 0;
      for (int b2 = 0; b2 < k; ++b2)
        rank += (cand[sel[b2]] < cand[sel[a]]) ||
                (cand[sel[b2]] == cand[sel[a]] && cidx[sel[b2]] < cidx[sel[a]]) ||
                (cand[sel[b2]] == cand[sel[a]] && cidx[sel[b2]] == cidx[sel[a]] && b2 < a);
      ord[rank] = a;
    }
  }
  __syncthreads();
  // LU factors of (Tri - lambda_r I), vector r at [i * k + r]
  double *lu_r = lw, *lu_u1 = lu_r + (int64_t)N * k, *lu_u2 = lu_u1 + (int64_t)N * k;
  double *lu_l = lu_u2 + (int64_t)N * k;
  int *piv = reinterpret_cast<int *>(lu_l + (int64_t)N * k);
  const double tiny = 2.2e-16 * tnorm;
  // solve L U v = v for vector r (one thread); v at stride vs
  auto solve = [&](int r, double *v, int64_t vs) {
    for (int i = 0; i < N - 1; ++i) {
      const int64_t o = (int64_t)i * k + r;
      const double l = lu_l[o];
      if (piv[o]) {
        const double t0 = v[i * vs];
        const double t1 = v[(i + 1) * vs];
        v[i * vs] = t1;
        v[(i + 1) * vs] = t0 - l * t1;
      } else {
        v[(i + 1) * vs] -= l * v[i * vs];
      }
    }
    double y1 = v[(N - 1) * vs] * lu_r[(int64_t)(N - 1) * k + r], y2 = 0.0;
    v[(N - 1) * vs] = y1;
    for (int i = N - 2; i >= 0; --i) {
      const int64_t o = (int64_t)i * k + r;
      const double yi = (v[i * vs] - lu_u1[o] * y1 - lu_u2[o] * y2) * lu_r[o];
      v[i * vs] = yi;
      y2 = y1;
      y1 = yi;
    }
  };
  if (tid < k) {  // concurrent phase: factor, then three plain inverse iterations per vector
    const int r = tid;
    const double shift = cand[sel[r]];
    double a = d[0] - shift, b = N > 1 ? e[0] : 0.0;
    for (int i = 0; i < N - 1; ++i) {
      const int64_t o = (int64_t)i * k + r;
      const double c = e[i], dn = d[i + 1] - shift, bn = i + 1 < N - 1 ? e[i + 1] : 0.0;
      double piv_d;
      if (fabs(a) >= fabs(c)) {  // no swap: rows (a b 0), (c dn bn)
        piv[o] = 0;
        const double l = (a != 0.0) ? c / a : 0.0;
        piv_d = a;
        lu_u1[o] = b;
        lu_u2[o] = 0.0;
        lu_l[o] = l;
        a = dn - l * b;
        b = bn;
      } else {  // swap: pivot row (c dn bn)
        piv[o] = 1;
        const double l = a / c;
        piv_d = c;
        lu_u1[o] = dn;
        lu_u2[o] = bn;
        lu_l[o] = l;
        a = b - l * dn;
        b = -l * bn;
      }
      if (piv_d == 0.0) piv_d = tiny;
      lu_r[o] = 1.0 / piv_d;
    }
    double last = (a == 0.0) ? tiny : a;
    if (fabs(last) < tiny) last = last < 0 ? -tiny : tiny;
    lu_r[(int64_t)(N - 1) * k + r] = 1.0 / last;
    double *v = Y + r;  // column r of Y (ld k)
    for (int i = 0; i < N; ++i)  // deterministic start: 1 + small index ramp
      v[(int64_t)i * k] = 1.0 + 1e-3 * (double)((i * 7 + r * 13) % 17);
    for (int iter = 0; iter < 3; ++iter) {
      solve(r, v, k);
      double s = 0.0;
      for (int i = 0; i < N; ++i) s = fma(v[(int64_t)i * k], v[(int64_t)i * k], s);
      const double inv = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
      for (int i = 0; i < N; ++i) v[(int64_t)i * k] *= inv;
    }
  }
  __syncthreads();
  auto block_sum = [&](double v) -> double {  // fixed order: lanes, then warps
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (lane == 0) s_red[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int q = 0; q < nw; ++q) t += s_red[q];
    __syncthreads();
    return t;
  };
  // serial phase, ascending eigenvalue order: two iterations with MGS inside the cluster.  The
  // vector's LU factors are staged in shared memory over d, e, e2 (no longer needed), so the
  // serial solve runs on shared-memory latencies
  double *sl_r = d, *sl_u1 = sl_r + N, *sl_u2 = sl_u1 + N, *sl_l = sl_u2 + N;
  int *sl_p = reinterpret_cast<int *>(sl_l + N);
  auto solve_s = [&]() {  // thread 0: L U y = y from the staged factors
    for (int i = 0; i < N - 1; ++i) {
      const double l = sl_l[i];
      if (sl_p[i]) {
        const double t0 = y[i], t1 = y[i + 1];
        y[i] = t1;
        y[i + 1] = t0 - l * t1;
      } else {
        y[i + 1] -= l * y[i];
      }
    }
    double y1 = y[N - 1] * sl_r[N - 1], y2 = 0.0;
    y[N - 1] = y1;
    for (int i = N - 2; i >= 0; --i) {
      const double yi = (y[i] - sl_u1[i] * y1 - sl_u2[i] * y2) * sl_r[i];
      y[i] = yi;
      y2 = y1;
      y1 = yi;
    }
  };
  for (int rr = 0; rr < k; ++rr) {
    const int r = ord[rr];
    const double shift = cand[sel[r]];
    for (int i = tid; i < N; i += nth) {
      const int64_t o = (int64_t)i * k + r;
      y[i] = Y[o];
      sl_r[i] = lu_r[o];
      sl_u1[i] = lu_u1[o];
      sl_u2[i] = lu_u2[o];
      sl_l[i] = lu_l[o];
      sl_p[i] = piv[o];
    }
    __syncthreads();
    for (int iter = 0; iter < 2; ++iter) {
      if (tid == 0) solve_s();
      __syncthreads();
      for (int q = 0; q < rr; ++q) {
        const int sq = ord[q];
        if (fabs(cand[sel[sq]] - shift) > 1e-3 * tnorm) continue;  // (uniform over the CTA)
        const double *yq = Y + sq;
        double part = 0.0;
        for (int i = tid; i < N; i += nth) part = fma(yq[(int64_t)i * k], y[i], part);
        const double dot = block_sum(part);
        for (int i = tid; i < N; i += nth) y[i] -= dot * yq[(int64_t)i * k];
        __syncthreads();
      }
      double part = 0.0;
      for (int i = tid; i < N; i += nth) part = fma(y[i], y[i], part);
      const double nrm = sqrt(block_sum(part));
      const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
      for (int i = tid; i < N; i += nth) y[i] *= inv;
      __syncthreads();
    }
    for (int i = tid; i < N; i += nth) Y[(int64_t)i * k + r] = y[i];
    if (tid == 0) {
      if (lam) lam[r] = cand[sel[r]];
      if (sigma) sigma[r] = fabs(cand[sel[r]]);
    }
    __syncthreads();
  }
}

// one CTA per vector: y <- H_0 H_1 ... H_{N-3} y, H_j = I - tau_j v_j v_j^T acting on [j+1, N)
__global__ void __launch_bounds__(256)
    k57_back(int N, int k, const double *__restrict__ H, const double *__restrict__ tau,
             double *__restrict__ Y) {
  __shared__ double red[256];
  __shared__ double yv[4096];  // N <= 4096
  const int tid = threadIdx.x, col = blockIdx.x;
  for (int i = tid; i < N; i += 256) yv[i] = Y[(int64_t)i * k + col];
  __syncthreads();
  for (int j = N - 3; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;
    const int m = N - j - 1;
    const double *v = H + (int64_t)j * N;
    double part = 0.0;
    for (int i = tid; i < m; i += 256) part = fma(v[i], yv[j + 1 + i], part);
    red[tid] = part;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
      if (tid < o) red[tid] += red[tid + o];
      __syncthreads();
    }
    const double f = t * red[0];
    __syncthreads();
    for (int i = tid; i < m; i += 256) yv[j + 1 + i] -= f * v[i];
    __syncthreads();
  }
  for (int i = tid; i < N; i += 256) Y[(int64_t)i * k + col] = yv[i];
}

// ------------------------------------------------------------------------------- small kernels
// order[r] = index of the r-th largest |W| (ties by index), r < k; lam/sigma of the selection;
// Vs (N x k) = V[:, order].
__global__ void k44_select(int N, int k, const double *__restrict__ W, const double *__restrict__ V,
                           int64_t ldv, double *__restrict__ lam, double *__restrict__ sigma,
                           double *__restrict__ Vs, int *__restrict__ order) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const double ai = fabs(W[i]);
    int r = 0;
    for (int j = 0; j < N; ++j) {
      const double aj = fabs(W[j]);
      r += (aj > ai) || (aj == ai && j < i);
    }
    if (r < k) {
      order[r] = i;
      if (lam) lam[r] = W[i];
      if (sigma) sigma[r] = ai;
      for (int row = 0; row < N; ++row) Vs[(int64_t)row * k + r] = V[(int64_t)row * ldv + i];
    }
  }
}

// S[r][c] = V[r][c] f(lam_c): f = 1/sqrt(lam) when lam > floor, else 0 (a dropped direction).
// floor = (rtol scale)^2 with scale^2 = max_c G0[c][c] when G0 != nullptr, else floor_abs.
__global__ void k45_scale_cols(int b, const double *__restrict__ V, const double *__restrict__ lam,
                               const double *__restrict__ G0, int64_t ldg0, double rtol,
                               double floor_abs, double *__restrict__ S) {
  double fl = floor_abs;
  if (G0) {
    double mx = 0.0;
    for (int c = 0; c < b; ++c) mx = fmax(mx, G0[(int64_t)c * ldg0 + c]);
    fl = rtol * rtol * mx;
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < b * b; e += gridDim.x * blockDim.x) {
    const int c = e % b;
    const double l = lam[c];
    S[e] = (l > fl) ? V[e] / sqrt(l) : 0.0;
  }
}

// Zs[i][c] = fp32(V[i][c]), Zs[i][b + c] = fp32(V[i][c] - fp32(V[i][c])): V = hi + lo to
// ~2^-48 relative, so A V = A hi + A lo through the fp32-input product (linearity).
__global__ void k46_split(int64_t n, int64_t b, const double *__restrict__ V, int64_t ldv,
                          float *__restrict__ Zs) {
  const int64_t total = n * b;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    const int64_t i = e / b, c = e - (e / b) * b;
    const double x = V[i * ldv + c];
    const float hi = (float)x;
    Zs[i * 2 * b + c] = hi;
    Zs[i * 2 * b + b + c] = (float)(x - (double)hi);
  }
}

// Y[i][c] = Yr[i][c] + Yr[i][b + c]
__global__ void k47_combine(int64_t n, int64_t b, const double *__restrict__ Yr,
                            double *__restrict__ Y, int64_t ldy) {
  const int64_t total = n * b;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    const int64_t i = e / b, c = e - (e / b) * b;
    Y[i * ldy + c] = Yr[i * 2 * b + c] + Yr[i * 2 * b + b + c];
  }
}

// D[r][c] (ldd) += alpha S[r][c] (lds), rows x cols
__global__ void k48_axpy2d(int64_t rows, int64_t cols, double alpha, const double *__restrict__ S,
                           int64_t lds, double *__restrict__ D, int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    const int64_t r = e / cols, c = e - (e / cols) * cols;
    D[r * ldd + c] += alpha * S[r * lds + c];
  }
}

// T = (T + T^T) / 2 in place (N x N, ldt); each unordered pair by one thread.
__global__ void k49_symmetrize(int64_t N, double *T, int64_t ldt) {
  const int64_t total = N * N;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    const int64_t r = e / N, c = e - (e / N) * N;
    if (c <= r) continue;
    const double v = 0.5 * (T[r * ldt + c] + T[c * ldt + r]);
    T[r * ldt + c] = v;
    T[c * ldt + r] = v;
  }
}

// ---- conjugate gradients (Thm. linear_system): device scalars, no host round trip ----
// part[blk] = sum over this CTA's fixed index set of x_i y_i (grid-stride, fixed tree).
constexpr int kDotBlocks = 296;
__global__ void __launch_bounds__(256)
    k50_dot(int64_t n, const double *__restrict__ x, const double *__restrict__ y,
            double *__restrict__ part) {
  __shared__ double sp[256];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    acc = fma(x[i], y[i], acc);
  sp[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if ((int)threadIdx.x < o) sp[threadIdx.x] += sp[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sp[0];
}

// CG state (device): [0] rs, [1] alpha, [2] beta, [3] target, [4] pAp, [5] rs_new, [6] conv,
// [7] iterations, [8] scratch
enum { CG_RS = 0, CG_ALPHA, CG_BETA, CG_TARGET, CG_PAP, CG_RSNEW, CG_CONV, CG_IT, CG_N };
static_assert(CG_CONV == CG_CONV_INDEX && CG_IT == CG_CONV_INDEX + 1, "CG state layout");

__device__ __forceinline__ double fold_parts(const double *part, int nb) {
  double s = 0.0;
  for (int i = 0; i < nb; ++i) s += part[i];
  return s;
}

// phase 0: rs = r.r, target = tol ||rhs|| (rhs = r at start), conv = sqrt(rs) <= target
// phase 1: pAp; alpha = rs / pAp (when not converged)
// phase 2: rs_new; conv = sqrt(rs_new) <= target; beta = rs_new / rs; rs = rs_new; it++
__global__ void k51_cg_scalars(int phase, const double *__restrict__ part, int nb, double tol,
                               double *__restrict__ st) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double v = fold_parts(part, nb);
  if (phase == 0) {
    st[CG_RS] = v;
    st[CG_TARGET] = tol * sqrt(v);
    st[CG_CONV] = (sqrt(v) <= st[CG_TARGET]) ? 1.0 : 0.0;
    st[CG_IT] = 0.0;
    st[CG_ALPHA] = st[CG_BETA] = 0.0;
  } else if (phase == 1) {
    st[CG_PAP] = v;
    if (st[CG_CONV] == 0.0) st[CG_ALPHA] = st[CG_RS] / v;
  } else {
    st[CG_RSNEW] = v;
    if (st[CG_CONV] == 0.0) {
      st[CG_CONV] = (sqrt(v) <= st[CG_TARGET]) ? 1.0 : 0.0;
      st[CG_BETA] = v / st[CG_RS];
      st[CG_RS] = v;
      st[CG_IT] += 1.0;
    }
  }
}

// x += alpha p, r -= alpha Ap (skipped once converged before this iteration)
__global__ void k52_cg_xr(int64_t n, const double *__restrict__ st, const double *__restrict__ p,
                          const double *__restrict__ Ap, double *__restrict__ x,
                          double *__restrict__ r) {
  if (st[CG_CONV] != 0.0) return;
  const double a = st[CG_ALPHA];
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
    x[i] = fma(a, p[i], x[i]);
    r[i] = fma(-a, Ap[i], r[i]);
  }
}

// p = r + beta p (skipped once converged)
__global__ void k53_cg_p(int64_t n, const double *__restrict__ st, const double *__restrict__ r,
                         double *__restrict__ p) {
  if (st[CG_CONV] != 0.0) return;
  const double b = st[CG_BETA];
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    p[i] = fma(b, p[i], r[i]);
}

// d = a - b (elementwise)
__global__ void k54_sub(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
                        double *__restrict__ d) {
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    d[i] = a[i] - b[i];
}

int grid1d(int64_t elems, int cap = 148 * 8) {
  int64_t b = (elems + 255) / 256;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

// ------------------------------------------------------------------------------- launchers
// the skinny kernels' shapes: TN with M <= 64, N <= 32 and a long K; NN with K <= 96, N <= 32
static bool skinny_tn(int ta, int64_t M, int64_t N, int64_t K) {
  return ta && M <= 64 && N <= 32 && K >= 4096;
}
static bool skinny_nn(int ta, int64_t N, int64_t K) { return !ta && K <= 96 && N <= 32; }
static int64_t skinny_tn_ctas(int64_t K, int sms) {
  int64_t c = (int64_t)sms * 4;
  const int64_t cap = (K + 8 * 64 - 1) / (8 * 64);  // at least 64 rows per warp
  return c < cap ? c : (cap < 1 ? 1 : cap);
}

size_t gemm_workspace(int ta, int64_t M, int64_t N, int64_t K, int sms) {
  const int64_t sp = gemm_splits(ta, M, N, K, sms);
  size_t b = sp > 1 ? (size_t)sp * (size_t)M * (size_t)N * sizeof(double) : 0;
  if (skinny_tn(ta, M, N, K))
    b = std::max(b, (size_t)skinny_tn_ctas(K, sms) * (size_t)M * (size_t)N * sizeof(double));
  return b;
}

template <int MT, int NT>
static int skinny_tn_t(int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                       int64_t lda, const double *B, int64_t ldb, double beta, double *C,
                       int64_t ldc, double *ws, int sms, cudaStream_t s) {
  const int64_t ctas = skinny_tn_ctas(K, sms);
  int64_t rpw = (K + ctas * 8 - 1) / (ctas * 8);
  rpw = (rpw + 15) / 16 * 16;
  if constexpr (MT == NT) {
    if (A == B && lda == ldb && M == N)
      k44_skinny_tn<MT, NT, true><<<(unsigned)ctas, 256, 0, s>>>(M, N, K, A, lda, B, ldb, rpw, ws);
    else
      k44_skinny_tn<MT, NT><<<(unsigned)ctas, 256, 0, s>>>(M, N, K, A, lda, B, ldb, rpw, ws);
  } else {
    k44_skinny_tn<MT, NT><<<(unsigned)ctas, 256, 0, s>>>(M, N, K, A, lda, B, ldb, rpw, ws);
  }
  const int64_t tot = M * N;
  k41b_gemm_fold_warp<<<(unsigned)((tot + 7) / 8), 256, 0, s>>>(M, N, ctas, ws, C, ldc, alpha,
                                                                beta);
  return 2;
}

template <int NT, int KQ, int TU>
static int skinny_nn_kt(int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                        int64_t lda, const double *B, int64_t ldb, double beta, double *C,
                        int64_t ldc, int sms, cudaStream_t s) {
  int64_t ctas = (int64_t)sms * 4;
  const int64_t need = ((M + 7) / 8 + 8 * TU - 1) / (8 * TU);
  if (ctas > need) ctas = need < 1 ? 1 : need;
  k45_skinny_nn<NT, KQ, TU><<<(unsigned)ctas, 256, 0, s>>>(M, N, K, A, lda, B, ldb, alpha, beta,
                                                           C, ldc);
  return 1;
}
template <int NT>
static int skinny_nn_t(int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                       int64_t lda, const double *B, int64_t ldb, double beta, double *C,
                       int64_t ldc, int sms, cudaStream_t s) {
  if (K <= 32)
    return skinny_nn_kt<NT, 8, 4>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sms, s);
  if (K <= 64)
    return skinny_nn_kt<NT, 16, 2>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sms, s);
  return skinny_nn_kt<NT, 24, 1>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sms, s);
}

int launch_gemm(int ta, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                double *ws, int sms, cudaStream_t s) {
  if (M < 1 || N < 1) return 0;
  if (K < 1) {  // C = beta C
    const int64_t tot = M * N;
    k41_gemm_fold<<<grid1d(tot), 256, 0, s>>>(M, N, 0, nullptr, C, ldc, 0.0, beta);
    return 1;
  }
  static const bool skinny_on = [] {
    const char *v = getenv("L1DM_SKINNY_GEMM");
    return v ? atoi(v) != 0 : true;
  }();
  if (skinny_on && skinny_tn(ta, M, N, K)) {
    const int mt = (int)((M + 7) / 8), nt = (int)((N + 7) / 8);
#define L1DM_TN(MT_, NT_) \
  if (mt == MT_ && nt == NT_) \
    return skinny_tn_t<MT_, NT_>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, sms, s);
#define L1DM_TN_M(MT_) L1DM_TN(MT_, 1) L1DM_TN(MT_, 2) L1DM_TN(MT_, 3) L1DM_TN(MT_, 4)
    L1DM_TN_M(1) L1DM_TN_M(2) L1DM_TN_M(3) L1DM_TN_M(4) L1DM_TN_M(5) L1DM_TN_M(6) L1DM_TN_M(7)
    L1DM_TN_M(8)
#undef L1DM_TN_M
#undef L1DM_TN
  }
  if (skinny_on && skinny_nn(ta, N, K)) {
    switch ((N + 7) / 8) {
      case 1: return skinny_nn_t<1>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sms, s);
      case 2: return skinny_nn_t<2>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sms, s);
      case 3: return skinny_nn_t<3>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sms, s);
      default: return skinny_nn_t<4>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sms, s);
    }
  }
  const int64_t sp = gemm_splits(ta, M, N, K, sms);
  const bool narrow = N <= 32;
  if (ta) {  // tile choice measured on B200 (profiles/r02e_gemm_tn_sweep.json)
    if (M <= 32 && narrow)  // Gram-sized: 32 x 32 tile, the 8 warps split K four ways
      return gemm_t<1, 2, 1, 4>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, sp, s);
    if (M <= 64 && narrow)  // 64 x 32 tile, K split two ways inside the CTA
      return gemm_t<1, 4, 1, 2>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, sp, s);
    return narrow ? gemm_t<1, 8, 1, 1>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, sp, s)
                  : gemm_t<1, 4, 2, 1>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, sp, s);
  }
  // the tall updates A W: 32 x 32 warp tiles (4 x 4 DMMA tiles per 8 fragment loads; measured
  // 1M x 64 x 640: 3.73 -> 3.09 ms, 1M x 32 x 32: 0.36 -> 0.23 ms in the same run)
  return narrow ? gemm_t<0, 8, 1, 1, 4>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, sp, s)
                : gemm_t<0, 4, 2, 1, 4>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, sp, s);
}

size_t jacobi_workspace(int64_t N) {
  const int64_t N2 = N + (N & 1);
  return (size_t)(2 * N * N + 6 * (N2 / 2) + kJacobiSweeps + 8) * sizeof(double);
}

// A (N x N, lda) symmetric, only read: W = eigenvalues (unsorted, the diagonal after
// convergence), V the eigenvectors (columns).  ws: jacobi_workspace(N) bytes.
int launch_jacobi(int64_t N, double *A, int64_t lda, double *W, double *V, int64_t ldv,
                  double *ws, int sms, cudaStream_t s, int *stats) {
  if (N < 1) return 0;
  if (N <= kSmallN) {
    const int N2 = (int)(N + (N & 1));
    const size_t sm = (2 * (size_t)N2 * (N2 + 1) + 3 * (size_t)(N2 / 2)) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k42_jacobi_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)((2 * (size_t)(kSmallN) * (kSmallN + 1) + 3 * kSmallN) *
                                 sizeof(double)));
      attr = true;
    }
    k42_jacobi_small<<<1, 1024, sm, s>>>((int)N, A, lda, W, V, ldv, stats);
    return 1;
  }
  // cooperative grid of 512-thread CTAs, one 2 x 2 block task per thread and step (measured on
  // B200 at N = 640: 52 ms; 16-CTA clusters or fewer, larger CTAs are slower: the steps are
  // latency-bound, not barrier-bound)
  const int64_t N2 = N + (N & 1);
  int Ni = (int)N;
  const double *Ac = A;
  void *args[] = {&Ni, &Ac, &lda, &W, &V, &ldv, &ws, &stats};
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k42_jacobi_grid, 512, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t want = ((N2 / 2) * (N2 / 2) + 511) / 512;
  int64_t blocks = (int64_t)sms * per_sm;
  if (blocks > want) blocks = want;
  if (blocks < 1) blocks = 1;
  cudaLaunchCooperativeKernel((void *)k42_jacobi_grid, dim3((unsigned)blocks), dim3(512), args, 0,
                              s);
  return 1;
}

// (+ the inverse iteration's LU factors: 5 N k doubles and N k ints, k <= 96)
size_t topk_workspace(int64_t N) {
  return (size_t)(2 * N * N + 5 * N + 8 + 6 * N * 96) * sizeof(double);
}

// The k eigenpairs of largest |lambda| of the symmetric A (N x N, lda; read only):
// lam[k], sigma[k] = |lam| in nonincreasing |lambda| order, Vs (N x k, ld k) the unit
// eigenvectors.  N <= 4096, k <= 96.  Returns the number of launches.
int launch_sym_topk(int64_t N, const double *A, int64_t lda, int64_t k, double *lam,
                    double *sigma, double *Vs, double *ws, int sms, cudaStream_t s) {
  if (N < 1 || k < 1) return 0;
  double *Ac = ws, *p = Ac + N * N, *H = p + N, *tau = H + N * N, *d = tau + N, *e = d + N;
  cudaMemcpy2DAsync(Ac, N * sizeof(double), A, lda * sizeof(double), N * sizeof(double), N,
                    cudaMemcpyDeviceToDevice, s);
  int launches = 1;
  if (N > 2) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k55_tridiag, 512, 0);
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (int64_t)sms * per_sm;
    static const int64_t cap = [] {
      const char *v = getenv("L1DM_TRIDIAG_CTAS");
      return v ? (int64_t)atoll(v) : (int64_t)0;
    }();
    if (cap > 0 && blocks > cap) blocks = cap;
    const int64_t want = (N * N + 511) / 512;
    if (blocks > want) blocks = want;
    if (blocks < 1) blocks = 1;
    int Ni = (int)N;
    void *args[] = {&Ni, &Ac, &p, &H, &tau, &d, &e};
    cudaLaunchCooperativeKernel((void *)k55_tridiag, dim3((unsigned)blocks), dim3(512), args, 0, s);
    ++launches;
  } else {
    // N <= 2: the matrix is already tridiagonal
    double *dd = d, *ee = e;
    cudaMemcpy2DAsync(dd, sizeof(double), Ac, (N + 1) * sizeof(double), sizeof(double), N,
                      cudaMemcpyDeviceToDevice, s);
    if (N == 2)
      cudaMemcpyAsync(ee, Ac + N, sizeof(double), cudaMemcpyDeviceToDevice, s);
    cudaMemsetAsync(tau, 0, N * sizeof(double), s);
  }
  const size_t sm = (size_t)((9 * N + 1) / 2 + N) * sizeof(double) +
                    (size_t)(2 * k) * sizeof(double) + (size_t)(4 * k) * sizeof(int) + 64;
  double *lw = e + N;  // LU factors of the inverse iteration (topk_workspace)
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k56_tri_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k56_tri_topk<<<1, 1024, sm, s>>>((int)N, (int)k, d, e, lam, sigma, Vs, lw);
  if (N > 2) k57_back<<<(unsigned)k, 256, 0, s>>>((int)N, (int)k, H, tau, Vs);
  return launches + 2;
}

// S (b x b) with V S orthonormal (CholeskyQR with column dropping, k43_chol_orth)
void launch_chol_orth(int64_t b, const double *G, int64_t ldg, const double *G0, int64_t ldg0,
                      double rtol, double floor_abs, double *S, cudaStream_t s) {
  const size_t sm = 2 * (size_t)b * (b + 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k43_chol_orth, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(2 * (size_t)kSmallN * (kSmallN + 1) * sizeof(double)));
    attr = true;
  }
  k43_chol_orth<<<1, 256, sm, s>>>((int)b, G, ldg, G0, ldg0, rtol, floor_abs, S);
}

void launch_select(int64_t N, int64_t k, const double *W, const double *V, int64_t ldv,
                   double *lam, double *sigma, double *Vs, int *order, cudaStream_t s) {
  k44_select<<<(unsigned)((N + 127) / 128), 128, 0, s>>>((int)N, (int)k, W, V, ldv, lam, sigma, Vs,
                                                         order);
}

void launch_scale_cols(int64_t b, const double *V, const double *lam, const double *G0,
                       int64_t ldg0, double rtol, double floor_abs, double *S, cudaStream_t s) {
  k45_scale_cols<<<grid1d(b * b), 256, 0, s>>>((int)b, V, lam, G0, ldg0, rtol, floor_abs, S);
}

void launch_split_hilo(int64_t n, int64_t b, const double *V, int64_t ldv, float *Zs,
                       cudaStream_t s) {
  k46_split<<<grid1d(n * b), 256, 0, s>>>(n, b, V, ldv, Zs);
}

void launch_combine_hilo(int64_t n, int64_t b, const double *Yr, double *Y, int64_t ldy,
                         cudaStream_t s) {
  k47_combine<<<grid1d(n * b), 256, 0, s>>>(n, b, Yr, Y, ldy);
}

void launch_axpy2d(int64_t rows, int64_t cols, double alpha, const double *S, int64_t lds,
                   double *D, int64_t ldd, cudaStream_t s) {
  if (rows < 1 || cols < 1) return;
  k48_axpy2d<<<grid1d(rows * cols), 256, 0, s>>>(rows, cols, alpha, S, lds, D, ldd);
}

void launch_symmetrize(int64_t N, double *T, int64_t ldt, cudaStream_t s) {
  k49_symmetrize<<<grid1d(N * N), 256, 0, s>>>(N, T, ldt);
}

int cg_dot_blocks() { return kDotBlocks; }
void launch_dot(int64_t n, const double *x, const double *y, double *part, cudaStream_t s) {
  k50_dot<<<kDotBlocks, 256, 0, s>>>(n, x, y, part);
}
void launch_cg_scalars(int phase, const double *part, double tol, double *st, cudaStream_t s) {
  k51_cg_scalars<<<1, 32, 0, s>>>(phase, part, kDotBlocks, tol, st);
}
void launch_cg_xr(int64_t n, const double *st, const double *p, const double *Ap, double *x,
                  double *r, cudaStream_t s) {
  k52_cg_xr<<<grid1d(n), 256, 0, s>>>(n, st, p, Ap, x, r);
}
void launch_cg_p(int64_t n, const double *st, const double *r, double *p, cudaStream_t s) {
  k53_cg_p<<<grid1d(n), 256, 0, s>>>(n, st, r, p);
}
void launch_sub(int64_t n, const double *a, const double *b, double *d, cudaStream_t s) {
  k54_sub<<<grid1d(n), 256, 0, s>>>(n, a, b, d);
}

}  // namespace l1dm
