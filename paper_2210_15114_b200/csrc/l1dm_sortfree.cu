// l1dm_sortfree.cu — the sort-free products: even-p l_p^p (p = 2 is
// the squared Euclidean matrix), Alg. "query_p_even" (Thm. even_p) with
// the binomial coefficients and y_j the garbled text drops (R19):
//
//   (x_i - x_j)^p = sum_t C(p,t) (-1)^t x_i^(p-t) x_j^t            (p even: no sign/abs)
//   y_ic = sum_k sum_t c_t x_ik^(p-t) W_t[k][c],   W_t[k][c] = sum_j x_jk^t z_jc,  c_t = C(p,t)(-1)^t
//        = S_c hp_i + sum_{t=1}^{p-1} c_t (X^(p-t) W_t)_ic + G_c,
//   S_c = sum_j z_jc,  hp_i = sum_k x_ik^p,  G_c = sum_k W_p[k][c]  (c_0 = c_p = 1 for even p).
//
// Two dense contractions, both fp64 FMAs on the CUDA cores (fp32 inputs, fp64 products and
// sums; tensor-core formats below fp64 cannot hold the 1e-9 bar — DESIGN.md §6b):
//   K12 moment reduce  W_t = (X^t)^T Z for t = 1..p, split over point chunks; each CTA owns a
//                      64 x 64 (coordinate, column) tile of one power and a chunk of points,
//                      staging X and Z sub-tiles in shared memory; partials per chunk
//   K13 moment fold    partials summed over chunks in fixed order (deterministic); S_c, G_c
//   K14 expand         per 64-point x 64-column tile: sum over k of the powers of x times the
//                      folded W (staged in shared memory), plus S_c hp_i + G_c
// Memory: X is read p+1 times, Z p times, Y written once; FLOPs ~2 n d m (2p - 1).
#include <cuda_runtime.h>

#include <cstdint>

#include "l1dm_device.cuh"
#include "l1dm_internal.h"

namespace l1dm {

namespace {

constexpr int kTile = 64;    // output tile (rows x columns) of K12 and K14
constexpr int kStepN = 16;   // points per shared-memory step of K12
constexpr int kStepK = 16;   // coordinates per shared-memory step of K14

__device__ __forceinline__ double powi(double x, int t) {
  double r = 1.0;
  for (int q = 0; q < t; ++q) r *= x;
  return r;
}

// grid: (k tiles, c tiles, p * chunks); block 16 x 16 threads, outputs (ty + 16u, tx + 16v).
__global__ void __launch_bounds__(256)
    k12_moment_reduce(const float *__restrict__ X, int64_t ldx, const float *__restrict__ Z,
                      int64_t ldz, int64_t n, int64_t d, int64_t m, int p, int64_t chunk,
                      int64_t nchunks, double *__restrict__ part) {
  // operands staged as fp64, x already raised to the CTA's power t: converted once per element
  // (not once per use), so the inner loop is 8 shared loads and 16 FMAs per point
  __shared__ double xs[kStepN][kTile];
  __shared__ double zs[kStepN][kTile];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t k0 = (int64_t)blockIdx.x * kTile, c0 = (int64_t)blockIdx.y * kTile;
  const int t = 1 + (int)(blockIdx.z % p);
  const int64_t ch = blockIdx.z / p;
  const int64_t i0 = ch * chunk, i1 = (i0 + chunk < n) ? i0 + chunk : n;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t base = i0; base < i1; base += kStepN) {
    __syncthreads();
    for (int e = threadIdx.x; e < kStepN * kTile; e += 256) {  // coalesced row pieces
      const int r = e / kTile, q = e - (e / kTile) * kTile;
      const int64_t i = base + r;
      const float xv = (i < i1 && k0 + q < d) ? __ldcs(X + i * ldx + k0 + q) : 0.0f;
      xs[r][q] = powi((double)xv, t);
      zs[r][q] = (i < i1 && c0 + q < m) ? (double)__ldcs(Z + i * ldz + c0 + q) : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < kStepN; ++r) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // rows ty + 16 q, columns tx + 16 q: conflict-free
        a[q] = xs[r][ty + 16 * q];
        b[q] = zs[r][tx + 16 * q];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
  }
  // part[ch][t-1][k][c]
  double *out = part + ((ch * p + (t - 1)) * d) * m;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t k = k0 + ty + 16 * u;
    if (k >= d) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t c = c0 + tx + 16 * v;
      if (c < m) out[k * m + c] = acc[u][v];
    }
  }
  (void)nchunks;
}

// W[t][k][c] = c_t * sum_ch part[ch][t][k][c]  (t = 1..p-1, scaled for the expand), plus
// S_c = sum_i z_ic (fixed-order two-level sum over point blocks) and G_c = sum_k W_p[k][c].
__global__ void __launch_bounds__(256)
    k13_moment_fold(const double *__restrict__ part, int64_t nchunks, int64_t d, int64_t m,
                    int p, double *__restrict__ W, double *__restrict__ G) {
  const int64_t total = (int64_t)p * d * m;
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
      W[e] = s;  // raw W_p, folded into G below
    }
  }
  (void)G;
}

__global__ void __launch_bounds__(256)
    k13_colsum(const double *__restrict__ Wp, const float *__restrict__ Z, int64_t ldz, int64_t n,
               int64_t d, int64_t m, double *__restrict__ S, double *__restrict__ G) {
  // one CTA per column: S_c = sum_i z_ic, G_c = sum_k W_p[k][c] (fixed order per thread, then
  // a fixed-shape tree)
  __shared__ double rs[256], rg[256];
  const int64_t c = blockIdx.x;
  double s = 0.0, g = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) s += (double)Z[i * ldz + c];
  for (int64_t k = threadIdx.x; k < d; k += 256) g += Wp[k * m + c];
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

// grid: (point tiles, column tiles); block 16 x 16 threads, 4 points x 4 columns each.
// Y[i][c] = S_c hp_i + G_c + sum_{t=1}^{p-1} sum_k x_ik^(p-t) Wc[t][k][c]  (Wc pre-scaled by c_t)
template <int P>
__global__ void __launch_bounds__(256)
    k14_moment_expand(const float *__restrict__ X, int64_t ldx, int64_t n, int64_t d, int64_t m,
                      const double *__restrict__ Wc, const double *__restrict__ S,
                      const double *__restrict__ G, double *__restrict__ Y, int64_t ldy) {
  constexpr int p = P;
  __shared__ float xs[kTile][kStepK + 1];
  __shared__ double ws[P - 1][kStepK][kTile];  // c_t W_t, t = 1..p-1
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = (int64_t)blockIdx.x * kTile, c0 = (int64_t)blockIdx.y * kTile;
  double acc[4][4], hp[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    hp[a] = 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  }
  for (int64_t kb = 0; kb < d; kb += kStepK) {
    __syncthreads();
    for (int e = threadIdx.x; e < kTile * kStepK; e += 256) {
      const int r = e / kStepK, q = e - (e / kStepK) * kStepK;
      const int64_t i = i0 + r, k = kb + q;
      xs[r][q] = (i < n && k < d) ? X[i * ldx + k] : 0.0f;
    }
    for (int e = threadIdx.x; e < (p - 1) * kStepK * kTile; e += 256) {
      const int tt = e / (kStepK * kTile), rem = e - tt * (kStepK * kTile);
      const int q = rem / kTile, cc = rem - (rem / kTile) * kTile;
      const int64_t k = kb + q, c = c0 + cc;
      ws[tt][q][cc] = (k < d && c < m) ? Wc[((int64_t)tt * d + k) * m + c] : 0.0;
    }
    __syncthreads();
    for (int q = 0; q < kStepK; ++q) {
      double xp[4][P + 1];  // x^0 .. x^p of this thread's 4 points
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double x = (double)xs[ty + 16 * u][q];
        xp[u][0] = 1.0;
#pragma unroll
        for (int e = 1; e <= P; ++e) xp[u][e] = xp[u][e - 1] * x;
      }
      if (kb + q < d) {
#pragma unroll
        for (int u = 0; u < 4; ++u) hp[u] += xp[u][p];
      }
#pragma unroll
      for (int tt = 1; tt < P; ++tt) {
        double b[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) b[v] = ws[tt - 1][q][tx + 16 * v];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double a = xp[u][p - tt];
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(a, b[v], acc[u][v]);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = i0 + ty + 16 * u;
    if (i >= n) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t c = c0 + tx + 16 * v;
      if (c < m) Y[i * ldy + c] = fma(S[c], hp[u], acc[u][v] + G[c]);
    }
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

void launch_embed(const float *X, int64_t ldx, int64_t n, int64_t d, const float *G, int64_t ldg,
                  int64_t k, float *Xp, int64_t ldp, cudaStream_t s) {
  const double beta = 0.79788456080286535588;  // sqrt(2 / pi)
  dim3 grid((unsigned)((n + kTile - 1) / kTile), (unsigned)((k + kTile - 1) / kTile));
  k16_embed<<<grid, 256, 0, s>>>(X, ldx, n, d, G, ldg, k, 1.0 / (beta * (double)k), Xp, ldp);
}

size_t bilinear_workspace(int64_t n, int64_t d, int64_t m, int sms) {
  // lpp_even's layout at p = 1 (partials | W | S | G) + V (d x m)
  return lpp_even_workspace(n, d, m, 1, nullptr, nullptr, sms) + (size_t)d * m * sizeof(double);
}

// Thm. maha: f(x, y) = x^T M y, A = X M X^T, Y = X (M (X^T Z)): Alg. 7's S = M X^T
// is never formed; W = X^T Z (k12 at p = 1), V = M W (k15), Y = X V (k14 with S = G = 0).
void launch_bilinear(const float *X, int64_t ldx, const double *M, const float *Z, int64_t ldz,
                     int64_t n, int64_t d, int64_t m, double *Y, int64_t ldy, double *ws, int sms,
                     cudaStream_t s) {
  int64_t nchunks = 1, chunk = n;
  lpp_even_workspace(n, d, m, 1, &nchunks, &chunk, sms);
  double *part = ws;
  double *W = part + (size_t)nchunks * d * m;
  double *S = W + (size_t)d * m;
  double *G = S + m;
  double *V = G + m;
  dim3 g12((unsigned)((d + kTile - 1) / kTile), (unsigned)((m + kTile - 1) / kTile),
           (unsigned)nchunks);
  k12_moment_reduce<<<g12, 256, 0, s>>>(X, ldx, Z, ldz, n, d, m, 1, chunk, nchunks, part);
  int64_t b13 = (d * m + 255) / 256;
  if (b13 > 148 * 8) b13 = 148 * 8;
  k13_moment_fold<<<(unsigned)b13, 256, 0, s>>>(part, nchunks, d, m, 1, W, G);
  k15_small_gemm<<<(unsigned)b13, 256, 0, s>>>(M, W, d, m, V);
  k15_zero<<<1, 256, 0, s>>>(S, 2 * m);  // S and G (adjacent): no h S or G term
  dim3 g14((unsigned)((n + kTile - 1) / kTile), (unsigned)((m + kTile - 1) / kTile));
  k14_moment_expand<2><<<g14, 256, 0, s>>>(X, ldx, n, d, m, V, S, G, Y, ldy);
}

size_t lpp_even_workspace(int64_t n, int64_t d, int64_t m, int p, int64_t *nchunks_out,
                          int64_t *chunk_out, int sms) {
  const int64_t tiles = ((d + kTile - 1) / kTile) * ((m + kTile - 1) / kTile) * p;
  int64_t nchunks = (4 * (int64_t)sms + tiles - 1) / tiles;  // ~4 CTAs per SM over all tiles
  const int64_t min_pts = 1024;
  if (nchunks * min_pts > n) nchunks = (n + min_pts - 1) / min_pts;
  if (nchunks < 1) nchunks = 1;
  const int64_t chunk = (n + nchunks - 1) / nchunks;
  nchunks = (n + chunk - 1) / chunk;
  if (nchunks_out) *nchunks_out = nchunks;
  if (chunk_out) *chunk_out = chunk;
  // partials | W (p x d x m) | S (m) | G (m)
  return ((size_t)nchunks * p * d * m + (size_t)p * d * m + 2 * (size_t)m) * sizeof(double);
}

void launch_lpp_even(const float *X, int64_t ldx, const float *Z, int64_t ldz, int64_t n,
                     int64_t d, int64_t m, int p, double *Y, int64_t ldy, double *ws, int sms,
                     cudaStream_t s) {
  int64_t nchunks = 1, chunk = n;
  lpp_even_workspace(n, d, m, p, &nchunks, &chunk, sms);
  double *part = ws;
  double *W = part + (size_t)nchunks * p * d * m;
  double *S = W + (size_t)p * d * m;
  double *G = S + m;
  dim3 g12((unsigned)((d + kTile - 1) / kTile), (unsigned)((m + kTile - 1) / kTile),
           (unsigned)(p * nchunks));
  k12_moment_reduce<<<g12, 256, 0, s>>>(X, ldx, Z, ldz, n, d, m, p, chunk, nchunks, part);
  int64_t b13 = ((int64_t)p * d * m + 255) / 256;
  if (b13 > 148 * 8) b13 = 148 * 8;
  k13_moment_fold<<<(unsigned)b13, 256, 0, s>>>(part, nchunks, d, m, p, W, G);
  k13_colsum<<<(unsigned)m, 256, 0, s>>>(W + (size_t)(p - 1) * d * m, Z, ldz, n, d, m, S, G);
  dim3 g14((unsigned)((n + kTile - 1) / kTile), (unsigned)((m + kTile - 1) / kTile));
  switch (p) {
    case 2: k14_moment_expand<2><<<g14, 256, 0, s>>>(X, ldx, n, d, m, W, S, G, Y, ldy); break;
    case 4: k14_moment_expand<4><<<g14, 256, 0, s>>>(X, ldx, n, d, m, W, S, G, Y, ldy); break;
    case 6: k14_moment_expand<6><<<g14, 256, 0, s>>>(X, ldx, n, d, m, W, S, G, Y, ldy); break;
    default: break;
  }
}

}  // namespace l1dm
