// l1dm_query.cu — Alg. 2 "matrix-vector Query for p=1" on sm_100a.
//
// Per query block Z (n x m) the library evaluates, for every point i and column c,
//   y_ic = 2 * sum_k U^k_{rank_k(i), c} + g_c - h_i S_c
//   U^k_r = v_r P_r - Q_r,  P/Q = exclusive prefix sums of s = z_{perm_k(r)} and t = v s
// which regroups Alg. 2's x_k(i)(S3-S4) + S2 - S1 so that each coordinate
// carries one fp64 array U instead of B_i and C_i.
//
//   K4 colsums     S = 1^T Z, g = h^T Z (fp64) — deterministic two-level reduction,
//                  the last CTA folds the partials in fixed order.
//   K5 scan        per (coordinate, column block) segment, tiles of sorted rows:
//                  gather Z rows through perm (vector loads), fp64 s and t = v*s,
//                  thread -> warp (shuffle) -> block scan, single-pass decoupled
//                  look-back across tiles (fp64 payloads of 2*mb values per tile,
//                  epoch-tagged flags, tiles claimed by atomic ticket), then U.
//   K6 accumulate  per point: gather U rows at rank[k][i] for every k of the chunk
//                  and accumulate in registers (no atomics); epilogue writes Y.
#include <cuda_runtime.h>

#include "l1dm_device.cuh"
#include "l1dm_internal.h"

namespace l1dm {

// ------------------------------------------------------------------ plan
static int pow2ceil(int64_t x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

bool make_plan(int64_t n, int64_t dl, int64_t m, int64_t l2_bytes, int64_t ws_limit,
               int vec_cap, QueryPlan *p) {
  if (n < 1 || dl < 1 || m < 1 || !p) return false;
  QueryPlan q{};
  q.vec = (m % 4 == 0) ? 4 : (m % 2 == 0) ? 2 : 1;
  if (q.vec > vec_cap) q.vec = vec_cap >= 2 && m % 2 == 0 ? 2 : 1;
  const int lpr_cap = (q.vec == 4) ? 16 : (q.vec == 2) ? 16 : 32;
  int64_t need = (m + q.vec - 1) / q.vec;
  q.lpr = pow2ceil(need);
  if (q.lpr > lpr_cap) q.lpr = lpr_cap;
  q.mb = q.vec * q.lpr;
  q.col_blocks = (int)((m + q.mb - 1) / q.mb);
  q.items = 8;
  q.rows_per_tile = 8 * (32 / q.lpr) * q.items;
  q.tiles_per_segment = (n + q.rows_per_tile - 1) / q.rows_per_tile;
  q.ldu = m;
  const size_t u_per_coord = (size_t)n * (size_t)q.ldu * sizeof(double);
  const size_t slots_per_coord = (size_t)q.col_blocks * (size_t)q.tiles_per_segment;
  const size_t lb_per_coord = slots_per_coord * (sizeof(uint32_t) + 2 * 2 * q.mb * sizeof(double));
  const size_t per_coord = u_per_coord + lb_per_coord;
  if (l2_bytes > 0 && (int64_t)(4 * per_coord) <= l2_bytes) {
    // small n*m: size each chunk's workspace to stay resident in L2 between K5 and K6
    q.l2_resident = 1;
    q.kc = (int64_t)((0.375 * (double)l2_bytes) / (double)per_coord);
  } else {
    q.l2_resident = 0;
    q.kc = (ws_limit > 0) ? (int64_t)((size_t)ws_limit / per_coord) : dl;
  }
  if (q.kc < 1) q.kc = 1;
  if (q.kc > dl) q.kc = dl;
  q.chunks = (dl + q.kc - 1) / q.kc;
  q.u_bytes = (size_t)q.kc * u_per_coord;
  q.lb_slots = (size_t)q.kc * slots_per_coord;
  q.workspace_bytes = (size_t)q.kc * per_coord + (size_t)kColsumBlocks * 2 * m * sizeof(double) +
                      2 * m * sizeof(double);
  q.v6 = (m % 2 == 0) ? 2 : 1;
  int64_t lanes = (m + q.v6 - 1) / q.v6;
  q.lpp = pow2ceil(lanes > 32 ? 32 : lanes);
  q.col_groups = (int)((m + (int64_t)q.lpp * q.v6 - 1) / ((int64_t)q.lpp * q.v6));
  *p = q;
  return true;
}

// ------------------------------------------------------------------ K4
// grid (kColsumBlocks, ceil(m/CW)); thread t: column cy*CW + t%CW, row lane t/CW.
__global__ void __launch_bounds__(256)
    k4_colsums(const float *__restrict__ Z, int64_t ldz, int64_t n, int64_t m,
               const double *__restrict__ hsum, double *__restrict__ part, double *__restrict__ Sg,
               unsigned *done_ctr, unsigned *tickets, int ntickets) {
  __shared__ double s_s[256];
  __shared__ double s_g[256];
  __shared__ bool s_last;
  const int tid = threadIdx.x;
  const int CW = (int)(m < 256 ? m : 256);
  const int RP = 256 / CW;
  const int ro = tid / CW;
  const int64_t c = (int64_t)blockIdx.y * CW + tid % CW;
  const int64_t rows_per_block = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = (r0 + rows_per_block < n) ? r0 + rows_per_block : n;
  double s = 0.0, g = 0.0;
  if (ro < RP && c < m) {
    for (int64_t r = r0 + ro; r < r1; r += RP) {
      const double z = (double)Z[r * ldz + c];
      s += z;
      g = fma(hsum[r], z, g);
    }
  }
  s_s[tid] = s;
  s_g[tid] = g;
  __syncthreads();
  if (ro == 0 && c < m) {
    for (int q = 1; q < RP; ++q) {
      s += s_s[q * CW + tid];
      g += s_g[q * CW + tid];
    }
    part[(int64_t)blockIdx.x * 2 * m + c] = s;
    part[(int64_t)blockIdx.x * 2 * m + m + c] = g;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned total = gridDim.x * gridDim.y;
    s_last = (atomicAdd(done_ctr, 1u) == total - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int64_t cc = tid; cc < m; cc += 256) {
    double S = 0.0, G = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      S += __ldcg(&part[(int64_t)b * 2 * m + cc]);
      G += __ldcg(&part[(int64_t)b * 2 * m + m + cc]);
    }
    Sg[cc] = S;
    Sg[m + cc] = G;
  }
  for (int t = tid; t < ntickets; t += 256) tickets[t] = 0u;
  if (tid == 0) *done_ctr = 0u;
}

void launch_colsums(const float *Z, int64_t ldz, int64_t n, int64_t m, const double *hsum,
                    double *part, double *Sg, unsigned *done_ctr, unsigned *tickets,
                    int ntickets, cudaStream_t s) {
  const int64_t CW = m < 256 ? m : 256;
  dim3 grid(kColsumBlocks, (unsigned)((m + CW - 1) / CW));
  k4_colsums<<<grid, 256, 0, s>>>(Z, ldz, n, m, hsum, part, Sg, done_ctr, tickets, ntickets);
}

// ------------------------------------------------------------------ K5
template <int VEC>
struct ZVec;
template <>
struct ZVec<1> {
  static __device__ __forceinline__ void load(const float *p, float *o) { o[0] = __ldg(p); }
};
template <>
struct ZVec<2> {
  static __device__ __forceinline__ void load(const float *p, float *o) {
    const float2 v = __ldg(reinterpret_cast<const float2 *>(p));
    o[0] = v.x;
    o[1] = v.y;
  }
};
template <>
struct ZVec<4> {
  static __device__ __forceinline__ void load(const float *p, float *o) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
  }
};

template <int VEC>
__device__ __forceinline__ void store_u(double *p, const double *u) {
  if constexpr (VEC == 1) {
    __stcs(p, u[0]);
  } else if constexpr (VEC == 2) {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(u[0], u[1]));
  } else {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(u[0], u[1]));
    __stcs(reinterpret_cast<double2 *>(p) + 1, make_double2(u[2], u[3]));
  }
}

template <int VEC, int LPR, int ITEMS>
__global__ void __launch_bounds__(256)
    k5_scan(const uint32_t *__restrict__ perm, const float *__restrict__ sval, int64_t ldn,
            int64_t n, const float *__restrict__ Z, int64_t ldz, int64_t m,
            double *__restrict__ U, int64_t ldu, int64_t k_first, int col_blocks,
            int64_t tiles_per_seg, uint32_t *flags, double *agg, double *incl, uint32_t epoch,
            unsigned *ticket, unsigned *timeout_flag) {
  constexpr int MB = VEC * LPR;
  constexpr int RPW = 32 / LPR;
  constexpr int ROWS_W = RPW * ITEMS;
  constexpr int ROWS_T = 8 * ROWS_W;
  constexpr int NP = 2 * MB;  // payload: (s, t) per column
  __shared__ double s_wt[8][NP];
  __shared__ double s_agg[NP];
  __shared__ double s_excl[NP];
  __shared__ unsigned s_ticket;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int rg = lane / LPR, cl = lane % LPR;
  if (tid == 0) s_ticket = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t t = s_ticket;
  const int64_t seg = t / tiles_per_seg;
  const int64_t tile = t - seg * tiles_per_seg;
  const int64_t kk = seg / col_blocks;
  const int cb = (int)(seg - kk * col_blocks);
  const int64_t k = k_first + kk;
  const int64_t r0 = tile * ROWS_T + (int64_t)w * ROWS_W + (int64_t)rg * ITEMS;
  const int col0 = cb * MB + cl * VEC;
  const bool col_ok = col0 < m;  // VEC divides m, so a lane's columns are all in or all out

  // ---- sorted-order inputs of this thread's ITEMS consecutive rows
  uint32_t p[ITEMS];
  float v[ITEMS];
  const uint32_t *pp = perm + k * ldn + r0;
  const float *vp = sval + k * ldn + r0;
  if (r0 + ITEMS <= n) {
#pragma unroll
    for (int j = 0; j < ITEMS; j += 4) {
      const uint4 a = __ldg(reinterpret_cast<const uint4 *>(pp + j));
      const float4 b = __ldg(reinterpret_cast<const float4 *>(vp + j));
      p[j] = a.x; p[j + 1] = a.y; p[j + 2] = a.z; p[j + 3] = a.w;
      v[j] = b.x; v[j + 1] = b.y; v[j + 2] = b.z; v[j + 3] = b.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const bool ok = r0 + j < n;
      p[j] = ok ? __ldg(pp + j) : 0u;
      v[j] = ok ? __ldg(vp + j) : 0.0f;
    }
  }
  // ---- gather z rows into sorted order ("in the order induced by T_i")
  float z[ITEMS][VEC];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if (col_ok && r0 + j < n) {
      ZVec<VEC>::load(Z + (int64_t)p[j] * ldz + col0, z[j]);
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) z[j][q] = 0.0f;
    }
  }
  // ---- thread totals of s and t = v*s (exact in fp64)
  double own_s[VEC], own_t[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) {
    own_s[q] = 0.0;
    own_t[q] = 0.0;
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const double vj = (double)v[j];
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      const double s = (double)z[j][q];
      own_s[q] += s;
      own_t[q] = fma(vj, s, own_t[q]);
    }
  }
  // ---- warp inclusive scan across the RPW row groups of the same column lane
  double ps[VEC], pt[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) {
    ps[q] = own_s[q];
    pt[q] = own_t[q];
  }
#pragma unroll
  for (int off = 1; off < RPW; off <<= 1) {
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      const double a = __shfl_up_sync(0xFFFFFFFFu, ps[q], off * LPR);
      const double b = __shfl_up_sync(0xFFFFFFFFu, pt[q], off * LPR);
      if (rg >= off) {
        ps[q] += a;
        pt[q] += b;
      }
    }
  }
  if (rg == RPW - 1) {
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      s_wt[w][2 * (cl * VEC + q)] = ps[q];
      s_wt[w][2 * (cl * VEC + q) + 1] = pt[q];
    }
  }
  __syncthreads();
  // ---- block: warp-exclusive prefixes in place, tile aggregate
  if (tid < NP) {
    double run = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) {
      const double c = s_wt[ww][tid];
      s_wt[ww][tid] = run;
      run += c;
    }
    s_agg[tid] = run;
  }
  __syncthreads();
  // ---- decoupled look-back across the tiles of this segment (warp 0)
  if (w == 0) {
    const int64_t slot0 = seg * tiles_per_seg;
    const int64_t me = slot0 + tile;
    double acc[(NP + 31) / 32];
#pragma unroll
    for (int u = 0; u < (NP + 31) / 32; ++u) acc[u] = 0.0;
    if (tile == 0) {
#pragma unroll
      for (int u = 0; u < (NP + 31) / 32; ++u) {
        const int comp = lane + 32 * u;
        if (comp < NP) __stcg(&incl[me * NP + comp], s_agg[comp]);
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_u32(&flags[me], (epoch << 2) | kFlagInclusive);
    } else {
#pragma unroll
      for (int u = 0; u < (NP + 31) / 32; ++u) {
        const int comp = lane + 32 * u;
        if (comp < NP) __stcg(&agg[me * NP + comp], s_agg[comp]);
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_u32(&flags[me], (epoch << 2) | kFlagAggregate);
      int64_t j = tile - 1;
      uint32_t spins = 0;
      for (;;) {
        uint32_t f = 0;
        if (lane == 0) {
          for (;;) {
            f = ld_acquire_u32(&flags[slot0 + j]);
            if ((f >> 2) == (epoch & 0x3FFFFFFFu) && (f & 3u) != kFlagInvalid) break;
            if (++spins > kSpinLimit) {
              atomicOr(timeout_flag, 1u);
              f = 0xFFFFFFFFu;  // give up (results invalid; host reports ETIMEOUT)
              break;
            }
            if (spins > 32) __nanosleep(32);
          }
        }
        f = __shfl_sync(0xFFFFFFFFu, f, 0);
        if (f == 0xFFFFFFFFu) break;
        const bool inc = (f & 3u) == kFlagInclusive;
        const double *src = (inc ? incl : agg) + (slot0 + j) * NP;
#pragma unroll
        for (int u = 0; u < (NP + 31) / 32; ++u) {
          const int comp = lane + 32 * u;
          if (comp < NP) acc[u] += __ldcg(src + comp);
        }
        if (inc) break;
        --j;
      }
#pragma unroll
      for (int u = 0; u < (NP + 31) / 32; ++u) {
        const int comp = lane + 32 * u;
        if (comp < NP) __stcg(&incl[me * NP + comp], acc[u] + s_agg[comp]);
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_u32(&flags[me], (epoch << 2) | kFlagInclusive);
    }
#pragma unroll
    for (int u = 0; u < (NP + 31) / 32; ++u) {
      const int comp = lane + 32 * u;
      if (comp < NP) s_excl[comp] = acc[u];
    }
  }
  __syncthreads();
  // ---- exclusive prefix at this thread's first row, then U along its rows
  double P[VEC], Q[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) {
    const int c2 = 2 * (cl * VEC + q);
    P[q] = s_excl[c2] + s_wt[w][c2] + (ps[q] - own_s[q]);
    Q[q] = s_excl[c2 + 1] + s_wt[w][c2 + 1] + (pt[q] - own_t[q]);
  }
  if (!col_ok) return;
  double *up = U + kk * n * ldu + r0 * ldu + col0;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if (r0 + j < n) {
      const double vj = (double)v[j];
      double u[VEC];
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        const double s = (double)z[j][q];
        u[q] = fma(vj, P[q], -Q[q]);  // U_r = v_r P_r - Q_r
        P[q] += s;
        Q[q] = fma(vj, s, Q[q]);
      }
      store_u<VEC>(up + (int64_t)j * ldu, u);
    }
  }
}

template <int VEC, int LPR>
static void launch_scan_t(const QueryPlan &p, const uint32_t *perm, const float *sval,
                          int64_t ldn, int64_t n, const float *Z, int64_t ldz, int64_t m,
                          double *U, int64_t k_first, int64_t kcc, uint32_t *flags, double *agg,
                          double *incl, uint32_t epoch, unsigned *ticket, unsigned *timeout_flag,
                          cudaStream_t s) {
  const int64_t blocks = kcc * p.col_blocks * p.tiles_per_segment;
  k5_scan<VEC, LPR, 8><<<(unsigned)blocks, 256, 0, s>>>(
      perm, sval, ldn, n, Z, ldz, m, U, p.ldu, k_first, p.col_blocks, p.tiles_per_segment, flags,
      agg, incl, epoch, ticket, timeout_flag);
}

void launch_scan(const QueryPlan &p, const uint32_t *perm, const float *sval, int64_t ldn,
                 int64_t n, const float *Z, int64_t ldz, int64_t m, double *U, int64_t k_first,
                 int64_t kcc, uint32_t *flags, double *agg, double *incl, uint32_t epoch,
                 unsigned *ticket, unsigned *timeout_flag, cudaStream_t s) {
#define L1DM_SCAN(V, L)                                                                     \
  launch_scan_t<V, L>(p, perm, sval, ldn, n, Z, ldz, m, U, k_first, kcc, flags, agg, incl, \
                      epoch, ticket, timeout_flag, s)
  switch (p.vec * 100 + p.lpr) {
    case 101: L1DM_SCAN(1, 1); break;
    case 102: L1DM_SCAN(1, 2); break;
    case 104: L1DM_SCAN(1, 4); break;
    case 108: L1DM_SCAN(1, 8); break;
    case 116: L1DM_SCAN(1, 16); break;
    case 132: L1DM_SCAN(1, 32); break;
    case 201: L1DM_SCAN(2, 1); break;
    case 202: L1DM_SCAN(2, 2); break;
    case 204: L1DM_SCAN(2, 4); break;
    case 208: L1DM_SCAN(2, 8); break;
    case 216: L1DM_SCAN(2, 16); break;
    case 401: L1DM_SCAN(4, 1); break;
    case 402: L1DM_SCAN(4, 2); break;
    case 404: L1DM_SCAN(4, 4); break;
    case 408: L1DM_SCAN(4, 8); break;
    case 416: L1DM_SCAN(4, 16); break;
    default: break;
  }
#undef L1DM_SCAN
}

// ------------------------------------------------------------------ K6
template <int V6>
struct UVec;
template <>
struct UVec<1> {
  static __device__ __forceinline__ void add(const double *p, double *a) { a[0] += __ldg(p); }
};
template <>
struct UVec<2> {
  static __device__ __forceinline__ void add(const double *p, double *a) {
    const double2 u = __ldg(reinterpret_cast<const double2 *>(p));
    a[0] += u.x;
    a[1] += u.y;
  }
};

template <int V6, int LPP, int UNR>
__global__ void __launch_bounds__(256)
    k6_accumulate(const uint32_t *__restrict__ rank, int64_t ldn, int64_t n,
                  const double *__restrict__ U, int64_t ldu, int64_t k_first, int64_t kcc,
                  const double *__restrict__ hsum, const double *__restrict__ Sg,
                  double *__restrict__ Y, int64_t ldy, int64_t m, int first_chunk) {
  constexpr int PPW = 32 / LPP;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * (8 * PPW) + (int64_t)w * PPW + lane / LPP;
  const int64_t c0 = (int64_t)blockIdx.y * (LPP * V6) + (int64_t)(lane % LPP) * V6;
  if (i >= n || c0 >= m) return;
  double acc[V6];
#pragma unroll
  for (int q = 0; q < V6; ++q) acc[q] = 0.0;
  const uint32_t *rp = rank + k_first * ldn + i;
  const double *ub = U + c0;
  const int64_t ustride = n * ldu;
  int64_t kk = 0;
  for (; kk + UNR <= kcc; kk += UNR) {
    uint32_t r[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) r[u] = __ldg(rp + (kk + u) * ldn);
#pragma unroll
    for (int u = 0; u < UNR; ++u) UVec<V6>::add(ub + (kk + u) * ustride + (int64_t)r[u] * ldu, acc);
  }
  for (; kk < kcc; ++kk) {
    const uint32_t r = __ldg(rp + kk * ldn);
    UVec<V6>::add(ub + kk * ustride + (int64_t)r * ldu, acc);
  }
  double *yp = Y + i * ldy + c0;
  if (first_chunk) {
    const double hi = hsum[i];
#pragma unroll
    for (int q = 0; q < V6; ++q) yp[q] = 2.0 * acc[q] + fma(-hi, Sg[c0 + q], Sg[m + c0 + q]);
  } else {
#pragma unroll
    for (int q = 0; q < V6; ++q) yp[q] = yp[q] + 2.0 * acc[q];
  }
}

template <int V6, int LPP>
static void launch_acc_t(const QueryPlan &p, const uint32_t *rank, int64_t ldn, int64_t n,
                         const double *U, int64_t k_first, int64_t kcc, const double *hsum,
                         const double *Sg, double *Y, int64_t ldy, int64_t m, bool first,
                         cudaStream_t s) {
  constexpr int PPB = 8 * (32 / LPP);
  dim3 grid((unsigned)((n + PPB - 1) / PPB), (unsigned)p.col_groups);
  k6_accumulate<V6, LPP, 8><<<grid, 256, 0, s>>>(rank, ldn, n, U, p.ldu, k_first, kcc, hsum, Sg,
                                                 Y, ldy, m, first ? 1 : 0);
}

void launch_accumulate(const QueryPlan &p, const uint32_t *rank, int64_t ldn, int64_t n,
                       const double *U, int64_t k_first, int64_t kcc, const double *hsum,
                       const double *Sg, double *Y, int64_t ldy, int64_t m, bool first_chunk,
                       cudaStream_t s) {
#define L1DM_ACC(V, L) \
  launch_acc_t<V, L>(p, rank, ldn, n, U, k_first, kcc, hsum, Sg, Y, ldy, m, first_chunk, s)
  switch (p.v6 * 100 + p.lpp) {
    case 101: L1DM_ACC(1, 1); break;
    case 102: L1DM_ACC(1, 2); break;
    case 104: L1DM_ACC(1, 4); break;
    case 108: L1DM_ACC(1, 8); break;
    case 116: L1DM_ACC(1, 16); break;
    case 132: L1DM_ACC(1, 32); break;
    case 201: L1DM_ACC(2, 1); break;
    case 202: L1DM_ACC(2, 2); break;
    case 204: L1DM_ACC(2, 4); break;
    case 208: L1DM_ACC(2, 8); break;
    case 216: L1DM_ACC(2, 16); break;
    case 232: L1DM_ACC(2, 32); break;
    default: break;
  }
#undef L1DM_ACC
}

}  // namespace l1dm
