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
#include <math_constants.h>

#include <cstdlib>

#include "l1dm_device.cuh"
#include "l1dm_internal.h"

namespace l1dm {

// ------------------------------------------------------------------ plan
static int pow2ceil(int64_t x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

static void plan_sizes(QueryPlan &q, int64_t n, int64_t dl, int64_t m, int64_t l2_bytes,
                       int64_t ws_limit) {
  q.mb = q.lpr * q.vc;
  q.col_blocks = (int)((m + q.mb - 1) / q.mb);
  q.items = scan_items(q.lpr, q.vc);
  q.rows_per_tile = 8 * (32 / q.lpr) * q.items;
  q.tiles_per_segment = (n + q.rows_per_tile - 1) / q.rows_per_tile;
  q.ldu = m;
  const size_t u_per_coord = (size_t)n * (size_t)q.ldu * sizeof(double);
  const size_t slots_per_coord = (size_t)q.col_blocks * (size_t)q.tiles_per_segment;
  const size_t lb_per_coord = slots_per_coord * (sizeof(uint32_t) + 2 * 2 * q.mb * sizeof(double));
  const size_t zs_per_coord = (q.mb == 1) ? (size_t)n * sizeof(float) : 0;  // m == 1 staging
  const size_t per_coord = u_per_coord + lb_per_coord + zs_per_coord;
  if (l2_bytes > 0 && (int64_t)(4 * per_coord) <= l2_bytes) {
    // small n*m: size each chunk's workspace to stay resident in L2 between K5 and K6
    q.l2_resident = 1;
    q.kc = (int64_t)((0.375 * (double)l2_bytes) / (double)per_coord);
  } else {
    q.l2_resident = 0;
    // one chunk's U is also capped: measured on B200, the rank gather of K6 drops from ~5.8
    // to ~3.2 TB/s when the chunk's U spans ~100 GB (c5, 96 coordinates), not at 64 GB.
    const size_t lim = (ws_limit > 0 && (size_t)ws_limit < kMaxChunkBytes) ? (size_t)ws_limit
                                                                           : kMaxChunkBytes;
    q.kc = (int64_t)(lim / per_coord);
  }
  if (q.kc < 1) q.kc = 1;
  if (q.kc > dl) q.kc = dl;
  q.chunks = (dl + q.kc - 1) / q.kc;
  q.u_bytes = (size_t)q.kc * u_per_coord;
  q.lb_slots = (size_t)q.kc * slots_per_coord;
  q.workspace_bytes = (size_t)q.kc * per_coord + (size_t)dl * 2 * m * sizeof(double) +
                      2 * m * sizeof(double);
}

bool make_plan(int64_t n, int64_t dl, int64_t m, int64_t l2_bytes, int64_t ws_limit,
               int vec_cap, int mode, QueryPlan *p) {
  if (n < 1 || dl < 1 || m < 1 || !p) return false;
  QueryPlan q{};
  // Columns per scan segment: the whole Z row when it fits one warp (two columns per lane
  // for 32 < m <= 64) — random row gathers from DRAM are only efficient when wide
  // (measured on B200: 64 B rows ~2.6 TB/s, 128 B ~4.5, 256 B ~5.5 of useful bandwidth).
  q.vc = (m > 32 && m % 2 == 0) ? 2 : 1;
  q.lpr = pow2ceil((m + q.vc - 1) / q.vc > 32 ? 32 : (m + q.vc - 1) / q.vc);
  // gather chunk (floats per cp.async): 16 B when rows/columns allow it
  auto pick_vec = [&](int mb) {
    int v = (m % 4 == 0) ? 4 : (m % 2 == 0) ? 2 : 1;
    if (v > vec_cap) v = (vec_cap >= 2 && m % 2 == 0) ? 2 : 1;
    while (v > mb) v >>= 1;
    return v;
  };
  q.vec = pick_vec(q.lpr * q.vc);
  plan_sizes(q, n, dl, m, l2_bytes, ws_limit);
  // Optional: split columns further (more, narrower segments) — off by default.
  static const int64_t target = [] {
    const char *e = getenv("L1DM_SCAN_SEGMENTS");  // tuning override
    return e ? atoll(e) : kScanTargetSegments;
  }();
  while (q.lpr * q.vc > 8 && q.kc * (int64_t)q.col_blocks < target) {
    if (q.vc == 2) q.vc = 1; else q.lpr /= 2;
    q.vec = pick_vec(q.lpr * q.vc);
    plan_sizes(q, n, dl, m, l2_bytes, ws_limit);
  }
  // Scatter mode: when a block of Y (n x mb fp64) and the matching block of Z fit in L2, the
  // scan adds 2U straight into Y with L2 atomics (no U workspace round trip through HBM, no
  // rank gather).  m == 1 uses the reduce-then-scan kernels; m > 1 runs one scan launch per
  // column block of mb columns over a column-block-major copy of Z.
  // mode (1 gather, 2 scatter), else L1DM_SCATTER=0/1, and L1DM_SCATTER_MB override.
  static const int scatter_env_ = [] {
    const char *e = getenv("L1DM_SCATTER");
    return e ? atoi(e) : -1;
  }();
  // an explicit per-handle mode (l1dm_set_query_mode) wins over the environment
  const int scatter_env = mode == 1 ? 0 : mode == 2 ? 1 : scatter_env_;
  static const int scatter_mb_env = [] {
    const char *e = getenv("L1DM_SCATTER_MB");
    return e ? atoi(e) : 0;
  }();
  int smb = 0;  // columns per scatter block (0: no scatter)
  if (m == 1) {
    smb = (scatter_env == 1 || (scatter_env < 0 && l2_bytes > 0 && n * 16 <= l2_bytes)) ? 1 : 0;
  } else if (scatter_env != 0) {
    if (scatter_mb_env > 0) {
      smb = scatter_mb_env;
    } else {
      // Measured on B200: per (point, coordinate, column block) the scatter scan
      // costs ~24 ps at mb = 8 and ~17-20 ps at mb = 4, i.e. ~3 and ~4.5-5 ps per update, against
      // ~3.6 (m = 64) to ~5 (m = 16) ps per update for the gather path.  So mb = 8 wins whenever
      // its Yt + Zt block (12 n mb bytes) roughly fits L2, mb = 4 only for narrow queries, and
      // tiny n (launch-bound) stays on the gather path.
      const double cap = kScatterL2Fraction * (double)l2_bytes;
      if (l2_bytes > 0 && n >= kScatterMinN) {
        if ((double)n * 8 * 12.0 <= cap) smb = 8;
        else if ((double)n * 4 * 12.0 <= cap && m <= kScatterNarrowM) smb = 4;
      }
      if (!smb && scatter_env == 1) smb = 4;
    }
    if (smb > 0) {
      if (smb > 16) smb = 16;
      smb = pow2ceil(smb);
      while (smb > 1 && smb >= 2 * m) smb >>= 1;
    }
  }
  q.scatter = smb > 0 ? 1 : 0;
  q.zt_floats = 0;
  if (q.scatter && m > 1) {
    q.vc = 1;
    q.lpr = smb;
    q.vec = smb >= 4 ? 4 : smb;  // Zt rows are smb floats, 16-B aligned blocks
    plan_sizes(q, n, dl, m, l2_bytes, ws_limit);
    q.items = 4 * smb;  // k5_scan_seq: 1024-row tiles, 4*mb consecutive rows per thread
    q.rows_per_tile = 1024;
    q.tiles_per_segment = (n + q.rows_per_tile - 1) / q.rows_per_tile;
    q.zt_floats = (int64_t)q.col_blocks * n * smb;
  }
  if (q.scatter) {
    q.kc = dl;  // every coordinate in one launch: nothing to hold between scan and accumulate
    q.chunks = 1;
    q.l2_resident = 1;
    q.u_bytes = 0;
    // m > 1: one launch per column block, the look-back state is reused between launches
    q.lb_slots = (size_t)dl * (m > 1 ? 1 : q.col_blocks) * q.tiles_per_segment;
    q.workspace_bytes = q.lb_slots * (sizeof(uint32_t) + 2 * 2 * q.mb * sizeof(double)) +
                        (m == 1 ? (size_t)dl * n * sizeof(float) : 0) +
                        (size_t)q.zt_floats * sizeof(float) +
                        (m > 1 ? (size_t)n * q.mb * sizeof(double) : 0) +
                        (size_t)dl * 2 * m * sizeof(double) + 2 * m * sizeof(double);
  }
  q.v6 = (m % 2 == 0) ? 2 : 1;
  int64_t lanes = (m + q.v6 - 1) / q.v6;
  q.lpp = pow2ceil(lanes > 32 ? 32 : lanes);
  q.col_groups = (int)((m + (int64_t)q.lpp * q.v6 - 1) / ((int64_t)q.lpp * q.v6));
  *p = q;
  return true;
}

// Plan of an l_p^p query with odd p > 1: every pass is the column-block seq scan
// with (p+1) moments per column.  Scatter when a block of Yt + Zt fits L2 (as for p = 1), else
// gather: the apply pass stores W in sorted order into the U workspace (chunks of kc
// coordinates) and k6 sums it over the chunk at rank (factor 1, no epilogue).
bool make_lp_plan(int64_t n, int64_t dl, int64_t m, int lp, int64_t l2_bytes, int64_t ws_limit,
                  int mode, QueryPlan *p) {
  if (n < 1 || dl < 1 || m < 1 || !p || lp < 3 || lp > 7 || !(lp & 1)) return false;
  QueryPlan base;
  if (!make_plan(n, dl, m, l2_bytes, ws_limit, 4, mode, &base)) return false;
  QueryPlan q = base;
  const bool scatter = base.scatter != 0;
  int mb;
  if (scatter) {
    mb = base.mb < 2 ? 2 : base.mb;  // seq kernels exist for mb = 2..16
  } else {
    mb = 16;                          // gather: Zt rows of 64 B from HBM
    while (mb > 2 && mb >= 2 * m) mb >>= 1;
  }
  const int K = lp + 1;
  q.scatter = scatter ? 1 : 0;
  q.mb = mb;
  q.lpr = mb;
  q.vc = 1;
  q.vec = mb >= 4 ? 4 : mb;
  q.col_blocks = (int)((m + mb - 1) / mb);
  q.items = 4 * mb;
  q.rows_per_tile = 1024;
  q.tiles_per_segment = (n + 1023) / 1024;
  q.zt_floats = (int64_t)q.col_blocks * n * mb;
  q.ldu = m;
  const size_t agg_per_coord = (size_t)q.tiles_per_segment * K * mb * sizeof(double);
  if (scatter) {
    q.kc = dl;
    q.chunks = 1;
    q.u_bytes = 0;
    q.l2_resident = 1;
  } else {
    const size_t per_coord = (size_t)n * m * sizeof(double) + agg_per_coord;
    const size_t lim = (ws_limit > 0 && (size_t)ws_limit < kMaxChunkBytes) ? (size_t)ws_limit
                                                                           : kMaxChunkBytes;
    q.kc = (int64_t)(lim / per_coord);
    if (q.kc < 1) q.kc = 1;
    if (q.kc > dl) q.kc = dl;
    q.chunks = (dl + q.kc - 1) / q.kc;
    q.u_bytes = (size_t)q.kc * n * m * sizeof(double);
    q.l2_resident = 0;
  }
  q.lb_slots = (size_t)q.kc * q.tiles_per_segment;
  q.workspace_bytes = q.u_bytes + q.lb_slots * K * mb * sizeof(double) +
                      (size_t)q.zt_floats * sizeof(float) +
                      (scatter ? (size_t)n * mb * sizeof(double) : 0) +
                      (size_t)dl * K * m * sizeof(double);
  *p = q;
  return true;
}

// ------------------------------------------------------------------ K4
// Query totals from the scan's segment totals: S_c = sum_j z_jc (coordinate 0's segment),
// g_c = sum_k T_kc = sum_j h_j z_jc, summed over the shard's coordinates in fixed order.
__global__ void __launch_bounds__(256)
    k4_totals(const double *__restrict__ segtot, int64_t ld_seg, int64_t dl, int64_t mc,
              double *__restrict__ S, double *__restrict__ g) {
  for (int64_t c = (int64_t)blockIdx.x * 256 + threadIdx.x; c < mc; c += (int64_t)gridDim.x * 256) {
    double gc = 0.0;
    for (int64_t k = 0; k < dl; ++k) gc += segtot[k * ld_seg + 2 * c + 1];
    S[c] = segtot[2 * c];
    g[c] = gc;
  }
}

void launch_totals(const double *segtot, int64_t ld_seg, int64_t dl, int64_t mc, double *S,
                   double *g, cudaStream_t s) {
  int64_t blocks = (mc + 255) / 256;
  if (blocks > 148) blocks = 148;
  k4_totals<<<(unsigned)blocks, 256, 0, s>>>(segtot, ld_seg, dl, mc, S, g);
}

// ------------------------------------------------------------------ K5
// One large tile per CTA.  Tiles are claimed by atomic ticket when the CTA starts (segments
// interleaved, so a tile's predecessor is nseg tickets older); a CTA never holds an
// unpublished ticket while it waits, so look-back waits are bounded by one tile's load
// latency.  perm/sval and the gathered Z rows of the tile are staged in shared memory with
// cp.async (the whole tile's loads are in flight at once), then the tile is scanned straight
// out of shared memory.
//
template <int VC>
__device__ __forceinline__ void lds_cols(const float *p, float *o) {
  if constexpr (VC == 1) {
    o[0] = *p;
  } else {
    const float2 v = *reinterpret_cast<const float2 *>(p);
    o[0] = v.x;
    o[1] = v.y;
  }
}
template <int VC>
__device__ __forceinline__ void stcs_cols(double *p, const double *u) {
  if constexpr (VC == 1) {
    __stcs(p, u[0]);
  } else {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(u[0], u[1]));
  }
}

// Lane mapping: lane = rg * LPR + cl owns columns [cl*VC, cl*VC+VC) of the segment
// (mb = LPR*VC columns) and,
// for j = 0..ITEMS-1, sorted row  w*ROWS_W + j*RPW + rg.  At fixed j a warp covers RPW
// consecutive rows x all mb columns: shared-memory reads are conflict-free and each warp
// store writes RPW full mb*8-byte row pieces of U.  The scan along rows is a warp scan over
// the RPW row groups per j plus a running carry across j.
template <int LPR, int VC, int ITEMS>
struct ScanCfg {
  static constexpr int MB = LPR * VC;
  static constexpr int NW = 8;
  static constexpr int NT = 32 * NW;
  static constexpr int RPW = 32 / LPR;
  static constexpr int ROWS_W = RPW * ITEMS;
  static constexpr int R = NW * ROWS_W;        // rows per tile
  static constexpr int NP = 2 * MB;            // look-back payload: (s, t) per column
  static constexpr int ZST = R * MB;           // floats of gathered Z per tile
  // dynamic smem: Z stage | sval | perm (+ small static arrays)
  static constexpr size_t SMEM = (size_t)ZST * 4 + (size_t)R * 4 * 2;
};


// Decoupled look-back (Merrill & Garland) for tile `tile` of the segment whose slots start at
// slot0: publishes the tile aggregate s_agg[NP] (epoch-tagged flag, release at gpu scope), sums
// the predecessors' payloads into s_excl[NP] (warp 0 polls a 32-predecessor window, all NT
// threads sum payloads), then publishes the inclusive prefix.  Waits are bounded by kSpinLimit
// (then *timeout_flag is raised and the results are invalid).  Called by all NT threads.
template <int NP, int NT>
__device__ __forceinline__ void lookback(int64_t slot0, int64_t tile, uint32_t *flags, double *agg,
                                         double *incl, uint32_t epoch, unsigned *timeout_flag,
                                         const double *s_agg, double *s_excl, double *s_red,
                                         int *s_q, int64_t *s_j) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t me = slot0 + tile;
  // payloads are read back within a few tiles: keep them from displacing L2-resident data
  const uint64_t pol = l2_policy_evict_first();
  if (tid < NP) s_excl[tid] = 0.0;
  if (tile == 0) {
    if (tid < NP) {
      st_f64_hint(&incl[me * NP + tid], s_agg[tid], pol);
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_u32(&flags[me], (epoch << 2) | kFlagInclusive);
    }
  } else {
    if (tid < NP) {
      st_f64_hint(&agg[me * NP + tid], s_agg[tid], pol);
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_u32(&flags[me], (epoch << 2) | kFlagAggregate);
    }
    int64_t j = tile - 1;  // nearest predecessor not yet summed
    for (;;) {
      // warp 0: lane l examines predecessor j - l; q = nearest inclusive prefix in the window
      if (w == 0) {
        const int64_t jl = j - lane;
        uint32_t f = (epoch << 2) | kFlagInclusive;  // jl < 0: empty prefix
        if (jl >= 0) {
          uint32_t spins = 0;
          for (;;) {
            f = ld_acquire_u32(&flags[slot0 + jl]);
            if ((f >> 2) == (epoch & 0x3FFFFFFFu) && (f & 3u) != kFlagInvalid) break;
            if (++spins > kSpinLimit) {
              atomicOr(timeout_flag, 1u);
              f = (epoch << 2) | kFlagInclusive;  // give up (results invalid; ETIMEOUT)
              break;
            }
            if (spins > 8) __nanosleep(32);
          }
        }
        const uint32_t inc_mask = __ballot_sync(0xFFFFFFFFu, (f & 3u) == kFlagInclusive);
        if (lane == 0) {
          *s_q = inc_mask ? __ffs(inc_mask) - 1 : 32;
          *s_j = j;
        }
      }
      __syncthreads();
      const int q = *s_q;
      const int64_t jw = *s_j;
      const int cnt = q < 32 ? q + 1 : 32;  // tiles jw .. jw-cnt+1 (the last one INCL if q<32)
      constexpr int GROUPS = NT / NP;       // all threads sum payloads, comp = tid % NP
      double part = 0.0;
      {
        const int comp = tid % NP, g = tid / NP;
        if (g < GROUPS) {
          for (int b = g; b < cnt; b += GROUPS) {
            const int64_t jj = jw - b;
            if (jj < 0) break;
            part += __ldcg((b == q ? incl : agg) + (slot0 + jj) * NP + comp);
          }
        }
      }
      s_red[tid] = part;
      __syncthreads();
      if (tid < NP) {
        double sum = 0.0;
#pragma unroll
        for (int g = 0; g < GROUPS; ++g) sum += s_red[g * NP + tid];
        s_excl[tid] += sum;
      }
      __syncthreads();
      if (q < 32) break;
      j = jw - 32;
    }
    if (tid < NP) {
      st_f64_hint(&incl[me * NP + tid], s_excl[tid] + s_agg[tid], pol);
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_u32(&flags[me], (epoch << 2) | kFlagInclusive);
    }
  }
}

template <int LPR, int VC, int CH>
__global__ void __launch_bounds__(256, 2)
    k5_scan(const uint32_t *__restrict__ perm, const float *__restrict__ sval, int64_t ldn,
            int64_t n, const float *__restrict__ Z, int64_t ldz, int64_t m,
            double *__restrict__ U, int64_t ldu, int64_t k_first, int col_blocks, int64_t nseg,
            int64_t total, uint32_t *flags, double *agg, double *incl, uint32_t epoch,
            unsigned *ticket, unsigned *timeout_flag, int64_t tiles_per_seg,
            double *__restrict__ segtot, int64_t ld_seg) {
  constexpr int ITEMS = scan_items(LPR, VC);
  using C = ScanCfg<LPR, VC, ITEMS>;
  constexpr int MB = C::MB, RPW = C::RPW, ROWS_W = C::ROWS_W, R = C::R, NP = C::NP, NW = C::NW;
  constexpr int NT = C::NT;
  constexpr int CPR = MB * 4 / CH;  // cp.async chunks per gathered row
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *zb = reinterpret_cast<float *>(smem_raw);        // [R][MB]
  float *vb = zb + C::ZST;                                 // [R]
  uint32_t *pb = reinterpret_cast<uint32_t *>(vb + R);     // [R]
  __shared__ double s_wt[NW * NP];  // per-warp totals, then warp-exclusive prefixes
  __shared__ double s_agg[NP];
  __shared__ double s_excl[NP];
  __shared__ double s_red[NT];
  __shared__ int64_t s_t;
  __shared__ int64_t s_j;
  __shared__ int s_q;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int rg = lane / LPR, cl = lane - (lane / LPR) * LPR;

  if (tid == 0) s_t = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t t = s_t;
  const int64_t tile = t / nseg;
  const int64_t seg = t - tile * nseg;
  const int64_t kk = seg / col_blocks;
  const int cb = (int)(seg - kk * col_blocks);
  const int64_t row0 = tile * R;
  const int64_t nrows = (n - row0 < R) ? (n - row0) : R;

  // ---- stage perm + sval of the tile (rows in [n, ldn) are padding: loaded, unused)
  {
    const uint32_t *pp = perm + (k_first + kk) * ldn + row0;
    const float *vp = sval + (k_first + kk) * ldn + row0;
    for (int c = tid; c < R / 4; c += NT) {
      const bool ok = row0 + 4 * c < ldn;
      cp_async<16>(pb + 4 * c, ok ? (const void *)(pp + 4 * c) : (const void *)perm, ok);
      cp_async<16>(vb + 4 * c, ok ? (const void *)(vp + 4 * c) : (const void *)sval, ok);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  }
  // ---- gather z rows into sorted order ("in the order induced by T_i")
  {
    const int64_t col_base = (int64_t)cb * MB;
    for (int e = tid; e < R * CPR; e += NT) {
      const int r = e / CPR, ch = e - (e / CPR) * CPR;
      const int64_t col = col_base + ch * (CH / 4);
      const bool ok = (r < nrows) && (col < m);
      const float *src = ok ? Z + (int64_t)pb[r] * ldz + col : Z;
      cp_async<CH>(zb + r * MB + ch * (CH / 4), src, ok);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  }
  const int64_t col = (int64_t)cb * MB + cl * VC;
  const bool col_ok = col < m;  // VC divides m: a lane's columns are all in or all out
  const int rbase = w * ROWS_W + rg;  // row of item j: rbase + j * RPW

  // ---- phase 1: warp totals of s = z and t = v z (fp64; products exact)
  double cs[VC], ct[VC];  // carry: sums over this warp's items so far (all row groups)
#pragma unroll
  for (int q = 0; q < VC; ++q) {
    cs[q] = 0.0;
    ct[q] = 0.0;
  }
#pragma unroll 4
  for (int j = 0; j < ITEMS; ++j) {
    const int r = rbase + j * RPW;
    float zz[VC];
    lds_cols<VC>(zb + r * MB + cl * VC, zz);     // zero-filled past n / past m
    const double vj = (r < nrows) ? (double)vb[r] : 0.0;
#pragma unroll
    for (int q = 0; q < VC; ++q) {
      double a = (double)zz[q], b = vj * (double)zz[q];
#pragma unroll
      for (int off = 1; off < RPW; off <<= 1) {  // reduce across the RPW row groups
        a += __shfl_xor_sync(0xFFFFFFFFu, a, off * LPR);
        b += __shfl_xor_sync(0xFFFFFFFFu, b, off * LPR);
      }
      cs[q] += a;
      ct[q] += b;
    }
  }
  if (rg == 0) {
#pragma unroll
    for (int q = 0; q < VC; ++q) {
      s_wt[w * NP + 2 * (cl * VC + q)] = cs[q];
      s_wt[w * NP + 2 * (cl * VC + q) + 1] = ct[q];
    }
  }
  __syncthreads();
  if (tid < NP) {  // warp-exclusive prefixes in place, tile aggregate
    double run = 0.0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) {
      const double c = s_wt[ww * NP + tid];
      s_wt[ww * NP + tid] = run;
      run += c;
    }
    s_agg[tid] = run;
  }
  __syncthreads();

  // ---- decoupled look-back (Merrill & Garland) across the tiles of this segment
  const int64_t slot0 = seg * tiles_per_seg;
  lookback<NP, NT>(slot0, tile, flags, agg, incl, epoch, timeout_flag, s_agg, s_excl, s_red, &s_q,
                   &s_j);
  // ---- the segment's totals (S = sum z, T_k = sum x z: Alg. 2's B_i[n], C_i[n])
  // feed the epilogue g - h_i S with g = sum_k T_k, so no extra pass over Z.
  if (tile == tiles_per_seg - 1 && tid < NP) {
    const int64_t c = (int64_t)cb * MB + tid / 2;
    if (c < m) segtot[(k_first + kk) * ld_seg + 2 * c + (tid & 1)] = s_excl[tid] + s_agg[tid];
  }
  // ---- phase 2: exclusive prefixes P, Q along the rows, U_r = v_r P_r - Q_r
  double P[VC], Q[VC];
#pragma unroll
  for (int q = 0; q < VC; ++q) {
    const int c2 = 2 * (cl * VC + q);
    P[q] = s_excl[c2] + s_wt[w * NP + c2];
    Q[q] = s_excl[c2 + 1] + s_wt[w * NP + c2 + 1];
  }
  double *ub = U + kk * n * ldu + (row0 + rbase) * ldu + col;
  if constexpr (RPW == 1) {
    // one row per warp step (a lane per column group): the exclusive prefixes are the carries
    const int nmine = (int)(nrows - rbase < ITEMS ? (nrows - rbase < 0 ? 0 : nrows - rbase)
                                                  : ITEMS);
    const float *zr = zb + rbase * MB + cl * VC;
    const float *vr = vb + rbase;
    if (col_ok) {
#pragma unroll 4
      for (int j = 0; j < nmine; ++j) {
        float zz[VC];
        lds_cols<VC>(zr + j * MB, zz);
        const double vj = (double)vr[j];
        double u[VC];
#pragma unroll
        for (int q = 0; q < VC; ++q) {
          const double sz = (double)zz[q];
          u[q] = fma(vj, P[q], -Q[q]);  // U_r = v_r P_r - Q_r
          P[q] += sz;
          Q[q] = fma(vj, sz, Q[q]);     // v z is exact in fp64: same as Q + v z
        }
        stcs_cols<VC>(ub + (int64_t)j * ldu, u);
      }
    }
  } else {
#pragma unroll 4
  for (int j = 0; j < ITEMS; ++j) {
    const int r = rbase + j * RPW;
    float zz[VC];
    lds_cols<VC>(zb + r * MB + cl * VC, zz);
    const double vj = (r < nrows) ? (double)vb[r] : 0.0;
    double u[VC];
#pragma unroll
    for (int q = 0; q < VC; ++q) {
      const double s = (double)zz[q], tt = vj * s;
      double a = s, b = tt;  // inclusive scan across the RPW row groups of this column
#pragma unroll
      for (int off = 1; off < RPW; off <<= 1) {
        const double a2 = __shfl_up_sync(0xFFFFFFFFu, a, off * LPR);
        const double b2 = __shfl_up_sync(0xFFFFFFFFu, b, off * LPR);
        if (rg >= off) {
          a += a2;
          b += b2;
        }
      }
      u[q] = fma(vj, P[q] + (a - s), -(Q[q] + (b - tt)));  // exclusive prefixes at row r
      // carry: this item's totals over all row groups (held by the last row group)
      P[q] += __shfl_sync(0xFFFFFFFFu, a, (RPW - 1) * LPR + cl);
      Q[q] += __shfl_sync(0xFFFFFFFFu, b, (RPW - 1) * LPR + cl);
    }
    if (col_ok && r < nrows) {
      stcs_cols<VC>(ub + (int64_t)j * RPW * ldu, u);
    }
  }
  }
}

// Column-block scan with thread-sequential rows ("seq"), used by scatter mode for m > 1 and by
// every l_p^p query with odd p > 1 (gather and scatter).  One column block of MB columns is
// read from the compact Zt block (row stride MB).  For P = 1 it evaluates U_r = v_r P_r - Q_r
// (DESIGN.md §2); for odd P, per column, the P+1 exclusive prefix moments
//   M_t(r) = sum_{r' < r} z_{perm(r')} v_{r'}^t,  t = 0..P,
// and the coordinate's whole contribution to point perm(r)
//   W_r = sum_t c_t v_r^(P-t) (2 M_t(r) - T_t),  c_t = C(P,t) (-1)^t,  T_t = M_t(n).
// Reduce-then-scan, no inter-CTA waits (ncu showed the decoupled look-back's barriers and
// fences dominating this L2-bound kernel):
//   SEQ_REDUCE       per tile: column totals of the P+1 moments     -> agg[seg][tile][NP]
//   k5_seq_prefix    per (segment, component): exclusive scan over tiles, segment totals T
//   SEQ_APPLY_RED    per tile: CTA scan + tile prefix; P = 1: 2U, P > 1: W, added into
//                    Yt[perm[r]][c] (row stride MB) by fp64 L2 reductions
//   SEQ_APPLY_STORE  the same value stored at U[r][c] in sorted order (gather mode, P > 1)
// Thread (g, c) owns ITEMS consecutive sorted rows of column c, so the row loop is a
// thread-sequential scan; only per-thread totals are scanned across the CTA (shuffles over the
// 32/MB groups of a warp, then across warps).  At each row step a warp touches 32/MB rows x MB
// consecutive columns: every reduction request is one row segment of Yt.
#ifndef L1DM_LB_ITEMS
#define L1DM_LB_ITEMS 4  // single-pass apply: consecutive rows per thread / mb (mb >= 2)
#endif
template <int MB, int P = 1, int NTT = 256, int IM = 4>
struct SeqCfg {
  static constexpr int NT = NTT, NW = NTT / 32;
  static constexpr int G = NT / MB;           // row groups per tile
  static constexpr int ITEMS = MB == 1 ? 8 : IM * MB;  // consecutive rows per thread
  static constexpr int R = G * ITEMS;         // 1024 rows per tile
  static constexpr int GPW = 32 / MB;         // groups per warp
  static constexpr int GS = ITEMS * MB + MB;  // padded floats per group of the Z stage
  static constexpr int PS = ITEMS + 4;        // padded words per group of perm / sval
  static constexpr int K = P + 1;             // moments per column
  static constexpr int NP = K * MB;           // payload per tile
  static constexpr int CH = MB * 4 >= 16 ? 16 : MB * 4;  // bytes per cp.async of a Z row
  static constexpr size_t SMEM = (size_t)G * GS * 4 + (size_t)G * PS * 4 * 2;
};
enum { SEQ_REDUCE = 0, SEQ_APPLY_RED = 1, SEQ_APPLY_STORE = 2, SEQ_APPLY_FX = 3 };
// SEQ_APPLY_FX (P = 1): the 2U values are added into Yt as 64-bit fixed-point integers,
// q = rint(2U 2^F_c) with column c's scale 2^F_c = fx[c] (launch_fx_scale below; fx points at
// the block's first column), by integer L2 reductions — integer addition is associative, so Yt
// (and Y) are bitwise reproducible whatever the order of the reductions (R16); the
// block write-out scales back by 2^-F_c.

// c_t = C(P, t) (-1)^t
template <int P>
__host__ __device__ constexpr double lp_coef(int t) {
  double b = 1.0;
  for (int q = 0; q < t; ++q) b = b * (double)(P - q) / (double)(q + 1);
  return (t & 1) ? -b : b;
}

template <int MB, int MODE, int P>
__global__ void __launch_bounds__(256)
    k5_scan_seq(const uint32_t *__restrict__ perm, const float *__restrict__ sval, int64_t ldn,
                int64_t n, const float *__restrict__ zt, int64_t mc, double *__restrict__ out,
                int64_t ldo, int64_t nseg, int64_t tiles_per_seg, double *__restrict__ agg,
                int64_t agg_ld, const double *__restrict__ segtot, int64_t ld_seg,
                const double *__restrict__ fx) {
  using C = SeqCfg<MB, P>;
  constexpr int NT = C::NT, NW = C::NW, ITEMS = C::ITEMS, R = C::R, GPW = C::GPW, GS = C::GS,
                PS = C::PS, K = C::K, NP = C::NP, CH = C::CH, CPR = MB * 4 / CH;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *zb = reinterpret_cast<float *>(smem_raw);              // [G][GS]
  float *vb = zb + C::G * GS;                                    // [G][PS]
  uint32_t *pb = reinterpret_cast<uint32_t *>(vb + C::G * PS);  // [G][PS]
  __shared__ double s_wt[NW * NP];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int c = lane % MB, gl = lane / MB, g = w * GPW + gl;
  const int64_t t = blockIdx.x;  // tiles are independent: no ticket, no waiting
  const int64_t tile = t / nseg;
  const int64_t kk = t - tile * nseg;  // segment = local coordinate
  const int64_t row0 = tile * R;
  const int64_t nrows = (n - row0 < R) ? (n - row0) : R;
  // L2 priorities: the sorted tables stream through (evict first); the Zt block and the Yt
  // accumulator are what must stay resident for the whole launch (evict last).
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  {
    const uint32_t *pp = perm + kk * ldn + row0;
    const float *vp = sval + kk * ldn + row0;
    for (int q = tid; q < R / 4; q += NT) {  // 4 consecutive rows, always inside one group
      const int r = 4 * q, dst = (r / ITEMS) * PS + (r % ITEMS);
      const bool ok = row0 + r < ldn;
      cp_async_hint<16>(pb + dst, ok ? (const void *)(pp + r) : (const void *)perm, ok, pol_stream);
      cp_async_hint<16>(vb + dst, ok ? (const void *)(vp + r) : (const void *)sval, ok, pol_stream);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    for (int e = tid; e < R * CPR; e += NT) {  // gather Zt rows into sorted order
      const int r = e / CPR, ch = e - (e / CPR) * CPR;
      const bool ok = r < nrows;
      const float *src =
          ok ? zt + (int64_t)pb[(r / ITEMS) * PS + (r % ITEMS)] * MB + ch * (CH / 4) : zt;
      cp_async_hint<CH>(zb + (r / ITEMS) * GS + (r % ITEMS) * MB + ch * (CH / 4), src, ok,
                        pol_keep);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  }
  const int rl0 = g * ITEMS;  // first row of this thread
  const int nmine = (int)(nrows - rl0 < ITEMS ? (nrows - rl0 < 0 ? 0 : nrows - rl0) : ITEMS);
  const float *zg = zb + g * GS + c;
  const float *vg = vb + g * PS;
  const uint32_t *pg = pb + g * PS;
  // ---- per-thread totals of the moments z v^t (fp64; for P = 1: s = z, t = v z, exact)
  double o[K];
#pragma unroll
  for (int q = 0; q < K; ++q) o[q] = 0.0;
#pragma unroll 4
  for (int j = 0; j < ITEMS; ++j) {
    const double z = (double)zg[j * MB];  // zero-filled past n
    const double v = j < nmine ? (double)vg[j] : 0.0;
    double zv = z;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      o[q] += zv;
      zv *= v;
    }
  }
  // ---- inclusive scan over the GPW groups of this warp (same column: lanes c + k*MB)
  double ps[K];
#pragma unroll
  for (int q = 0; q < K; ++q) ps[q] = o[q];
#pragma unroll
  for (int off = 1; off < GPW; off <<= 1) {
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const double a = __shfl_up_sync(0xFFFFFFFFu, ps[q], off * MB);
      if (gl >= off) ps[q] += a;
    }
  }
  if (gl == GPW - 1) {
#pragma unroll
    for (int q = 0; q < K; ++q) s_wt[w * NP + K * c + q] = ps[q];
  }
  __syncthreads();
  double *ag = agg + (kk * tiles_per_seg + tile) * agg_ld;  // tile totals (REDUCE: agg_ld = NP)
  if constexpr (MODE == SEQ_REDUCE) {
    if (tid < NP) {
      double run = 0.0;
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) run += s_wt[ww * NP + tid];
      ag[tid] = run;
    }
    return;
  } else {
    // exclusive prefix of this thread's first row: tile prefix + earlier warps + earlier groups
    double M[K];
#pragma unroll
    for (int q = 0; q < K; ++q) M[q] = __ldg(ag + K * c + q) + ps[q] - o[q];
    for (int ww = 0; ww < w; ++ww) {
#pragma unroll
      for (int q = 0; q < K; ++q) M[q] += s_wt[ww * NP + K * c + q];
    }
    double fxs = 0.0;  // SEQ_APPLY_FX: this column's fixed-point scale 2^F_c
    if constexpr (MODE == SEQ_APPLY_FX) fxs = c < mc ? __ldg(fx + c) : 0.0;
    double cT[K];  // P > 1: c_t T_t, the coordinate's totals of this column (prefix pass)
#pragma unroll
    for (int q = 0; q < K; ++q)
      cT[q] = (P > 1 && c < mc) ? lp_coef<P>(q) * __ldg(segtot + kk * ld_seg + K * c + q) : 0.0;
    if (c < mc) {
#pragma unroll 4
      for (int j = 0; j < ITEMS; ++j) {
        if (j >= nmine) break;
        const double z = (double)zg[j * MB], v = (double)vg[j];
        double val;
        if constexpr (P == 1) {
          val = 2.0 * fma(v, M[0], -M[1]);  // 2 U_r = 2 (v_r P_r - Q_r)
        } else {
          // sum_t c_t v^(P-t) (2 M_t - T_t) in Horner form over descending powers of v:
          // a_t = 2 c_t M_t - c_t T_t, val = (..(a_0 v + a_1) v + ..) v + a_P
          val = fma(2.0 * lp_coef<P>(0), M[0], -cT[0]);
#pragma unroll
          for (int q = 1; q < K; ++q) val = fma(val, v, fma(2.0 * lp_coef<P>(q), M[q], -cT[q]));
        }
        double zv = z;
#pragma unroll
        for (int q = 0; q < K; ++q) {
          M[q] += zv;
          zv *= v;
        }
        if constexpr (MODE == SEQ_APPLY_RED) {
          red_add_f64(out + (int64_t)pg[j] * ldo + c, val, pol_keep);
        } else if constexpr (MODE == SEQ_APPLY_FX) {
          const unsigned long long q = (unsigned long long)__double2ll_rn(val * fxs);
          asm volatile("red.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(
                           reinterpret_cast<unsigned long long *>(out) + (int64_t)pg[j] * ldo + c),
                       "l"(q), "l"(pol_keep)
                       : "memory");
        } else {
          __stcs(out + (kk * n + row0 + rl0 + j) * ldo + c, val);  // U[kk][r][c]
        }
      }
    }
  }
}

// Exclusive scan of each (segment, component) over the segment's tiles, in place (one warp per
// (segment, component)), and the segment totals for the epilogue.
__global__ void __launch_bounds__(256)
    k5_seq_prefix(double *__restrict__ agg, int64_t nseg, int64_t tiles_per_seg, int np,
                  int64_t ncomp, double *__restrict__ segtot, int64_t ld_seg) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (wid >= nseg * np) return;
  const int64_t seg = wid / np;
  const int comp = (int)(wid - seg * np);
  double *ag = agg + seg * tiles_per_seg * np + comp;
  double carry = 0.0;
  for (int64_t base = 0; base < tiles_per_seg; base += 32) {
    const int64_t j = base + lane;
    const double x = j < tiles_per_seg ? ag[j * np] : 0.0;
    double a = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double a2 = __shfl_up_sync(0xFFFFFFFFu, a, off);
      if (lane >= off) a += a2;
    }
    if (j < tiles_per_seg) ag[j * np] = carry + a - x;
    carry += __shfl_sync(0xFFFFFFFFu, a, 31);
  }
  if (lane == 0 && comp < ncomp) segtot[seg * ld_seg + comp] = carry;
}

template <int MB, int P>
static void launch_seq_t(const QueryPlan &p, const uint32_t *perm, const float *sval, int64_t ldn,
                         int64_t n, const float *zt, int64_t mc, double *out, int64_t ldo,
                         bool store, int64_t kcc, double *agg, int64_t agg_ld, double *segtot,
                         int64_t ld_seg, int phase, cudaStream_t s, const double *fx) {
  using C = SeqCfg<MB, P>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k5_scan_seq<MB, SEQ_REDUCE, P>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaFuncSetAttribute(k5_scan_seq<MB, SEQ_APPLY_RED, P>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaFuncSetAttribute(k5_scan_seq<MB, SEQ_APPLY_STORE, P>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (P == 1)
      cudaFuncSetAttribute(k5_scan_seq<MB, SEQ_APPLY_FX, P>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    attr = true;
  }
  const int64_t total = kcc * p.tiles_per_segment;
  if (phase != 1) {
    k5_scan_seq<MB, SEQ_REDUCE, P><<<(unsigned)total, C::NT, C::SMEM, s>>>(
        perm, sval, ldn, n, zt, mc, out, ldo, kcc, p.tiles_per_segment, agg, C::NP, segtot,
        ld_seg, nullptr);
    const int64_t warps = kcc * C::NP;
    k5_seq_prefix<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(agg, kcc, p.tiles_per_segment,
                                                              C::NP, C::K * mc, segtot, ld_seg);
  }
  if (phase != 0) {
    auto kern = store ? k5_scan_seq<MB, SEQ_APPLY_STORE, P>
                      : (P == 1 && fx) ? k5_scan_seq<MB, SEQ_APPLY_FX, P>
                                       : k5_scan_seq<MB, SEQ_APPLY_RED, P>;
    kern<<<(unsigned)total, C::NT, C::SMEM, s>>>(perm, sval, ldn, n, zt, mc, out, ldo, kcc,
                                                 p.tiles_per_segment, agg,
                                                 agg_ld > 0 ? agg_ld : C::NP, segtot, ld_seg, fx);
  }
}

void launch_scan_seq(const QueryPlan &p, int lp, const uint32_t *perm, const float *sval,
                     int64_t ldn, int64_t n, const float *zt, int64_t mc, double *out,
                     int64_t ldo, bool store, int64_t kcc, double *agg, double *segtot,
                     int64_t ld_seg, int phase, cudaStream_t s, int64_t agg_ld,
                     const double *fx) {
#define L1DM_SEQ(MB, P)                                                                         \
  launch_seq_t<MB, P>(p, perm, sval, ldn, n, zt, mc, out, ldo, store, kcc, agg, agg_ld, segtot, \
                      ld_seg, phase, s, fx)
#define L1DM_SEQ_P(MB)                         \
  switch (lp) {                                \
    case 1: L1DM_SEQ(MB, 1); break;            \
    case 3: L1DM_SEQ(MB, 3); break;            \
    case 5: L1DM_SEQ(MB, 5); break;            \
    case 7: L1DM_SEQ(MB, 7); break;            \
    default: break;                            \
  }
  switch (p.mb) {
    case 2: L1DM_SEQ_P(2); break;
    case 4: L1DM_SEQ_P(4); break;
    case 8: L1DM_SEQ_P(8); break;
    case 16: L1DM_SEQ_P(16); break;
    default: break;
  }
#undef L1DM_SEQ_P
#undef L1DM_SEQ
}

// Look-back status word of k5_scan_lb: [63:4] the 60-bit signed fixed-point value, [3:2] the
// launch's epoch mod 4, [1:0] the flag (0 = not published).  One 8-byte access: a reader sees a
// value with its own tag.  Every launch rewrites every word of its geometry (and the words are
// zeroed when the geometry changes), so a stale word is from the previous launch: two epoch
// bits tell them apart with margin.
__device__ __forceinline__ unsigned long long lb_word(long long v, uint32_t ep, uint32_t flag) {
  return ((unsigned long long)v << 4) | (unsigned long long)((ep << 2) | flag);
}

// Single-pass scatter apply (P = 1, fixed-point Yt): the tile's exclusive prefixes of s = z and
// t = v z come from a decoupled look-back (Merrill & Garland) over the earlier tiles of its
// segment instead of a separate tile-totals pass over Z — the Zt rows the apply gathers anyway
// give the tile aggregates.  The look-back runs in 64-bit fixed point (per column, 2^Fz for the
// s sums, 2^Fv for the t sums; launch_fx_scale), so the prefix a tile receives is the exact
// integer sum of its predecessors' rounded aggregates whichever of them it walks over: Y stays
// bitwise reproducible (R16).  Each status word is 8 bytes {value, epoch, flag}
// (lb_word; no separate flag, no fences; epochs count this kernel's launches per handle, and
// the words are zeroed whenever the slot geometry changes).  Warp 0's lanes
// 0..2MB-1 each walk back one component, kLBW predecessors per round trip: first while the
// tile's Z gathers are in flight (non-blocking: it stops at the first unpublished predecessor),
// then, once the tile's own aggregate is known, it publishes INCLUSIVE directly when the walk
// finished (the common case) or AGGREGATE and waits.  Tile order is blockIdx order with the
// segments interleaved (CTAs are dispatched in increasing blockIdx, so every tile a CTA waits
// for is resident or done — the single-pass scan's usual forward-progress argument); waits are
// bounded by kSpinLimit (then *timeout_flag is raised).
//
// P > 1 (odd l_p^p): K = P + 1 moments z v^t per column, all prefixed by the same
// look-back (K mb components, one lane each), and each row adds only the prefix part of its term,
// 2 sum_t c_t v^(P-t) M_t, into a fp64 block accumulator (fp64 reductions, yt points at doubles):
// the coordinate totals' part, sum_k sum_t c_t x_ik^(P-t) T_kt, is one DMMA expansion after the
// last block (launch_lp_totals_expand), so no pass has to know the totals before the apply.
template <int MB, int NTT, int P>
__global__ void __launch_bounds__(NTT, (P <= 3 ? 1280 : 768) / NTT)  // 5 (3 for P >= 5) x 256 thr/SM
    k5_scan_lb(const uint32_t *__restrict__ perm, const float *__restrict__ sval, int64_t ldn,
               int64_t n, const float *__restrict__ zt, int64_t mc, unsigned long long *__restrict__ yt,
               int64_t nseg, int64_t tiles_per_seg, unsigned long long *__restrict__ lbst,
               uint32_t epoch,
               unsigned *timeout_flag, const double *__restrict__ fx,
               const double *__restrict__ fa, int64_t fa_ld, double *__restrict__ segtot,
               int64_t ld_seg) {
  using C = SeqCfg<MB, P, NTT, L1DM_LB_ITEMS>;
  constexpr int NT = C::NT, NW = C::NW, ITEMS = C::ITEMS, R = C::R, GPW = C::GPW, GS = C::GS,
                PS = C::PS, NP = C::NP, CH = C::CH, CPR = MB * 4 / CH, K = P + 1;
  constexpr int kLBW = 4;  // predecessors loaded per look-back round trip
  static_assert(NP <= 64 && NT >= 64, "one look-back lane per component (warps 0 and 1)");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *zb = reinterpret_cast<float *>(smem_raw);              // [G][GS]
  float *vb = zb + C::G * GS;                                    // [G][PS]
  uint32_t *pb = reinterpret_cast<uint32_t *>(vb + C::G * PS);  // [G][PS]
  __shared__ double s_wt[NW * NP];
  __shared__ double s_excl[NP];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int c = lane % MB, gl = lane / MB, g = w * GPW + gl;
  const int64_t t = blockIdx.x;
  const int64_t tile = t / nseg;
  const int64_t kk = t - tile * nseg;
  const int64_t row0 = tile * R;
  const int64_t nrows = (n - row0 < R) ? (n - row0) : R;
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  {
    const uint32_t *pp = perm + kk * ldn + row0;
    const float *vp = sval + kk * ldn + row0;
    for (int q = tid; q < R / 4; q += NT) {
      const int r = 4 * q, dst = (r / ITEMS) * PS + (r % ITEMS);
      const bool ok = row0 + r < ldn;
      cp_async_hint<16>(pb + dst, ok ? (const void *)(pp + r) : (const void *)perm, ok, pol_stream);
      cp_async_hint<16>(vb + dst, ok ? (const void *)(vp + r) : (const void *)sval, ok, pol_stream);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    for (int e = tid; e < R * CPR; e += NT) {  // gather Zt rows into sorted order
      const int r = e / CPR, ch = e - (e / CPR) * CPR;
      const bool ok = r < nrows;
      const float *src =
          ok ? zt + (int64_t)pb[(r / ITEMS) * PS + (r % ITEMS)] * MB + ch * (CH / 4) : zt;
      cp_async_hint<CH>(zb + (r / ITEMS) * GS + (r % ITEMS) * MB + ch * (CH / 4), src, ok,
                        pol_keep);
    }
    cp_async_commit();
  }
  // ---- look-back, first part (overlaps the gathers): component e = 2 cc + q of this lane
  const int e = NP <= 32 ? lane : 32 * w + lane, cc = e / K, q = e - (e / K) * K;
  const bool lb_lane = NP <= 32 ? (w == 0 && lane < NP) : (w < 2 && e < NP);
  unsigned long long *st = lbst + (kk * tiles_per_seg) * NP + e;
  const uint32_t ep2 = epoch & 3u;
  const uint64_t pol_lb = pol_stream;  // status words are read back within a few tiles
  long long excl = 0;
  int64_t j = tile - 1;  // nearest predecessor not summed yet
  bool done = tile == 0;
  // one round trip: sum the published predecessors in the window; returns whether any was
  auto walk = [&]() {
    unsigned long long sv[kLBW];
#pragma unroll
    for (int u = 0; u < kLBW; ++u)
      sv[u] = (j - u >= 0) ? ld_relaxed_u64_hint(st + (j - u) * NP, pol_lb)
                           : lb_word(0, ep2, kFlagInclusive);
    int u = 0;
    for (; u < kLBW; ++u) {
      const uint32_t tg = (uint32_t)sv[u] & 0xFu;
      if ((tg >> 2) != ep2 || (tg & 3u) == kFlagInvalid) break;
      excl += (long long)sv[u] >> 4;  // the 60-bit signed value
      if ((tg & 3u) == kFlagInclusive) {
        done = true;
        return true;
      }
    }
    j -= u;
    return u > 0;
  };
  if (lb_lane)
    while (!done && walk()) {
    }
  cp_async_wait_all();
  __syncthreads();
  const int rl0 = g * ITEMS;
  const int nmine = (int)(nrows - rl0 < ITEMS ? (nrows - rl0 < 0 ? 0 : nrows - rl0) : ITEMS);
  const float *zg = zb + g * GS + c;
  const float *vg = vb + g * PS;
  const uint32_t *pg = pb + g * PS;
  double o[K];  // this thread's totals of the moments z v^t (P = 1: s = z, t = v z; fp64, fixed order)
#pragma unroll
  for (int q = 0; q < K; ++q) o[q] = 0.0;
#pragma unroll 4
  for (int jj = 0; jj < ITEMS; ++jj) {
    const double z = (double)zg[jj * MB];  // zero-filled past n
    const double v = jj < nmine ? (double)vg[jj] : 0.0;
    double zv = z;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      o[q] += zv;  // (q = 1: z v is exact in fp64, so this equals fma(v, z, o))
      zv *= v;
    }
  }
  double ps[K];
#pragma unroll
  for (int q = 0; q < K; ++q) ps[q] = o[q];
#pragma unroll
  for (int off = 1; off < GPW; off <<= 1) {
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const double a = __shfl_up_sync(0xFFFFFFFFu, ps[q], off * MB);
      if (gl >= off) ps[q] += a;
    }
  }
  if (gl == GPW - 1) {
#pragma unroll
    for (int q = 0; q < K; ++q) s_wt[w * NP + K * c + q] = ps[q];
  }
  __syncthreads();
  if (lb_lane) {
    // the tile aggregate of component e (warps in order) in fixed point
    double a = 0.0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) a += s_wt[ww * NP + e];
    const bool live = cc < mc;
    const double sc = live ? __ldg(fa + (2 * q) * fa_ld + cc) : 0.0;
    const double isc = live ? __ldg(fa + (2 * q + 1) * fa_ld + cc) : 0.0;
    const long long qa = __double2ll_rn(a * sc);
    if (!done) {
      st_relaxed_u64_hint(st + tile * NP, lb_word(qa, ep2, kFlagAggregate), pol_lb);
      uint32_t spins = 0;
      while (!done) {
        if (walk()) continue;
        if (++spins > kSpinLimit) {
          atomicOr(timeout_flag, 1u);
          break;
        }
        if (spins > 16) __nanosleep(32);
      }
    }
    st_relaxed_u64_hint(st + tile * NP, lb_word(excl + qa, ep2, kFlagInclusive), pol_lb);
    s_excl[e] = (double)excl * isc;
    if (tile == tiles_per_seg - 1 && live) segtot[kk * ld_seg + e] = (double)(excl + qa) * isc;
  }
  __syncthreads();
  // exclusive prefix of this thread's first row: tile prefix + earlier warps + earlier groups
  double M[K];
#pragma unroll
  for (int q2 = 0; q2 < K; ++q2) M[q2] = s_excl[K * c + q2] + ps[q2] - o[q2];
  for (int ww = 0; ww < w; ++ww) {
#pragma unroll
    for (int q2 = 0; q2 < K; ++q2) M[q2] += s_wt[ww * NP + K * c + q2];
  }
  if (c < mc) {
    double fxs2 = 0.0;  // P = 1: 2 2^F_c (the factor 2 of 2U folded into the exact scaling)
    if constexpr (P == 1) fxs2 = 2.0 * __ldg(fx + c);
#pragma unroll 4
    for (int jj = 0; jj < ITEMS; ++jj) {
      if (jj >= nmine) break;
      const double z = (double)zg[jj * MB], v = (double)vg[jj];
      if constexpr (P == 1) {
        const double u = fma(v, M[0], -M[1]);  // U_r = v_r P_r - Q_r; adds 2 U_r
        M[0] += z;
        M[1] = fma(v, z, M[1]);
        const unsigned long long qv = (unsigned long long)__double2ll_rn(u * fxs2);
        asm volatile("red.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(
                         yt + (int64_t)pg[jj] * MB + c),
                     "l"(qv), "l"(pol_keep)
                     : "memory");
      } else {
        // 2 sum_t c_t v^(P-t) M_t in Horner form over descending powers of v
        double val = 2.0 * lp_coef<P>(0) * M[0];
#pragma unroll
        for (int q2 = 1; q2 < K; ++q2) val = fma(val, v, 2.0 * lp_coef<P>(q2) * M[q2]);
        double zv = z;
#pragma unroll
        for (int q2 = 0; q2 < K; ++q2) {
          M[q2] += zv;
          zv *= v;
        }
        red_add_f64(reinterpret_cast<double *>(yt) + (int64_t)pg[jj] * MB + c, val, pol_keep);
      }
    }
  }
}

// threads per k5_scan_lb CTA: 128 (512-row tiles) for mb >= 2, 256 (2048-row tiles) for mb = 1,
// or L1DM_LB_NT (tuning override, 128 or 256)
static int scan_lb_threads(int mb) {
  static const int env = [] {
    const char *e = getenv("L1DM_LB_NT");
    return e ? atoi(e) : 0;
  }();
  if (env == 128 || env == 256) return env;
  return mb == 1 ? 256 : 128;
}

int scan_lb_rows(int mb) { return scan_lb_threads(mb) * (mb == 1 ? 8 : L1DM_LB_ITEMS); }

void launch_scan_lb(int mb, const uint32_t *perm, const float *sval, int64_t ldn, int64_t n,
                    const float *zt, int64_t mc, unsigned long long *yt, int64_t kcc,
                    void *lbst, uint32_t epoch,
                    unsigned *timeout_flag, const double *fx, const double *fa, int64_t fa_ld,
                    double *segtot, int64_t ld_seg, cudaStream_t s, int lp) {
  const int nt = scan_lb_threads(mb);
  const int64_t tiles_per_seg = (n + scan_lb_rows(mb) - 1) / scan_lb_rows(mb);
  const int64_t total = kcc * tiles_per_seg;
#define L1DM_LB(MB, NTT, P)                                                                    \
  {                                                                                            \
    using C = SeqCfg<MB, P, NTT, L1DM_LB_ITEMS>;                                               \
    static bool attr = false;                                                                  \
    if (!attr) {                                                                               \
      cudaFuncSetAttribute(k5_scan_lb<MB, NTT, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,\
                           (int)C::SMEM);                                                      \
      attr = true;                                                                             \
    }                                                                                          \
    k5_scan_lb<MB, NTT, P><<<(unsigned)total, C::NT, C::SMEM, s>>>(                            \
        perm, sval, ldn, n, zt, mc, yt, kcc, tiles_per_seg,                                    \
        static_cast<unsigned long long *>(lbst), epoch, timeout_flag, fx, fa, fa_ld, segtot,   \
        ld_seg);                                                                               \
  }
#define L1DM_LB_NT(NTT)                                                      \
  if (lp == 1) {                                                             \
    switch (mb) {                                                            \
      case 1: L1DM_LB(1, NTT, 1) break;                                      \
      case 2: L1DM_LB(2, NTT, 1) break;                                      \
      case 4: L1DM_LB(4, NTT, 1) break;                                      \
      case 8: L1DM_LB(8, NTT, 1) break;                                      \
      case 16: L1DM_LB(16, NTT, 1) break;                                    \
      default: break;                                                        \
    }                                                                        \
  } else if (lp == 3) {                                                      \
    switch (mb) {                                                            \
      case 2: L1DM_LB(2, NTT, 3) break;                                      \
      case 4: L1DM_LB(4, NTT, 3) break;                                      \
      case 8: L1DM_LB(8, NTT, 3) break;                                      \
      case 16: L1DM_LB(16, NTT, 3) break;                                    \
      default: break;                                                        \
    }                                                                        \
  } else if (lp == 5) {                                                      \
    switch (mb) {                                                            \
      case 2: L1DM_LB(2, NTT, 5) break;                                      \
      case 4: L1DM_LB(4, NTT, 5) break;                                      \
      case 8: L1DM_LB(8, NTT, 5) break;                                      \
      default: break;                                                        \
    }                                                                        \
  } else if (lp == 7) {                                                      \
    switch (mb) {                                                            \
      case 2: L1DM_LB(2, NTT, 7) break;                                      \
      case 4: L1DM_LB(4, NTT, 7) break;                                      \
      case 8: L1DM_LB(8, NTT, 7) break;                                      \
      default: break;                                                        \
    }                                                                        \
  }
  if (nt == 256) {
    L1DM_LB_NT(256)
  } else {
    L1DM_LB_NT(128)
  }
#undef L1DM_LB_NT
#undef L1DM_LB
}

// Whether launch_scan_lb has a kernel for (mb, lp): one look-back lane per component in warps 0
// and 1, (lp + 1) mb <= 64.
bool scan_lb_supported(int mb, int lp) {
  if (lp == 1 || lp == 3) return mb == 1 || mb == 2 || mb == 4 || mb == 8 || mb == 16;
  if (lp == 5 || lp == 7) return mb == 2 || mb == 4 || mb == 8;
  return false;
}

// Tile totals of every column at once for the P = 1 scatter scan (one pass over the sorted
// tables and the full Z rows, instead of one reduce pass per column block): per (segment,
// 1024-row tile) and column c, (sum z, sum v z) -> agg[seg][tile][2c + {0,1}], the same layout
// the per-block reduce writes with NP = 2m.  Each warp sums 128 consecutive sorted rows: the
// row's perm/sval are warp-uniform loads, the Z row (m floats) is read with lanes over columns
// (coalesced), so the gathers are whole Z rows from HBM (c3: 256 B) — the efficient width.
template <int NCL>
__global__ void __launch_bounds__(256)
    k5_reduce_all(const uint32_t *__restrict__ perm, const float *__restrict__ sval, int64_t ldn,
                  int64_t n, const float *__restrict__ Z, int64_t ldz, int64_t m, int64_t nseg,
                  int64_t tiles_per_seg, double *__restrict__ agg) {
  // a CTA covers two consecutive 1024-row tiles (warps 0-3 the first, 4-7 the second): half as
  // many CTAs, twice the rows per warp (measured: 6.9 -> 6.4 ms at c3), per-tile outputs as before
  constexpr int R = 1024, NW = 8, TPC = L1DM_RA_TILES, RW = TPC * R / NW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *s_part = reinterpret_cast<double *>(smem_raw);  // [NW][2m]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t = blockIdx.x;
  const int64_t pair = t / nseg;  // (group of TPC tiles)
  const int64_t kk = t - pair * nseg;
  const int64_t r0 = pair * TPC * R + (int64_t)w * RW;
  const int64_t r1 = (r0 + RW < n) ? r0 + RW : n;
  const uint32_t *pp = perm + kk * ldn;
  const float *vp = sval + kk * ldn;
  double cs[NCL], ct[NCL];
#pragma unroll
  for (int j = 0; j < NCL; ++j) {
    cs[j] = 0.0;
    ct[j] = 0.0;
  }
  int64_t r = r0;
  for (; r + 4 <= r1; r += 4) {  // 4 rows in flight per warp
    uint32_t pr[4];
    float vr[4], zr[4][NCL];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      pr[u] = __ldg(pp + r + u);
      vr[u] = __ldg(vp + r + u);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < NCL; ++j) {
        const int64_t c = lane + 32 * j;
        zr[u][j] = (c < m) ? __ldg(Z + (int64_t)pr[u] * ldz + c) : 0.0f;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < NCL; ++j) {
        const double z = (double)zr[u][j];
        cs[j] += z;
        ct[j] = fma((double)vr[u], z, ct[j]);
      }
  }
  for (; r < r1; ++r) {
    const uint32_t pr = __ldg(pp + r);
    const double v = (double)__ldg(vp + r);
#pragma unroll
    for (int j = 0; j < NCL; ++j) {
      const int64_t c = lane + 32 * j;
      const double z = (c < m) ? (double)__ldg(Z + (int64_t)pr * ldz + c) : 0.0;
      cs[j] += z;
      ct[j] = fma(v, z, ct[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < NCL; ++j) {
    const int64_t c = lane + 32 * j;
    if (c < m) {
      s_part[w * 2 * m + 2 * c] = cs[j];
      s_part[w * 2 * m + 2 * c + 1] = ct[j];
    }
  }
  __syncthreads();
  for (int half = 0; half < TPC; ++half) {
    const int64_t tile = TPC * pair + half;
    if (tile >= tiles_per_seg) break;
    double *ag = agg + (kk * tiles_per_seg + tile) * 2 * m;
    for (int64_t e = threadIdx.x; e < 2 * m; e += 256) {
      double a = 0.0;
#pragma unroll
      for (int ww = 0; ww < NW / TPC; ++ww) a += s_part[(half * NW / TPC + ww) * 2 * m + e];
      ag[e] = a;
    }
  }
}

bool launch_reduce_all(const uint32_t *perm, const float *sval, int64_t ldn, int64_t n,
                       const float *Z, int64_t ldz, int64_t m, int64_t kcc, int64_t tiles_per_seg,
                       double *agg, double *segtot, cudaStream_t s) {
  if (m > 256) return false;
  const int64_t total = kcc * ((tiles_per_seg + L1DM_RA_TILES - 1) / L1DM_RA_TILES);
  const size_t smem = (size_t)8 * 2 * m * sizeof(double);
#define L1DM_RA(NCL)                                                                            \
  {                                                                                             \
    static bool attr = false;                                                                   \
    if (!attr) {                                                                                \
      cudaFuncSetAttribute(k5_reduce_all<NCL>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                           32768);                                                              \
      attr = true;                                                                              \
    }                                                                                           \
    k5_reduce_all<NCL><<<(unsigned)total, 256, smem, s>>>(perm, sval, ldn, n, Z, ldz, m, kcc,   \
                                                          tiles_per_seg, agg);                  \
  }
  if (m <= 32) L1DM_RA(1)
  else if (m <= 64) L1DM_RA(2)
  else if (m <= 128) L1DM_RA(4)
  else L1DM_RA(8)
#undef L1DM_RA
  const int64_t warps = kcc * 2 * m;
  k5_seq_prefix<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(agg, kcc, tiles_per_seg, (int)(2 * m),
                                                            2 * m, segtot, 2 * m);
  return true;
}

// Single-column variant (m == 1).  Here a tile is cheap (4 B of Z per row, gathered from
// L2) and the decoupled look-back's latency dominates, so the scan is done as
// reduce-then-scan with no inter-CTA waits at all:
//   M1_REDUCE  per tile: (sum z, sum v z)                         -> m1agg[seg][tile]
//   k5_m1_prefix  per segment: exclusive scan over its tiles       -> m1agg (in place), segtot
//   M1_APPLY   per tile: U along the rows from the tile's prefix, stored (sorted order)
//              or, in scatter mode, added as 2U into Y[perm[r]] with L2 atomics.
// Each thread owns ITEMS *consecutive* sorted rows (thread-sequential scan, one warp scan per
// tile); shared-memory rows are padded (4 floats every 32) so its 128-bit reads are
// bank-conflict free.
constexpr int kM1Items = L1DM_M1_ROW_ITEMS;
constexpr int kM1Rows = 256 * kM1Items;  // rows per tile
__device__ __forceinline__ int m1_pad(int r) { return r + (r >> 5) * 4; }

enum { M1_REDUCE = 0, M1_APPLY_STORE = 1, M1_APPLY_SCATTER = 2 };

template <int MODE>
__global__ void __launch_bounds__(256, L1DM_M1_MINB)
    k5_scan_m1(const uint32_t *__restrict__ perm, const float *__restrict__ sval, int64_t ldn,
               int64_t n, const float *__restrict__ Z, int64_t ldz, double *__restrict__ U,
               int64_t ldu, int64_t k_first, int64_t nseg, int64_t tiles_per_seg,
               double *__restrict__ m1agg, float *__restrict__ zs) {
  constexpr int ITEMS = kM1Items, R = kM1Rows, NW = 8;
  constexpr int RP = R + R / 8;  // padded length
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *zb = reinterpret_cast<float *>(smem_raw);     // [RP]
  float *vb = zb + RP;                                  // [RP]
  uint32_t *pb = reinterpret_cast<uint32_t *>(vb + RP);  // [RP]
  __shared__ double s_w[NW][2];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t t = blockIdx.x;  // tiles are independent: no ticket, no waiting
  const int64_t tile = t / nseg;
  const int64_t seg = t - tile * nseg;  // local coordinate
  const int64_t row0 = tile * R;
  const int64_t nrows = (n - row0 < R) ? (n - row0) : R;
  float *zsp = zs + seg * ldn + row0;  // z in sorted order, written by the reduce pass
  {
    const uint32_t *pp = perm + (k_first + seg) * ldn + row0;
    const float *vp = sval + (k_first + seg) * ldn + row0;
    for (int c = tid; c < R / 4; c += 256) {
      const bool ok = row0 + 4 * c < ldn;
      if (MODE == M1_REDUCE || MODE == M1_APPLY_SCATTER)
        cp_async<16>(pb + m1_pad(4 * c), ok ? (const void *)(pp + 4 * c) : (const void *)perm, ok);
      cp_async<16>(vb + m1_pad(4 * c), ok ? (const void *)(vp + 4 * c) : (const void *)sval, ok);
      if (MODE != M1_REDUCE)  // the apply pass streams z back in sorted order: no second gather
        cp_async<16>(zb + m1_pad(4 * c), ok ? (const void *)(zsp + 4 * c) : (const void *)zs, ok);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    if constexpr (MODE == M1_REDUCE) {
      for (int r = tid; r < R; r += 256) {  // gather z into sorted order
        const bool ok = r < nrows;
        cp_async<4>(zb + m1_pad(r), ok ? (const void *)(Z + (int64_t)pb[m1_pad(r)] * ldz) : Z, ok);
      }
      cp_async_commit();
      cp_async_wait_all();
      __syncthreads();
      for (int c = tid; c < R / 4; c += 256)  // keep it for the apply pass (coalesced)
        if (row0 + 4 * c < ldn)
          __stcg(reinterpret_cast<float4 *>(zsp + 4 * c),
                 *reinterpret_cast<const float4 *>(zb + m1_pad(4 * c)));
    }
  }
  const int rl0 = tid * ITEMS;  // this thread's first row
  const int b0 = m1_pad(rl0);   // padded start (16 rows never straddle a 32-row group)
  const int nmine = (int)(nrows - rl0 < ITEMS ? (nrows - rl0 < 0 ? 0 : nrows - rl0) : ITEMS);
  double os = 0.0, ot = 0.0;
#pragma unroll
  for (int q = 0; q < ITEMS / 4; ++q) {
    const float4 a = *reinterpret_cast<const float4 *>(zb + b0 + 4 * q);
    const float4 b = *reinterpret_cast<const float4 *>(vb + b0 + 4 * q);
    const float zz[4] = {a.x, a.y, a.z, a.w}, vv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // padding rows: z is zero-filled
      os += (double)zz[u];
      ot = fma(4 * q + u < nmine ? (double)vv[u] : 0.0, (double)zz[u], ot);
    }
  }
  double ps = os, pt = ot;  // warp inclusive scan of the thread totals
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double a = __shfl_up_sync(0xFFFFFFFFu, ps, off);
    const double b = __shfl_up_sync(0xFFFFFFFFu, pt, off);
    if (lane >= off) {
      ps += a;
      pt += b;
    }
  }
  if (lane == 31) {
    s_w[w][0] = ps;
    s_w[w][1] = pt;
  }
  __syncthreads();
  double *ag = m1agg + (seg * tiles_per_seg + tile) * 2;
  if constexpr (MODE == M1_REDUCE) {
    if (tid < 2) {
      double run = 0.0;
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) run += s_w[ww][tid];
      ag[tid] = run;
    }
    return;
  } else {
    // exclusive prefix of this thread's first row: tile prefix + earlier warps + earlier lanes
    double P = __ldg(ag) + ps - os, Q = __ldg(ag + 1) + pt - ot;
    for (int ww = 0; ww < w; ++ww) {
      P += s_w[ww][0];
      Q += s_w[ww][1];
    }
    double *up = U + seg * n * ldu + (row0 + rl0) * ldu;  // store mode: this thread's U rows
#pragma unroll
    for (int q = 0; q < ITEMS / 4; ++q) {
      const float4 a = *reinterpret_cast<const float4 *>(zb + b0 + 4 * q);
      const float4 b = *reinterpret_cast<const float4 *>(vb + b0 + 4 * q);
      const uint4 c = *reinterpret_cast<const uint4 *>(pb + b0 + 4 * q);
      const float zz[4] = {a.x, a.y, a.z, a.w}, vv[4] = {b.x, b.y, b.z, b.w};
      const uint32_t pr[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = 4 * q + u;
        const double vj = j < nmine ? (double)vv[u] : 0.0, sz = (double)zz[u];
        const double uu = fma(vj, P, -Q);  // U_r = v_r P_r - Q_r
        P += sz;
        Q = fma(vj, sz, Q);
        if (j < nmine) {
          if constexpr (MODE == M1_APPLY_SCATTER) {
            atomicAdd(U + (int64_t)pr[u] * ldu, 2.0 * uu);
          } else {
            __stcs(up + (int64_t)j * ldu, uu);
          }
        }
      }
    }
  }
}

// Exclusive scan of each segment's tile aggregates (one warp per segment, in place), and the
// segment totals for the epilogue.
__global__ void __launch_bounds__(256)
    k5_m1_prefix(double *__restrict__ m1agg, int64_t nseg, int64_t tiles_per_seg, int64_t k_first,
                 double *__restrict__ segtot) {
  const int lane = threadIdx.x & 31;
  const int64_t seg = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (seg >= nseg) return;
  double *ag = m1agg + seg * tiles_per_seg * 2;
  double cs = 0.0, ct = 0.0;
  for (int64_t base = 0; base < tiles_per_seg; base += 32) {
    const int64_t j = base + lane;
    const double s = j < tiles_per_seg ? ag[2 * j] : 0.0;
    const double t = j < tiles_per_seg ? ag[2 * j + 1] : 0.0;
    double a = s, b = t;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double a2 = __shfl_up_sync(0xFFFFFFFFu, a, off);
      const double b2 = __shfl_up_sync(0xFFFFFFFFu, b, off);
      if (lane >= off) {
        a += a2;
        b += b2;
      }
    }
    if (j < tiles_per_seg) {
      ag[2 * j] = cs + a - s;
      ag[2 * j + 1] = ct + b - t;
    }
    cs += __shfl_sync(0xFFFFFFFFu, a, 31);
    ct += __shfl_sync(0xFFFFFFFFu, b, 31);
  }
  if (lane == 0) {
    segtot[(k_first + seg) * 2] = cs;
    segtot[(k_first + seg) * 2 + 1] = ct;
  }
}

template <int LPR, int VC, int CH>
static void launch_scan_t(const QueryPlan &p, const uint32_t *perm, const float *sval,
                          int64_t ldn, int64_t n, const float *Z, int64_t ldz, int64_t m,
                          double *U, int64_t k_first, int64_t kcc, uint32_t *flags, double *agg,
                          double *incl, uint32_t epoch, unsigned *ticket, unsigned *timeout_flag,
                          double *segtot, int64_t ld_seg, cudaStream_t s) {
  using C = ScanCfg<LPR, VC, scan_items(LPR, VC)>;
  auto kern = k5_scan<LPR, VC, CH>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k5_scan<LPR, VC, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM);
    attr = true;
  }
  const int64_t nseg = kcc * p.col_blocks;
  const int64_t total = nseg * p.tiles_per_segment;
  kern<<<(unsigned)total, C::NT, C::SMEM, s>>>(perm, sval, ldn, n, Z, ldz, m, U, p.ldu, k_first,
                                               p.col_blocks, nseg, total, flags, agg, incl, epoch,
                                               ticket, timeout_flag, p.tiles_per_segment, segtot,
                                               ld_seg);
}

void launch_scan(const QueryPlan &p, const uint32_t *perm, const float *sval, int64_t ldn,
                 int64_t n, const float *Z, int64_t ldz, int64_t m, double *U, int64_t k_first,
                 int64_t kcc, uint32_t *flags, double *agg, double *incl, uint32_t epoch,
                 unsigned *ticket, unsigned *timeout_flag, double *segtot, int64_t ld_seg,
                 float *zs, cudaStream_t s) {
#define L1DM_SCAN(L, V, CH)                                                                    \
  launch_scan_t<L, V, CH>(p, perm, sval, ldn, n, Z, ldz, m, U, k_first, kcc, flags,              \
                          agg, incl, epoch, ticket, timeout_flag, segtot, ld_seg, s)
  // p.lpr lanes per row, p.mb / p.lpr columns per lane, p.vec floats per cp.async chunk
  if (p.mb == 1) {
    // reduce-then-scan, no look-back (the agg workspace holds 2 doubles per tile)
    const size_t smem = (size_t)(kM1Rows + kM1Rows / 8) * 4 * 3;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k5_scan_m1<M1_REDUCE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      cudaFuncSetAttribute(k5_scan_m1<M1_APPLY_STORE>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k5_scan_m1<M1_APPLY_SCATTER>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    const int64_t nseg = kcc;
    const int64_t total = nseg * p.tiles_per_segment;
    k5_scan_m1<M1_REDUCE><<<(unsigned)total, 256, smem, s>>>(
        perm, sval, ldn, n, Z, ldz, U, p.ldu, k_first, nseg, p.tiles_per_segment, agg, zs);
    k5_m1_prefix<<<(unsigned)((nseg + 7) / 8), 256, 0, s>>>(agg, nseg, p.tiles_per_segment,
                                                             k_first, segtot);
    auto kern = p.scatter ? k5_scan_m1<M1_APPLY_SCATTER> : k5_scan_m1<M1_APPLY_STORE>;
    kern<<<(unsigned)total, 256, smem, s>>>(perm, sval, ldn, n, Z, ldz, U, p.ldu, k_first, nseg,
                                            p.tiles_per_segment, agg, zs);
    (void)flags;
    (void)incl;
    (void)epoch;
    (void)ticket;
    (void)timeout_flag;
    return;
  }
  const int vc = p.mb / p.lpr;
  switch (vc * 10000 + p.vec * 100 + p.lpr) {
    case 10101: L1DM_SCAN(1, 1, 4); break;
    case 10102: L1DM_SCAN(2, 1, 4); break;
    case 10104: L1DM_SCAN(4, 1, 4); break;
    case 10108: L1DM_SCAN(8, 1, 4); break;
    case 10116: L1DM_SCAN(16, 1, 4); break;
    case 10132: L1DM_SCAN(32, 1, 4); break;
    case 10202: L1DM_SCAN(2, 1, 8); break;
    case 10204: L1DM_SCAN(4, 1, 8); break;
    case 10208: L1DM_SCAN(8, 1, 8); break;
    case 10216: L1DM_SCAN(16, 1, 8); break;
    case 10232: L1DM_SCAN(32, 1, 8); break;
    case 10404: L1DM_SCAN(4, 1, 16); break;
    case 10408: L1DM_SCAN(8, 1, 16); break;
    case 10416: L1DM_SCAN(16, 1, 16); break;
    case 10432: L1DM_SCAN(32, 1, 16); break;
    case 20232: L1DM_SCAN(32, 2, 8); break;
    case 20432: L1DM_SCAN(32, 2, 16); break;
    default: break;
  }
#undef L1DM_SCAN
}

// ------------------------------------------------------------------ scatter-mode epilogue
// Y[i][c] += g_c - h_i S_c after the scatter scans (Y was zeroed before them).
__global__ void __launch_bounds__(256)
    k7_epilogue(const double *__restrict__ hsum, const double *__restrict__ Sg,
                double *__restrict__ Y, int64_t ldy, int64_t i0, int64_t i1, int64_t m) {
  const int64_t total = (i1 - i0) * m;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    const int64_t i = i0 + e / m, c = e - (e / m) * m;
    Y[i * ldy + c] += fma(-hsum[i], Sg[c], Sg[m + c]);
  }
}

void launch_epilogue(const double *hsum, const double *Sg, double *Y, int64_t ldy, int64_t i0,
                     int64_t i1, int64_t m, cudaStream_t s) {
  if (i1 <= i0) return;
  int64_t blocks = ((i1 - i0) * m + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k7_epilogue<<<(unsigned)blocks, 256, 0, s>>>(hsum, Sg, Y, ldy, i0, i1, m);
}

// Scatter mode, m > 1: Y[i][c0 + c] = Yt[i][c] + g_c - h_i S_c for one column block (Yt is the
// block's compact L2-resident accumulator, mb doubles per point).  S == nullptr (l_p, p > 1:
// the apply pass already added the whole contribution): Y[i][c0 + c] = Yt[i][c].
// PUSH: the row goes to its owner's inbox slot (peer memory over NVLink) at
// column pc0 + c — the block's output pass is the collective's send.
template <bool PUSH>
__global__ void __launch_bounds__(256)
    k9_block_out(const double *__restrict__ yt, int mb, int64_t mc, const double *__restrict__ hsum,
                 const double *__restrict__ S, const double *__restrict__ g, double *__restrict__ Y,
                 int64_t ldy, int64_t i0, int64_t i1, PeerDst pd, int64_t pc0,
                 const double *__restrict__ fx) {
  const int64_t total = (i1 - i0) * mc;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    const int64_t i = i0 + e / mc, c = e - (e / mc) * mc;
    // fixed-point Yt (SEQ_APPLY_FX): fx = the block's inverse scales 2^-F_c
    const double v = fx ? (double)reinterpret_cast<const long long *>(yt)[i * mb + c] * __ldg(fx + c)
                        : yt[i * mb + c];
    const double out = S ? v + fma(-hsum[i], S[c], g[c]) : v;
    if constexpr (PUSH) {
      peer_row(pd, i)[pc0 + c] = out;
    } else {
      __stcs(Y + i * ldy + c, out);
    }
  }
  if constexpr (PUSH) __threadfence_system();  // the sends precede the signal kernel's flag
}

void launch_block_out(const double *yt, int mb, int64_t mc, const double *hsum, const double *S,
                      const double *g, double *Y, int64_t ldy, int64_t i0, int64_t i1,
                      cudaStream_t s, const PeerDst *pd, int64_t pc0, const double *fx) {
  if (i1 <= i0) return;
  int64_t blocks = ((i1 - i0) * mc + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (pd && pd->world > 0)
    k9_block_out<true><<<(unsigned)blocks, 256, 0, s>>>(yt, mb, mc, hsum, S, g, Y, ldy, i0, i1,
                                                        *pd, pc0, fx);
  else
    k9_block_out<false><<<(unsigned)blocks, 256, 0, s>>>(yt, mb, mc, hsum, S, g, Y, ldy, i0, i1,
                                                         PeerDst{}, 0, fx);
}

// Block write-out of the single-pass fixed-point apply (k5_scan_lb), with the block's query totals
// folded in (no k4_totals launch): S_c = coordinate 0's segment total of s, g_c = sum_k T_kc
// (warp per column, lanes over k, a fixed butterfly: every CTA derives the same values; CTA 0
// also stores them to Sg), then Y[i][c0 + c] = Yt[i][c] 2^-F_c + g_c - h_i S_c for rows
// [i0, i1), two columns per thread (16-byte loads, and stores when Y allows).
template <bool PUSH>
__global__ void __launch_bounds__(256)
    k9f_block_out(const unsigned long long *__restrict__ yt, int mb, int64_t mc,
                  const double *__restrict__ hsum, const double *__restrict__ segtot,
                  int64_t ld_seg, int64_t dl, double *__restrict__ Sg, int64_t m_all,
                  double *__restrict__ Y, int64_t ldy, int64_t i0, int64_t i1, PeerDst pd,
                  int64_t pc0, const double *__restrict__ fx_inv, int vec) {
  __shared__ double s_S[32], s_g[32], s_f[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c = w; c < mb; c += 8) {
    double gk = 0.0;
    if (c < mc)
      for (int64_t k = lane; k < dl; k += 32) gk += __ldg(segtot + k * ld_seg + 2 * c + 1);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) gk += __shfl_xor_sync(0xFFFFFFFFu, gk, off);
    if (lane == 0) {
      const double S = c < mc ? __ldg(segtot + 2 * c) : 0.0;
      s_S[c] = S;
      s_g[c] = gk;
      s_f[c] = c < mc ? __ldg(fx_inv + c) : 0.0;
      if (blockIdx.x == 0 && c < mc) {
        Sg[c] = S;
        Sg[m_all + c] = gk;
      }
    }
  }
  __syncthreads();
  const int hp = mb > 1 ? mb >> 1 : 1;  // column pairs per row (mb = 1: one column)
  // mb is a power of two (the planner's blocks): row and pair by shift and mask — a 64-bit
  // division per element made this pass ALU-bound
  const int hsh = __ffs(hp) - 1;
  const int64_t total = (i1 - i0) * hp;
  const int64_t stride = (int64_t)gridDim.x * 256;
  // four elements per thread in flight (loads first): one 16-byte load per iteration left the
  // pass latency-bound at ~2.8 TB/s
  constexpr int U = 4;
  for (int64_t e0 = (int64_t)blockIdx.x * 256 + threadIdx.x; e0 < total; e0 += U * stride) {
    ulonglong2 q[U];
    double hv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      q[u] = make_ulonglong2(0ull, 0ull);
      hv[u] = 0.0;
      if (e < total) {
        const int64_t i = i0 + (e >> hsh);
        const int c = mb > 1 ? 2 * (int)(e & (hp - 1)) : 0;
        if (mb > 1)
          q[u] = __ldcs(reinterpret_cast<const ulonglong2 *>(yt + i * mb + c));
        else
          q[u] = make_ulonglong2(__ldcs(yt + i), 0ull);
        hv[u] = __ldg(hsum + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      if (e >= total) break;
      const int64_t i = i0 + (e >> hsh);
      const int c = mb > 1 ? 2 * (int)(e & (hp - 1)) : 0;
      if (c >= mc) continue;
      const double h = hv[u];
      const double o0 = (double)(long long)q[u].x * s_f[c] + fma(-h, s_S[c], s_g[c]);
      const double o1 = c + 1 < mc ? (double)(long long)q[u].y * s_f[c + 1] +
                                         fma(-h, s_S[c + 1], s_g[c + 1])
                                   : 0.0;
      if constexpr (PUSH) {
        double *row = peer_row(pd, i) + pc0 + c;
        row[0] = o0;
        if (c + 1 < mc) row[1] = o1;
      } else {
        double *yo = Y + i * ldy + c;
        if (vec && c + 1 < mc) {
          __stcs(reinterpret_cast<double2 *>(yo), make_double2(o0, o1));
        } else {
          __stcs(yo, o0);
          if (c + 1 < mc) __stcs(yo + 1, o1);
        }
      }
    }
  }
  if constexpr (PUSH) __threadfence_system();  // the sends precede the signal kernel's flag
}

void launch_block_out_fx(const unsigned long long *yt, int mb, int64_t mc, const double *hsum,
                         const double *segtot, int64_t ld_seg, int64_t dl, double *Sg,
                         int64_t m_all, double *Y, int64_t ldy, int64_t i0, int64_t i1,
                         cudaStream_t s, const PeerDst *pd, int64_t pc0, const double *fx_inv) {
  if (i1 <= i0) return;
  int64_t blocks = ((i1 - i0) * (mb > 1 ? mb / 2 : 1) + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  const int vec = (reinterpret_cast<uintptr_t>(Y) % 16 == 0 && ldy % 2 == 0) ? 1 : 0;
  if (pd && pd->world > 0)
    k9f_block_out<true><<<(unsigned)blocks, 256, 0, s>>>(yt, mb, mc, hsum, segtot, ld_seg, dl,
                                                         Sg, m_all, Y, ldy, i0, i1, *pd, pc0,
                                                         fx_inv, vec);
  else
    k9f_block_out<false><<<(unsigned)blocks, 256, 0, s>>>(yt, mb, mc, hsum, segtot, ld_seg, dl,
                                                          Sg, m_all, Y, ldy, i0, i1, PeerDst{}, 0,
                                                          fx_inv, vec);
}

// The fixed-point scales of a query (SEQ_APPLY_FX), one per column c.  Every term
// 2U^k_r = 2 (v_r P_r - Q_r) satisfies |2U^k| <= 4 Mx_k Sz_c (|P_r| and |Q_r| / Mx_k are partial
// sums of |z|), Mx_k the largest |x| of coordinate k (the ends of its sorted row) and Sz_c the
// column sum of |z|; a point's block row, a sum over the dl coordinates, stays below
// B_c = 4 Sz_c sum_k Mx_k (x 1.0001 for the bound's own rounding).  F_c = 61 - ceil(log2 B_c)
// keeps every partial sum below 2^61 in magnitude: fx[c] = 2^F_c, fx[m + c] = 2^-F_c.  Each
// term is rounded once to 2^-F_c (<= 2^-(F_c+1) absolute, about 2^-63 B_c), the sum is exact.
// The scale itself must not depend on the order of any floating-point sum (else F_c could flip
// at a power of two from run to run): k8_zt writes per-CTA partial sums (its threads folded in
// order) while it builds the Zt blocks, k8c adds them in a fixed lane/butterfly order.
__global__ void __launch_bounds__(256)
    k8c_fx_scale(const double *__restrict__ part, int64_t nparts, int64_t m,
                 const uint32_t *__restrict__ sval_bits, int64_t ldn, int64_t n, int64_t dl,
                 double *__restrict__ fx) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // sum_k Mx_k: lanes over k, a fixed butterfly (every warp computes it)
  double mx = 0.0, mxx = 0.0;  // sum_k Mx_k and max_k Mx_k
  for (int64_t k = lane; k < dl; k += 32) {
    const double mk = fmax(fabs((double)__uint_as_float(sval_bits[k * ldn])),
                           fabs((double)__uint_as_float(sval_bits[k * ldn + n - 1])));
    mx += mk;
    mxx = fmax(mxx, mk);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mx += __shfl_xor_sync(0xFFFFFFFFu, mx, off);
    mxx = fmax(mxx, __shfl_xor_sync(0xFFFFFFFFu, mxx, off));
  }
  // F = 61 - ilogb(B) - 1 (B > 0 finite), clamped: B 2^F < 2^61
  auto scale_exp = [](double B, int top) {
    int F = 0;
    if (B > 0.0 && isfinite(B)) {
      F = top - ilogb(B) - 1;
      if (F > 1000) F = 1000;
      if (F < -1000) F = -1000;
    }
    return F;
  };
  // column c: lanes over the CTA partials (strided, in order), then a fixed butterfly
  for (int64_t c = (int64_t)blockIdx.x * 8 + w; c < m; c += (int64_t)gridDim.x * 8) {
    double sz = 0.0;
    for (int64_t t = lane; t < nparts; t += 32) sz += part[t * m + c];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sz += __shfl_xor_sync(0xFFFFFFFFu, sz, off);
    if (lane != 0) continue;
    // B = 0: the column is zero, any scale.  2^ilogb(B) <= B < 2^(ilogb+1): B < 2^(61 - F).
    // Tiny data take large F (2^F stays finite up to F = 1000, i.e. B >= 2^-939 keeps the full
    // 61 bits; fp32 inputs give B >= ~2^-300)
    const int F = scale_exp(4.0 * mx * sz * 1.0001, 61);
    fx[c] = ldexp(1.0, F);
    fx[m + c] = ldexp(1.0, -F);
    const bool bad = !isfinite(sz);  // a NaN / Inf in column c: the column's Y is NaN (the
    if (bad) {                       // fixed-point path would otherwise hide it)
      fx[c] = 0.0;
      fx[m + c] = CUDART_NAN;
    }
    // the single-pass apply's look-back (k5_scan_lb): every partial sum of s = z over a
    // coordinate is bounded by sz, of t = v z by max_k Mx_k sz; the rounded tile aggregates'
    // sums stay below 2^58 (the look-back words carry 60-bit signed values)
    const int Fz = scale_exp(sz * 1.0001, 58), Fv = scale_exp(mxx * sz * 1.0001, 58);
    fx[2 * m + c] = ldexp(1.0, Fz);
    fx[3 * m + c] = bad ? CUDART_NAN : ldexp(1.0, -Fz);
    fx[4 * m + c] = ldexp(1.0, Fv);
    fx[5 * m + c] = bad ? CUDART_NAN : ldexp(1.0, -Fv);
  }
}

// Look-back scales for the odd-p single pass: per column c and moment t = 0..lp, 2^F with
// max_k Mx_k^t sum_i |z_ic| 2^F < 2^58 (every partial sum of z v^t over a coordinate is below the
// bound), summed in the same fixed orders as k8c_fx_scale.
__global__ void __launch_bounds__(256)
    k8e_lb_scales(const double *__restrict__ part, int64_t nparts, int64_t m,
                  const uint32_t *__restrict__ sval_bits, int64_t ldn, int64_t n, int64_t dl,
                  int lp, double *__restrict__ fa) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double mxx = 0.0;
  for (int64_t k = lane; k < dl; k += 32)
    mxx = fmax(mxx, fmax(fabs((double)__uint_as_float(sval_bits[k * ldn])),
                         fabs((double)__uint_as_float(sval_bits[k * ldn + n - 1]))));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mxx = fmax(mxx, __shfl_xor_sync(0xFFFFFFFFu, mxx, off));
  for (int64_t c = (int64_t)blockIdx.x * 8 + w; c < m; c += (int64_t)gridDim.x * 8) {
    double sz = 0.0;
    for (int64_t t = lane; t < nparts; t += 32) sz += part[t * m + c];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sz += __shfl_xor_sync(0xFFFFFFFFu, sz, off);
    if (lane != 0) continue;
    const bool bad = !isfinite(sz);  // NaN / Inf in column c: NaN prefixes, so Y's column is NaN
    double B = sz * 1.0001;
    for (int t = 0; t <= lp; ++t) {
      int F = 0;
      if (B > 0.0 && isfinite(B)) {
        F = 58 - ilogb(B) - 1;
        if (F > 1000) F = 1000;
        if (F < -1000) F = -1000;
      }
      fa[(2 * t) * m + c] = ldexp(1.0, F);
      fa[(2 * t + 1) * m + c] = bad ? CUDART_NAN : ldexp(1.0, -F);
      B *= mxx;
    }
  }
}

void launch_lb_scales(const double *part, int64_t nparts, int64_t m, const uint32_t *sval_bits,
                      int64_t ldn, int64_t n, int64_t dl, int lp, double *fa, cudaStream_t s) {
  k8e_lb_scales<<<(unsigned)((m + 7) / 8), 256, 0, s>>>(part, nparts, m, sval_bits, ldn, n, dl,
                                                        lp, fa);
}

// X in point order from the sorted tables, xr[perm[k][r] dl + k] = sval[k][r]: the odd-p single
// pass needs x_ik^(p-t) by point for its totals expansion (launch_lp_totals_expand); built once
// per handle on the first such query.
__global__ void __launch_bounds__(256)
    k3x_unsort(const uint32_t *__restrict__ perm, const float *__restrict__ sval, int64_t ldn,
               int64_t n, int64_t dl, float *__restrict__ xr) {
  const int64_t k = blockIdx.y;
  for (int64_t r = (int64_t)blockIdx.x * 256 + threadIdx.x; r < n; r += (int64_t)gridDim.x * 256)
    xr[(int64_t)perm[k * ldn + r] * dl + k] = sval[k * ldn + r];
}

void launch_unsort(const uint32_t *perm, const float *sval, int64_t ldn, int64_t n, int64_t dl,
                   float *xr, cudaStream_t s) {
  int64_t bx = (n + 255) / 256;
  if (bx > 1024) bx = 1024;
  k3x_unsort<<<dim3((unsigned)bx, (unsigned)dl), 256, 0, s>>>(perm, sval, ldn, n, dl, xr);
}

void launch_fx_scale(const double *part, int64_t nparts, int64_t m, const uint32_t *sval_bits,
                     int64_t ldn, int64_t n, int64_t dl, double *fx, cudaStream_t s) {
  k8c_fx_scale<<<(unsigned)((m + 7) / 8), 256, 0, s>>>(part, nparts, m, sval_bits, ldn, n, dl,
                                                       fx);
}

// ------------------------------------------------------------------ runs mode
// For tie-heavy coordinates (<= 256 distinct values each) Alg. 2 collapses to its distinct
// values: with H_j = sum of z over run j, P_j / Q_j the exclusive prefixes over runs of H and
// v H, every point of run j sees U^k = v_j P_j - Q_j (the prefix at any row of a run differs
// only by equal-value terms, which contribute 0 — P:173 / P:205), so
//   y_i = 2 sum_k U^k[runid_k(i)] + g - h_i S,  U^k[j] = v_j P_j - Q_j
// R1  H[k][j][c] += z_ic for j = runid[k][i] (fp64 L2 reductions into an L2-resident table,
//     points read in point order: no sorted-order gather at all)
// R2  per (k, c): the prefix over runs, U in place, segment totals (S, T_k) for k4_totals
// R3  per point tile: U^k staged in shared memory per coordinate, y accumulated in registers.
__global__ void __launch_bounds__(256)
    k20_runs_hist(const uint8_t *__restrict__ runid, int64_t ldn, int64_t n, int64_t dl,
                  const float *__restrict__ Z, int64_t ldz, int64_t m, int kg,
                  double *__restrict__ H, int copies) {
  // lane -> (point p within the warp's group of 32/L, column c), L = min(32, pow2 >= m)
  const int L = m >= 32 ? 32 : (m > 16 ? 32 : m > 8 ? 16 : m > 4 ? 8 : m > 2 ? 4 : m > 1 ? 2 : 1);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int pg = lane / L, cl = lane - (lane / L) * L;
  const int ppw = 32 / L;  // points per warp step
  const int64_t k0 = (int64_t)blockIdx.y * kg;
  const int64_t k1 = (k0 + kg < dl) ? k0 + kg : dl;
  const int64_t pts_per_cta = 8 * ppw * 16;  // 16 steps per warp
  const int64_t i_base = (int64_t)blockIdx.x * pts_per_cta + (int64_t)w * ppw * 16;
  const uint64_t pol = l2_policy_evict_last();
  // narrow tables (few coordinates) are spread over `copies` replicas, a warp on one of them:
  // a table of a few thousand 128-byte lines loads the L2 slices unevenly, and how unevenly
  // depends on where the allocation landed (runs_copies); folded by k20b_fold before the scan
  H += (int64_t)((blockIdx.x * 8 + w) % (unsigned)copies) * (dl * 256 * m);
  for (int step = 0; step < 16; ++step) {
    const int64_t i = i_base + (int64_t)step * ppw + pg;
    if (i >= n) break;
    for (int64_t c0 = 0; c0 < m; c0 += L) {
      const int64_t c = c0 + cl;
      if (c >= m) continue;
      const float z = __ldg(Z + i * ldz + c);
      for (int64_t k = k0; k < k1; ++k) {
        const uint32_t j = __ldg(runid + k * ldn + i);
        red_add_f64(H + ((k * 256 + j) * m + c), (double)z, pol);
      }
    }
  }
}

// H[e] += H[e + r T] for the replicas r = 1 .. copies - 1 (in that order), T = dl 256 m.
__global__ void __launch_bounds__(256)
    k20b_fold(double *__restrict__ H, int64_t T, int copies) {
  const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (e >= T) return;
  double a = H[e];
  for (int r = 1; r < copies; ++r) a += H[e + (int64_t)r * T];
  H[e] = a;
}

// Replicas of the run table for the histogram's reductions: enough that they spread over
// ~100 k 128-byte lines, at most 8 (measured on c5: 12 coordinates x 8 replicas 4.34 -> 3.48 ms
// per query, 96 coordinates x 4 replicas 24.19 -> 23.8 ms; 8 replicas there no better).
int runs_copies(int64_t dl, int64_t m) {
#if L1DM_RUNS_COPIES
  const int64_t lines = dl * 256 * m * 8 / 128;
  int c = 1;
  while (c < 8 && lines * c * 2 <= 98304) c *= 2;
  return c;
#else
  (void)dl; (void)m;
  return 1;
#endif
}

__global__ void __launch_bounds__(256)
    k21_runs_scan(double *__restrict__ H, const float *__restrict__ rvals,
                  const uint32_t *__restrict__ nruns, int64_t dl, int64_t m,
                  double *__restrict__ segtot) {
  const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (e >= dl * m) return;
  const int64_t k = e / m, c = e - (e / m) * m;
  const uint32_t R = nruns[k];
  double P = 0.0, Q = 0.0;
  uint32_t j = 0;
  // eight runs' H and values loaded before the in-place stores (the sequential form waits one
  // L2 round trip per run: 256 of them per query whatever dl is); same order of additions
  for (; j + 8 <= R; j += 8) {
    double h8[8];
    float v8[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h8[u] = H[(k * 256 + j + u) * m + c];
      v8[u] = rvals[k * 256 + j + u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double v = (double)v8[u];
      H[(k * 256 + j + u) * m + c] = fma(v, P, -Q);
      P += h8[u];
      Q = fma(v, h8[u], Q);
    }
  }
  for (; j < R; ++j) {
    double *hp = H + (k * 256 + j) * m + c;
    const double h = *hp, v = (double)rvals[k * 256 + j];
    *hp = fma(v, P, -Q);  // U at run j (exclusive prefixes)
    P += h;
    Q = fma(v, h, Q);
  }
  segtot[k * 2 * m + 2 * c] = P;      // S_c (every coordinate's total of z)
  segtot[k * 2 * m + 2 * c + 1] = Q;  // T_kc
}

// grid: point tiles of 256 points x column chunks of MC; block 256 threads; thread (p, c):
// p = tid / MC + (256 / MC) u for u < MC, c = c0 + tid % MC.
template <int MC>
__global__ void __launch_bounds__(256)
    k22_runs_expand(const uint8_t *__restrict__ runid, int64_t ldn, int64_t n, int64_t dl,
                    const double *__restrict__ U, const uint32_t *__restrict__ nruns, int64_t m,
                    const double *__restrict__ hsum, const double *__restrict__ Sg,
                    double *__restrict__ Y, int64_t ldy, int64_t i_begin) {
  constexpr int PT = 256;               // points per CTA
  constexpr int PPP = 256 / MC;         // points per pass of the CTA's threads
  constexpr int NP = PT / PPP;          // points per thread (= MC)
  __shared__ double us[256 * MC];       // U^k[j][c0 .. c0 + MC)
  const int tid = threadIdx.x;
  const int cl = tid % MC, pr = tid / MC;
  const int64_t i0 = i_begin + (int64_t)blockIdx.x * PT, c0 = (int64_t)blockIdx.y * MC;
  const int64_t c = c0 + cl;
  double acc[NP];
#pragma unroll
  for (int u = 0; u < NP; ++u) acc[u] = 0.0;
  for (int64_t k = 0; k < dl; ++k) {
    const int R = (int)nruns[k];
    __syncthreads();
    for (int e = tid; e < R * MC; e += 256) {
      const int j = e / MC, q = e - (e / MC) * MC;
      us[e] = (c0 + q < m) ? __ldg(U + (k * 256 + j) * m + c0 + q) : 0.0;
    }
    __syncthreads();
    const uint8_t *rk = runid + k * ldn;
#pragma unroll
    for (int u = 0; u < NP; ++u) {
      const int64_t i = i0 + pr + (int64_t)PPP * u;
      if (i < n) acc[u] += us[(int)__ldg(rk + i) * MC + cl];
    }
  }
  if (c >= m) return;
#pragma unroll
  for (int u = 0; u < NP; ++u) {
    const int64_t i = i0 + pr + (int64_t)PPP * u;
    if (i < n) Y[i * ldy + c] = 2.0 * acc[u] + fma(-hsum[i], Sg[c], Sg[m + c]);
  }
}

// Expansion without staging: a point's V lanes sum U^k[runid][c0 .. c0 + V) straight from the
// L2-resident table (dl x 256 x m fp64) — the staged kernel above copies each coordinate's
// table into shared memory once per 256 points, i.e. as many L2 bytes as the points read.
template <int V, int LPP, int UNR, bool LP = false>
__global__ void __launch_bounds__(256)
    k22_runs_gather(const uint8_t *__restrict__ runid, int64_t ldn, int64_t n, int64_t dl,
                    const double *__restrict__ U, int64_t m, const double *__restrict__ hsum,
                    const double *__restrict__ Sg, double *__restrict__ Y, int64_t ldy,
                    int64_t i_begin) {
  constexpr int PPW = 32 / LPP;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = i_begin + (int64_t)blockIdx.x * (8 * PPW) + (int64_t)w * PPW + lane / LPP;
  const int64_t c0 = (int64_t)blockIdx.y * (LPP * V) + (int64_t)(lane % LPP) * V;
  if (i >= n || c0 >= m) return;
  double acc[V];
#pragma unroll
  for (int q = 0; q < V; ++q) acc[q] = 0.0;
  const uint8_t *rp = runid + i;
  const double *ub = U + c0;
  int64_t k = 0;
  for (; k + UNR <= dl; k += UNR) {
    uint32_t r[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) r[u] = __ldg(rp + (k + u) * ldn);
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const double *p = ub + ((k + u) * 256 + r[u]) * m;
      if constexpr (V == 2) {
        const double2 v = __ldg(reinterpret_cast<const double2 *>(p));
        acc[0] += v.x;
        acc[1] += v.y;
      } else {
        acc[0] += __ldg(p);
      }
    }
  }
  if constexpr (UNR > 4) {  // the remainder four run ids at a time before the singles
    for (; k + 4 <= dl; k += 4) {
      uint32_t r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = __ldg(rp + (k + u) * ldn);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double *p = ub + ((k + u) * 256 + r[u]) * m;
        if constexpr (V == 2) {
          const double2 v = __ldg(reinterpret_cast<const double2 *>(p));
          acc[0] += v.x;
          acc[1] += v.y;
        } else {
          acc[0] += __ldg(p);
        }
      }
    }
  }
  for (; k < dl; ++k) {
    const double *p = ub + (k * 256 + __ldg(rp + k * ldn)) * m;
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] += __ldg(p + q);
  }
#pragma unroll
  for (int q = 0; q < V; ++q)
    Y[i * ldy + c0 + q] = LP ? acc[q]  // l_p^p: the table holds each coordinate's whole term
                             : 2.0 * acc[q] + fma(-hsum[i], Sg[c0 + q], Sg[m + c0 + q]);
}

// Odd p (DESIGN.md §2b over runs, §2f): with H_j = sum of z over run j (the histogram), per
// (coordinate, column) the totals T_t = sum_j v_j^t H_j, then in run order the exclusive
// moments M_t(j) and W_j = sum_t c_t v_j^(P-t) (2 M_t(j) - T_t) in place of H — the same value
// every row of run j gets in the sorted scan (rows of the run itself contribute |v - v|^p = 0).
template <int P>
__global__ void __launch_bounds__(256)
    k21_runs_scan_lp(double *__restrict__ H, const float *__restrict__ rvals,
                     const uint32_t *__restrict__ nruns, int64_t dl, int64_t m) {
  constexpr int K = P + 1;
  const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (e >= dl * m) return;
  const int64_t k = e / m, c = e - (e / m) * m;
  const uint32_t R = nruns[k];
  double T[K], M[K];
#pragma unroll
  for (int t = 0; t < K; ++t) T[t] = M[t] = 0.0;
#pragma unroll 8  // eight runs' loads in flight (no stores in this loop)
  for (uint32_t j = 0; j < R; ++j) {
    const double h = H[(k * 256 + j) * m + c], v = (double)rvals[k * 256 + j];
    double hv = h;
#pragma unroll
    for (int t = 0; t < K; ++t) {
      T[t] += hv;
      hv *= v;
    }
  }
  for (uint32_t j0 = 0; j0 < R; j0 += 8) {
    // the next eight runs' H and values loaded before the in-place stores (as k21_runs_scan)
    double h8[8];
    float v8[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t ju = j0 + u < R ? j0 + u : R - 1;
      h8[u] = H[(k * 256 + ju) * m + c];
      v8[u] = rvals[k * 256 + ju];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t j = j0 + u;
      if (j >= R) break;
      double *hp = H + (k * 256 + j) * m + c;
      const double h = h8[u], v = (double)v8[u];
      double vp[K];
      vp[0] = 1.0;
#pragma unroll
      for (int t = 1; t < K; ++t) vp[t] = vp[t - 1] * v;
      double w = 0.0;
#pragma unroll
      for (int t = 0; t < K; ++t) {
        double b = 1.0;  // c_t = C(P, t) (-1)^t
        for (int q = 0; q < t; ++q) b = b * (double)(P - q) / (double)(q + 1);
        w = fma(((t & 1) ? -b : b) * vp[P - t], fma(2.0, M[t], -T[t]), w);
      }
      *hp = w;
      double hv = h;
#pragma unroll
      for (int t = 0; t < K; ++t) {
        M[t] += hv;
        hv *= v;
      }
    }
  }
}

// Coordinates per run-histogram CTA: at most L1DM_RUNS_KG, balanced over the grid.y slices so
// no slice is a thin tail (dl = 128 -> 2 x 64, not 96 + 32; dl = 97 -> 49 + 48).
static int runs_kg(int64_t dl) {
  const int64_t slices = (dl + L1DM_RUNS_KG - 1) / L1DM_RUNS_KG;
  return (int)((dl + slices - 1) / (slices < 1 ? 1 : slices));
}

void launch_runs_lp(const uint8_t *runid, int64_t ldn, int64_t n, int64_t dl, const float *rvals,
                    const uint32_t *nruns, const float *Z, int64_t ldz, int64_t m, int lp,
                    double *H, double *Y, int64_t ldy, int phase, cudaStream_t s) {
  // phase 0: R1 as for l1 (the run sums of z), then the p-moment scan over runs in place of
  // the l1 prefix; phase 1: the expansion without the l1 epilogue (no g - h S for p > 1)
  if (phase == 0) {
    const int copies = runs_copies(dl, m);
    cudaMemsetAsync(H, 0, (size_t)copies * dl * 256 * m * sizeof(double), s);
    const int L = m >= 32 ? 32 : (m > 16 ? 32 : m > 8 ? 16 : m > 4 ? 8 : m > 2 ? 4 : m > 1 ? 2 : 1);
    const int64_t pts_per_cta = 8 * (32 / L) * 16;
    const int kg = runs_kg(dl);
    dim3 g1((unsigned)((n + pts_per_cta - 1) / pts_per_cta), (unsigned)((dl + kg - 1) / kg));
    k20_runs_hist<<<g1, 256, 0, s>>>(runid, ldn, n, dl, Z, ldz, m, kg, H, copies);
    if (copies > 1)
      k20b_fold<<<(unsigned)((dl * 256 * m + 255) / 256), 256, 0, s>>>(H, dl * 256 * m, copies);
    const unsigned g2 = (unsigned)((dl * m + 255) / 256);
    switch (lp) {
      case 3: k21_runs_scan_lp<3><<<g2, 256, 0, s>>>(H, rvals, nruns, dl, m); break;
      case 5: k21_runs_scan_lp<5><<<g2, 256, 0, s>>>(H, rvals, nruns, dl, m); break;
      case 7: k21_runs_scan_lp<7><<<g2, 256, 0, s>>>(H, rvals, nruns, dl, m); break;
      default: break;
    }
    return;
  }
  auto g = [&](auto kern, int LPP, int V) {
    const int ppb = 8 * (32 / LPP);
    dim3 grid((unsigned)((n + ppb - 1) / ppb), (unsigned)((m + V * LPP - 1) / (V * LPP)));
    kern<<<grid, 256, 0, s>>>(runid, ldn, n, dl, H, m, nullptr, nullptr, Y, ldy, 0);
  };
  if (m % 2 == 0) {
    const int64_t lpp = m / 2;
    if (lpp <= 1) g(k22_runs_gather<2, 1, 8, true>, 1, 2);
    else if (lpp <= 2) g(k22_runs_gather<2, 2, 8, true>, 2, 2);
    else if (lpp <= 4) g(k22_runs_gather<2, 4, 8, true>, 4, 2);
    else if (lpp <= 8) g(k22_runs_gather<2, 8, L1DM_RUNS_UNR, true>, 8, 2);
    else if (lpp <= 16) g(k22_runs_gather<2, 16, 8, true>, 16, 2);
    else g(k22_runs_gather<2, 32, 8, true>, 32, 2);
  } else {
    if (m <= 1) g(k22_runs_gather<1, 1, 8, true>, 1, 1);
    else if (m <= 2) g(k22_runs_gather<1, 2, 8, true>, 2, 1);
    else if (m <= 4) g(k22_runs_gather<1, 4, 8, true>, 4, 1);
    else if (m <= 8) g(k22_runs_gather<1, 8, 8, true>, 8, 1);
    else if (m <= 16) g(k22_runs_gather<1, 16, 8, true>, 16, 1);
    else g(k22_runs_gather<1, 32, 8, true>, 32, 1);
  }
}

void launch_runs_query(const uint8_t *runid, int64_t ldn, int64_t n, int64_t dl, const float *rvals,
                       const uint32_t *nruns, const float *Z, int64_t ldz, int64_t m, double *H,
                       double *segtot, const double *hsum, double *Sg, double *Y, int64_t ldy,
                       int phase, cudaStream_t s, int64_t i0, int64_t i1) {
  if (phase == 0) {
    const int copies = runs_copies(dl, m);
    cudaMemsetAsync(H, 0, (size_t)copies * dl * 256 * m * sizeof(double), s);
    const int L = m >= 32 ? 32 : (m > 16 ? 32 : m > 8 ? 16 : m > 4 ? 8 : m > 2 ? 4 : m > 1 ? 2 : 1);
    const int64_t pts_per_cta = 8 * (32 / L) * 16;
    const int kg = runs_kg(dl);
    dim3 g1((unsigned)((n + pts_per_cta - 1) / pts_per_cta), (unsigned)((dl + kg - 1) / kg));
    k20_runs_hist<<<g1, 256, 0, s>>>(runid, ldn, n, dl, Z, ldz, m, kg, H, copies);
    if (copies > 1)
      k20b_fold<<<(unsigned)((dl * 256 * m + 255) / 256), 256, 0, s>>>(H, dl * 256 * m, copies);
    const int64_t t2 = dl * m;
    k21_runs_scan<<<(unsigned)((t2 + 255) / 256), 256, 0, s>>>(H, rvals, nruns, dl, m, segtot);
    return;
  }
  // phase 1: expand (Sg = S, g from the segment totals, computed by the caller)
  if (i1 < 0) i1 = n;
  if (i1 <= i0) return;
  auto run = [&](auto kern, int MC) {  // points [i0, i1): the kernel bounds rows by i1 via n
    dim3 g3((unsigned)((i1 - i0 + 255) / 256), (unsigned)((m + MC - 1) / MC));
    kern<<<g3, 256, 0, s>>>(runid, ldn, i1, dl, H, nruns, m, hsum, Sg, Y, ldy, i0);
  };
  static const int gather_env = [] {
    const char *e = getenv("L1DM_RUNS_GATHER");
    return e ? atoi(e) : -1;
  }();
  // default: the unstaged gather (measured on B200, c5: expand 19.2 -> 8.5 ms); lanes cover
  // V = 2 columns (even m) or 1, LPP lanes per point, wide m in several column groups
  if (gather_env != 0) {
    auto g = [&](auto kern, int LPP, int V) {
      const int ppb = 8 * (32 / LPP);
      dim3 grid((unsigned)((i1 - i0 + ppb - 1) / ppb), (unsigned)((m + V * LPP - 1) / (V * LPP)));
      kern<<<grid, 256, 0, s>>>(runid, ldn, i1, dl, H, m, hsum, Sg, Y, ldy, i0);
    };
    // narrow coordinate shards (dl < 16, e.g. c5 at G = 8: 12): 4 run ids in flight per step,
    // so the unrolled body covers the shard instead of the one-at-a-time tail loop
    const bool narrow = dl < 16;
    if (m % 2 == 0) {
      const int64_t lpp = m / 2;
      if (narrow) {
        if (lpp <= 1) g(k22_runs_gather<2, 1, 4>, 1, 2);
        else if (lpp <= 2) g(k22_runs_gather<2, 2, 4>, 2, 2);
        else if (lpp <= 4) g(k22_runs_gather<2, 4, 4>, 4, 2);
        else if (lpp <= 8) {
          if (dl >= 8) g(k22_runs_gather<2, 8, 8>, 8, 2);  // 8 + a 4-wide remainder (c5 at G = 8: 12)
          else g(k22_runs_gather<2, 8, 4>, 8, 2);
        }
        else if (lpp <= 16) g(k22_runs_gather<2, 16, 4>, 16, 2);
        else g(k22_runs_gather<2, 32, 4>, 32, 2);
      } else if (lpp <= 1) g(k22_runs_gather<2, 1, 8>, 1, 2);
      else if (lpp <= 2) g(k22_runs_gather<2, 2, 8>, 2, 2);
      else if (lpp <= 4) g(k22_runs_gather<2, 4, 8>, 4, 2);
      else if (lpp <= 8) g(k22_runs_gather<2, 8, L1DM_RUNS_UNR>, 8, 2);
      else if (lpp <= 16) g(k22_runs_gather<2, 16, 8>, 16, 2);
      else g(k22_runs_gather<2, 32, 8>, 32, 2);
    } else {
      if (narrow) {
        if (m <= 1) g(k22_runs_gather<1, 1, 4>, 1, 1);
        else if (m <= 2) g(k22_runs_gather<1, 2, 4>, 2, 1);
        else if (m <= 4) g(k22_runs_gather<1, 4, 4>, 4, 1);
        else if (m <= 8) g(k22_runs_gather<1, 8, 4>, 8, 1);
        else if (m <= 16) g(k22_runs_gather<1, 16, 4>, 16, 1);
        else g(k22_runs_gather<1, 32, 4>, 32, 1);
      } else if (m <= 1) g(k22_runs_gather<1, 1, 8>, 1, 1);
      else if (m <= 2) g(k22_runs_gather<1, 2, 8>, 2, 1);
      else if (m <= 4) g(k22_runs_gather<1, 4, 8>, 4, 1);
      else if (m <= 8) g(k22_runs_gather<1, 8, 8>, 8, 1);
      else if (m <= 16) g(k22_runs_gather<1, 16, 8>, 16, 1);
      else g(k22_runs_gather<1, 32, 8>, 32, 1);
    }
    return;
  }
  if (m <= 4) run(k22_runs_expand<4>, 4);
  else if (m <= 8) run(k22_runs_expand<8>, 8);
  else run(k22_runs_expand<16>, 16);
}

// Y[i][c] = Yb[c / mb][i][c % mb]: column-block-major (l1dm_matvec_colblocks) to row-major.
__global__ void __launch_bounds__(256)
    k10_unblock(const double *__restrict__ Yb, int64_t n, int64_t m, int64_t mb,
                double *__restrict__ Y, int64_t ldy) {
  const int64_t total = n * m;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    const int64_t i = e / m, c = e - (e / m) * m;
    Y[i * ldy + c] = Yb[((c / mb) * n + i) * mb + (c % mb)];
  }
}

void launch_unblock(const double *Yb, int64_t n, int64_t m, int64_t mb, double *Y, int64_t ldy,
                    cudaStream_t s) {
  int64_t blocks = (n * m + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k10_unblock<<<(unsigned)blocks, 256, 0, s>>>(Yb, n, m, mb, Y, ldy);
}

// Y[i][c] *= a (TV = a * l1 with a = 1/2).
__global__ void __launch_bounds__(256)
    k10_scale(double *__restrict__ Y, int64_t ldy, int64_t n, int64_t m, double a) {
  const int64_t total = n * m;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    const int64_t i = e / m, c = e - (e / m) * m;
    Y[i * ldy + c] *= a;
  }
}

void launch_scale(double *Y, int64_t ldy, int64_t n, int64_t m, double a, cudaStream_t s) {
  int64_t blocks = (n * m + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k10_scale<<<(unsigned)blocks, 256, 0, s>>>(Y, ldy, n, m, a);
}

// Simplex statistics of a prepared handle: out[0] = max_i |h_i - 1|, out[1] = min_k sval[k][0]
// (the smallest coordinate value overall).  One CTA; n and dl are small enough per handle for
// a grid-stride loop to be negligible next to prepare.
__global__ void __launch_bounds__(1024)
    k11_simplex_stats(const double *__restrict__ hsum, int64_t n, const float *__restrict__ sval,
                      int64_t ldn, int64_t dl, double *__restrict__ out) {
  __shared__ double s_a[32], s_b[32];
  double a = 0.0, b = 1e300;
  for (int64_t i = threadIdx.x; i < n; i += 1024) a = fmax(a, fabs(hsum[i] - 1.0));
  for (int64_t k = threadIdx.x; k < dl; k += 1024) b = fmin(b, (double)sval[k * ldn]);
  for (int off = 16; off; off >>= 1) {
    a = fmax(a, __shfl_xor_sync(0xFFFFFFFFu, a, off));
    b = fmin(b, __shfl_xor_sync(0xFFFFFFFFu, b, off));
  }
  if ((threadIdx.x & 31) == 0) {
    s_a[threadIdx.x >> 5] = a;
    s_b[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < 32; ++q) {
      a = fmax(a, s_a[q]);
      b = fmin(b, s_b[q]);
    }
    out[0] = a;
    out[1] = b;
  }
}

void launch_simplex_stats(const double *hsum, int64_t n, const float *sval, int64_t ldn,
                          int64_t dl, double *out, cudaStream_t s) {
  k11_simplex_stats<<<1, 1024, 0, s>>>(hsum, n, sval, ldn, dl, out);
}

// ------------------------------------------------------------------ scatter-mode Z blocks
// Zt[cb][i][0..mb) = Z[i][cb*mb ..] zero-padded past m.  Thread e -> (row i = e / cb_count,
// block cb = e % cb_count): a warp reads whole Z rows and writes full sectors of each block.
// With part != nullptr (scatter m > 1: the fixed-point scales, launch_fx_scale) the pass also
// sums |z| per column: the grid is a multiple of cb_count threads, so a thread's block is fixed;
// each CTA folds its threads' sums per column in thread order into part[blockIdx][m].
template <int MB>
__global__ void __launch_bounds__(256)
    k8_zt(const float *__restrict__ Z, int64_t ldz, int64_t n, int64_t m, int64_t ncb,
          float *__restrict__ zt, int vec4, double *__restrict__ part) {
  const int64_t total = n * ncb;
  float acc[MB];
#pragma unroll
  for (int q = 0; q < MB; ++q) acc[q] = 0.0f;
  double dacc[MB];
#pragma unroll
  for (int q = 0; q < MB; ++q) dacc[q] = 0.0;
  int cnt = 0;
  const int64_t stride = (int64_t)gridDim.x * 256;
  int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if constexpr (MB % 4 == 0) {
    // whole-block rows, 4 rows in flight per thread (loads of all four issued first); the
    // stride is a multiple of ncb, so a thread stays on one column block
    if (vec4 && m % MB == 0) {
      for (; e + 3 * stride < total; e += 4 * stride) {
        float4 t[4][MB / 4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t eu = e + u * stride, i = eu / ncb, cb = eu - i * ncb;
          const float4 *src = reinterpret_cast<const float4 *>(Z + i * ldz + cb * MB);
#pragma unroll
          for (int q = 0; q < MB / 4; ++q) t[u][q] = __ldcs(src + q);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t eu = e + u * stride, i = eu / ncb, cb = eu - i * ncb;
          float4 *dst = reinterpret_cast<float4 *>(zt + (cb * n + i) * MB);
#pragma unroll
          for (int q = 0; q < MB / 4; ++q) dst[q] = t[u][q];
          if (part) {
#pragma unroll
            for (int q = 0; q < MB / 4; ++q) {
              acc[4 * q] += fabsf(t[u][q].x);
              acc[4 * q + 1] += fabsf(t[u][q].y);
              acc[4 * q + 2] += fabsf(t[u][q].z);
              acc[4 * q + 3] += fabsf(t[u][q].w);
            }
            if (++cnt == 64) {
#pragma unroll
              for (int q = 0; q < MB; ++q) {
                dacc[q] += (double)acc[q];
                acc[q] = 0.0f;
              }
              cnt = 0;
            }
          }
        }
      }
    }
  }
  for (; e < total; e += stride) {
    const int64_t i = e / ncb, cb = e - (e / ncb) * ncb;
    const int64_t c0 = cb * MB;
    const float *src = Z + i * ldz + c0;
    float *dst = zt + (cb * n + i) * MB;
    float v[MB];
    bool done = false;
    if constexpr (MB % 4 == 0) {
      if (vec4 && c0 + MB <= m) {
#pragma unroll
        for (int q = 0; q < MB; q += 4) {
          const float4 t = __ldcs(reinterpret_cast<const float4 *>(src + q));
          reinterpret_cast<float4 *>(dst)[q / 4] = t;
          v[q] = t.x; v[q + 1] = t.y; v[q + 2] = t.z; v[q + 3] = t.w;
        }
        done = true;
      }
    }
    if (!done) {
#pragma unroll
      for (int q = 0; q < MB; ++q) {
        v[q] = (c0 + q < m) ? __ldcs(src + q) : 0.0f;
        dst[q] = v[q];
      }
    }
    if (part) {  // |z| sums: fp32 runs of 64 rows, folded into fp64 (a bound only)
#pragma unroll
      for (int q = 0; q < MB; ++q) acc[q] += fabsf(v[q]);
      if (++cnt == 64) {
#pragma unroll
        for (int q = 0; q < MB; ++q) {
          dacc[q] += (double)acc[q];
          acc[q] = 0.0f;
        }
        cnt = 0;
      }
    }
  }
  if (!part) return;
  constexpr int QC = MB < 16 ? MB : 16;  // columns of a block per shared-memory round
  __shared__ double s_acc[256 * QC];
  const int64_t base = (int64_t)blockIdx.x * 256;
#pragma unroll
  for (int q0 = 0; q0 < MB; q0 += QC) {
#pragma unroll
    for (int q = 0; q < QC; ++q) s_acc[threadIdx.x * QC + q] = dacc[q0 + q] + (double)acc[q0 + q];
    __syncthreads();
    for (int64_t c = threadIdx.x; c < m; c += 256) {
      const int64_t cb = c / MB, q = c - cb * MB;
      if (q < q0 || q >= q0 + QC) continue;
      int64_t t0 = (cb - base % ncb) % ncb;  // first thread of this CTA on block cb
      if (t0 < 0) t0 += ncb;
      double sum = 0.0;
      for (int64_t t = t0; t < 256; t += ncb) sum += s_acc[t * QC + (q - q0)];
      part[(int64_t)blockIdx.x * m + c] = sum;
    }
    __syncthreads();
  }
}

int64_t launch_zt(const float *Z, int64_t ldz, int64_t n, int64_t m, int mb, float *zt,
                  cudaStream_t s, double *colabs_part) {
  const int64_t ncb = (m + mb - 1) / mb;
  const int vec4 = (ldz % 4 == 0 && reinterpret_cast<uintptr_t>(Z) % 16 == 0) ? 1 : 0;
  int64_t blocks = (n * ncb + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  // with the |z| sums: whole multiples of ncb CTAs keep every thread on one block
  if (colabs_part) blocks = (blocks + ncb - 1) / ncb * ncb;
  switch (mb) {
    case 1: k8_zt<1><<<(unsigned)blocks, 256, 0, s>>>(Z, ldz, n, m, ncb, zt, vec4, colabs_part); break;
    case 2: k8_zt<2><<<(unsigned)blocks, 256, 0, s>>>(Z, ldz, n, m, ncb, zt, vec4, colabs_part); break;
    case 4: k8_zt<4><<<(unsigned)blocks, 256, 0, s>>>(Z, ldz, n, m, ncb, zt, vec4, colabs_part); break;
    case 8: k8_zt<8><<<(unsigned)blocks, 256, 0, s>>>(Z, ldz, n, m, ncb, zt, vec4, colabs_part); break;
    case 16: k8_zt<16><<<(unsigned)blocks, 256, 0, s>>>(Z, ldz, n, m, ncb, zt, vec4, colabs_part); break;
    case 32: k8_zt<32><<<(unsigned)blocks, 256, 0, s>>>(Z, ldz, n, m, ncb, zt, vec4, colabs_part); break;
    default: break;
  }
  return blocks;
}

int64_t zt_max_ctas(int64_t m, int mb) {
  const int64_t ncb = (m + mb - 1) / mb;
  return (148 * 16 + ncb - 1) / ncb * ncb;
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

template <int V6, int LPP, int UNR, bool PUSH>
__global__ void __launch_bounds__(256)
    k6_accumulate(const uint32_t *__restrict__ rank, int64_t ldn, int64_t n,
                  const double *__restrict__ U, int64_t ldu, int64_t k_first, int64_t kcc,
                  const double *__restrict__ hsum, const double *__restrict__ Sg,
                  double *__restrict__ Y, int64_t ldy, int64_t m, int first_chunk,
                  int last_chunk, unsigned *ticket, int64_t i_begin, int64_t i_end, double factor,
                  int epilogue, PeerDst pd) {
  constexpr int PPW = 32 / LPP;
  // the chunk's scan has completed (stream order): re-arm its ticket for the next query
  if (ticket && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *ticket = 0u;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = i_begin + (int64_t)blockIdx.x * (8 * PPW) + (int64_t)w * PPW + lane / LPP;
  const int64_t c0 = (int64_t)blockIdx.y * (LPP * V6) + (int64_t)(lane % LPP) * V6;
  if (i >= i_end || c0 >= m) {
    if constexpr (PUSH) __threadfence_system();
    return;
  }
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
  double val[V6];
#pragma unroll
  for (int q = 0; q < V6; ++q) val[q] = factor * acc[q];
  if (!first_chunk) {
#pragma unroll
    for (int q = 0; q < V6; ++q) val[q] += yp[q];
  }
  if (last_chunk && epilogue) {
    const double hi = hsum[i];
#pragma unroll
    for (int q = 0; q < V6; ++q) val[q] += fma(-hi, Sg[c0 + q], Sg[m + c0 + q]);  // g - h_i S
  }
  if constexpr (PUSH) {
    // last chunk: the finished partial row goes straight to its owner's inbox slot (peer
    // stores over NVLink, overlapping the rest of the grid's gathers), then a system fence so
    // the signal kernel's flag is ordered after every send
    if (last_chunk) {
      double *dp = peer_row(pd, i) + c0;
#pragma unroll
      for (int q = 0; q < V6; ++q) dp[q] = val[q];
      __threadfence_system();
      return;
    }
  }
#pragma unroll
  for (int q = 0; q < V6; ++q) yp[q] = val[q];
}

template <int V6, int LPP>
static void launch_acc_t(const QueryPlan &p, const uint32_t *rank, int64_t ldn, int64_t n,
                         const double *U, int64_t k_first, int64_t kcc, const double *hsum,
                         const double *Sg, double *Y, int64_t ldy, int64_t m, bool first,
                         bool last, unsigned *ticket, int64_t i0, int64_t i1, double factor,
                         bool epilogue, const PeerDst *pd, cudaStream_t s) {
  constexpr int PPB = 8 * (32 / LPP);
  dim3 grid((unsigned)((i1 - i0 + PPB - 1) / PPB), (unsigned)p.col_groups);
  if (pd && pd->world > 0 && last)
    k6_accumulate<V6, LPP, L1DM_ACC_UNR, true><<<grid, 256, 0, s>>>(
        rank, ldn, n, U, p.ldu, k_first, kcc, hsum, Sg, Y, ldy, m, first ? 1 : 0, 1, ticket, i0,
        i1, factor, epilogue ? 1 : 0, *pd);
  else
    k6_accumulate<V6, LPP, L1DM_ACC_UNR, false><<<grid, 256, 0, s>>>(
        rank, ldn, n, U, p.ldu, k_first, kcc, hsum, Sg, Y, ldy, m, first ? 1 : 0, last ? 1 : 0,
        ticket, i0, i1, factor, epilogue ? 1 : 0, PeerDst{});
}

void launch_accumulate(const QueryPlan &p, const uint32_t *rank, int64_t ldn, int64_t n,
                       const double *U, int64_t k_first, int64_t kcc, const double *hsum,
                       const double *Sg, double *Y, int64_t ldy, int64_t m, bool first_chunk,
                       bool last_chunk, unsigned *ticket, int64_t i0, int64_t i1,
                       cudaStream_t s, double factor, bool epilogue, const PeerDst *pd) {
  if (i1 <= i0) return;
#define L1DM_ACC(V, L)                                                                   \
  launch_acc_t<V, L>(p, rank, ldn, n, U, k_first, kcc, hsum, Sg, Y, ldy, m, first_chunk, \
                     last_chunk, ticket, i0, i1, factor, epilogue, pd, s)
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
