// l1dm_internal.h — host-side declarations shared by the library's translation units.
// Product code only; never included by oracle/ (and vice versa).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace l1dm {

// Look-back flag states (low 2 bits of an epoch-tagged word).
constexpr uint32_t kFlagInvalid = 0;
constexpr uint32_t kFlagAggregate = 1;
constexpr uint32_t kFlagInclusive = 2;

// Spin bound for every look-back wait: after this many polls the waiter gives up,
// raises the handle's timeout flag and proceeds (results then invalid, status ETIMEOUT).
constexpr uint32_t kSpinLimit = 1u << 26;

// ---------------- prepare (Alg. 1) ----------------
constexpr int kSortThreads = 256;
#ifndef L1DM_SORT_ITEMS
#define L1DM_SORT_ITEMS 18  // keys per thread per onesweep tile (18 x 256 = 4608 with the bulk-copy loads: c3 prepare 3.59 -> 3.53 ms; 24 no longer fits ptxas at 2 CTAs/SM)
#endif
#ifndef L1DM_SORT_MINB
#define L1DM_SORT_MINB 2  // 2 CTAs per SM (104 KB of shared memory each); 3 x 4096-key tiles: c3 3.77 ms
#endif
#ifndef L1DM_SORT_TMA
#define L1DM_SORT_TMA 1  // tile loads by 1-D bulk copies (one thread, mbarrier) instead of cp.async
#endif
constexpr int kSortItems = L1DM_SORT_ITEMS;             // keys per thread per onesweep tile
constexpr int kSortTile = kSortThreads * kSortItems;    // 4608 keys
constexpr int kHistChunk = 16384;                       // keys per histogram CTA

void launch_keys(const float *X, int64_t n, int64_t ldx, int64_t k0, int64_t dl, int64_t ldn,
                 uint32_t *key, double *hsum, unsigned *nonfinite, cudaStream_t s);
// per (segment, pass): exclusive digit scan -> dbase (pass-major dl x 256 blocks); ntrivial[p]
// counts the segments whose pass-p digit is constant (zeroed by the caller)
void launch_digit_base(const uint32_t *hist, int64_t n, int64_t dl, uint32_t *dbase,
                       unsigned *ntrivial, cudaStream_t s);
void launch_hist(const uint32_t *key, int64_t n, int64_t ldn, int64_t dl, uint32_t *hist,
                 cudaStream_t s);
// One stable LSD pass over all dl segments.  first: values are implicit point indices.
// last: writes sval (decoded floats) to kout, perm to vout and rank[k][perm] = r.
void sort_prof_print(cudaStream_t s);  // debug builds (L1DM_SORT_PROF) only
void launch_sort_pass(bool first, bool last, const uint32_t *kin, const uint32_t *vin,
                      uint32_t *kout, uint32_t *vout, uint32_t *rank, int64_t n, int64_t ldn,
                      int64_t dl, int shift, const uint32_t *digit_base,
                      unsigned long long *status, uint32_t epoch, unsigned *ticket,
                      unsigned *timeout_flag, cudaStream_t s);
// rank[k][perm[k][r]] = r, segment-major (K3; used when the last pass does not scatter it).
void launch_rank(const uint32_t *perm, uint32_t *rank, int64_t n, int64_t ldn, int64_t dl,
                 cudaStream_t s);
// No pass needed (every digit constant in every segment): identity order.
void launch_identity_emit(const uint32_t *key, float *sval, uint32_t *perm, uint32_t *rank,
                          int64_t n, int64_t ldn, int64_t dl, cudaStream_t s);

// Runs of equal values (tie-heavy coordinates): run-start counts per 4096-row
// tile (cnt: dl x runs_tiles(n)); then, given exclusive per-tile offsets, runid[k][i] (u8,
// point order) and rvals[k][0..R_k) (the distinct values, ascending; R_k <= 256).
int64_t runs_tiles(int64_t n);
// flag |= 1 when some coordinate has > 256 distinct values among 4096 sampled sorted positions
void launch_runs_sample(const float *sval, int64_t n, int64_t ldn, int64_t dl, unsigned *flag,
                        cudaStream_t s);
void launch_runs_count(const float *sval, int64_t n, int64_t ldn, int64_t dl, uint32_t *cnt,
                       cudaStream_t s);
void launch_runs_emit(const float *sval, int64_t n, int64_t ldn, int64_t dl,
                      const uint32_t *tile_off, float *rvals, cudaStream_t s);
// runid[k][i] from X (point-major, the prepare's input) by binary search in rvals.
void launch_runs_ids(const float *X, int64_t n, int64_t ldx, int64_t k0, int64_t dl, int64_t ldn,
                     const float *rvals, const uint32_t *nruns, uint8_t *runid, cudaStream_t s);

// ---------------- query (Alg. 2) ----------------
// Rows per thread in a scan tile (8 warps, VC columns per lane): the tile stages about
// 96 KB of perm/sval/Z in shared memory, so two CTAs fit per SM.
#ifndef L1DM_M1_ITEMS
#define L1DM_M1_ITEMS 32
#endif
// Stage budget (bytes of gathered Z + sval + perm per tile).  Measured on B200 (c4, c3 gather,
// c5 gather): 64 KiB for one-row-per-warp-step tiles (lpr = 32: 3 CTAs per SM, fewer look-backs
// than 4 smaller CTAs), 96 KiB otherwise.
#ifndef L1DM_SCAN_SMEM
#define L1DM_SCAN_SMEM(lpr) ((lpr) == 32 ? 65536 : 98304)
#endif
#ifndef L1DM_RA_TILES
#define L1DM_RA_TILES 2  // 1024-row tiles per reduce-all CTA (a power of two <= 8)
#endif
#ifndef L1DM_ACC_UNR
#define L1DM_ACC_UNR 8  // gather-mode accumulate: coordinates' rank + U loads in flight per lane
#endif
#ifndef L1DM_RUNS_KG
#define L1DM_RUNS_KG 96  // coordinates per run-histogram CTA (measured c5 step: kg 8 -> 32 cut 366 -> 303 ms; with 16 run ids in flight 32 -> 96: 273 -> 268 ms)
#endif
#ifndef L1DM_RUNS_COPIES
#define L1DM_RUNS_COPIES 1  // replicate narrow run tables for the histogram's reductions (runs_copies)
#endif
#ifndef L1DM_RUNS_UNR
#define L1DM_RUNS_UNR 16  // coordinates' run ids in flight per lane in the expansion (8.4 -> 5.2 ms)
#endif
#ifndef L1DM_M1_ROW_ITEMS
#define L1DM_M1_ROW_ITEMS 8  // m = 1 scan: consecutive rows per thread (tile = 256 x this); 8 measured best (c2: 16 -> 8 cut the scan 0.91 -> 0.72 ms)
#endif
#ifndef L1DM_M1_MINB
#define L1DM_M1_MINB 4
#endif
__host__ __device__ constexpr int scan_items(int lpr, int vc) {
  return (lpr == 1 && vc == 1) ? L1DM_M1_ROW_ITEMS : lpr == 1 ? L1DM_M1_ITEMS
                  : ((L1DM_SCAN_SMEM(lpr) / (1024 * vc + 2048 / lpr)) / 4 * 4 > 64
                         ? 64
                         : (L1DM_SCAN_SMEM(lpr) / (1024 * vc + 2048 / lpr)) / 4 * 4);
}
// Largest query workspace chunk (U + look-back state) in bytes.
constexpr size_t kMaxChunkBytes = (size_t)72 << 30;
// Independent (coordinate, column block) scan segments the planner aims for per chunk.
constexpr int64_t kScanTargetSegments = 0;
// Scatter mode for m > 1 (measured crossovers): a Y block plus its Z block
// (12 n mb bytes) may be up to this multiple of L2; mb = 4 only for m <= kScatterNarrowM; and
// n >= kScatterMinN (below it the per-block launches dominate).
constexpr double kScatterL2Fraction = 1.25;
constexpr int64_t kScatterNarrowM = 24;
constexpr int64_t kScatterMinN = 1 << 17;
struct QueryPlan {
  int vec;            // fp32 Z elements per cp.async gather chunk (1, 2, 4)
  int lpr;            // lanes per sorted row in the scan = columns per segment
  int vc;             // columns per lane (1, or 2 when 32 < m <= 64)
  int mb;             // columns per scan segment (= lpr * vc)
  int col_blocks;     // ceil(m / mb)
  int items;          // consecutive sorted rows per thread
  int rows_per_tile;  // 8 warps * (32/lpr) * items
  int64_t tiles_per_segment;
  int64_t kc;         // coordinates per chunk
  int64_t chunks;
  int l2_resident;
  int scatter;        // 1: scan adds 2U into Y with L2 atomics (Y block fits L2); 0: U + rank gather
  int64_t zt_floats;  // scatter with m > 1: column-block-major copy of Z (col_blocks x n x mb)
  int64_t ldu;        // U row length (doubles) = m
  size_t u_bytes;     // kc * n * ldu * 8
  size_t lb_slots;    // kc * col_blocks * tiles_per_segment
  size_t workspace_bytes;
  // accumulate kernel
  int v6;             // doubles per lane (1 or 2)
  int lpp;            // lanes per point
  int col_groups;     // grid.y of the accumulate kernel
};

// vec_cap: widest fp32 vector the caller's Z allows (4: 16-B aligned rows, 2: 8-B, 1).
// mode: 0 automatic, 1 gather (U + rank gather), 2 scatter (L2 atomics into Y).
bool make_plan(int64_t n, int64_t dl, int64_t m, int64_t l2_bytes, int64_t ws_limit,
               int vec_cap, int mode, QueryPlan *p);

// ---------------- peer-memory collective (l1dm_peer.cu) ----------------
// Row destinations of a rank's partial Y in the owners' inboxes: owner o holds rows
// [row0[o], row0[o+1]) and this rank's slot in o's inbox is slot[o] (mapped in this process;
// row stride ld = m).  world == 0: no push (the product writes its own Y).
constexpr int kMaxPeers = 16;
struct PeerDst {
  int world;
  int64_t ld;
  int64_t row0[kMaxPeers + 1];
  double *slot[kMaxPeers];
};
__device__ __forceinline__ double *peer_row(const PeerDst &d, int64_t i) {
  int o = (int)((i * d.world) / d.row0[d.world]);  // even split: within one of the owner
  if (o >= d.world) o = d.world - 1;
  while (o > 0 && d.row0[o] > i) --o;
  while (o + 1 < d.world && d.row0[o + 1] <= i) ++o;
  return d.slot[o] + (i - d.row0[o]) * d.ld;
}
// rows [row0[o], row0[o+1]) of n for o = 0..world-1: floor(o n / world)
inline int64_t peer_row0(int64_t n, int world, int o) { return (n * o) / world; }
// dst rows <- src rows [i0, i1) (m doubles each, src row stride lds) at their owners.
void launch_push_rows(const double *src, int64_t lds, int64_t m, int64_t i0, int64_t i1,
                      const PeerDst &pd, cudaStream_t s);
// flags[o][index] = epoch (system-scope release) for o = 0..world-1, after a system fence.
void launch_peer_signal(unsigned *const *flags, int world, int index, unsigned epoch,
                        cudaStream_t s);
// Owner side: wait for flags[0..world) == epoch (bounded; *timeout |= 1 on expiry), then
// out_t[(row0 + r) * ld_t + c] = sum_g slot_g[r][c] (g = 0..world-1, fixed order) for every
// target t (targets[t], ld_t; mapped peer memory or local), rows r < rows, c < m.
void launch_peer_reduce(const unsigned *flags, int world, unsigned epoch, const double *inbox,
                        int64_t rows, int64_t m, int64_t row0, double *const *targets,
                        const int64_t *ld_t, int ntargets, unsigned *timeout, cudaStream_t s);
// Wait until flags[0..count) == epoch (bounded; *timeout |= 1 on expiry).
void launch_peer_wait(const unsigned *flags, int count, unsigned epoch, unsigned *timeout,
                      cudaStream_t s);

// Scatter mode: Y[i][c] += g_c - h_i S_c.
void launch_epilogue(const double *hsum, const double *Sg, double *Y, int64_t ldy, int64_t i0,
                     int64_t i1, int64_t m, cudaStream_t s);
// S and g of mc columns from the scan's per-segment totals (coordinate rows of ld_seg doubles,
// (S, T) pairs per column): S_c = coordinate 0's S, g_c = sum_k T_kc.
void launch_totals(const double *segtot, int64_t ld_seg, int64_t dl, int64_t mc, double *S,
                   double *g, cudaStream_t s);
// Scatter mode, m > 1: Y[i][c] = Yt[i][c] + g_c - h_i S_c for points [i0, i1), mc columns
// (S == nullptr: Y[i][c] = Yt[i][c]).
void launch_block_out(const double *yt, int mb, int64_t mc, const double *hsum, const double *S,
                      const double *g, double *Y, int64_t ldy, int64_t i0, int64_t i1,
                      cudaStream_t s, const PeerDst *pd = nullptr, int64_t pc0 = 0,
                      const double *fx = nullptr);
// (pd: the rows go to their owners' inbox slots at column pc0 instead of Y.)
// segtot: per-coordinate rows of ld_seg doubles ((S, T) per column); zs: m == 1 only, kc x ldn
// floats (z in sorted order between the reduce and apply passes).
void launch_scan(const QueryPlan &p, const uint32_t *perm, const float *sval, int64_t ldn,
                 int64_t n, const float *Z, int64_t ldz, int64_t m, double *U, int64_t k_first,
                 int64_t kcc, uint32_t *flags, double *agg, double *incl, uint32_t epoch,
                 unsigned *ticket, unsigned *timeout_flag, double *segtot, int64_t ld_seg,
                 float *zs, cudaStream_t s);
// Column-block "seq" scan (k5_scan_seq; scatter mode for m > 1 and every odd lp > 1 query):
// one column block (mc <= mb columns of the compact Zt block) over kcc coordinates, as reduce /
// prefix / apply launches (agg: kcc x tiles x (lp+1) mb doubles; segtot rows of ld_seg doubles,
// (lp+1) moments per column).  Apply adds its per-row value into out[perm[r]][c] with fp64 L2
// reductions (store = false: the block accumulator Yt, ldo = mb) or stores it at out[r][c] in
// sorted order (store = true: the U workspace of gather mode, ldo = m).  rows_per_tile = 1024.
// phase: 0 reduce + prefix, 1 apply, 2 both.  lp in {1, 3, 5, 7}.
void launch_scan_seq(const QueryPlan &p, int lp, const uint32_t *perm, const float *sval,
                     int64_t ldn, int64_t n, const float *zt, int64_t mc, double *out,
                     int64_t ldo, bool store, int64_t kcc, double *agg, double *segtot,
                     int64_t ld_seg, int phase, cudaStream_t s, int64_t agg_ld = 0,
                     const double *fx = nullptr);
// (fx: lp = 1 apply in deterministic fixed point — out is an int64 block, fx = the block's
//  per-column scales 2^F_c.)
// fx[c] = 2^F_c, fx[m + c] = 2^-F_c for the query: F_c from a bound on column c of Yt (the
// column's |z| sum, from the nparts x m per-CTA partials launch_zt wrote, and the shard's |x|),
// every sum in a fixed order.
void launch_fx_scale(const double *part, int64_t nparts, int64_t m, const uint32_t *sval_bits,
                     int64_t ldn, int64_t n, int64_t dl, double *fx, cudaStream_t s);
// Single-pass P = 1 scatter apply of one column block (k5_scan_lb): the tile prefixes by a
// fixed-point decoupled look-back (lbst: kcc x tiles x 2 mb 16-byte words, zeroed once; epoch
// distinct per launch), reductions into the int64
// block accumulator yt at scales fx (2^F_c), fa = the look-back scales (rows of fa_ld doubles:
// 2^Fz, 2^-Fz, 2^Fv, 2^-Fv), segment totals of s and t into segtot (rows of ld_seg).
// Block write-out after k5_scan_lb (mb even): S and g of the block from segtot (rows of ld_seg,
// dl coordinates) stored to Sg[c] / Sg[m_all + c], Y rows [i0, i1) = Yt 2^-F + g - h S (or the
// owners' inbox rows with pd).
void launch_block_out_fx(const unsigned long long *yt, int mb, int64_t mc, const double *hsum,
                         const double *segtot, int64_t ld_seg, int64_t dl, double *Sg,
                         int64_t m_all, double *Y, int64_t ldy, int64_t i0, int64_t i1,
                         cudaStream_t s, const PeerDst *pd, int64_t pc0, const double *fx_inv);
int scan_lb_rows(int mb);  // rows per k5_scan_lb tile (lbst: kcc x ceil(n / rows) x 2 mb words)
void launch_scan_lb(int mb, const uint32_t *perm, const float *sval, int64_t ldn, int64_t n,
                    const float *zt, int64_t mc, unsigned long long *yt, int64_t kcc,
                    void *lbst, uint32_t epoch, unsigned *timeout_flag, const double *fx,
                    const double *fa, int64_t fa_ld, double *segtot, int64_t ld_seg,
                    cudaStream_t s, int lp = 1);
// (lp in {3, 5, 7}: (lp + 1) moments, yt points at a fp64 block accumulator, fx unused, fa rows
//  (2t, 2t + 1) = the scale of moment t and its inverse; segtot rows of ld_seg hold (lp + 1) mc
//  moments per coordinate; the totals' part of the value is added by launch_lp_totals_expand.)
bool scan_lb_supported(int mb, int lp);
// Odd p in one pass: Y -= E, E_ic = sum_k sum_t C(p,t) (-1)^t x_ik^(p-t) T_ktc from the apply's
// segment totals (segtot rows of ld_seg, (p+1) moments per column) and X in point order (n x dl,
// row stride ldx); work: lp_totals_workspace bytes.  Returns the kernels launched.
size_t lp_totals_workspace(int64_t dl, int64_t m, int p);
int launch_lp_totals_expand(const float *X, int64_t ldx, int64_t n, int64_t dl, int64_t m,
                            const double *segtot, int64_t ld_seg, int p, double *work, double *Y,
                            int64_t ldy, cudaStream_t s);
// X in point order from the sorted tables: xr[perm[k][r] * dl + k] = sval[k][r] (once per handle).
void launch_unsort(const uint32_t *perm, const float *sval, int64_t ldn, int64_t n, int64_t dl,
                   float *xr, cudaStream_t s);
// Look-back scales of (lp + 1) moments per column (fa rows 2t, 2t + 1: 2^F_t and 2^-F_t, F_t from
// the bound max_k Mx_k^t sum_i |z_ic| < 2^58), from launch_zt's |z| partials.
void launch_lb_scales(const double *part, int64_t nparts, int64_t m, const uint32_t *sval_bits,
                      int64_t ldn, int64_t n, int64_t dl, int lp, double *fa, cudaStream_t s);
// (agg_ld: the apply's stride between tiles in agg, 0 = the block's own payload (lp+1) mb.)
// P = 1, m <= 256: tile totals of all m columns in one pass over full Z rows + the prefix
// (agg: kcc x tiles x 2m, segtot rows of 2m).  The per-block apply then reads agg + 2 c0 with
// agg_ld = 2m.  Returns false (nothing launched) for m > 256.
bool launch_reduce_all(const uint32_t *perm, const float *sval, int64_t ldn, int64_t n,
                       const float *Z, int64_t ldz, int64_t m, int64_t kcc, int64_t tiles_per_seg,
                       double *agg, double *segtot, cudaStream_t s);
// Zt[cb][i][0..mb) = Z[i][cb*mb + ..] (zero-padded past m): the scatter mode's per-block Z.
// With colabs_part (zt_max_ctas(m, mb) x m doubles) also the per-CTA column sums of |z| for
// launch_fx_scale; returns the number of CTAs (partials).
int64_t launch_zt(const float *Z, int64_t ldz, int64_t n, int64_t m, int mb, float *zt,
                  cudaStream_t s, double *colabs_part = nullptr);
int64_t zt_max_ctas(int64_t m, int mb);
void launch_accumulate(const QueryPlan &p, const uint32_t *rank, int64_t ldn, int64_t n,
                       const double *U, int64_t k_first, int64_t kcc, const double *hsum,
                       const double *Sg, double *Y, int64_t ldy, int64_t m, bool first_chunk,
                       bool last_chunk, unsigned *ticket, int64_t i0, int64_t i1,
                       cudaStream_t s, double factor = 2.0,
                       bool epilogue = true,   // points [i0, i1); Y (+)= factor * sum_k U (+ g - h S)
                       const PeerDst *pd = nullptr);  // last chunk: rows to their owners' slots
// l_p^p, odd p in {3, 5, 7}: plan over the seq kernels.
bool make_lp_plan(int64_t n, int64_t dl, int64_t m, int lp, int64_t l2_bytes, int64_t ws_limit,
                  int mode, QueryPlan *p);
// Runs mode.  phase 0: H (dl x 256 x m, zeroed here) <- run sums of Z, then U
// in place and segtot (rows of 2m: S, T_k); phase 1: Y = 2 sum_k U[k][runid] + g - h S with
// Sg = (S, g) from launch_totals.
int runs_copies(int64_t dl, int64_t m);  // replicas of the [dl][256][m] run table the histogram needs
void launch_runs_query(const uint8_t *runid, int64_t ldn, int64_t n, int64_t dl, const float *rvals,
                       const uint32_t *nruns, const float *Z, int64_t ldz, int64_t m, double *H,
                       double *segtot, const double *hsum, double *Sg, double *Y, int64_t ldy,
                       int phase, cudaStream_t s, int64_t i0 = 0, int64_t i1 = -1);
// Runs mode for odd p in {3, 5, 7}: Y = sum_k W^k[runid_k(i)] with W^k the whole per-run
// l_p^p term (histogram, p-moment scan over runs, expansion); H: dl x 256 x m fp64 scratch.
void launch_runs_lp(const uint8_t *runid, int64_t ldn, int64_t n, int64_t dl, const float *rvals,
                    const uint32_t *nruns, const float *Z, int64_t ldz, int64_t m, int lp,
                    double *H, double *Y, int64_t ldy, int phase, cudaStream_t s);
// (phase 0: histogram + p-moment scan; phase 1: expansion.)
// Y (row-major, ldy) <- Yb (column-block-major blocks of n x mb).
void launch_unblock(const double *Yb, int64_t n, int64_t m, int64_t mb, double *Y, int64_t ldy,
                    cudaStream_t s);
// Y[i][c] *= a over n x m.
void launch_scale(double *Y, int64_t ldy, int64_t n, int64_t m, double a, cudaStream_t s);
// out[0] = max_i |h_i - 1|, out[1] = min over every prepared coordinate value (device doubles).
void launch_simplex_stats(const double *hsum, int64_t n, const float *sval, int64_t ldn,
                          int64_t dl, double *out, cudaStream_t s);

// ---------------- sort-free products (l1dm_sortfree.cu, NEXT-4) ----------------
// Even p in {2, 4, 6}: Y = A_p Z with (A_p)_ij = ||x_i - x_j||_p^p, no preprocessing.
// ws: lpp_even_workspace() bytes of device memory.
size_t lpp_even_workspace(int64_t n, int64_t d, int64_t m, int p, int64_t *nchunks_out,
                          int64_t *chunk_out, int sms);
int launch_lpp_even(const float *X, int64_t ldx, const float *Z, int64_t ldz, int64_t n,
                     int64_t d, int64_t m, int p, double *Y, int64_t ldy, double *ws, int sms,
                     cudaStream_t s);

// Thm. maha's bilinear form f(x, y) = x^T M y (M: d x d fp64 row-major, device): Y = X M X^T Z.
size_t bilinear_workspace(int64_t n, int64_t d, int64_t m, int sms);
int launch_bilinear(const float *X, int64_t ldx, const double *M, const float *Z, int64_t ldz,
                     int64_t n, int64_t d, int64_t m, double *Y, int64_t ldy, double *ws, int sms,
                     cudaStream_t s);

// Thm. l2embed: Xp (n x k fp32, ldp) = X G^T / (beta k), beta = sqrt(2/pi); G: k x d fp32.
int launch_embed(const float *X, int64_t ldx, int64_t n, int64_t d, const float *G, int64_t ldg,
                  int64_t k, float *Xp, int64_t ldp, cudaStream_t s);

// ---------------- dense fp64 steps of the matrix-free consumers (l1dm_dense.cu, NEXT-2) ----
size_t gemm_workspace(int ta, int64_t M, int64_t N, int64_t K, int sms);
int launch_gemm(int ta, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                double *ws, int sms, cudaStream_t s);
size_t jacobi_workspace(int64_t N);
int launch_jacobi(int64_t N, double *A, int64_t lda, double *W, double *V, int64_t ldv,
                  double *ws, int sms, cudaStream_t s, int *stats = nullptr);
size_t topk_workspace(int64_t N);
int launch_sym_topk(int64_t N, const double *A, int64_t lda, int64_t k, double *lam,
                    double *sigma, double *Vs, double *ws, int sms, cudaStream_t s);
void launch_chol_orth(int64_t b, const double *G, int64_t ldg, const double *G0, int64_t ldg0,
                      double rtol, double floor_abs, double *S, cudaStream_t s);
void launch_select(int64_t N, int64_t k, const double *W, const double *V, int64_t ldv,
                   double *lam, double *sigma, double *Vs, int *order, cudaStream_t s);
void launch_scale_cols(int64_t b, const double *V, const double *lam, const double *G0,
                       int64_t ldg0, double rtol, double floor_abs, double *S, cudaStream_t s);
void launch_split_hilo(int64_t n, int64_t b, const double *V, int64_t ldv, float *Zs,
                       cudaStream_t s);
void launch_combine_hilo(int64_t n, int64_t b, const double *Yr, double *Y, int64_t ldy,
                         cudaStream_t s);
void launch_axpy2d(int64_t rows, int64_t cols, double alpha, const double *S, int64_t lds,
                   double *D, int64_t ldd, cudaStream_t s);
void launch_symmetrize(int64_t N, double *T, int64_t ldt, cudaStream_t s);
int cg_dot_blocks();
// CG device state: doubles [CG_CONV_INDEX] = converged flag, [CG_CONV_INDEX + 1] = iterations
constexpr int CG_CONV_INDEX = 6;
void launch_dot(int64_t n, const double *x, const double *y, double *part, cudaStream_t s);
void launch_cg_scalars(int phase, const double *part, double tol, double *st, cudaStream_t s);
void launch_cg_xr(int64_t n, const double *st, const double *p, const double *Ap, double *x,
                  double *r, cudaStream_t s);
void launch_cg_p(int64_t n, const double *st, const double *r, double *p, cudaStream_t s);
void launch_sub(int64_t n, const double *a, const double *b, double *d, cudaStream_t s);

}  // namespace l1dm
