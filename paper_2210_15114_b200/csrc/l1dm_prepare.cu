// l1dm_prepare.cu — Alg. 1 "Preprocessing" on sm_100a.
//
// For every coordinate k of the shard: a STABLE ascending sort of x_{.k}
// producing sval[k][r] (T_k), perm[k][r] (the order pi^k) and
// rank[k][i] ("position of x_i(k) in the order of T_k").  Layout is
// coordinate-major with row stride ldn = round_up(n, 32) so every row is
// 128-byte aligned.
//
//   K0 keys      X (row-major) -> key[k][i] orderable u32, h[i] = sum_k x_ik (fp64),
//                non-finite flag.  Tiled smem transpose, coalesced both sides.
//   K1 hist      one read of the keys -> all four 8-bit digit histograms per segment.
//   K2 pass      onesweep LSD pass: warp multisplit ranking (8 ballots), per-digit
//                decoupled look-back across tiles (one 64-bit word per digit holds
//                flag | epoch | count), smem staging so the scatter is run-coalesced.
//                Passes whose digit is constant in every segment are skipped.
//                The last pass decodes sval, writes perm and scatters rank (K3 fused).
//   emit         identity tables when no pass is needed.
#include <cuda_runtime.h>

#include <cstdio>
#include <type_traits>

#include "l1dm_device.cuh"
#include "l1dm_internal.h"

namespace l1dm {

// ------------------------------------------------------------------ K0
constexpr int kT0Points = 64;
constexpr int kT0Coords = 32;

__global__ void __launch_bounds__(256)
    k0_keys(const float *__restrict__ X, int64_t n, int64_t ldx, int64_t k0, int64_t dl,
            int64_t ldn, uint32_t *__restrict__ key, double *__restrict__ hsum,
            unsigned *__restrict__ nonfinite) {
  __shared__ float tile[kT0Points][kT0Coords + 1];
  const int64_t i0 = (int64_t)blockIdx.x * kT0Points;
  const int tid = threadIdx.x;
  constexpr int PER = kT0Points * kT0Coords / 256;  // elements per thread per chunk
  // the next chunk's values are loaded into registers while the current one is written out
  float xr[PER];
  auto load = [&](int64_t kt) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + 256 * u;
      const int p = e / kT0Coords, c = e % kT0Coords;
      const int64_t i = i0 + p, k = kt + c;
      xr[u] = (i < n && k < dl) ? __ldg(X + i * ldx + k0 + k) : 0.0f;
    }
  };
  double hacc = 0.0;  // threads with (tid & 3) == 0: point i0 + tid / 4
  int bad = 0;
  load(0);
  for (int64_t kt = 0; kt < dl; kt += kT0Coords) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + 256 * u;
      if (!isfinite(xr[u])) bad = 1;
      tile[e / kT0Coords][e % kT0Coords] = xr[u];
    }
    __syncthreads();
    if (kt + kT0Coords < dl) load(kt + kT0Coords);
    {  // h_i: 4 threads per point, 8 coordinates each, then a fixed 2-level tree
      const int p = tid >> 2, q = tid & 3;
      double part = 0.0;
#pragma unroll
      for (int c = 0; c < kT0Coords / 4; ++c) part += (double)tile[p][q * (kT0Coords / 4) + c];
      part += __shfl_xor_sync(0xFFFFFFFFu, part, 1);
      part += __shfl_xor_sync(0xFFFFFFFFu, part, 2);
      hacc += part;  // (zero past dl and past n)
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + 256 * u;
      const int c = e / kT0Points, p = e % kT0Points;
      const int64_t i = i0 + p, k = kt + c;
      if (i < n && k < dl) key[k * ldn + i] = float_to_key(tile[p][c]);
    }
    __syncthreads();
  }
  if ((tid & 3) == 0 && i0 + (tid >> 2) < n) hsum[i0 + (tid >> 2)] = hacc;
  if (__syncthreads_or(bad) && tid == 0) atomicOr(nonfinite, 1u);
}

// K0 with 16-byte accesses (X rows 16-byte aligned at the shard's first coordinate, dl % 4 == 0):
// two float4 loads and two uint4 key stores per thread per 64 x 32 chunk instead of 8 + 8 scalar
// ones; the same h_i summation order as k0_keys.
__global__ void __launch_bounds__(256)
    k0_keys_v4(const float *__restrict__ X, int64_t n, int64_t ldx, int64_t k0, int64_t dl,
               int64_t ldn, uint32_t *__restrict__ key, double *__restrict__ hsum,
               unsigned *__restrict__ nonfinite) {
  __shared__ float tile[kT0Points][kT0Coords + 1];
  const int64_t i0 = (int64_t)blockIdx.x * kT0Points;
  const int tid = threadIdx.x;
  float4 xr[2];
  auto load = [&](int64_t kt) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = tid + 256 * u;
      const int p = e >> 3, q = e & 7;
      const int64_t i = i0 + p, k = kt + 4 * q;
      xr[u] = (i < n && k < dl) ? __ldcs(reinterpret_cast<const float4 *>(X + i * ldx + k0 + k))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  double hacc = 0.0;
  int bad = 0;
  load(0);
  for (int64_t kt = 0; kt < dl; kt += kT0Coords) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = tid + 256 * u;
      const int p = e >> 3, q = e & 7;
      const float v[4] = {xr[u].x, xr[u].y, xr[u].z, xr[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!isfinite(v[j])) bad = 1;
        tile[p][4 * q + j] = v[j];
      }
    }
    __syncthreads();
    if (kt + kT0Coords < dl) load(kt + kT0Coords);
    {  // h_i: 4 threads per point, 8 coordinates each, then a fixed 2-level tree (as k0_keys)
      const int p = tid >> 2, q = tid & 3;
      double part = 0.0;
#pragma unroll
      for (int c = 0; c < kT0Coords / 4; ++c) part += (double)tile[p][q * (kT0Coords / 4) + c];
      part += __shfl_xor_sync(0xFFFFFFFFu, part, 1);
      part += __shfl_xor_sync(0xFFFFFFFFu, part, 2);
      hacc += part;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = tid + 256 * u;
      const int c = e >> 4, pq = e & 15;
      const int64_t k = kt + c, i = i0 + 4 * pq;
      if (k >= dl) continue;
      uint32_t kv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) kv[j] = float_to_key(tile[4 * pq + j][c]);
      uint32_t *dst = key + k * ldn + i;
      if (i + 4 <= n) {
        __stcg(reinterpret_cast<uint4 *>(dst), make_uint4(kv[0], kv[1], kv[2], kv[3]));
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (i + j < n) dst[j] = kv[j];
      }
    }
    __syncthreads();
  }
  if ((tid & 3) == 0 && i0 + (tid >> 2) < n) hsum[i0 + (tid >> 2)] = hacc;
  if (__syncthreads_or(bad) && tid == 0) atomicOr(nonfinite, 1u);
}

void launch_keys(const float *X, int64_t n, int64_t ldx, int64_t k0, int64_t dl, int64_t ldn,
                 uint32_t *key, double *hsum, unsigned *nonfinite, cudaStream_t s) {
  dim3 grid((unsigned)((n + kT0Points - 1) / kT0Points));
  if (ldx % 4 == 0 && k0 % 4 == 0 && dl % 4 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0)
    k0_keys_v4<<<grid, 256, 0, s>>>(X, n, ldx, k0, dl, ldn, key, hsum, nonfinite);
  else
    k0_keys<<<grid, 256, 0, s>>>(X, n, ldx, k0, dl, ldn, key, hsum, nonfinite);
}

// ------------------------------------------------------------------ K1
__global__ void __launch_bounds__(256)
    k1_hist(const uint32_t *__restrict__ key, int64_t n, int64_t ldn,
            uint32_t *__restrict__ hist) {
  __shared__ uint32_t sh[4 * 256];
  const int tid = threadIdx.x;
  for (int b = tid; b < 1024; b += 256) sh[b] = 0;
  __syncthreads();
  const int64_t seg = blockIdx.y;
  const uint32_t *kp = key + seg * ldn;
  const int64_t r0 = (int64_t)blockIdx.x * kHistChunk;
  const int64_t r1 = (r0 + kHistChunk < n) ? r0 + kHistChunk : n;
  // r0 is a multiple of 4 and rows are 128-B aligned: vector body, scalar tail.
  const int64_t body = r0 + ((r1 - r0) & ~(int64_t)3);
  for (int64_t r = r0 + 4 * tid; r < body; r += 4 * 256) {
    const uint4 q = *reinterpret_cast<const uint4 *>(kp + r);
    const uint32_t v[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      atomicAdd(&sh[0 * 256 + (v[u] & 255u)], 1u);
      atomicAdd(&sh[1 * 256 + ((v[u] >> 8) & 255u)], 1u);
      atomicAdd(&sh[2 * 256 + ((v[u] >> 16) & 255u)], 1u);
      atomicAdd(&sh[3 * 256 + (v[u] >> 24)], 1u);
    }
  }
  for (int64_t r = body + tid; r < r1; r += 256) {
    const uint32_t v = kp[r];
    atomicAdd(&sh[0 * 256 + (v & 255u)], 1u);
    atomicAdd(&sh[1 * 256 + ((v >> 8) & 255u)], 1u);
    atomicAdd(&sh[2 * 256 + ((v >> 16) & 255u)], 1u);
    atomicAdd(&sh[3 * 256 + (v >> 24)], 1u);
  }
  __syncthreads();
  for (int b = tid; b < 1024; b += 256)
    if (sh[b]) atomicAdd(&hist[seg * 1024 + b], sh[b]);
}

void launch_hist(const uint32_t *key, int64_t n, int64_t ldn, int64_t dl, uint32_t *hist,
                 cudaStream_t s) {
  dim3 grid((unsigned)((n + kHistChunk - 1) / kHistChunk), (unsigned)dl);
  k1_hist<<<grid, 256, 0, s>>>(key, n, ldn, hist);
}

// Digit bases on the device: per (segment k, pass p) the exclusive scan of the 256-bin histogram
// -> dbase[(p dl + k) 256 + b] (the layout k2_pass reads), and ntrivial[p] += 1 when the digit
// is constant over the segment (some bin holds all n keys).  The host reads back four words.
__global__ void __launch_bounds__(256)
    k1b_digit_base(const uint32_t *__restrict__ hist, int64_t n, int64_t dl,
                   uint32_t *__restrict__ dbase, unsigned *__restrict__ ntrivial) {
  const int64_t k = blockIdx.x;
  const int p = blockIdx.y, b = threadIdx.x, lane = b & 31, w = b >> 5;
  const uint32_t c = hist[k * 1024 + p * 256 + b];
  uint32_t incl = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, off);
    if (lane >= off) incl += y;
  }
  __shared__ uint32_t s_w[8];
  if (lane == 31) s_w[w] = incl;
  const int triv = __syncthreads_or(c == (uint32_t)n);
  uint32_t pre = 0;
  for (int ww = 0; ww < w; ++ww) pre += s_w[ww];
  dbase[((int64_t)p * dl + k) * 256 + b] = pre + incl - c;
  if (b == 0 && triv) atomicAdd(ntrivial + p, 1u);
}

void launch_digit_base(const uint32_t *hist, int64_t n, int64_t dl, uint32_t *dbase,
                       unsigned *ntrivial, cudaStream_t s) {
  k1b_digit_base<<<dim3((unsigned)dl, 4), 256, 0, s>>>(hist, n, dl, dbase, ntrivial);
}

// ------------------------------------------------------------------ K2
#ifdef L1DM_SORT_PROF
// debug build only: per-phase SM cycles of k2_pass summed over CTAs (thread 0's view)
__device__ unsigned long long g_sort_prof[8];
#define SORT_T(k)                                                        \
  do {                                                                   \
    if (threadIdx.x == 0) {                                              \
      const long long now = clock64();                                   \
      atomicAdd(&g_sort_prof[k], (unsigned long long)(now - prof_last)); \
      prof_last = now;                                                   \
    }                                                                    \
  } while (0)
__global__ void k_sort_prof_print() {
  printf("[sort prof] ticket %llu load+ballots %llu chain %llu digits+lookback %llu scan %llu "
         "stage %llu scatter %llu\n",
         g_sort_prof[0], g_sort_prof[1], g_sort_prof[2], g_sort_prof[3], g_sort_prof[4],
         g_sort_prof[5], g_sort_prof[6]);
  for (int i = 0; i < 8; ++i) g_sort_prof[i] = 0;
}
void sort_prof_print(cudaStream_t s) { k_sort_prof_print<<<1, 1, 0, s>>>(); }
#else
#define SORT_T(k) \
  do {            \
  } while (0)
void sort_prof_print(cudaStream_t) {}
#endif

// Status word per (segment, tile, digit): [63:62] flag, [61:32] epoch (30 bits), [31:0] count.
__device__ __forceinline__ unsigned long long pack_status(uint32_t flag, uint32_t epoch,
                                                          uint32_t cnt) {
  return ((unsigned long long)flag << 62) |
         ((unsigned long long)(epoch & 0x3FFFFFFFu) << 32) | (unsigned long long)cnt;
}

#if L1DM_SORT_TMA
// thread 0 of a sort CTA: tile t's keys (and values unless vin is null) into dst by 1-D bulk
// copies completing on bar.  Out of line: inlined into k2_pass, ptxas (12.9) fails register
// allocation ("register count of 7": the predicate file) under the ballot loop's pressure.
__device__ __noinline__ void sort_tile_bulk_load(const uint32_t *kin, const uint32_t *vin,
                                                 uint32_t *dst, uint64_t *bar, int64_t t,
                                                 int64_t nseg, int64_t ldn) {
  const int64_t tile = t / nseg, seg = t - tile * nseg;
  const int64_t base = tile * kSortTile, off = seg * ldn + base;
  const unsigned bytes = 4u * (unsigned)(ldn - base < kSortTile ? ldn - base : kSortTile);
  mbar_expect_tx(bar, vin ? 2 * bytes : bytes);
  bulk_g2s(dst, kin + off, bytes, bar);
  if (vin) bulk_g2s(dst + kSortTile, vin + off, bytes, bar);
}
__device__ __noinline__ void sort_tile_wait(uint64_t *bar, unsigned parity) { mbar_wait(bar, parity); }
#endif

// Persistent onesweep pass: each CTA loops over tiles claimed by an atomic ticket, and the
// next tile's keys/values are already in flight (cp.async into the other half of a shared
// double buffer) while the current one is ranked, looked back and scattered — ncu/clock64
// showed the one-tile-per-CTA version spending ~4 of its ~12 us per tile waiting for the
// ticket and its loads.  A CTA claims tickets in increasing order and processes them in that
// order, so the smallest unfinished ticket always belongs to a tile being processed whose
// predecessors are done: the look-back waits cannot deadlock.
template <bool FIRST, bool LAST>
__global__ void __launch_bounds__(kSortThreads, L1DM_SORT_MINB)
    k2_pass(const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin,
            uint32_t *__restrict__ kout, uint32_t *__restrict__ vout, uint32_t *__restrict__ rank,
            int64_t n, int64_t ldn, int64_t nseg, int64_t tiles_per_seg, int shift,
            const uint32_t *__restrict__ digit_base, unsigned long long *status, uint32_t epoch,
            unsigned *ticket, unsigned *timeout_flag) {
  constexpr int W = kSortThreads / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t *s_in = reinterpret_cast<uint32_t *>(smem_raw);  // [2][2][kSortTile] keys | vals
  __shared__ uint32_t s_whist[W][256];   // per-warp digit counts, then warp-exclusive offsets
  __shared__ uint32_t s_gbase[256];      // segment-relative start of this tile's run of each
                                         // digit minus its tile-local start
                                         // (n < 2^32: every in-segment offset fits 32 bits)
  __shared__ uint32_t s_wsum[W];
  __shared__ unsigned s_tk[2];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t total = nseg * tiles_per_seg;
  // stage tile t (keys, and values unless FIRST) into half b of the input buffer
#if L1DM_SORT_TMA
  // one thread moves each contiguous key / value tile with a 1-D bulk copy (TMA engine) that
  // completes on the half's mbarrier; rows are padded to ldn (a multiple of 32 keys), so every
  // copy is a multiple of 128 bytes from a 128-byte aligned address
  __shared__ uint64_t s_bar[2];
  uint32_t phase = 0;  // bit b: parity of the next completion of half b
  auto issue = [&](int64_t t, int b) {
    unsigned tx;  // %tid.x re-read here: a predicate held across the loop exhausts the file
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tx));
    if (tx == 0 && t < total)
      sort_tile_bulk_load(kin, FIRST ? nullptr : vin, s_in + (size_t)b * 2 * kSortTile, &s_bar[b],
                          t, nseg, ldn);
  };
#else
  auto issue = [&](int64_t t, int b) {
    if (t < total) {
      const int64_t tile = t / nseg, seg = t - (t / nseg) * nseg;
      const int64_t base = tile * kSortTile, off = seg * ldn + base;
      uint32_t *dk = s_in + (size_t)b * 2 * kSortTile, *dv = dk + kSortTile;
      for (int c = tid; c < kSortTile / 4; c += kSortThreads) {
        const bool ok = base + 4 * c < ldn;  // rows are padded to ldn (multiple of 32)
        cp_async<16>(dk + 4 * c, ok ? (const void *)(kin + off + 4 * c) : (const void *)kin, ok);
        if (!FIRST)
          cp_async<16>(dv + 4 * c, ok ? (const void *)(vin + off + 4 * c) : (const void *)vin, ok);
      }
    }
    cp_async_commit();  // (an empty group past the last ticket keeps the group count uniform)
  };
#endif
  if (tid == 0) {
#if L1DM_SORT_TMA
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init_fence();
#endif
    s_tk[0] = atomicAdd(ticket, 1u);
    s_tk[1] = atomicAdd(ticket, 1u);
  }
  __syncthreads();
  int64_t t_cur = s_tk[0], t_nxt = s_tk[1];
  issue(t_cur, 0);
  issue(t_nxt, 1);
  int cur = 0;
#ifdef L1DM_SORT_PROF
  long long prof_last = clock64();
#endif
  while (t_cur < total) {
#if L1DM_SORT_TMA
    sort_tile_wait(&s_bar[cur], (phase >> cur) & 1u);  // t_cur's tile (t_nxt's may be in flight)
    phase ^= 1u << cur;
#else
    cp_async_wait_group<1>();  // t_cur's group (t_nxt's may still be in flight)
#endif
    for (int b = tid; b < W * 256; b += kSortThreads) (&s_whist[0][0])[b] = 0;
    __syncthreads();
    SORT_T(0);
    const int64_t tile = t_cur / nseg;
    const int64_t seg = t_cur - tile * nseg;
    const int64_t base = tile * kSortTile;
    const int64_t seg_off = seg * ldn;
    const int tile_valid = (int)((n - base < kSortTile) ? (n - base) : kSortTile);
    // 32-bit tile-local indices from here on (the pass is instruction-bound: ncu shows the SM
    // issuing integer ALU most of the time, so 64-bit index arithmetic per key is not free)
    const uint32_t base32 = (uint32_t)base;

    // the digit-ordered stage: the input half this tile was loaded from (free once every thread
    // holds its items in registers)
    uint32_t *s_keys = s_in + (size_t)cur * 2 * kSortTile, *s_vals = s_keys + kSortTile;
    // the tile body, specialised for full tiles (no per-item validity tests: only the last tile
    // of a segment is partial)
    auto tile_body = [&](auto full_c) {
    constexpr bool FULL = decltype(full_c)::value;
    // ---- items (warp-striped: warp w owns [w*32*ITEMS, (w+1)*32*ITEMS), item j at +j*32+lane)
    uint32_t keys[kSortItems];
    uint32_t vals[kSortItems];
    uint16_t lrank[kSortItems];
    const int wbase = w * 32 * kSortItems;
    {
      const uint32_t *sk = s_in + (size_t)cur * 2 * kSortTile, *sv = sk + kSortTile;
#pragma unroll
      for (int j = 0; j < kSortItems; ++j) {
        const int e = wbase + j * 32 + lane;
        const bool valid = FULL || e < tile_valid;
        keys[j] = valid ? sk[e] : 0u;
        vals[j] = FIRST ? base32 + (uint32_t)e : (valid ? sv[e] : 0u);
      }
    }
    // ---- warp multisplit: stable rank of each key among equal digits of its warp
    const uint32_t lt = lanemask_lt();
    // lanes holding the same digit: 8 ballots (one per digit bit) — MATCH.ANY's latency made it
    // the top stall of this kernel on sm_100a (ncu short_scoreboard).  The ballots of all items
    // are independent (issued back to back); only the per-warp digit counters form a chain.
    uint32_t peers[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const bool valid = FULL || wbase + j * 32 + lane < tile_valid;
      const uint32_t dgt = (keys[j] >> shift) & 255u;
#ifdef L1DM_SORT_MATCH
      // invalid lanes match only themselves (256 + lane is no digit)
      const uint32_t pm = __match_any_sync(0xFFFFFFFFu, valid ? dgt : 256u + lane);
#else
      uint32_t pm = FULL ? 0xFFFFFFFFu : __ballot_sync(0xFFFFFFFFu, valid);
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        // one LOP3 to a predicate, the vote, a select and a 3-input LOP3 per bit
        uint32_t bal, m;
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
            "and.b32 t, %2, %3;\n\tsetp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\tselp.b32 %1, 0, 0xffffffff, p;\n\t}"
            : "=r"(bal), "=r"(m)
            : "r"(dgt), "r"(1u << b));
        pm &= bal ^ m;
      }
#endif
      peers[j] = valid ? pm : 0u;
    }
    SORT_T(1);
    // the leader of each digit group bumps the warp's counter; one full-warp shuffle hands
    // every lane its leader's old count (a shuffle per peer-group mask would serialise groups)
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const uint32_t pm = peers[j];
      const int leader = (FULL || pm) ? __ffs(pm) - 1 : lane;
      uint32_t old = 0;
      if ((FULL || pm) && lane == leader)
        old = atomicAdd(&s_whist[w][(keys[j] >> shift) & 255u], (uint32_t)__popc(pm));
      old = __shfl_sync(0xFFFFFFFFu, old, leader);
      lrank[j] = (uint16_t)(old + __popc(pm & lt));
    }
    __syncthreads();  // every thread has its items: half `cur` is free for the tile after next
    SORT_T(2);

    // ---- per digit (thread d): warp-exclusive offsets and the tile count
    const int dgt = tid;  // kSortThreads == 256 digits
    uint32_t cnt = 0;
#pragma unroll
    for (int ww = 0; ww < W; ++ww) {
      const uint32_t c = s_whist[ww][dgt];
      s_whist[ww][dgt] = cnt;
      cnt += c;
    }
    // ---- decoupled look-back over earlier tiles of this segment, per digit
    unsigned long long *st = status + (seg * tiles_per_seg) * 256;
    uint64_t excl = 0;
    if (tile == 0) {
      st_relaxed_u64(&st[dgt], pack_status(kFlagInclusive, epoch, cnt));
    } else {
      st_relaxed_u64(&st[tile * 256 + dgt], pack_status(kFlagAggregate, epoch, cnt));
      // walk back from tile - 1, reading a window of kLB predecessors per round trip (the
      // reads are independent; they are consumed in order and the walk resumes at the first
      // one that is not published yet)
      constexpr int kLB = 4;
      int64_t j = tile - 1;
      uint32_t spins = 0;
      bool done = false;
      while (!done) {
        unsigned long long sv[kLB];
#pragma unroll
        for (int q = 0; q < kLB; ++q)
          sv[q] = (j - q >= 0) ? ld_relaxed_u64(&st[(j - q) * 256 + dgt])
                               : pack_status(kFlagInclusive, epoch, 0);  // before tile 0: empty
        int q = 0;
        for (; q < kLB; ++q) {
          const uint32_t f = (uint32_t)(sv[q] >> 62);
          const uint32_t ep = (uint32_t)(sv[q] >> 32) & 0x3FFFFFFFu;
          if (ep != (epoch & 0x3FFFFFFFu) || f == kFlagInvalid) break;
          excl += (uint32_t)sv[q];
          if (f == kFlagInclusive) {
            done = true;
            break;
          }
        }
        if (done) break;
        j -= q;
        if (q == 0) {  // the nearest unsummed predecessor is not published yet
          if (++spins > kSpinLimit) {
            atomicOr(timeout_flag, 1u);
            break;
          }
          if (spins > 64) __nanosleep(64);
        }
      }
      st_relaxed_u64(&st[tile * 256 + dgt], pack_status(kFlagInclusive, epoch,
                                                        (uint32_t)(excl + cnt)));
    }
    const uint32_t gb = digit_base[seg * 256 + dgt] + (uint32_t)excl;
    SORT_T(3);

    // ---- block exclusive scan of the tile's digit counts -> the tile start of each digit
    uint32_t incl_scan = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl_scan, off);
      if (lane >= off) incl_scan += y;
    }
    if (lane == 31) s_wsum[w] = incl_scan;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int ww = 0; ww < W; ++ww)
      if (ww < w) wpre += s_wsum[ww];
    // fold the tile start into this digit's per-warp offsets (staging: one shared load per key)
    // and into the global base (scatter: gpos = s_gbase[d] + e, modulo 2^32)
    const uint32_t ts = wpre + incl_scan - cnt;
#pragma unroll
    for (int ww = 0; ww < W; ++ww) s_whist[ww][dgt] += ts;
    s_gbase[dgt] = gb - ts;
    __syncthreads();
    SORT_T(4);

    // ---- stage the tile in digit order (stable: warp order, then item, then lane)
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const int idx = wbase + j * 32 + lane;
      if (FULL || idx < tile_valid) {
        const uint32_t d = (keys[j] >> shift) & 255u;
        const uint32_t lp = s_whist[w][d] + lrank[j];
        s_keys[lp] = keys[j];
        s_vals[lp] = vals[j];
      }
    }
    __syncthreads();
    SORT_T(5);
    };
    if (tile_valid == kSortTile)
      tile_body(std::true_type{});
    else
      tile_body(std::false_type{});

    // ---- scatter: consecutive e inside a digit run go to consecutive global slots
    {
      uint32_t *ko = kout + seg_off, *vo = vout + seg_off;
      uint32_t *ro = rank ? rank + seg_off : nullptr;
      // opaque segment pointers: each store address is then one IMAD.WIDE.U32 of the 32-bit
      // slot (ncu: the compiler otherwise re-derived seg * ldn + gpos in 64 bits per store)
      asm("" : "+l"(ko), "+l"(vo));
#pragma unroll 4
      for (int e = tid; e < tile_valid; e += kSortThreads) {
        const uint32_t k = s_keys[e];
        const uint32_t v = s_vals[e];
        const uint32_t d = (k >> shift) & 255u;
        const uint32_t gpos = s_gbase[d] + (uint32_t)e;
        if (LAST) {
          st_global_u32(ko + gpos, __float_as_uint(key_to_float(k)));  // sval
          st_global_u32(vo + gpos, v);                                 // perm
          if (ro) ro[v] = gpos;                         // rank = perm^-1 (K3 fused)
        } else {
          st_global_u32(ko + gpos, k);
          st_global_u32(vo + gpos, v);
        }
      }
    }
    SORT_T(6);
    // claim the tile after next only now: a CTA holds at most two tickets (the one it works on
    // and the one in flight), which keeps the tiles a look-back may wait for close behind
    // (claiming it at the top of the tile, to hide the atomic's latency, measured 1% slower)
    if (tid == 0) s_tk[0] = atomicAdd(ticket, 1u);
#if L1DM_SORT_TMA
    fence_proxy_async_smem();  // this thread's reads of half `cur` before the bulk copy into it
#endif
    __syncthreads();  // s_keys / s_vals / s_gbase are reused by the next tile
    const int64_t t_nn = s_tk[0];
    issue(t_nn, cur);
    t_cur = t_nxt;
    t_nxt = t_nn;
    cur ^= 1;
  }
#if !L1DM_SORT_TMA
  cp_async_wait_all();
#endif
}

void launch_sort_pass(bool first, bool last, const uint32_t *kin, const uint32_t *vin,
                      uint32_t *kout, uint32_t *vout, uint32_t *rank, int64_t n, int64_t ldn,
                      int64_t dl, int shift, const uint32_t *digit_base,
                      unsigned long long *status, uint32_t epoch, unsigned *ticket,
                      unsigned *timeout_flag, cudaStream_t s) {
  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  // persistent grid: every CTA resident (the look-back needs no more), at most one per tile
  static int ctas = 0;
  const size_t smem = (size_t)4 * kSortTile * sizeof(uint32_t);  // 2 halves x (keys | vals)
  if (!ctas) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k2_pass<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k2_pass<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k2_pass<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k2_pass<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k2_pass<false, false>, kSortThreads, smem);
    ctas = sms * (per > 0 ? per : 1);
  }
  const int64_t work = tiles * dl;
  dim3 grid((unsigned)(work < ctas ? work : ctas));
#define L1DM_PASS(F, L)                                                                     \
  k2_pass<F, L><<<grid, kSortThreads, smem, s>>>(kin, vin, kout, vout, rank, n, ldn, dl, tiles, \
                                                 shift, digit_base, status, epoch, ticket,   \
                                                 timeout_flag)
  if (first && last)
    L1DM_PASS(true, true);
  else if (first)
    L1DM_PASS(true, false);
  else if (last)
    L1DM_PASS(false, true);
  else
    L1DM_PASS(false, false);
#undef L1DM_PASS
}

// ------------------------------------------------------------------ K3 rank
// rank[k][perm[k][r]] = r.  Blocks are segment-major (x fastest), so the 4n-byte rank row of
// one coordinate is written while it is L2-resident and leaves L2 as whole sectors.
constexpr int kRankRows = 4096;
__global__ void __launch_bounds__(256)
    k3_rank(const uint32_t *__restrict__ perm, uint32_t *__restrict__ rank, int64_t n,
            int64_t ldn) {
  const int64_t seg = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * kRankRows;
  const uint32_t *pp = perm + seg * ldn;
  uint32_t *rp = rank + seg * ldn;
  // the perm stream must not evict the rank row being filled: a sector that leaves L2 before
  // its 8 words arrive costs a DRAM read-modify-write (ncu: 3x write amplification on c4)
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  for (int64_t r = r0 + 4 * threadIdx.x; r < r0 + kRankRows && r < n; r += 4 * 256) {
    if (r + 4 <= n) {
      const uint4 q = ld_stream_u4_hint(pp + r, pol_stream);
      st_u32_hint(rp + q.x, (uint32_t)r, pol_keep);
      st_u32_hint(rp + q.y, (uint32_t)(r + 1), pol_keep);
      st_u32_hint(rp + q.z, (uint32_t)(r + 2), pol_keep);
      st_u32_hint(rp + q.w, (uint32_t)(r + 3), pol_keep);
    } else {
      for (int64_t u = r; u < n; ++u) rp[pp[u]] = (uint32_t)u;
    }
  }
}

void launch_rank(const uint32_t *perm, uint32_t *rank, int64_t n, int64_t ldn, int64_t dl,
                 cudaStream_t s) {
  dim3 grid((unsigned)((n + kRankRows - 1) / kRankRows), (unsigned)dl);
  k3_rank<<<grid, 256, 0, s>>>(perm, rank, n, ldn);
}

// ------------------------------------------------------------------ identity emit
__global__ void __launch_bounds__(256)
    k3_identity(const uint32_t *__restrict__ key, float *__restrict__ sval,
                uint32_t *__restrict__ perm, uint32_t *__restrict__ rank, int64_t n, int64_t ldn) {
  const int64_t seg = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
    sval[seg * ldn + i] = key_to_float(key[seg * ldn + i]);
    perm[seg * ldn + i] = (uint32_t)i;
    rank[seg * ldn + i] = (uint32_t)i;
  }
}

void launch_identity_emit(const uint32_t *key, float *sval, uint32_t *perm, uint32_t *rank,
                          int64_t n, int64_t ldn, int64_t dl, cudaStream_t s) {
  int64_t bx = (n + 255) / 256;
  if (bx > 4096) bx = 4096;
  dim3 grid((unsigned)bx, (unsigned)dl);
  k3_identity<<<grid, 256, 0, s>>>(key, sval, perm, rank, n, ldn);
}

// ------------------------------------------------------------------ runs (tie-heavy data)
// A coordinate whose sorted values take few distinct values (P:173 / P:205: ties) is also kept
// as runs: rvals[k][j] = the j-th distinct value (ascending), runid[k][i] = j for point i (u8,
// so at most 256 runs).  K_r1 counts run starts per 4096-row tile; the host turns the counts
// into per-tile offsets and decides (every coordinate needs <= 256 runs); K_r2 emits both.
constexpr int kRunTile = 4096;

// A thread's 16 consecutive sorted values of a 4096-row tile (four 16-byte loads; zero past n)
// and the value before its first row (the previous lane's last, the previous tile's last row for
// lane 0 of warp 0, a shared-memory hand-off between warps).
struct RunRows {
  uint32_t v[16];
  uint32_t prev;
};
__device__ __forceinline__ void load_run_rows(const float *v, int64_t n, int64_t r0, RunRows &o,
                                              uint32_t *s_last) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t rt = r0 + (int64_t)tid * 16;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t r = rt + 4 * q;
    if (r + 4 <= n) {  // rows are 128-byte aligned (ldn) and r is a multiple of 4
      const uint4 u = *reinterpret_cast<const uint4 *>(v + r);
      o.v[4 * q] = u.x;
      o.v[4 * q + 1] = u.y;
      o.v[4 * q + 2] = u.z;
      o.v[4 * q + 3] = u.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) o.v[4 * q + u] = r + u < n ? __float_as_uint(v[r + u]) : 0u;
    }
  }
  uint32_t p = __shfl_up_sync(0xFFFFFFFFu, o.v[15], 1);
  if (lane == 31) s_last[w] = o.v[15];
  __syncthreads();
  if (lane == 0) p = w > 0 ? s_last[w - 1] : (r0 > 0 ? __float_as_uint(v[r0 - 1]) : 0u);
  o.prev = p;
}

__global__ void __launch_bounds__(256)
    k_runs_count(const float *__restrict__ sval, int64_t n, int64_t ldn, int64_t tiles,
                 uint32_t *__restrict__ cnt) {
  static_assert(kRunTile == 256 * 16, "16 rows per thread");
  __shared__ uint32_t s_last[8], s_c[8];
  const int64_t seg = blockIdx.y, tile = blockIdx.x;
  const int64_t r0 = tile * kRunTile;
  RunRows rr;
  load_run_rows(sval + seg * ldn, n, r0, rr, s_last);
  const int64_t rt = r0 + (int64_t)threadIdx.x * 16;
  uint32_t c = 0, prev = rr.prev;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    c += (rt + j < n && (rt + j == 0 || rr.v[j] != prev)) ? 1u : 0u;
    prev = rr.v[j];
  }
  c = __reduce_add_sync(0xFFFFFFFFu, c);
  if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += s_c[w];
    cnt[seg * tiles + tile] = t;
  }
}

__global__ void __launch_bounds__(256)
    k_runs_emit(const float *__restrict__ sval, int64_t n, int64_t ldn, int64_t tiles,
                const uint32_t *__restrict__ tile_off, float *__restrict__ rvals) {
  __shared__ uint32_t s_last[8], s_w[8];
  const int64_t seg = blockIdx.y, tile = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t r0 = tile * kRunTile;
  RunRows rr;
  load_run_rows(sval + seg * ldn, n, r0, rr, s_last);
  const int64_t rt = r0 + (int64_t)tid * 16;
  uint32_t f = 0, cnt = 0, prev = rr.prev;  // f: bit j = row rt + j starts a run
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (rt + j < n && (rt + j == 0 || rr.v[j] != prev)) {
      f |= 1u << j;
      ++cnt;
    }
    prev = rr.v[j];
  }
  if (!__syncthreads_or(cnt)) return;  // no run starts in this tile
  uint32_t inc = cnt;  // block exclusive scan of the per-thread counts
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, off);
    if (lane >= off) inc += y;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  uint32_t run = tile_off[seg * tiles + tile] + inc - cnt;  // run starts before this thread
  for (int ww = 0; ww < w; ++ww) run += s_w[ww];
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (f & (1u << j)) rvals[seg * 256 + run++] = __uint_as_float(rr.v[j]);
}

// runid[k][i] = the index of x_ik among rvals[k][0..R_k) (binary search; -0.0 == +0.0 as in
// the sort's key canonicalisation).  Tiles of 64 points x 32 coordinates of X staged in shared
// memory (as K0), so X is read in whole rows and runid written in whole segments.
// grid (point blocks of kIdPoints, 32-coordinate chunks): a chunk's distinct values are staged
// once per CTA and serve kIdPoints / 64 point tiles (staging them per 64 points read 32 KB of
// L2 per 8 KB of X)
constexpr int kIdPoints = 1024;
__global__ void __launch_bounds__(256)
    k_runs_ids(const float *__restrict__ X, int64_t n, int64_t ldx, int64_t k0, int64_t dl,
               int64_t ldn, const float *__restrict__ rvals, const uint32_t *__restrict__ nruns,
               uint8_t *__restrict__ runid) {
  __shared__ float tile[kT0Points][kT0Coords + 1];
  // padded rows (one float per 32): the search's power-of-two strides spread over the banks
  __shared__ float s_vals[kT0Coords][256 + 8];
  __shared__ uint32_t s_nr[kT0Coords];
  const int tid = threadIdx.x;
  const int64_t kt = (int64_t)blockIdx.y * kT0Coords;
  for (int e = tid; e < kT0Coords * 256; e += 256) {
    const int c = e / 256, j = e % 256;
    s_vals[c][j + (j >> 5)] = (kt + c < dl) ? rvals[(kt + c) * 256 + j] : 0.0f;
  }
  if (tid < kT0Coords) s_nr[tid] = (kt + tid < dl) ? nruns[kt + tid] : 1u;
  for (int sub = 0; sub < kIdPoints / kT0Points; ++sub) {
    const int64_t i0 = (int64_t)blockIdx.x * kIdPoints + (int64_t)sub * kT0Points;
    if (i0 >= n) break;
    __syncthreads();
    for (int e = tid; e < kT0Points * kT0Coords; e += 256) {
      const int p = e / kT0Coords, c = e % kT0Coords;
      const int64_t i = i0 + p, k = kt + c;
      tile[p][c] = (i < n && k < dl) ? X[i * ldx + k0 + k] : 0.0f;
    }
    __syncthreads();
    // the largest j with rvals[j] <= x (== x: present): a fixed 8-step branchless search per
    // element, the 8 elements of a thread interleaved (independent shared-memory chains)
    constexpr int PE = kT0Points * kT0Coords / 256;
    float xs[PE];
    int pos[PE], nr[PE];
#pragma unroll
    for (int u = 0; u < PE; ++u) {
      const int e = tid + 256 * u;
      const int c = e / kT0Points, p = e % kT0Points;
      xs[u] = tile[p][c];
      nr[u] = (int)s_nr[c];
      pos[u] = 0;
    }
#pragma unroll
    for (int step = 128; step > 0; step >>= 1) {
#pragma unroll
      for (int u = 0; u < PE; ++u) {
        const int c = (tid + 256 * u) / kT0Points;
        const int t = pos[u] + step;
        if (t < nr[u] && s_vals[c][t + (t >> 5)] <= xs[u]) pos[u] = t;
      }
    }
#pragma unroll
    for (int u = 0; u < PE; ++u) {
      const int e = tid + 256 * u;
      const int c = e / kT0Points, p = e % kT0Points;
      const int64_t i = i0 + p, k = kt + c;
      if (i < n && k < dl) runid[k * ldn + i] = (uint8_t)pos[u];
    }
  }
}

// A cheap necessary test before the exact count: the distinct values among 4096 evenly spaced
// sorted positions of a coordinate are a subset of its distinct values, so more than 256 of them
// rules runs mode out for the shard (float data: one small kernel instead of a full read of
// sval).  flag |= 1 when some coordinate fails.
__global__ void __launch_bounds__(256)
    k_runs_sample(const float *__restrict__ sval, int64_t n, int64_t ldn,
                  unsigned *__restrict__ flag) {
  constexpr int S = 4096;
  const float *v = sval + (int64_t)blockIdx.x * ldn;
  uint32_t c = 0;
  for (int j = threadIdx.x; j < S; j += 256) {
    const int64_t r = (int64_t)j * n / S, rp = (int64_t)(j - 1) * n / S;
    c += (j == 0 || (r != rp && __float_as_uint(v[r]) != __float_as_uint(v[rp]))) ? 1u : 0u;
  }
  c = __reduce_add_sync(0xFFFFFFFFu, c);
  __shared__ uint32_t s_c[8];
  if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += s_c[w];
    if (t > 256) atomicOr(flag, 1u);
  }
}

void launch_runs_sample(const float *sval, int64_t n, int64_t ldn, int64_t dl, unsigned *flag,
                        cudaStream_t s) {
  k_runs_sample<<<(unsigned)dl, 256, 0, s>>>(sval, n, ldn, flag);
}

int64_t runs_tiles(int64_t n) { return (n + kRunTile - 1) / kRunTile; }

void launch_runs_count(const float *sval, int64_t n, int64_t ldn, int64_t dl, uint32_t *cnt,
                       cudaStream_t s) {
  dim3 grid((unsigned)runs_tiles(n), (unsigned)dl);
  k_runs_count<<<grid, 256, 0, s>>>(sval, n, ldn, runs_tiles(n), cnt);
}

void launch_runs_emit(const float *sval, int64_t n, int64_t ldn, int64_t dl,
                      const uint32_t *tile_off, float *rvals, cudaStream_t s) {
  dim3 grid((unsigned)runs_tiles(n), (unsigned)dl);
  k_runs_emit<<<grid, 256, 0, s>>>(sval, n, ldn, runs_tiles(n), tile_off, rvals);
}

void launch_runs_ids(const float *X, int64_t n, int64_t ldx, int64_t k0, int64_t dl, int64_t ldn,
                     const float *rvals, const uint32_t *nruns, uint8_t *runid, cudaStream_t s) {
  dim3 grid((unsigned)((n + kIdPoints - 1) / kIdPoints), (unsigned)((dl + kT0Coords - 1) / kT0Coords));
  k_runs_ids<<<grid, 256, 0, s>>>(X, n, ldx, k0, dl, ldn, rvals, nruns, runid);
}

}  // namespace l1dm
