// l1dm_peer.cu — the cross-GPU sum of the partial Y_g over peer
// memory instead of NCCL.
//
// A = sum_k A^(k), so rank g's coordinate shard yields a partial Y_g and Y = sum_g Y_g.
// Rows are owned in contiguous blocks (owner o: [floor(o n / G), floor((o+1) n / G))).  Each
// rank's final query pass (k6_accumulate's last chunk, or k9_block_out in scatter mode) stores
// every finished partial row straight into its owner's inbox slot — peer stores over NVLink,
// overlapping the rest of the pass — and a one-warp kernel then raises the rank's arrival flag
// at every owner (system-scope release after a system fence).  The owner waits for all G
// arrivals, sums the G slots of its rows in fixed rank order (deterministic), and stores the
// reduced rows into each target's result buffer (the root for reduce, every rank for
// all-reduce), raising a second flag there; targets wait for all owners.  Waits are bounded
// (kSpinLimit polls, then the caller's timeout word is set and the result is invalid).
// Inboxes are double-buffered by epoch parity: rank g can only start query e+2's push after its
// reduce of e+1, which saw owner o's arrival for e+1 — issued after o's reduce of e finished
// reading the buffer that e+2 reuses.  Result buffers need no second copy: owner o stores e+1
// into target t only after t's arrival for e+1, which follows t's copy-out of e.
#include <cuda_runtime.h>

#include "l1dm_device.cuh"
#include "l1dm_internal.h"

namespace l1dm {
namespace {

__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u32(unsigned *p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Rows [i0, i1) of a locally computed partial (the modes whose final pass is not fused with the
// push: m = 1 scatter, runs) to their owners' slots; one thread per double.
__global__ void __launch_bounds__(256)
    k30_push_rows(const double *__restrict__ src, int64_t lds, int64_t m, int64_t i0, int64_t i1,
                  PeerDst pd) {
  const int64_t total = (i1 - i0) * m;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    const int64_t i = i0 + e / m, c = e - (e / m) * m;
    peer_row(pd, i)[c] = src[i * lds + c];
  }
  __threadfence_system();
}

struct FlagTab {
  unsigned *p[kMaxPeers];
};

// One warp: lane o raises flags[o][index] after a system-scope fence (every earlier kernel on
// this stream has completed; its peer stores were fenced at system scope by their threads).
__global__ void k31_peer_signal(FlagTab flags, int world, int index, unsigned epoch) {
  __threadfence_system();
  const int o = threadIdx.x;
  if (o < world) st_release_sys_u32(flags.p[o] + index, epoch);
}

__device__ __forceinline__ void wait_flags(const unsigned *flags, int count, unsigned epoch,
                                           unsigned *timeout) {
  // One bound for the whole wait (not per flag), and any waiter that sees the rank's timeout
  // word raised (by another CTA, or an earlier wait) gives up at once: a dead peer costs one
  // kSpinLimit, not one per CTA and flag.
  uint32_t spins = 0;
  for (int g = 0; g < count; ++g) {
    // epochs only grow: a flag already past this epoch (a fast peer's next query) counts
    while ((int)(ld_acquire_sys_u32(flags + g) - epoch) < 0) {
      if (++spins > kSpinLimit) {
        atomicOr(timeout, 1u);
        return;
      }
      if ((spins & 63u) == 0 && *(volatile unsigned *)timeout) return;
      if (spins > 16) __nanosleep(128);
    }
  }
}

struct TargetTab {
  double *p[kMaxPeers];
  int64_t ld[kMaxPeers];
};

// Owner side: all G arrivals, then the fixed-order sum of the G slots into every target.
__global__ void __launch_bounds__(256)
    k32_peer_reduce(const unsigned *__restrict__ flags, int world, unsigned epoch,
                    const double *__restrict__ inbox, int64_t rows, int64_t m, int64_t row0,
                    TargetTab tg, int ntargets, unsigned *timeout) {
  if (threadIdx.x == 0) wait_flags(flags, world, epoch, timeout);
  __syncthreads();
  const int64_t total = rows * m, slot = rows * m;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * 256) {
    double v = 0.0;
    for (int g = 0; g < world; ++g) v += __ldcv(inbox + g * slot + e);  // peers wrote it
    const int64_t r = e / m, c = e - (e / m) * m;
    for (int t = 0; t < ntargets; ++t) tg.p[t][(row0 + r) * tg.ld[t] + c] = v;
  }
  __threadfence_system();
}

__global__ void k33_peer_wait(const unsigned *flags, int count, unsigned epoch,
                              unsigned *timeout) {
  if (threadIdx.x == 0) wait_flags(flags, count, epoch, timeout);
}

int grid_for(int64_t elems) {
  int64_t b = (elems + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

void launch_push_rows(const double *src, int64_t lds, int64_t m, int64_t i0, int64_t i1,
                      const PeerDst &pd, cudaStream_t s) {
  if (i1 <= i0) return;
  k30_push_rows<<<grid_for((i1 - i0) * m), 256, 0, s>>>(src, lds, m, i0, i1, pd);
}

void launch_peer_signal(unsigned *const *flags, int world, int index, unsigned epoch,
                        cudaStream_t s) {
  FlagTab t{};
  for (int o = 0; o < world && o < kMaxPeers; ++o) t.p[o] = flags[o];
  k31_peer_signal<<<1, 32, 0, s>>>(t, world, index, epoch);
}

void launch_peer_reduce(const unsigned *flags, int world, unsigned epoch, const double *inbox,
                        int64_t rows, int64_t m, int64_t row0, double *const *targets,
                        const int64_t *ld_t, int ntargets, unsigned *timeout, cudaStream_t s) {
  TargetTab tg{};
  for (int t = 0; t < ntargets && t < kMaxPeers; ++t) {
    tg.p[t] = targets[t];
    tg.ld[t] = ld_t[t];
  }
  k32_peer_reduce<<<grid_for(rows * m), 256, 0, s>>>(flags, world, epoch, inbox, rows, m, row0,
                                                     tg, ntargets, timeout);
}

void launch_peer_wait(const unsigned *flags, int count, unsigned epoch, unsigned *timeout,
                      cudaStream_t s) {
  k33_peer_wait<<<1, 32, 0, s>>>(flags, count, epoch, timeout);
}

}  // namespace l1dm
