// l1dm_api.cu — host runtime and the C ABI declared in include/l1dm.h.
//
// Owns the handle lifecycle, device buffers, the query planner, launch sequencing,
// host<->device staging for host pointers, per-kernel event timing and error mapping.
// Every compute step runs in the kernels of l1dm_prepare.cu / l1dm_query.cu; there
// is no host (CPU) evaluation path.
#include <atomic>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <map>
#include <mutex>
#include <unordered_map>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "l1dm.h"
#include "l1dm_internal.h"

using namespace l1dm;

namespace {

thread_local std::string g_err;

l1dm_status fail(l1dm_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      l1dm_status st_ = (e_ == cudaErrorMemoryAllocation) ? L1DM_ENOMEM : L1DM_ECUDA;         \
      return fail(st_, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__,      \
                  __LINE__);                                                                  \
    }                                                                                         \
  } while (0)

enum TimingKind { kPrep = 0, kColsums, kScan, kAcc, kCopy, kNumKinds };

struct TimedPair {
  int kind;
  cudaEvent_t a, b;
};

// Process-wide cache of device blocks released by handles (prepare transients, query
// workspace), so that successive handles — one per bench step, one per shard — reuse memory
// instead of paying cudaMalloc/cudaFree of tens of GB each time.  Blocks enter the cache only
// after their stream has been synchronised; a request takes the smallest cached block of at
// least the requested size (and at most 1.25x of it).  The cache holds at most half of the
// device memory, is flushed when an allocation fails, and l1dm_release_cached() empties it.
class BlockCache {
 public:
  static BlockCache &get() {
    static BlockCache c;
    return c;
  }
  static bool debug() {
    static const bool d = getenv("L1DM_DEBUG_ALLOC") != nullptr;
    return d;
  }
  cudaError_t alloc(void **p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    bytes = (bytes + ((size_t)2 << 20) - 1) & ~(((size_t)2 << 20) - 1);  // 2 MiB granules
    {
      std::lock_guard<std::mutex> g(mu_);
      auto &m = free_[dev];
      auto it = m.lower_bound(bytes);
      if (it != m.end() && it->first <= bytes + bytes / 4) {
        *p = it->second;
        sizes_[*p] = {it->first, dev};
        cached_[dev] -= it->first;
        m.erase(it);
        return cudaSuccess;
      }
    }
    const size_t rounded = bytes;
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMalloc(p, rounded);
    if (debug())
      fprintf(stderr, "[l1dm] cudaMalloc %zu B: %.3f ms\n", rounded,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count());
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      release_all(dev);
      cudaMemPool_t pool;  // and what the stream-ordered pool keeps (keep_default_pool)
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaDeviceSynchronize();
        cudaMemPoolTrimTo(pool, 0);
      }
      e = cudaMalloc(p, rounded);
    }
    if (e == cudaSuccess) {
      std::lock_guard<std::mutex> g(mu_);
      sizes_[*p] = {rounded, dev};
    }
    return e;
  }
  // p must not be in use by any queued work (callers synchronise first).  The block is filed
  // under the device it was allocated on (recorded at alloc), whatever device is current.
  void free(void *p) {
    if (!p) return;
    std::lock_guard<std::mutex> g(mu_);
    auto sz = sizes_.find(p);
    if (sz == sizes_.end()) {
      cudaFree(p);
      return;
    }
    const size_t bytes = sz->second.first;
    const int dev = sz->second.second;
    sizes_.erase(sz);
    if (limit_[dev] == 0) {
      int cur = 0;
      cudaGetDevice(&cur);
      if (cur != dev) cudaSetDevice(dev);
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      limit_[dev] = tot / 2;
      if (cur != dev) cudaSetDevice(cur);
    }
    if (cached_[dev] + bytes > limit_[dev]) {
      if (debug()) fprintf(stderr, "[l1dm] cache full: cudaFree %zu B\n", bytes);
      cudaFree(p);
      return;
    }
    free_[dev].emplace(bytes, p);
    cached_[dev] += bytes;
  }
  void release_all(int dev) {
    std::lock_guard<std::mutex> g(mu_);
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != dev && !free_[dev].empty()) cudaSetDevice(dev);
    for (auto &kv : free_[dev]) cudaFree(kv.second);
    if (cur != dev && !free_[dev].empty()) cudaSetDevice(cur);
    free_[dev].clear();
    cached_[dev] = 0;
  }
  size_t cached(int dev) {
    std::lock_guard<std::mutex> g(mu_);
    return cached_[dev];
  }

 private:
  std::mutex mu_;
  std::map<int, std::multimap<size_t, void *>> free_;
  std::map<int, size_t> cached_, limit_;
  std::unordered_map<void *, std::pair<size_t, int>> sizes_;  // block -> (bytes, device)
};

template <typename T>
struct DevBuf {
  T *p = nullptr;
  size_t count = 0;
  cudaStream_t s_last = nullptr;  // stream of the latest ensure (the block's user)
  DevBuf() = default;
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  // a block still held at scope exit (a function-local buffer, an early error return) goes
  // back to the cache once its stream is idle — never leaked, never reused while in use
  ~DevBuf() {
    if (p) {
      cudaStreamSynchronize(s_last);
      release();
    }
  }
  cudaError_t ensure(size_t c, bool zero, cudaStream_t s) {
    s_last = s;
    if (c <= count && p) return cudaSuccess;
    if (p) {
      if (BlockCache::debug()) fprintf(stderr, "[l1dm] grow %zu -> %zu elems (sync)\n", count, c);
      cudaStreamSynchronize(s);  // queued work on s may still use the old block
      BlockCache::get().free(p);
      p = nullptr;
      count = 0;
    }
    void *q = nullptr;
    cudaError_t e = BlockCache::get().alloc(&q, std::max<size_t>(c, 1) * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      return e;
    }
    p = static_cast<T *>(q);
    count = c;
    if (zero) return cudaMemsetAsync(p, 0, std::max<size_t>(c, 1) * sizeof(T), s);
    return cudaSuccess;
  }
  void release() {  // callers synchronise the streams that used the block first
    if (p) BlockCache::get().free(p);
    p = nullptr;
    count = 0;
  }
};

bool is_device_pointer(const void *ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();  // clear: unknown pointers are host memory
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

struct l1dm_ctx {
  int device = -1;
  int64_t n = 0, dl = 0, k_begin = 0, k_end = 0, ldn = 0;
  int64_t l2_bytes = 0;
  cudaStream_t stream = nullptr;       // prepare stream; default for l1dm_matvec
  cudaStream_t last_stream = nullptr;  // stream of the latest l1dm_matvec_ex
  bool own_stream = false;
  // prepared state (Alg. 1)
  DevBuf<uint32_t> sval_bits;  // fp32 bits
  DevBuf<uint32_t> perm;
  DevBuf<uint32_t> rank;
  DevBuf<double> hsum;
  // runs of equal values (every coordinate <= 256 distinct values)
  bool has_runs = false;
  bool rank_ready = false;  // rank = perm^-1 is built on first use (gather-mode queries only)
  DevBuf<uint8_t> runid;   // [dl][ldn] run index of point i
  DevBuf<float> rvals;     // [dl][256] distinct values, ascending
  DevBuf<uint32_t> nruns;  // [dl]
  DevBuf<double> rtab;     // [copies][dl][256][m] query table: H (replicas folded into the first), then U in place
  // query workspace
  DevBuf<double> U;
  DevBuf<uint32_t> flags;
  DevBuf<double> agg, incl;
  DevBuf<double> part, Sg;
  DevBuf<float> zs;            // m == 1: gathered z in sorted order (reduce -> apply pass)
  DevBuf<float> zt;            // scatter mode, m > 1: column-block-major copy of Z
  DevBuf<double> yt;           // scatter mode, m > 1: one column block's accumulator (n x mb)
  DevBuf<double> fxbuf;        // scatter mode, m > 1: fixed-point scales (6m) + their scratch
  DevBuf<unsigned long long> lbst;  // scatter mode, m > 1: single-pass apply look-back words
  DevBuf<float> xr;                 // X in point order (n x dl), built for odd-p single passes
  bool xr_ready = false;
  uint32_t lb_epoch = 0;            // k5_scan_lb launches (their words carry it mod 4)
  int64_t lb_geom = -1;             // slot geometry the words were written with
  DevBuf<unsigned> ctr;        // [0] colsum done counter, [1] timeout flag, [2..] scan tickets
  size_t ws_limit = 0;
  int mode = 0;  // L1DM_MODE_*
  bool full_rows = false;     // prepared coordinates are every coordinate of X's rows
  int simplex = -1;           // TV precondition, checked once: -1 unknown, 0 violated, 1 holds
  double simplex_dev = 0.0, simplex_min = 0.0;
  uint32_t epoch = 1;
  // host staging (synchronous path: pageable host buffers)
  DevBuf<float> Zstage;
  DevBuf<double> Ystage;
  DevBuf<double> ypush;  // peer push: the partial Y when the final pass is not fused (or chunked)
  // asynchronous pinned-host pipeline: two staging slots, H2D / D2H on their own streams so
  // query q's copies overlap query q-1's compute (DESIGN.md §7 e2e)
  DevBuf<float> Zpin[2];
  DevBuf<double> Ypin[2];
  cudaStream_t cp_in = nullptr, cp_out = nullptr;
  cudaEvent_t ev_in[2] = {}, ev_done[2] = {}, ev_out[2] = {};
  unsigned pin_slot = 0;
  // plan cache
  int64_t plan_m = -1;
  size_t plan_ws = 0;
  int plan_vec_cap = 0;
  size_t plan_ws_limit = 0;
  int plan_mode = -1;
  QueryPlan plan{};
  // timing
  bool timing = false;
  std::vector<TimedPair> pending;
  std::vector<cudaEvent_t> pool;
  double prep_ms = 0.0;
  double ms[kNumKinds] = {0, 0, 0, 0, 0};
  int64_t launches[kNumKinds] = {0, 0, 0, 0, 0};
  int64_t queries = 0;
  int64_t kernel_launches = 0;
  int64_t scan_pairs = 0, acc_pairs = 0, m_last = 0;
};

namespace {

cudaEvent_t take_event(l1dm_ctx *h) {
  if (!h->pool.empty()) {
    cudaEvent_t e = h->pool.back();
    h->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct TimedScope {
  l1dm_ctx *h;
  int kind;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  TimedScope(l1dm_ctx *h_, int kind_, cudaStream_t s_) : h(h_), kind(kind_), s(s_) {
    if (h->timing) {
      a = take_event(h);
      cudaEventRecord(a, s);
    }
  }
  ~TimedScope() {
    if (a) {
      cudaEvent_t b = take_event(h);
      cudaEventRecord(b, s);
      h->pending.push_back({kind, a, b});
    }
  }
};

// The device's default stream-ordered pool keeps freed memory (release threshold = max): with
// the default threshold of 0 every Krylov / CG call re-mapped its multi-GB basis (c3 top-16:
// ~80-120 ms of host-side cudaMallocAsync per call beside 480 ms of device work).
static void keep_default_pool() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

// NVTX range over an entry point (named ranges for profilers; header-only NVTX 3,
// a no-op unless a tool is attached).
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Makes h's device current for a scope (calls that only synchronise or release a handle's
// resources may come from a thread whose current device is another one).
struct DeviceGuard {
  int prev = -1, dev = -1;
  explicit DeviceGuard(int d) : dev(d) {
    cudaGetDevice(&prev);
    if (dev >= 0 && prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (dev >= 0 && prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};

l1dm_status check_device(l1dm_ctx *h) {
  int cur = -1;
  CUDA_TRY(cudaGetDevice(&cur));
  if (cur != h->device)
    return fail(L1DM_EDEVICE, "handle belongs to device %d but device %d is current", h->device,
                cur);
  return L1DM_OK;
}

l1dm_status check_arch(int *dev_out) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(L1DM_EDEVICE, "no CUDA device available (%s)",
                e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
  }
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  int major = 0, minor = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (major != 10 || minor != 0)
    return fail(L1DM_EDEVICE, "library is built for sm_100a only; device %d is sm_%d%d", dev, major,
                minor);
  *dev_out = dev;
  return L1DM_OK;
}

void destroy(l1dm_ctx *h) {
  if (!h) return;
  // a handle may be freed (or garbage-collected) while another device is current: every
  // stream, event and block below belongs to h->device
  int cur = -1;
  cudaGetDevice(&cur);
  if (h->device >= 0 && cur != h->device) cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  if (h->last_stream != h->stream) cudaStreamSynchronize(h->last_stream);
  for (auto &p : h->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : h->pool) cudaEventDestroy(e);
  h->sval_bits.release();
  h->perm.release();
  h->rank.release();
  h->runid.release();
  h->rvals.release();
  h->nruns.release();
  h->rtab.release();
  h->hsum.release();
  h->U.release();
  h->flags.release();
  h->agg.release();
  h->incl.release();
  h->part.release();
  h->Sg.release();
  h->ctr.release();
  if (h->cp_in) cudaStreamSynchronize(h->cp_in);
  if (h->cp_out) cudaStreamSynchronize(h->cp_out);
  h->Zstage.release();
  h->Ystage.release();
  h->ypush.release();
  for (int q = 0; q < 2; ++q) {
    h->Zpin[q].release();
    h->Ypin[q].release();
    for (cudaEvent_t e : {h->ev_in[q], h->ev_done[q], h->ev_out[q]})
      if (e) cudaEventDestroy(e);
  }
  if (h->cp_in) cudaStreamDestroy(h->cp_in);
  if (h->cp_out) cudaStreamDestroy(h->cp_out);
  h->zs.release();
  h->zt.release();
  h->yt.release();
  h->fxbuf.release();
  h->lbst.release();
  h->xr.release();
  h->lb_geom = -1;
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  const int hdev = h->device;
  delete h;
  if (hdev >= 0 && cur >= 0 && cur != hdev) cudaSetDevice(cur);
}

// --------------------------------------------------------------------- prepare
l1dm_status prepare_impl(const float *X, int64_t n, int64_t ld_x, int64_t k_begin, int64_t k_end,
                         void *stream, l1dm_ctx *h) {
  int dev = 0;
  l1dm_status st = check_arch(&dev);
  if (st != L1DM_OK) return st;
  h->device = dev;
  h->n = n;
  h->k_begin = k_begin;
  h->k_end = k_end;
  h->full_rows = (k_begin == 0 && k_end == ld_x);
  h->dl = k_end - k_begin;
  h->ldn = (n + 31) / 32 * 32;
  int l2 = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  h->l2_bytes = l2;
  // CUDA convention: a NULL stream is the legacy default stream (implicitly ordered
  // with every blocking stream, e.g. torch's default stream).
  h->stream = (cudaStream_t)stream;
  h->own_stream = false;
  cudaStream_t s = h->stream;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  CUDA_TRY(cudaEventCreate(&ev0));
  CUDA_TRY(cudaEventCreate(&ev1));
  CUDA_TRY(cudaEventRecord(ev0, s));
  static const bool dbg = getenv("L1DM_DEBUG_PREP") != nullptr;  // phase timing to stderr
  const auto t_start = std::chrono::steady_clock::now();
  auto lap = [&](const char *what) {
    if (!dbg) return;
    cudaStreamSynchronize(s);
    fprintf(stderr, "[l1dm prep] %-28s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start)
                .count());
  };

  const int64_t dl = h->dl, ldn = h->ldn;
  const size_t elems = (size_t)dl * (size_t)ldn;

  // X may live on the host: stage it (only the rows are needed, all columns copied).
  const float *Xd = X;
  DevBuf<float> Xstage;
  if (!is_device_pointer(X)) {
    CUDA_TRY(Xstage.ensure((size_t)n * (size_t)ld_x, false, s));
    CUDA_TRY(cudaMemcpyAsync(Xstage.p, X, (size_t)n * (size_t)ld_x * sizeof(float),
                             cudaMemcpyHostToDevice, s));
    Xd = Xstage.p;
  }
  DevBuf<uint32_t> keyA, keyB, valA, valB, hist, dbase;
  DevBuf<unsigned long long> status;
  DevBuf<unsigned> ctrl;  // [0] nonfinite [1] timeout [2] ticket [3] runs [4..8) trivial passes
  CUDA_TRY(ctrl.ensure(8, true, s));
  CUDA_TRY(keyA.ensure(elems, false, s));
  CUDA_TRY(h->hsum.ensure((size_t)n, false, s));
  CUDA_TRY(hist.ensure((size_t)dl * 1024, true, s));

  lap("alloc keyA/rank/hsum/hist");
  launch_keys(Xd, n, ld_x, k_begin, dl, ldn, keyA.p, h->hsum.p, ctrl.p + 0, s);
  h->kernel_launches++;
  launch_hist(keyA.p, n, ldn, dl, hist.p, s);
  h->kernel_launches++;
  CUDA_TRY(dbase.ensure((size_t)4 * dl * 256, false, s));
  launch_digit_base(hist.p, n, dl, dbase.p, ctrl.p + 4, s);
  h->kernel_launches++;
  CUDA_TRY(cudaGetLastError());
  unsigned flags_h[8];
  CUDA_TRY(cudaMemcpyAsync(flags_h, ctrl.p, sizeof(flags_h), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  lap("keys + hist + readback");
  if (flags_h[0]) {
    Xstage.release();
    keyA.release();
    hist.release();
    ctrl.release();
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    return fail(L1DM_ENONFINITE, "X holds a non-finite value in coordinates [%lld, %lld)",
                (long long)k_begin, (long long)k_end);
  }
  // Passes whose digit is constant in every segment are the identity: skip them.
  std::vector<int> passes;
  for (int p = 0; p < 4; ++p)
    if (flags_h[4 + p] != (unsigned)dl) passes.push_back(p);
  const int P = (int)passes.size();
  if (P == 0) {
    // keyA holds the keys; emit in place (sval bits over keyA), perm into valA.
    CUDA_TRY(valA.ensure(elems, false, s));
    CUDA_TRY(h->rank.ensure(elems, false, s));
    launch_identity_emit(keyA.p, reinterpret_cast<float *>(keyA.p), valA.p, h->rank.p, n, ldn, dl,
                         s);
    h->rank_ready = true;
    h->kernel_launches++;
    h->sval_bits.p = keyA.p;
    h->sval_bits.count = keyA.count;
    keyA.p = nullptr;
    keyA.count = 0;
    h->perm.p = valA.p;
    h->perm.count = valA.count;
    valA.p = nullptr;
    valA.count = 0;
  } else {
    CUDA_TRY(keyB.ensure(elems, false, s));
    CUDA_TRY(valB.ensure(elems, false, s));
    if (P > 1) CUDA_TRY(valA.ensure(elems, false, s));
    const int64_t tiles = (n + kSortTile - 1) / kSortTile;
    CUDA_TRY(status.ensure((size_t)dl * tiles * 256, true, s));
    static const bool fused_rank = getenv("L1DM_FUSED_RANK") != nullptr;  // tuning switch
    if (fused_rank) CUDA_TRY(h->rank.ensure(elems, false, s));
    lap("alloc sort buffers");
    uint32_t *kb[2] = {keyA.p, keyB.p};
    uint32_t *vb[2] = {valA.p, valB.p};
    for (int i = 0; i < P; ++i) {
      const int p = passes[i];
      CUDA_TRY(cudaMemsetAsync(ctrl.p + 2, 0, sizeof(unsigned), s));
      const uint32_t ep = h->epoch++;
      launch_sort_pass(i == 0, i == P - 1, kb[i & 1], vb[i & 1], kb[(i + 1) & 1], vb[(i + 1) & 1],
                       fused_rank ? h->rank.p : nullptr, n, ldn, dl, 8 * p,
                       dbase.p + (size_t)p * dl * 256, status.p, ep, ctrl.p + 2, ctrl.p + 1, s);
      h->kernel_launches++;
      sort_prof_print(s);  // no-op unless built with L1DM_SORT_PROF
      CUDA_TRY(cudaGetLastError());
    }
    // without the fused variant, rank (only gather-mode queries read it) is built lazily by
    // ensure_rank: scatter and runs queries never pay for it
    h->rank_ready = fused_rank;
    const int fin = P & 1;
    DevBuf<uint32_t> *kbuf[2] = {&keyA, &keyB};
    DevBuf<uint32_t> *vbuf[2] = {&valA, &valB};
    std::swap(h->sval_bits.p, kbuf[fin]->p);
    std::swap(h->sval_bits.count, kbuf[fin]->count);
    std::swap(h->perm.p, vbuf[fin]->p);
    std::swap(h->perm.count, vbuf[fin]->count);
  }
  lap("sort passes + rank");
  // runs: count run starts per tile; keep runid / rvals when every coordinate has <= 256
  {
    static const bool runs_env = [] {
      const char *e = getenv("L1DM_RUNS");
      return e ? atoi(e) != 0 : true;
    }();
    const int64_t rt = runs_tiles(n);
    bool maybe = runs_env && n >= 2;
    if (maybe) {  // necessary condition on a sample first (ctrl[3]: 1 = too many values)
      launch_runs_sample(reinterpret_cast<const float *>(h->sval_bits.p), n, ldn, dl, ctrl.p + 3,
                         s);
      h->kernel_launches++;
      unsigned too_many = 0;
      CUDA_TRY(cudaMemcpyAsync(&too_many, ctrl.p + 3, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      maybe = too_many == 0;
    }
    if (maybe) {
      DevBuf<uint32_t> rcnt;
      CUDA_TRY(rcnt.ensure((size_t)dl * rt, false, s));
      launch_runs_count(reinterpret_cast<const float *>(h->sval_bits.p), n, ldn, dl, rcnt.p, s);
      h->kernel_launches++;
      std::vector<uint32_t> cnt((size_t)dl * rt), off((size_t)dl * rt), nr((size_t)dl);
      CUDA_TRY(cudaMemcpyAsync(cnt.data(), rcnt.p, cnt.size() * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      bool ok = true;
      for (int64_t k = 0; k < dl; ++k) {
        uint32_t run = 0;
        for (int64_t t = 0; t < rt; ++t) {
          off[(size_t)k * rt + t] = run;
          run += cnt[(size_t)k * rt + t];
        }
        nr[(size_t)k] = run;
        if (run > 256) ok = false;
      }
      if (ok) {
        CUDA_TRY(rcnt.ensure((size_t)dl * rt, false, s));
        CUDA_TRY(cudaMemcpyAsync(rcnt.p, off.data(), off.size() * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, s));
        CUDA_TRY(h->runid.ensure((size_t)dl * ldn, false, s));
        CUDA_TRY(h->rvals.ensure((size_t)dl * 256, true, s));
        CUDA_TRY(h->nruns.ensure((size_t)dl, false, s));
        CUDA_TRY(cudaMemcpyAsync(h->nruns.p, nr.data(), nr.size() * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, s));
        launch_runs_emit(reinterpret_cast<const float *>(h->sval_bits.p), n, ldn, dl, rcnt.p,
                         h->rvals.p, s);
        launch_runs_ids(Xd, n, ld_x, k_begin, dl, ldn, h->rvals.p, h->nruns.p, h->runid.p, s);
        h->kernel_launches += 2;
        h->has_runs = true;
      }
      CUDA_TRY(cudaStreamSynchronize(s));  // rcnt and the host vectors go out of scope
      rcnt.release();
    }
  }
  lap("runs");
  Xstage.release();  // (the runs ids read X)
  CUDA_TRY(cudaEventRecord(ev1, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaMemcpy(flags_h, ctrl.p, sizeof(flags_h), cudaMemcpyDeviceToHost));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  h->prep_ms = ms;
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  keyA.release();
  keyB.release();
  valA.release();
  valB.release();
  hist.release();
  dbase.release();
  status.release();
  ctrl.release();
  lap("release transients");
  if (flags_h[1]) return fail(L1DM_ETIMEOUT, "sort look-back wait exceeded its bound");
  return L1DM_OK;
}

// --------------------------------------------------------------------- query
int vec_cap_for(const float *Z, int64_t ldz) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(Z);
  if (ldz % 4 == 0 && a % 16 == 0) return 4;
  if (ldz % 2 == 0 && a % 8 == 0) return 2;
  return 1;
}

l1dm_status ensure_plan(l1dm_ctx *h, int64_t m, int vec_cap) {
  // a cached plan for this (m, alignment, limit) stands: the free-memory probe below
  // (cudaMemGetInfo) costs host time on every query otherwise
  if (h->plan_m == m && h->plan_vec_cap == vec_cap && h->plan_ws_limit == h->ws_limit &&
      h->plan_mode == h->mode)
    return L1DM_OK;
  size_t ws = h->ws_limit;
  QueryPlan p;
  if (ws == 0) {
    // A plan whose whole workspace is small (scatter mode, runs, narrow gathers) does not depend
    // on the free memory: take it without the probe — cudaMemGetInfo occasionally stalls the
    // host for milliseconds (measured: up to 7 ms on B200), idling the GPU on a new handle's
    // first query.  An allocation that still fails flushes the block cache and retries.
    constexpr size_t kNoProbeBytes = (size_t)2 << 30;
    if (make_plan(h->n, h->dl, m, h->l2_bytes, (int64_t)kNoProbeBytes, vec_cap, h->mode, &p) &&
        p.chunks == 1 && p.workspace_bytes <= kNoProbeBytes) {
      ws = kNoProbeBytes;
    } else {
      size_t fr = 0, tot = 0;
      CUDA_TRY(cudaMemGetInfo(&fr, &tot));
      ws = (size_t)(0.75 * (double)(fr + BlockCache::get().cached(h->device) +
                                   h->U.count * sizeof(double) +
                                   h->agg.count * sizeof(double) * 2));
    }
  }
  if (h->plan_m == m && h->plan_ws == ws && h->plan_vec_cap == vec_cap) return L1DM_OK;
  if (!make_plan(h->n, h->dl, m, h->l2_bytes, (int64_t)ws, vec_cap, h->mode, &p))
    return fail(L1DM_EINVAL, "no query plan for n=%lld d=%lld m=%lld", (long long)h->n,
                (long long)h->dl, (long long)m);
  h->plan = p;
  h->plan_m = m;
  h->plan_ws = ws;
  h->plan_vec_cap = vec_cap;
  h->plan_ws_limit = h->ws_limit;
  h->plan_mode = h->mode;
  return L1DM_OK;
}

// nblocks/events: the pass that completes Y (the last chunk's accumulate, or the scatter-mode
// epilogue) is launched per contiguous point block, and events[b] is recorded after block b.
// Runs mode is used when the prepared data has runs tables (every coordinate <= 256 distinct
// values) and the mode is AUTO or RUNS.
bool use_runs(const l1dm_ctx *h) {
  return h->has_runs && (h->mode == L1DM_MODE_AUTO || h->mode == L1DM_MODE_RUNS);
}

// blocked (scatter mode, m > 1 only): Y is column-block-major — block cb at Y + cb n mb with
// row stride mb — and events[cb] is recorded once block cb is final (nblocks = col_blocks).
// rank[k][perm[k][r]] = r (K3), built the first time a query needs it (gather mode's
// accumulate, the l_p gather path, debug export): the scatter and runs strategies never read it
l1dm_status ensure_rank(l1dm_ctx *h, cudaStream_t s) {
  if (h->rank_ready) return L1DM_OK;
  CUDA_TRY(h->rank.ensure((size_t)h->dl * (size_t)h->ldn, false, s));
  launch_rank(h->perm.p, h->rank.p, h->n, h->ldn, h->dl, s);
  CUDA_TRY(cudaGetLastError());
  h->kernel_launches++;
  h->rank_ready = true;
  return L1DM_OK;
}

// pd (peer push): the final pass stores each finished row into its owner's inbox
// slot instead of Y (gather mode's last accumulate, scatter mode's block write-out); Y is then
// only the gather mode's scratch between coordinate chunks.  Callers pass pd only when
// push_fusable() holds.
l1dm_status matvec_device(l1dm_ctx *h, const float *Z, int64_t ldz, int64_t m, double *Y,
                          int64_t ldy, cudaStream_t s, int64_t nblocks = 1,
                          void *const *events = nullptr, bool blocked = false,
                          const PeerDst *pd = nullptr) {
  if (nblocks < 1) nblocks = 1;
  auto block_range = [&](int64_t b, int64_t &i0, int64_t &i1) {
    i0 = (h->n * b) / nblocks;
    i1 = (h->n * (b + 1)) / nblocks;
  };
  if (!blocked && use_runs(h)) {
    // runs mode: tie-heavy coordinates, no sorted-order gather at all
    CUDA_TRY(h->rtab.ensure((size_t)runs_copies(h->dl, m) * h->dl * 256 * m, false, s));
    CUDA_TRY(h->part.ensure((size_t)h->dl * 2 * m, false, s));
    CUDA_TRY(h->Sg.ensure((size_t)2 * m, false, s));
    {
      TimedScope ts(h, kScan, s);
      launch_runs_query(h->runid.p, h->ldn, h->n, h->dl, h->rvals.p, h->nruns.p, Z, ldz, m,
                        h->rtab.p, h->part.p, h->hsum.p, h->Sg.p, Y, ldy, 0, s);
      h->kernel_launches += 2;
      h->launches[kScan]++;
      if (h->timing) h->scan_pairs += h->n * h->dl;
    }
    {
      TimedScope ts(h, kColsums, s);
      launch_totals(h->part.p, 2 * m, h->dl, m, h->Sg.p, h->Sg.p + m, s);
      h->kernel_launches++;
      h->launches[kColsums]++;
    }
    {
      TimedScope ts(h, kAcc, s);
      for (int64_t b = 0; b < nblocks; ++b) {
        int64_t i0, i1;
        block_range(b, i0, i1);
        launch_runs_query(h->runid.p, h->ldn, h->n, h->dl, h->rvals.p, h->nruns.p, Z, ldz, m,
                          h->rtab.p, h->part.p, h->hsum.p, h->Sg.p, Y, ldy, 1, s, i0, i1);
        h->kernel_launches++;
        if (events && events[b]) CUDA_TRY(cudaEventRecord((cudaEvent_t)events[b], s));
      }
      h->launches[kAcc]++;
      if (h->timing) h->acc_pairs += h->n * h->dl;
    }
    CUDA_TRY(cudaGetLastError());
    h->queries++;
    h->m_last = m;
    return L1DM_OK;
  }
  const auto dbg_t0 = std::chrono::steady_clock::now();
  l1dm_status st = ensure_plan(h, m, vec_cap_for(Z, ldz));
  if (st != L1DM_OK) return st;
  if (BlockCache::debug())
    fprintf(stderr, "[l1dm] ensure_plan %.3f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - dbg_t0)
                .count());
  const QueryPlan &p = h->plan;
  if (!p.scatter) CUDA_TRY(h->U.ensure((size_t)p.kc * (size_t)h->n * (size_t)p.ldu, false, s));
  if (p.mb == 1) CUDA_TRY(h->zs.ensure((size_t)p.kc * (size_t)h->ldn, false, s));
  CUDA_TRY(h->flags.ensure(p.lb_slots, true, s));
  CUDA_TRY(h->agg.ensure(p.lb_slots * 2 * p.mb, false, s));
  CUDA_TRY(h->incl.ensure(p.lb_slots * 2 * p.mb, false, s));
  CUDA_TRY(h->part.ensure((size_t)h->dl * 2 * m, false, s));  // per-segment totals
  CUDA_TRY(h->Sg.ensure((size_t)2 * m, false, s));
  const size_t nticket = (size_t)p.chunks;
  if (h->ctr.count < 2 + nticket) {
    CUDA_TRY(h->ctr.ensure(2 + nticket, true, s));  // tickets start at 0
  }
  if (p.zt_floats) {
    CUDA_TRY(h->zt.ensure((size_t)p.zt_floats, false, s));
    CUDA_TRY(h->yt.ensure((size_t)h->n * p.mb, false, s));
  }
  if (BlockCache::debug())
    fprintf(stderr, "[l1dm] plan + workspace %.3f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - dbg_t0)
                .count());
  // scatter mode: by default the single-pass apply (k5_scan_lb; tile prefixes by a fixed-point
  // look-back inside the apply, no pass over Z beyond the gathers the apply makes anyway) for
  // every m, m = 1 included (one 1-column block); L1DM_SCATTER_LB=0 selects the two-pass forms
  // (m = 1: reduce / prefix / apply with fp64 atomics into Y; m > 1: a reduce pass for the tile
  // totals, then the apply)
  static const bool lb_env = [] {
    const char *e = getenv("L1DM_SCATTER_LB");
    return e ? atoi(e) != 0 : true;
  }();
  if (p.scatter && m == 1 && lb_env) {
    CUDA_TRY(h->zt.ensure((size_t)h->n, false, s));
    CUDA_TRY(h->yt.ensure((size_t)h->n, false, s));
  }
  if (p.scatter && m == 1 && !lb_env) {
    // scatter mode, m == 1, two-pass: zero Y, reduce/prefix/apply over every coordinate adding
    // 2U into Y, then the epilogue g - h_i S
    CUDA_TRY(cudaMemset2DAsync(Y, (size_t)ldy * sizeof(double), 0, sizeof(double), (size_t)h->n, s));
    {
      TimedScope ts(h, kScan, s);
      const uint32_t ep = h->epoch++;
      if (h->epoch >= (1u << 30)) h->epoch = 1;
      QueryPlan ps = p;
      ps.ldu = ldy;  // the scan adds straight into Y's rows
      launch_scan(ps, h->perm.p, reinterpret_cast<const float *>(h->sval_bits.p), h->ldn, h->n,
                  Z, ldz, m, Y, 0, h->dl, h->flags.p, h->agg.p, h->incl.p, ep, h->ctr.p + 2,
                  h->ctr.p + 1, h->part.p, 2 * m, h->zs.p, s);
      h->kernel_launches += 3;  // reduce, prefix, apply
      h->launches[kScan]++;
      if (h->timing) h->scan_pairs += h->n * h->dl;
    }
    {
      TimedScope ts(h, kColsums, s);
      launch_totals(h->part.p, 2 * m, h->dl, m, h->Sg.p, h->Sg.p + m, s);
      h->kernel_launches++;
      h->launches[kColsums]++;
    }
    {
      TimedScope ts(h, kAcc, s);
      for (int64_t b = 0; b < nblocks; ++b) {
        int64_t i0, i1;
        block_range(b, i0, i1);
        launch_epilogue(h->hsum.p, h->Sg.p, Y, ldy, i0, i1, m, s);
        h->kernel_launches++;
        if (events && events[b]) CUDA_TRY(cudaEventRecord((cudaEvent_t)events[b], s));
      }
      h->launches[kAcc]++;
    }
    CUDA_TRY(cudaMemsetAsync(h->ctr.p + 2, 0, sizeof(unsigned), s));  // re-arm the ticket
  } else if (p.scatter) {
    // scatter mode, m > 1: per column block of mb columns (Zt, the block's compact copy of Z),
    // the reduce / prefix / apply scan adds 2U into a compact L2-resident accumulator Yt
    // (n x mb), then Y's block columns = Yt + g - h_i S.  Timing kinds: scan =
    // reduce + prefix (tile totals), accumulate = apply (U and the reductions into Yt),
    // colsums = Zt, totals and the block write-out.
    const float *sval = reinterpret_cast<const float *>(h->sval_bits.p);
    // deterministic accumulation (R16): the block accumulator Yt holds 64-bit fixed
    // point at per-column scales from a bound on |Yt|; integer reductions are associative, so Y
    // is bitwise reproducible run to run.  The Zt pass also sums |z| per column for the bound.
    CUDA_TRY(h->fxbuf.ensure(6 * (size_t)m + (size_t)zt_max_ctas(m, p.mb) * m, false, s));
    double *fx = h->fxbuf.p;
    {
      TimedScope ts(h, kColsums, s);
      const int64_t nparts = launch_zt(Z, ldz, h->n, m, p.mb, h->zt.p, s, h->fxbuf.p + 6 * m);
      launch_fx_scale(h->fxbuf.p + 6 * m, nparts, m, h->sval_bits.p, h->ldn, h->n, h->dl, fx, s);
      h->kernel_launches += 2;
      h->launches[kColsums]++;
    }
    // tile prefixes: by default a decoupled look-back inside each block's apply (k5_scan_lb);
    // L1DM_SCATTER_LB=0: the two-pass form below (one reduce pass over full Z rows for every
    // column block at once for m <= 256, else a reduce pass per block over its Zt block)
    const bool single = lb_env;

    if (single) {
      // every launch rewrites all dl x tiles x 2mb words, so a stale word on the same geometry is
      // the previous launch's (another epoch mod 4); on a new geometry the words are zeroed
      const int64_t lbt = (h->n + scan_lb_rows(p.mb) - 1) / scan_lb_rows(p.mb);
      const size_t words = (size_t)h->dl * lbt * 2 * p.mb;
      const int64_t geom = (int64_t)words * 64 + p.mb;
      CUDA_TRY(h->lbst.ensure(words, false, s));
      if (geom != h->lb_geom) {
        CUDA_TRY(cudaMemsetAsync(h->lbst.p, 0, words * sizeof(unsigned long long), s));
        h->lb_geom = geom;
      }
    }
    static const bool reduce_all_env = [] {
      const char *e = getenv("L1DM_REDUCE_ALL");
      return e ? atoi(e) != 0 : true;
    }();
    bool all = false;
    if (!single && reduce_all_env && m <= 256) {
      TimedScope ts(h, kScan, s);
      CUDA_TRY(h->agg.ensure((size_t)h->dl * p.tiles_per_segment * 2 * m, false, s));
      all = launch_reduce_all(h->perm.p, sval, h->ldn, h->n, Z, ldz, m, h->dl,
                              p.tiles_per_segment, h->agg.p, h->part.p, s);
      h->kernel_launches += 2;  // reduce-all, prefix
      h->launches[kScan]++;
      if (h->timing) h->scan_pairs += h->n * h->dl * p.col_blocks;
    }
    for (int cb = 0; cb < p.col_blocks; ++cb) {
      const int64_t c0 = (int64_t)cb * p.mb;
      const int64_t mc = std::min<int64_t>(p.mb, m - c0);
      const bool last = cb == p.col_blocks - 1;
      const float *ztb = h->zt.p + (size_t)cb * h->n * p.mb;
      if (!all && !single) {
        TimedScope ts(h, kScan, s);
        launch_scan_seq(p, 1, h->perm.p, sval, h->ldn, h->n, ztb, mc, h->yt.p, p.mb, false,
                        h->dl, h->agg.p, h->part.p + 2 * c0, 2 * m, 0, s);
        h->kernel_launches += 2;  // reduce, prefix
        h->launches[kScan]++;
        if (h->timing) h->scan_pairs += h->n * h->dl;
      }
      {
        TimedScope ts(h, kAcc, s);
        // (clearing Yt in the write-out's pass instead, as it reads it, measured 7x slower for
        // that kernel than this memset: c3 G = 8 shard query 3.94 vs 2.77 ms)
        CUDA_TRY(cudaMemsetAsync(h->yt.p, 0, (size_t)h->n * p.mb * sizeof(double), s));
        if (single) {
          const uint32_t ep = ++h->lb_epoch;
          launch_scan_lb(p.mb, h->perm.p, sval, h->ldn, h->n, ztb, mc,
                         reinterpret_cast<unsigned long long *>(h->yt.p), h->dl,
                         h->lbst.p, ep, h->ctr.p + 1, fx + c0,
                         fx + 2 * m + c0, m, h->part.p + 2 * c0, 2 * m, s);
        } else {
          launch_scan_seq(p, 1, h->perm.p, sval, h->ldn, h->n, ztb, mc, h->yt.p, p.mb, false,
                          h->dl, all ? h->agg.p + 2 * c0 : h->agg.p, h->part.p + 2 * c0, 2 * m,
                          1, s, all ? 2 * m : 0, fx + c0);
        }
        h->kernel_launches++;  // apply
        h->launches[kAcc]++;
        if (h->timing) h->acc_pairs += h->n * h->dl;
      }
      if (single) {
        // S, g of the block folded into the write-out (no k4_totals launch)
        TimedScope ts(h, kColsums, s);
        unsigned long long *ytq = reinterpret_cast<unsigned long long *>(h->yt.p);
        const int64_t nb = last ? nblocks : 1;
        if (blocked) {
          launch_block_out_fx(ytq, p.mb, mc, h->hsum.p, h->part.p + 2 * c0, 2 * m, h->dl,
                              h->Sg.p + c0, m, Y + (size_t)cb * h->n * p.mb, p.mb, 0, h->n, s,
                              nullptr, 0, fx + m + c0);
          if (events && events[cb]) CUDA_TRY(cudaEventRecord((cudaEvent_t)events[cb], s));
        }
        for (int64_t b = 0; !blocked && b < nb; ++b) {
          int64_t i0 = 0, i1 = h->n;
          if (last) block_range(b, i0, i1);
          launch_block_out_fx(ytq, p.mb, mc, h->hsum.p, h->part.p + 2 * c0, 2 * m, h->dl,
                              h->Sg.p + c0, m, Y + c0, ldy, i0, i1, s, pd, c0, fx + m + c0);
          if (last && events && events[b]) CUDA_TRY(cudaEventRecord((cudaEvent_t)events[b], s));
        }
        h->kernel_launches += blocked ? 1 : nb;  // block out(s)
        h->launches[kColsums]++;
      } else {
        TimedScope ts(h, kColsums, s);
        launch_totals(h->part.p + 2 * c0, 2 * m, h->dl, mc, h->Sg.p + c0, h->Sg.p + m + c0, s);
        const int64_t nb = last ? nblocks : 1;
        if (blocked) {
          launch_block_out(h->yt.p, p.mb, mc, h->hsum.p, h->Sg.p + c0, h->Sg.p + m + c0,
                           Y + (size_t)cb * h->n * p.mb, p.mb, 0, h->n, s, nullptr, 0, fx + m + c0);
          if (events && events[cb]) CUDA_TRY(cudaEventRecord((cudaEvent_t)events[cb], s));
        }
        for (int64_t b = 0; !blocked && b < nb; ++b) {
          int64_t i0 = 0, i1 = h->n;
          if (last) block_range(b, i0, i1);
          launch_block_out(h->yt.p, p.mb, mc, h->hsum.p, h->Sg.p + c0, h->Sg.p + m + c0, Y + c0,
                           ldy, i0, i1, s, pd, c0, fx + m + c0);
          if (last && events && events[b]) CUDA_TRY(cudaEventRecord((cudaEvent_t)events[b], s));
        }
        h->kernel_launches += 1 + nb;  // totals, block out(s)
        h->launches[kColsums]++;
      }
    }
  }
  if (!p.scatter) {
    l1dm_status rs = ensure_rank(h, s);
    if (rs != L1DM_OK) return rs;
  }
  for (int64_t c = 0; !p.scatter && c < p.chunks; ++c) {
    const int64_t k_first = c * p.kc;
    const int64_t kcc = std::min<int64_t>(p.kc, h->dl - k_first);
    const bool last = (c == p.chunks - 1);
    {
      TimedScope ts(h, kScan, s);
      const uint32_t ep = h->epoch++;
      if (h->epoch >= (1u << 30)) h->epoch = 1;
      launch_scan(p, h->perm.p, reinterpret_cast<const float *>(h->sval_bits.p), h->ldn, h->n, Z,
                  ldz, m, h->U.p, k_first, kcc, h->flags.p, h->agg.p, h->incl.p, ep,
                  h->ctr.p + 2 + c, h->ctr.p + 1, h->part.p, 2 * m, h->zs.p, s);
      h->kernel_launches += (p.mb == 1) ? 3 : 1;  // m == 1: reduce, prefix, apply
      h->launches[kScan]++;
      if (h->timing) h->scan_pairs += h->n * kcc;
    }
    if (last) {
      TimedScope ts(h, kColsums, s);
      launch_totals(h->part.p, 2 * m, h->dl, m, h->Sg.p, h->Sg.p + m, s);  // S, g from the segment totals
      h->kernel_launches++;
      h->launches[kColsums]++;
    }
    {
      TimedScope ts(h, kAcc, s);
      const int64_t nb = last ? nblocks : 1;
      for (int64_t b = 0; b < nb; ++b) {
        int64_t i0 = 0, i1 = h->n;
        if (last) block_range(b, i0, i1);
        launch_accumulate(p, h->rank.p, h->ldn, h->n, h->U.p, k_first, kcc, h->hsum.p, h->Sg.p,
                          Y, ldy, m, c == 0, last, b == 0 ? h->ctr.p + 2 + c : nullptr, i0, i1,
                          s, 2.0, true, pd);
        h->kernel_launches++;
        if (last && events && events[b]) CUDA_TRY(cudaEventRecord((cudaEvent_t)events[b], s));
      }
      h->launches[kAcc]++;
      if (h->timing) h->acc_pairs += h->n * kcc;
    }
  }
  CUDA_TRY(cudaGetLastError());
  h->queries++;
  h->m_last = m;
  return L1DM_OK;
}

// l_p^p query, odd p > 1: Zt, then per column block the seq scan with p+1
// moments; scatter mode adds each coordinate's whole term into Yt (then Y's block columns =
// Yt), gather mode stores it in sorted order into U and k6 sums U over each coordinate chunk.
l1dm_status lp_device(l1dm_ctx *h, int lp, const float *Z, int64_t ldz, int64_t m, double *Y,
                      int64_t ldy, cudaStream_t s) {
  if (use_runs(h)) {  // tie-heavy data: the run-level form serves every odd p
    CUDA_TRY(h->rtab.ensure((size_t)runs_copies(h->dl, m) * h->dl * 256 * m, false, s));
    {
      TimedScope ts(h, kScan, s);
      launch_runs_lp(h->runid.p, h->ldn, h->n, h->dl, h->rvals.p, h->nruns.p, Z, ldz, m, lp,
                     h->rtab.p, Y, ldy, 0, s);
      h->kernel_launches += 2;  // histogram, p-moment scan
      h->launches[kScan]++;
    }
    {
      TimedScope ts(h, kAcc, s);
      launch_runs_lp(h->runid.p, h->ldn, h->n, h->dl, h->rvals.p, h->nruns.p, Z, ldz, m, lp,
                     h->rtab.p, Y, ldy, 1, s);
      h->kernel_launches++;  // expansion
      h->launches[kAcc]++;
      if (h->timing) h->acc_pairs += h->n * h->dl;
    }
    CUDA_TRY(cudaGetLastError());
    h->queries++;
    h->m_last = m;
    return L1DM_OK;
  }
  size_t ws = h->ws_limit;
  QueryPlan p;
  if (ws == 0) {  // the free-memory probe only when the workspace is large (see ensure_plan)
    constexpr size_t kNoProbeBytes = (size_t)2 << 30;
    if (make_lp_plan(h->n, h->dl, m, lp, h->l2_bytes, (int64_t)kNoProbeBytes, h->mode, &p) &&
        p.chunks == 1 && p.workspace_bytes <= kNoProbeBytes) {
      ws = kNoProbeBytes;
    } else {
      size_t fr = 0, tot = 0;
      CUDA_TRY(cudaMemGetInfo(&fr, &tot));
      ws = (size_t)(0.75 * (double)(fr + BlockCache::get().cached(h->device) +
                                   h->U.count * sizeof(double)));
    }
  }
  if (!make_lp_plan(h->n, h->dl, m, lp, h->l2_bytes, (int64_t)ws, h->mode, &p))
    return fail(L1DM_EINVAL, "no l_p plan for p=%d n=%lld d=%lld m=%lld", lp, (long long)h->n,
                (long long)h->dl, (long long)m);
  const int K = lp + 1;
  const int64_t ld_seg = (int64_t)K * m;
  const float *sval = reinterpret_cast<const float *>(h->sval_bits.p);
  CUDA_TRY(h->zt.ensure((size_t)p.zt_floats, false, s));
  CUDA_TRY(h->agg.ensure(p.lb_slots * (size_t)K * p.mb, false, s));
  CUDA_TRY(h->part.ensure((size_t)h->dl * ld_seg, false, s));
  if (p.scatter) {
    CUDA_TRY(h->yt.ensure((size_t)h->n * p.mb, false, s));
  } else {
    CUDA_TRY(h->U.ensure((size_t)p.kc * (size_t)h->n * (size_t)m, false, s));
    l1dm_status rs = ensure_rank(h, s);  // the accumulate gathers U at each point's rank
    if (rs != L1DM_OK) return rs;
  }
  static const bool lb_env = [] {
    const char *e = getenv("L1DM_SCATTER_LB");
    return e ? atoi(e) != 0 : true;
  }();
  if (p.scatter && lb_env && scan_lb_supported(p.mb, lp)) {
    // single pass: per column block the apply prefixes all p + 1 moments by the
    // fixed-point look-back and adds 2 sum_t c_t v^(p-t) M_t; after the last block one DMMA
    // expansion subtracts the totals' part, sum_k sum_t c_t x_ik^(p-t) T_kt (X rebuilt in point
    // order from the sorted tables once per handle)
    if (h->ctr.count < 3) CUDA_TRY(h->ctr.ensure(3, true, s));  // [1]: the timeout word
    if (!h->xr_ready) {
      CUDA_TRY(h->xr.ensure((size_t)h->n * h->dl, false, s));
      launch_unsort(h->perm.p, sval, h->ldn, h->n, h->dl, h->xr.p, s);
      h->kernel_launches++;
      h->xr_ready = true;
    }
    CUDA_TRY(h->fxbuf.ensure(2 * (size_t)K * m + (size_t)zt_max_ctas(m, p.mb) * m, false, s));
    double *fa = h->fxbuf.p;
    {
      TimedScope ts(h, kColsums, s);
      const int64_t nparts = launch_zt(Z, ldz, h->n, m, p.mb, h->zt.p, s, fa + 2 * (size_t)K * m);
      launch_lb_scales(fa + 2 * (size_t)K * m, nparts, m, h->sval_bits.p, h->ldn, h->n, h->dl, lp,
                       fa, s);
      h->kernel_launches += 2;
      h->launches[kColsums]++;
    }
    const int64_t lbt = (h->n + scan_lb_rows(p.mb) - 1) / scan_lb_rows(p.mb);
    const size_t words = (size_t)h->dl * lbt * K * p.mb;
    const int64_t geom = ((int64_t)words * 64 + p.mb) * 8 + K;
    CUDA_TRY(h->lbst.ensure(words, false, s));
    if (geom != h->lb_geom) {
      CUDA_TRY(cudaMemsetAsync(h->lbst.p, 0, words * sizeof(unsigned long long), s));
      h->lb_geom = geom;
    }
    for (int cb = 0; cb < p.col_blocks; ++cb) {
      const int64_t c0 = (int64_t)cb * p.mb;
      const int64_t mc = std::min<int64_t>(p.mb, m - c0);
      const float *ztb = h->zt.p + (size_t)cb * h->n * p.mb;
      TimedScope ts(h, kAcc, s);
      CUDA_TRY(cudaMemsetAsync(h->yt.p, 0, (size_t)h->n * p.mb * sizeof(double), s));
      const uint32_t ep = ++h->lb_epoch;
      launch_scan_lb(p.mb, h->perm.p, sval, h->ldn, h->n, ztb, mc,
                     reinterpret_cast<unsigned long long *>(h->yt.p), h->dl, h->lbst.p, ep,
                     h->ctr.p + 1, nullptr, fa + c0, m, h->part.p + K * c0, ld_seg, s, lp);
      launch_block_out(h->yt.p, p.mb, mc, nullptr, nullptr, nullptr, Y + c0, ldy, 0, h->n, s);
      h->kernel_launches += 2;
      h->launches[kAcc]++;
      if (h->timing) h->acc_pairs += h->n * h->dl;
    }
    {
      TimedScope ts(h, kColsums, s);
      CUDA_TRY(h->agg.ensure(lp_totals_workspace(h->dl, m, lp) / sizeof(double) + 1, false, s));
      h->kernel_launches += launch_lp_totals_expand(h->xr.p, h->dl, h->n, h->dl, m, h->part.p,
                                                    ld_seg, lp, h->agg.p, Y, ldy, s);
      h->launches[kColsums]++;
    }
    CUDA_TRY(cudaGetLastError());
    h->queries++;
    h->m_last = m;
    return L1DM_OK;
  }
  {
    TimedScope ts(h, kColsums, s);
    launch_zt(Z, ldz, h->n, m, p.mb, h->zt.p, s);
    h->kernel_launches++;
    h->launches[kColsums]++;
  }
  for (int64_t c = 0; c < p.chunks; ++c) {
    const int64_t k_first = c * p.kc;
    const int64_t kcc = std::min<int64_t>(p.kc, h->dl - k_first);
    const uint32_t *perm = h->perm.p + k_first * h->ldn;
    const float *sv = sval + k_first * h->ldn;
    double *seg = h->part.p + k_first * ld_seg;
    for (int cb = 0; cb < p.col_blocks; ++cb) {
      const int64_t c0 = (int64_t)cb * p.mb;
      const int64_t mc = std::min<int64_t>(p.mb, m - c0);
      const float *ztb = h->zt.p + (size_t)cb * h->n * p.mb;
      {
        TimedScope ts(h, kScan, s);
        launch_scan_seq(p, lp, perm, sv, h->ldn, h->n, ztb, mc, nullptr, 0, false, kcc, h->agg.p,
                        seg + K * c0, ld_seg, 0, s);
        h->kernel_launches += 2;
        h->launches[kScan]++;
        if (h->timing) h->scan_pairs += h->n * kcc;
      }
      TimedScope ts(h, kAcc, s);
      if (p.scatter) {
        CUDA_TRY(cudaMemsetAsync(h->yt.p, 0, (size_t)h->n * p.mb * sizeof(double), s));
        launch_scan_seq(p, lp, perm, sv, h->ldn, h->n, ztb, mc, h->yt.p, p.mb, false, kcc,
                        h->agg.p, seg + K * c0, ld_seg, 1, s);
        launch_block_out(h->yt.p, p.mb, mc, nullptr, nullptr, nullptr, Y + c0, ldy, 0, h->n, s);
        h->kernel_launches += 2;
      } else {
        launch_scan_seq(p, lp, perm, sv, h->ldn, h->n, ztb, mc, h->U.p + c0, m, true, kcc,
                        h->agg.p, seg + K * c0, ld_seg, 1, s);
        h->kernel_launches++;
      }
      h->launches[kAcc]++;
      if (h->timing) h->acc_pairs += h->n * kcc;
    }
    if (!p.scatter) {
      TimedScope ts(h, kAcc, s);
      launch_accumulate(p, h->rank.p, h->ldn, h->n, h->U.p, k_first, kcc, h->hsum.p, h->Sg.p, Y,
                        ldy, m, c == 0, c == p.chunks - 1, nullptr, 0, h->n, s, 1.0, false);
      h->kernel_launches++;
    }
  }
  CUDA_TRY(cudaGetLastError());
  h->queries++;
  h->m_last = m;
  return L1DM_OK;
}

l1dm_status read_timeout(l1dm_ctx *h) {
  if (!h->ctr.p) return L1DM_OK;
  unsigned f = 0;
  CUDA_TRY(cudaMemcpy(&f, h->ctr.p + 1, sizeof(unsigned), cudaMemcpyDeviceToHost));
  if (f) {
    unsigned zero = 0;
    cudaMemcpy(h->ctr.p + 1, &zero, sizeof(unsigned), cudaMemcpyHostToDevice);
    return fail(L1DM_ETIMEOUT, "scan look-back wait exceeded its bound; results invalid");
  }
  return L1DM_OK;
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

l1dm_status l1dm_prepare_ex(const float *X, int64_t n, int64_t ld_x, int64_t k_begin,
                            int64_t k_end, void *stream, l1dm_handle *out) {
  NvtxRange nvtx_("l1dm_prepare_ex");
  g_err.clear();
  if (!out) return fail(L1DM_EINVAL, "out is NULL");
  *out = nullptr;
  if (!X) return fail(L1DM_EINVAL, "X is NULL");
  if (n < 1 || n > (int64_t)0xFFFFFFFFLL)
    return fail(L1DM_EINVAL, "n=%lld out of range [1, 2^32)", (long long)n);
  if (k_begin < 0 || k_end <= k_begin || k_end > ld_x)
    return fail(L1DM_EINVAL, "coordinate range [%lld,%lld) invalid for ld_x=%lld",
                (long long)k_begin, (long long)k_end, (long long)ld_x);
  l1dm_ctx *h = new (std::nothrow) l1dm_ctx();
  if (!h) return fail(L1DM_ENOMEM, "host allocation failed");
  l1dm_status st = prepare_impl(X, n, ld_x, k_begin, k_end, stream, h);
  if (st != L1DM_OK) {
    std::string keep = g_err;
    destroy(h);
    g_err = keep;
    return st;
  }
  *out = h;
  return L1DM_OK;
}

l1dm_status l1dm_prepare(const float *X, int64_t n, int64_t d, l1dm_handle *out) {
  if (d < 1) {
    if (out) *out = nullptr;
    return fail(L1DM_EINVAL, "d=%lld < 1", (long long)d);
  }
  return l1dm_prepare_ex(X, n, d, 0, d, nullptr, out);
}

}  // extern "C"

namespace {

enum QueryKind { kQueryL1 = 0, kQueryLp = 1, kQueryTV = 2 };

// TV precondition (Thm. tv; "rows of X on the probability simplex"):
// every prepared coordinate >= 0 and, for a handle holding whole rows, |sum_k x_ik - 1| <=
// 1e-9 + d 2^-23 (fp32 rows of a distribution carry ~2^-24 relative rounding per entry,
// DESIGN.md reading R17).  Computed once per handle (the prepared state is immutable).
l1dm_status check_simplex(l1dm_ctx *h, cudaStream_t s) {
  if (h->simplex < 0) {
    DevBuf<double> out;
    CUDA_TRY(out.ensure(2, false, s));
    launch_simplex_stats(h->hsum.p, h->n, reinterpret_cast<const float *>(h->sval_bits.p), h->ldn,
                         h->dl, out.p, s);
    double host[2];
    CUDA_TRY(cudaMemcpyAsync(host, out.p, sizeof(host), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    out.release();
    h->simplex_dev = host[0];
    h->simplex_min = host[1];
    const double tol = 1e-9 + (double)h->dl * std::ldexp(1.0, -23);
    h->simplex = (host[1] >= 0.0 && (!h->full_rows || host[0] <= tol)) ? 1 : 0;
  }
  if (!h->simplex)
    return fail(L1DM_ENOTSIMPLEX,
                "rows are not on the probability simplex (min coordinate %.3g, max |sum - 1| "
                "%.3g%s)", h->simplex_min, h->simplex_dev,
                h->full_rows ? "" : "; row sums not checkable on a coordinate shard");
  return L1DM_OK;
}

l1dm_status dispatch(l1dm_ctx *h, int kind, int lp, const float *Z, int64_t ldz, int64_t m,
                     double *Y, int64_t ldy, cudaStream_t s, int64_t nblocks = 1,
                     void *const *events = nullptr) {
  if (kind == kQueryTV) {
    l1dm_status st = check_simplex(h, s);
    if (st != L1DM_OK) return st;
  }
  if (kind == kQueryLp && lp > 1) return lp_device(h, lp, Z, ldz, m, Y, ldy, s);
  l1dm_status st = matvec_device(h, Z, ldz, m, Y, ldy, s, nblocks, events);
  if (st == L1DM_OK && kind == kQueryTV) {
    TimedScope ts(h, kAcc, s);
    launch_scale(Y, ldy, h->n, m, 0.5, s);  // TV(x, y) = ||x - y||_1 / 2
    h->kernel_launches++;
  }
  return st;
}

// 2-D copy of `rows` rows of `width` bytes; a contiguous block (pitches == width) goes as one
// 1-D copy (the 2-D engine path moves narrow rows one by one: ~100x slower for m = 1).
cudaError_t copy_rows(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width,
                      size_t rows, cudaMemcpyKind kind, cudaStream_t s) {
  if (dpitch == width && spitch == width) return cudaMemcpyAsync(dst, src, width * rows, kind, s);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, kind, s);
}

bool is_pinned_host(const void *ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Pinned host Z and Y: asynchronous, stream-ordered like device buffers (l1dm_sync before
// reading Y or reusing Z).  Slot q&1: H2D of Z on cp_in (after the compute that last read the
// slot), the query on the handle's stream, D2H of Y on cp_out; consecutive calls overlap.
l1dm_status pinned_pipeline(l1dm_ctx *h, int kind, int lp, const float *Z, int64_t ld_z, int64_t m,
                            double *Y, int64_t ld_y, cudaStream_t s) {
  if (!h->cp_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->cp_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&h->cp_out, cudaStreamNonBlocking));
    for (int q = 0; q < 2; ++q) {
      CUDA_TRY(cudaEventCreateWithFlags(&h->ev_in[q], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&h->ev_done[q], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&h->ev_out[q], cudaEventDisableTiming));
    }
  }
  const unsigned q = h->pin_slot++ & 1u;
  if (h->Zpin[q].count < (size_t)h->n * m || h->Ypin[q].count < (size_t)h->n * m) {
    // (re)allocation: drain every user of the slot first
    CUDA_TRY(cudaStreamSynchronize(h->cp_in));
    CUDA_TRY(cudaStreamSynchronize(h->cp_out));
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(h->Zpin[q].ensure((size_t)h->n * (size_t)m, false, s));
    CUDA_TRY(h->Ypin[q].ensure((size_t)h->n * (size_t)m, false, s));
  }
  CUDA_TRY(cudaStreamWaitEvent(h->cp_in, h->ev_done[q], 0));  // slot's Z no longer read
  {
    TimedScope ts(h, kCopy, h->cp_in);
    CUDA_TRY(copy_rows(h->Zpin[q].p, (size_t)m * sizeof(float), Z, (size_t)ld_z * sizeof(float),
                       (size_t)m * sizeof(float), (size_t)h->n, cudaMemcpyHostToDevice, h->cp_in));
  }
  CUDA_TRY(cudaEventRecord(h->ev_in[q], h->cp_in));
  CUDA_TRY(cudaStreamWaitEvent(s, h->ev_in[q], 0));
  CUDA_TRY(cudaStreamWaitEvent(s, h->ev_out[q], 0));  // slot's Y copied out
  l1dm_status st = dispatch(h, kind, lp, h->Zpin[q].p, m, m, h->Ypin[q].p, m, s);
  if (st != L1DM_OK) return st;
  CUDA_TRY(cudaEventRecord(h->ev_done[q], s));
  CUDA_TRY(cudaStreamWaitEvent(h->cp_out, h->ev_done[q], 0));
  {
    TimedScope ts(h, kCopy, h->cp_out);
    CUDA_TRY(copy_rows(Y, (size_t)ld_y * sizeof(double), h->Ypin[q].p, (size_t)m * sizeof(double),
                       (size_t)m * sizeof(double), (size_t)h->n, cudaMemcpyDeviceToHost,
                       h->cp_out));
  }
  CUDA_TRY(cudaEventRecord(h->ev_out[q], h->cp_out));
  return L1DM_OK;
}

// Argument checks, host-buffer staging and the call: shared by the l1, l_p and TV entries.
l1dm_status query_entry(l1dm_handle h, int kind, int lp, const float *Z, int64_t ld_z, int64_t m,
                        double *Y, int64_t ld_y, void *stream) {
  g_err.clear();
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  if (!Z || !Y) return fail(L1DM_EINVAL, "Z or Y is NULL");
  if (m < 1 || ld_z < m || ld_y < m)
    return fail(L1DM_EINVAL, "m=%lld ld_z=%lld ld_y=%lld invalid", (long long)m, (long long)ld_z,
                (long long)ld_y);
  if (kind == kQueryLp && (lp < 1 || lp > 7 || !(lp & 1)))
    return fail(L1DM_EINVAL, "p=%d: odd p in {1, 3, 5, 7} only (even p needs no sort)", lp);
  l1dm_status st = check_device(h);
  if (st != L1DM_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;  // NULL: legacy default stream
  h->last_stream = s;
  const bool zdev = is_device_pointer(Z), ydev = is_device_pointer(Y);
  if (zdev && ydev) return dispatch(h, kind, lp, Z, ld_z, m, Y, ld_y, s);
  if (is_pinned_host(Z) && is_pinned_host(Y)) return pinned_pipeline(h, kind, lp, Z, ld_z, m, Y, ld_y, s);
  // pageable host buffers: stage through library-owned device memory; synchronous
  const float *Zd = Z;
  int64_t ldzd = ld_z;
  if (!zdev) {
    CUDA_TRY(h->Zstage.ensure((size_t)h->n * (size_t)m, false, s));
    TimedScope ts(h, kCopy, s);
    CUDA_TRY(copy_rows(h->Zstage.p, (size_t)m * sizeof(float), Z, (size_t)ld_z * sizeof(float),
                       (size_t)m * sizeof(float), (size_t)h->n, cudaMemcpyHostToDevice, s));
    Zd = h->Zstage.p;
    ldzd = m;
  }
  double *Yd = Y;
  int64_t ldyd = ld_y;
  if (!ydev) {
    CUDA_TRY(h->Ystage.ensure((size_t)h->n * (size_t)m, false, s));
    Yd = h->Ystage.p;
    ldyd = m;
  }
  st = dispatch(h, kind, lp, Zd, ldzd, m, Yd, ldyd, s);
  if (st != L1DM_OK) return st;
  if (!ydev) {
    TimedScope ts(h, kCopy, s);
    CUDA_TRY(copy_rows(Y, (size_t)ld_y * sizeof(double), Yd, (size_t)m * sizeof(double),
                       (size_t)m * sizeof(double), (size_t)h->n, cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  return read_timeout(h);
}

}  // namespace

extern "C" {

l1dm_status l1dm_matvec_ex(l1dm_handle h, const float *Z, int64_t ld_z, int64_t m, double *Y,
                           int64_t ld_y, void *stream) {
  NvtxRange nvtx_("l1dm_matvec_ex");
  return query_entry(h, kQueryL1, 1, Z, ld_z, m, Y, ld_y, stream);
}

l1dm_status l1dm_matvec_lp_ex(l1dm_handle h, int p, const float *Z, int64_t ld_z, int64_t m,
                              double *Y, int64_t ld_y, void *stream) {
  NvtxRange nvtx_("l1dm_matvec_lp_ex");
  return query_entry(h, kQueryLp, p, Z, ld_z, m, Y, ld_y, stream);
}

l1dm_status l1dm_matvec_lp(l1dm_handle h, int p, const float *Z, int64_t m, double *Y) {
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  return query_entry(h, kQueryLp, p, Z, m, m, Y, m, (void *)h->stream);
}

l1dm_status l1dm_tv_matvec_ex(l1dm_handle h, const float *Z, int64_t ld_z, int64_t m, double *Y,
                              int64_t ld_y, void *stream) {
  NvtxRange nvtx_("l1dm_tv_matvec_ex");
  return query_entry(h, kQueryTV, 1, Z, ld_z, m, Y, ld_y, stream);
}

l1dm_status l1dm_tv_matvec(l1dm_handle h, const float *Z, int64_t m, double *Y) {
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  return query_entry(h, kQueryTV, 1, Z, m, m, Y, m, (void *)h->stream);
}

}  // extern "C"

namespace {

std::atomic<int64_t> g_handleless_launches{0};

// Shared by the handle-free sort-free entries: argument checks, host staging through the
// stream-ordered allocator, the launch, the copy back.  M (bilinear only): d x d fp64.
l1dm_status sortfree_entry(const float *X, int64_t n, int64_t ld_x, int64_t d, int p,
                           const double *M, const float *Z, int64_t ld_z, int64_t m, double *Y,
                           int64_t ld_y, void *stream) {
  g_err.clear();
  const bool bilinear = (p == 0);
  if (!X || !Z || !Y || (bilinear && !M)) return fail(L1DM_EINVAL, "X, M, Z or Y is NULL");
  if (n < 1 || d < 1 || m < 1 || ld_x < d || ld_z < m || ld_y < m)
    return fail(L1DM_EINVAL, "n=%lld d=%lld m=%lld ld_x=%lld ld_z=%lld ld_y=%lld invalid",
                (long long)n, (long long)d, (long long)m, (long long)ld_x, (long long)ld_z,
                (long long)ld_y);
  if (!bilinear && p != 2 && p != 4 && p != 6)
    return fail(L1DM_EINVAL, "p=%d: even p in {2, 4, 6} only", p);
  int dev = 0;
  l1dm_status st = check_arch(&dev);
  if (st != L1DM_OK) return st;
  int sms = 148;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t s = (cudaStream_t)stream;
  const bool xdev = is_device_pointer(X), zdev = is_device_pointer(Z), ydev = is_device_pointer(Y);
  const bool mdev = bilinear && is_device_pointer(M);
  // stream-ordered scratch (cudaMallocAsync): the call stays asynchronous for device buffers
  const size_t wsb = bilinear ? bilinear_workspace(n, d, m, sms)
                              : lpp_even_workspace(n, d, m, p, nullptr, nullptr, sms);
  void *ws = nullptr, *xs = nullptr, *zs = nullptr, *ys = nullptr, *ms = nullptr;
  auto release = [&]() {
    for (void *q : {ws, xs, zs, ys, ms})
      if (q) cudaFreeAsync(q, s);
  };
  keep_default_pool();
  cudaError_t e = cudaMallocAsync(&ws, wsb, s);
  const float *Xd = X, *Zd = Z;
  const double *Md = M;
  double *Yd = Y;
  int64_t ldxd = ld_x, ldzd = ld_z, ldyd = ld_y;
  if (e == cudaSuccess && !xdev) {
    e = cudaMallocAsync(&xs, (size_t)n * d * sizeof(float), s);
    if (e == cudaSuccess)
      e = copy_rows(xs, (size_t)d * sizeof(float), X, (size_t)ld_x * sizeof(float),
                    (size_t)d * sizeof(float), (size_t)n, cudaMemcpyHostToDevice, s);
    Xd = static_cast<const float *>(xs);
    ldxd = d;
  }
  if (e == cudaSuccess && !zdev) {
    e = cudaMallocAsync(&zs, (size_t)n * m * sizeof(float), s);
    if (e == cudaSuccess)
      e = copy_rows(zs, (size_t)m * sizeof(float), Z, (size_t)ld_z * sizeof(float),
                    (size_t)m * sizeof(float), (size_t)n, cudaMemcpyHostToDevice, s);
    Zd = static_cast<const float *>(zs);
    ldzd = m;
  }
  if (e == cudaSuccess && bilinear && !mdev) {
    e = cudaMallocAsync(&ms, (size_t)d * d * sizeof(double), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ms, M, (size_t)d * d * sizeof(double), cudaMemcpyHostToDevice, s);
    Md = static_cast<const double *>(ms);
  }
  if (e == cudaSuccess && !ydev) {
    e = cudaMallocAsync(&ys, (size_t)n * m * sizeof(double), s);
    Yd = static_cast<double *>(ys);
    ldyd = m;
  }
  if (e != cudaSuccess) {
    release();
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? L1DM_ENOMEM : L1DM_ECUDA, "sort-free setup: %s",
                cudaGetErrorString(e));
  }
  g_handleless_launches +=
      bilinear
          ? launch_bilinear(Xd, ldxd, Md, Zd, ldzd, n, d, m, Yd, ldyd, static_cast<double *>(ws),
                            sms, s)
          : launch_lpp_even(Xd, ldxd, Zd, ldzd, n, d, m, p, Yd, ldyd, static_cast<double *>(ws),
                            sms, s);
  e = cudaGetLastError();
  if (e == cudaSuccess && !ydev)
    e = copy_rows(Y, (size_t)ld_y * sizeof(double), Yd, (size_t)m * sizeof(double),
                  (size_t)m * sizeof(double), (size_t)n, cudaMemcpyDeviceToHost, s);
  release();
  if (e == cudaSuccess && !(xdev && zdev && ydev && (!bilinear || mdev)))
    e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(L1DM_ECUDA, "sort-free query: %s", cudaGetErrorString(e));
  return L1DM_OK;
}

}  // namespace

extern "C" {

l1dm_status l1dm_lpp_even_matvec(const float *X, int64_t n, int64_t ld_x, int64_t d, int p,
                                 const float *Z, int64_t ld_z, int64_t m, double *Y, int64_t ld_y,
                                 void *stream) {
  NvtxRange nvtx_("l1dm_lpp_even_matvec");
  if (p == 0) return fail(L1DM_EINVAL, "p=0: even p in {2, 4, 6} only");
  return sortfree_entry(X, n, ld_x, d, p, nullptr, Z, ld_z, m, Y, ld_y, stream);
}

l1dm_status l1dm_bilinear_matvec(const float *X, int64_t n, int64_t ld_x, int64_t d,
                                 const double *M, const float *Z, int64_t ld_z, int64_t m,
                                 double *Y, int64_t ld_y, void *stream) {
  NvtxRange nvtx_("l1dm_bilinear_matvec");
  return sortfree_entry(X, n, ld_x, d, 0, M, Z, ld_z, m, Y, ld_y, stream);
}

l1dm_status l1dm_l2_embed(const float *X, int64_t n, int64_t ld_x, int64_t d, const float *G,
                          int64_t k, float *Xp, int64_t ld_p, void *stream) {
  NvtxRange nvtx_("l1dm_l2_embed");
  g_err.clear();
  if (!X || !G || !Xp) return fail(L1DM_EINVAL, "X, G or Xp is NULL");
  if (n < 1 || d < 1 || k < 1 || ld_x < d || ld_p < k)
    return fail(L1DM_EINVAL, "n=%lld d=%lld k=%lld ld_x=%lld ld_p=%lld invalid", (long long)n,
                (long long)d, (long long)k, (long long)ld_x, (long long)ld_p);
  int dev = 0;
  l1dm_status st = check_arch(&dev);
  if (st != L1DM_OK) return st;
  if (!is_device_pointer(X) || !is_device_pointer(G) || !is_device_pointer(Xp))
    return fail(L1DM_EINVAL, "l1dm_l2_embed needs device X, G and Xp");
  cudaStream_t s = (cudaStream_t)stream;
  g_handleless_launches += launch_embed(X, ld_x, n, d, G, d, k, Xp, ld_p, s);
  CUDA_TRY(cudaGetLastError());
  return L1DM_OK;
}

l1dm_status l1dm_matvec_pipelined(l1dm_handle h, const float *Z, int64_t ld_z, int64_t m,
                                  double *Y, int64_t ld_y, void *stream, int64_t point_blocks,
                                  void *const *block_events) {
  NvtxRange nvtx_("l1dm_matvec_pipelined");
  g_err.clear();
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  if (!Z || !Y) return fail(L1DM_EINVAL, "Z or Y is NULL");
  if (m < 1 || ld_z < m || ld_y < m || point_blocks < 1 || point_blocks > h->n)
    return fail(L1DM_EINVAL, "m=%lld ld_z=%lld ld_y=%lld point_blocks=%lld invalid", (long long)m,
                (long long)ld_z, (long long)ld_y, (long long)point_blocks);
  l1dm_status st = check_device(h);
  if (st != L1DM_OK) return st;
  if (!is_device_pointer(Z) || !is_device_pointer(Y))
    return fail(L1DM_EINVAL, "l1dm_matvec_pipelined needs device Z and Y");
  cudaStream_t s = (cudaStream_t)stream;
  h->last_stream = s;
  return matvec_device(h, Z, ld_z, m, Y, ld_y, s, point_blocks, block_events);
}

// ---------------------------------------------------------------- peer-memory collective
l1dm_status l1dm_ipc_alloc(size_t bytes, void **dptr, void *handle) {
  g_err.clear();
  if (!dptr || !handle || bytes == 0) return fail(L1DM_EINVAL, "dptr/handle NULL or bytes == 0");
  int dev = 0;
  l1dm_status st = check_arch(&dev);
  if (st != L1DM_OK) return st;
  void *p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? L1DM_ENOMEM : L1DM_ECUDA, "cudaMalloc(%zu): %s",
                bytes, cudaGetErrorString(e));
  }
  CUDA_TRY(cudaMemset(p, 0, bytes));
  cudaIpcMemHandle_t hd;
  e = cudaIpcGetMemHandle(&hd, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    cudaGetLastError();
    return fail(L1DM_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  }
  memcpy(handle, &hd, sizeof(hd));
  *dptr = p;
  return L1DM_OK;
}

l1dm_status l1dm_ipc_free(void *dptr) {
  g_err.clear();
  if (dptr) CUDA_TRY(cudaFree(dptr));
  return L1DM_OK;
}

l1dm_status l1dm_ipc_open(const void *handle, void **dptr) {
  g_err.clear();
  if (!handle || !dptr) return fail(L1DM_EINVAL, "handle or dptr is NULL");
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle, sizeof(hd));
  CUDA_TRY(cudaIpcOpenMemHandle(dptr, hd, cudaIpcMemLazyEnablePeerAccess));
  return L1DM_OK;
}

l1dm_status l1dm_ipc_close(void *dptr) {
  g_err.clear();
  if (dptr) CUDA_TRY(cudaIpcCloseMemHandle(dptr));
  return L1DM_OK;
}

namespace {
l1dm_status check_peers(const l1dm_peer_t *pr, int64_t n, int64_t m) {
  if (!pr) return fail(L1DM_EINVAL, "peers is NULL");
  if (pr->n < 1 || pr->m < 1 || n != pr->n || m != pr->m)
    return fail(L1DM_EINVAL, "n=%lld m=%lld do not match the peer buffers (n=%lld m=%lld)",
                (long long)n, (long long)m, (long long)pr->n, (long long)pr->m);
  if (pr->world < 1 || pr->world > L1DM_MAX_PEERS || pr->rank < 0 || pr->rank >= pr->world)
    return fail(L1DM_EINVAL, "world=%d rank=%d invalid (1 <= world <= %d)", pr->world, pr->rank,
                L1DM_MAX_PEERS);
  for (int o = 0; o < pr->world; ++o)
    if (!pr->inbox[o] || !pr->flags[o])
      return fail(L1DM_EINVAL, "inbox/flags of rank %d not mapped", o);
  if (!pr->timeout) return fail(L1DM_EINVAL, "timeout word is NULL");
  return L1DM_OK;
}
}  // namespace

l1dm_status l1dm_matvec_push(l1dm_handle h, const float *Z, int64_t ld_z, int64_t m,
                             const l1dm_peer_t *peers, unsigned epoch, void *stream) {
  NvtxRange nvtx_("l1dm_matvec_push");
  g_err.clear();
  if (!h || !Z) return fail(L1DM_EINVAL, "handle or Z is NULL");
  if (m < 1 || ld_z < m) return fail(L1DM_EINVAL, "m=%lld ld_z=%lld invalid", (long long)m,
                                     (long long)ld_z);
  l1dm_status st = check_peers(peers, h->n, m);
  if (st != L1DM_OK) return st;
  if (epoch == 0) return fail(L1DM_EINVAL, "epoch 0 is reserved (the flags' initial value)");
  st = check_device(h);
  if (st != L1DM_OK) return st;
  if (!is_device_pointer(Z)) return fail(L1DM_EINVAL, "l1dm_matvec_push needs a device Z");
  cudaStream_t s = (cudaStream_t)stream;
  h->last_stream = s;
  const int G = peers->world, g = peers->rank;
  PeerDst pd{};
  pd.world = G;
  pd.ld = m;
  for (int o = 0; o <= G; ++o) pd.row0[o] = peer_row0(h->n, G, o);
  const size_t par = epoch & 1u;  // inbox half of this epoch (double-buffered, see l1dm_peer.cu)
  for (int o = 0; o < G; ++o)
    pd.slot[o] = peers->inbox[o] +
                 (par * G + (size_t)g) * (size_t)(pd.row0[o + 1] - pd.row0[o]) * m;
  // fused when the final pass is k6 (gather) or k9 (scatter, m > 1); otherwise the partial is
  // computed locally and pushed by k30
  bool fused = false;
  if (!use_runs(h)) {
    st = ensure_plan(h, m, vec_cap_for(Z, ld_z));
    if (st != L1DM_OK) return st;
    fused = !(h->plan.scatter && m == 1);
  }
  const bool need_scratch = !fused || (!h->plan.scatter && h->plan.chunks > 1);
  if (need_scratch) CUDA_TRY(h->ypush.ensure((size_t)h->n * (size_t)m, false, s));
  if (fused) {
    st = matvec_device(h, Z, ld_z, m, h->ypush.p, m, s, 1, nullptr, false, &pd);
  } else {
    st = matvec_device(h, Z, ld_z, m, h->ypush.p, m, s);
    if (st == L1DM_OK) {
      launch_push_rows(h->ypush.p, m, m, 0, h->n, pd, s);
      h->kernel_launches++;
    }
  }
  if (st != L1DM_OK) return st;
  launch_peer_signal(peers->flags, G, g, epoch, s);  // arrival of rank g at every owner
  h->kernel_launches++;
  CUDA_TRY(cudaGetLastError());
  return L1DM_OK;
}

l1dm_status l1dm_peer_reduce(const l1dm_peer_t *peers, int64_t n, int64_t m, unsigned epoch,
                             unsigned targets, void *stream) {
  NvtxRange nvtx_("l1dm_peer_reduce");
  g_err.clear();
  l1dm_status st = check_peers(peers, n, m);
  if (st != L1DM_OK) return st;
  if (n < 1 || m < 1 || epoch == 0) return fail(L1DM_EINVAL, "n, m >= 1 and epoch > 0 required");
  const int G = peers->world, g = peers->rank;
  double *tp[L1DM_MAX_PEERS];
  int64_t tl[L1DM_MAX_PEERS];
  unsigned *tf[L1DM_MAX_PEERS];
  int nt = 0;
  for (int t = 0; t < G; ++t) {
    if (!((targets >> t) & 1u)) continue;
    if (!peers->ybuf[t]) return fail(L1DM_EINVAL, "target %d has no result buffer mapped", t);
    tp[nt] = peers->ybuf[t];
    tl[nt] = m;
    tf[nt] = peers->flags[t];
    ++nt;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t r0 = peer_row0(n, G, g), r1 = peer_row0(n, G, g + 1);
  const double *half = peers->inbox[g] + (size_t)(epoch & 1u) * G * (size_t)(r1 - r0) * m;
  launch_peer_reduce(peers->flags[g], G, epoch, half, r1 - r0, m, r0, tp, tl, nt,
                     peers->timeout, s);
  if (nt) launch_peer_signal(tf, nt, G + g, epoch, s);  // owner g's rows are at every target
  CUDA_TRY(cudaGetLastError());
  return L1DM_OK;
}

l1dm_status l1dm_peer_wait(const l1dm_peer_t *peers, unsigned epoch, int64_t n, int64_t m,
                           double *Y, int64_t ld_y, void *stream) {
  NvtxRange nvtx_("l1dm_peer_wait");
  g_err.clear();
  l1dm_status st = check_peers(peers, n, m);
  if (st != L1DM_OK) return st;
  if (epoch == 0) return fail(L1DM_EINVAL, "epoch 0 is reserved");
  const int G = peers->world, g = peers->rank;
  cudaStream_t s = (cudaStream_t)stream;
  launch_peer_wait(peers->flags[g] + G, G, epoch, peers->timeout, s);
  if (Y) {
    if (!peers->ybuf[g]) return fail(L1DM_EINVAL, "this rank has no result buffer");
    if (n < 1 || m < 1 || ld_y < m) return fail(L1DM_EINVAL, "n, m, ld_y invalid");
    CUDA_TRY(copy_rows(Y, (size_t)ld_y * sizeof(double), peers->ybuf[g], (size_t)m * sizeof(double),
                       (size_t)m * sizeof(double), (size_t)n, cudaMemcpyDeviceToDevice, s));
  }
  CUDA_TRY(cudaGetLastError());
  return L1DM_OK;
}

l1dm_status l1dm_peer_check(const l1dm_peer_t *peers, void *stream) {
  g_err.clear();
  if (!peers || !peers->timeout) return fail(L1DM_EINVAL, "peers or timeout word is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned f = 0;
  CUDA_TRY(cudaMemcpyAsync(&f, peers->timeout, sizeof(f), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (f) {
    const unsigned zero = 0;
    CUDA_TRY(cudaMemcpy(peers->timeout, &zero, sizeof(zero), cudaMemcpyHostToDevice));
    return fail(L1DM_ETIMEOUT, "a peer flag wait exceeded its bound; the result is invalid");
  }
  return L1DM_OK;
}

l1dm_status l1dm_query_layout(l1dm_handle h, int64_t m, int64_t *scatter, int64_t *mb,
                              int64_t *col_blocks) {
  g_err.clear();
  if (!h || m < 1) return fail(L1DM_EINVAL, "handle is NULL or m < 1");
  l1dm_status st = ensure_plan(h, m, 4);
  if (st != L1DM_OK) return st;
  if (scatter) *scatter = use_runs(h) ? 0 : h->plan.scatter;  // runs: point-block overlap
  if (mb) *mb = h->plan.mb;
  if (col_blocks) *col_blocks = h->plan.col_blocks;
  return L1DM_OK;
}

l1dm_status l1dm_query_strategy(l1dm_handle h, int64_t m, int *strategy) {
  g_err.clear();
  if (!h || m < 1 || !strategy) return fail(L1DM_EINVAL, "handle/strategy NULL or m < 1");
  if (use_runs(h)) {
    *strategy = L1DM_STRATEGY_RUNS;
    return L1DM_OK;
  }
  l1dm_status st = ensure_plan(h, m, 4);
  if (st != L1DM_OK) return st;
  *strategy = h->plan.scatter ? L1DM_STRATEGY_SCATTER : L1DM_STRATEGY_GATHER;
  return L1DM_OK;
}

l1dm_status l1dm_matvec_colblocks(l1dm_handle h, const float *Z, int64_t ld_z, int64_t m,
                                  double *Yb, void *stream, int64_t nevents,
                                  void *const *events) {
  NvtxRange nvtx_("l1dm_matvec_colblocks");
  g_err.clear();
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  if (!Z || !Yb || m < 2 || ld_z < m)
    return fail(L1DM_EINVAL, "Z/Yb NULL, m < 2 or ld_z < m");
  l1dm_status st = check_device(h);
  if (st != L1DM_OK) return st;
  if (!is_device_pointer(Z) || !is_device_pointer(Yb))
    return fail(L1DM_EINVAL, "l1dm_matvec_colblocks needs device Z and Yb");
  st = ensure_plan(h, m, vec_cap_for(Z, ld_z));
  if (st != L1DM_OK) return st;
  if (!h->plan.scatter)
    return fail(L1DM_EINVAL, "column-block output needs the scatter strategy (plan is gather)");
  if (nevents != 0 && nevents != h->plan.col_blocks)
    return fail(L1DM_EINVAL, "nevents=%lld, plan has %d column blocks", (long long)nevents,
                h->plan.col_blocks);
  cudaStream_t s = (cudaStream_t)stream;
  h->last_stream = s;
  return matvec_device(h, Z, ld_z, m, Yb, h->plan.mb, s, h->plan.col_blocks,
                       nevents ? events : nullptr, true);
}

l1dm_status l1dm_unblock(const double *Yb, int64_t n, int64_t m, int64_t mb, double *Y,
                         int64_t ld_y, void *stream) {
  g_err.clear();
  if (!Yb || !Y || n < 1 || m < 1 || mb < 1 || ld_y < m)
    return fail(L1DM_EINVAL, "invalid unblock arguments");
  int dev = 0;
  l1dm_status st = check_arch(&dev);
  if (st != L1DM_OK) return st;
  launch_unblock(Yb, n, m, mb, Y, ld_y, (cudaStream_t)stream);
  CUDA_TRY(cudaGetLastError());
  return L1DM_OK;
}

l1dm_status l1dm_matvec(l1dm_handle h, const float *Z, int64_t m, double *Y) {
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  return l1dm_matvec_ex(h, Z, m, m, Y, m, (void *)h->stream);
}

void l1dm_free(l1dm_handle h) { destroy(h); }

l1dm_status l1dm_sync(l1dm_handle h) {
  g_err.clear();
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  DeviceGuard dg(h->device);
  if (h->cp_in) CUDA_TRY(cudaStreamSynchronize(h->cp_in));
  if (h->cp_out) CUDA_TRY(cudaStreamSynchronize(h->cp_out));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (h->last_stream != h->stream) CUDA_TRY(cudaStreamSynchronize(h->last_stream));
  return read_timeout(h);
}

l1dm_status l1dm_shape(l1dm_handle h, int64_t *n, int64_t *d_local, int64_t *k_begin,
                       int64_t *k_end) {
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  if (n) *n = h->n;
  if (d_local) *d_local = h->dl;
  if (k_begin) *k_begin = h->k_begin;
  if (k_end) *k_end = h->k_end;
  return L1DM_OK;
}

size_t l1dm_workspace_bytes(l1dm_handle h, int64_t m) {
  if (!h || m < 1) return 0;
  QueryPlan p;
  int64_t ws = (int64_t)h->ws_limit;
  if (ws == 0) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return 0;
    ws = (int64_t)(0.75 * (double)fr);
  }
  if (!make_plan(h->n, h->dl, m, h->l2_bytes, ws, 4, h->mode, &p)) return 0;
  return p.workspace_bytes;
}

l1dm_status l1dm_set_query_mode(l1dm_handle h, int mode) {
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  if (mode < L1DM_MODE_AUTO || mode > L1DM_MODE_RUNS)
    return fail(L1DM_EINVAL, "unknown query mode %d", mode);
  if (mode == L1DM_MODE_RUNS && !h->has_runs)
    return fail(L1DM_EINVAL, "runs mode needs <= 256 distinct values in every coordinate");
  h->mode = mode;
  h->plan_m = -1;
  return L1DM_OK;
}

l1dm_status l1dm_set_workspace_limit(l1dm_handle h, size_t bytes) {
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  h->ws_limit = bytes;
  h->plan_m = -1;
  return L1DM_OK;
}

l1dm_status l1dm_plan(int64_t n, int64_t d_local, int64_t m, int64_t l2_bytes,
                      int64_t workspace_limit, l1dm_plan_t *out) {
  return l1dm_plan_ex(n, d_local, m, l2_bytes, workspace_limit, L1DM_MODE_AUTO, out);
}

l1dm_status l1dm_plan_ex(int64_t n, int64_t d_local, int64_t m, int64_t l2_bytes,
                         int64_t workspace_limit, int mode, l1dm_plan_t *out) {
  if (!out) return fail(L1DM_EINVAL, "out is NULL");
  if (mode < L1DM_MODE_AUTO || mode > L1DM_MODE_SCATTER)
    return fail(L1DM_EINVAL, "unknown query mode %d", mode);
  QueryPlan p;
  if (!make_plan(n, d_local, m, l2_bytes, workspace_limit, 4, mode, &p))
    return fail(L1DM_EINVAL, "invalid sizes n=%lld d=%lld m=%lld", (long long)n,
                (long long)d_local, (long long)m);
  out->mb = p.mb;
  out->col_blocks = p.col_blocks;
  out->vec = p.vec;
  out->lanes_per_row = p.lpr;
  out->rows_per_tile = p.rows_per_tile;
  out->tiles_per_segment = p.tiles_per_segment;
  out->kc = p.kc;
  out->chunks = p.chunks;
  out->l2_resident = p.l2_resident;
  out->workspace_bytes = (int64_t)p.workspace_bytes;
  out->scatter = p.scatter;
  return L1DM_OK;
}

l1dm_status l1dm_timing_enable(l1dm_handle h, int enable) {
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  h->timing = enable != 0;
  return L1DM_OK;
}

l1dm_status l1dm_timing_read(l1dm_handle h, l1dm_timing_t *out, int reset) {
  if (!h || !out) return fail(L1DM_EINVAL, "handle or out is NULL");
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (h->last_stream != h->stream) CUDA_TRY(cudaStreamSynchronize(h->last_stream));
  for (auto &tp : h->pending) {
    float ms = 0.f;
    cudaEventSynchronize(tp.b);
    if (cudaEventElapsedTime(&ms, tp.a, tp.b) == cudaSuccess) h->ms[tp.kind] += ms;
    h->pool.push_back(tp.a);
    h->pool.push_back(tp.b);
  }
  h->pending.clear();
  out->prep_ms = h->prep_ms;
  out->colsums_ms = h->ms[kColsums];
  out->scan_ms = h->ms[kScan];
  out->accumulate_ms = h->ms[kAcc];
  out->copy_ms = h->ms[kCopy];
  out->colsums_launches = h->launches[kColsums];
  out->scan_launches = h->launches[kScan];
  out->accumulate_launches = h->launches[kAcc];
  out->queries = h->queries;
  out->kernel_launches = h->kernel_launches;
  out->scan_pairs = h->scan_pairs;
  out->accumulate_pairs = h->acc_pairs;
  out->m_last = h->m_last;
  if (reset) {
    h->scan_pairs = 0;
    h->acc_pairs = 0;
    for (int k = 0; k < kNumKinds; ++k) {
      h->ms[k] = 0.0;
      h->launches[k] = 0;
    }
    h->queries = 0;
    h->kernel_launches = 0;
  }
  return L1DM_OK;
}

l1dm_status l1dm_debug_export(l1dm_handle h, float *sval, uint32_t *perm, uint32_t *rank,
                              double *hsum) {
  if (!h) return fail(L1DM_EINVAL, "handle is NULL");
  l1dm_status st = check_device(h);
  if (st != L1DM_OK) return st;
  const size_t row = (size_t)h->n * sizeof(uint32_t);
  const size_t pitch = (size_t)h->ldn * sizeof(uint32_t);
  if (sval)
    CUDA_TRY(cudaMemcpy2DAsync(sval, row, h->sval_bits.p, pitch, row, (size_t)h->dl,
                               cudaMemcpyDefault, h->stream));
  if (perm)
    CUDA_TRY(cudaMemcpy2DAsync(perm, row, h->perm.p, pitch, row, (size_t)h->dl, cudaMemcpyDefault,
                               h->stream));
  if (rank) {
    st = ensure_rank(h, h->stream);
    if (st != L1DM_OK) return st;
    CUDA_TRY(cudaMemcpy2DAsync(rank, row, h->rank.p, pitch, row, (size_t)h->dl, cudaMemcpyDefault,
                               h->stream));
  }
  if (hsum)
    CUDA_TRY(cudaMemcpyAsync(hsum, h->hsum.p, (size_t)h->n * sizeof(double), cudaMemcpyDefault,
                             h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return L1DM_OK;
}

l1dm_status l1dm_release_cached(void) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  BlockCache::get().release_all(dev);
  return L1DM_OK;
}

const char *l1dm_last_error(void) { return g_err.c_str(); }

int64_t l1dm_handleless_launches(void) { return g_handleless_launches.load(); }

const char *l1dm_version(void) { return "l1dm 0.1.0 (sm_100a)"; }

}  // extern "C"

// ============================================================================================
// Matrix-free consumers (include/l1dm.h): block Krylov and
// conjugate gradients with every dense step on the device (l1dm_dense.cu) and A touched only
// through the operator's block product.
// ============================================================================================
namespace {

// One stream-ordered scratch allocation carved into aligned pieces; freed (stream-ordered) on
// scope exit.
struct Scratch {
  cudaStream_t s;
  char *base = nullptr;
  size_t used = 0, cap = 0;
  explicit Scratch(cudaStream_t s_) : s(s_) {}
  ~Scratch() {
    if (base) cudaFreeAsync(base, s);
  }
  cudaError_t reserve(size_t bytes) {
    cap = bytes;
    keep_default_pool();
    return cudaMallocAsync(reinterpret_cast<void **>(&base), bytes ? bytes : 256, s);
  }
  template <typename T>
  T *take(size_t count) {
    const size_t off = (used + 255) & ~(size_t)255;
    used = off + count * sizeof(T);
    return reinterpret_cast<T *>(base + off);
  }
  static size_t bytes_for(size_t count, size_t elem) { return ((count * elem + 255) & ~(size_t)255); }
};

l1dm_status op_check(const l1dm_operator_t *op, int64_t *n_out) {
  if (!op) return fail(L1DM_EINVAL, "operator is NULL");
  switch (op->kind) {
    case L1DM_OP_SORTED: {
      if (!op->h) return fail(L1DM_EINVAL, "sorted operator without a handle");
      if (op->p != 1 && op->p != 3 && op->p != 5 && op->p != 7)
        return fail(L1DM_EINVAL, "sorted operator: p=%d not in {1, 3, 5, 7}", op->p);
      l1dm_status st = check_device(op->h);
      if (st != L1DM_OK) return st;
      *n_out = op->h->n;
      return L1DM_OK;
    }
    case L1DM_OP_EVEN:
    case L1DM_OP_BILINEAR:
      if (!op->X || (op->kind == L1DM_OP_BILINEAR && !op->M))
        return fail(L1DM_EINVAL, "operator X (or M) is NULL");
      if (op->n < 1 || op->d < 1 || op->ld_x < op->d)
        return fail(L1DM_EINVAL, "operator n=%lld d=%lld ld_x=%lld invalid", (long long)op->n,
                    (long long)op->d, (long long)op->ld_x);
      if (op->kind == L1DM_OP_EVEN && op->p != 2 && op->p != 4 && op->p != 6)
        return fail(L1DM_EINVAL, "even operator: p=%d not in {2, 4, 6}", op->p);
      if (!is_device_pointer(op->X) || (op->kind == L1DM_OP_BILINEAR && !is_device_pointer(op->M)))
        return fail(L1DM_EINVAL, "operator X and M must be device memory");
      *n_out = op->n;
      return L1DM_OK;
    default:
      return fail(L1DM_EINVAL, "unknown operator kind %d", op->kind);
  }
}

// Y = A Z for an fp32 block (the operator's own product, stream-ordered)
l1dm_status op_apply_f32(const l1dm_operator_t *op, const float *Z, int64_t ldz, int64_t m,
                         double *Y, int64_t ldy, cudaStream_t s) {
  switch (op->kind) {
    case L1DM_OP_SORTED:
      return op->p == 1 ? l1dm_matvec_ex(op->h, Z, ldz, m, Y, ldy, s)
                        : l1dm_matvec_lp_ex(op->h, op->p, Z, ldz, m, Y, ldy, s);
    case L1DM_OP_EVEN:
      return l1dm_lpp_even_matvec(op->X, op->n, op->ld_x, op->d, op->p, Z, ldz, m, Y, ldy, s);
    default:
      return l1dm_bilinear_matvec(op->X, op->n, op->ld_x, op->d, op->M, Z, ldz, m, Y, ldy, s);
  }
}

// Y = A V for fp64 V through the fp32 product: [hi | lo] in one product of 2b columns
l1dm_status op_apply_f64(const l1dm_operator_t *op, int64_t n, const double *V, int64_t ldv,
                         int64_t b, double *Y, int64_t ldy, float *zs, double *yr,
                         cudaStream_t s) {
  launch_split_hilo(n, b, V, ldv, zs, s);
  l1dm_status st = op_apply_f32(op, zs, 2 * b, 2 * b, yr, 2 * b, s);
  if (st != L1DM_OK) return st;
  launch_combine_hilo(n, b, yr, Y, ldy, s);
  return L1DM_OK;
}

int device_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

extern "C" {

l1dm_status l1dm_gemm(int trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                      int64_t lda, const double *B, int64_t ldb, double beta, double *C,
                      int64_t ldc, void *stream) {
  NvtxRange nvtx_("l1dm_gemm");
  g_err.clear();
  if (!C || (K > 0 && (!A || !B))) return fail(L1DM_EINVAL, "A, B or C is NULL");
  if (M < 1 || N < 1 || K < 0 || ldc < N || (K > 0 && (ldb < N || lda < (trans_a ? M : K))))
    return fail(L1DM_EINVAL, "gemm sizes M=%lld N=%lld K=%lld lda=%lld ldb=%lld ldc=%lld invalid",
                (long long)M, (long long)N, (long long)K, (long long)lda, (long long)ldb,
                (long long)ldc);
  int dev = 0;
  l1dm_status st = check_arch(&dev);
  if (st != L1DM_OK) return st;
  if ((K > 0 && (!is_device_pointer(A) || !is_device_pointer(B))) || !is_device_pointer(C))
    return fail(L1DM_EINVAL, "l1dm_gemm takes device pointers");
  cudaStream_t s = (cudaStream_t)stream;
  const int sms = device_sms();
  Scratch sc(s);
  CUDA_TRY(sc.reserve(gemm_workspace(trans_a ? 1 : 0, M, N, K, sms)));
  g_handleless_launches += launch_gemm(trans_a ? 1 : 0, M, N, K, alpha, A, lda, B, ldb, beta, C,
                                       ldc, reinterpret_cast<double *>(sc.base), sms, s);
  CUDA_TRY(cudaGetLastError());
  return L1DM_OK;
}

l1dm_status l1dm_syevj(int64_t N, const double *A, int64_t lda, double *W, double *V, int64_t ldv,
                       void *stream) {
  NvtxRange nvtx_("l1dm_syevj");
  g_err.clear();
  if (!A || !W || !V) return fail(L1DM_EINVAL, "A, W or V is NULL");
  if (N < 1 || lda < N || ldv < N || N > (1 << 15))
    return fail(L1DM_EINVAL, "syevj N=%lld lda=%lld ldv=%lld invalid", (long long)N,
                (long long)lda, (long long)ldv);
  int dev = 0;
  l1dm_status st = check_arch(&dev);
  if (st != L1DM_OK) return st;
  if (!is_device_pointer(A) || !is_device_pointer(W) || !is_device_pointer(V))
    return fail(L1DM_EINVAL, "l1dm_syevj takes device pointers");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc(s);
  const bool big = false;  // both Jacobi variants only read A
  CUDA_TRY(sc.reserve(Scratch::bytes_for(jacobi_workspace(N), 1) +
                      (big ? Scratch::bytes_for((size_t)N * N, sizeof(double)) : 0) + 512));
  double *ws = sc.take<double>(jacobi_workspace(N) / sizeof(double) + 1);
  double *Acp = const_cast<double *>(A);
  int64_t ld = lda;
  if (big) {
    Acp = sc.take<double>((size_t)N * N);
    CUDA_TRY(cudaMemcpy2DAsync(Acp, N * sizeof(double), A, lda * sizeof(double),
                               N * sizeof(double), N, cudaMemcpyDeviceToDevice, s));
    ld = N;
  }
  static const bool dbg = getenv("L1DM_DEBUG_JACOBI") != nullptr;
  int *stats = dbg ? sc.take<int>(4) : nullptr;
  g_handleless_launches += launch_jacobi(N, Acp, ld, W, V, ldv, ws, device_sms(), s, stats);
  CUDA_TRY(cudaGetLastError());
  if (dbg) {
    int hs = -1;
    cudaMemcpyAsync(&hs, stats, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "[l1dm] syevj N=%lld sweeps=%d\n", (long long)N, hs);
  }
  return L1DM_OK;
}

l1dm_status l1dm_syev_topk(int64_t N, const double *A, int64_t lda, int64_t k, double *lam,
                           double *V, int64_t ldv, void *stream) {
  NvtxRange nvtx_("l1dm_syev_topk");
  g_err.clear();
  if (!A || !lam || !V) return fail(L1DM_EINVAL, "A, lam or V is NULL");
  if (N < 1 || N > 4096 || k < 1 || k > 96 || k > N || lda < N || ldv < k)
    return fail(L1DM_EINVAL, "syev_topk N=%lld k=%lld lda=%lld ldv=%lld invalid (N <= 4096, "
                "k <= min(N, 96))", (long long)N, (long long)k, (long long)lda, (long long)ldv);
  int dev = 0;
  l1dm_status st = check_arch(&dev);
  if (st != L1DM_OK) return st;
  if (!is_device_pointer(A) || !is_device_pointer(lam) || !is_device_pointer(V))
    return fail(L1DM_EINVAL, "l1dm_syev_topk takes device pointers");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc(s);
  CUDA_TRY(sc.reserve(Scratch::bytes_for(topk_workspace(N), 1) +
                      Scratch::bytes_for((size_t)N * k, sizeof(double)) + 512));
  double *ws = sc.take<double>(topk_workspace(N) / sizeof(double) + 1);
  double *Vs = sc.take<double>((size_t)N * k);
  g_handleless_launches += launch_sym_topk(N, A, lda, k, lam, nullptr, Vs, ws, device_sms(), s);
  CUDA_TRY(cudaMemcpy2DAsync(V, ldv * sizeof(double), Vs, k * sizeof(double), k * sizeof(double),
                             N, cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(cudaGetLastError());
  return L1DM_OK;
}

l1dm_status l1dm_op_apply(const l1dm_operator_t *op, const double *V, int64_t ldv, int64_t b,
                          double *Y, int64_t ldy, void *stream) {
  NvtxRange nvtx_("l1dm_op_apply");
  g_err.clear();
  int64_t n = 0;
  l1dm_status st = op_check(op, &n);
  if (st != L1DM_OK) return st;
  if (!V || !Y || b < 1 || ldv < b || ldy < b)
    return fail(L1DM_EINVAL, "V/Y NULL or b=%lld ldv=%lld ldy=%lld invalid", (long long)b,
                (long long)ldv, (long long)ldy);
  if (!is_device_pointer(V) || !is_device_pointer(Y))
    return fail(L1DM_EINVAL, "l1dm_op_apply takes device pointers");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc(s);
  CUDA_TRY(sc.reserve(Scratch::bytes_for((size_t)n * 2 * b, sizeof(float)) +
                      Scratch::bytes_for((size_t)n * 2 * b, sizeof(double))));
  float *zs = sc.take<float>((size_t)n * 2 * b);
  double *yr = sc.take<double>((size_t)n * 2 * b);
  g_handleless_launches += 2;
  return op_apply_f64(op, n, V, ldv, b, Y, ldy, zs, yr, s);
}

}  // extern "C"

namespace {
// Y = A V (n x b fp64 blocks, leading dimensions given), stream-ordered on the core's stream
using ApplyF64 = std::function<l1dm_status(const double *V, int64_t ldv, int64_t b, double *Y,
                                           int64_t ldy)>;

l1dm_status krylov_core(int64_t n, const ApplyF64 &apply_f64, int64_t k, int64_t block,
                        int64_t depth, const double *Pi, double *sigma, double *lam, double *Z,
                        int64_t ldz, cudaStream_t s, l1dm_krylov_info_t *info) {
  l1dm_status st = L1DM_OK;  // (arguments checked by the entry points: krylov_args)
  const int64_t b = block, q = depth, Qw = block * depth;
  const int sms = device_sms();
  // scratch: basis, Krylov block, orthogonalisation temporaries, T and its eigenvectors
  const size_t gws = std::max({gemm_workspace(1, Qw, b, n, sms), gemm_workspace(1, b, b, n, sms)});
  size_t bytes = 0;
  auto add = [&](size_t count, size_t el) { bytes += Scratch::bytes_for(count, el); };
  add((size_t)n * Qw, 8);                    // Qb
  add((size_t)n * b, 8);                     // W
  add((size_t)n * b, 8);                     // Vt
  for (int i = 0; i < 4; ++i) add((size_t)b * b, 8);  // G0, G, Gv, S
  add((size_t)b, 8);                         // lamb
  add((size_t)Qw * b, 8);                    // Ct
  add((size_t)Qw * Qw, 8);                   // T
  add((size_t)Qw * k, 8);                    // Vs
  add(gws / 8 + 1, 8);
  add(topk_workspace(Qw) / 8 + 1, 8);
  Scratch sc(s);
  CUDA_TRY(sc.reserve(bytes));
  double *Qb = sc.take<double>((size_t)n * Qw), *W = sc.take<double>((size_t)n * b);
  double *Vt = sc.take<double>((size_t)n * b);
  double *G0 = sc.take<double>(b * b), *G = sc.take<double>(b * b);
  double *Gv = sc.take<double>(b * b), *S = sc.take<double>(b * b);
  double *lamb = sc.take<double>(b), *Ct = sc.take<double>(Qw * b);
  double *T = sc.take<double>(Qw * Qw);
  double *Vs = sc.take<double>(Qw * k);
  double *gw = sc.take<double>(gws / 8 + 1);
  double *tw = sc.take<double>(topk_workspace(Qw) / 8 + 1);
  CUDA_TRY(cudaMemsetAsync(T, 0, (size_t)Qw * Qw * sizeof(double), s));

  std::vector<cudaEvent_t> evs;
  auto ev = [&]() {
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    evs.push_back(e);
  };
  auto release_events = [&]() {
    for (auto e : evs) cudaEventDestroy(e);
    evs.clear();
  };
  int64_t launches = 0, products = 0;
  std::vector<std::pair<size_t, size_t>> prod_ev;
  auto apply = [&](const double *V, int64_t ldv, double *Y) -> l1dm_status {
    const size_t e0 = evs.size();
    ev();
    l1dm_status r = apply_f64(V, ldv, b, Y, b);
    ev();
    prod_ev.push_back({e0, e0 + 1});
    ++products;
    launches += 2;
    return r;
  };
  auto gemm = [&](int ta, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                  int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc) {
    launches += launch_gemm(ta, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, gw, sms, s);
  };
  // Gram-based orthonormalisation (CholeskyQR) resolves column residuals down to ~sqrt(eps) of
  // the block's largest column norm; columns whose residual is below kDropRtol of it are
  // rounding noise (a rank-deficient block: Krylov space exhausted), dropped as zero columns
  constexpr double kDropRtol = 1e-7;
  ev();  // total start
  st = apply(Pi, b, W);  // A Pi: the first Krylov block
  int64_t cols = 0;
  for (int64_t j = 0; j < q && st == L1DM_OK; ++j) {
    gemm(1, b, b, n, 1.0, W, b, W, b, 0.0, G0, b);  // column norms before projection (drop floor)
    if (cols > 0) {
      // block Gram-Schmidt against the basis, twice: first against the last two blocks (the
      // block Lanczos three-term recurrence: in exact arithmetic A Q_{j-1} has no component on
      // older blocks), then against the whole basis (full re-orthogonalisation).  The
      // coefficients add up to column block j-1 of T = Q^T A Q (rows 0..cols): W = A Q_{j-1}.
      for (int pass = 0; pass < 2; ++pass) {
        const int64_t c0 = pass == 0 ? std::max<int64_t>(0, cols - 2 * b) : 0, cw = cols - c0;
        gemm(1, cw, b, n, 1.0, Qb + c0, Qw, W, b, 0.0, Ct, b);
        gemm(0, n, b, cw, -1.0, Qb + c0, Qw, Ct, b, 1.0, W, b);
        launch_axpy2d(cw, b, 1.0, Ct, b, T + c0 * Qw + (j - 1) * b, Qw, s);
        ++launches;
      }
    }
    // orthonormal basis of the block's column space: CholeskyQR with column dropping, twice
    // (CholeskyQR2)
    const double *src = W;
    double *dst = Vt;
    int64_t ldd = b;
    for (int rep = 0; rep < 2; ++rep) {
      gemm(1, b, b, n, 1.0, src, b, src, b, 0.0, G, b);
      launch_chol_orth(b, G, b, rep == 0 ? G0 : nullptr, b, kDropRtol, 0.25, S, s);
      gemm(0, n, b, b, 1.0, src, b, S, b, 0.0, dst, ldd);
      launches += 1;
      src = Vt;
      dst = Qb + cols;
      ldd = Qw;
    }
    if (cols > 0)  // R = Q_j^T W: rows cols..cols+b of T's column block j-1
      gemm(1, b, b, n, 1.0, Qb + cols, Qw, W, b, 0.0, T + cols * Qw + (j - 1) * b, Qw);
    cols += b;
    st = apply(Qb + (cols - b), Qw, W);  // A Q_j: next Krylov block and T's column block j
  }
  if (st != L1DM_OK) {
    cudaStreamSynchronize(s);
    release_events();
    return st;
  }
  gemm(1, Qw, b, n, 1.0, Qb, Qw, W, b, 0.0, T + (q - 1) * b, Qw);  // last column block of T
  launch_symmetrize(Qw, T, Qw, s);
  // the k Ritz pairs of largest |lambda|: Householder tridiagonalisation, bisection, inverse
  // iteration, back-transformation (l1dm_dense.cu)
  launches += 1 + launch_sym_topk(Qw, T, Qw, k, lam, sigma, Vs, tw, sms, s);
  if (Z) gemm(0, n, k, Qw, 1.0, Qb, Qw, Vs, k, 0.0, Z, ldz);
  ev();  // total end
  cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    release_events();
    return fail(L1DM_ECUDA, "block krylov: %s", cudaGetErrorString(e));
  }
  if (info) {
    info->products = products;
    info->columns = products * 2 * b;
    info->block = b;
    info->depth = q;
    float ms = 0.0f;
    double pm = 0.0;
    for (auto &pe : prod_ev) {
      cudaEventElapsedTime(&ms, evs[pe.first], evs[pe.second]);
      pm += ms;
    }
    info->product_ms = pm;
    cudaEventElapsedTime(&ms, evs.front(), evs.back());
    info->total_ms = ms;
  }
  g_handleless_launches += launches;
  release_events();
  return L1DM_OK;
}

l1dm_status cg_core(int64_t n, const ApplyF64 &apply_f64, const double *bvec, double *x,
                    double tol, int64_t maxit, int normal_equations, cudaStream_t s,
                    l1dm_cg_info_t *info) {
  l1dm_status st = L1DM_OK;
  const int nb = cg_dot_blocks();
  Scratch sc(s);
  CUDA_TRY(sc.reserve(4 * Scratch::bytes_for(n, 8) + Scratch::bytes_for(nb, 8) +
                      Scratch::bytes_for(16, 8)));
  double *r = sc.take<double>(n), *p = sc.take<double>(n), *Ap = sc.take<double>(n);
  double *tmp = sc.take<double>(n);
  double *part = sc.take<double>(nb);
  double *stv = sc.take<double>(16);
  double *hflag = nullptr;  // pinned: [chunk parity][conv, it]
  CUDA_TRY(cudaHostAlloc(reinterpret_cast<void **>(&hflag), 4 * sizeof(double), 0));
  cudaEvent_t cev[2] = {nullptr, nullptr};
  cudaEventCreateWithFlags(&cev[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&cev[1], cudaEventDisableTiming);
  auto cleanup = [&]() {
    cudaStreamSynchronize(s);
    cudaFreeHost(hflag);
    cudaEventDestroy(cev[0]);
    cudaEventDestroy(cev[1]);
  };
  int64_t products = 0, launches = 0;
  auto A = [&](const double *v, double *out) -> l1dm_status {
    ++products;
    launches += 2;
    return apply_f64(v, 1, 1, out, 1);
  };
  // rhs into r (normal equations: A b), x = 0, p = r
  if (normal_equations) st = A(bvec, r);
  else if (cudaMemcpyAsync(r, bvec, n * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    st = fail(L1DM_ECUDA, "cg: copy of b failed");
  if (st != L1DM_OK) {
    cleanup();
    return st;
  }
  cudaMemsetAsync(x, 0, n * sizeof(double), s);
  cudaMemcpyAsync(p, r, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  launch_dot(n, r, r, part, s);
  launch_cg_scalars(0, part, tol, stv, s);
  launches += 2;
  constexpr int64_t kChunk = 8;  // iterations between host looks at the flag
  int64_t issued = 0, chunk = 0;
  bool stop = false;
  while (!stop && issued < maxit) {
    const int64_t it_here = std::min(kChunk, maxit - issued);
    for (int64_t i = 0; i < it_here && st == L1DM_OK; ++i) {
      if (normal_equations) {
        st = A(p, tmp);
        if (st == L1DM_OK) st = A(tmp, Ap);
      } else {
        st = A(p, Ap);
      }
      launch_dot(n, p, Ap, part, s);
      launch_cg_scalars(1, part, tol, stv, s);
      launch_cg_xr(n, stv, p, Ap, x, r, s);
      launch_dot(n, r, r, part, s);
      launch_cg_scalars(2, part, tol, stv, s);
      launch_cg_p(n, stv, r, p, s);
      launches += 6;
    }
    if (st != L1DM_OK) break;
    issued += it_here;
    const int slot = (int)(chunk & 1);
    cudaMemcpyAsync(hflag + 2 * slot, stv + CG_CONV_INDEX, 2 * sizeof(double),
                    cudaMemcpyDeviceToHost, s);
    cudaEventRecord(cev[slot], s);
    if (chunk > 0) {  // the previous chunk's flag (this chunk is already queued behind it)
      cudaEventSynchronize(cev[slot ^ 1]);
      if (hflag[2 * (slot ^ 1)] != 0.0) stop = true;
    }
    ++chunk;
  }
  if (st != L1DM_OK) {
    cleanup();
    return st;
  }
  // final state and the true residual ||A x - b|| / ||b||
  double hst[2] = {0.0, 0.0};
  cudaMemcpyAsync(hst, stv + CG_CONV_INDEX, 2 * sizeof(double), cudaMemcpyDeviceToHost, s);
  st = A(x, tmp);
  if (st != L1DM_OK) {
    cleanup();
    return st;
  }
  launch_sub(n, tmp, bvec, tmp, s);
  std::vector<double> hp(2 * nb);
  launch_dot(n, tmp, tmp, part, s);
  cudaMemcpyAsync(hp.data(), part, nb * sizeof(double), cudaMemcpyDeviceToHost, s);
  launch_dot(n, bvec, bvec, part, s);
  cudaMemcpyAsync(hp.data() + nb, part, nb * sizeof(double), cudaMemcpyDeviceToHost, s);
  launches += 3;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  cleanup();
  if (e != cudaSuccess) return fail(L1DM_ECUDA, "cg: %s", cudaGetErrorString(e));
  double rr = 0.0, bb = 0.0;
  for (int i = 0; i < nb; ++i) {
    rr += hp[i];
    bb += hp[nb + i];
  }
  if (info) {
    info->iterations = (int64_t)hst[1];
    info->converged = hst[0] != 0.0;
    info->residual = std::sqrt(rr) / std::max(std::sqrt(bb), 1e-300);
    info->products = products;
  }
  g_handleless_launches += launches;
  return L1DM_OK;
}


// The fp64 product of an l1dm_operator_t: the hi/lo split through the operator's own product,
// with scratch for blocks up to bmax columns
struct OpApply {
  const l1dm_operator_t *op;
  int64_t n;
  cudaStream_t s;
  Scratch sc;
  float *zs = nullptr;
  double *yr = nullptr;
  int64_t bmax = 0;
  OpApply(const l1dm_operator_t *o, int64_t n_, cudaStream_t s_) : op(o), n(n_), s(s_), sc(s_) {}
  cudaError_t reserve(int64_t b) {
    bmax = b;
    cudaError_t e = sc.reserve(Scratch::bytes_for((size_t)n * 2 * b, sizeof(float)) +
                               Scratch::bytes_for((size_t)n * 2 * b, sizeof(double)));
    if (e != cudaSuccess) return e;
    zs = sc.take<float>((size_t)n * 2 * b);
    yr = sc.take<double>((size_t)n * 2 * b);
    return cudaSuccess;
  }
  ApplyF64 fn() {
    return [this](const double *V, int64_t ldv, int64_t b, double *Y, int64_t ldy) {
      return op_apply_f64(op, n, V, ldv, b, Y, ldy, zs, yr, s);
    };
  }
};

// a caller-supplied product (l1dm_apply_fn): e.g. a coordinate-sharded partial plus the
// cross-GPU all-reduce
ApplyF64 callback_apply(l1dm_apply_fn fn, void *user, cudaStream_t s) {
  return [fn, user, s](const double *V, int64_t ldv, int64_t b, double *Y, int64_t ldy) {
    const int rc = fn(user, V, ldv, b, Y, ldy, (void *)s);
    return rc == 0 ? L1DM_OK : fail(rc < 0 && rc >= L1DM_ENOTSIMPLEX ? (l1dm_status)rc : L1DM_ECUDA,
                                    "the caller's product callback returned %d", rc);
  };
}

l1dm_status krylov_args(int64_t n, int64_t k, int64_t b, int64_t q, const double *Pi,
                        const double *sigma, const double *lam, const double *Z, int64_t ldz) {
  if (!Pi || !sigma) return fail(L1DM_EINVAL, "Pi or sigma is NULL");
  const int64_t Qw = b * q;
  if (n < 1 || k < 1 || b < k || b > 96 || q < 1 || Qw > n || Qw > 4096 || (Z && ldz < k))
    return fail(L1DM_EINVAL, "krylov k=%lld block=%lld depth=%lld (n=%lld) invalid: need 1 <= k "
                "<= block <= 96, depth >= 1, block*depth <= min(n, 4096)", (long long)k, (long long)b,
                (long long)q, (long long)n);
  for (const void *ptr : {(const void *)Pi, (const void *)sigma, (const void *)lam,
                          (const void *)Z})
    if (ptr && !is_device_pointer(ptr)) return fail(L1DM_EINVAL, "krylov buffers must be device memory");
  return L1DM_OK;
}

}  // namespace

extern "C" {

l1dm_status l1dm_block_krylov(const l1dm_operator_t *op, int64_t k, int64_t block, int64_t depth,
                              const double *Pi, double *sigma, double *lam, double *Z,
                              int64_t ldz, void *stream, l1dm_krylov_info_t *info) {
  NvtxRange nvtx_("l1dm_block_krylov");
  g_err.clear();
  int64_t n = 0;
  l1dm_status st = op_check(op, &n);
  if (st != L1DM_OK) return st;
  st = krylov_args(n, k, block, depth, Pi, sigma, lam, Z, ldz);
  if (st != L1DM_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  OpApply oa(op, n, s);
  CUDA_TRY(oa.reserve(block));
  return krylov_core(n, oa.fn(), k, block, depth, Pi, sigma, lam, Z, ldz, s, info);
}

l1dm_status l1dm_block_krylov_cb(int64_t n, l1dm_apply_fn apply, void *user, int64_t k,
                                 int64_t block, int64_t depth, const double *Pi, double *sigma,
                                 double *lam, double *Z, int64_t ldz, void *stream,
                                 l1dm_krylov_info_t *info) {
  NvtxRange nvtx_("l1dm_block_krylov_cb");
  g_err.clear();
  if (!apply) return fail(L1DM_EINVAL, "apply callback is NULL");
  int dev = 0;
  l1dm_status st = check_arch(&dev);
  if (st != L1DM_OK) return st;
  st = krylov_args(n, k, block, depth, Pi, sigma, lam, Z, ldz);
  if (st != L1DM_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  return krylov_core(n, callback_apply(apply, user, s), k, block, depth, Pi, sigma, lam, Z, ldz,
                     s, info);
}

l1dm_status l1dm_cg(const l1dm_operator_t *op, const double *bvec, double *x, double tol,
                    int64_t maxit, int normal_equations, void *stream, l1dm_cg_info_t *info) {
  NvtxRange nvtx_("l1dm_cg");
  g_err.clear();
  int64_t n = 0;
  l1dm_status st = op_check(op, &n);
  if (st != L1DM_OK) return st;
  if (!bvec || !x || maxit < 0 || !(tol >= 0.0))
    return fail(L1DM_EINVAL, "b/x NULL, maxit < 0 or tol invalid");
  if (!is_device_pointer(bvec) || !is_device_pointer(x))
    return fail(L1DM_EINVAL, "l1dm_cg takes device b and x");
  cudaStream_t s = (cudaStream_t)stream;
  OpApply oa(op, n, s);
  CUDA_TRY(oa.reserve(1));
  return cg_core(n, oa.fn(), bvec, x, tol, maxit, normal_equations, s, info);
}

l1dm_status l1dm_cg_cb(int64_t n, l1dm_apply_fn apply, void *user, const double *bvec, double *x,
                       double tol, int64_t maxit, int normal_equations, void *stream,
                       l1dm_cg_info_t *info) {
  NvtxRange nvtx_("l1dm_cg_cb");
  g_err.clear();
  if (!apply || !bvec || !x || n < 1 || maxit < 0 || !(tol >= 0.0))
    return fail(L1DM_EINVAL, "apply/b/x NULL, n < 1, maxit < 0 or tol invalid");
  int dev = 0;
  l1dm_status st = check_arch(&dev);
  if (st != L1DM_OK) return st;
  if (!is_device_pointer(bvec) || !is_device_pointer(x))
    return fail(L1DM_EINVAL, "l1dm_cg_cb takes device b and x");
  cudaStream_t s = (cudaStream_t)stream;
  return cg_core(n, callback_apply(apply, user, s), bvec, x, tol, maxit, normal_equations, s,
                 info);
}

}  // extern "C"
