// l2_probe.cu — measures the L2-side ceilings that bound the scatter-mode query
// on the local B200 and prints one JSON object (committed as profiles/l2_peaks.json):
//   red_row8_adds_per_s   fp64 reductions, 8 consecutive doubles (one 64-B row) per request,
//                         random rows of an L2-resident 64 MiB buffer (the apply pass's REDs)
//   gather_sector_GBps    random 32-B sector reads of an L2-resident 32 MiB buffer (Zt gathers)
//   stream_read_GBps      sequential reads of an L2-resident 32 MiB buffer
// Row indices come from a streamed index array (4 B per row, like perm).  CUDA-event timed,
// best of 5 after a warm-up launch.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void fill_idx(uint32_t *idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    idx[i] = (uint32_t)x;
  }
}
// W lanes per W*8-byte row (32/W rows per warp step), U steps in flight per thread
template <int W, int U>
__global__ void __launch_bounds__(256) red_rows(const uint32_t *idx, int64_t rows, double *y,
                                                uint32_t yrows) {
  constexpr int G = 32 / W;
  const int lane = threadIdx.x & 31, c = lane % W, g = lane / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * G * U; base < rows; base += nw * G * U) {
    uint32_t p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) p[u] = __ldcs(idx + base + u * G + g);
#pragma unroll
    for (int u = 0; u < U; ++u) atomicAdd(y + (int64_t)(p[u] % yrows) * W + c, 1.0);
  }
}
// one 32-B sector per row: 8 lanes x 4 B
__global__ void __launch_bounds__(256) gather_sectors(const uint32_t *idx, int64_t rows,
                                                      const float *z, uint32_t zrows,
                                                      float *out) {
  const int lane = threadIdx.x & 31, c = lane & 7, g = lane >> 3;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int64_t base = warp * 16; base < rows; base += nw * 16) {
    uint32_t p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) p[u] = __ldcs(idx + base + u * 4 + g);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += __ldcg(z + (int64_t)(p[u] % zrows) * 8 + c);
  }
  if (acc == 1.2345f) out[0] = acc;
}
// W lanes per W*8-byte row, row indices hashed in registers (no index stream: the reduction
// rate alone), U reductions in flight per thread
template <int W, int U>
__global__ void __launch_bounds__(256) red_rows_hash(int64_t rows, double *y, uint32_t yrows) {
  constexpr int G = 32 / W;
  const int lane = threadIdx.x & 31, c = lane % W, g = lane / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * G * U; base < rows; base += nw * G * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t x = (uint32_t)(base + u * G + g) * 0x9E3779B1u;
      x ^= x >> 15;
      x *= 0x85EBCA77u;
      x ^= x >> 13;
      atomicAdd(y + (int64_t)(x % yrows) * W + c, 1.0);
    }
  }
}
// the runs histogram's pattern: a warp's reductions land in one coordinate's 256-row table
// (rows of W*8 bytes; 96 tables), the run within the table random, the coordinate varying with
// the loop (as k in k20_runs_hist)
template <int W, int U>
__global__ void __launch_bounds__(256) red_tables(int64_t rows, double *y, uint32_t ntab) {
  constexpr int G = 32 / W;
  const int lane = threadIdx.x & 31, c = lane % W, g = lane / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * G * U; base < rows; base += nw * G * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t x = (uint32_t)(base + u * G + g) * 0x9E3779B1u;
      x ^= x >> 15;
      x *= 0x85EBCA77u;
      x ^= x >> 13;
      const uint32_t tab = (uint32_t)((warp + u) % ntab);
      atomicAdd(y + ((int64_t)tab * 256 + (x & 255u)) * W + c, 1.0);
    }
  }
}
// one random 4-byte element per lane (32 rows per warp request): the m = 1 reduce pass's pattern
__global__ void __launch_bounds__(256) gather_lanes(const uint32_t *idx, int64_t rows,
                                                    const float *z, uint32_t zwords, float *out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  float acc = 0.f;
  for (int64_t r = tid; r < rows; r += nt * 4) {
    uint32_t p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) p[u] = (r + u * nt < rows) ? __ldcs(idx + r + u * nt) : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += __ldcg(z + (p[u] % zwords));
  }
  if (acc == 1.2345f) out[0] = acc;
}
// one random fp64 reduction per lane (the m = 1 apply pass's pattern)
__global__ void __launch_bounds__(256) red_lanes(const uint32_t *idx, int64_t rows, double *y,
                                                 uint32_t ywords) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = tid; r < rows; r += nt * 4) {
    uint32_t p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) p[u] = (r + u * nt < rows) ? __ldcs(idx + r + u * nt) : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (r + u * nt < rows) atomicAdd(y + (p[u] % ywords), 1.0);
  }
}
__global__ void __launch_bounds__(256) stream_read(const float4 *z, int64_t n4, int reps,
                                                   float *out) {
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
      const float4 v = __ldcg(z + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 1.2345f) out[0] = acc;
}
// the ceiling sweep: W lanes per W*8-byte row, U reductions in flight per thread, hashed rows of
// a ytab-row buffer; `local` > 0 confines each warp's reductions to one of `local` sub-tables of
// 256 rows (the locality of the runs histogram's per-coordinate tables)
template <int W, int U>
__global__ void __launch_bounds__(256) red_sweep(int64_t rows, double *y, uint32_t ytab,
                                                 uint32_t local) {
  constexpr int G = 32 / W;
  const int lane = threadIdx.x & 31, c = lane % W, g = lane / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * G * U; base < rows; base += nw * G * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t x = (uint32_t)(base + u * G + g) * 0x9E3779B1u;
      x ^= x >> 15;
      x *= 0x85EBCA77u;
      x ^= x >> 13;
      const uint32_t row = local ? (uint32_t)((warp + u) % local) * 256u + (x & 255u) : x % ytab;
      atomicAdd(y + (int64_t)row * W + c, 1.0);
    }
  }
}
// the runs histogram's own reduction stream (k20_runs_hist at c5: m = 16 columns, 16 lanes per
// 128-B row, 2 points per warp step, the point's 96 coordinates in turn, each into its 256-row
// table at a pseudo-random run id): run ids hashed, z = 1 (no loads), tables dl x 256 x m
__global__ void __launch_bounds__(256) red_runs_exact(int64_t npts, int dl, double *H,
                                                      int copies = 1) {
  constexpr int L = 16, m = 16, ppw = 2;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int pg = lane / L, cl = lane % L;
  const int64_t pts_per_cta = 8 * ppw * 16;
  const int64_t i_base = (int64_t)blockIdx.x * pts_per_cta + (int64_t)w * ppw * 16;
  // replicated tables (runs_copies in the library): a warp on replica (8 blockIdx.x + w) % copies
  H += (int64_t)((blockIdx.x * 8 + w) % (unsigned)copies) * ((int64_t)dl * 256 * m);
  for (int step = 0; step < 16; ++step) {
    const int64_t i = i_base + (int64_t)step * ppw + pg;
    if (i >= npts) break;
    for (int k = 0; k < dl; ++k) {
      uint32_t x = (uint32_t)(i * 97 + k) * 0x9E3779B1u;
      x ^= x >> 15;
      x *= 0x85EBCA77u;
      x ^= x >> 13;
      atomicAdd(H + (((int64_t)k * 256 + (x & 255u)) * m + cl), 1.0);
    }
  }
}
template <typename F>
static float best_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int i = 0; i < 5; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}
int main() {
  int dev = 0, sms = 0, l2 = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int64_t rows = 1ll << 27;
  uint32_t *idx;
  double *y;
  float *z, *out;
  if (cudaMalloc(&idx, rows * 4) || cudaMalloc(&y, 64ll << 20) || cudaMalloc(&z, 32ll << 20) ||
      cudaMalloc(&out, 64)) {
    printf("{\"error\": \"alloc\"}\n");
    return 1;
  }
  cudaMemset(y, 0, 64ll << 20);
  cudaMemset(z, 0, 32ll << 20);
  fill_idx<<<sms * 8, 256>>>(idx, rows);
  const int grid = sms * 8;
  const uint32_t yrows = (uint32_t)((64ll << 20) / 64), zrows = (uint32_t)((32ll << 20) / 32);
  const float t_red = best_ms([&] { red_rows<8, 4><<<grid, 256>>>(idx, rows, y, yrows); });
  // deeper: 16 reductions in flight per thread (the apply / histogram kernels keep many)
  const float t_red16 = best_ms([&] { red_rows<8, 16><<<grid, 256>>>(idx, rows, y, yrows); });
  const float t_red_w16 =
      best_ms([&] { red_rows<16, 16><<<grid, 256>>>(idx, rows, y, yrows / 2); });
  const float t_hash8 = best_ms([&] { red_rows_hash<8, 16><<<grid, 256>>>(rows, y, yrows); });
  const float t_hash16_small =
      best_ms([&] { red_rows_hash<16, 16><<<grid, 256>>>(rows, y, (4u << 20) / 128); });
  const float t_tables = best_ms([&] { red_tables<16, 16><<<grid, 256>>>(rows, y, 96); });
  // a 4 MiB table (the runs histogram's: dl x 256 x m fp64, 3 MiB at c5)
  const float t_red_w16_small =
      best_ms([&] { red_rows<16, 16><<<grid, 256>>>(idx, rows, y, (4u << 20) / 128); });
  const float t_gat = best_ms([&] { gather_sectors<<<grid, 256>>>(idx, rows, z, zrows, out); });
  const float t_gl = best_ms([&] { gather_lanes<<<grid, 256>>>(idx, rows, z, zrows * 8, out); });
  const float t_rl = best_ms([&] { red_lanes<<<grid, 256>>>(idx, rows, y, yrows * 8); });
  // c2's exact buffer sizes (m = 1 scatter: z is 4 MiB, Y is 8 MiB)
  const float t_gl4 = best_ms([&] { gather_lanes<<<grid, 256>>>(idx, rows, z, 1u << 20, out); });
  const float t_rl8 = best_ms([&] { red_lanes<<<grid, 256>>>(idx, rows, y, 1u << 20); });
  const int reps = 64;
  const float t_str = best_ms([&] {
    stream_read<<<grid, 256>>>(reinterpret_cast<const float4 *>(z), (32ll << 20) / 16, reps, out);
  });
  // ceiling sweep over row width (32-256 B), buffer size (1-64 MiB), locality and grid size:
  // the largest fp64 reduction rate any pattern reaches is the L2 reduction ceiling
  double best_rate = 0.0;
  char best_cfg[160] = "";
  printf("{\"sweep\": [");
  bool first = true;
  auto rec = [&](const char *name, int w, double mib, int loc, int gmul, float ms) {
    const double rate = rows * (double)w / (ms * 1e-3);
    printf("%s{\"kernel\": \"%s\", \"row_bytes\": %d, \"MiB\": %.3g, \"local_tables\": %d, "
           "\"ctas_per_sm\": %d, \"adds_per_s\": %.4g}",
           first ? "" : ", ", name, w * 8, mib, loc, gmul, rate);
    first = false;
    if (rate > best_rate) {
      best_rate = rate;
      snprintf(best_cfg, sizeof(best_cfg), "%s, %d-B rows, %.3g MiB, local %d, %d CTAs/SM", name,
               w * 8, mib, loc, gmul);
    }
  };
  for (int gmul : {4, 8, 16}) {
    const int gg = sms * gmul;
    for (double mib : {1.0, 3.0, 8.0, 32.0, 64.0}) {
      const uint32_t b = (uint32_t)(mib * (1 << 20));
      rec("hashed", 4, mib, 0, gmul, best_ms([&] { red_sweep<4, 16><<<gg, 256>>>(rows, y, b / 32, 0); }));
      rec("hashed", 8, mib, 0, gmul, best_ms([&] { red_sweep<8, 16><<<gg, 256>>>(rows, y, b / 64, 0); }));
      rec("hashed", 16, mib, 0, gmul, best_ms([&] { red_sweep<16, 16><<<gg, 256>>>(rows, y, b / 128, 0); }));
      rec("hashed", 32, mib, 0, gmul, best_ms([&] { red_sweep<32, 8><<<gg, 256>>>(rows, y, b / 256, 0); }));
    }
    for (int loc : {16, 96, 256}) {
      rec("local_tables", 8, loc * 256 * 64 / 1048576.0, loc, gmul,
          best_ms([&] { red_sweep<8, 16><<<gg, 256>>>(rows, y, 0, (uint32_t)loc); }));
      rec("local_tables", 16, loc * 256 * 128 / 1048576.0, loc, gmul,
          best_ms([&] { red_sweep<16, 16><<<gg, 256>>>(rows, y, 0, (uint32_t)loc); }));
    }
  }
  {  // the runs histogram's exact stream (c5: n = 2^23 points x 96 coordinates x 16 columns)
    const int64_t npts = 1ll << 23;
    const float ms = best_ms([&] { red_runs_exact<<<(unsigned)(npts / 256), 256>>>(npts, 96, y); });
    const double rate = (double)npts * 96 * 16 / (ms * 1e-3);
    printf("%s{\"kernel\": \"runs_histogram_exact\", \"row_bytes\": 128, \"MiB\": 3, "
           "\"adds_per_s\": %.4g}", first ? "" : ", ", rate);
    if (rate > best_rate) {
      best_rate = rate;
      snprintf(best_cfg, sizeof(best_cfg), "runs_histogram_exact (k20's stream, 3 MiB tables)");
    }
    // the same stream on replicated tables, as the library runs it (runs_copies): 96 coordinates
    // x 4 and 8 replicas, and a G = 8 shard's 12 coordinates x 1 and 8 replicas
    for (int cfg = 0; cfg < 4; ++cfg) {
      const int dlc = cfg < 2 ? 96 : 12, cp = cfg == 0 ? 4 : (cfg == 2 ? 1 : 8);
      const float msr = best_ms(
          [&] { red_runs_exact<<<(unsigned)(npts / 256), 256>>>(npts, dlc, y, cp); });
      const double r = (double)npts * dlc * 16 / (msr * 1e-3);
      printf(", {\"kernel\": \"runs_histogram_replicas\", \"row_bytes\": 128, \"coords\": %d, "
             "\"replicas\": %d, \"MiB\": %.3g, \"adds_per_s\": %.4g}", dlc, cp,
             dlc * 256 * 128.0 * cp / 1048576.0, r);
      if (r > best_rate) {
        best_rate = r;
        snprintf(best_cfg, sizeof(best_cfg),
                 "runs_histogram_replicas (k20's stream, %d coordinates x %d replicas)", dlc, cp);
      }
    }
  }
  printf("], \"red_ceiling_adds_per_s\": %.4g, \"red_ceiling_config\": \"%s\", ", best_rate,
         best_cfg);
  const cudaError_t e = cudaGetLastError();
  printf("\"gather_lane_per_s\": %.4g, \"red_lane_per_s\": %.4g, ", rows / (t_gl * 1e-3),
         rows / (t_rl * 1e-3));
  printf("\"gather_lane_4MiB_per_s\": %.4g, \"red_lane_8MiB_per_s\": %.4g, ",
         rows / (t_gl4 * 1e-3), rows / (t_rl8 * 1e-3));
  printf("\"red_row8_deep_adds_per_s\": %.4g, \"red_row16_deep_adds_per_s\": %.4g, "
         "\"red_row16_4MiB_adds_per_s\": %.4g, \"red_row8_hashed_adds_per_s\": %.4g, "
         "\"red_row16_4MiB_hashed_adds_per_s\": %.4g, \"red_runs_tables_adds_per_s\": %.4g, ",
         rows * 8.0 / (t_red16 * 1e-3), rows * 16.0 / (t_red_w16 * 1e-3),
         rows * 16.0 / (t_red_w16_small * 1e-3), rows * 8.0 / (t_hash8 * 1e-3),
         rows * 16.0 / (t_hash16_small * 1e-3), rows * 16.0 / (t_tables * 1e-3));
  printf("\"red_row8_adds_per_s\": %.4g, \"gather_sector_GBps\": %.1f, "
         "\"stream_read_GBps\": %.1f, \"sms\": %d, \"l2_bytes\": %d, \"sm_clock_khz\": %d, "
         "\"status\": \"%s\", \"how\": \"tools/l2_probe.cu: 2^27 random rows, L2-resident "
         "buffers (RED 64 MiB, gather 32 MiB), best of 5 CUDA-event timings\"}\n",
         rows * 8.0 / (t_red * 1e-3), rows * 32.0 / (t_gat * 1e-3) / 1e9,
         (32ll << 20) * (double)reps / (t_str * 1e-3) / 1e9, sms, l2, clk, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
