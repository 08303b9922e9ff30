// gather_bench.cu -- random 512-byte row gather microbenchmark on B200 (sm_100a).
//
// The SaCD MTTKRP is a stream of random gathers of fp64 factor rows of
// R_pad = 64 doubles (512 B), each scaled by the nonzero's value and accumulated into a
// per-warp register row.  This program measures that access pattern alone, so the MTTKRP's
// composite roofline has a MEASURED gather peak, and it tests the
// alternative transports the round-1 review proposed:
//   ldg   : one warp per stream chunk; the row index reaches the lanes by shuffle, x by a
//           shared-memory broadcast; every lane loads its 16-byte chunk of the row with
//           LDG.128 (the production kernel's transport), one row ahead;
//   bulk  : the lane that holds a row's index issues one cp.async.bulk (TMA bulk copy,
//           UBLKCP) of the whole 512-byte row into a per-warp shared-memory ring slot with
//           an mbarrier; the warp waits on the slot and reads it with LDS.128 (no index
//           shuffle, no L1 allocation: every row comes from L2);
//   ldg256: ldg with 256-bit loads, two 16-lane workers per warp (two rows per shuffle);
//   hot   : ldg, but rows with index < HOT are read from a copy staged in shared memory at
//           kernel start (one generic load; the Zipf head of the b-factor).
// Index streams: uniform over the table, or Zipf(s) with rank = index (heavy rows first,
// as in the c3 / c4 generators).  Tables: L1-resident (100 KB), L2-resident (5 MB, c4's W),
// HBM-sized (256 MB / 512 MB, c4's V / U).
//
// Output: one JSON line per case on stdout.  Build: nvcc -O3 -std=c++17
//   -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/gather_bench tools/gather_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

constexpr int RW = 64;  // doubles per row (512 B)

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double *p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// ------------------------------------------------------------------ ldg (+ optional hot rows)
// HOT > 0: rows [0, HOT) staged in dynamic shared memory by the block at start.
template <int HOT>
__global__ void __launch_bounds__(1024) g_ldg(const double *__restrict__ tab, const uint32_t *__restrict__ idx,
                                              const double *__restrict__ xs, long long n, long long per,
                                              double *__restrict__ out) {
  extern __shared__ __align__(16) double hot[];
  __shared__ double xsb[2][1024];
  const int lane = threadIdx.x & 31;
  if (HOT > 0) {
    for (int x = threadIdx.x; x < HOT * RW / 2; x += blockDim.x)
      reinterpret_cast<double2 *>(hot)[x] = reinterpret_cast<const double2 *>(tab)[x];
    __syncthreads();
  }
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long e0 = w * per, e1 = min(n, e0 + per);
  double f0 = 0.0, f1 = 0.0;
  int par = 0;
  const int wbase = threadIdx.x & ~31;
  auto rowp = [&](uint32_t r) -> const double2 * {
    if (HOT > 0 && r < (uint32_t)HOT) return reinterpret_cast<const double2 *>(hot + (size_t)r * RW) + lane;
    return reinterpret_cast<const double2 *>(tab + (size_t)r * RW) + lane;
  };
  for (long long base = e0; base < e1; base += 32) {
    uint32_t my = 0;
    double xl = 0.0;
    if (base + lane < e1) {
      my = ld_stream_u32(idx + base + lane);
      xl = ld_stream_f64(xs + base + lane);
    }
    par ^= 1;
    xsb[par][threadIdx.x] = xl;
    __syncwarp();
    double2 b[2];
    b[0] = *rowp(__shfl_sync(0xffffffffu, my, 0));
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j + 1 < 32) b[(j + 1) & 1] = *rowp(__shfl_sync(0xffffffffu, my, j + 1));
      const double x = xsb[par][wbase + j];
      f0 = fma(x, b[j & 1].x, f0);
      f1 = fma(x, b[j & 1].y, f1);
    }
  }
  out[w * RW + 2 * lane] = f0;
  out[w * RW + 2 * lane + 1] = f1;
}

// ------------------------------------------------------------------ ldg256
// Two 16-lane workers per warp: every lane loads its 32-byte quarter-chunk of a 512-byte row
// with one 256-bit load (LDG.E.ENL2.256, sm_100), so one shuffle delivers the indices of two
// rows (each half-warp reads its own source lane) and one load instruction moves 1 KB.
__device__ __forceinline__ void ldg256(const double *p, double &a, double &b, double &c, double &d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__global__ void __launch_bounds__(1024) g_ldg256(const double *__restrict__ tab, const uint32_t *__restrict__ idx,
                                                 const double *__restrict__ xs, long long n, long long per,
                                                 double *__restrict__ out) {
  __shared__ double xsb[2][1024];
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long e0 = w * per, e1 = min(n, e0 + per);
  double f[4] = {0.0, 0.0, 0.0, 0.0};
  int par = 0;
  const int wbase = threadIdx.x & ~31;
  for (long long base = e0; base < e1; base += 32) {
    uint32_t my = 0;
    double xl = 0.0;
    if (base + lane < e1) {
      my = ld_stream_u32(idx + base + lane);
      xl = ld_stream_f64(xs + base + lane);
    }
    par ^= 1;
    xsb[par][threadIdx.x] = xl;
    __syncwarp();
    double b[2][4];
    {
      const uint32_t r = __shfl_sync(0xffffffffu, my, half);
      ldg256(tab + (size_t)r * RW + 4 * hl, b[0][0], b[0][1], b[0][2], b[0][3]);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j + 1 < 16) {
        const uint32_t r = __shfl_sync(0xffffffffu, my, 2 * (j + 1) + half);
        ldg256(tab + (size_t)r * RW + 4 * hl, b[(j + 1) & 1][0], b[(j + 1) & 1][1], b[(j + 1) & 1][2],
               b[(j + 1) & 1][3]);
      }
      const double x = xsb[par][wbase + 2 * j + half];
#pragma unroll
      for (int e = 0; e < 4; ++e) f[e] = fma(x, b[j & 1][e], f[e]);
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) f[e] += __shfl_xor_sync(0xffffffffu, f[e], 16);
  if (half == 0)
#pragma unroll
    for (int e = 0; e < 4; ++e) out[w * RW + 4 * hl + e] = f[e];
}

// ------------------------------------------------------------------ bulk copies
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void bulk_row(void *dst, const void *src, uint64_t *bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst), b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(RW * 8) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
               "l"(src), "r"(RW * 8), "r"(b)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(b),
      "r"(phase)
      : "memory");
}

// S slots per warp; row t of the warp's stream goes to slot t % S and is issued S - 1 rows
// ahead by the lane holding its index (the current batch, or the next batch's indices).
template <int S>
__global__ void __launch_bounds__(256) g_bulk(const double *__restrict__ tab, const uint32_t *__restrict__ idx,
                                              const double *__restrict__ xs, long long n, long long per,
                                              double *__restrict__ out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  double *ring = reinterpret_cast<double *>(sm) + (size_t)wp * S * RW;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + (size_t)(blockDim.x >> 5) * S * RW * 8) + wp * S;
  __shared__ double xsb[2][256];
  if (lane < S) mbar_init(bars + lane, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long e0 = w * per, e1 = min(n, e0 + per);
  double f0 = 0.0, f1 = 0.0;
  unsigned phases = 0;  // bit s = parity to wait for on slot s
  int par = 0;
  const int wbase = threadIdx.x & ~31;
  uint32_t my = 0, nx = 0;
  if (e0 + lane < e1) my = ld_stream_u32(idx + e0 + lane);
  // prologue: rows 0 .. S-2 of the stream
  for (int j = 0; j < S - 1; ++j)
    if (lane == j && e0 + j < e1) bulk_row(ring + (j % S) * RW, tab + (size_t)my * RW, bars + (j % S));
  long long t = 0;  // stream position of the row being consumed
  for (long long base = e0; base < e1; base += 32) {
    nx = 0;
    if (base + 32 + lane < e1) nx = ld_stream_u32(idx + base + 32 + lane);
    double xl = (base + lane < e1) ? ld_stream_f64(xs + base + lane) : 0.0;
    par ^= 1;
    xsb[par][threadIdx.x] = xl;
    __syncwarp();
    const int cnt = (int)min(32LL, e1 - base);
    for (int j = 0; j < cnt; ++j, ++t) {
      // issue row t + S - 1 (its slot was consumed at t - 1; the warp is past those reads)
      const long long ti = t + S - 1;
      const int jj = j + S - 1;
      if (base + jj < e1) {
        const int sl = (int)(ti % S);
        const uint32_t r = jj < 32 ? my : nx;
        if (lane == (jj & 31)) bulk_row(ring + sl * RW, tab + (size_t)r * RW, bars + sl);
      }
      const int s = (int)(t % S);
      mbar_wait(bars + s, (phases >> s) & 1u);
      phases ^= 1u << s;
      const double2 b = reinterpret_cast<const double2 *>(ring + s * RW)[lane];
      const double x = xsb[par][wbase + j];
      f0 = fma(x, b.x, f0);
      f1 = fma(x, b.y, f1);
      __syncwarp();
    }
    my = nx;
  }
  out[w * RW + 2 * lane] = f0;
  out[w * RW + 2 * lane + 1] = f1;
}

// ------------------------------------------------------------------ host
static std::vector<uint32_t> make_idx(long long n, long long T, double s, uint64_t seed) {
  std::vector<uint32_t> v((size_t)n);
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  if (s <= 0) {
    for (auto &x : v) x = (uint32_t)std::min<long long>(T - 1, (long long)(U(g) * T));
    return v;
  }
  std::vector<double> cdf((size_t)T);
  double acc = 0.0;
  for (long long k = 0; k < T; ++k) cdf[(size_t)k] = (acc += std::pow((double)(k + 1), -s));
  for (auto &c : cdf) c /= acc;
  for (auto &x : v) x = (uint32_t)std::min<long long>(T - 1, std::lower_bound(cdf.begin(), cdf.end(), U(g)) - cdf.begin());
  return v;
}

int main(int argc, char **argv) {
  // gather_bench [n] [table filter] [dist filter] [kernel filter]: filters are substrings
  // (e.g. "L2_5MB" "zipf" "ldg_w32" for one case under ncu)
  const long long n = argc > 1 ? atoll(argv[1]) : (1LL << 26);
  const std::string ftab = argc > 2 ? argv[2] : "", fdist = argc > 3 ? argv[3] : "", fker = argc > 4 ? argv[4] : "";
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  CK(cudaFuncSetAttribute(g_ldg<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 0));
  CK(cudaFuncSetAttribute(g_ldg<192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * RW * 8));
  CK(cudaFuncSetAttribute(g_ldg<384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 384 * RW * 8));
  CK(cudaFuncSetAttribute(g_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * (RW * 8 + 8)));
  CK(cudaFuncSetAttribute(g_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8 * (RW * 8 + 8)));
  CK(cudaFuncSetAttribute(g_bulk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16 * (RW * 8 + 8)));
  const long long Tmax = 1000000;
  double *tab = nullptr, *xs = nullptr, *out = nullptr;
  uint32_t *idx = nullptr;
  CK(cudaMalloc(&tab, (size_t)Tmax * RW * 8));
  CK(cudaMalloc(&xs, (size_t)n * 8));
  CK(cudaMalloc(&idx, (size_t)n * 4));
  CK(cudaMalloc(&out, (size_t)sms * 64 * 32 * RW * 8));
  {
    std::vector<double> h((size_t)Tmax * RW);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761u) % 1000) * 1e-3;
    CK(cudaMemcpy(tab, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    std::vector<double> hx((size_t)n, 1.0);
    CK(cudaMemcpy(xs, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice));
  }
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  struct Tab { const char *name; long long T; };
  const Tab tabs[] = {{"L1_100KB", 200}, {"L2_5MB", 10000}, {"HBM_256MB", 500000}, {"HBM_512MB", 1000000}};
  const double dists[] = {0.0, 1.2};
  for (const Tab &tb : tabs) {
    if (!ftab.empty() && std::string(tb.name).find(ftab) == std::string::npos) continue;
    for (double s : dists) {
      if (!fdist.empty() && std::string(s > 0 ? "zipf1.2" : "uniform").find(fdist) == std::string::npos) continue;
      std::vector<uint32_t> hi = make_idx(n, tb.T, s, 12345);
      CK(cudaMemcpy(idx, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));
      auto run = [&](const char *kname, auto launch) {
        if (!fker.empty() && std::string(kname) != fker) return;
        launch();
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        const int reps = 5;
        CK(cudaEventRecord(a));
        for (int r = 0; r < reps; ++r) launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, a, b));
        ms /= reps;
        const double gbs = (double)n * RW * 8 / (ms * 1e-3) / 1e9;
        printf("{\"table\": \"%s\", \"rows\": %lld, \"dist\": \"%s\", \"kernel\": \"%s\", \"gathers\": %lld, "
               "\"ms\": %.4f, \"row_GBps\": %.1f, \"Grows_per_s\": %.3f}\n",
               tb.name, tb.T, s > 0 ? "zipf1.2" : "uniform", kname, n, ms, gbs, n / (ms * 1e-3) / 1e9);
        fflush(stdout);
      };
      for (int wps : {8, 16, 32, 48, 64}) {  // resident warps per SM, static partition
        const int bs = 256;
        const int bps = wps * 32 / bs;
        const long long nw = (long long)sms * bps * (bs / 32);
        const long long per = ((n + nw - 1) / nw + 31) / 32 * 32;
        char nm[64];
        snprintf(nm, sizeof nm, "ldg_w%d", wps);
        run(nm, [&] { g_ldg<0><<<sms * bps, bs>>>(tab, idx, xs, n, per, out); });
      }
      for (int hotk : {192, 384}) {
        const int bs = 1024;  // one block per SM, 32 warps
        const long long nw = (long long)sms * 32;
        const long long per = ((n + nw - 1) / nw + 31) / 32 * 32;
        char nm[64];
        snprintf(nm, sizeof nm, "hot%d_w32", hotk);
        if (hotk <= tb.T) {
          if (hotk == 192) run(nm, [&] { g_ldg<192><<<sms, bs, 192 * RW * 8>>>(tab, idx, xs, n, per, out); });
          else run(nm, [&] { g_ldg<384><<<sms, bs, 384 * RW * 8>>>(tab, idx, xs, n, per, out); });
        }
      }
      {
        const int bs = 1024;
        const long long nw = (long long)sms * 32;
        const long long per = ((n + nw - 1) / nw + 31) / 32 * 32;
        run("ldg_w32_1blk", [&] { g_ldg<0><<<sms, bs>>>(tab, idx, xs, n, per, out); });
      }
      for (int wps : {16, 32, 48, 64}) {  // 256-bit loads, two rows per warp instruction
        const int bs = 256;
        const int bps = wps * 32 / bs;
        const long long nw = (long long)sms * bps * (bs / 32);
        const long long per = ((n + nw - 1) / nw + 31) / 32 * 32;
        char nm[64];
        snprintf(nm, sizeof nm, "ldg256_w%d", wps);
        run(nm, [&] { g_ldg256<<<sms * bps, bs>>>(tab, idx, xs, n, per, out); });
      }
      for (int S : {4, 8, 16}) {
        for (int bps : {1, 2, 4, 6}) {
          const int bs = 256;
          const size_t smem = (size_t)8 * S * (RW * 8 + 8);
          if (smem * bps > 220 * 1024) continue;
          const long long nw = (long long)sms * bps * 8;
          const long long per = ((n + nw - 1) / nw + 31) / 32 * 32;
          char nm[64];
          snprintf(nm, sizeof nm, "bulk_S%d_w%d", S, bps * 8);
          if (S == 4) run(nm, [&] { g_bulk<4><<<sms * bps, bs, smem>>>(tab, idx, xs, n, per, out); });
          if (S == 8) run(nm, [&] { g_bulk<8><<<sms * bps, bs, smem>>>(tab, idx, xs, n, per, out); });
          if (S == 16) run(nm, [&] { g_bulk<16><<<sms * bps, bs, smem>>>(tab, idx, xs, n, per, out); });
        }
      }
    }
  }
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"clock_khz\": %d}\n", prop.name, sms, prop.l2CacheSize,
         prop.clockRate);
  return 0;
}
