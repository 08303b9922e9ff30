// kernels.cu -- the SaCD sweep on B200 (sm_100a): sparse MTTKRP, Gram-Hadamard H,
// the fused column-wise SaCD row update, Gram refresh and the objective.
//
// Paper: arXiv 2003.03572 ("P:n" = PAPER.md line n).  Readings C1-C19: DESIGN.md s3.
//   MTTKRP      m_ir = sum_{e in Omega^(n)_i} x_e a_(e,r) b_(e,r)      Eq 9
//   H           H = G_a * G_b                                         Eq 10
//   row update  for r = 0..R-1 (Gauss-Seidel within the row, C9):
//                 g = -m_r + sum_j u_j h_jr                           Eq 14
//                 u' = max(0, u_r - g/h_rr), d = u' - u_r              Eq 11-13
//                 z = -g d - (L_r/2) d^2                               Eq 20
//                 select: FIRST z>0 | EQ24 z-zprev>0 | EQ27 zprev-z>0  Alg 1, Eq 24/27
//                 if selected u_r <- u'; zprev_r <- z                  P:598 (C8)
//   objective   f = ||X||^2 - 2 sum_s w_s.m^W_s + 1^T(G_U*G_V*G_W)1   Eq 6-7, C1
//
// Determinism: no floating-point atomics anywhere; every reduction has a fixed order, so
// reruns are bitwise identical (unchanged elements recompute the same z exactly).
//
// The kernels live in fragments included below (one translation unit): k_mttkrp.inc.cuh
// (A3), k_rows.inc.cuh (A2 H / branch, A4 row update), k_gram.inc.cuh (Gram refresh),
// k_pass.inc.cuh (pass records / objective, delta exchange, sharding helpers, predict).
// This file keeps the helpers, the launch implementations (Impl) and the C++ entry points.
#include <math.h>

#include <nccl.h>

#include "sacd_internal.cuh"

namespace sacd {

namespace {

#ifdef SACD_DEBUG
__device__ DebugBounds g_dbg;
__global__ void k_set_dbg(DebugBounds b) { g_dbg = b; }
#define SACD_DBG(x) x
#else
#define SACD_DBG(x)
#endif

// ------------------------------------------------------------------ small helpers
inline int grid1d(long long n, int block = 256) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

template <typename Real>
struct V16;
template <>
struct V16<float> {
  using T = float4;
  static constexpr int N = 4;
  __device__ static inline void get(const T &v, float *o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
  __device__ static inline T make(const float *o) { return make_float4(o[0], o[1], o[2], o[3]); }
};
template <>
struct V16<double> {
  using T = double2;
  static constexpr int N = 2;
  __device__ static inline void get(const T &v, double *o) { o[0] = v.x; o[1] = v.y; }
  __device__ static inline T make(const double *o) { return make_double2(o[0], o[1]); }
};

// Streaming loads for the nonzero arrays: read once per pass, keep L1 for factor rows.
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream_f32(const float *p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// Row-update loads (not volatile, so the compiler may batch them): M and z_prev stream through
// once per pass and must not evict H, which every block of the pass re-reads from L1.
__device__ __forceinline__ double ld_stream_f64(const double *p) {  // read-only in the kernel
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_na_f64(const double *p) {  // coherent, no L1 allocation
  double v;
  asm("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_keep_f64(const double *p) {  // read-only, kept in L1
  double v;
  asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Asynchronous global -> shared copies (LDGSTS): the row-block staging of the row-update
// kernels keeps every load in flight at once instead of one register round trip per element.
template <int BYTES>
__device__ __forceinline__ void cp_async(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(sa), "l"(gmem), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Reading C12: rand(seed, tag, ctr) = mix64(mix64(seed ^ tag) + (ctr + 1) * golden)
#ifndef SACD_ROWS_WARPS
#define SACD_ROWS_WARPS 4  // warps (x 32 rows) per block of the dynamic fp64 row update (2: 4 CTAs/SM, 3: 6 warps/SM, both slower)
#endif

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// M (the MTTKRP result) and Z (z_prev) are stored "TT": 32-row tiles, column-major inside a
// tile, so the thread-per-row update reads and writes them as contiguous 256-byte warp
// accesses.  Element (i, c) of a matrix with row pitch RT lives at tt(i, c).
template <int RT>
__host__ __device__ __forceinline__ long long tt(long long i, int c) {
  return (i >> 5) * (32LL * RT) + (long long)c * 32 + (i & 31);
}

template <int RT>
__host__ __device__ constexpr int rows_per_block() {
  return RT <= 64 ? 128 : (RT == 128 ? 64 : 32);
}

template <typename Real, int RT>
__host__ __device__ constexpr bool h_in_smem() {
  return (size_t)RT * RT * sizeof(Real) <= 64 * 1024;
}

template <typename Real, int RT, bool HS = h_in_smem<Real, RT>()>
__host__ __device__ constexpr size_t rows_smem_bytes() {
  return (HS ? (size_t)RT * RT * sizeof(Real) : 0) + (size_t)rows_per_block<RT>() * (RT + 1) * sizeof(Real);
}

template <int RT>
__host__ __device__ constexpr int gram_tg() {
  return RT <= 16 ? RT : (RT <= 128 ? 16 : 32);
}

// ------------------------------------------------------------------ init (Alg 1 input, C12)
template <typename Real>
__global__ void k_init_factors(Real *__restrict__ F, long long I, int R, int RT, unsigned long long seed,
                               unsigned long long off) {
  const unsigned long long base = mix64(seed ^ 1ULL);  // tag INIT = 1
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < I * RT;
       x += (long long)gridDim.x * blockDim.x) {
    const long long i = x / RT;
    const int r = (int)(x - i * RT);
    Real v = Real(0);
    if (r < R) {
      const unsigned long long ctr = off + (unsigned long long)i * R + r;
      const unsigned long long u = mix64(base + (ctr + 1ULL) * 0x9E3779B97F4A7C15ULL);
      v = (Real)((double)(u >> 40) * (1.0 / 16777216.0));
    }
    F[x] = v;
  }
}

#include "k_mttkrp.inc.cuh"
#include "k_rows.inc.cuh"
#include "k_gram.inc.cuh"
#include "k_pass.inc.cuh"

// ------------------------------------------------------------------ launch implementations
template <typename Real, int RT>
struct Impl {
  static int mttkrp(Context &c, int mode, void *out_v) {
    ModeData &md = c.m[mode];
    return mttkrp_on(c, mode, md.items, md.n_items, md.splits, md.n_splits, md.chunks, md.n_chunks,
                     reinterpret_cast<Real *>(out_v),
                     reinterpret_cast<Real *>(c.partial));
  }

  // the dynamically scheduled lean kernel (one worker per warp): a grid of resident blocks
  // only, items from c.item_ctr (reset here, stream-ordered)
  // SW = 32: one worker per warp (k_mttkrp_lean_dyn); SW < 32: 32/SW workers per warp
  // (k_mttkrp_lean_dyn_sw), each taking its own items from the counter
  template <int D, int MINB, int XS, int SW = 32, int PF = 0>
  static void launch_dyn(Context &c, const WorkItem *items, long long n_items, const uint4 *nzm, const Real *A,
                         const Real *B, Real *out, Real *partial) {
    auto go = [&](auto kern) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
      if (per_sm < 1) per_sm = 1;
      const long long need = (n_items * SW + 255) / 256;
      const long long grid = std::min<long long>(need, (long long)per_sm * c.num_sms);
      cudaMemsetAsync(c.item_ctr, 0, sizeof(unsigned long long), c.stream);
      kern<<<(unsigned)std::max<long long>(1, grid), 256, 0, c.stream>>>(items, n_items, nzm, A, B, out, partial,
                                                                         c.item_ctr, (Real)c.xu);
    };
    if constexpr (SW == 32) go(k_mttkrp_lean_dyn<Real, RT, D, MINB, PF, XS>);
    else go(k_mttkrp_lean_dyn_sw<Real, RT, SW, D, MINB, PF, XS>);
  }

  static int mttkrp_on(Context &c, int mode, const WorkItem *items, long long n_items, const SplitRow *splits,
                       long long n_splits, const FixChunk *chunks, long long n_chunks, Real *out, Real *partial) {
    ModeData &md = c.m[mode];
    const Real *A = reinterpret_cast<const Real *>(c.m[md.a].F);
    const Real *B = reinterpret_cast<const Real *>(c.m[md.b].F);
#ifdef SACD_DEBUG
    {
      const DebugBounds db{c.nnz, c.m[md.a].I, c.m[md.b].I, md.I, c.max_slots, c.max_chunks};
      k_set_dbg<<<1, 1, 0, c.stream>>>(db);
    }
#endif
    int pe = prof_begin(c, 0);
    if (n_items > 0) {
      const int wpb = 8;
      const long long blocks = (n_items + wpb - 1) / wpb;
      if constexpr (RT >= 32) {
        // (NB gathers in flight per warp, min blocks per SM); opt.mttkrp_variant selects a
        // tuning variant (0 = default, measured on B200 with tools/mttkrp_tune.py:
        // occupancy beats deeper per-warp batching).
#ifdef SACD_TUNING
        // measured tuning variants (tools/mttkrp_tune.py; built only with -DSACD_TUNING, so the
        // default library carries only the default kernels)
        const int var = c.opt.mttkrp_variant;
        auto go = [&](auto kern) {
          kern<<<(unsigned)blocks, wpb * 32, 0, c.stream>>>(items, n_items, md.idx_a, md.idx_b, md.val, md.idx_n, A,
                                                           B, out, partial);
        };
        constexpr int SW = sub_warp_lanes<Real, RT>();
        const long long sblocks = (n_items * SW + 255) / 256;
        auto gos = [&](auto kern) {
          kern<<<(unsigned)sblocks, 256, 0, c.stream>>>(items, n_items, md.nzm, A, B, out, partial);
        };
        if (var != 0) {
          if (var == 1) go(k_mttkrp_fiber<Real, RT, 1, fiber_min_blocks<Real, RT>()>);
        else if (var == 10) gos(k_mttkrp_sw<Real, RT, SW, 1, 4>);
        else if (var == 11) gos(k_mttkrp_sw<Real, RT, SW, 2, 4>);
        else if (var == 12) gos(k_mttkrp_sw<Real, RT, SW, 4, 4>);
        else if (var == 13) gos(k_mttkrp_sw<Real, RT, SW, 4, 3>);
        else if (var == 14) gos(k_mttkrp_sw<Real, RT, SW, 8, 2>);
        else if (var == 15) gos(k_mttkrp_sw<Real, RT, SW, 2, 6>);
        else if (var >= 50 && var < 60) {
          // round-2 occupancy / broadcast variants of the fp64 R = 64 kernel (c4)
          if constexpr (sizeof(Real) == 8 && RT == 64) {
            const bool ux = c.uniform_x;
            if (var == 50) launch_dyn<1, 4, 1>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 51) launch_dyn<1, 4, 3, 16>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 52) launch_dyn<1, 3, 3, 16>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 53 && ux) launch_dyn<1, 6, 4>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 54 && ux) launch_dyn<1, 4, 4>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 55 && ux) launch_dyn<1, 4, 4, 16>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 56) launch_dyn<2, 4, 1>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 57) launch_dyn<1, 5, 1>(c, items, n_items, md.nzm, A, B, out, partial);
            else launch_dyn<1, 6, 1>(c, items, n_items, md.nzm, A, B, out, partial);
          }
        }
        else if (var >= 60 && var < 70) {
          // L1 policy of the row gathers (the fp64 R = 64 kernel on a uniform-valued tensor, c4)
          if constexpr (sizeof(Real) == 8 && RT == 64) {
            const bool ux = c.uniform_x;
            if (var == 60 && ux) launch_dyn<1, 6, 4, 32, 4>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 60) launch_dyn<1, 6, 1, 32, 4>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 61 && ux) launch_dyn<1, 6, 4, 32, 5>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 61) launch_dyn<1, 6, 1, 32, 5>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 62 && ux) launch_dyn<1, 6, 4, 32, 6>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 62) launch_dyn<1, 6, 1, 32, 6>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 63 && ux) launch_dyn<1, 6, 4, 32, 7>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (var == 63) launch_dyn<1, 6, 1, 32, 7>(c, items, n_items, md.nzm, A, B, out, partial);
            else if (ux) launch_dyn<1, 6, 4>(c, items, n_items, md.nzm, A, B, out, partial);
            else launch_dyn<1, 6, 1>(c, items, n_items, md.nzm, A, B, out, partial);
          }
        }
        else if (var >= 20 && var < 50) {
          // lean kernel: E elements per lane -> SW = RT / E lanes per worker
          constexpr int VEC = V16<Real>::N;
          constexpr int E8 = 8 < VEC ? VEC : 8;
          constexpr int SW8 = RT / E8 > 32 ? 32 : (RT / E8 < 1 ? 1 : RT / E8);
          constexpr int E4 = 4 < VEC ? VEC : 4;
          constexpr int SW4 = RT / E4 > 32 ? 32 : (RT / E4 < 1 ? 1 : RT / E4);
          auto gol = [&](auto kern, int sw) {
            const long long lb = (n_items * sw + 255) / 256;
            kern<<<(unsigned)lb, 256, 0, c.stream>>>(items, n_items, md.nzm, A, B, out, partial, Real(0));
          };
          if constexpr (RT / VEC <= 32) {
            if (var == 26 || var == 27 || var == 28) {
              constexpr int EL = sizeof(Real) == 8 ? E4 : E8;
              constexpr int SWL = sizeof(Real) == 8 ? SW4 : SW8;
              const uint32_t *cmA = c.m[md.a].cmask, *cmB = c.m[md.b].cmask;
              (void)EL;
              auto gok = [&](auto kern) {
                const long long lb = (n_items * SWL + 255) / 256;
                kern<<<(unsigned)lb, 256, 0, c.stream>>>(items, n_items, md.nzm, A, B, cmA, cmB, out, partial);
              };
              if (var == 26) gok(k_mttkrp_skip<Real, RT, SWL, 1, sizeof(Real) == 8 ? 3 : 2>);
              else if (var == 27) gok(k_mttkrp_skip<Real, RT, SWL, 2, 2>);
              else gok(k_mttkrp_skip<Real, RT, SWL, 1, 2>);
              SACD_CUDA_TRY(cudaGetLastError());
              SACD_TRY(prof_end(c, 0, pe));
              goto fixup;
            }
          }
          if (var == 20) gol(k_mttkrp_lean<Real, RT, SW4, 1, 4>, SW4);
          else if (var == 21) gol(k_mttkrp_lean<Real, RT, SW4, 2, 3>, SW4);
          else if (var == 22) gol(k_mttkrp_lean<Real, RT, SW8, 1, 2>, SW8);
          else if (var == 23) gol(k_mttkrp_lean<Real, RT, SW8, 1, 3>, SW8);
          else if (var == 24) gol(k_mttkrp_lean<Real, RT, SW4, 1, 3>, SW4);
          else if (var == 45) gol(k_mttkrp_lean<Real, RT, SW4, 1, 3, 1>, SW4);
          else if (var == 46) gol(k_mttkrp_lean<Real, RT, SW4, 1, 3, 2>, SW4);
          else if (var == 47) gol(k_mttkrp_lean<Real, RT, SW4, 1, 3, 3>, SW4);
          else if (var == 48) gol(k_mttkrp_lean<Real, RT, SW8, 1, 2, 1>, SW8);
          else if (var == 49) gol(k_mttkrp_lean<Real, RT, SW8, 1, 2, 3>, SW8);
          // shared-memory broadcast of x (XS = 1) or of the b index and x (XS = 2)
          else if (var == 30) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 1, 5, 0, 1>, sub_warp_lanes<Real, RT>());
          else if (var == 31) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 1, 5, 0, 2>, sub_warp_lanes<Real, RT>());
          else if (var == 32) gol(k_mttkrp_lean<Real, RT, SW4, 1, 3, 0, 1>, SW4);
          else if (var == 33) gol(k_mttkrp_lean<Real, RT, SW4, 1, 3, 0, 2>, SW4);
          else if (var == 34) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 2, 5, 0, 2>, sub_warp_lanes<Real, RT>());
          else if (var == 35) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 1, 6, 0, 1>, sub_warp_lanes<Real, RT>());
          else if (var == 36) gol(k_mttkrp_lean<Real, RT, SW8, 1, 2, 0, 1>, SW8);
          else if (var == 39) {
            if constexpr (sizeof(Real) == 8 && RT == 64) launch_dyn<1, 6, 1>(c, items, n_items, md.nzm, A, B, out, partial);
            if constexpr (sizeof(Real) == 8 && RT == 128) launch_dyn<1, 3, 1>(c, items, n_items, md.nzm, A, B, out, partial);
            if constexpr (sizeof(Real) == 8 && RT == 256) launch_dyn<1, 2, 1>(c, items, n_items, md.nzm, A, B, out, partial);
            if constexpr (sizeof(Real) == 8 && RT == 32) {
              auto kern = k_mttkrp_lean_dyn_sw<Real, RT, 16, 1, 5, 0, 2>;
              int per_sm = 0;
              cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
              const long long need = (n_items * 16 + 255) / 256;
              const long long grid = std::min<long long>(need, (long long)std::max(1, per_sm) * c.num_sms);
              cudaMemsetAsync(c.item_ctr, 0, sizeof(unsigned long long), c.stream);
              kern<<<(unsigned)std::max<long long>(1, grid), 256, 0, c.stream>>>(items, n_items, md.nzm, A, B, out,
                                                                                 partial, c.item_ctr, Real(0));
            }
          }
          else if (var == 40) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 1, 6>, sub_warp_lanes<Real, RT>());
          else if (var == 41) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 1, 5>, sub_warp_lanes<Real, RT>());
          else if (var == 42) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 2, 5>, sub_warp_lanes<Real, RT>());
          else if (var == 43) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 2, 4>, sub_warp_lanes<Real, RT>());
          else if (var == 44) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 1, 8>, sub_warp_lanes<Real, RT>());
          else gol(k_mttkrp_lean<Real, RT, SW8, 2, 2>, SW8);
        }
        } else
#endif
        if (sizeof(Real) == 8 && RT >= 256) {
          // fp64, R > 128: one warp per item, 8 fp64 columns per lane, x broadcast through
          // shared memory (variant 36; c5 R=256: 12.7 ms per sweep vs 13.7 with shuffles,
          // variant 22, and 28.6 for the warp fiber kernel, variant 1)
          // Dynamically scheduled (items from a counter; c5 R=256 12.6 vs 13.1 ms, variant 39).
          if constexpr (sizeof(Real) == 8 && RT == 256) {
            if (c.uniform_x) launch_dyn<1, 2, 4>(c, items, n_items, md.nzm, A, B, out, partial);
            else launch_dyn<1, 2, 1>(c, items, n_items, md.nzm, A, B, out, partial);
          }
        } else if (sizeof(Real) == 8 && (RT == 64 || (RT == 32 && md.n_fibers > 0 && c.nnz >= 2 * md.n_fibers))) {
          // fp64, R = 33..64 (and R = 17..32 with a mean fiber length >= 2, the Zipf config
          // c3): one warp per item (2 fp64 columns per lane at R = 64) at 48 registers / 40
          // warps per SM (variant 41: c4 13.65 vs 15.17 ms per sweep, c3 1.22 vs 1.28).  x
          // reaches the lanes through a shared-memory broadcast (XS = 1: one L1 wavefront
          // instead of two shuffles on the L1-data-path-bound kernel; variant 30: c4 12.11 vs
          // 13.66 ms, c5 R=64 4.02 vs 4.42); with two workers per warp (R = 32) the b index
          // and x go as one 16-byte broadcast (XS = 2; variant 31: c3 1.195 vs 1.227 ms).
          if constexpr (sizeof(Real) == 8 && RT == 64) {
            // R = 64: 40 registers / 48 warps per SM (variant 35: c4 11.75 vs 12.11 ms), dynamically
            // scheduled from a work counter (variant 39: c4 11.06, c5 R=64 3.29 vs 3.82 ms; a
            // sharded rank's launch covers only ~2 waves of items, where the static grid lost
            // up to a third to the last wave)
            // A tensor whose values are all equal (binary interactions, c4) needs no per-nonzero
            // x at all (XS = 4; exact: x * b with the same x): c4 MTTKRP 11.12 -> 10.98 ms per
            // sweep (variant 53, profiles/r02_mttkrp_variants_c4.txt)
            if (c.uniform_x) launch_dyn<1, 6, 4>(c, items, n_items, md.nzm, A, B, out, partial);
            else launch_dyn<1, 6, 1>(c, items, n_items, md.nzm, A, B, out, partial);
          } else if constexpr (sizeof(Real) == 8 && RT == 32) {
            // two workers per warp, each taking items from the work counter (c3 0.98 vs
            // 1.09 ms per sweep for the static grid)
            auto kern = k_mttkrp_lean_dyn_sw<Real, RT, 16, 1, 5, 0, 2>;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
            const long long need = (n_items * 16 + 255) / 256;
            const long long grid = std::min<long long>(need, (long long)std::max(1, per_sm) * c.num_sms);
            cudaMemsetAsync(c.item_ctr, 0, sizeof(unsigned long long), c.stream);
            kern<<<(unsigned)std::max<long long>(1, grid), 256, 0, c.stream>>>(items, n_items, md.nzm, A, B, out,
                                                                               partial, c.item_ctr, Real(0));
          }
        } else if (sizeof(Real) == 8 && RT == 128) {
          // fp64, R = 65..128: 4 columns per lane, one warp per item, x broadcast through shared
          // memory (variant 32: c5 R=128 6.54 vs 6.95 ms, c4 R=128 21.5 vs 26.0 ms per sweep)
          if constexpr (sizeof(Real) == 8 && RT == 128) {
            // dynamically scheduled (variant 39: c5 R=128 6.38 vs 6.58, c4 R=128 18.8 vs 21.6 ms)
            if (c.uniform_x) launch_dyn<1, 3, 4>(c, items, n_items, md.nzm, A, B, out, partial);
            else launch_dyn<1, 3, 1>(c, items, n_items, md.nzm, A, B, out, partial);
          }
        } else {
          // default (measured on B200, tools/mttkrp_tune.py): the lean sub-warp kernel with
          // 4 fp64 / 8 fp32 columns per lane
          constexpr int VEC = V16<Real>::N;
          constexpr int EL = sizeof(Real) == 8 ? (4 < VEC ? VEC : 4) : (8 < VEC ? VEC : 8);
          constexpr int SWL = RT / EL > 32 ? 32 : (RT / EL < 1 ? 1 : RT / EL);
          constexpr int MB = sizeof(Real) == 8 ? 3 : 2;
          const long long lb = (n_items * SWL + 255) / 256;
          k_mttkrp_lean<Real, RT, SWL, 1, MB><<<(unsigned)lb, 256, 0, c.stream>>>(items, n_items, md.nzm, A, B, out,
                                                                                 partial);
        }
      } else {
        k_mttkrp<Real, RT><<<(unsigned)blocks, wpb * 32, 0, c.stream>>>(items, n_items, md.row_ptr, md.idx_a,
                                                                       md.idx_b, md.val, A, B, out, partial);
      }
    }
    SACD_CUDA_TRY(cudaGetLastError());
    SACD_TRY(prof_end(c, 0, pe));
#ifdef SACD_TUNING
  fixup:
#endif
    if (n_splits > 0) {
      pe = prof_begin(c, 1);
      Real *buf = reinterpret_cast<Real *>(c.fixbuf);
      k_fix1<Real, RT><<<(unsigned)((n_chunks + 7) / 8), 256, 0, c.stream>>>(chunks, n_chunks, partial, buf, out);
      k_fix2<Real, RT><<<(unsigned)((n_splits + 7) / 8), 256, 0, c.stream>>>(splits, n_splits, buf, out);
      SACD_CUDA_TRY(cudaGetLastError());
      SACD_TRY(prof_end(c, 1, pe));
    }
    return SACD_OK;
  }

  // ---- sharded engine -------------------------------------------------
  // With the peer-memory exchange and emulated ranks, every shard has its own factor
  // replicas: while a shard's kernels are launched the context's factor pointers are that
  // shard's replicas (restored to shard 0's on scope exit).
  struct ReplicaScope {
    Context &c;
    void *saved[3];
    ReplicaScope(Context &cc, const Shard &sh) : c(cc) {
      for (int k = 0; k < 3; ++k) {
        saved[k] = c.m[k].F;
        if (c.p2p && sh.Frep[k]) c.m[k].F = sh.Frep[k];
      }
    }
    ~ReplicaScope() {
      for (int k = 0; k < 3; ++k) c.m[k].F = saved[k];
    }
  };

  // flag barrier of the peer-memory exchange: every shard signals before any waits (emulated
  // ranks share one stream; across processes each rank has one shard)
  static void p2p_barrier(Context &c) {
    for (Shard &sh : c.shards) k_p2p_signal<<<1, 32, 0, c.stream>>>(sh.d_peer_flags, c.G, sh.rank, sh.epoch);
    for (Shard &sh : c.shards) k_p2p_wait<<<1, 32, 0, c.stream>>>(sh.flags, c.G, sh.rank, sh.epoch);
  }

  // the stats slots [ti, md, E, Ech, Gram] of the G ranks as this context reads them
  static double *stats_array(Context &c) { return (c.p2p && c.G > 1) ? c.shards[0].xstats_r : c.xstats; }

  // Each rank computes the MTTKRP of its nonzero range; the head partials (rows whose
  // first nonzero is on a lower rank) are exchanged and added by the owners in rank order.
  static int sharded_mttkrp_merge(Context &c, int mode) {
    for (Shard &sh : c.shards) {
      ReplicaScope rs(c, sh);
      SACD_TRY(mttkrp_on(c, mode, sh.items[mode], sh.n_items[mode], sh.splits[mode], sh.n_splits[mode],
                         sh.chunks[mode], sh.n_chunks[mode],
                         reinterpret_cast<Real *>(sh.M), reinterpret_cast<Real *>(sh.partial)));
    }
    if (c.p2p && c.G > 1) {
      // peer memory: every rank stores its head partial into slot `rank` of every rank's
      // arrays, then a flag barrier; each rank merges from its own arrays
      for (Shard &sh : c.shards)
        k_pack_head_p2p<Real, RT><<<1, 256, 0, c.stream>>>(sh.plan[mode].head, reinterpret_cast<const Real *>(sh.M),
                                                           sh.d_px, reinterpret_cast<Real *const *>(sh.d_pr), c.G,
                                                           sh.rank);
      p2p_barrier(c);
      for (Shard &sh : c.shards)
        k_merge_heads<Real, RT><<<1, 256, 0, c.stream>>>(c.G, sh.plan[mode].rlo, sh.plan[mode].rhi, sh.xid_r,
                                                         reinterpret_cast<const Real *>(sh.xrow_r),
                                                         reinterpret_cast<Real *>(sh.M));
      SACD_CUDA_TRY(cudaGetLastError());
      return SACD_OK;
    }
    Real *xrow = reinterpret_cast<Real *>(c.xrow);
    for (Shard &sh : c.shards)
      k_pack_head<Real, RT><<<1, 256, 0, c.stream>>>(sh.plan[mode].head, reinterpret_cast<const Real *>(sh.M),
                                                     c.xid + sh.rank, xrow + (long long)sh.rank * RT);
    SACD_CUDA_TRY(cudaGetLastError());
    if (c.comm) {
      SACD_TRY(nccl_allgather_inplace(c, c.xid, 1, 2));
      SACD_TRY(nccl_allgather_inplace(c, c.xrow, RT, sizeof(Real) == 8 ? 0 : 1));
    }
    for (Shard &sh : c.shards)
      k_merge_heads<Real, RT><<<1, 256, 0, c.stream>>>(c.G, sh.plan[mode].rlo, sh.plan[mode].rhi, c.xid, xrow,
                                                       reinterpret_cast<Real *>(sh.M));
    SACD_CUDA_TRY(cudaGetLastError());
    return SACD_OK;
  }

  static int sharded_mode_update(Context &c, int mode, int branch_override, bool begin_sweep, bool end_sweep,
                                 uint8_t *dec) {
    ModeData &md = c.m[mode];
    if (begin_sweep) k_sweep_begin<<<1, 32, 0, c.stream>>>(c.st);
    SACD_TRY(sharded_mttkrp_merge(c, mode));
    SACD_TRY(prepare(c, mode, branch_override, begin_sweep, 1));
    // p2p: the DMMA row kernels (fp64, R <= 64) store the changed chunks into the peers
    // themselves; the other row kernels are followed by k_p2p_push against a pass-start snapshot
    const bool fused_push = c.p2p && c.G > 1 && rows_push(c);
    if (c.delta || (c.p2p && !fused_push)) SACD_TRY(delta_snapshot(c, mode));
    const long long TR = rows_tr(c, 0);
    const long long slot = 4 + (long long)c.R * c.R;
    for (Shard &sh : c.shards) {
      ReplicaScope rs(c, sh);
      const long long rlo = sh.plan[mode].rlo, rhi = sh.plan[mode].rhi;
      const long long nblk = (rhi - rlo + TR - 1) / TR;
      double *ti_part = sh.row_part, *md_part = sh.row_part + c.max_row_blocks;
      long long *e_part = sh.cnt_part, *ech_part = sh.cnt_part + c.max_row_blocks;
      int pe = prof_begin(c, 3);
      int gn = 0;
      c.rows_peers = fused_push ? reinterpret_cast<void *const *>(sh.d_peerF[mode]) : nullptr;
      c.rows_me = sh.rank;
      if (nblk > 0)
        SACD_TRY(rows(c, nblk, rlo, rhi, mode, reinterpret_cast<const Real *>(sh.M), dec, ti_part, md_part, e_part,
                      ech_part, 0, gram_fused(c) ? sh.gram_part : nullptr, &gn));
      c.rows_peers = nullptr;
      SACD_CUDA_TRY(cudaGetLastError());
      SACD_TRY(prof_end(c, 3, pe));
      pe = prof_begin(c, 4);
      double *sl = ((c.p2p && c.G > 1) ? sh.xstats_r : c.xstats) + sh.rank * slot;
      if (gn == 0) {
        gn = gram_partial(c, rlo, rhi, reinterpret_cast<const Real *>(md.F), sh.gram_part);
      }
      k_gram_reduce<<<gram_reduce_blocks(c.R), 256, 0, c.stream>>>(c.R, gn, sh.gram_part, sl + 4);
      SACD_CUDA_TRY(cudaGetLastError());
      SACD_TRY(prof_end(c, 4, pe));
      k_finalize<<<1, 1024, 0, c.stream>>>(mode, nblk, ti_part, md_part, e_part, ech_part, nullptr, nullptr,
                                           nullptr, c.R, c.st, 8, sl);
      SACD_CUDA_TRY(cudaGetLastError());
      if (c.p2p && c.G > 1)  // this shard's stats slot into the other ranks' arrays
        k_push_slot<<<4, 256, 0, c.stream>>>(sl, sh.d_ps, slot, sh.rank * slot, c.G, sh.rank);
      if (c.p2p && !fused_push && rhi > rlo && c.G > 1)  // this shard's changed chunks into the peers' replicas
        k_p2p_push<Real><<<4 * c.num_sms, 256, 0, c.stream>>>(
            rlo * RT, rhi * RT, reinterpret_cast<const Real *>(md.F), reinterpret_cast<const Real *>(c.Fold),
            reinterpret_cast<Real *const *>(sh.d_peerF[mode]), c.G, sh.rank);
      SACD_CUDA_TRY(cudaGetLastError());
    }
    if (c.p2p && c.G > 1) {  // rows and stats pushed: one flag barrier
      p2p_barrier(c);
      SACD_CUDA_TRY(cudaGetLastError());
    } else if (c.comm) {
      SACD_TRY(nccl_allgather_inplace(c, c.xstats, (size_t)slot, 0));
    }
    int pe = prof_begin(c, 5);
    k_finalize_global<<<1, 1024, 0, c.stream>>>(mode, c.G, c.R, stats_array(c), md.G, c.m[0].G, c.m[1].G, c.m[2].G,
                                                c.st, 32 | 1 | (end_sweep ? 6 : 0));
    SACD_CUDA_TRY(cudaGetLastError());
    SACD_TRY(prof_end(c, 5, pe));
    if (c.p2p) {
      // rows already exchanged through peer memory
    } else if (c.delta) {
      SACD_TRY(delta_exchange(c, mode));
    } else if (c.comm) {
      SACD_TRY(nccl_broadcast_rows(c, mode));
    }
    SACD_TRY(chunk_mask(c, mode));
    return SACD_OK;
  }

  // snapshot of the local shards' owned rows before the pass (delta exchange)
  static int delta_snapshot(Context &c, int mode) {
    const size_t rb = (size_t)c.pitch * sizeof(Real);
    for (Shard &sh : c.shards) {
      const long long rlo = sh.plan[mode].rlo, rhi = sh.plan[mode].rhi;
      if (rhi > rlo)
        SACD_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char *>(c.Fold) + rlo * rb,
                                      reinterpret_cast<const char *>(c.m[mode].F) + rlo * rb, (rhi - rlo) * rb,
                                      cudaMemcpyDeviceToDevice, c.stream));
    }
    return SACD_OK;
  }

  // every owner compacts the changed elements of its rows into its list slot; the
  // lists travel instead of the rows (NCCL: list lengths all-gathered, then one grouped
  // broadcast per owner of the index and value arrays; full rows when that is smaller, as in
  // the first sweeps).  Emulated ranks exercise the same lists on one replica: the owned
  // rows are reset to the snapshot and every list is applied, so a compaction or apply error
  // changes the factors.
  static int delta_exchange(Context &c, int mode) {
    Real *F = reinterpret_cast<Real *>(c.m[mode].F);
    Real *Fo = reinterpret_cast<Real *>(c.Fold);
    Real *V = reinterpret_cast<Real *>(c.dval);
    for (Shard &sh : c.shards) {
      const int q = sh.rank;
      const long long lo = sh.plan[mode].rlo * c.pitch, hi = sh.plan[mode].rhi * c.pitch;
      k_delta_count<Real><<<kDeltaBlocks, 256, 0, c.stream>>>(lo, hi, F, Fo, c.dblk);
      k_delta_write<Real><<<kDeltaBlocks, 256, 0, c.stream>>>(lo, hi, F, Fo, c.dblk, c.didx + c.doff[q], V + c.doff[q],
                                                              c.dcnt + q);
    }
    SACD_CUDA_TRY(cudaGetLastError());
    const size_t rb = (size_t)c.pitch * sizeof(Real);
    if (!c.comm) {  // emulated ranks: reset the owned rows, apply every list in rank order
      for (Shard &sh : c.shards) {
        const long long rlo = sh.plan[mode].rlo, rhi = sh.plan[mode].rhi;
        if (rhi > rlo)
          SACD_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char *>(F) + rlo * rb,
                                        reinterpret_cast<const char *>(Fo) + rlo * rb, (rhi - rlo) * rb,
                                        cudaMemcpyDeviceToDevice, c.stream));
      }
      for (int q = 0; q < c.G; ++q)
        k_delta_apply<Real><<<kDeltaBlocks, 256, 0, c.stream>>>(c.didx + c.doff[q], V + c.doff[q], c.dcnt + q, F);
      SACD_CUDA_TRY(cudaGetLastError());
      return SACD_OK;
    }
    if (c.capturing) return nccl_broadcast_rows(c, mode);  // kernel count only; never replayed
    // a small factor (c4's W: 5 MB) goes as full rows: cheaper than the host round trip for
    // the list lengths
    if ((double)c.m[mode].I * c.pitch * sizeof(Real) < 16.0 * (1 << 20)) {
      long long nf = 0;
      for (int q = 0; q < c.G; ++q) nf += (c.all_plans[mode][q].rhi - c.all_plans[mode][q].rlo) * c.pitch;
      c.full_equiv += nf;
      return nccl_broadcast_rows(c, mode);
    }
    SACD_TRY(nccl_allgather_inplace(c, c.dcnt, 1, 2));
    std::vector<long long> h(c.G);
    SACD_CUDA_TRY(cudaMemcpyAsync(h.data(), c.dcnt, (size_t)c.G * 8, cudaMemcpyDeviceToHost, c.stream));
    SACD_CUDA_TRY(cudaStreamSynchronize(c.stream));
    long long nd = 0, nf = 0;
    for (int q = 0; q < c.G; ++q) {
      nd += h[q];
      nf += (c.all_plans[mode][q].rhi - c.all_plans[mode][q].rlo) * c.pitch;
    }
    c.full_equiv += nf;
    if (nd * (long long)(4 + sizeof(Real)) >= nf * (long long)sizeof(Real)) return nccl_broadcast_rows(c, mode);
    c.delta_sent += nd;
    const ncclDataType_t t = sizeof(Real) == 8 ? ncclFloat64 : ncclFloat32;
    ncclResult_t r = ncclGroupStart();
    for (int q = 0; q < c.G && r == ncclSuccess; ++q) {
      if (h[q] == 0) continue;
      r = ncclBroadcast(c.didx + c.doff[q], c.didx + c.doff[q], (size_t)h[q], ncclUint32, q,
                        reinterpret_cast<ncclComm_t>(c.comm), c.stream);
      if (r == ncclSuccess)
        r = ncclBroadcast(V + c.doff[q], V + c.doff[q], (size_t)h[q], t, q, reinterpret_cast<ncclComm_t>(c.comm),
                          c.stream);
    }
    const ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess) {
      set_error(std::string("ncclBroadcast (delta): ") + ncclGetErrorString(r != ncclSuccess ? r : r2));
      return SACD_ENCCL;
    }
    for (int q = 0; q < c.G; ++q)
      if (q != c.me && h[q] > 0)
        k_delta_apply<Real><<<kDeltaBlocks, 256, 0, c.stream>>>(c.didx + c.doff[q], V + c.doff[q], c.dcnt + q, F);
    SACD_CUDA_TRY(cudaGetLastError());
    return SACD_OK;
  }

  static int sharded_initial_fit(Context &c) {
    SACD_TRY(sharded_mttkrp_merge(c, 2));
    ModeData &md = c.m[2];
    constexpr int TR = rows_per_block<RT>();
    const long long slot = 4 + (long long)c.R * c.R;
    for (Shard &sh : c.shards) {
      const long long rlo = sh.plan[2].rlo, rhi = sh.plan[2].rhi;
      const long long nblk = (rhi - rlo + TR - 1) / TR;
      double *ti_part = sh.row_part, *md_part = sh.row_part + c.max_row_blocks;
      long long *e_part = sh.cnt_part, *ech_part = sh.cnt_part + c.max_row_blocks;
      if (nblk > 0)
        k_fm_dot<Real, RT><<<(unsigned)nblk, TR, 0, c.stream>>>(rlo, rhi, c.R, md.row_ptr,
                                                                reinterpret_cast<const Real *>(md.F),
                                                                reinterpret_cast<const Real *>(sh.M), ti_part,
                                                                md_part, e_part, ech_part);
      double *sl = ((c.p2p && c.G > 1) ? sh.xstats_r : c.xstats) + sh.rank * slot;
      k_finalize<<<1, 1024, 0, c.stream>>>(2, nblk, ti_part, md_part, e_part, ech_part, nullptr, nullptr, nullptr,
                                           c.R, c.st, 8, sl);
      if (c.p2p && c.G > 1) k_push_slot<<<4, 256, 0, c.stream>>>(sl, sh.d_ps, slot, sh.rank * slot, c.G, sh.rank);
    }
    SACD_CUDA_TRY(cudaGetLastError());
    if (c.p2p && c.G > 1) p2p_barrier(c);
    else if (c.comm) SACD_TRY(nccl_allgather_inplace(c, c.xstats, (size_t)slot, 0));
    k_finalize_global<<<1, 1024, 0, c.stream>>>(2, c.G, c.R, stats_array(c), nullptr, c.m[0].G, c.m[1].G, c.m[2].G,
                                                c.st, 2);
    SACD_CUDA_TRY(cudaGetLastError());
    return SACD_OK;
  }

  // merged MTTKRP of every shard's owned rows into c.M (entry point sacd_mttkrp)
  static int sharded_mttkrp_api(Context &c, int mode) {
    const size_t bytes = (size_t)((c.m[mode].I + 31) / 32 * 32) * RT * sizeof(Real);
    for (Shard &sh : c.shards) SACD_CUDA_TRY(cudaMemsetAsync(sh.M, 0, bytes, c.stream));
    SACD_TRY(sharded_mttkrp_merge(c, mode));
    for (Shard &sh : c.shards) {
      const long long rlo = sh.plan[mode].rlo, rhi = sh.plan[mode].rhi;
      if (rhi > rlo)
        k_copy_rows_tt<Real, RT><<<grid1d((rhi - rlo) * RT), 256, 0, c.stream>>>(
            rlo, rhi, reinterpret_cast<const Real *>(sh.M), reinterpret_cast<Real *>(c.M));
    }
    SACD_CUDA_TRY(cudaGetLastError());
    return SACD_OK;
  }

  // Gram partials of rows [rlo, rhi) of F: DMMA (fp64 tensor cores) for fp64 with RT >= 32
  // (opt.reserved[2] = 1 selects the FMA kernel), else the shared-memory FMA kernel
  // number of row ranges of a Gram over rows [rlo, rhi): c.gram_blocks, fewer for a short
  // range (a sharded rank's slice) so that no range is under 64 rows
  static int gram_ranges(const Context &c, long long rlo, long long rhi) {
    return (int)std::max<long long>(1, std::min<long long>(c.gram_blocks, (rhi - rlo + 63) / 64));
  }

  // Writes the partials of rows [rlo, rhi) of F to part[0 .. n) and returns n (the count
  // k_gram_reduce sums).  fp64 R <= 64: k_gram_stream (cp.async ring + DMMA), one partial per
  // resident CTA (at most gram_cap, at least 32 rows each); opt.reserved[2] = 3 keeps the
  // panel-pair DMMA kernel, 1 the FMA kernel (A/B)
  static int gram_partial(Context &c, long long rlo, long long rhi, const Real *F, double *part) {
    const int nb = gram_ranges(c, rlo, rhi);
    if constexpr (kGramStream) {
      if (c.opt.reserved[2] != 1 && c.opt.reserved[2] != 3) {
        int per_sm = 0;
        auto kern = k_gram_stream<RT, kGramStages>;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, gram_stream_smem_bytes<RT, kGramStages>());
        const long long nch = std::max<long long>(1, (rhi - rlo + 31) / 32);
        const int n = (int)std::min<long long>(std::min<long long>((long long)std::max(1, per_sm) * c.num_sms,
                                                                   (long long)c.gram_cap),
                                               nch);
        kern<<<(unsigned)n, 128, gram_stream_smem_bytes<RT, kGramStages>(), c.stream>>>(
            rlo, rhi, c.R, reinterpret_cast<const double *>(F), part);
        return n;
      }
    }
    if constexpr (sizeof(Real) == 8 && RT >= 32) {
      if (c.opt.reserved[2] != 1) {
        constexpr int NP = RT / 32;
        k_gram_dmma<RT><<<dim3(nb, NP * (NP + 1) / 2), 128, 0, c.stream>>>(
            rlo, rhi, c.R, reinterpret_cast<const double *>(F), part);
        return nb;
      }
    }
    constexpr int GT = gram_gt<RT>();
    constexpr int TG = gram_tg<GT>();
    constexpr int NB = RT / GT;
    k_gram_partial<Real, RT><<<dim3(nb, NB * (NB + 1) / 2), TG * TG, 0, c.stream>>>(rlo, rhi, c.R, F, part);
    return nb;
  }

  static int gram(Context &c, int mode) {
    ModeData &md = c.m[mode];
    int pe = prof_begin(c, 4);
    const int nb = gram_partial(c, 0, md.I, reinterpret_cast<const Real *>(md.F), c.gram_part);
    k_gram_reduce<<<gram_reduce_blocks(c.R), 256, 0, c.stream>>>(c.R, nb, c.gram_part, md.G);
    SACD_CUDA_TRY(cudaGetLastError());
    SACD_TRY(chunk_mask(c, mode));
    return prof_end(c, 4, pe);
  }

  // chunk support masks of F_mode (used by the skipping MTTKRP of the other modes)
  static int chunk_mask(Context &c, int mode) {
#ifndef SACD_TUNING
    (void)c;
    (void)mode;
    return SACD_OK;
#else
    const int var = c.opt.mttkrp_variant;
    if (var < 26 || var > 28) return SACD_OK;  // only the support-skipping variants read them
    if constexpr (RT / V16<Real>::N <= 32) {
      ModeData &md = c.m[mode];
      if (md.I > 0)
        k_chunk_mask<Real, RT><<<grid1d(md.I * 32), 256, 0, c.stream>>>(reinterpret_cast<const Real *>(md.F), md.I,
                                                                         md.cmask);
      SACD_CUDA_TRY(cudaGetLastError());
    }
    return SACD_OK;
#endif
  }

  static int prepare(Context &c, int mode, int branch_override, bool begin_sweep, int write_state) {
    ModeData &md = c.m[mode];
    int pe = prof_begin(c, 2);
    k_prepare<Real, RT><<<1, 1024, 0, c.stream>>>(mode, c.R, c.m[md.a].G, c.m[md.b].G, c.Hd,
                                                 reinterpret_cast<Real *>(c.Hr), c.st, branch_override,
                                                 begin_sweep ? 1 : 0, c.opt.variant, write_state);
    SACD_CUDA_TRY(cudaGetLastError());
    return prof_end(c, 2, pe);
  }

  static int mode_update(Context &c, int mode, int branch_override, bool begin_sweep, bool end_sweep,
                         uint8_t *dec) {
    ModeData &md = c.m[mode];
    Real *M = reinterpret_cast<Real *>(c.M);
    if (begin_sweep) k_sweep_begin<<<1, 32, 0, c.stream>>>(c.st);
    SACD_TRY(mttkrp(c, mode, M));
    SACD_TRY(prepare(c, mode, branch_override, begin_sweep, 1));
    const int vflags0 = c.opt.variant == SACD_VARIANT_SNAPSHOT ? 2 : (c.opt.variant == SACD_VARIANT_JACOBI ? 1 : 0);
    const long long TR = rows_tr(c, vflags0);
    const long long nblk = (md.I + TR - 1) / TR;
    double *ti_part = c.row_part, *md_part = c.row_part + c.max_row_blocks;
    long long *e_part = c.cnt_part, *ech_part = c.cnt_part + c.max_row_blocks;
    int gn = 0;
    int pe = prof_begin(c, 3);
    if (c.opt.variant == SACD_VARIANT_SNAPSHOT) {
      // (1) snapshot scores from the rows at pass start, (2) ti^k and this pass's branch,
      // (3) the Gauss-Seidel pass gated by the snapshot (reading C10')
      SACD_TRY(rows(c, nblk, 0, md.I, mode, M, nullptr, ti_part, md_part, e_part, ech_part, 1 | 2));
      k_snapshot_branch<<<1, 1024, 0, c.stream>>>(mode, nblk, ti_part, c.st, branch_override);
      SACD_TRY(rows(c, nblk, 0, md.I, mode, M, dec, ti_part, md_part, e_part, ech_part, 4));
    } else {
      SACD_TRY(rows(c, nblk, 0, md.I, mode, M, dec, ti_part, md_part, e_part, ech_part,
                    c.opt.variant == SACD_VARIANT_JACOBI ? 1 : 0, gram_fused(c) ? c.gram_part : nullptr, &gn));
    }
    SACD_CUDA_TRY(cudaGetLastError());
    SACD_TRY(prof_end(c, 3, pe));
    if (gn > 0) {  // the row kernel wrote one Gram partial per CTA: fixed-order reduce only
      pe = prof_begin(c, 4);
      k_gram_reduce<<<gram_reduce_blocks(c.R), 256, 0, c.stream>>>(c.R, gn, c.gram_part, md.G);
      SACD_CUDA_TRY(cudaGetLastError());
      SACD_TRY(prof_end(c, 4, pe));
    } else {
      SACD_TRY(gram(c, mode));
    }
    pe = prof_begin(c, 5);
    const int flags = 1 | (end_sweep ? 6 : 0);
    k_finalize<<<1, 1024, 0, c.stream>>>(mode, nblk, ti_part, md_part, e_part, ech_part, c.m[0].G, c.m[1].G,
                                         c.m[2].G, c.R, c.st, flags, nullptr);
    SACD_CUDA_TRY(cudaGetLastError());
    return prof_end(c, 5, pe);
  }

  static int initial_fit(Context &c) {
    Real *M = reinterpret_cast<Real *>(c.M);
    SACD_TRY(mttkrp(c, 2, M));
    ModeData &md = c.m[2];
    constexpr int TR = rows_per_block<RT>();
    const long long nblk = (md.I + TR - 1) / TR;
    double *ti_part = c.row_part, *md_part = c.row_part + c.max_row_blocks;
    long long *e_part = c.cnt_part, *ech_part = c.cnt_part + c.max_row_blocks;
    k_fm_dot<Real, RT><<<(unsigned)nblk, TR, 0, c.stream>>>(0, md.I, c.R, md.row_ptr, reinterpret_cast<const Real *>(md.F), M,
                                                            ti_part, md_part, e_part, ech_part);
    k_finalize<<<1, 1024, 0, c.stream>>>(2, nblk, ti_part, md_part, e_part, ech_part, c.m[0].G, c.m[1].G, c.m[2].G,
                                         c.R, c.st, 2, nullptr);
    SACD_CUDA_TRY(cudaGetLastError());
    return SACD_OK;
  }

  // predictions (out) and / or the squared-error sum (sse) at n device coordinates
  static int predict(Context &c, const uint32_t *coords, long long n, const float *vals, double *out, double *part,
                     double *sse) {
    const long long nb = (n + 7) / 8;
    if (n > 0)
      k_predict<Real, RT><<<(unsigned)nb, 256, 0, c.stream>>>(
          coords, n, reinterpret_cast<const Real *>(c.m[0].F), reinterpret_cast<const Real *>(c.m[1].F),
          reinterpret_cast<const Real *>(c.m[2].F), vals, out, part);
    if (sse) k_sum_parts<<<1, 1024, 0, c.stream>>>(part, n > 0 ? nb : 0, sse);
    SACD_CUDA_TRY(cudaGetLastError());
    return SACD_OK;
  }

  // the fused row update over rows [rlo, rhi) (nblk blocks); opt.reserved[0] = 1 reads H
  // from global memory (L1) instead of staging it in shared memory
  // rows per block of the row-update launch for these flags (the DMMA kernel: kMmaWarps x 32)
  static constexpr bool kRowsMma = sizeof(Real) == 8 && RT <= 64 && rows_per_block<RT>() == 128;
  static constexpr bool kRowsMmaBig = sizeof(Real) == 8 && RT >= 128;
  static constexpr int kMmaWarps = 4;  // the fused-Gram kernel; 5 (160 rows, 2 blocks per SM) measured 2.41 vs 1.72 ms: L1 too small
  static constexpr int kDynWarps = SACD_ROWS_WARPS;  // the dynamic / static row kernels
  // the Gram of the updated factor: a separate streaming kernel (k_gram_stream) after the row
  // update, or fused into the row update (k_sacd_rows_mma_gram; c4 rows + Gram 1.93 ms per
  // sweep fused vs 1.87 streaming)
  static constexpr bool kGramStream = sizeof(Real) == 8 && RT <= 64;
  static constexpr int kGramStages = 4;
  // the default fp64 R <= 64 row kernels (dynamic or with the fused Gram) push changed
  // chunks to the peers in their write-back
  static bool rows_push(const Context &c) {
    if constexpr (kRowsMma) return c.opt.reserved[0] == 0;
    return false;
  }
  // opt.reserved[2]: 0 = by size (fused while max I_n x R <= 2^20: small configs are launch-
  // bound and the fused kernel saves the Gram launch, c1 / c2 / c5 R <= 32; the streaming
  // kernel is faster from c3 / c5 R = 64 up), 2 = fused, 4 = streaming
  static bool gram_fused(const Context &c) {
    if constexpr (kRowsMma) {
      if (c.opt.reserved[0] != 0) return false;
      if (c.opt.reserved[2] == 2) return true;
      if (c.opt.reserved[2] != 0) return false;
      const long long imax = std::max(c.m[0].I, std::max(c.m[1].I, c.m[2].I));
      return imax * (long long)c.R <= (1LL << 20);
    }
    return false;
  }
  static int rows_tr(const Context &c, int vflags) {
    if constexpr (kRowsMma) {
      if ((c.opt.reserved[0] == 0 || c.opt.reserved[0] == 5 || c.opt.reserved[0] == 6) && vflags == 0)
        return gram_fused(c) ? kMmaWarps * 32 : kDynWarps * 32;
    }
    if constexpr (kRowsMmaBig) {
      if (c.opt.reserved[0] == 0 && vflags == 0) return 32;
    }
    return rows_per_block<RT>();
  }

  static int rows(Context &c, long long nblk, long long rlo, long long rhi, int mode, const Real *M, uint8_t *dec,
                  double *ti_part, double *md_part, long long *e_part, long long *ech_part, int vflags = 0,
                  double *gram_out = nullptr, int *gram_n = nullptr) {
    constexpr int TR = rows_per_block<RT>();
    ModeData &md = c.m[mode];
    if (gram_n) *gram_n = 0;
    auto go = [&](auto kern, size_t smem) {
      if (nblk > 0)
        kern<<<(unsigned)nblk, TR, smem, c.stream>>>(rlo, rhi, c.R, mode, c.opt.l_mode, md.row_ptr, M,
                                                      reinterpret_cast<Real *>(md.F), reinterpret_cast<Real *>(md.Z),
                                                      reinterpret_cast<const Real *>(c.Hr), c.st, dec, ti_part,
                                                      md_part, e_part, ech_part, vflags,
                                                      reinterpret_cast<Real *>(c.Zs));
    };
    if constexpr (kRowsMma) {
      if (gram_out && c.opt.reserved[0] == 0 && vflags == 0) {
        // default for fp64, R <= 64 with the Gram refresh fused (k_sacd_rows_mma_gram):
        // contiguous row-block ranges per CTA, one Gram partial per CTA into gram_out
        if (nblk > 0) {
          int per_sm = 0;
          auto kern = k_sacd_rows_mma_gram<RT, kMmaWarps>;
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMmaWarps * 32,
                                                        rows_mma_smem_bytes<RT, kMmaWarps>());
          const long long grid = std::min(std::min(nblk, (long long)std::max(1, per_sm) * c.num_sms),
                                          (long long)c.gram_cap);
          kern<<<(unsigned)grid, kMmaWarps * 32, rows_mma_smem_bytes<RT, kMmaWarps>(), c.stream>>>(
              rlo, rhi, c.R, mode, c.opt.l_mode, md.row_ptr, reinterpret_cast<const double *>(M),
              reinterpret_cast<double *>(md.F), reinterpret_cast<double *>(md.Z),
              reinterpret_cast<const double *>(c.Hr), c.st, dec, ti_part, md_part, e_part, ech_part, nblk, gram_out,
              reinterpret_cast<double *const *>(c.rows_peers), c.G, c.rows_me);
          if (gram_n) *gram_n = (int)grid;
        }
        SACD_CUDA_TRY(cudaGetLastError());
        return SACD_OK;
      }
      if ((c.opt.reserved[0] == 0 || c.opt.reserved[0] == 5) && vflags == 0) {
        // fp64, R <= 64 without the fused Gram: out-of-block gradient on DMMA, row blocks taken
        // from a work counter (c4 1.684 vs 1.720 ms per sweep for the static grid, variant 6)
        if (nblk > 0) {
          int per_sm = 0;
          auto kern = k_sacd_rows_mma_dyn<RT, kDynWarps>;
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDynWarps * 32,
                                                        rows_mma_smem_bytes<RT, kDynWarps>());
          const long long grid = std::min<long long>(nblk, (long long)std::max(1, per_sm) * c.num_sms);
          cudaMemsetAsync(c.item_ctr + 1, 0, sizeof(unsigned long long), c.stream);
          kern<<<(unsigned)grid, kDynWarps * 32, rows_mma_smem_bytes<RT, kDynWarps>(), c.stream>>>(
              rlo, rhi, c.R, mode, c.opt.l_mode, md.row_ptr, reinterpret_cast<const double *>(M),
              reinterpret_cast<double *>(md.F), reinterpret_cast<double *>(md.Z),
              reinterpret_cast<const double *>(c.Hr), c.st, dec, ti_part, md_part, e_part, ech_part, nblk,
              c.item_ctr + 1, reinterpret_cast<double *const *>(c.rows_peers), c.G, c.rows_me);
        }
        SACD_CUDA_TRY(cudaGetLastError());
        return SACD_OK;
      }
      if (c.opt.reserved[0] == 6 && vflags == 0) {  // the static grid (one block per row block)
        if (nblk > 0)
          k_sacd_rows_mma<RT, kDynWarps><<<(unsigned)nblk, kDynWarps * 32, rows_mma_smem_bytes<RT, kDynWarps>(),
                                            c.stream>>>(
              rlo, rhi, c.R, mode, c.opt.l_mode, md.row_ptr, reinterpret_cast<const double *>(M),
              reinterpret_cast<double *>(md.F), reinterpret_cast<double *>(md.Z),
              reinterpret_cast<const double *>(c.Hr), c.st, dec, ti_part, md_part, e_part, ech_part);
        SACD_CUDA_TRY(cudaGetLastError());
        return SACD_OK;
      }
    }
    if constexpr (kRowsMmaBig) {
      if (c.opt.reserved[0] == 0 && vflags == 0) {  // fp64, R > 64: DMMA gradient, one warp per block
        if (nblk > 0)
          k_sacd_rows_mma_big<RT><<<(unsigned)nblk, 32, rows_mma_big_smem_bytes<RT>(), c.stream>>>(
              rlo, rhi, c.R, mode, c.opt.l_mode, md.row_ptr, reinterpret_cast<const double *>(M),
              reinterpret_cast<double *>(md.F), reinterpret_cast<double *>(md.Z),
              reinterpret_cast<const double *>(c.Hr), c.st, dec, ti_part, md_part, e_part, ech_part);
        SACD_CUDA_TRY(cudaGetLastError());
        return SACD_OK;
      }
    }
    // reserved[0]: 1 = the FMA kernel with H read from global memory (L1), else (0 for the
    // other pitches / precisions, 2) the FMA kernel with H staged in shared memory
    if (c.opt.reserved[0] == 1) go(k_sacd_rows<Real, RT, false>, rows_smem_bytes<Real, RT, false>());
    else go(k_sacd_rows<Real, RT, h_in_smem<Real, RT>()>, rows_smem_bytes<Real, RT>());
    SACD_CUDA_TRY(cudaGetLastError());
    return SACD_OK;
  }

  static int setup(Context &c) {
    SACD_CUDA_TRY(cudaFuncSetAttribute(k_sacd_rows<Real, RT, h_in_smem<Real, RT>()>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_smem_bytes<Real, RT>()));
    SACD_CUDA_TRY(cudaFuncSetAttribute(k_sacd_rows<Real, RT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)rows_smem_bytes<Real, RT, false>()));
    if constexpr (kRowsMma) {
      SACD_CUDA_TRY(cudaFuncSetAttribute(k_sacd_rows_mma<RT, kDynWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)rows_mma_smem_bytes<RT, kDynWarps>()));
      SACD_CUDA_TRY(cudaFuncSetAttribute(k_sacd_rows_mma_dyn<RT, kDynWarps>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)rows_mma_smem_bytes<RT, kDynWarps>()));
      SACD_CUDA_TRY(cudaFuncSetAttribute(k_sacd_rows_mma_gram<RT, kMmaWarps>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)rows_mma_smem_bytes<RT, kMmaWarps>()));
    }
    if constexpr (kGramStream) {
      SACD_CUDA_TRY(cudaFuncSetAttribute(k_gram_stream<RT, kGramStages>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)gram_stream_smem_bytes<RT, kGramStages>()));
    }
    if constexpr (kRowsMmaBig)
      SACD_CUDA_TRY(cudaFuncSetAttribute(k_sacd_rows_mma_big<RT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)rows_mma_big_smem_bytes<RT>()));
    return SACD_OK;
  }
};

#define SACD_DISPATCH(c, EXPR)                                   \
  do {                                                           \
    const bool f64_ = (c).opt.precision == SACD_F64;             \
    switch ((c).pitch) {                                         \
      case 8:                                                    \
        if (f64_) { using I_ = Impl<double, 8>; return EXPR; }   \
        else { using I_ = Impl<float, 8>; return EXPR; }         \
      case 16:                                                   \
        if (f64_) { using I_ = Impl<double, 16>; return EXPR; }  \
        else { using I_ = Impl<float, 16>; return EXPR; }        \
      case 32:                                                   \
        if (f64_) { using I_ = Impl<double, 32>; return EXPR; }  \
        else { using I_ = Impl<float, 32>; return EXPR; }        \
      case 64:                                                   \
        if (f64_) { using I_ = Impl<double, 64>; return EXPR; }  \
        else { using I_ = Impl<float, 64>; return EXPR; }        \
      case 128:                                                  \
        if (f64_) { using I_ = Impl<double, 128>; return EXPR; } \
        else { using I_ = Impl<float, 128>; return EXPR; }       \
      case 256:                                                  \
        if (f64_) { using I_ = Impl<double, 256>; return EXPR; } \
        else { using I_ = Impl<float, 256>; return EXPR; }       \
      default:                                                   \
        set_error("bad pitch");                                  \
        return SACD_EINVAL;                                      \
    }                                                            \
  } while (0)

}  // namespace

size_t real_size(const Context &c) { return c.opt.precision == SACD_F64 ? 8 : 4; }

long long rows_block_for(const Context &c) {
  switch (c.pitch) {
    case 128: return 64;
    case 256: return 32;
    default: return 128;
  }
}

int launch_setup(Context &c) { SACD_DISPATCH(c, I_::setup(c)); }

int launch_init_factors(Context &c, uint64_t seed) {
  unsigned long long off = 0;
  for (int n = 0; n < 3; ++n) {
    ModeData &md = c.m[n];
    if (c.opt.precision == SACD_F64)
      k_init_factors<double><<<grid1d(md.I * c.pitch), 256, 0, c.stream>>>(reinterpret_cast<double *>(md.F), md.I,
                                                                             c.R, c.pitch, seed, off);
    else
      k_init_factors<float><<<grid1d(md.I * c.pitch), 256, 0, c.stream>>>(reinterpret_cast<float *>(md.F), md.I,
                                                                            c.R, c.pitch, seed, off);
    off += (unsigned long long)md.I * c.R;
  }
  SACD_CUDA_TRY(cudaGetLastError());
  return SACD_OK;
}

int launch_mttkrp(Context &c, int mode, void *out) { SACD_DISPATCH(c, I_::mttkrp(c, mode, out)); }

int launch_gram(Context &c, int mode) { SACD_DISPATCH(c, I_::gram(c, mode)); }

int launch_hessian_only(Context &c, int mode) { SACD_DISPATCH(c, I_::prepare(c, mode, -1, false, 0)); }

int launch_mode_update(Context &c, int mode, int branch_override, bool begin_sweep, bool end_sweep,
                       uint8_t *decisions_dev) {
  SACD_DISPATCH(c, I_::mode_update(c, mode, branch_override, begin_sweep, end_sweep, decisions_dev));
}

int launch_initial_fit(Context &c) { SACD_DISPATCH(c, I_::initial_fit(c)); }

__global__ void k_unpack_nzm(const uint4 *__restrict__ nzm, long long n, uint32_t *__restrict__ ia,
                             uint32_t *__restrict__ ib, float *__restrict__ v) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const uint4 r = nzm[e];
    ia[e] = r.x;
    ib[e] = r.y;
    v[e] = __uint_as_float(r.z);
  }
}

int launch_unpack_nzm(Context &c, const uint4 *nzm, long long nnz, uint32_t *ia, uint32_t *ib, float *v) {
  if (nnz > 0) k_unpack_nzm<<<grid1d(nnz), 256, 0, c.stream>>>(nzm, nnz, ia, ib, v);
  SACD_CUDA_TRY(cudaGetLastError());
  return SACD_OK;
}

int launch_range_check(Context &c, const uint32_t *coords, long long n, int *flag) {
  if (n > 0) k_range_check<<<grid1d(n), 256, 0, c.stream>>>(coords, n, c.dims[0], c.dims[1], c.dims[2], flag);
  SACD_CUDA_TRY(cudaGetLastError());
  return SACD_OK;
}

int launch_predict(Context &c, const uint32_t *coords, long long n, const float *vals, double *out, double *part,
                   double *sse) {
  SACD_DISPATCH(c, I_::predict(c, coords, n, vals, out, part, sse));
}

int launch_sharded_mode_update(Context &c, int mode, int branch_override, bool begin_sweep, bool end_sweep,
                               uint8_t *decisions_dev) {
  SACD_DISPATCH(c, I_::sharded_mode_update(c, mode, branch_override, begin_sweep, end_sweep, decisions_dev));
}

int launch_sharded_mttkrp(Context &c, int mode) { SACD_DISPATCH(c, I_::sharded_mttkrp_api(c, mode)); }

int launch_sharded_initial_fit(Context &c) { SACD_DISPATCH(c, I_::sharded_initial_fit(c)); }

// ------------------------------------------------------------------ NCCL transport
int nccl_allgather_inplace(Context &c, void *buf, size_t count, int dtype) {
  const ncclDataType_t t = dtype == 0 ? ncclFloat64 : (dtype == 1 ? ncclFloat32 : ncclInt64);
  const size_t esz = dtype == 1 ? 4 : 8;
  const ncclResult_t r = ncclAllGather(reinterpret_cast<char *>(buf) + (size_t)c.me * count * esz, buf, count, t,
                                       reinterpret_cast<ncclComm_t>(c.comm), c.stream);
  if (r != ncclSuccess) {
    set_error(std::string("ncclAllGather: ") + ncclGetErrorString(r));
    return SACD_ENCCL;
  }
  return SACD_OK;
}

// All-gather-v of the updated factor rows: one in-place broadcast per owner, grouped.
int nccl_broadcast_rows(Context &c, int mode) {
  const size_t rs = real_size(c);
  const ncclDataType_t t = rs == 8 ? ncclFloat64 : ncclFloat32;
  char *F = reinterpret_cast<char *>(c.m[mode].F);
  ncclResult_t r = ncclGroupStart();
  for (int q = 0; q < c.G && r == ncclSuccess; ++q) {
    const ShardPlan &p = c.all_plans[mode][q];
    const size_t cnt = (size_t)(p.rhi - p.rlo) * c.pitch;
    if (cnt == 0) continue;
    char *ptr = F + (size_t)p.rlo * c.pitch * rs;
    r = ncclBroadcast(ptr, ptr, cnt, t, q, reinterpret_cast<ncclComm_t>(c.comm), c.stream);
  }
  const ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess) {
    set_error(std::string("ncclBroadcast: ") + ncclGetErrorString(r != ncclSuccess ? r : r2));
    return SACD_ENCCL;
  }
  return SACD_OK;
}

int launch_convert_in(Context &c, const double *src_dev, long long rows, void *dst, bool ttl) {
  if (c.opt.precision == SACD_F64)
    k_convert_in<double><<<grid1d(rows * c.pitch), 256, 0, c.stream>>>(src_dev, rows, c.R, c.pitch,
                                                                        reinterpret_cast<double *>(dst), ttl);
  else
    k_convert_in<float><<<grid1d(rows * c.pitch), 256, 0, c.stream>>>(src_dev, rows, c.R, c.pitch,
                                                                       reinterpret_cast<float *>(dst), ttl);
  SACD_CUDA_TRY(cudaGetLastError());
  return SACD_OK;
}

int launch_convert_out(Context &c, const void *src, long long rows, double *dst_dev, bool ttl) {
  if (c.opt.precision == SACD_F64)
    k_convert_out<double><<<grid1d(rows * c.R), 256, 0, c.stream>>>(reinterpret_cast<const double *>(src), rows, c.R,
                                                                     c.pitch, dst_dev, ttl);
  else
    k_convert_out<float><<<grid1d(rows * c.R), 256, 0, c.stream>>>(reinterpret_cast<const float *>(src), rows, c.R,
                                                                    c.pitch, dst_dev, ttl);
  SACD_CUDA_TRY(cudaGetLastError());
  return SACD_OK;
}

}  // namespace sacd
