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
#include <math.h>

#include <nccl.h>

#include "sacd_internal.cuh"

namespace sacd {

namespace {

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

// Reading C12: rand(seed, tag, ctr) = mix64(mix64(seed ^ tag) + (ctr + 1) * golden)
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

// ------------------------------------------------------------------ sparse MTTKRP
// One warp per work item.  Lanes tile the row's R columns with 16-byte vectors (float4 /
// double2); when a row needs fewer than 32 lanes, the warp splits into G groups that take
// every G-th nonzero of the row and are combined by a fixed xor-shuffle tree at row end.
template <typename Real, int RT>
__global__ void __launch_bounds__(256) k_mttkrp(const WorkItem *__restrict__ items, long long n_items,
                                                const long long *__restrict__ row_ptr,
                                                const uint32_t *__restrict__ ia, const uint32_t *__restrict__ ib,
                                                const float *__restrict__ val, const Real *__restrict__ A,
                                                const Real *__restrict__ B, Real *__restrict__ M,
                                                Real *__restrict__ partial) {
  using VV = V16<Real>;
  using VT = typename VV::T;
  constexpr int VEC = VV::N;
  constexpr int NV = RT / VEC;
  constexpr int LPN = NV < 32 ? NV : 32;
  constexpr int VPL = NV / LPN;
  constexpr int G = 32 / LPN;
  const int lane = threadIdx.x & 31;
  const long long item = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= n_items) return;
  const WorkItem it = items[item];
  const int grp = lane / LPN, sub = lane % LPN;
  for (int row = it.row0; row < it.row1; ++row) {
    long long s = row_ptr[row], t = row_ptr[row + 1];
    if (s < it.nz0) s = it.nz0;
    if (t > it.nz1) t = it.nz1;
    Real acc[VPL][VEC];
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int c = 0; c < VEC; ++c) acc[v][c] = Real(0);
    for (long long e = s + grp; e < t; e += G) {
      const Real x = (Real)ld_stream_f32(val + e);
      const VT *ap = reinterpret_cast<const VT *>(A + (long long)(ld_stream_u32(ia + e) & kIdxMask) * RT);
      const VT *bp = reinterpret_cast<const VT *>(B + (long long)(ld_stream_u32(ib + e) & kIdxMask) * RT);
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        Real av[VEC], bv[VEC];
        VV::get(__ldg(ap + sub + v * LPN), av);
        VV::get(__ldg(bp + sub + v * LPN), bv);
#pragma unroll
        for (int c = 0; c < VEC; ++c) acc[v][c] = fma(x * av[c], bv[c], acc[v][c]);
      }
    }
#pragma unroll
    for (int off = LPN; off < 32; off <<= 1)
#pragma unroll
      for (int v = 0; v < VPL; ++v)
#pragma unroll
        for (int c = 0; c < VEC; ++c) acc[v][c] += __shfl_xor_sync(0xffffffffu, acc[v][c], off);
    if (grp == 0) {
      if (it.slot >= 0) {
        VT *dv = reinterpret_cast<VT *>(partial + it.slot * RT);
#pragma unroll
        for (int v = 0; v < VPL; ++v) dv[sub + v * LPN] = VV::make(acc[v]);
      } else {
        VT *dv = reinterpret_cast<VT *>(M + (long long)row * RT);
#pragma unroll
        for (int v = 0; v < VPL; ++v) dv[sub + v * LPN] = VV::make(acc[v]);
      }
    }
  }
}

// Wide-row MTTKRP (R > 16): one warp per work item, lane l owns columns [l*E, l*E+E),
// E = RT/32, so every factor-row gather is one coalesced RT*sizeof(Real)-byte warp access.
//  * The warp loads 32 nonzeros' (idx_a|flags, idx_b, x, row) with coalesced streaming
//    loads and broadcasts them by shuffle.
//  * Fiber factoring: the layout is sorted by (i_n, i_a, i_b), so a run of
//    equal i_a inside a row is a fiber, and m_i = sum_fibers a_(i_a) * (sum_e x_e b_(i_b(e))):
//    one a-row gather per fiber.  Fiber / row starts are precomputed flag bits of idx_a
//    (built with the layout), so the per-nonzero path is: 3 shuffles, one b-row gather
//    (prefetched one nonzero ahead), E FMAs.
//  * Rows are flushed to M[row] when a row starts; empty rows are never touched (the row
//    update reads row_ptr and uses m = 0 for them).  Split items (slot >= 0) hold a segment
//    of one heavy row and flush to their partial slot.
// Default occupancy target of k_mttkrp_fiber (measured on B200 with tools/mttkrp_tune.py:
// the kernel is latency-bound, so the most resident warps that fit without spilling win).
template <typename Real, int RT>
__host__ __device__ constexpr int fiber_min_blocks() {
  return (RT / 32) * sizeof(Real) <= 8 ? 7 : ((RT / 32) * sizeof(Real) <= 16 ? 6 : ((RT / 32) * sizeof(Real) <= 32 ? 4 : 2));
}

template <typename Real, int E>
struct LaneRow {
  Real v[E];
  __device__ __forceinline__ void load(const Real *p) {
    if constexpr (E * sizeof(Real) >= 16) {
      using VV = V16<Real>;
#pragma unroll
      for (int k = 0; k < (int)(E * sizeof(Real) / 16); ++k)
        VV::get(__ldg(reinterpret_cast<const typename VV::T *>(p) + k), v + k * VV::N);
    } else if constexpr (E * sizeof(Real) == 8) {
      if constexpr (sizeof(Real) == 8) {
        v[0] = __ldg(p);
      } else {
        const float2 t = __ldg(reinterpret_cast<const float2 *>(p));
        v[0] = t.x;
        v[1] = t.y;
      }
    } else {
      v[0] = __ldg(p);
    }
  }
  __device__ __forceinline__ void store(Real *p) const {
    if constexpr (E * sizeof(Real) >= 16) {
      using VV = V16<Real>;
#pragma unroll
      for (int k = 0; k < (int)(E * sizeof(Real) / 16); ++k)
        reinterpret_cast<typename VV::T *>(p)[k] = VV::make(v + k * VV::N);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k) p[k] = v[k];
    }
  }
};

template <typename Real, int RT, int NB, int MINB>
__global__ void __launch_bounds__(256, MINB) k_mttkrp_fiber(const WorkItem *__restrict__ items, long long n_items,
                                                      const uint32_t *__restrict__ ia,
                                                      const uint32_t *__restrict__ ib,
                                                      const float *__restrict__ val,
                                                      const uint32_t *__restrict__ in_,
                                                      const Real *__restrict__ A, const Real *__restrict__ B,
                                                      Real *__restrict__ M, Real *__restrict__ partial) {
  constexpr int E = RT / 32;
  const int lane = threadIdx.x & 31;
  const long long item = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= n_items) return;
  const WorkItem it = items[item];
  if (it.nz0 >= it.nz1) return;
  const Real *Al = A + lane * E;
  const Real *Bl = B + lane * E;
  LaneRow<Real, E> arow;
  Real acc[E], facc[E];
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = facc[k] = arow.v[k] = Real(0);
  long long cur_row = -1;
  Real *Ml = M + lane * E;
  auto flush = [&]() {
    LaneRow<Real, E> o;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      o.v[k] = acc[k];
      acc[k] = Real(0);
    }
    if (it.slot >= 0) o.store(partial + it.slot * RT + lane * E);
    else if (cur_row >= 0) o.store(Ml + cur_row * RT);
  };
  auto step = [&](uint32_t fa, float xf, const LaneRow<Real, E> &b, uint32_t my_n, int j) {
    if (fa & kFiberStart) {
#pragma unroll
      for (int k = 0; k < E; ++k) {            // close the previous fiber: acc += a * facc
        acc[k] = fma(arow.v[k], facc[k], acc[k]);
        facc[k] = Real(0);
      }
      if (fa & kRowStart) {
        flush();
        cur_row = __shfl_sync(0xffffffffu, my_n, j);
      }
      arow.load(Al + (long long)(fa & kIdxMask) * RT);
    }
    const Real x = (Real)xf;
#pragma unroll
    for (int k = 0; k < E; ++k) facc[k] = fma(x, b.v[k], facc[k]);
  };
  for (long long base = it.nz0; base < it.nz1; base += 32) {
    const int cnt = (int)min(32LL, it.nz1 - base);
    uint32_t my_a = 0, my_b = 0, my_n = 0;
    float my_x = 0.f;
    if (lane < cnt) {
      my_a = ld_stream_u32(ia + base + lane);
      my_b = ld_stream_u32(ib + base + lane);
      my_x = ld_stream_f32(val + base + lane);
      my_n = ld_stream_u32(in_ + base + lane);
    }
    if (base == it.nz0 && lane == 0) my_a |= kFiberStart | kRowStart;  // an item starts a row/fiber
    // batches of NB b-row gathers in flight per warp, then consumed in order
    for (int jb = 0; jb < cnt; jb += NB) {
      LaneRow<Real, E> bb[NB];
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        const uint32_t eb = __shfl_sync(0xffffffffu, my_b, (jb + u) & 31);
        if (jb + u < cnt) bb[u].load(Bl + (long long)(eb & kIdxMask) * RT);
      }
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        const int j = (jb + u) & 31;
        const uint32_t fa = __shfl_sync(0xffffffffu, my_a, j);
        const float xf = __shfl_sync(0xffffffffu, my_x, j);
        if (jb + u < cnt) step(fa, xf, bb[u], my_n, j);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = fma(arow.v[k], facc[k], acc[k]);
  flush();
}

// Sub-warp fiber MTTKRP (R > 16): a worker of SW lanes (8, 16 or 32) per work item, so one
// warp runs 32/SW items at once and every shuffle instruction serves all of them.
//  * Lane l of a worker owns the 16-byte column chunks k*SW + l (k < NV), so each chunk
//    load of a factor row is one contiguous SW*16-byte access (full sectors).
//  * The fiber / row flag bits ride on idx_b (layout.cu), so a nonzero costs two shuffles
//    (b index + flags, value); the a index and the row id are fetched only at fiber / row
//    starts.  The next batch's metadata is prefetched one batch ahead.
//  * NB b-rows (and, with PA, the a-rows of fibers starting among them) are issued before
//    any is consumed, so a worker keeps NB gathers in flight.
// Same arithmetic and order as k_mttkrp_fiber: m_i = sum_fibers a (.) (sum_e x_e b_e).
template <typename Real, int RT>
__host__ __device__ constexpr int sub_warp_lanes() {  // 16 bytes of a row per lane, at most 32 lanes
  return RT * (int)sizeof(Real) / 16 > 32 ? 32 : RT * (int)sizeof(Real) / 16;
}

template <typename Real, int RT, int SW>
struct SubRow {
  using VV = V16<Real>;
  using VT = typename VV::T;
  static constexpr int NV = RT / VV::N / SW;  // 16-byte chunks per lane
  static constexpr int E = NV * VV::N;
  Real v[E];
  // p = row base + lane * VEC
  __device__ __forceinline__ void load(const Real *p) {
#pragma unroll
    for (int k = 0; k < NV; ++k) VV::get(__ldg(reinterpret_cast<const VT *>(p) + k * SW), v + k * VV::N);
  }
  __device__ __forceinline__ void store(Real *p) const { store_from(p, v); }
  __device__ static __forceinline__ void store_from(Real *p, const Real (&x)[E]) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      Real t[VV::N];
#pragma unroll
      for (int c = 0; c < VV::N; ++c) t[c] = x[k * VV::N + c];
      reinterpret_cast<VT *>(p)[k * SW] = VV::make(t);
    }
  }
};

__device__ __forceinline__ uint4 ld_stream_u4(const uint4 *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Chunk support mask of each factor row: bit k = 16-byte chunk k (elements
// [k*VEC, (k+1)*VEC)) holds a nonzero.  One warp per row (lane k tests chunk k); rows of at
// most 32 chunks (RT * sizeof(Real) <= 512).  SaCD's projection leaves most factor entries
// exactly zero (tools/factor_stats.py: ~80% on c4), and the skipping MTTKRP uses these masks
// to gather only chunks where both the a-row and the b-row are nonzero.
template <typename Real, int RT>
__global__ void __launch_bounds__(256) k_chunk_mask(const Real *__restrict__ F, long long I,
                                                   uint32_t *__restrict__ cmask) {
  using VV = V16<Real>;
  constexpr int NCH = RT / VV::N;
  static_assert(NCH <= 32, "chunk masks hold at most 32 chunks");
  const int lane = threadIdx.x & 31;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long row = w0; row < I; row += nw) {
    bool nz = false;
    if (lane < NCH) {
      Real v[VV::N];
      VV::get(__ldg(reinterpret_cast<const typename VV::T *>(F + row * RT) + lane), v);
#pragma unroll
      for (int c = 0; c < VV::N; ++c) nz |= (v[c] != Real(0));
    }
    const uint32_t m = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) cmask[row] = m;
  }
}

template <typename Real, int RT, int SW, int NB, int MINB>
__global__ void __launch_bounds__(256, MINB) k_mttkrp_sw(const WorkItem *__restrict__ items, long long n_items,
                                                        const uint4 *__restrict__ nzm,
                                                        const Real *__restrict__ A, const Real *__restrict__ B,
                                                        Real *__restrict__ M, Real *__restrict__ partial) {
  using SR = SubRow<Real, RT, SW>;
  constexpr int E = SR::E;
  constexpr int VEC = V16<Real>::N;
  static_assert(SR::NV >= 1, "row narrower than a sub-warp of 16-byte chunks");
  const int lane = threadIdx.x & (SW - 1);
  const unsigned mask = SW == 32 ? 0xffffffffu : (((1u << SW) - 1u) << (threadIdx.x & 31 & ~(SW - 1)));
  const int shift = threadIdx.x & 31 & ~(SW - 1);  // this worker's lanes in a ballot
  const long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / SW;
  if (item >= n_items) return;
  const long long nz0 = items[item].nz0, nz1 = items[item].nz1;
  const int slot = (int)items[item].slot;
  if (nz0 >= nz1) return;
  const Real *Al = A + lane * VEC;
  const Real *Bl = B + lane * VEC;
  SR arow, anext;
  Real acc[E], facc[E];
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = facc[k] = arow.v[k] = anext.v[k] = Real(0);
  int cur_row = -1;
  bool need_next = true;  // the a-row of the next fiber start is not in flight yet
  for (long long base = nz0; base < nz1; base += SW) {
    const int cnt = (int)min((long long)SW, nz1 - base);
    // this batch's metadata: lane l holds nonzero base + l as {a|flags, b|flags, x, row}
    uint4 my = make_uint4(0u, 0u, 0u, 0u);
    if (lane < cnt) my = __ldg(nzm + base + lane);
    if (base + SW + lane < nz1) asm volatile("prefetch.global.L1 [%0];" ::"l"(nzm + base + SW + lane));
    if (base == nz0 && lane == 0) my.y |= kFiberStart | kRowStart;  // an item starts a row and a fiber
    // fiber starts of this batch (bit j = nonzero base + j)
    const unsigned fmask = (__ballot_sync(mask, (my.y & kFiberStart) != 0) >> shift) &
                           (SW == 32 ? 0xffffffffu : ((1u << SW) - 1u));
    if (need_next && fmask) {
      const int j0 = __ffs(fmask) - 1;
      anext.load(Al + (long long)(__shfl_sync(mask, my.x, j0, SW) & kIdxMask) * RT);
      need_next = false;
    }
    for (int jb = 0; jb < cnt; jb += NB) {
      SR bb[NB];
      uint32_t fb[NB];
      float xf[NB];
#pragma unroll
      for (int u = 0; u < NB; ++u) {  // NB gathers in flight (rows past cnt read row 0: harmless)
        const int j = (jb + u) & (SW - 1);
        fb[u] = __shfl_sync(mask, my.y, j, SW);
        xf[u] = __uint_as_float(__shfl_sync(mask, my.z, j, SW));
        bb[u].load(Bl + (long long)(fb[u] & kIdxMask) * RT);
      }
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        if (jb + u < cnt) {
          const int j = jb + u;
          if (fb[u] & kFiberStart) {
#pragma unroll
            for (int k = 0; k < E; ++k) {  // close the previous fiber: acc += a * facc
              acc[k] = fma(arow.v[k], facc[k], acc[k]);
              facc[k] = Real(0);
            }
            if (fb[u] & kRowStart) {
              const int nrow = (int)__shfl_sync(mask, my.w, j, SW);
              if (slot >= 0) SR::store_from(partial + (long long)slot * RT + lane * VEC, acc);
              else if (cur_row >= 0) SR::store_from(M + (long long)cur_row * RT + lane * VEC, acc);
#pragma unroll
              for (int k = 0; k < E; ++k) acc[k] = Real(0);
              cur_row = nrow;
            }
#pragma unroll
            for (int k = 0; k < E; ++k) arow.v[k] = anext.v[k];
            // issue the a-row of the next fiber start (in this batch, else at the next batch)
            const unsigned rest = j + 1 < 32 ? (fmask & ~((2u << j) - 1u)) : 0u;
            if (rest) {
              const int jn = __ffs(rest) - 1;
              anext.load(Al + (long long)(__shfl_sync(mask, my.x, jn, SW) & kIdxMask) * RT);
            } else {
              need_next = true;
            }
          }
          const Real x = (Real)xf[u];
#pragma unroll
          for (int k = 0; k < E; ++k) facc[k] = fma(x, bb[u].v[k], facc[k]);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = fma(arow.v[k], facc[k], acc[k]);
  if (slot >= 0) SR::store_from(partial + (long long)slot * RT + lane * VEC, acc);
  else if (cur_row >= 0) SR::store_from(M + (long long)cur_row * RT + lane * VEC, acc);
}

// Lean sub-warp fiber MTTKRP.  The MTTKRP is issue-bound (ncu: ~34 warp instructions per
// nonzero in the warp-per-item kernel), so this kernel minimises instructions per nonzero:
//  * SW lanes per worker (32/SW workers per warp), each lane holding E = RT/SW columns, so
//    every shuffle / address / branch instruction serves 32/SW nonzeros at once;
//  * the batch loop is fully unrolled over SW nonzeros; entries past the end carry x = 0,
//    b = 0 and no flags, so they add exact zeros instead of needing predicates;
//  * b-rows are prefetched D nonzeros ahead (registers renamed by the unroll), and the
//    next batch's 16-byte metadata is in flight while the current batch is consumed.
// Same arithmetic and order as k_mttkrp_fiber (bitwise-equal results).
// Prefetch of a batch's factor rows into L2 (PF = 1: a-rows of fiber starts; 3: also the
// b-rows) or L1 (PF = 2: a-rows): the per-fiber a-row gathers miss L2 on big factors and
// their latency is otherwise exposed at the next fiber close, ~2.7 nonzeros later.
template <typename Real, int RT, int PF>
__device__ __forceinline__ void prefetch_rows(const uint4 &m, bool valid, const Real *A, const Real *B) {
  constexpr int LINES = (RT * (int)sizeof(Real) + 127) / 128;
  if (!valid) return;
  if (m.y & kFiberStart) {
    const char *pa = reinterpret_cast<const char *>(A + (long long)(m.x & kIdxMask) * RT);
#pragma unroll
    for (int k = 0; k < LINES; ++k) {
      if (PF == 2) asm volatile("prefetch.global.L1 [%0];" ::"l"(pa + 128 * k));
      else asm volatile("prefetch.global.L2 [%0];" ::"l"(pa + 128 * k));
    }
  }
  if (PF == 3) {
    const char *pb = reinterpret_cast<const char *>(B + (long long)(m.y & kIdxMask) * RT);
#pragma unroll
    for (int k = 0; k < LINES; ++k) asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + 128 * k));
  }
}

// XS: how the batch's per-nonzero b index / x reach every lane of the worker: 0 = warp
// shuffles (1 for the b index, 2 for x in fp64), 1 = x through a shared-memory broadcast
// (one wavefront instead of two shuffles), 2 = the b index and x as one 16-byte
// shared-memory broadcast per nonzero.
template <typename Real, int RT, int SW, int D, int MINB, int PF = 0, int XS = 0>
__global__ void __launch_bounds__(256, MINB) k_mttkrp_lean(const WorkItem *__restrict__ items, long long n_items,
                                                          const uint4 *__restrict__ nzm,
                                                          const Real *__restrict__ A, const Real *__restrict__ B,
                                                          Real *__restrict__ M, Real *__restrict__ partial) {
  using SR = SubRow<Real, RT, SW>;
  constexpr int E = SR::E;
  constexpr int VEC = V16<Real>::N;
  static_assert(SR::NV >= 1, "row narrower than a sub-warp of 16-byte chunks");
  const int lane = threadIdx.x & (SW - 1);
  const unsigned mask = SW == 32 ? 0xffffffffu : (((1u << SW) - 1u) << (threadIdx.x & 31 & ~(SW - 1)));
  const long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / SW;
  if (item >= n_items) return;
  const long long nz0 = items[item].nz0, nz1 = items[item].nz1;
  const int slot = (int)items[item].slot;
  const Real *Al = A + lane * VEC;
  const Real *Bl = B + lane * VEC;
  __shared__ __align__(16) Real xsb[XS == 1 ? 2 : 1][XS == 1 ? 256 : 1];
  __shared__ __align__(16) uint4 rsb[XS == 2 ? 2 : 1][XS == 2 ? 256 : 1];
  const int wbase = threadIdx.x & ~(SW - 1);
  int par = 0;
  SR arow;
  Real acc[E], facc[E];
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = facc[k] = arow.v[k] = Real(0);
  int cur_row = -1;
  uint4 my = make_uint4(0u, 0u, 0u, 0u);
  if (nz0 + lane < nz1) my = ld_stream_u4(nzm + nz0 + lane);
  uint4 nx = make_uint4(0u, 0u, 0u, 0u);  // PF: metadata one batch ahead, rows prefetched
  if constexpr (PF > 0) {
    if (nz0 + SW + lane < nz1) nx = ld_stream_u4(nzm + nz0 + SW + lane);
    prefetch_rows<Real, RT, PF>(my, nz0 + lane < nz1, A, B);
  }
  if (lane == 0) my.y |= kFiberStart | kRowStart;  // an item starts a row and a fiber
  for (long long base = nz0; base < nz1; base += SW) {
    uint4 nx2 = make_uint4(0u, 0u, 0u, 0u);
    if constexpr (PF > 0) {
      if (base + 2 * SW + lane < nz1) nx2 = ld_stream_u4(nzm + base + 2 * SW + lane);
      prefetch_rows<Real, RT, PF>(nx, base + SW + lane < nz1, A, B);
    } else {
      nx = make_uint4(0u, 0u, 0u, 0u);  // lanes past the end must carry x = 0 and no flags
      if (base + SW + lane < nz1) nx = ld_stream_u4(nzm + base + SW + lane);
    }
    // x of this lane's nonzero, converted once per batch (F2F runs on the narrow XU pipe:
    // converting per nonzero in every lane of the worker made the fp64 kernel XU-bound)
    const Real xl = (Real)__uint_as_float(my.z);
    if constexpr (XS == 1) {
      par ^= 1;
      xsb[par][threadIdx.x] = xl;
      __syncwarp(mask);
    } else if constexpr (XS == 2) {
      par ^= 1;
      uint4 r;
      r.x = my.y;
      r.y = 0u;
      if constexpr (sizeof(Real) == 8) {
        r.z = (uint32_t)__double2loint((double)xl);
        r.w = (uint32_t)__double2hiint((double)xl);
      } else {
        r.z = __float_as_uint((float)xl);
        r.w = 0u;
      }
      rsb[par][threadIdx.x] = r;
      __syncwarp(mask);
    }
    uint32_t fb[SW];
    Real xr[D + 1];
    SR bb[D + 1];
    auto fetch = [&](int j) {  // b index + flags (and, XS == 2, x) of nonzero j of the batch
      if constexpr (XS == 2) {
        const uint4 r = rsb[par][wbase + j];
        fb[j] = r.x;
        if constexpr (sizeof(Real) == 8) xr[j % (D + 1)] = __hiloint2double((int)r.w, (int)r.z);
        else xr[j % (D + 1)] = __uint_as_float(r.z);
      } else {
        fb[j] = __shfl_sync(mask, my.y, j, SW);
      }
    };
#pragma unroll
    for (int j = 0; j < D && j < SW; ++j) {
      fetch(j);
      bb[j % (D + 1)].load(Bl + (long long)(fb[j] & kIdxMask) * RT);
    }
#pragma unroll
    for (int j = 0; j < SW; ++j) {
      if (j + D < SW) {
        fetch(j + D);
        bb[(j + D) % (D + 1)].load(Bl + (long long)(fb[j + D] & kIdxMask) * RT);
      }
      Real x;
      if constexpr (XS == 2) x = xr[j % (D + 1)];
      else if constexpr (XS == 1) x = xsb[par][wbase + j];
      else x = __shfl_sync(mask, xl, j, SW);
      if (fb[j] & kFiberStart) {
#pragma unroll
        for (int k = 0; k < E; ++k) {  // close the previous fiber: acc += a * facc
          acc[k] = fma(arow.v[k], facc[k], acc[k]);
          facc[k] = Real(0);
        }
        if (fb[j] & kRowStart) {
          if (slot >= 0) SR::store_from(partial + (long long)slot * RT + lane * VEC, acc);
          else if (cur_row >= 0) SR::store_from(M + (long long)cur_row * RT + lane * VEC, acc);
#pragma unroll
          for (int k = 0; k < E; ++k) acc[k] = Real(0);
          cur_row = (int)__shfl_sync(mask, my.w, j, SW);
        }
        arow.load(Al + (long long)(__shfl_sync(mask, my.x, j, SW) & kIdxMask) * RT);
      }
#pragma unroll
      for (int k = 0; k < E; ++k) facc[k] = fma(x, bb[j % (D + 1)].v[k], facc[k]);
    }
    my = nx;
    if constexpr (PF > 0) nx = nx2;
  }
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = fma(arow.v[k], facc[k], acc[k]);
  if (slot >= 0) SR::store_from(partial + (long long)slot * RT + lane * VEC, acc);
  else if (cur_row >= 0) SR::store_from(M + (long long)cur_row * RT + lane * VEC, acc);
}

// Support-skipping lean MTTKRP (exact).  Per nonzero, only the 16-byte chunks where both the
// fiber's a-row and the nonzero's b-row are nonzero (chunk masks, k_chunk_mask) are gathered
// and accumulated; a-rows are gathered only on their nonzero chunks.  Bitwise equal to the
// dense kernels: a skipped b chunk is zero (x*0 adds an exact zero), and a column whose a
// entry is zero only ever enters M as fma(0, facc, acc) = acc.  Lane l of a worker owns the
// chunks k*SW + l, i.e. bit k*SW + l of a mask.  The masks of a batch's nonzeros are
// gathered one batch ahead (lane l: masks of its nonzero's a- and b-rows).
template <typename Real, int RT, int SW, int D, int MINB>
__global__ void __launch_bounds__(256, MINB) k_mttkrp_skip(const WorkItem *__restrict__ items, long long n_items,
                                                          const uint4 *__restrict__ nzm,
                                                          const Real *__restrict__ A, const Real *__restrict__ B,
                                                          const uint32_t *__restrict__ cmA,
                                                          const uint32_t *__restrict__ cmB,
                                                          Real *__restrict__ M, Real *__restrict__ partial) {
  using SR = SubRow<Real, RT, SW>;
  using VV = V16<Real>;
  using VT = typename VV::T;
  constexpr int E = SR::E;
  constexpr int NV = SR::NV;
  constexpr int VEC = VV::N;
  static_assert(NV >= 1, "row narrower than a sub-warp of 16-byte chunks");
  static_assert(RT / VEC <= 32, "chunk masks hold at most 32 chunks");
  const int lane = threadIdx.x & (SW - 1);
  const unsigned mask = SW == 32 ? 0xffffffffu : (((1u << SW) - 1u) << (threadIdx.x & 31 & ~(SW - 1)));
  const long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / SW;
  if (item >= n_items) return;
  const long long nz0 = items[item].nz0, nz1 = items[item].nz1;
  const int slot = (int)items[item].slot;
  const Real *Al = A + lane * VEC;
  const Real *Bl = B + lane * VEC;
  Real arow[E], acc[E], facc[E];
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = facc[k] = arow[k] = Real(0);
  uint32_t am_cur = 0;  // chunk mask of the current fiber's a-row
  int cur_row = -1;
  // batch t: metadata `my` and the combined / a masks of its nonzeros; batch t+1: `nx`
  // (metadata) whose masks are gathered at the start of batch t; batch t+2: `nx2`.
  uint4 my = make_uint4(0u, 0u, 0u, 0u), nx = make_uint4(0u, 0u, 0u, 0u);
  if (nz0 + lane < nz1) my = ld_stream_u4(nzm + nz0 + lane);
  if (nz0 + SW + lane < nz1) nx = ld_stream_u4(nzm + nz0 + SW + lane);
  if (lane == 0) my.y |= kFiberStart | kRowStart;  // an item starts a row and a fiber
  uint32_t my_am = 0, my_m = 0;
  if (nz0 + lane < nz1) {
    my_am = __ldg(cmA + (my.x & kIdxMask));
    my_m = my_am & __ldg(cmB + (my.y & kIdxMask));
  }
  for (long long base = nz0; base < nz1; base += SW) {
    uint4 nx2 = make_uint4(0u, 0u, 0u, 0u);
    if (base + 2 * SW + lane < nz1) nx2 = ld_stream_u4(nzm + base + 2 * SW + lane);
    uint32_t nx_am = 0, nx_m = 0;
    if (base + SW + lane < nz1) {
      nx_am = __ldg(cmA + (nx.x & kIdxMask));
      nx_m = nx_am & __ldg(cmB + (nx.y & kIdxMask));
    }
    const Real xl = (Real)__uint_as_float(my.z);  // one XU conversion per lane per batch
    uint32_t fb[SW], mb[SW];
    Real bb[D + 1][E];
    auto issue = [&](int j) {
      fb[j] = __shfl_sync(mask, my.y, j, SW);
      mb[j] = __shfl_sync(mask, my_m, j, SW);
      const VT *p = reinterpret_cast<const VT *>(Bl + (long long)(fb[j] & kIdxMask) * RT);
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if ((mb[j] >> (k * SW + lane)) & 1u) VV::get(__ldg(p + k * SW), &bb[j % (D + 1)][k * VEC]);
    };
#pragma unroll
    for (int j = 0; j < D && j < SW; ++j) issue(j);
#pragma unroll
    for (int j = 0; j < SW; ++j) {
      if (j + D < SW) issue(j + D);
      const Real x = __shfl_sync(mask, xl, j, SW);
      if (fb[j] & kFiberStart) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {  // close the previous fiber on its a-row's nonzero chunks
          const bool on = (am_cur >> (k * SW + lane)) & 1u;
#pragma unroll
          for (int cc = 0; cc < VEC; ++cc) {
            if (on) acc[k * VEC + cc] = fma(arow[k * VEC + cc], facc[k * VEC + cc], acc[k * VEC + cc]);
            facc[k * VEC + cc] = Real(0);
          }
        }
        if (fb[j] & kRowStart) {
          if (slot >= 0) SR::store_from(partial + (long long)slot * RT + lane * VEC, acc);
          else if (cur_row >= 0) SR::store_from(M + (long long)cur_row * RT + lane * VEC, acc);
#pragma unroll
          for (int k = 0; k < E; ++k) acc[k] = Real(0);
          cur_row = (int)__shfl_sync(mask, my.w, j, SW);
        }
        am_cur = __shfl_sync(mask, my_am, j, SW);
        const VT *p = reinterpret_cast<const VT *>(Al + (long long)(__shfl_sync(mask, my.x, j, SW) & kIdxMask) * RT);
#pragma unroll
        for (int k = 0; k < NV; ++k)
          if ((am_cur >> (k * SW + lane)) & 1u) VV::get(__ldg(p + k * SW), &arow[k * VEC]);
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        if ((mb[j] >> (k * SW + lane)) & 1u) {
#pragma unroll
          for (int cc = 0; cc < VEC; ++cc)
            facc[k * VEC + cc] = fma(x, bb[j % (D + 1)][k * VEC + cc], facc[k * VEC + cc]);
        }
      }
    }
    my = nx;
    nx = nx2;
    my_am = nx_am;
    my_m = nx_m;
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const bool on = (am_cur >> (k * SW + lane)) & 1u;
#pragma unroll
    for (int cc = 0; cc < VEC; ++cc)
      if (on) acc[k * VEC + cc] = fma(arow[k * VEC + cc], facc[k * VEC + cc], acc[k * VEC + cc]);
  }
  if (slot >= 0) SR::store_from(partial + (long long)slot * RT + lane * VEC, acc);
  else if (cur_row >= 0) SR::store_from(M + (long long)cur_row * RT + lane * VEC, acc);
}

// Heavy rows split across items: M_row = sum of the row's partial slots, in two levels so
// that a row with thousands of slots (a 10%-of-nnz slice) is summed in parallel:
//   level 1: one warp per FixChunk sums its <= kFixChunk slots (4 independent running sums
//            over slots j = u mod 4, combined in u order) -> M[row] or a level-2 row;
//   level 2: one warp per split row with several chunks sums its chunk rows in order.
// Fixed orders throughout: deterministic.
template <typename Real, int RT>
__global__ void __launch_bounds__(256) k_fix1(const FixChunk *__restrict__ chunks, long long n,
                                              const Real *__restrict__ partial, Real *__restrict__ buf,
                                              Real *__restrict__ M) {
  constexpr int CPL = RT >= 32 ? RT / 32 : 1;  // columns per lane: c = lane + 32 q
  const int lane = threadIdx.x & 31;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n) return;
  const FixChunk fc = chunks[w];
  Real acc[4][CPL];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int q = 0; q < CPL; ++q) acc[u][q] = Real(0);
  for (int j0 = 0; j0 < fc.nslots; j0 += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (j0 + u < fc.nslots) {
        const Real *p = partial + (fc.slot0 + j0 + u) * RT;
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          if (lane + 32 * q < RT) acc[u][q] += p[lane + 32 * q];
      }
    }
  }
  Real *dst = fc.out < 0 ? M + (long long)(-fc.out - 1) * RT : buf + (long long)fc.out * RT;
#pragma unroll
  for (int q = 0; q < CPL; ++q)
    if (lane + 32 * q < RT) dst[lane + 32 * q] = (acc[0][q] + acc[1][q]) + (acc[2][q] + acc[3][q]);
}

template <typename Real, int RT>
__global__ void __launch_bounds__(256) k_fix2(const SplitRow *__restrict__ splits, long long n,
                                              const Real *__restrict__ buf, Real *__restrict__ M) {
  constexpr int CPL = RT >= 32 ? RT / 32 : 1;
  const int lane = threadIdx.x & 31;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n) return;
  const SplitRow sr = splits[w];
  const long long nch = (sr.nslots + kFixChunk - 1) / kFixChunk;
  if (nch <= 1) return;  // written by level 1
  Real acc[CPL];
#pragma unroll
  for (int q = 0; q < CPL; ++q) acc[q] = Real(0);
  for (long long k = 0; k < nch; ++k) {
    const Real *p = buf + (sr.chunk0 + k) * RT;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
      if (lane + 32 * q < RT) acc[q] += p[lane + 32 * q];
  }
#pragma unroll
  for (int q = 0; q < CPL; ++q)
    if (lane + 32 * q < RT) M[(long long)sr.row * RT + lane + 32 * q] = acc[q];
}

// ------------------------------------------------------------------ H, L and the branch
// H = G_a * G_b (Eq 10), L = ||H||_F (Alg 1), branch by reading C10.
template <typename Real, int RT>
__global__ void __launch_bounds__(1024) k_prepare(int mode, int R, const double *__restrict__ Ga,
                                                  const double *__restrict__ Gb, double *__restrict__ Hd,
                                                  Real *__restrict__ Hr, DevState *st, int branch_override,
                                                  int begin_sweep, int variant, int write_state) {
  __shared__ double red[1024];
  double ss = 0.0;
  for (int x = threadIdx.x; x < RT * RT; x += blockDim.x) {
    const int r = x / RT, t = x - (x / RT) * RT;
    double h = 0.0;
    if (r < R && t < R) {
      h = Ga[r * R + t] * Gb[r * R + t];
      Hd[r * R + t] = h;
      ss += h * h;
    }
    Hr[x] = (Real)h;
  }
  red[threadIdx.x] = ss;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0 && write_state) {
    if (begin_sweep) st->k += 1;
    int br;
    if (branch_override >= 0) br = branch_override;
    else if (variant == SACD_VARIANT_SELECT_OFF || st->nhist[mode] == 0) br = SACD_BR_FIRST;
    else if (st->nhist[mode] == 1) br = SACD_BR_EQ24;
    else br = (st->ti1[mode] > st->ti2[mode]) ? SACD_BR_EQ27 : SACD_BR_EQ24;
    st->branch[mode] = br;
    st->Lfrob[mode] = sqrt(red[0]);
  }
}

// ------------------------------------------------------------------ fused row update
// One thread per row (rows are independent given A and B: Eq ucap).  The block's
// rows are staged in shared memory with an odd stride (RT+1) so the per-thread column
// walk is bank-conflict free; H is staged in shared memory when it fits.
template <typename Real, int RT, bool HS>
__global__ void __launch_bounds__(rows_per_block<RT>())
    k_sacd_rows(long long row_begin, long long row_end, int R, int mode, int l_mode,
                const long long *__restrict__ row_ptr,
                const Real *__restrict__ M, Real *__restrict__ F,
                Real *__restrict__ Z, const Real *__restrict__ Hr, const DevState *__restrict__ st,
                uint8_t *__restrict__ dec, double *__restrict__ ti_part, double *__restrict__ md_part,
                long long *__restrict__ e_part, long long *__restrict__ ech_part, int vflags = 0,
                Real *__restrict__ Zs = nullptr) {
  // vflags (reading variants): 1 = JACOBI gradients from the rows at pass start
  // (Lemma 2 literal); 2 = SCORE only (with 1: the snapshot z of every element into Zs, ti,
  // no update); 4 = SNAP (Gauss-Seidel updates gated by the snapshot Zs, z_prev <- Zs)
  const bool jac = vflags & 1, score = vflags & 2, snap = vflags & 4;
  constexpr int TR = rows_per_block<RT>();
  constexpr int US = RT + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real *Hs = reinterpret_cast<Real *>(smem_raw);
  Real *Us = reinterpret_cast<Real *>(smem_raw + (HS ? (size_t)RT * RT * sizeof(Real) : 0));
  __shared__ double red_d[2][TR / 32];
  __shared__ long long red_l[2][TR / 32];

  const int tid = threadIdx.x;
  const long long row0 = row_begin + (long long)blockIdx.x * TR;
  const int nrows = (int)min((long long)TR, row_end - row0);
  if (HS) {
    constexpr int PER = 16 / (int)sizeof(Real);
    for (int x = tid; x < RT * RT / PER; x += TR) cp_async<16>(Hs + PER * x, Hr + PER * x);
  }
  const Real *Fg = F + row0 * RT;
  for (int x = tid; x < nrows * RT; x += TR) cp_async<(int)sizeof(Real)>(Us + (x / RT) * US + (x % RT), Fg + x);
  cp_async_wait_all();
  __syncthreads();
  const Real *H = HS ? Hs : Hr;
  const int branch = st->branch[mode];
  const Real Lf = (Real)st->Lfrob[mode];

  using VV = V16<Real>;
  using VT = typename VV::T;
  constexpr int VEC = VV::N;
  constexpr int C = 8;  // column block: each u_j read from shared memory feeds C FMAs
  double ti = 0.0, md = 0.0;
  long long E = 0, Ech = 0;
  // M is row-major (written by the MTTKRP as whole rows): each warp transposes the 32 x C
  // block of its rows through a small shared tile, so global reads stay coalesced.
  __shared__ Real Mst[TR / 32][32][C + 1];
  const int lane = tid & 31, wp = tid >> 5;
  const bool active = tid < nrows;
  {
    const long long row = row0 + tid;
    Real *u = Us + tid * US;
    const bool empty = active ? row_ptr[row] == row_ptr[row + 1] : true;  // empty slice: m = 0
    Real *zp = Z + tt<RT>(active ? row : row0, 0);         // z_prev in the TT layout
    Real *zsp = (score || snap) ? Zs + tt<RT>(active ? row : row0, 0) : nullptr;
    for (int c0 = 0; c0 < R; c0 += C) {
      __syncwarp();
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const int x = lane + 32 * k, rl = x / C, cl = x % C;
        const long long rg = row0 + wp * 32 + rl;
        Mst[wp][rl][cl] = (rg < row_end) ? M[rg * RT + c0 + cl] : Real(0);
      }
      __syncwarp();
      if (!active) continue;
      // (1) out-of-block part of the gradient with the current row (columns < c0 already
      //     updated), Eq 14:  acc_q = sum_{j not in block} u_j h_(j, c0+q)   (H symmetric)
      Real acc[C];
#pragma unroll
      for (int q = 0; q < C; ++q) acc[q] = Real(0);
      auto accumulate = [&](int j) {
        const Real uj = u[j];
        const VT *hj = reinterpret_cast<const VT *>(H + j * RT + c0);
#pragma unroll
        for (int x = 0; x < C / VEC; ++x) {
          Real hv[VEC];
          VV::get(hj[x], hv);
#pragma unroll
          for (int y = 0; y < VEC; ++y) acc[x * VEC + y] = fma(uj, hv[y], acc[x * VEC + y]);
        }
      };
#pragma unroll 4
      for (int j = 0; j < c0; ++j) accumulate(j);
#pragma unroll 4
      for (int j = c0 + C; j < R; ++j) accumulate(j);
      Real mv[C], zv[C], ub[C], zs[C];
#pragma unroll
      for (int q = 0; q < C; ++q) {
        mv[q] = Mst[wp][lane][q];
        zv[q] = score ? Real(0) : zp[32 * (c0 + q)];
        zs[q] = snap ? zsp[32 * (c0 + q)] : Real(0);
      }
#pragma unroll
      for (int q = 0; q < C; ++q) ub[q] = u[c0 + q];
      if (empty) {
#pragma unroll
        for (int q = 0; q < C; ++q) mv[q] = Real(0);
      }
      // (2) Gauss-Seidel inside the block (C9): column r adds the in-block terms from the
      //     CURRENT block values ub (never by subtracting old ones, so a gradient whose
      //     other terms are exactly zero is computed exactly, as in the oracle).
#pragma unroll
      for (int q = 0; q < C; ++q) {
        const int r = c0 + q;
        if (r < R) {
          const Real *Hr_ = H + r * RT;
          const Real h = Hr_[r];
          Real z = Real(0);
          bool sel = false;
          if (h != Real(0)) {
            Real sg = acc[q];
#pragma unroll
            for (int qq = 0; qq < C; ++qq) sg = fma(jac ? u[c0 + qq] : ub[qq], Hr_[c0 + qq], sg);
            const Real g = sg - mv[q];                     // Eq 14
            const Real ur = ub[q];
            const Real un = fmax(Real(0), ur - g / h);     // Eq 11-13
            const Real d = un - ur;                        // Eq 12
            const Real L = l_mode ? Lf : h;
            z = -g * d - (L * Real(0.5)) * d * d;          // Eq 20
            const Real zpr = zv[q];
            const Real zg = snap ? zs[q] : z;  // the score the gate sees
            sel = !score && ((branch == SACD_BR_FIRST) ? (zg > Real(0))
                                                       : ((branch == SACD_BR_EQ24) ? (zg - zpr > Real(0))
                                                                                   : (zpr - zg > Real(0))));
            if (sel) {
              ub[q] = un;
              E += 1;
              if (d != Real(0)) Ech += 1;
            }
          }
          if (snap) z = zs[q];
          zv[q] = z;                                       // z_prev <- z always (C8)
          ti += (double)z;                                 // Eq 25
          md += (double)ub[q] * (double)mv[q];
          if (dec && !score) dec[row * R + r] = (uint8_t)sel;
        }
      }
      if (score) {
#pragma unroll
        for (int q = 0; q < C; ++q) zsp[32 * (c0 + q)] = zv[q];
        continue;
      }
      if (jac) {  // the staged rows keep the pass-start values; updates go straight to F
#pragma unroll
        for (int q = 0; q < C; ++q)
          if (c0 + q < R) F[row * RT + c0 + q] = ub[q];
      } else {
#pragma unroll
        for (int q = 0; q < C; ++q) u[c0 + q] = ub[q];
      }
#pragma unroll
      for (int q = 0; q < C; ++q) zp[32 * (c0 + q)] = zv[q];
    }
  }
  __syncthreads();
  Real *Fo = F + row0 * RT;
  if (!jac && !score)
    for (int x = tid; x < nrows * RT; x += TR) Fo[x] = Us[(x / RT) * US + (x % RT)];

  // fixed-order block reduction of (ti, md, E, Ech)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ti += __shfl_xor_sync(0xffffffffu, ti, o);
    md += __shfl_xor_sync(0xffffffffu, md, o);
    E += __shfl_xor_sync(0xffffffffu, E, o);
    Ech += __shfl_xor_sync(0xffffffffu, Ech, o);
  }
  const int w = tid >> 5;
  if ((tid & 31) == 0) {
    red_d[0][w] = ti;
    red_d[1][w] = md;
    red_l[0][w] = E;
    red_l[1][w] = Ech;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    long long c = 0, d = 0;
    for (int k = 0; k < TR / 32; ++k) {
      a += red_d[0][k];
      b += red_d[1][k];
      c += red_l[0][k];
      d += red_l[1][k];
    }
    ti_part[blockIdx.x] = a;
    md_part[blockIdx.x] = b;
    e_part[blockIdx.x] = c;
    ech_part[blockIdx.x] = d;
  }
}

// Fused row update with the out-of-block gradient on the fp64 tensor cores (Real = double,
// RT <= 64).  Same semantics and per-row order of operations as k_sacd_rows: for column block
// [c0, c0+8) the out-of-block part acc_q = sum_{j not in block} u_j h_(j,c0+q) of every row
// of a warp (32 rows) is one (32 x RT) x (RT x 8) product of the CURRENT rows (columns < c0
// already updated this pass, Gauss-Seidel C9) with H, issued as DMMA m8n8k4 (4 row tiles x
// the k-steps outside the block, in ascending k); the in-block Gauss-Seidel step then runs
// one thread per row exactly as in k_sacd_rows.  Fragments: A[m][k] = u[8mt+m][4kk+k] held
// by lane (g = lane >> 2, t = lane & 3) as Us[8mt+g][4kk+t]; B[k][n] = H[4kk+k][c0+n] as
// H[4kk+t][c0+g] (from L1: H is read-only and shared by every block); C[g][2t + {0,1}].
// The accumulator tile and the block's M tile are transposed to one-row-per-thread through
// a per-warp shared tile.  Shared memory: Us (rows x (RT+2), conflict-free for both the
// fragment reads and the 16-byte row walks) + 32 x 18 doubles per warp.
template <int RT, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_sacd_rows_mma(long long row_begin, long long row_end, int R, int mode, int l_mode,
                    const long long *__restrict__ row_ptr, const double *__restrict__ M, double *__restrict__ F,
                    double *__restrict__ Z, const double *__restrict__ H, const DevState *__restrict__ st,
                    uint8_t *__restrict__ dec, double *__restrict__ ti_part, double *__restrict__ md_part,
                    long long *__restrict__ e_part, long long *__restrict__ ech_part) {
  constexpr int TR = WPB * 32;
  constexpr int US = RT + 2;
  constexpr int C = 8;
  constexpr int TS = 2 * C + 2;
  constexpr int NKS = RT / 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *Us = reinterpret_cast<double *>(smem_raw);
  double *Hd = Us + TR * US + WPB * 32 * TS;  // the 8 x 8 diagonal blocks of H: [RT/8][8][8]
  __shared__ double red_d[2][WPB];
  __shared__ long long red_l[2][WPB];

  const int tid = threadIdx.x;
  const int lane = tid & 31, wp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  double *Tw = Us + TR * US + wp * 32 * TS;
  const long long row0 = row_begin + (long long)blockIdx.x * TR;
  const int nrows = (int)min((long long)TR, row_end - row0);
  const double *Fg = F + row0 * RT;
  static_assert(((RT + 2) * 8) % 16 == 0, "row stride must keep 16-byte chunks aligned");
  for (int x = tid; x < TR * RT / 2; x += TR) {  // 16-byte chunks
    const int r = (2 * x) / RT, col = (2 * x) % RT;
    if (r < nrows) cp_async<16>(Us + r * US + col, Fg + 2 * x);
    else *reinterpret_cast<double2 *>(Us + r * US + col) = make_double2(0.0, 0.0);
  }
  cp_async_wait_all();
  for (int x = tid; x < RT * C; x += TR) {
    const int b = x / (C * C), q = (x / C) % C, qq = x % C;
    Hd[x] = H[(b * C + q) * RT + b * C + qq];
  }
  __syncthreads();
  const int branch = st->branch[mode];
  const double Lf = st->Lfrob[mode];
  const int kmax = (R + 3) / 4;  // k-steps past R multiply zero padding

  double ti = 0.0, md = 0.0;
  long long E = 0, Ech = 0;
  const bool active = tid < nrows;
  const long long row = row0 + tid;
  double *u = Us + tid * US;
  const bool empty = active ? row_ptr[row] == row_ptr[row + 1] : true;  // empty slice: m = 0
  double *zp = Z + tt<RT>(active ? row : row0, 0);
  const double *Uw = Us + (wp * 32 + g) * US + t;

  // software pipeline over column blocks: the B fragments, the M tile and this thread's
  // z_prev of block c0 + 8 are loaded while block c0 is processed (all read-only here)
  double bf[NKS], mt[C], zv[C];
  auto load_block = [&](int c, double (&b)[NKS], double (&mm)[C], double (&zz)[C]) {
    const int kb = c / 4;
#pragma unroll
    for (int kk = 0; kk < NKS; ++kk)
      b[kk] = (kk == kb || kk == kb + 1 || kk >= kmax) ? 0.0 : __ldg(H + (4 * kk + t) * RT + c + g);
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const int x = lane + 32 * k, rl = x / C, cl = x % C;
      const long long rg = row0 + wp * 32 + rl;
      mm[k] = (rg < row_end) ? __ldg(M + rg * RT + c + cl) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < C; ++q) zz[q] = (active && c + q < RT) ? zp[32 * (c + q)] : 0.0;
  };
  load_block(0, bf, mt, zv);
  for (int c0 = 0; c0 < R; c0 += C) {
    double bfn[NKS], mtn[C], zvn[C];
    if (c0 + C < R) load_block(c0 + C, bfn, mtn, zvn);
    // (1) out-of-block gradient of the warp's 32 rows on the tensor cores: all k-steps
    //     unrolled, the block's own k-steps (and those past R) with a zero B fragment (adding
    //     0 * a leaves an accumulator unchanged); even / odd k-steps in two sets of tiles
    double cacc[2][4][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int m = 0; m < 4; ++m) cacc[h][m][0] = cacc[h][m][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < NKS; ++kk) {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double a = Uw[8 * m * US + 4 * kk];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(cacc[kk & 1][m][0]), "+d"(cacc[kk & 1][m][1])
                     : "d"(a), "d"(bf[kk]));
      }
    }
    // (2) accumulators and the block's M tile to one row per thread
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      Tw[(8 * m + g) * TS + 2 * t] = cacc[0][m][0] + cacc[1][m][0];
      Tw[(8 * m + g) * TS + 2 * t + 1] = cacc[0][m][1] + cacc[1][m][1];
    }
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const int x = lane + 32 * k, rl = x / C, cl = x % C;
      Tw[rl * TS + C + cl] = mt[k];
    }
    __syncwarp();
    if (active) {
      double acc[C], mv[C], ub[C];
#pragma unroll
      for (int q = 0; q < C; ++q) {
        acc[q] = Tw[lane * TS + q];
        mv[q] = empty ? 0.0 : Tw[lane * TS + C + q];
        ub[q] = u[c0 + q];
      }
      const double *Hb = Hd + (c0 / C) * C * C;
      // (3) in-block Gauss-Seidel (C9), as k_sacd_rows
#pragma unroll
      for (int q = 0; q < C; ++q) {
        const int r = c0 + q;
        if (r < R) {
          const double h = Hb[q * C + q];
          double z = 0.0;
          bool sel = false;
          if (h != 0.0) {
            double sg = acc[q];
#pragma unroll
            for (int qq = 0; qq < C; ++qq) sg = fma(ub[qq], Hb[q * C + qq], sg);
            const double gr = sg - mv[q];                  // Eq 14
            const double ur = ub[q];
            const double un = fmax(0.0, ur - gr / h);      // Eq 11-13
            const double d = un - ur;                      // Eq 12
            const double L = l_mode ? Lf : h;
            z = -gr * d - (L * 0.5) * d * d;               // Eq 20
            const double zpr = zv[q];
            sel = (branch == SACD_BR_FIRST) ? (z > 0.0)
                                            : ((branch == SACD_BR_EQ24) ? (z - zpr > 0.0) : (zpr - z > 0.0));
            if (sel) {
              ub[q] = un;
              E += 1;
              if (d != 0.0) Ech += 1;
            }
          }
          zv[q] = z;                                       // z_prev <- z always (C8)
          ti += z;                                         // Eq 25
          md += ub[q] * mv[q];
          if (dec) dec[row * R + r] = (uint8_t)sel;
        }
      }
#pragma unroll
      for (int q = 0; q < C; ++q) u[c0 + q] = ub[q];
#pragma unroll
      for (int q = 0; q < C; ++q) zp[32 * (c0 + q)] = zv[q];
    }
    __syncwarp();  // the updated block columns feed the next block's fragments; Tw is reused
#pragma unroll
    for (int kk = 0; kk < NKS; ++kk) bf[kk] = bfn[kk];
#pragma unroll
    for (int q = 0; q < C; ++q) {
      mt[q] = mtn[q];
      zv[q] = zvn[q];
    }
  }
  __syncthreads();
  double *Fo = F + row0 * RT;
  for (int x = tid; x < nrows * RT; x += TR) Fo[x] = Us[(x / RT) * US + (x % RT)];

  // fixed-order block reduction of (ti, md, E, Ech)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ti += __shfl_xor_sync(0xffffffffu, ti, o);
    md += __shfl_xor_sync(0xffffffffu, md, o);
    E += __shfl_xor_sync(0xffffffffu, E, o);
    Ech += __shfl_xor_sync(0xffffffffu, Ech, o);
  }
  if (lane == 0) {
    red_d[0][wp] = ti;
    red_d[1][wp] = md;
    red_l[0][wp] = E;
    red_l[1][wp] = Ech;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    long long c = 0, d = 0;
    for (int k = 0; k < WPB; ++k) {
      a += red_d[0][k];
      b += red_d[1][k];
      c += red_l[0][k];
      d += red_l[1][k];
    }
    ti_part[blockIdx.x] = a;
    md_part[blockIdx.x] = b;
    e_part[blockIdx.x] = c;
    ech_part[blockIdx.x] = d;
  }
}

// The same row update for R > 64 (fp64): one warp (32 rows) per block; the B fragments of
// a column block (R/4 k-steps) are loaded 16 k-steps at a time, the next chunk in flight
// while the current one feeds the DMMAs; the in-block H values come from L1.  The FMA
// kernel this replaces waited on one L2 round trip of H per 4 gradient terms.
template <int RT>
__global__ void __launch_bounds__(32)
    k_sacd_rows_mma_big(long long row_begin, long long row_end, int R, int mode, int l_mode,
                        const long long *__restrict__ row_ptr, const double *__restrict__ M, double *__restrict__ F,
                        double *__restrict__ Z, const double *__restrict__ H, const DevState *__restrict__ st,
                        uint8_t *__restrict__ dec, double *__restrict__ ti_part, double *__restrict__ md_part,
                        long long *__restrict__ e_part, long long *__restrict__ ech_part) {
  constexpr int US = RT + 2;
  constexpr int C = 8;
  constexpr int TS = 2 * C + 2;
  constexpr int KC = 16;  // k-steps per B-fragment chunk
  static_assert(RT % (4 * KC) == 0, "R pitch must be a multiple of 64");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *Us = reinterpret_cast<double *>(smem_raw);
  double *Tw = Us + 32 * US;
  const int lane = threadIdx.x;
  const int g = lane >> 2, t = lane & 3;
  const long long row0 = row_begin + (long long)blockIdx.x * 32;
  const int nrows = (int)min(32LL, row_end - row0);
  const double *Fg = F + row0 * RT;
  static_assert(((RT + 2) * 8) % 16 == 0, "row stride must keep 16-byte chunks aligned");
  for (int x = lane; x < 32 * RT / 2; x += 32) {
    const int r = (2 * x) / RT, col = (2 * x) % RT;
    if (r < nrows) cp_async<16>(Us + r * US + col, Fg + 2 * x);
    else *reinterpret_cast<double2 *>(Us + r * US + col) = make_double2(0.0, 0.0);
  }
  cp_async_wait_all();
  __syncwarp();
  const int branch = st->branch[mode];
  const double Lf = st->Lfrob[mode];
  const int kmax = (R + 3) / 4;

  double ti = 0.0, md = 0.0;
  long long E = 0, Ech = 0;
  const bool active = lane < nrows;
  const long long row = row0 + lane;
  double *u = Us + lane * US;
  const bool empty = active ? row_ptr[row] == row_ptr[row + 1] : true;
  double *zp = Z + tt<RT>(active ? row : row0, 0);
  const double *Uw = Us + g * US + t;
  for (int c0 = 0; c0 < R; c0 += C) {
    const int kb = c0 / 4;
    double mt[C], zv[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const int x = lane + 32 * k, rl = x / C, cl = x % C;
      const long long rg = row0 + rl;
      mt[k] = (rg < row_end) ? __ldg(M + rg * RT + c0 + cl) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < C; ++q) zv[q] = active ? zp[32 * (c0 + q)] : 0.0;
    double cacc[2][4][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int m = 0; m < 4; ++m) cacc[h][m][0] = cacc[h][m][1] = 0.0;
    auto load_chunk = [&](int k0, double (&b)[KC]) {
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        const int kk = k0 + j;
        b[j] = (kk == kb || kk == kb + 1 || kk >= kmax) ? 0.0 : __ldg(H + (4 * kk + t) * RT + c0 + g);
      }
    };
    double bc[KC], bn[KC];
    load_chunk(0, bc);
    for (int k0 = 0; k0 < kmax; k0 += KC) {
      if (k0 + KC < kmax) load_chunk(k0 + KC, bn);
#pragma unroll
      for (int j = 0; j < KC; ++j) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const double a = Uw[8 * m * US + 4 * (k0 + j)];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(cacc[j & 1][m][0]), "+d"(cacc[j & 1][m][1])
                       : "d"(a), "d"(bc[j]));
        }
      }
#pragma unroll
      for (int j = 0; j < KC; ++j) bc[j] = bn[j];
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      Tw[(8 * m + g) * TS + 2 * t] = cacc[0][m][0] + cacc[1][m][0];
      Tw[(8 * m + g) * TS + 2 * t + 1] = cacc[0][m][1] + cacc[1][m][1];
    }
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const int x = lane + 32 * k, rl = x / C, cl = x % C;
      Tw[rl * TS + C + cl] = mt[k];
    }
    __syncwarp();
    if (active) {
      double acc[C], mv[C], ub[C];
#pragma unroll
      for (int q = 0; q < C; ++q) {
        acc[q] = Tw[lane * TS + q];
        mv[q] = empty ? 0.0 : Tw[lane * TS + C + q];
        ub[q] = u[c0 + q];
      }
#pragma unroll
      for (int q = 0; q < C; ++q) {
        const int r = c0 + q;
        if (r < R) {
          const double *Hr_ = H + (long long)r * RT + c0;
          const double h = __ldg(Hr_ + q);
          double z = 0.0;
          bool sel = false;
          if (h != 0.0) {
            double sg = acc[q];
#pragma unroll
            for (int qq = 0; qq < C; ++qq) sg = fma(ub[qq], __ldg(Hr_ + qq), sg);
            const double gr = sg - mv[q];                  // Eq 14
            const double ur = ub[q];
            const double un = fmax(0.0, ur - gr / h);      // Eq 11-13
            const double d = un - ur;                      // Eq 12
            const double L = l_mode ? Lf : h;
            z = -gr * d - (L * 0.5) * d * d;               // Eq 20
            const double zpr = zv[q];
            sel = (branch == SACD_BR_FIRST) ? (z > 0.0)
                                            : ((branch == SACD_BR_EQ24) ? (z - zpr > 0.0) : (zpr - z > 0.0));
            if (sel) {
              ub[q] = un;
              E += 1;
              if (d != 0.0) Ech += 1;
            }
          }
          zv[q] = z;
          ti += z;
          md += ub[q] * mv[q];
          if (dec) dec[row * R + r] = (uint8_t)sel;
        }
      }
#pragma unroll
      for (int q = 0; q < C; ++q) u[c0 + q] = ub[q];
#pragma unroll
      for (int q = 0; q < C; ++q) zp[32 * (c0 + q)] = zv[q];
    }
    __syncwarp();
  }
  double *Fo = F + row0 * RT;
  for (int x = lane; x < nrows * RT; x += 32) Fo[x] = Us[(x / RT) * US + (x % RT)];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ti += __shfl_xor_sync(0xffffffffu, ti, o);
    md += __shfl_xor_sync(0xffffffffu, md, o);
    E += __shfl_xor_sync(0xffffffffu, E, o);
    Ech += __shfl_xor_sync(0xffffffffu, Ech, o);
  }
  if (lane == 0) {
    ti_part[blockIdx.x] = ti;
    md_part[blockIdx.x] = md;
    e_part[blockIdx.x] = E;
    ech_part[blockIdx.x] = Ech;
  }
}

template <int RT>
__host__ __device__ constexpr size_t rows_mma_big_smem_bytes() {
  return (size_t)32 * (RT + 2) * 8 + (size_t)32 * 18 * 8;
}

template <int RT, int WPB>
__host__ __device__ constexpr size_t rows_mma_smem_bytes() {
  return (size_t)WPB * 32 * (RT + 2) * 8 + (size_t)WPB * 32 * 18 * 8 + (size_t)RT * 8 * 8;
}

// sum_r F_ir M_ir per row block (initial objective f^0)
template <typename Real, int RT>
__global__ void k_fm_dot(long long row_begin, long long row_end, int R, const long long *__restrict__ row_ptr,
                         const Real *__restrict__ F,
                         const Real *__restrict__ M,
                         double *__restrict__ ti_part, double *__restrict__ md_part, long long *__restrict__ e_part,
                         long long *__restrict__ ech_part) {
  constexpr int TR = rows_per_block<RT>();
  __shared__ double red[TR];
  const long long row = row_begin + (long long)blockIdx.x * TR + threadIdx.x;
  double s = 0.0;
  if (row < row_end && row_ptr[row] != row_ptr[row + 1])
    for (int r = 0; r < R; ++r) s += (double)F[row * RT + r] * (double)M[row * RT + r];
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int k = 0; k < TR; ++k) a += red[k];
    md_part[blockIdx.x] = a;
    ti_part[blockIdx.x] = 0.0;
    e_part[blockIdx.x] = 0;
    ech_part[blockIdx.x] = 0;
  }
}

// ------------------------------------------------------------------ Gram G = F^T F (fp64)
// Fixed grid: blockIdx.x = a contiguous row range, blockIdx.y = a pair (bi <= bj) of GT-wide
// column panels (one pair unless R > 128).  Each thread owns a T x T tile; inside a
// diagonal panel pair only tiles with ty <= tx work.  Partials are reduced in block order.
template <int RT>
__host__ __device__ constexpr int gram_gt() {
  return RT < 128 ? RT : 128;
}

template <typename Real, int RT>
__global__ void __launch_bounds__(gram_tg<gram_gt<RT>()>() * gram_tg<gram_gt<RT>()>())
    k_gram_partial(long long row_begin, long long row_end, int R, const Real *__restrict__ F,
                   double *__restrict__ part) {
  // Thread (ty, tx) of a TG x TG grid owns entries (bi*GT + ty + TG*a, bj*GT + tx + TG*b),
  // a, b < T: for a fixed staged row the warp reads TG consecutive values (conflict-free)
  // and a few broadcast ones.  A diagonal panel pair also computes its lower half
  // (redundant); the reduce reads the (min, max) entry.
  constexpr int GT = gram_gt<RT>();
  constexpr int TG = gram_tg<GT>();
  constexpr int T = GT / TG;
  constexpr int CH = GT >= 128 ? 16 : 32;
  __shared__ double Fa[CH][GT + 1];
  __shared__ double Fb[CH][GT + 1];
  constexpr int NB = RT / GT;
  int bi = 0, bj = 0;
  {
    int y = blockIdx.y;
    for (int a = 0; a < NB; ++a) {
      if (y < NB - a) {
        bi = a;
        bj = a + y;
        break;
      }
      y -= NB - a;
    }
  }
  const int tid = threadIdx.x;
  const int ty = tid / TG, tx = tid % TG;
  const long long per = (row_end - row_begin + gridDim.x - 1) / gridDim.x;
  const long long i0 = row_begin + (long long)blockIdx.x * per;
  const long long i1 = min(row_end, i0 + per);
  double acc[T][T];
#pragma unroll
  for (int a = 0; a < T; ++a)
#pragma unroll
    for (int b = 0; b < T; ++b) acc[a][b] = 0.0;
  for (long long c0 = i0; c0 < i1; c0 += CH) {
    const int nr = (int)min((long long)CH, i1 - c0);
    __syncthreads();
    for (int x = tid; x < nr * GT; x += TG * TG) {
      const int k = x / GT, col = x % GT;
      Fa[k][col] = (double)F[(c0 + k) * RT + bi * GT + col];
      Fb[k][col] = (double)F[(c0 + k) * RT + bj * GT + col];
    }
    __syncthreads();
    for (int k = 0; k < nr; ++k) {
      double av[T], bv[T];
#pragma unroll
      for (int a = 0; a < T; ++a) av[a] = Fa[k][ty + TG * a];
#pragma unroll
      for (int b = 0; b < T; ++b) bv[b] = Fb[k][tx + TG * b];
#pragma unroll
      for (int a = 0; a < T; ++a)
#pragma unroll
        for (int b = 0; b < T; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
  }
  double *p = part + (long long)blockIdx.x * R * R;
#pragma unroll
  for (int a = 0; a < T; ++a)
#pragma unroll
    for (int b = 0; b < T; ++b) {
      const int r = bi * GT + ty + TG * a, t = bj * GT + tx + TG * b;
      if (r < R && t < R) p[r * R + t] = acc[a][b];
    }
}

// fp64 Gram on the tensor cores (DMMA, mma.sync m8n8k4 f64): G = F^T F as a GEMM with
// M = N = RT (columns) and K = rows.  blockIdx.x = a contiguous row range (as
// k_gram_partial), blockIdx.y = an upper-triangle pair (qi <= qj) of 32-column panels; the
// 4 warps of a block take 4 contiguous sub-ranges of the rows (multiples of 4), each lane
// holding a 32 x 32 quadrant as 4 x 4 m8n8 tiles, and the warps' quadrants are summed in
// warp order through shared memory.  Fragments (PTX m8n8k4 .f64): A[m][k] = F[i0+k][r0+m]
// is held by lane (g = lane >> 2, t = lane & 3) as F[i0+t][r0+g]; B[k][n] = F[i0+k][c0+n]
// as F[i0+t][c0+g]; C[g][2t + {0,1}].  Same partial contract as k_gram_partial (entries
// r <= t of every panel pair are written; the reduce reads those).
template <int RT>
__global__ void __launch_bounds__(128) k_gram_dmma(long long row_begin, long long row_end, int R,
                                                   const double *__restrict__ F, double *__restrict__ part) {
  constexpr int NP = RT / 32;
  int qi = 0, qj = 0;
  {
    int y = blockIdx.y;
    for (int a = 0; a < NP; ++a) {
      if (y < NP - a) {
        qi = a;
        qj = a + y;
        break;
      }
      y -= NP - a;
    }
  }
  __shared__ double red[3][32 * 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const long long per = (row_end - row_begin + gridDim.x - 1) / gridDim.x;
  const long long b0 = row_begin + (long long)blockIdx.x * per;
  const long long b1 = min(row_end, b0 + per);
  const long long wper = ((b1 - b0 + 3) / 4 + 3) / 4 * 4;  // rows per warp, multiple of 4
  const long long i0 = min(b1, b0 + w * wper), i1 = min(b1, i0 + wper);
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const double *Fa = F + qi * 32 + g;
  const double *Fb = F + qj * 32 + g;
  for (long long r0 = i0; r0 < i1; r0 += 8) {
    double av[2][4], bv[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long row = r0 + 4 * h + t;
      const bool ok = row < i1;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        av[h][m] = ok ? __ldg(Fa + row * RT + 8 * m) : 0.0;
        bv[h][m] = ok ? __ldg(Fb + row * RT + 8 * m) : 0.0;
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                       : "d"(av[h][a]), "d"(bv[h][b]));
  }
  // fixed-order sum of the 4 warps' quadrants
  if (w > 0) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) red[w - 1][(8 * a + g) * 32 + 8 * b + 2 * t + e] = acc[a][b][e];
  }
  __syncthreads();
  if (w == 0) {
    double *p = part + (long long)blockIdx.x * R * R;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int x = (8 * a + g) * 32 + 8 * b + 2 * t + e;
          const double v = ((acc[a][b][e] + red[0][x]) + red[1][x]) + red[2][x];
          const int r = qi * 32 + 8 * a + g, c = qj * 32 + 8 * b + 2 * t + e;
          if (r < R && c < R && (qi < qj || r <= c)) p[r * R + c] = v;
        }
  }
}

// G[r][t] = sum over blocks (in order) of the upper-triangle partial; mirrored exactly.
__global__ void k_gram_reduce(int R, int nblk, const double *__restrict__ part, double *__restrict__ G) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= R * R) return;
  const int r = x / R, t = x % R;
  const int src = (r <= t) ? (r * R + t) : (t * R + r);
  // (an entry with r <= t lies in panel pair (r/GT, t/GT) with bi <= bj, which wrote it)
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += part[(long long)b * R * R + src];
  G[x] = s;
}

// ------------------------------------------------------------------ finalize a mode pass
// flags: 1 = record the pass (ti/E/history), 2 = compute f (needs all three Grams),
//        4 = push a stats-ring record (end of sweep)
// Record a finished pass in the device state (thread 0 only).
// flags: 1 = record the pass (ti/E/history), 2 = compute f, 4 = push a stats-ring record.
__device__ void apply_pass(DevState *st, int mode, double ti, double md, long long E, long long Ech, double mn,
                           int flags) {
  if (flags & 1) {
    st->ti_cur[mode] = ti;
    st->E[mode] = E;
    st->Ech[mode] = Ech;
    st->ti2[mode] = st->ti1[mode];
    st->ti1[mode] = ti;
    st->nhist[mode] += 1;
  }
  if (mode == 2) st->mdot = md;
  if (flags & 2) {
    const double f = st->xnorm2 - 2.0 * md + mn;
    st->f = f;
    st->fit = st->xnorm2 > 0.0 ? 1.0 - sqrt(f > 0.0 ? f : 0.0) / sqrt(st->xnorm2) : 0.0;
  }
  if (flags & 4) {
    sacd_iter_stats &rec = st->ring[st->ring_count % kRing];
    rec.k = st->k;
    rec.objective = st->f;
    rec.fit = st->fit;
    for (int n = 0; n < 3; ++n) {
      rec.branch[n] = st->branch[n];
      rec.ti[n] = st->ti_cur[n];
      rec.E[n] = st->E[n];
      rec.E_changed[n] = st->Ech[n];
    }
    st->ring_count += 1;
  }
}

// Fixed-order reduction of the per-block partials of a pass.  flags as apply_pass, plus
// 8 = local: write (ti, md, E, Ech) to local_out[0..3] and leave the state alone (sharded).
__global__ void __launch_bounds__(1024) k_finalize(int mode, long long nblk, const double *__restrict__ ti_part,
                                                   const double *__restrict__ md_part,
                                                   const long long *__restrict__ e_part,
                                                   const long long *__restrict__ ech_part, const double *G0,
                                                   const double *G1, const double *G2, int R, DevState *st,
                                                   int flags, double *local_out) {
  __shared__ double sd[3][1024];
  __shared__ long long sl[2][1024];
  const int tid = threadIdx.x;
  double ti = 0.0, md = 0.0, mn = 0.0;
  long long E = 0, Ech = 0;
  for (long long b = tid; b < nblk; b += 1024) {
    ti += ti_part[b];
    md += md_part[b];
    E += e_part[b];
    Ech += ech_part[b];
  }
  if ((flags & 2) && !(flags & 8))
    for (int x = tid; x < R * R; x += 1024) mn += G0[x] * G1[x] * G2[x];
  sd[0][tid] = ti;
  sd[1][tid] = md;
  sd[2][tid] = mn;
  sl[0][tid] = E;
  sl[1][tid] = Ech;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (tid < o) {
      sd[0][tid] += sd[0][tid + o];
      sd[1][tid] += sd[1][tid + o];
      sd[2][tid] += sd[2][tid + o];
      sl[0][tid] += sl[0][tid + o];
      sl[1][tid] += sl[1][tid + o];
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (flags & 8) {
      local_out[0] = sd[0][0];
      local_out[1] = sd[1][0];
      local_out[2] = (double)sl[0][0];
      local_out[3] = (double)sl[1][0];
    } else {
      apply_pass(st, mode, sd[0][0], sd[1][0], sl[0][0], sl[1][0], sd[2][0], flags);
    }
  }
}

// ------------------------------------------------------------------ delta exchange
// Changed elements of F over [lo, hi) (element indices of the padded row-major factor),
// compared bit for bit against Fold (so a +0 / -0 flip is sent too and every replica stays
// bitwise identical).  Two passes over a fixed grid of kDeltaBlocks contiguous chunks: count,
// then write in index order (warp ballots + block prefix), so the lists are deterministic.
template <typename Real>
__device__ __forceinline__ bool elem_changed(const Real *F, const Real *Fo, long long i) {
  if constexpr (sizeof(Real) == 8)
    return __double_as_longlong(F[i]) != __double_as_longlong(Fo[i]);
  else
    return __float_as_uint(F[i]) != __float_as_uint(Fo[i]);
}

template <typename Real>
__global__ void __launch_bounds__(256) k_delta_count(long long lo, long long hi, const Real *__restrict__ F,
                                                     const Real *__restrict__ Fo, int *__restrict__ blk) {
  __shared__ int red[8];
  const long long per = (hi - lo + gridDim.x - 1) / gridDim.x;
  const long long b0 = lo + (long long)blockIdx.x * per, b1 = min(hi, b0 + per);
  int n = 0;
  for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) n += elem_changed(F, Fo, i);
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    blk[blockIdx.x] = t;
  }
}

template <typename Real>
__global__ void __launch_bounds__(256) k_delta_write(long long lo, long long hi, const Real *__restrict__ F,
                                                     const Real *__restrict__ Fo, const int *__restrict__ blk,
                                                     uint32_t *__restrict__ idx, Real *__restrict__ val,
                                                     long long *__restrict__ count) {
  __shared__ int wcnt[8];
  __shared__ long long base_s;
  const long long per = (hi - lo + gridDim.x - 1) / gridDim.x;
  const long long b0 = lo + (long long)blockIdx.x * per, b1 = min(hi, b0 + per);
  if (threadIdx.x == 0) {
    long long b = 0;
    for (int k = 0; k < (int)blockIdx.x; ++k) b += blk[k];
    base_s = b;
    if (blockIdx.x == gridDim.x - 1) *count = b + blk[blockIdx.x];
  }
  __syncthreads();
  long long base = base_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (long long t0 = b0; t0 < b1; t0 += blockDim.x) {
    const long long i = t0 + threadIdx.x;
    const bool ch = i < b1 && elem_changed(F, Fo, i);
    const unsigned bal = __ballot_sync(0xffffffffu, ch);
    if (lane == 0) wcnt[w] = __popc(bal);
    __syncthreads();
    int before = 0, tot = 0;
    for (int k = 0; k < 8; ++k) {
      before += k < w ? wcnt[k] : 0;
      tot += wcnt[k];
    }
    if (ch) {
      const long long o = base + before + __popc(bal & ((1u << lane) - 1u));
      idx[o] = (uint32_t)i;
      val[o] = F[i];
    }
    base += tot;
    __syncthreads();
  }
}

template <typename Real>
__global__ void k_delta_apply(const uint32_t *__restrict__ idx, const Real *__restrict__ val,
                              const long long *__restrict__ count, Real *__restrict__ F) {
  const long long n = *count;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    F[idx[k]] = val[k];
}

// Snapshot variant (reading C10'): ti^k = fixed-order sum of the score pass's block partials
// (the same tree as k_finalize, so the recorded ti equals it bitwise); the branch of THIS
// pass: k == 1 (no history) the z > 0 rule, else Eq 27 iff ti^k > ti^{k-1}.
__global__ void __launch_bounds__(1024) k_snapshot_branch(int mode, long long nblk, const double *__restrict__ ti_part,
                                                          DevState *st, int branch_override) {
  __shared__ double sd[1024];
  const int tid = threadIdx.x;
  double ti = 0.0;
  for (long long b = tid; b < nblk; b += 1024) ti += ti_part[b];
  sd[tid] = ti;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (tid < o) sd[tid] += sd[tid + o];
    __syncthreads();
  }
  if (tid == 0) {
    int br;
    if (branch_override >= 0) br = branch_override;
    else if (st->nhist[mode] == 0) br = SACD_BR_FIRST;
    else br = (sd[0] > st->ti1[mode]) ? SACD_BR_EQ27 : SACD_BR_EQ24;
    st->branch[mode] = br;
  }
}

// ------------------------------------------------------------------ sharded-engine kernels
// Every rank q writes its head row id / partial row into slot q of the exchange buffers
// and its (ti, md, E, Ech, Gram partial) into slot q of the stats buffer; NCCL all-gathers
// them in place (or, with emulated ranks on one GPU, they are already all local).
template <typename Real, int RT>
__global__ void k_pack_head(long long head, const Real *__restrict__ M, long long *__restrict__ id_slot,
                            Real *__restrict__ row_slot) {
  for (int c = threadIdx.x; c < RT; c += blockDim.x) row_slot[c] = head >= 0 ? M[head * RT + c] : Real(0);
  if (threadIdx.x == 0) *id_slot = head;
}

template <typename Real, int RT>
__global__ void k_copy_rows_tt(long long rlo, long long rhi, const Real *__restrict__ src, Real *__restrict__ dst) {
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < (rhi - rlo) * RT;
       x += (long long)gridDim.x * blockDim.x) {
    const long long i = rlo + x / RT;
    const int c = (int)(x % RT);
    dst[i * RT + c] = src[i * RT + c];
  }
}

// The owner adds the head partials of the other ranks to its rows, in rank order.
template <typename Real, int RT>
__global__ void k_merge_heads(int G, long long rlo, long long rhi, const long long *__restrict__ ids,
                              const Real *__restrict__ rows, Real *__restrict__ M) {
  for (int q = 0; q < G; ++q) {
    const long long id = ids[q];
    if (id >= rlo && id < rhi)
      for (int c = threadIdx.x; c < RT; c += blockDim.x) M[id * RT + c] += rows[(long long)q * RT + c];
  }
}

// Sum the G ranks' slots in rank order: Gram (if flags & 32) and (ti, md, E, Ech); then
// apply the pass to the device state.  stats slot layout: [ti, md, E, Ech, Gram R x R].
__global__ void __launch_bounds__(1024) k_finalize_global(int mode, int G, int R, const double *__restrict__ stats,
                                                          double *Gout, const double *G0, const double *G1,
                                                          const double *G2, DevState *st, int flags) {
  __shared__ double red[1024];
  const int tid = threadIdx.x;
  const long long slot = 4 + (long long)R * R;
  if (flags & 32) {
    for (int x = tid; x < R * R; x += 1024) {
      double s = 0.0;
      for (int q = 0; q < G; ++q) s += stats[q * slot + 4 + x];
      Gout[x] = s;
    }
    __syncthreads();
  }
  double mn = 0.0;
  if (flags & 2)
    for (int x = tid; x < R * R; x += 1024) mn += G0[x] * G1[x] * G2[x];
  red[tid] = mn;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  if (tid == 0) {
    double ti = 0.0, md = 0.0, E = 0.0, Ech = 0.0;
    for (int q = 0; q < G; ++q) {
      ti += stats[q * slot + 0];
      md += stats[q * slot + 1];
      E += stats[q * slot + 2];
      Ech += stats[q * slot + 3];
    }
    apply_pass(st, mode, ti, md, (long long)E, (long long)Ech, red[0], flags & 7);
  }
}

// host-order fp64 (rows x R) <-> device Real (row-major with pitch RT, or TT tiles)
__device__ __forceinline__ long long dev_index(long long i, int r, int RT, bool ttl) {
  return ttl ? (i >> 5) * (32LL * RT) + (long long)r * 32 + (i & 31) : i * RT + r;
}

template <typename Real>
__global__ void k_convert_in(const double *__restrict__ src, long long rows, int R, int RT, Real *__restrict__ dst,
                             bool ttl) {
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < rows * RT;
       x += (long long)gridDim.x * blockDim.x) {
    const long long i = x / RT;
    const int r = (int)(x - i * RT);
    dst[dev_index(i, r, RT, ttl)] = r < R ? (Real)src[i * R + r] : Real(0);
  }
}

template <typename Real>
__global__ void k_convert_out(const Real *__restrict__ src, long long rows, int R, int RT, double *__restrict__ dst,
                              bool ttl) {
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < rows * R;
       x += (long long)gridDim.x * blockDim.x) {
    const long long i = x / R;
    const int r = (int)(x - i * R);
    dst[x] = (double)src[dev_index(i, r, RT, ttl)];
  }
}


// ------------------------------------------------------------------ held-out evaluation
// Eq 8 at test coordinates: one warp per entry, lane l multiplies columns
// l, l+32, ... and the warp sums them by a fixed xor tree.  With vals != nullptr also the
// squared error (Eq 30), reduced per block in a fixed order into part[block].
template <typename Real, int RT>
__global__ void __launch_bounds__(256) k_predict(const uint32_t *__restrict__ coords, long long n,
                                                 const Real *__restrict__ U, const Real *__restrict__ V,
                                                 const Real *__restrict__ W, const float *__restrict__ vals,
                                                 double *__restrict__ out, double *__restrict__ part) {
  constexpr int CPL = RT >= 32 ? RT / 32 : 1;
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const long long e = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double se = 0.0;
  if (e < n) {
    const long long q = coords[3 * e], p = coords[3 * e + 1], s = coords[3 * e + 2];
    double xh = 0.0;
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int c = lane + 32 * k;
      if (c < RT) xh += (double)U[q * RT + c] * (double)V[p * RT + c] * (double)W[s * RT + c];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xh += __shfl_xor_sync(0xffffffffu, xh, o);
    if (lane == 0) {
      if (out) out[e] = xh;
      if (vals) {
        const double d = (double)vals[e] - xh;
        se = d * d;
      }
    }
  }
  if (part) {
    if (lane == 0) red[wp] = se;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int k = 0; k < 8; ++k) t += red[k];
      part[blockIdx.x] = t;
    }
  }
}

__global__ void k_range_check(const uint32_t *__restrict__ coords, long long n, long long d0, long long d1,
                              long long d2, int *__restrict__ flag) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    if (coords[3 * e] >= d0 || coords[3 * e + 1] >= d1 || coords[3 * e + 2] >= d2) atomicOr(flag, 1);
}

// fixed-order sum of the block partials (one block)
__global__ void __launch_bounds__(1024) k_sum_parts(const double *__restrict__ part, long long nb,
                                                    double *__restrict__ out) {
  __shared__ double sd[1024];
  double t = 0.0;
  for (long long b = threadIdx.x; b < nb; b += 1024) t += part[b];
  sd[threadIdx.x] = t;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) sd[threadIdx.x] += sd[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sd[0];
}

// ------------------------------------------------------------------ launch implementations
template <typename Real, int RT>
struct Impl {
  static int mttkrp(Context &c, int mode, void *out_v) {
    ModeData &md = c.m[mode];
    return mttkrp_on(c, mode, md.items, md.n_items, md.splits, md.n_splits, md.chunks, md.n_chunks,
                     reinterpret_cast<Real *>(out_v),
                     reinterpret_cast<Real *>(c.partial));
  }

  static int mttkrp_on(Context &c, int mode, const WorkItem *items, long long n_items, const SplitRow *splits,
                       long long n_splits, const FixChunk *chunks, long long n_chunks, Real *out, Real *partial) {
    ModeData &md = c.m[mode];
    const Real *A = reinterpret_cast<const Real *>(c.m[md.a].F);
    const Real *B = reinterpret_cast<const Real *>(c.m[md.b].F);
    int pe = prof_begin(c, 0);
    if (n_items > 0) {
      const int wpb = 8;
      const long long blocks = (n_items + wpb - 1) / wpb;
      if constexpr (RT >= 32) {
        // (NB gathers in flight per warp, min blocks per SM); opt.mttkrp_variant selects a
        // tuning variant (0 = default, measured on B200 with tools/mttkrp_tune.py:
        // occupancy beats deeper per-warp batching).
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
        if (var == 1) go(k_mttkrp_fiber<Real, RT, 1, fiber_min_blocks<Real, RT>()>);
        else if (var == 10) gos(k_mttkrp_sw<Real, RT, SW, 1, 4>);
        else if (var == 11) gos(k_mttkrp_sw<Real, RT, SW, 2, 4>);
        else if (var == 12) gos(k_mttkrp_sw<Real, RT, SW, 4, 4>);
        else if (var == 13) gos(k_mttkrp_sw<Real, RT, SW, 4, 3>);
        else if (var == 14) gos(k_mttkrp_sw<Real, RT, SW, 8, 2>);
        else if (var == 15) gos(k_mttkrp_sw<Real, RT, SW, 2, 6>);
        else if (var >= 20 && var < 50) {
          // lean kernel: E elements per lane -> SW = RT / E lanes per worker
          constexpr int VEC = V16<Real>::N;
          constexpr int E8 = 8 < VEC ? VEC : 8;
          constexpr int SW8 = RT / E8 > 32 ? 32 : (RT / E8 < 1 ? 1 : RT / E8);
          constexpr int E4 = 4 < VEC ? VEC : 4;
          constexpr int SW4 = RT / E4 > 32 ? 32 : (RT / E4 < 1 ? 1 : RT / E4);
          auto gol = [&](auto kern, int sw) {
            const long long lb = (n_items * sw + 255) / 256;
            kern<<<(unsigned)lb, 256, 0, c.stream>>>(items, n_items, md.nzm, A, B, out, partial);
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
          else if (var == 40) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 1, 6>, sub_warp_lanes<Real, RT>());
          else if (var == 41) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 1, 5>, sub_warp_lanes<Real, RT>());
          else if (var == 42) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 2, 5>, sub_warp_lanes<Real, RT>());
          else if (var == 43) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 2, 4>, sub_warp_lanes<Real, RT>());
          else if (var == 44) gol(k_mttkrp_lean<Real, RT, sub_warp_lanes<Real, RT>(), 1, 8>, sub_warp_lanes<Real, RT>());
          else gol(k_mttkrp_lean<Real, RT, SW8, 2, 2>, SW8);
        }
        else if (sizeof(Real) == 8 && RT >= 256) {
          // fp64, R > 128: one warp per item, 8 fp64 columns per lane, x broadcast through
          // shared memory (variant 36; c5 R=256: 12.7 ms per sweep vs 13.7 with shuffles,
          // variant 22, and 28.6 for the warp fiber kernel, variant 1)
          constexpr int SWW = RT / 8 > 32 ? 32 : RT / 8;
          const long long lb = (n_items * SWW + 255) / 256;
          k_mttkrp_lean<Real, RT, SWW, 1, 2, 0, 1><<<(unsigned)lb, 256, 0, c.stream>>>(items, n_items, md.nzm, A, B,
                                                                                      out, partial);
        } else if (sizeof(Real) == 8 && (RT == 64 || (RT == 32 && md.n_fibers > 0 && c.nnz >= 2 * md.n_fibers))) {
          // fp64, R = 33..64 (and R = 17..32 with a mean fiber length >= 2, the Zipf config
          // c3): one warp per item (2 fp64 columns per lane at R = 64) at 48 registers / 40
          // warps per SM (variant 41: c4 13.65 vs 15.17 ms per sweep, c3 1.22 vs 1.28).  x
          // reaches the lanes through a shared-memory broadcast (XS = 1: one L1 wavefront
          // instead of two shuffles on the L1-data-path-bound kernel; variant 30: c4 12.11 vs
          // 13.66 ms, c5 R=64 4.02 vs 4.42); with two workers per warp (R = 32) the b index
          // and x go as one 16-byte broadcast (XS = 2; variant 31: c3 1.195 vs 1.227 ms).
          if constexpr (sizeof(Real) == 8 && (RT == 64 || RT == 32)) {
            constexpr int SWF = sub_warp_lanes<Real, RT>();
            const long long lb = (n_items * SWF + 255) / 256;
            // R = 64: 40 registers / 48 warps per SM (variant 35: c4 11.75 vs 12.11 ms, c5 R=64
            // 3.82 vs 4.02; small spills at the batch boundary)
            k_mttkrp_lean<Real, RT, SWF, 1, SWF == 32 ? 6 : 5, 0, SWF == 32 ? 1 : 2><<<(unsigned)lb, 256, 0, c.stream>>>(
                items, n_items, md.nzm, A, B, out, partial);
          }
        } else if (sizeof(Real) == 8 && RT == 128) {
          // fp64, R = 65..128: 4 columns per lane, one warp per item, x broadcast through shared
          // memory (variant 32: c5 R=128 6.54 vs 6.95 ms, c4 R=128 21.5 vs 26.0 ms per sweep)
          if constexpr (sizeof(Real) == 8 && RT == 128) {
            const long long lb = (n_items * 32 + 255) / 256;
            k_mttkrp_lean<Real, RT, 32, 1, 3, 0, 1><<<(unsigned)lb, 256, 0, c.stream>>>(items, n_items, md.nzm, A,
                                                                                       B, out, partial);
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
  fixup:
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
  // Each rank computes the MTTKRP of its nonzero range; the head partials (rows whose
  // first nonzero is on a lower rank) are exchanged and added by the owners in rank order.
  static int sharded_mttkrp_merge(Context &c, int mode) {
    for (Shard &sh : c.shards)
      SACD_TRY(mttkrp_on(c, mode, sh.items[mode], sh.n_items[mode], sh.splits[mode], sh.n_splits[mode],
                         sh.chunks[mode], sh.n_chunks[mode],
                         reinterpret_cast<Real *>(sh.M), reinterpret_cast<Real *>(sh.partial)));
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
    SACD_TRY(sharded_mttkrp_merge(c, mode));
    SACD_TRY(prepare(c, mode, branch_override, begin_sweep, 1));
    if (c.delta) SACD_TRY(delta_snapshot(c, mode));
    const long long TR = rows_tr(c, 0);
    constexpr int GT = gram_gt<RT>();
    constexpr int TG = gram_tg<GT>();
    constexpr int NBP = RT / GT;
    const long long slot = 4 + (long long)c.R * c.R;
    for (Shard &sh : c.shards) {
      const long long rlo = sh.plan[mode].rlo, rhi = sh.plan[mode].rhi;
      const long long nblk = (rhi - rlo + TR - 1) / TR;
      double *ti_part = sh.row_part, *md_part = sh.row_part + c.max_row_blocks;
      long long *e_part = sh.cnt_part, *ech_part = sh.cnt_part + c.max_row_blocks;
      int pe = prof_begin(c, 3);
      if (nblk > 0)
        SACD_TRY(rows(c, nblk, rlo, rhi, mode, reinterpret_cast<const Real *>(sh.M), dec, ti_part, md_part, e_part,
                      ech_part));
      SACD_CUDA_TRY(cudaGetLastError());
      SACD_TRY(prof_end(c, 3, pe));
      pe = prof_begin(c, 4);
      double *sl = c.xstats + sh.rank * slot;
      gram_partial(c, rlo, rhi, reinterpret_cast<const Real *>(md.F), sh.gram_part);
      k_gram_reduce<<<(c.R * c.R + 255) / 256, 256, 0, c.stream>>>(c.R, c.gram_blocks, sh.gram_part, sl + 4);
      SACD_CUDA_TRY(cudaGetLastError());
      SACD_TRY(prof_end(c, 4, pe));
      k_finalize<<<1, 1024, 0, c.stream>>>(mode, nblk, ti_part, md_part, e_part, ech_part, nullptr, nullptr,
                                           nullptr, c.R, c.st, 8, sl);
      SACD_CUDA_TRY(cudaGetLastError());
    }
    if (c.comm) SACD_TRY(nccl_allgather_inplace(c, c.xstats, (size_t)slot, 0));
    int pe = prof_begin(c, 5);
    k_finalize_global<<<1, 1024, 0, c.stream>>>(mode, c.G, c.R, c.xstats, md.G, c.m[0].G, c.m[1].G, c.m[2].G, c.st,
                                                32 | 1 | (end_sweep ? 6 : 0));
    SACD_CUDA_TRY(cudaGetLastError());
    SACD_TRY(prof_end(c, 5, pe));
    if (c.delta) SACD_TRY(delta_exchange(c, mode));
    else if (c.comm) SACD_TRY(nccl_broadcast_rows(c, mode));
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
      k_finalize<<<1, 1024, 0, c.stream>>>(2, nblk, ti_part, md_part, e_part, ech_part, nullptr, nullptr, nullptr,
                                           c.R, c.st, 8, c.xstats + sh.rank * slot);
    }
    SACD_CUDA_TRY(cudaGetLastError());
    if (c.comm) SACD_TRY(nccl_allgather_inplace(c, c.xstats, (size_t)slot, 0));
    k_finalize_global<<<1, 1024, 0, c.stream>>>(2, c.G, c.R, c.xstats, nullptr, c.m[0].G, c.m[1].G, c.m[2].G, c.st,
                                                2);
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
  static void gram_partial(Context &c, long long rlo, long long rhi, const Real *F, double *part) {
    if constexpr (sizeof(Real) == 8 && RT >= 32) {
      if (c.opt.reserved[2] != 1) {
        constexpr int NP = RT / 32;
        k_gram_dmma<RT><<<dim3(c.gram_blocks, NP * (NP + 1) / 2), 128, 0, c.stream>>>(
            rlo, rhi, c.R, reinterpret_cast<const double *>(F), part);
        return;
      }
    }
    constexpr int GT = gram_gt<RT>();
    constexpr int TG = gram_tg<GT>();
    constexpr int NB = RT / GT;
    k_gram_partial<Real, RT><<<dim3(c.gram_blocks, NB * (NB + 1) / 2), TG * TG, 0, c.stream>>>(rlo, rhi, c.R, F,
                                                                                              part);
  }

  static int gram(Context &c, int mode) {
    ModeData &md = c.m[mode];
    int pe = prof_begin(c, 4);
    gram_partial(c, 0, md.I, reinterpret_cast<const Real *>(md.F), c.gram_part);
    k_gram_reduce<<<(c.R * c.R + 255) / 256, 256, 0, c.stream>>>(c.R, c.gram_blocks, c.gram_part, md.G);
    SACD_CUDA_TRY(cudaGetLastError());
    SACD_TRY(chunk_mask(c, mode));
    return prof_end(c, 4, pe);
  }

  // chunk support masks of F_mode (used by the skipping MTTKRP of the other modes)
  static int chunk_mask(Context &c, int mode) {
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
    SACD_TRY(mttkrp(c, mode, M));
    SACD_TRY(prepare(c, mode, branch_override, begin_sweep, 1));
    const int vflags0 = c.opt.variant == SACD_VARIANT_SNAPSHOT ? 2 : (c.opt.variant == SACD_VARIANT_JACOBI ? 1 : 0);
    const long long TR = rows_tr(c, vflags0);
    const long long nblk = (md.I + TR - 1) / TR;
    double *ti_part = c.row_part, *md_part = c.row_part + c.max_row_blocks;
    long long *e_part = c.cnt_part, *ech_part = c.cnt_part + c.max_row_blocks;
    int pe = prof_begin(c, 3);
    if (c.opt.variant == SACD_VARIANT_SNAPSHOT) {
      // (1) snapshot scores from the rows at pass start, (2) ti^k and this pass's branch,
      // (3) the Gauss-Seidel pass gated by the snapshot (reading C10')
      SACD_TRY(rows(c, nblk, 0, md.I, mode, M, nullptr, ti_part, md_part, e_part, ech_part, 1 | 2));
      k_snapshot_branch<<<1, 1024, 0, c.stream>>>(mode, nblk, ti_part, c.st, branch_override);
      SACD_TRY(rows(c, nblk, 0, md.I, mode, M, dec, ti_part, md_part, e_part, ech_part, 4));
    } else {
      SACD_TRY(rows(c, nblk, 0, md.I, mode, M, dec, ti_part, md_part, e_part, ech_part,
                    c.opt.variant == SACD_VARIANT_JACOBI ? 1 : 0));
    }
    SACD_CUDA_TRY(cudaGetLastError());
    SACD_TRY(prof_end(c, 3, pe));
    SACD_TRY(gram(c, mode));
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
  static constexpr int kMmaWarps = 4;  // 5 (160 rows, 2 blocks per SM) measured 2.41 vs 1.72 ms: L1 too small
  static int rows_tr(const Context &c, int vflags) {
    if constexpr (kRowsMma) {
      if (c.opt.reserved[0] == 0 && vflags == 0) return kMmaWarps * 32;
    }
    if constexpr (kRowsMmaBig) {
      if (c.opt.reserved[0] == 0 && vflags == 0) return 32;
    }
    return rows_per_block<RT>();
  }

  static int rows(Context &c, long long nblk, long long rlo, long long rhi, int mode, const Real *M, uint8_t *dec,
                  double *ti_part, double *md_part, long long *e_part, long long *ech_part, int vflags = 0) {
    constexpr int TR = rows_per_block<RT>();
    ModeData &md = c.m[mode];
    auto go = [&](auto kern, size_t smem) {
      if (nblk > 0)
        kern<<<(unsigned)nblk, TR, smem, c.stream>>>(rlo, rhi, c.R, mode, c.opt.l_mode, md.row_ptr, M,
                                                      reinterpret_cast<Real *>(md.F), reinterpret_cast<Real *>(md.Z),
                                                      reinterpret_cast<const Real *>(c.Hr), c.st, dec, ti_part,
                                                      md_part, e_part, ech_part, vflags,
                                                      reinterpret_cast<Real *>(c.Zs));
    };
    if constexpr (kRowsMma) {
      if (c.opt.reserved[0] == 0 && vflags == 0) {  // default for fp64, R <= 64: out-of-block gradient on DMMA
        if (nblk > 0)
          k_sacd_rows_mma<RT, kMmaWarps><<<(unsigned)nblk, kMmaWarps * 32, rows_mma_smem_bytes<RT, kMmaWarps>(),
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
    if constexpr (kRowsMma)
      SACD_CUDA_TRY(cudaFuncSetAttribute(k_sacd_rows_mma<RT, kMmaWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)rows_mma_smem_bytes<RT, kMmaWarps>()));
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
