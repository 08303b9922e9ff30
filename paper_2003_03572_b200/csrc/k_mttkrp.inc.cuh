// k_mttkrp.inc.cuh -- part of kernels.cu (included inside namespace sacd { namespace { ... } }).
// Sparse MTTKRP kernels (A3): the R <= 16 grouped kernel, the lean record-driven
// fiber-factored kernels and their measured tuning variants, the split-row fix-ups.
// Paper citations "P:n" are PAPER.md lines; readings Cn / L1 / C10' are DESIGN.md section 3.
// NOT a standalone header: it relies on the helpers defined at the top of kernels.cu.

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
  SACD_DBG(SACD_DASSERT(it.nz0 < it.nz1 && it.nz1 <= g_dbg.nnz && it.slot < g_dbg.nslots && it.row0 < it.row1 &&
                        it.row1 <= g_dbg.In));
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
      const uint32_t ea = ld_stream_u32(ia + e) & kIdxMask, eb = ld_stream_u32(ib + e) & kIdxMask;
      SACD_DBG(SACD_DASSERT(ea < g_dbg.Ia && eb < g_dbg.Ib));
      const VT *ap = reinterpret_cast<const VT *>(A + (long long)ea * RT);
      const VT *bp = reinterpret_cast<const VT *>(B + (long long)eb * RT);
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
  // the same load with an L1 policy: H = 1 no L1 allocation, 2 L1 evict_first, 3 L1 evict_last
  template <int H>
  __device__ __forceinline__ void load_hint(const Real *p) {
    if constexpr (H == 0) {
      load(p);
    } else {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        uint4 r;
        const void *q = reinterpret_cast<const VT *>(p) + k * SW;
        if constexpr (H == 1)
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(q));
        else if constexpr (H == 2)
          asm volatile("ld.global.nc.L1::evict_first.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(q));
        else
          asm volatile("ld.global.nc.L1::evict_last.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(q));
        VT t;
        static_assert(sizeof(VT) == 16, "16-byte chunks");
        memcpy(&t, &r, 16);
        VV::get(t, v + k * VV::N);
      }
    }
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
// shared-memory broadcast per nonzero, 3 = as 2 with the workers' slots padded apart (two
// workers of a warp read different banks: one wavefront serves both), 4 = every value of the
// tensor equals xu (e.g. binary tensors; detected at sacd_init): no x broadcast at all, x =
// xu for the batch's nonzeros and 0 past the item's end.
template <int XS>
__device__ __forceinline__ int xs_slot(int t) {
  return XS == 3 ? t + (t >> 4) : t;
}

template <typename Real, int RT, int SW, int D, int PFX, int XS>
__device__ __forceinline__ void lean_item(long long item, const WorkItem *__restrict__ items,
                                          const uint4 *__restrict__ nzm, const Real *__restrict__ A,
                                          const Real *__restrict__ B, Real *__restrict__ M,
                                          Real *__restrict__ partial, Real xu) {
  using SR = SubRow<Real, RT, SW>;
  constexpr int E = SR::E;
  constexpr int VEC = V16<Real>::N;
  static_assert(SR::NV >= 1, "row narrower than a sub-warp of 16-byte chunks");
  // PFX >= 4 (tuning): L1 policy of the row gathers instead of a prefetch.  4: a-rows without
  // L1 allocation, 5: a-rows evict_first, 6: a-rows without allocation + b-rows evict_last,
  // 7: b-rows evict_last
  constexpr int PF = PFX >= 4 ? 0 : PFX;
  constexpr int AH = (PFX == 4 || PFX == 6) ? 1 : (PFX == 5 ? 2 : 0);
  constexpr int BH = (PFX == 6 || PFX == 7) ? 3 : 0;
  const int lane = threadIdx.x & (SW - 1);
  const unsigned mask = SW == 32 ? 0xffffffffu : (((1u << SW) - 1u) << (threadIdx.x & 31 & ~(SW - 1)));
  const long long nz0 = items[item].nz0, nz1 = items[item].nz1;
  const int slot = (int)items[item].slot;
  SACD_DBG(SACD_DASSERT(nz0 >= 0 && nz0 < nz1 && nz1 <= g_dbg.nnz && slot < g_dbg.nslots));
  const Real *Al = A + lane * VEC;
  const Real *Bl = B + lane * VEC;
  __shared__ __align__(16) Real xsb[XS == 1 ? 2 : 1][XS == 1 ? 256 : 1];
  __shared__ __align__(16) uint4 rsb[(XS == 2 || XS == 3) ? 2 : 1][(XS == 2 || XS == 3) ? 272 : 1];
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
    } else if constexpr (XS == 2 || XS == 3) {
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
      rsb[par][xs_slot<XS>(threadIdx.x)] = r;
      __syncwarp(mask);
    }
    uint32_t fb[SW];
    Real xr[D + 1];
    SR bb[D + 1];
    auto fetch = [&](int j) {  // b index + flags (and, XS == 2, x) of nonzero j of the batch
      if constexpr (XS == 2 || XS == 3) {
        const uint4 r = rsb[par][xs_slot<XS>(wbase + j)];
        fb[j] = r.x;
        if constexpr (sizeof(Real) == 8) xr[j % (D + 1)] = __hiloint2double((int)r.w, (int)r.z);
        else xr[j % (D + 1)] = __uint_as_float(r.z);
      } else {
        fb[j] = __shfl_sync(mask, my.y, j, SW);
      }
      SACD_DBG(SACD_DASSERT((fb[j] & kIdxMask) < g_dbg.Ib));
    };
#pragma unroll
    for (int j = 0; j < D && j < SW; ++j) {
      fetch(j);
      bb[j % (D + 1)].template load_hint<BH>(Bl + (long long)(fb[j] & kIdxMask) * RT);
    }
#pragma unroll
    for (int j = 0; j < SW; ++j) {
      if (j + D < SW) {
        fetch(j + D);
        bb[(j + D) % (D + 1)].template load_hint<BH>(Bl + (long long)(fb[j + D] & kIdxMask) * RT);
      }
      Real x;
      if constexpr (XS == 2 || XS == 3) x = xr[j % (D + 1)];
      else if constexpr (XS == 1) x = xsb[par][wbase + j];
      else if constexpr (XS == 4) x = (base + j < nz1) ? xu : Real(0);
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
          SACD_DBG(SACD_DASSERT(cur_row >= 0 && cur_row < g_dbg.In));
        }
        const uint32_t ai = __shfl_sync(mask, my.x, j, SW) & kIdxMask;
        SACD_DBG(SACD_DASSERT(ai < g_dbg.Ia));
        arow.template load_hint<AH>(Al + (long long)ai * RT);
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

template <typename Real, int RT, int SW, int D, int MINB, int PF = 0, int XS = 0>
__global__ void __launch_bounds__(256, MINB) k_mttkrp_lean(const WorkItem *__restrict__ items, long long n_items,
                                                          const uint4 *__restrict__ nzm,
                                                          const Real *__restrict__ A, const Real *__restrict__ B,
                                                          Real *__restrict__ M, Real *__restrict__ partial,
                                                          Real xu = Real(0)) {
  const long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / SW;
  if (item >= n_items) return;
  lean_item<Real, RT, SW, D, PF, XS>(item, items, nzm, A, B, M, partial, xu);
}

// Dynamic scheduling (one worker per warp): a fixed grid of resident warps takes items from
// a device counter (reset to 0 before the launch), so no launch ends on a partly-filled
// last wave -- that tail grew to ~50% of a sharded rank's MTTKRP, whose launch covers only
// about 2 waves of items.  Results do not depend on which warp takes which item.
// The same for SW < 32 (several workers per warp): every worker takes its own items.
template <typename Real, int RT, int SW, int D, int MINB, int PF = 0, int XS = 0>
__global__ void __launch_bounds__(256, MINB) k_mttkrp_lean_dyn_sw(const WorkItem *__restrict__ items,
                                                                 long long n_items, const uint4 *__restrict__ nzm,
                                                                 const Real *__restrict__ A, const Real *__restrict__ B,
                                                                 Real *__restrict__ M, Real *__restrict__ partial,
                                                                 unsigned long long *__restrict__ counter,
                                                                 Real xu = Real(0)) {
  const int lane = threadIdx.x & (SW - 1);
  const unsigned mask = SW == 32 ? 0xffffffffu : (((1u << SW) - 1u) << (threadIdx.x & 31 & ~(SW - 1)));
  for (;;) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(counter, 1ull);
    it = __shfl_sync(mask, it, 0, SW);
    if ((long long)it >= n_items) break;
    __syncwarp(mask);
    lean_item<Real, RT, SW, D, PF, XS>((long long)it, items, nzm, A, B, M, partial, xu);
  }
}

template <typename Real, int RT, int D, int MINB, int PF = 0, int XS = 0>
__global__ void __launch_bounds__(256, MINB) k_mttkrp_lean_dyn(const WorkItem *__restrict__ items, long long n_items,
                                                              const uint4 *__restrict__ nzm,
                                                              const Real *__restrict__ A, const Real *__restrict__ B,
                                                              Real *__restrict__ M, Real *__restrict__ partial,
                                                              unsigned long long *__restrict__ counter,
                                                              Real xu = Real(0)) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(counter, 1ull);
    it = __shfl_sync(0xffffffffu, it, 0);
    if ((long long)it >= n_items) break;
    __syncwarp();  // the warp's shared broadcast slots may still be read for its previous item
    lean_item<Real, RT, 32, D, PF, XS>((long long)it, items, nzm, A, B, M, partial, xu);
  }
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
  SACD_DBG(SACD_DASSERT(fc.slot0 >= 0 && fc.slot0 + fc.nslots <= g_dbg.nslots && fc.out < g_dbg.nchunk_rows &&
                        (fc.out >= 0 || -fc.out - 1 < g_dbg.In)));
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
  SACD_DBG(SACD_DASSERT(sr.row >= 0 && sr.row < g_dbg.In && sr.chunk0 + (nch > 1 ? nch : 0) <= g_dbg.nchunk_rows));
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

