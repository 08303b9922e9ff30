// k_rows.inc.cuh -- part of kernels.cu (included inside namespace sacd { namespace { ... } }).
// H, L and the branch (A2) and the fused SaCD row update (A4): FMA and DMMA kernels.
// Paper citations "P:n" are PAPER.md lines; readings Cn / L1 / C10' are DESIGN.md section 3.
// NOT a standalone header: it relies on the helpers defined at the top of kernels.cu.

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

// Fused row update with the gradient on the fp64 tensor cores (Real = double, RT <= 64).
// Same semantics and per-row order of the column steps as k_sacd_rows (Gauss-Seidel C9).
// For column block [c0, c0+8) the out-of-block part acc_q = sum_{j not in block} u_j h_(j,c0+q)
// of every row of a warp (32 rows) is one (32 x RT) x (RT x 8) product of the CURRENT rows
// (columns < c0 already updated this pass) with H, issued as DMMA m8n8k4 (4 row tiles x the
// k-steps outside the block, in ascending k).  The in-block Gauss-Seidel step then runs one
// thread per row: the in-block terms of the columns not yet visited are added up front, the
// term of column q' with its final value right after column q' is decided, so g of column q
// (Eq 14) sees every earlier update and the dependent chain per column is one FMA deep.
// g / h is the correctly rounded quotient: q0 = g * (1/h), r = fma(-q0, h, g) (exact),
// q = fma(r, 1/h, q0) with 1/h correctly rounded (Markstein's theorem; 1/h once per CTA).
// Fragments: A[m][k] = u[8mt+m][4kk+k] held by lane (g = lane >> 2, t = lane & 3) as
// Us[8mt+g][4kk+t]; B[k][n] = H[4kk+k][c0+n] as H[4kk+t][c0+g] (from L1: H is read-only and
// shared by every block); C[g][2t + {0,1}].  The accumulator tile and the block's M tile are
// transposed to one-row-per-thread through a per-warp shared tile.  Shared memory: Us (rows x
// (RT+4): the row pitch is 4 mod 16 doubles, so the fragment reads of a half-warp (4 rows x 4
// columns) and the Gram panel reads hit 16 distinct bank pairs, and 16-byte chunks stay
// aligned) + 32 x 18 doubles per warp + the 8 x 8 diagonal blocks of H, 1 / h_rr, the branch
// rule and ||H||_F (loaded once per CTA by rows_mma_prologue).
template <int RT>
__host__ __device__ constexpr int rows_mma_us() {
  return RT + 4;
}
template <int RT, int WPB>
__device__ __forceinline__ double *rows_mma_hd(unsigned char *smem_raw) {
  return reinterpret_cast<double *>(smem_raw) + WPB * 32 * rows_mma_us<RT>() + WPB * 32 * 18;
}
// H's diagonal 8 x 8 blocks ([RT/8][8][8]) and the reciprocals 1 / h_rr (0 where h_rr = 0)
// into shared memory; H is fixed for the whole pass.  Ends with __syncthreads.
template <int RT, int WPB>
__device__ __forceinline__ void rows_mma_prologue(const double *__restrict__ H, const DevState *__restrict__ st,
                                                  int mode, int l_mode) {
  constexpr int C = 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *Hd = rows_mma_hd<RT, WPB>(smem_raw);
  double *Ri = Hd + RT * C;
  for (int x = threadIdx.x; x < RT * C; x += WPB * 32) {
    const int b = x / (C * C), q = (x / C) % C, qq = x % C;
    Hd[x] = H[(b * C + q) * RT + b * C + qq];
  }
  for (int r = threadIdx.x; r < RT; r += WPB * 32) {
    const double h = H[r * RT + r];
    Ri[r] = h != 0.0 ? 1.0 / h : 0.0;
    Ri[RT + 2 + r] = (l_mode ? st->Lfrob[mode] : h) * 0.5;  // L / 2 of Eq 20 (exact halving)
  }
  if (threadIdx.x == 0) {  // the pass's branch rule and ||H||_F, also fixed for the launch
    Ri[RT] = (double)st->branch[mode];
    Ri[RT + 1] = st->Lfrob[mode];
  }
  __syncthreads();
}

// Issue the staging of row block rb's factor rows into Us (cp.async, rows past the range
// zero-filled); rows_mma_block waits for it.
template <int RT, int WPB>
__device__ __forceinline__ void rows_mma_stage(long long rb, long long row_begin, long long row_end,
                                               const double *__restrict__ F) {
  constexpr int TR = WPB * 32;
  constexpr int US = rows_mma_us<RT>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *Us = reinterpret_cast<double *>(smem_raw);
  const long long row0 = row_begin + rb * TR;
  const int nrows = (int)min((long long)TR, row_end - row0);
  const double *Fg = F + row0 * RT;
  for (int x = threadIdx.x; x < TR * RT / 2; x += TR) {  // 16-byte chunks
    const int r = (2 * x) / RT, col = (2 * x) % RT;
    if (r < nrows) cp_async<16>(Us + r * US + col, Fg + 2 * x);
    else *reinterpret_cast<double2 *>(Us + r * US + col) = make_double2(0.0, 0.0);
  }
}

// Is this thread's row of block rb an empty slice (m = 0)?  false past the range.
template <int WPB>
__device__ __forceinline__ bool rows_mma_empty(long long rb, long long row_begin, long long row_end,
                                               const long long *__restrict__ row_ptr) {
  const long long row = row_begin + rb * (WPB * 32) + threadIdx.x;
  return row < row_end ? __ldg(row_ptr + row) == __ldg(row_ptr + row + 1) : true;
}

template <int RT, int WPB>
__device__ __forceinline__ void rows_mma_block(long long rb, long long row_begin, long long row_end, int R, int mode,
                    int l_mode,
                    const long long *__restrict__ row_ptr, const double *__restrict__ M, double *__restrict__ F,
                    double *__restrict__ Z, const double *__restrict__ H, const DevState *__restrict__ st,
                    uint8_t *__restrict__ dec, double *__restrict__ ti_part, double *__restrict__ md_part,
                    long long *__restrict__ e_part, long long *__restrict__ ech_part,
                    double *const *__restrict__ peers = nullptr, int G = 0, int me = 0,
                    const long long *next_rb = nullptr, long long nblk = 0, bool empty_in = false,
                    bool *empty_next = nullptr) {
  constexpr int TR = WPB * 32;
  constexpr int US = rows_mma_us<RT>();
  constexpr int C = 8;
  constexpr int TS = 2 * C + 2;
  constexpr int NKS = RT / 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *Us = reinterpret_cast<double *>(smem_raw);
  const double *Hd = rows_mma_hd<RT, WPB>(smem_raw);  // [RT/8][8][8], then 1 / h_rr [RT]
  const double *Ri = Hd + RT * C;
  __shared__ double red_d[2][WPB];
  __shared__ long long red_l[2][WPB];

  const int tid = threadIdx.x;
  const int lane = tid & 31, wp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  double *Tw = Us + TR * US + wp * 32 * TS;
  const long long row0 = row_begin + rb * TR;
  const int nrows = (int)min((long long)TR, row_end - row0);
  static_assert((US * 8) % 16 == 0, "row stride must keep 16-byte chunks aligned");
  const bool active = tid < nrows;
  const long long row = row0 + tid;
  // the block's staging (rows_mma_stage) is in flight; the empty-slice flag (m = 0) comes
  // from the caller (the dynamic kernel loads it one block ahead)
  const bool empty = empty_next ? empty_in : rows_mma_empty<WPB>(rb, row_begin, row_end, row_ptr);
  const int branch = (int)Ri[RT];
  // the branch rule as one sign test: FIRST z > 0 (z_prev taken as 0), EQ24 z - z_prev > 0,
  // EQ27 z_prev - z > 0, i.e. -(z - z_prev) > 0 (IEEE subtraction is antisymmetric, negation
  // and z - 0 are exact)
  const bool first = branch == SACD_BR_FIRST;
  const double sgn = branch == SACD_BR_EQ27 ? -1.0 : 1.0;
  const double *Lh = Ri + RT + 2;
  double *zp = Z + tt<RT>(active ? row : row0, 0);
  const double *Uw = Us + (wp * 32 + g) * US + t;

  // software pipeline over column blocks: the B fragments, the M tile and this thread's
  // z_prev of block c0 + 8 are loaded while block c0 is processed (all read-only here)
  double bf[NKS], mt[C], zv[C];
  auto load_block = [&](int c, double (&b)[NKS], double (&mm)[C], double (&zz)[C]) {
    // unconditional loads (no select right behind them, so they stay in flight for a whole
    // block): H's padding rows are zero, rows past the range read the last row and
    // inactive threads read row0's z_prev (neither is used)
#pragma unroll
    for (int kk = 0; kk < NKS; ++kk) b[kk] = ld_keep_f64(H + (4 * kk + t) * RT + c + g);
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const int x = lane + 32 * k, rl = x / C, cl = x % C;
      const long long rg = min(row0 + wp * 32 + rl, row_end - 1);
      mm[k] = ld_stream_f64(M + rg * RT + c + cl);
    }
#pragma unroll
    for (int q = 0; q < C; ++q) zz[q] = first ? 0.0 : ld_na_f64(zp + 32 * (c + q));  // FIRST: not read
  };
  load_block(0, bf, mt, zv);
  cp_async_wait_all();
  __syncthreads();

  double ti = 0.0, md = 0.0;
  unsigned E = 0, Ech = 0;  // per thread at most 64 x (its rows) < 2^32
  double *u = Us + tid * US;
  for (int c0 = 0; c0 < R; c0 += C) {
    double bfn[NKS], mtn[C], zvn[C];
    if (c0 + C < R) load_block(c0 + C, bfn, mtn, zvn);
    // (1) out-of-block part of the warp's 32 rows on the tensor cores: the block's own two
    //     k-steps are skipped (a uniform branch), the k-steps past R multiply zero padding
    //     (A and H); even / odd k-steps in two sets of tiles
    double cacc[2][4][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int m = 0; m < 4; ++m) cacc[h][m][0] = cacc[h][m][1] = 0.0;
    const int kb = c0 / 4;
#pragma unroll
    for (int kk = 0; kk < NKS; ++kk) {
      if (kk == kb || kk == kb + 1) continue;
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
      }
#pragma unroll
      for (int q = 0; q < C; q += 2) {
        const double2 v = *reinterpret_cast<const double2 *>(u + c0 + q);
        ub[q] = v.x;
        ub[q + 1] = v.y;
      }
      const double *Hb = Hd + (c0 / C) * C * C;
      unsigned selbits = 0;
      // (3) in-block Gauss-Seidel (C9).  acc_q starts as the out-of-block sum; the in-block
      //     terms of the columns not yet visited (q' >= q: their values at block start) are
      //     added now, independently per column, and the term of column q' < q is added with
      //     its final value as soon as column q' is decided, so every term enters once with
      //     the value the sequential sweep sees, an all-zero row sums to exactly 0, and the
      //     dependent chain per column is one FMA deep
#pragma unroll
      for (int q = 0; q < C; ++q)
#pragma unroll
        for (int qq = q; qq < C; ++qq) acc[q] = fma(ub[qq], Hb[q * C + qq], acc[q]);
      // padding columns (r >= R) have h = 0 (H is zero-padded) and u = m = 0: they take the
      // h = 0 path (z = 0, no selection) and add exact zeros, so no r < R test is needed.
      // Column q + 1's gradient depends on column q only through u_q's final value, which is
      // u_q or the candidate u'_q: both versions of column q + 1's g and u' are computed
      // while column q's z and gate are still in flight, and the gate picks one.  The picked
      // values are exactly the sequential ones; the dependent chain per column shrinks to the
      // gate (d, z, z - z_prev) and one select.
      auto cand = [&](double gr, double ur, double h, double ri) {  // max(0, u - g / h), Eq 11-13
        const double q0 = gr * ri;                                  // g / h, correctly rounded
        const double qr = fma(-q0, h, gr);
        const double ut = ur - fma(qr, ri, q0);
        return ut > 0.0 ? ut : 0.0;                                 // a zero's sign is immaterial
      };
      double gr = acc[0] - mv[0];                                   // Eq 14
      double un = cand(gr, ub[0], Hb[0], Ri[c0]);
#pragma unroll
      for (int q = 0; q < C; ++q) {
        const int r = c0 + q;
        const double h = Hb[q * C + q];
        const double ur = ub[q];
        const double d = un - ur;                                   // Eq 12
        double z = -gr * d - Lh[r] * d * d;                         // Eq 20 (Lh = L / 2)
        const bool sel = h != 0.0 && (z - zv[q]) * sgn > 0.0;
        if (h == 0.0) z = 0.0;
        double grn = 0.0, unn = 0.0;
        if (q + 1 < C) {
          const double hqn = Hb[q * C + q + 1], hn = Hb[(q + 1) * C + q + 1], rin = Ri[r + 1];
          const double g0 = fma(ur, hqn, acc[q + 1]) - mv[q + 1];  // column q kept u_q
          const double g1 = fma(un, hqn, acc[q + 1]) - mv[q + 1];  // column q took u'_q
          const double u0 = cand(g0, ub[q + 1], hn, rin), u1 = cand(g1, ub[q + 1], hn, rin);
          grn = sel ? g1 : g0;
          unn = sel ? u1 : u0;
        }
        if (sel) {
          ub[q] = un;
          E += 1;
          if (d != 0.0) Ech += 1;
          selbits |= 1u << q;
        }
#pragma unroll
        for (int q2 = q + 2; q2 < C; ++q2) acc[q2] = fma(ub[q], Hb[q * C + q2], acc[q2]);
        zv[q] = z;                                                  // z_prev <- z always (C8)
        ti += z;                                                    // Eq 25
        md += ub[q] * mv[q];
        gr = grn;
        un = unn;
      }
      if (dec) {
#pragma unroll
        for (int q = 0; q < C; ++q)
          if (c0 + q < R) dec[row * R + c0 + q] = (uint8_t)((selbits >> q) & 1u);
      }
#pragma unroll
      for (int q = 0; q < C; q += 2) *reinterpret_cast<double2 *>(u + c0 + q) = make_double2(ub[q], ub[q + 1]);
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
  if (peers) {
    // peer-memory exchange fused into the write-back (sharded engine, exchange = p2p): every
    // 16-byte chunk of the block's rows that differs from the pass-start value still in F is
    // also stored into every peer's replica, so the NVLink traffic of one block overlaps the
    // compute of the others
    for (int x = tid; x < nrows * RT / 2; x += TR) {
      const int r = (2 * x) / RT, col = (2 * x) % RT;
      const double2 nv = make_double2(Us[r * US + col], Us[r * US + col + 1]);
      const double2 ov = reinterpret_cast<const double2 *>(Fo)[x];
      if (__double_as_longlong(nv.x) != __double_as_longlong(ov.x) ||
          __double_as_longlong(nv.y) != __double_as_longlong(ov.y)) {
        for (int p = 0; p < G; ++p)
          if (p != me) reinterpret_cast<double2 *>(peers[p] + row0 * RT)[x] = nv;
      }
      reinterpret_cast<double2 *>(Fo)[x] = nv;
    }
  } else {
    for (int x = tid; x < nrows * RT / 2; x += TR) {
      const int r = (2 * x) / RT, col = (2 * x) % RT;
      reinterpret_cast<double2 *>(Fo)[x] = *reinterpret_cast<const double2 *>(Us + r * US + col);
    }
  }
  if (next_rb) {  // Us is free once every thread has read it: stage the next block now, so
                  // its loads overlap this block's reductions and the next block's start
    __syncthreads();
    const long long nb = *next_rb;
    if (nb < nblk) {
      rows_mma_stage<RT, WPB>(nb, row_begin, row_end, F);
      if (empty_next) *empty_next = rows_mma_empty<WPB>(nb, row_begin, row_end, row_ptr);
    }
  }

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
    ti_part[rb] = a;
    md_part[rb] = b;
    e_part[rb] = c;
    ech_part[rb] = d;
  }
}


template <int RT, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_sacd_rows_mma(long long row_begin, long long row_end, int R, int mode, int l_mode,
                    const long long *__restrict__ row_ptr, const double *__restrict__ M, double *__restrict__ F,
                    double *__restrict__ Z, const double *__restrict__ H, const DevState *__restrict__ st,
                    uint8_t *__restrict__ dec, double *__restrict__ ti_part, double *__restrict__ md_part,
                    long long *__restrict__ e_part, long long *__restrict__ ech_part) {
  rows_mma_stage<RT, WPB>(blockIdx.x, row_begin, row_end, F);
  rows_mma_prologue<RT, WPB>(H, st, mode, l_mode);
  rows_mma_block<RT, WPB>(blockIdx.x, row_begin, row_end, R, mode, l_mode, row_ptr, M, F, Z, H, st, dec, ti_part,
                          md_part, e_part, ech_part);
}

// Dynamically scheduled: a grid of resident blocks takes 128-row blocks from a device counter
// (reset before the launch), so a launch of few waves (a sharded rank's rows) does not end
// on a partly filled wave.  The partials are indexed by the row block, as in the static grid.
template <int RT, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_sacd_rows_mma_dyn(long long row_begin, long long row_end, int R, int mode, int l_mode,
                        const long long *__restrict__ row_ptr, const double *__restrict__ M, double *__restrict__ F,
                        double *__restrict__ Z, const double *__restrict__ H, const DevState *__restrict__ st,
                        uint8_t *__restrict__ dec, double *__restrict__ ti_part, double *__restrict__ md_part,
                        long long *__restrict__ e_part, long long *__restrict__ ech_part, long long nblk,
                        unsigned long long *__restrict__ counter, double *const *__restrict__ peers = nullptr,
                        int G = 0, int me = 0) {
  // the next block's index is taken at the start of the current one, and its staging is
  // issued as soon as the current block's rows are written back (rows_mma_block)
  __shared__ long long rb_s[2];
  if (threadIdx.x == 0) rb_s[0] = (long long)atomicAdd(counter, 1ull);
  rows_mma_prologue<RT, WPB>(H, st, mode, l_mode);  // ends with __syncthreads
  long long rb = rb_s[0];
  bool empty = true;
  if (rb < nblk) {
    rows_mma_stage<RT, WPB>(rb, row_begin, row_end, F);
    empty = rows_mma_empty<WPB>(rb, row_begin, row_end, row_ptr);
  }
  for (int it = 1; rb < nblk; it ^= 1) {
    // slot it was last read before the previous block's closing barrier
    if (threadIdx.x == 0) rb_s[it] = (long long)atomicAdd(counter, 1ull);
    bool empty_nx = true;
    rows_mma_block<RT, WPB>(rb, row_begin, row_end, R, mode, l_mode, row_ptr, M, F, Z, H, st, dec, ti_part, md_part,
                            e_part, ech_part, peers, G, me, rb_s + it, nblk, empty, &empty_nx);
    empty = empty_nx;
    __syncthreads();  // thread 0's partial writes and rb_s[it] reads are done
    rb = rb_s[it];
  }
}

// Gram refresh fused into the row update (Eq 10's G_n = F_n^T F_n of the factor just
// updated): after a 128-row block is final in shared memory (Us), the block's contribution
// Us^T Us is added on the fp64 tensor cores to a per-CTA accumulator held in registers, so
// the updated factor is never re-read from HBM for its Gram.  The upper-triangle 8 x 8 tiles
// (ti <= tj) of the RT x RT Gram are dealt round-robin to the CTA's warps (tile q -> warp
// q mod WPB, at most ceil(P(P+1)/2 / WPB) tiles per warp, P = RT / 8); each tile is a chain of
// m8n8k4 DMMAs over the block's rows, 4 at a time: A[m][k] = Us[4kk + k][8ti + m] held by lane
// (g, t) as Us[4kk + t][8ti + g], B[k][n] = Us[4kk + k][8tj + n] as Us[4kk + t][8tj + g],
// C[g][2t + e] = G[8ti + g][8tj + 2t + e].  Rows past the range are zero in Us (the staging
// zero-fills them), padding columns are zero in F.
template <int RT, int WPB>
struct GramAcc {
  static constexpr int P = RT / 8;
  static constexpr int NT = P * (P + 1) / 2;
  static constexpr int TPW = (NT + WPB - 1) / WPB;
  double c[TPW][2];
  __device__ __forceinline__ static void tile_ij(int q, int &ti, int &tj) {  // q-th upper tile, row major
    ti = 0;
    while (q >= P - ti) {
      q -= P - ti;
      ++ti;
    }
    tj = ti + q;
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < TPW; ++k) c[k][0] = c[k][1] = 0.0;
  }
  // k-steps outer, tiles inner: the warp's TPW accumulator chains are independent, so their
  // DMMAs overlap (a tile-outer loop made one dependent chain of TPW * rows / 4 DMMAs); the
  // P panel fragments of a k-step are loaded once and shared by the tiles.  The warp index is
  // a template argument so that every tile's two panels are compile-time register picks.
  __host__ __device__ static constexpr int tile_i(int q) {
    int ti = 0;
    while (q >= P - ti) {
      q -= P - ti;
      ++ti;
    }
    return ti;
  }
  __host__ __device__ static constexpr int tile_j(int q) {
    int ti = 0;
    while (q >= P - ti) {
      q -= P - ti;
      ++ti;
    }
    return ti + q;
  }
  template <int W, int K>
  __device__ __forceinline__ void mma_tiles(const double (&pf)[P]) {
    if constexpr (K < TPW) {
      constexpr int q = W + WPB * K;
      if constexpr (q < NT) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[K][0]), "+d"(c[K][1])
                     : "d"(pf[tile_i(q)]), "d"(pf[tile_j(q)]));
      }
      mma_tiles<W, K + 1>(pf);
    }
  }
  template <int W>
  __device__ __forceinline__ void add_block_w(const double *Us, int US, int nrows_pad, int lane) {
    const int g = lane >> 2, t = lane & 3;
    const double *p0 = Us + t * US + g;
    for (int r0 = 0; r0 < nrows_pad; r0 += 4) {
      double pf[P];
#pragma unroll
      for (int j = 0; j < P; ++j) pf[j] = p0[r0 * US + 8 * j];
      mma_tiles<W, 0>(pf);
    }
  }
  // a chunk of NR (compile-time) rows, fully unrolled so the panel loads of later k-steps
  // are issued ahead of the DMMAs
  template <int W, int NR, int US>
  __device__ __forceinline__ void add_chunk_w(const double *Us, int lane) {
    const int g = lane >> 2, t = lane & 3;
    const double *p0 = Us + t * US + g;
#pragma unroll
    for (int r0 = 0; r0 < NR; r0 += 4) {
      double pf[P];
#pragma unroll
      for (int j = 0; j < P; ++j) pf[j] = p0[r0 * US + 8 * j];
      mma_tiles<W, 0>(pf);
    }
  }
  template <int NR, int US>
  __device__ __forceinline__ void add_chunk(const double *Us, int wp, int lane) {
    static_assert(WPB == 4, "add_chunk dispatches 4 warps");
    switch (wp) {
      case 0: add_chunk_w<0, NR, US>(Us, lane); break;
      case 1: add_chunk_w<1, NR, US>(Us, lane); break;
      case 2: add_chunk_w<2, NR, US>(Us, lane); break;
      default: add_chunk_w<3, NR, US>(Us, lane); break;
    }
  }
  __device__ __forceinline__ void add_block(const double *Us, int US, int nrows_pad, int wp, int lane) {
    static_assert(WPB == 4, "add_block dispatches 4 warps");
    switch (wp) {
      case 0: add_block_w<0>(Us, US, nrows_pad, lane); break;
      case 1: add_block_w<1>(Us, US, nrows_pad, lane); break;
      case 2: add_block_w<2>(Us, US, nrows_pad, lane); break;
      default: add_block_w<3>(Us, US, nrows_pad, lane); break;
    }
  }
  // upper-triangle entries (r <= t) of this CTA's partial: the k_gram_reduce contract
  __device__ __forceinline__ void store(double *part, int R, int wp, int lane) const {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int k = 0; k < TPW; ++k) {
      const int q = wp + WPB * k;
      if (q < NT) {
        int ti, tj;
        tile_ij(q, ti, tj);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 8 * ti + g, cc = 8 * tj + 2 * t + e;
          if (r < R && cc < R && r <= cc) part[r * R + cc] = c[k][e];
        }
      }
    }
  }
};

// Gram partials G_b = sum of u u^T over rows [row_begin, row_end) of F (fp64, RT <= 64; Eq 10's
// G_n = F_n^T F_n of the factor just updated), streamed through shared memory: CTA b takes
// the 32-row chunks [b * nch / grid, (b + 1) * nch / grid) (a fixed assignment, so its
// partial and the fixed-order k_gram_reduce are deterministic), stages them with cp.async
// into an S-deep ring at the conflict-free row pitch of the row update, S - 1 chunks ahead,
// and adds each chunk's u u^T on the fp64 tensor cores with GramAcc (36 upper 8 x 8 tiles
// for R = 64, 9 per warp).  Rows past the range are zero-filled.  Partial b goes to
// part[b] (upper entries r <= t, the k_gram_reduce contract).
template <int RT, int S>
__host__ __device__ constexpr size_t gram_stream_smem_bytes() {
  return (size_t)S * 32 * rows_mma_us<RT>() * 8;
}
template <int RT, int S>
__global__ void __launch_bounds__(128) k_gram_stream(long long row_begin, long long row_end, int R,
                                                     const double *__restrict__ F, double *__restrict__ part) {
  constexpr int US = rows_mma_us<RT>();
  constexpr int CH = 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *ring = reinterpret_cast<double *>(smem_raw);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const long long nch = (row_end - row_begin + CH - 1) / CH;
  const long long c0 = nch * blockIdx.x / gridDim.x, c1 = nch * (blockIdx.x + 1) / gridDim.x;
  auto stage = [&](long long ch) {
    double *dst = ring + (int)((ch - c0) % S) * CH * US;
    const long long r0 = row_begin + ch * CH;
    const int nr = (int)min((long long)CH, row_end - r0);
    const double *src = F + r0 * RT;
    for (int x = threadIdx.x; x < CH * RT / 2; x += 128) {  // 16-byte chunks
      const int r = (2 * x) / RT, col = (2 * x) % RT;
      if (r < nr) cp_async<16>(dst + r * US + col, src + 2 * x);
      else *reinterpret_cast<double2 *>(dst + r * US + col) = make_double2(0.0, 0.0);
    }
  };
  GramAcc<RT, 4> acc;
  acc.zero();
#pragma unroll
  for (int k = 0; k < S - 1; ++k) {
    if (c0 + k < c1) stage(c0 + k);
    cp_async_commit();
  }
  for (long long ch = c0; ch < c1; ++ch) {
    if (ch + S - 1 < c1) stage(ch + S - 1);  // the slot of chunk ch - 1, released below
    cp_async_commit();
    cp_async_wait_group<S - 1>();  // this thread's copies of chunk ch are done
    __syncthreads();               // ... and every thread's copies and zero fills
    acc.template add_chunk<CH, US>(ring + (int)((ch - c0) % S) * CH * US, wp, lane);
    __syncthreads();  // chunk ch's slot is restaged next iteration
  }
  acc.store(part + (long long)blockIdx.x * R * R, R, wp, lane);
}

// Row update with the fused Gram: CTA b takes the contiguous row blocks
// [b * nblk / grid, (b + 1) * nblk / grid) in order (a fixed assignment, so the Gram partial of
// each CTA, and the fixed-order reduce over CTAs, are deterministic), and writes its Gram
// partial to part[blockIdx.x].
template <int RT, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_sacd_rows_mma_gram(long long row_begin, long long row_end, int R, int mode, int l_mode,
                         const long long *__restrict__ row_ptr, const double *__restrict__ M, double *__restrict__ F,
                         double *__restrict__ Z, const double *__restrict__ H, const DevState *__restrict__ st,
                         uint8_t *__restrict__ dec, double *__restrict__ ti_part, double *__restrict__ md_part,
                         long long *__restrict__ e_part, long long *__restrict__ ech_part, long long nblk,
                         double *__restrict__ gram_part, double *const *__restrict__ peers = nullptr, int G = 0,
                         int me = 0) {
  constexpr int TR = WPB * 32;
  constexpr int US = rows_mma_us<RT>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const double *Us = reinterpret_cast<const double *>(smem_raw);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  rows_mma_prologue<RT, WPB>(H, st, mode, l_mode);
  GramAcc<RT, WPB> acc;
  acc.zero();
  const long long b0 = nblk * blockIdx.x / gridDim.x, b1 = nblk * (blockIdx.x + 1) / gridDim.x;
  for (long long rb = b0; rb < b1; ++rb) {
    rows_mma_stage<RT, WPB>(rb, row_begin, row_end, F);
    rows_mma_block<RT, WPB>(rb, row_begin, row_end, R, mode, l_mode, row_ptr, M, F, Z, H, st, dec, ti_part, md_part,
                            e_part, ech_part, peers, G, me);
    // Us holds the block's final rows (rows past the range are zero): add them to the Gram
    const int nrows = (int)min((long long)TR, row_end - (row_begin + rb * TR));
    acc.add_block(Us, US, (nrows + 3) & ~3, wp, lane);
    __syncthreads();  // the next block's staging overwrites Us
  }
  acc.store(gram_part + (long long)blockIdx.x * R * R, R, wp, lane);
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
  return (size_t)WPB * 32 * rows_mma_us<RT>() * 8 + (size_t)WPB * 32 * 18 * 8 + (size_t)RT * 8 * 8 + (size_t)(2 * RT + 2) * 8;
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

