// k_gram.inc.cuh -- part of kernels.cu (included inside namespace sacd { namespace { ... } }).
// Gram G = F^T F (A2 refresh): the DMMA and FMA partial kernels and the fixed-order reduce.
// Paper citations "P:n" are PAPER.md lines; readings Cn / L1 / C10' are DESIGN.md section 3.
// NOT a standalone header: it relies on the helpers defined at the top of kernels.cu.

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

// G[r][t] = G[t][r] = the fixed-order sum over the nblk partials of upper entry (r, t): one
// warp per upper entry, lane l sums partials l, l + 32, ... in order, then a fixed xor tree
// (deterministic; a thread per entry with a 296-long serial chain left this reduce at
// ~180 GB/s, 0.16 ms per c4 sweep).  An entry with r <= t lies in a panel pair / tile with
// bi <= bj, which wrote it.
__global__ void __launch_bounds__(256) k_gram_reduce(int R, int nblk, const double *__restrict__ part,
                                                     double *__restrict__ G) {
  const int w = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  const int nup = R * (R + 1) / 2;
  if (w >= nup) return;
  int r = 0, q = w;  // the w-th upper entry, row major
  while (q >= R - r) {
    q -= R - r;
    ++r;
  }
  const int t = r + q;
  const long long src = (long long)r * R + t;
  double s = 0.0;
  for (int b = lane; b < nblk; b += 32) s += part[(long long)b * R * R + src];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    G[r * R + t] = s;
    G[t * R + r] = s;
  }
}

inline unsigned gram_reduce_blocks(int R) { return (unsigned)((R * (R + 1) / 2 * 32 + 255) / 256); }

