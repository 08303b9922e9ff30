// layout.cu -- per-mode sorted nonzero layout, built once on device by sacd_init.
//
// The paper's slices Omega^U_q, Omega^V_p, Omega^W_s (Table 2) become,
// per mode n, the nonzeros sorted by the key (i_n, i_a, i_b) where a is the longer other
// mode (ties -> lower mode id; reading L1) and b the remaining one, so the fiber-
// factored MTTKRP gathers the shorter factor per nonzero; row_ptr[i] .. row_ptr[i+1] is the
// slice of row i.  This replaces the unfolding X_(n) (Lemma 4), which
// is never materialised.  Keys are unique (duplicates are rejected), so the order
// is unique and equals the oracle's bit for bit.
//
// Steps (all on device): validate -> 64-bit keys -> cub radix sort of (key, position) ->
// duplicate check -> gather idx_a, idx_b, val -> row_ptr by binary search -> ||X||^2.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "sacd_internal.cuh"

namespace sacd {

namespace {

__global__ void k_validate(const uint32_t *__restrict__ coords, const float *__restrict__ vals, long long nnz,
                           long long d0, long long d1, long long d2, int *__restrict__ flags) {
  // flags: 1 = index out of range, 2 = non-finite value, 8 = the values are not all equal
  // (bitwise) to vals[0]; bit 8 clear means a uniform-valued tensor (e.g. binary), for which
  // the MTTKRP needs no per-nonzero value at all
  const uint32_t v0 = nnz > 0 ? __float_as_uint(vals[0]) : 0u;
  bool diff = false;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    const uint32_t q = coords[3 * e], p = coords[3 * e + 1], s = coords[3 * e + 2];
    if (q >= d0 || p >= d1 || s >= d2) atomicOr(flags, 1);
    if (!isfinite(vals[e])) atomicOr(flags, 2);
    diff |= __float_as_uint(vals[e]) != v0;
  }
  if (__any_sync(0xffffffffu, diff) && (threadIdx.x & 31) == 0) atomicOr(flags, 8);
}

__global__ void k_make_keys(const uint32_t *__restrict__ coords, long long nnz, int n, int a, int b,
                            unsigned long long Ia, unsigned long long Ib, unsigned long long *__restrict__ keys,
                            uint32_t *__restrict__ pos) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    const unsigned long long in = coords[3 * e + n], ia = coords[3 * e + a], ib = coords[3 * e + b];
    keys[e] = (in * Ia + ia) * Ib + ib;
    pos[e] = (uint32_t)e;
  }
}

__global__ void k_check_dup(const unsigned long long *__restrict__ keys, long long nnz, int *__restrict__ flags) {
  for (long long e = 1 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x)
    if (keys[e] == keys[e - 1]) atomicOr(flags, 4);
}

// Gather the sorted entries; idx_a and idx_b get the fiber-start / row-start flag bits and idx_n
// the row index (both derived from the sorted keys).
__global__ void k_gather(const uint32_t *__restrict__ coords, const float *__restrict__ vals,
                         const uint32_t *__restrict__ pos, const unsigned long long *__restrict__ keys,
                         long long nnz, int a, int b, unsigned long long Ib, unsigned long long IaIb,
                         uint32_t *__restrict__ ia, uint32_t *__restrict__ ib, uint32_t *__restrict__ in_,
                         float *__restrict__ v, uint4 *__restrict__ nzm, unsigned long long *__restrict__ nfib) {
  for (long long e0 = blockIdx.x * (long long)blockDim.x; e0 < nnz; e0 += (long long)gridDim.x * blockDim.x) {
    const long long e = e0 + threadIdx.x;  // warp-uniform loop: the fiber count uses a ballot
    bool fs = false;
    if (e < nnz) {
    const long long p = pos[e];
    const unsigned long long k = keys[e];
    const unsigned long long row = k / IaIb;
    bool row_start = true, fiber_start = true;
    if (e > 0) {
      const unsigned long long kp = keys[e - 1];
      row_start = (kp / IaIb) != row;
      fiber_start = (kp / Ib) != (k / Ib);
    }
    const uint32_t fl = (fiber_start ? kFiberStart : 0u) | (row_start ? kRowStart : 0u);
    const uint32_t xa = coords[3 * p + a] | fl, xb = coords[3 * p + b] | fl;
    const float x = vals[p];
    if (ia) {  // SoA copies only when a kernel of this context reads them (layout_needs_soa)
      ia[e] = xa;
      ib[e] = xb;
      in_[e] = (uint32_t)row;
      v[e] = x;
    }
    nzm[e] = make_uint4(xa, xb, __float_as_uint(x), (uint32_t)row);
    fs = fiber_start;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, fs);
    if ((threadIdx.x & 31) == 0 && bal) atomicAdd(nfib, (unsigned long long)__popc(bal));
  }
}

// row_ptr[i] = #keys < i * (Ia*Ib)   (lower bound), i = 0..I
__global__ void k_row_ptr(const unsigned long long *__restrict__ keys, long long nnz, long long I,
                          unsigned long long stride, long long *__restrict__ row_ptr) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= I;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long target = (unsigned long long)i * stride;
    long long lo = 0, hi = nnz;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    row_ptr[i] = lo;
  }
}

// ||X||^2 = sum x^2 in fp64: fixed grid of per-block partials, then one block in order.
constexpr int kNormBlocks = 296;
__global__ void k_norm_partial(const uint4 *__restrict__ nzm, long long nnz, double *__restrict__ part) {
  __shared__ double sh[256];
  const long long per = (nnz + gridDim.x - 1) / gridDim.x;
  const long long e0 = blockIdx.x * per, e1 = min(nnz, e0 + per);
  double s = 0.0;
  for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const double x = (double)__uint_as_float(nzm[e].z);
    s += x * x;
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_norm_final(const double *__restrict__ part, int n, DevState *st) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; i++) s += part[i];
    st->xnorm2 = s;
  }
}

inline int grid_for(long long n) {
  long long g = (n + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

__global__ void k_widen(const uint32_t *__restrict__ a, long long n, unsigned long long *__restrict__ b) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    b[e] = a[e];
}

int bits_for(unsigned long long maxkey) {
  int b = 1;
  while (b < 64 && (maxkey >> b) != 0) b++;
  return b;
}

}  // namespace

// ---- a-blocked execution order (MTTKRP locality for modes with long slices) ----------
// The MTTKRP of mode n gathers one a-row per fiber.  When F_a is much larger than L2 and
// the slices are long (few rows), consecutive work items touch a-rows spread over all of
// F_a.  Regrouping the nonzeros by a-block (i_a / ablk_rows) keeps one block of F_a
// (<= ~40 MB) hot in L2 while every slice is swept: the order becomes (blk, i_n, i_a, i_b),
// a stable regrouping of the canonical order, and every (blk, row) run is a row segment
// whose partial the split-row fix-up sums in block order (deterministic).
__global__ void k_block_keys(const uint32_t *__restrict__ ia, long long nnz, long long ablk_rows,
                             uint32_t *__restrict__ keys, uint32_t *__restrict__ pos) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    keys[e] = (uint32_t)((long long)(ia[e] & kIdxMask) / ablk_rows);
    pos[e] = (uint32_t)e;
  }
}

// blocked nzm + segment-start flags: segment = maximal run of equal (blk, row)
__global__ void k_block_gather(const uint32_t *__restrict__ perm, const uint32_t *__restrict__ blk,
                               const uint32_t *__restrict__ ia, const uint32_t *__restrict__ ib,
                               const uint32_t *__restrict__ in_, const float *__restrict__ v, long long nnz,
                               uint4 *__restrict__ nzm, uint32_t *__restrict__ seg_flag) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    const uint32_t p = perm[e];
    const uint32_t a = ia[p] & kIdxMask, b = ib[p] & kIdxMask, row = in_[p];
    bool seg = true, fib = true;
    if (e > 0) {
      const uint32_t q = perm[e - 1];
      seg = blk[e] != blk[e - 1] || in_[q] != row;
      fib = seg || (ia[q] & kIdxMask) != a;
    }
    const uint32_t fl = (fib ? kFiberStart : 0u) | (seg ? kRowStart : 0u);
    nzm[e] = make_uint4(a | fl, b | fl, __float_as_uint(v[p]), row);
    seg_flag[e] = seg ? 1u : 0u;
  }
}

__global__ void k_seg_list(const uint32_t *__restrict__ seg_flag, const unsigned long long *__restrict__ seg_idx,
                           const uint32_t *__restrict__ nzm_row, long long nnz, long long *__restrict__ seg_start,
                           int *__restrict__ seg_row) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x)
    if (seg_flag[e]) {
      const unsigned long long k = seg_idx[e];  // exclusive prefix count of segment starts
      seg_start[k] = e;
      seg_row[k] = (int)nzm_row[4 * e + 3];
    }
}

int build_blocked_order(Context &c, int n, long long ablk_rows, std::vector<long long> &seg_start,
                        std::vector<int> &seg_row) {
  ModeData &md = c.m[n];
  const long long nnz = c.nnz;
  cudaStream_t s = c.stream;
  uint32_t *keys = nullptr, *keys2 = nullptr, *pos = nullptr, *perm = nullptr, *flag = nullptr;
  unsigned long long *idx = nullptr, *flag64 = nullptr;
  long long *d_start = nullptr;
  int *d_row = nullptr;
  void *temp = nullptr;
  size_t tb = 0, tb2 = 0;
  const size_t ne = (size_t)nnz;
  SACD_CUDA_TRY(pool_alloc(&keys, ne * 4, c.device, s));
  SACD_CUDA_TRY(pool_alloc(&keys2, ne * 4, c.device, s));
  SACD_CUDA_TRY(pool_alloc(&pos, ne * 4, c.device, s));
  SACD_CUDA_TRY(pool_alloc(&perm, ne * 4, c.device, s));
  SACD_CUDA_TRY(pool_alloc(&flag, ne * 4, c.device, s));
  SACD_CUDA_TRY(pool_alloc(&flag64, ne * 8, c.device, s));
  SACD_CUDA_TRY(pool_alloc(&idx, ne * 8, c.device, s));
  const long long nblk = (md.I > 0 ? (c.dims[md.a] + ablk_rows - 1) / ablk_rows : 1);
  const int end_bit = bits_for((unsigned long long)std::max(1LL, nblk - 1));
  k_block_keys<<<grid_for(nnz), 256, 0, s>>>(md.idx_a, nnz, ablk_rows, keys, pos);
  SACD_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, pos, perm, (int)nnz, 0, end_bit, s));
  SACD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb2, flag64, idx, (int)nnz, s));
  SACD_CUDA_TRY(pool_alloc(&temp, std::max(tb, tb2), c.device, s));
  SACD_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, tb, keys, keys2, pos, perm, (int)nnz, 0, end_bit, s));
  k_block_gather<<<grid_for(nnz), 256, 0, s>>>(perm, keys2, md.idx_a, md.idx_b, md.idx_n, md.val, nnz, md.nzm, flag);
  k_widen<<<grid_for(nnz), 256, 0, s>>>(flag, nnz, flag64);
  SACD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(temp, tb2, flag64, idx, (int)nnz, s));
  unsigned long long nseg = 0, last = 0;
  uint32_t lastf = 0;
  SACD_CUDA_TRY(cudaMemcpyAsync(&last, idx + nnz - 1, 8, cudaMemcpyDeviceToHost, s));
  SACD_CUDA_TRY(cudaMemcpyAsync(&lastf, flag + nnz - 1, 4, cudaMemcpyDeviceToHost, s));
  SACD_CUDA_TRY(cudaStreamSynchronize(s));
  nseg = last + lastf;
  SACD_CUDA_TRY(pool_alloc(&d_start, (size_t)nseg * 8, c.device, s));
  SACD_CUDA_TRY(pool_alloc(&d_row, (size_t)nseg * 4, c.device, s));
  k_seg_list<<<grid_for(nnz), 256, 0, s>>>(flag, idx, reinterpret_cast<const uint32_t *>(md.nzm), nnz, d_start,
                                           d_row);
  SACD_CUDA_TRY(cudaGetLastError());
  seg_start.resize(nseg);
  seg_row.resize(nseg);
  SACD_CUDA_TRY(cudaMemcpyAsync(seg_start.data(), d_start, (size_t)nseg * 8, cudaMemcpyDeviceToHost, s));
  SACD_CUDA_TRY(cudaMemcpyAsync(seg_row.data(), d_row, (size_t)nseg * 4, cudaMemcpyDeviceToHost, s));
  SACD_CUDA_TRY(cudaStreamSynchronize(s));
  cudaFreeAsync(keys, s);
  cudaFreeAsync(keys2, s);
  cudaFreeAsync(pos, s);
  cudaFreeAsync(perm, s);
  cudaFreeAsync(flag, s);
  cudaFreeAsync(flag64, s);
  cudaFreeAsync(idx, s);
  cudaFreeAsync(d_start, s);
  cudaFreeAsync(d_row, s);
  cudaFreeAsync(temp, s);
  SACD_CUDA_TRY(cudaStreamSynchronize(s));
  return SACD_OK;
}

int build_layouts(Context &c, const uint32_t *coords, const float *vals) {
  const long long nnz = c.nnz;
  cudaStream_t s = c.stream;
  int *flags = nullptr;
  InitTimer tm;
  SACD_CUDA_TRY(pool_alloc(&flags, 4 * sizeof(unsigned long long), c.device, s));  // flags | fiber counts [3]
  SACD_CUDA_TRY(cudaMemsetAsync(flags, 0, 4 * sizeof(unsigned long long), s));
  unsigned long long *nfib = reinterpret_cast<unsigned long long *>(flags) + 1;
  if (nnz > 0)
    k_validate<<<grid_for(nnz), 256, 0, s>>>(coords, vals, nnz, c.dims[0], c.dims[1], c.dims[2], flags);
  int hflags = 0;
  SACD_CUDA_TRY(cudaMemcpyAsync(&hflags, flags, sizeof(int), cudaMemcpyDeviceToHost, s));
  SACD_CUDA_TRY(cudaStreamSynchronize(s));
  if (hflags & 1) {
    set_error("sacd_init: coordinate index out of range");
    cudaFreeAsync(flags, s);
    return SACD_ERANGE;
  }
  if (hflags & 2) {
    set_error("sacd_init: non-finite value");
    cudaFreeAsync(flags, s);
    return SACD_ENONFINITE;
  }
  c.uniform_x = nnz > 0 && !(hflags & 8);
  if (c.uniform_x) {
    float x0 = 0.f;
    SACD_CUDA_TRY(cudaMemcpyAsync(&x0, vals, sizeof(float), cudaMemcpyDeviceToHost, s));
    SACD_CUDA_TRY(cudaStreamSynchronize(s));
    c.xu = (double)x0;
  }

  unsigned long long *keys = nullptr, *keys2 = nullptr;
  uint32_t *pos = nullptr, *pos2 = nullptr;
  void *temp = nullptr;
  size_t temp_bytes = 0;
  const size_t ne = (size_t)(nnz > 0 ? nnz : 1);
  SACD_CUDA_TRY(pool_alloc(&keys, ne * 8, c.device, s));
  SACD_CUDA_TRY(pool_alloc(&keys2, ne * 8, c.device, s));
  SACD_CUDA_TRY(pool_alloc(&pos, ne * 4, c.device, s));
  SACD_CUDA_TRY(pool_alloc(&pos2, ne * 4, c.device, s));
  if (nnz > 0) {
    SACD_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, keys2, pos, pos2, (int)nnz, 0, 64, s));
    SACD_CUDA_TRY(pool_alloc(&temp, temp_bytes, c.device, s));
  }
  for (int n = 0; n < 3; n++) {
    ModeData &md = c.m[n];
    const int a = md.a, b = md.b;
    const unsigned long long Ia = (unsigned long long)c.dims[a], Ib = (unsigned long long)c.dims[b];
    const bool soa = layout_needs_soa(c);
    if (soa) {
      SACD_CUDA_TRY(pool_alloc(&md.idx_a, ne * 4, c.device, s));
      SACD_CUDA_TRY(pool_alloc(&md.idx_b, ne * 4, c.device, s));
      SACD_CUDA_TRY(pool_alloc(&md.idx_n, ne * 4, c.device, s));
      SACD_CUDA_TRY(pool_alloc(&md.val, ne * 4, c.device, s));
    }
    SACD_CUDA_TRY(pool_alloc(&md.nzm, ne * 16, c.device, s));
    SACD_CUDA_TRY(pool_alloc(&md.row_ptr, (size_t)(md.I + 1) * 8, c.device, s));
    c.device_bytes += (long long)ne * (soa ? 32 : 16) + (md.I + 1) * 8;
    tm.mark(s, "  layout: allocations");
    if (nnz > 0) {
      k_make_keys<<<grid_for(nnz), 256, 0, s>>>(coords, nnz, n, a, b, Ia, Ib, keys, pos);
      tm.mark(s, "  layout: keys");
      const int end_bit = bits_for((unsigned long long)c.dims[n] * Ia * Ib - 1ULL);
      SACD_CUDA_TRY(
          cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys2, pos, pos2, (int)nnz, 0, end_bit, s));
      tm.mark(s, "  layout: radix sort");
      k_check_dup<<<grid_for(nnz), 256, 0, s>>>(keys2, nnz, flags);
      k_gather<<<grid_for(nnz), 256, 0, s>>>(coords, vals, pos2, keys2, nnz, a, b, Ib, Ia * Ib, md.idx_a, md.idx_b,
                                             md.idx_n, md.val, md.nzm, nfib + n);
      tm.mark(s, "  layout: dup check + gather");
    }
    k_row_ptr<<<grid_for(md.I + 1), 256, 0, s>>>(keys2, nnz, md.I, Ia * Ib, md.row_ptr);
    SACD_CUDA_TRY(cudaGetLastError());
    tm.mark(s, "  layout: row_ptr");
  }
  SACD_CUDA_TRY(cudaMemcpyAsync(&hflags, flags, sizeof(int), cudaMemcpyDeviceToHost, s));
  unsigned long long hfib[3] = {0, 0, 0};
  SACD_CUDA_TRY(cudaMemcpyAsync(hfib, nfib, sizeof(hfib), cudaMemcpyDeviceToHost, s));
  // ||X||^2 in mode-0 layout order
  double *part = nullptr;
  SACD_CUDA_TRY(pool_alloc(&part, kNormBlocks * sizeof(double), c.device, s));
  k_norm_partial<<<kNormBlocks, 256, 0, s>>>(c.m[0].nzm, nnz, part);  // mode-0 order, canonical here
  k_norm_final<<<1, 32, 0, s>>>(part, kNormBlocks, c.st);
  SACD_CUDA_TRY(cudaGetLastError());
  SACD_CUDA_TRY(cudaStreamSynchronize(s));
  cudaFreeAsync(part, s);
  cudaFreeAsync(keys, s);
  cudaFreeAsync(keys2, s);
  cudaFreeAsync(pos, s);
  cudaFreeAsync(pos2, s);
  if (temp) cudaFreeAsync(temp, s);
  cudaFreeAsync(flags, s);
  SACD_CUDA_TRY(cudaStreamSynchronize(s));
  if (hflags & 4) {
    set_error("sacd_init: duplicate coordinate");
    return SACD_EDUP;
  }
  for (int n = 0; n < 3; ++n) c.m[n].n_fibers = (long long)hfib[n];
  return SACD_OK;
}

}  // namespace sacd
