// k_pass.inc.cuh -- part of kernels.cu (included inside namespace sacd { namespace { ... } }).
// Pass records and the objective (A5), the delta exchange, the sharded-
// engine helper kernels and held-out evaluation (f3).
// Paper citations "P:n" are PAPER.md lines; readings Cn / L1 / C10' are DESIGN.md section 3.
// NOT a standalone header: it relies on the helpers defined at the top of kernels.cu.

// ------------------------------------------------------------------ per-sweep device time
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// First kernel of every sweep (eager or captured): the start time of the sweep.
__global__ void k_sweep_begin(DevState *st) {
  if (threadIdx.x == 0) st->t_begin = globaltimer_ns();
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
    rec.ms = (double)(globaltimer_ns() - st->t_begin) * 1e-6;
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

// ------------------------------------------------------------------ peer-memory exchange
// After the owner's row update, every 16-byte chunk of its owned rows [lo, hi) (element
// indices of the row-major factor) that differs bit for bit from the pass-start snapshot Fo
// is stored directly into every peer's replica at the same offset (NVLink stores through
// IPC-mapped pointers across processes; other shards' replicas with emulated ranks).  No
// lists, no counts on the host, no NCCL: the whole exchange is kernels, so the sweep graph
// captures it.  Unchanged chunks are already equal on every replica (all start equal and
// receive the same stores), so the replicas stay bitwise identical.
template <typename Real>
__global__ void __launch_bounds__(256) k_p2p_push(long long lo, long long hi, const Real *__restrict__ F,
                                                  const Real *__restrict__ Fo, Real *const *__restrict__ peers,
                                                  int G, int me) {
  constexpr int PER = 16 / (int)sizeof(Real);
  const long long c0 = lo / PER, c1 = hi / PER;  // lo, hi are whole rows (multiples of the pitch)
  const uint4 *Fc = reinterpret_cast<const uint4 *>(F);
  const uint4 *Oc = reinterpret_cast<const uint4 *>(Fo);
  for (long long k = c0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; k < c1;
       k += (long long)gridDim.x * blockDim.x) {
    const uint4 a = Fc[k], b = Oc[k];
    if (a.x != b.x || a.y != b.y || a.z != b.z || a.w != b.w) {
      for (int p = 0; p < G; ++p)
        if (p != me) reinterpret_cast<uint4 *>(peers[p])[k] = a;
    }
  }
}

// This rank has pushed its rows: make them visible system-wide, advance the pass counter and
// raise flag[me] = counter in every peer's flag array.
__global__ void k_p2p_signal(unsigned long long *const *__restrict__ peer_flags, int G, int me,
                             unsigned long long *__restrict__ epoch) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  const unsigned long long e = *epoch + 1;
  *epoch = e;
  for (int p = 0; p < G; ++p)
    if (p != me) {
      unsigned long long *f = peer_flags[p] + me;
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
    }
}

// Wait until every peer has raised its flag for this pass (flags live in this rank's memory);
// a peer that never arrives traps after ~20 s (a sticky ECUDA instead of a hang).
__global__ void k_p2p_wait(const unsigned long long *__restrict__ flags, int G, int me,
                           const unsigned long long *__restrict__ epoch) {
  if (threadIdx.x != 0) return;
  const unsigned long long e = *epoch;
  const unsigned long long t0 = globaltimer_ns();
  for (int p = 0; p < G; ++p) {
    if (p == me) continue;
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + p) : "memory");
      if (v >= e) break;
      if (globaltimer_ns() - t0 > 20000000000ULL) __trap();
      __nanosleep(200);
    }
  }
  __threadfence_system();
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
// Peer-memory exchange of the small per-rank slots (exchange = p2p): this rank's head
// partial (row id + row) into slot `me` of EVERY rank's exchange arrays (its own included),
// and its stats slot [ti, md, E, Ech, Gram] into every other rank's stats array.  A flag
// barrier (k_p2p_signal / k_p2p_wait) follows before anyone reads them, so a sweep needs no
// NCCL at all.
template <typename Real, int RT>
__global__ void k_pack_head_p2p(long long head, const Real *__restrict__ M, long long *const *__restrict__ ids,
                                Real *const *__restrict__ rows, int G, int me) {
  for (int p = 0; p < G; ++p) {
    for (int c = threadIdx.x; c < RT; c += blockDim.x) rows[p][(long long)me * RT + c] = head >= 0 ? M[head * RT + c] : Real(0);
    if (threadIdx.x == 0) ids[p][me] = head;
  }
}

__global__ void k_push_slot(const double *__restrict__ src, double *const *__restrict__ dst, long long count,
                            long long off, int G, int me) {
  for (int p = 0; p < G; ++p)
    if (p != me)
      for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < count; x += (long long)gridDim.x * blockDim.x)
        dst[p][off + x] = src[x];
}

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

