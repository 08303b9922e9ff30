// capi.cu -- the C ABI of libsacd (include/sacd.h): context lifetime, the MTTKRP work
// partition (host-side planning over row_ptr, done once at init), the sweep CUDA graph,
// teacher-forcing entry points and profiling.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include <nccl.h>

#include "sacd_internal.cuh"

struct sacd_ctx : public sacd::Context {};

namespace sacd {

static thread_local std::string g_err;
void set_error(const std::string &m) { g_err = m; }

// ------------------------------------------------------------------ profiling events
static int prof_flush(Context &c) {
  if (c.ev_pending.empty()) {
    c.ev_next = 0;
    return SACD_OK;
  }
  SACD_CUDA_TRY(cudaStreamSynchronize(c.stream));
  for (auto &p : c.ev_pending) {
    float ms = 0.f;
    SACD_CUDA_TRY(cudaEventElapsedTime(&ms, c.ev_pool[p.second], c.ev_pool[p.second + 1]));
    c.prof_ms[p.first] += ms;
    c.prof_n[p.first] += 1;
  }
  c.ev_pending.clear();
  c.ev_next = 0;
  return SACD_OK;
}

int prof_begin(Context &c, int kclass) {
  (void)kclass;
  if (!c.opt.profile) return -1;
  if (c.ev_next + 2 > 16384) {
    if (prof_flush(c) != SACD_OK) return -1;
  }
  while (c.ev_pool.size() < c.ev_next + 2) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    c.ev_pool.push_back(e);
  }
  const int idx = (int)c.ev_next;
  c.ev_next += 2;
  if (cudaEventRecord(c.ev_pool[idx], c.stream) != cudaSuccess) return -1;
  return idx;
}

int prof_end(Context &c, int kclass, int idx) {
  if (idx < 0) return SACD_OK;
  SACD_CUDA_TRY(cudaEventRecord(c.ev_pool[idx + 1], c.stream));
  c.ev_pending.push_back({kclass, idx});
  return SACD_OK;
}

// ------------------------------------------------------------------ slice sharding
// lower_bound over row_ptr[0..I]: first r with row_ptr[r] >= x
static long long lower_row(const long long *rp, long long I, long long x) {
  long long lo = 0, hi = I + 1;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (rp[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

ShardPlan plan_shard(const long long *rp, long long I, int world, int rank) {
  ShardPlan p;
  const long long nnz = rp[I];
  p.lo = (long long)((__int128)rank * nnz / world);
  p.hi = (long long)((__int128)(rank + 1) * nnz / world);
  p.rlo = std::min(lower_row(rp, I, p.lo), I);
  p.rhi = (rank == world - 1) ? I : std::min(lower_row(rp, I, p.hi), I);
  if (p.rhi < p.rlo) p.rhi = p.rlo;
  p.head = -1;
  if (p.lo < p.hi && (p.rlo >= I || rp[p.rlo] > p.lo)) p.head = p.rlo - 1;
  return p;
}

// ------------------------------------------------------------------ MTTKRP work partition
// Work items over the nonzero range [lo, hi) of one mode: whole rows with <= T local
// nonzeros in total and <= maxrows rows per item; a row with more than T local nonzeros,
// or one cut by the range boundary (sharded engine), is split into row-relative segments
// of T nonzeros, each writing a partial slot that k_fixup sums in slot order into M[row]
// (deterministic).  Rows without local nonzeros get no item: the row update reads row_ptr
// and uses m = 0 for empty slices.
static void build_items(const std::vector<long long> &rp, long long I, long long lo, long long hi, long long T,
                        long long maxrows, std::vector<WorkItem> &items, std::vector<SplitRow> &splits,
                        long long &nslots) {
  items.clear();
  splits.clear();
  nslots = 0;
  if (lo >= hi) return;
  // the row containing nonzero lo: rp[r] <= lo < rp[r+1]
  long long r = (long long)(std::upper_bound(rp.begin(), rp.begin() + I + 1, lo) - rp.begin()) - 1;
  while (r < I && rp[r] < hi) {
    const long long s0 = std::max(rp[r], lo), e0 = std::min(rp[r + 1], hi);
    const long long len = e0 - s0;
    if (len <= 0) {
      ++r;
      continue;
    }
    const bool clipped = rp[r] < lo || rp[r + 1] > hi;
    if (clipped || len > T) {
      const long long nseg = (len + T - 1) / T;
      SplitRow sr;
      sr.slot0 = nslots;
      sr.nslots = nseg;
      sr.row = (int)r;
      sr.chunk0 = 0;
      for (long long q = 0; q < nseg; ++q) {
        WorkItem w;
        w.nz0 = s0 + q * T;
        w.nz1 = std::min(s0 + (q + 1) * T, e0);
        w.row0 = (int)r;
        w.row1 = (int)(r + 1);
        w.slot = nslots++;
        items.push_back(w);
      }
      splits.push_back(sr);
      ++r;
      continue;
    }
    long long j = r, tot = 0;
    while (j < I && j - r < maxrows && rp[j] < hi) {
      const long long l = rp[j + 1] - rp[j];
      if (rp[j + 1] > hi || l > T) break;
      if (tot + l > T && j > r) break;
      tot += l;
      ++j;
    }
    WorkItem w;
    w.nz0 = rp[r];
    w.nz1 = rp[j];
    w.row0 = (int)r;
    w.row1 = (int)j;
    w.slot = -1;
    items.push_back(w);
    r = j;
  }
}

// Work items over the segments of an a-blocked execution order (layout.cu,
// build_blocked_order): every (blk, row) segment is cut into T-nonzero items, each writing
// a partial slot; a row's slots are contiguous and ordered by block, then by position, so
// the split-row fix-up sums the row in execution order (deterministic).
static void build_items_segments(const std::vector<long long> &seg_start, const std::vector<int> &seg_row,
                                 long long nnz, long long I, long long T, std::vector<WorkItem> &items,
                                 std::vector<SplitRow> &splits, long long &nslots) {
  items.clear();
  splits.clear();
  const size_t ns = seg_start.size();
  std::vector<long long> cnt((size_t)I, 0), slot0((size_t)I, 0), next((size_t)I, 0);
  for (size_t k = 0; k < ns; ++k) {
    const long long len = (k + 1 < ns ? seg_start[k + 1] : nnz) - seg_start[k];
    cnt[(size_t)seg_row[k]] += (len + T - 1) / T;
  }
  nslots = 0;
  for (long long r = 0; r < I; ++r) {
    slot0[(size_t)r] = nslots;
    if (cnt[(size_t)r] > 0) {
      SplitRow sr;
      sr.slot0 = nslots;
      sr.nslots = cnt[(size_t)r];
      sr.row = (int)r;
      sr.chunk0 = 0;
      splits.push_back(sr);
    }
    nslots += cnt[(size_t)r];
  }
  for (size_t k = 0; k < ns; ++k) {
    const long long e0 = seg_start[k], e1 = k + 1 < ns ? seg_start[k + 1] : nnz;
    const int r = seg_row[k];
    for (long long z = e0; z < e1; z += T) {
      WorkItem w;
      w.nz0 = z;
      w.nz1 = std::min(z + T, e1);
      w.row0 = r;
      w.row1 = r + 1;
      w.slot = slot0[(size_t)r] + next[(size_t)r]++;
      items.push_back(w);
    }
  }
}

// Does the selected MTTKRP kernel read the 16-byte nonzero records (nzm)?  Only those
// kernels can run an a-blocked execution order (the warp fiber kernel, variant 1, and the
// R <= 16 kernel read the canonical SoA arrays).
static bool mttkrp_reads_nzm(const Context &c) {
  if (c.pitch < 32 || c.opt.mttkrp_variant == 1) return false;
  return true;
}

// two-level fix-up plan of a split-row list (sets SplitRow::chunk0)
static void plan_fixup(std::vector<SplitRow> &splits, std::vector<FixChunk> &chunks) {
  chunks.clear();
  for (SplitRow &sr : splits) {
    const long long nch = (sr.nslots + kFixChunk - 1) / kFixChunk;
    sr.chunk0 = (int)chunks.size();
    for (long long q = 0; q < nch; ++q) {
      FixChunk fc;
      fc.slot0 = sr.slot0 + q * kFixChunk;
      fc.nslots = (int)std::min<long long>(kFixChunk, sr.nslots - q * kFixChunk);
      fc.out = nch == 1 ? -(sr.row + 1) : (int)chunks.size();
      chunks.push_back(fc);
    }
  }
}

template <typename T>
static int upload(T **dst, const std::vector<T> &v) {
  SACD_CUDA_TRY(cudaMalloc(dst, std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!v.empty()) SACD_CUDA_TRY(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return SACD_OK;
}

// Capture one sweep as a CUDA graph (replayed by sacd_iterate unless profiling), and count
// the libsacd kernels it launches (NCCL's own kernels excluded).
static int capture_graph(Context &c) {
  if (c.graph_exec) {
    cudaGraphExecDestroy(c.graph_exec);
    c.graph_exec = nullptr;
  }
  if (c.graph) {
    cudaGraphDestroy(c.graph);
    c.graph = nullptr;
  }
  const int saved_profile = c.opt.profile;
  c.opt.profile = 0;
  SACD_CUDA_TRY(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  int rc = SACD_OK;
  c.capturing = true;
  for (int n = 0; n < 3 && rc == SACD_OK; ++n)
    rc = c.sharded ? launch_sharded_mode_update(c, n, SACD_BR_AUTO, n == 0, n == 2, nullptr)
                   : launch_mode_update(c, n, SACD_BR_AUTO, n == 0, n == 2, nullptr);
  c.capturing = false;
  c.opt.profile = saved_profile;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(c.stream, &g);
  if (rc != SACD_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  SACD_CUDA_TRY(e);
  size_t nn = 0;
  SACD_CUDA_TRY(cudaGraphGetNodes(g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  if (nn) SACD_CUDA_TRY(cudaGraphGetNodes(g, nodes.data(), &nn));
  c.kernels_per_sweep = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nd, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp;
    const char *name = nullptr;
    if (cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess && cudaFuncGetName(&name, kp.func) == cudaSuccess &&
        name && strstr(name, "sacd"))
      c.kernels_per_sweep += 1;
  }
  cudaGetLastError();
  // the NCCL delta exchange reads the list lengths on the host: its sweeps run eagerly
  if (!c.opt.use_graph || (c.delta && c.comm)) {
    cudaGraphDestroy(g);
    return SACD_OK;
  }
  c.graph = g;
  SACD_CUDA_TRY(cudaGraphInstantiate(&c.graph_exec, c.graph, 0));
  return SACD_OK;
}

static int sweep_eager(Context &c) {
  for (int n = 0; n < 3; ++n)
    SACD_TRY(c.sharded ? launch_sharded_mode_update(c, n, SACD_BR_AUTO, n == 0, n == 2, nullptr)
                       : launch_mode_update(c, n, SACD_BR_AUTO, n == 0, n == 2, nullptr));
  return SACD_OK;
}

// The library's device memory pool (sacd_internal.cuh): one per device, created on first
// use, never destroyed (its memory is reused by every later context on that device).
cudaMemPool_t device_pool(int device) {
  static std::mutex mu;
  static std::vector<cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0) device = 0;
  if ((int)pools.size() <= device) pools.resize(device + 1, nullptr);
  if (!pools[device]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {  // fall back to the default pool
      cudaGetLastError();
      if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return nullptr;
    }
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    unsigned long long thr = total_b / 4;
    if (const char *e = getenv("SACD_POOL_RELEASE_MB")) thr = strtoull(e, nullptr, 10) << 20;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    cudaGetLastError();
    pools[device] = pool;
  }
  return pools[device];
}

static void destroy(sacd_ctx *c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  if (c->graph) cudaGraphDestroy(c->graph);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (int n = 0; n < 3; ++n) {
    ModeData &m = c->m[n];
    cudaFree(m.idx_a);
    cudaFree(m.idx_b);
    cudaFree(m.idx_n);
    cudaFree(m.val);
    cudaFree(m.nzm);
    cudaFree(m.row_ptr);
    cudaFree(m.items);
    cudaFree(m.splits);
    cudaFree(m.chunks);
    cudaFree(m.F);
    cudaFree(m.Z);
    cudaFree(m.G);
    cudaFree(m.cmask);
  }
  cudaFree(c->st);
  cudaFree(c->M);
  cudaFree(c->Zs);
  cudaFree(c->item_ctr);
  cudaFree(c->Fold);
  cudaFree(c->didx);
  cudaFree(c->dval);
  cudaFree(c->dcnt);
  cudaFree(c->dblk);
  cudaFree(c->partial);
  cudaFree(c->fixbuf);
  cudaFree(c->Hr);
  cudaFree(c->Hd);
  cudaFree(c->row_part);
  cudaFree(c->cnt_part);
  cudaFree(c->gram_part);
  cudaFree(c->decisions);
  for (Shard &sh : c->shards) {
    for (void *p : sh.ipc_opened) cudaIpcCloseMemHandle(p);
    for (int n = 0; n < 3; ++n) {
      cudaFree(sh.items[n]);
      cudaFree(sh.splits[n]);
      cudaFree(sh.chunks[n]);
      cudaFree(sh.d_peerF[n]);
      if (sh.own_rep) cudaFree(sh.Frep[n]);
    }
    cudaFree(sh.flags);
    cudaFree(sh.epoch);
    cudaFree(sh.d_peer_flags);
    cudaFree(sh.d_px);
    cudaFree(sh.d_pr);
    cudaFree(sh.d_ps);
    if (sh.xid_r && sh.xid_r != c->xid) {
      cudaFree(sh.xid_r);
      cudaFree(sh.xrow_r);
      cudaFree(sh.xstats_r);
    }
    cudaFree(sh.M);
    cudaFree(sh.partial);
    cudaFree(sh.row_part);
    cudaFree(sh.cnt_part);
    cudaFree(sh.gram_part);
  }
  cudaFree(c->xid);
  cudaFree(c->xrow);
  cudaFree(c->xstats);
  if (c->pin) cudaFreeHost(c->pin);
  for (auto e : c->pin_ev)
    if (e) cudaEventDestroy(e);
  if (c->comm) ncclCommDestroy(reinterpret_cast<ncclComm_t>(c->comm));
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;  // memory from the library's pool stays mapped there for the next context
}

// Layout key (i_n, i_a, i_b): a = the LONGER other mode (ties -> lower mode id), b = the
// shorter one, so the per-nonzero gathers hit the smaller, cache-resident factor and the
// per-fiber gathers the larger one (reading L1).
static int other_modes(const long long dims[3], int n, int *a, int *b) {
  const int o1 = (n + 1) % 3, o2 = (n + 2) % 3;
  const int lo = std::min(o1, o2), hi = std::max(o1, o2);
  if (dims[hi] > dims[lo]) {
    *a = hi;
    *b = lo;
  } else {
    *a = lo;
    *b = hi;
  }
  return 0;
}

#define CTX_CHECK(ctx)                                              \
  do {                                                              \
    if (!(ctx)) {                                                   \
      set_error("null context");                                    \
      return SACD_EINVAL;                                           \
    }                                                               \
    if ((ctx)->dead) {                                              \
      set_error("context is dead after a CUDA/NCCL error");         \
      return SACD_ECUDA;                                            \
    }                                                               \
    if (cudaSetDevice((ctx)->device) != cudaSuccess) {              \
      set_error("cudaSetDevice failed");                            \
      return SACD_ECUDA;                                            \
    }                                                               \
  } while (0)

// Any ECUDA/ENCCL result kills the context (sticky).
static int sticky(Context *c, int rc) {
  if (rc == SACD_ECUDA || rc == SACD_ENCCL) c->dead = true;
  return rc;
}

// Device-resident inputs may have been produced on any stream (e.g. PyTorch's current
// stream), which the context's non-blocking stream does not order against: synchronise the
// device before reading them.  Host inputs need nothing (the copies are from pageable or
// pinned memory the caller owns).
static int sync_if_device(const void *a, const void *b) {
  for (const void *p : {a, b}) {
    if (!p) continue;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();  // unregistered host memory on older drivers
      continue;
    }
    if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
      SACD_CUDA_TRY(cudaDeviceSynchronize());
      return SACD_OK;
    }
  }
  return SACD_OK;
}

// Peer-memory exchange (opt.reserved[3] = 2) setup, after the factors exist and hold the
// init: every shard's flags, pass counter and device arrays of the G ranks' replica pointers.
//  * emulated ranks: shard q > 0 gets its own replicas (copies of the init), so the pushes
//    of one shard into the others' replicas are real stores to other memory;
//  * NCCL ranks (one shard per process): the CUDA IPC handles of every rank's three factors
//    and flag array are all-gathered over NCCL and opened (NVLink peer mappings).
static int setup_p2p(Context *c) {
  const size_t rs = real_size(*c);
  cudaStream_t s = c->stream;
  const int G = c->G;
  const size_t xrow_bytes = (size_t)G * c->pitch * rs, xst_bytes = (size_t)G * (4 + (size_t)c->R * c->R) * 8;
  for (Shard &sh : c->shards) {
    if (sh.rank == c->shards[0].rank) {  // the context's own exchange arrays
      sh.xid_r = c->xid;
      sh.xrow_r = c->xrow;
      sh.xstats_r = c->xstats;
    } else {  // emulated ranks: every shard its own arrays
      SACD_CUDA_TRY(cudaMalloc(&sh.xid_r, (size_t)G * 8));
      SACD_CUDA_TRY(cudaMalloc(&sh.xrow_r, xrow_bytes));
      SACD_CUDA_TRY(cudaMalloc(&sh.xstats_r, xst_bytes));
    }
    SACD_CUDA_TRY(cudaMalloc(&sh.flags, (size_t)G * 8));
    SACD_CUDA_TRY(cudaMemsetAsync(sh.flags, 0, (size_t)G * 8, s));
    SACD_CUDA_TRY(cudaMalloc(&sh.epoch, 8));
    SACD_CUDA_TRY(cudaMemsetAsync(sh.epoch, 0, 8, s));
    for (int n = 0; n < 3; ++n) {
      if (c->opt.emulate_ranks > 1 && sh.rank > 0) {
        const size_t b = (size_t)c->m[n].I * c->pitch * rs;
        SACD_CUDA_TRY(cudaMalloc(&sh.Frep[n], b));
        SACD_CUDA_TRY(cudaMemcpyAsync(sh.Frep[n], c->m[n].F, b, cudaMemcpyDeviceToDevice, s));
        sh.own_rep = true;
        c->device_bytes += (long long)b;
      } else {
        sh.Frep[n] = c->m[n].F;
      }
    }
  }
  // host tables for every rank q: ptrF[q][n] (factor replicas), ptrX[q][k] (k = 0 flags,
  // 1 head ids, 2 head rows, 3 stats)
  constexpr int NH = 7;  // IPC handles per rank: 3 factors + 4 exchange arrays
  std::vector<void *> ptrF((size_t)G * 3, nullptr), ptrX((size_t)G * 4, nullptr);
  if (c->opt.emulate_ranks > 1 || G == 1) {
    for (Shard &sh : c->shards) {
      for (int n = 0; n < 3; ++n) ptrF[(size_t)sh.rank * 3 + n] = sh.Frep[n];
      ptrX[(size_t)sh.rank * 4 + 0] = sh.flags;
      ptrX[(size_t)sh.rank * 4 + 1] = sh.xid_r;
      ptrX[(size_t)sh.rank * 4 + 2] = sh.xrow_r;
      ptrX[(size_t)sh.rank * 4 + 3] = sh.xstats_r;
    }
  } else {
    Shard &sh = c->shards[0];
    cudaIpcMemHandle_t mine[NH];
    for (int n = 0; n < 3; ++n) SACD_CUDA_TRY(cudaIpcGetMemHandle(&mine[n], sh.Frep[n]));
    SACD_CUDA_TRY(cudaIpcGetMemHandle(&mine[3], sh.flags));
    SACD_CUDA_TRY(cudaIpcGetMemHandle(&mine[4], sh.xid_r));
    SACD_CUDA_TRY(cudaIpcGetMemHandle(&mine[5], sh.xrow_r));
    SACD_CUDA_TRY(cudaIpcGetMemHandle(&mine[6], sh.xstats_r));
    const size_t hb = sizeof(mine);
    char *dh = nullptr;
    SACD_CUDA_TRY(cudaMalloc(&dh, hb * G));
    SACD_CUDA_TRY(cudaMemcpyAsync(dh + hb * c->me, mine, hb, cudaMemcpyHostToDevice, s));
    const ncclResult_t r = ncclAllGather(dh + hb * c->me, dh, hb, ncclChar, reinterpret_cast<ncclComm_t>(c->comm), s);
    if (r != ncclSuccess) {
      set_error(std::string("ncclAllGather (IPC handles): ") + ncclGetErrorString(r));
      cudaFree(dh);
      return SACD_ENCCL;
    }
    std::vector<cudaIpcMemHandle_t> all((size_t)G * NH);
    SACD_CUDA_TRY(cudaMemcpyAsync(all.data(), dh, hb * G, cudaMemcpyDeviceToHost, s));
    SACD_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(dh);
    void *own[NH] = {sh.Frep[0], sh.Frep[1], sh.Frep[2], sh.flags, sh.xid_r, sh.xrow_r, sh.xstats_r};
    for (int q = 0; q < G; ++q) {
      for (int k = 0; k < NH; ++k) {
        void *ptr = nullptr;
        if (q == c->me) {
          ptr = own[k];
        } else {
          const cudaError_t e = cudaIpcOpenMemHandle(&ptr, all[(size_t)q * NH + k], cudaIpcMemLazyEnablePeerAccess);
          if (e != cudaSuccess) {
            cudaGetLastError();
            set_error(std::string("sacd_init: peer-memory exchange needs CUDA IPC / P2P between the ranks' GPUs (") +
                      cudaGetErrorString(e) + "); use the NCCL exchange (opt.reserved[3] = 0 or 1)");
            return SACD_ECUDA;
          }
          sh.ipc_opened.push_back(ptr);
        }
        if (k < 3) ptrF[(size_t)q * 3 + k] = ptr;
        else ptrX[(size_t)q * 4 + (k - 3)] = ptr;
      }
    }
  }
  for (Shard &sh : c->shards) {
    for (int n = 0; n < 3; ++n) {
      std::vector<void *> v((size_t)G);
      for (int q = 0; q < G; ++q) v[(size_t)q] = ptrF[(size_t)q * 3 + n];
      SACD_CUDA_TRY(cudaMalloc(&sh.d_peerF[n], (size_t)G * sizeof(void *)));
      SACD_CUDA_TRY(cudaMemcpy(sh.d_peerF[n], v.data(), (size_t)G * sizeof(void *), cudaMemcpyHostToDevice));
    }
    void **tabs[4] = {reinterpret_cast<void **>(&sh.d_peer_flags), reinterpret_cast<void **>(&sh.d_px),
                      reinterpret_cast<void **>(&sh.d_pr), reinterpret_cast<void **>(&sh.d_ps)};
    for (int k = 0; k < 4; ++k) {
      std::vector<void *> v((size_t)G);
      for (int q = 0; q < G; ++q) v[(size_t)q] = ptrX[(size_t)q * 4 + k];
      SACD_CUDA_TRY(cudaMalloc(tabs[k], (size_t)G * sizeof(void *)));
      SACD_CUDA_TRY(cudaMemcpy(*tabs[k], v.data(), (size_t)G * sizeof(void *), cudaMemcpyHostToDevice));
    }
  }
  SACD_CUDA_TRY(cudaStreamSynchronize(s));
  return SACD_OK;
}

// Copy factor `mode` (replica of shard 0) into the other shards' replicas (emulated ranks with
// the peer-memory exchange) after a host write (sacd_set_factors).
static int sync_replicas(Context *c, int mode) {
  if (!c->p2p) return SACD_OK;
  const size_t b = (size_t)c->m[mode].I * c->pitch * real_size(*c);
  for (Shard &sh : c->shards)
    if (sh.own_rep && sh.Frep[mode] != c->m[mode].F)
      SACD_CUDA_TRY(cudaMemcpyAsync(sh.Frep[mode], c->m[mode].F, b, cudaMemcpyDeviceToDevice, c->stream));
  return SACD_OK;
}

static int init_impl(Context *c, const uint32_t *coords, const float *vals, uint64_t seed) {
  const size_t rs = real_size(*c);
  cudaStream_t s = c->stream;
  InitTimer tm;
  SACD_TRY(sync_if_device(coords, vals));
  SACD_CUDA_TRY(cudaMalloc(&c->st, sizeof(DevState)));
  SACD_CUDA_TRY(cudaMemsetAsync(c->st, 0, sizeof(DevState), s));
  for (int n = 0; n < 3; ++n) {
    c->m[n].I = c->dims[n];
    other_modes(c->dims, n, &c->m[n].a, &c->m[n].b);
  }
  // tensor to device (host or device source; UVA picks the direction)
  uint32_t *dc = nullptr;
  float *dv = nullptr;
  const size_t ne = (size_t)(c->nnz > 0 ? c->nnz : 1);
  SACD_CUDA_TRY(pool_alloc(&dc, ne * 12, c->device, s));
  SACD_CUDA_TRY(pool_alloc(&dv, ne * 4, c->device, s));
  if (c->nnz > 0) {
    SACD_CUDA_TRY(cudaMemcpyAsync(dc, coords, (size_t)c->nnz * 12, cudaMemcpyDefault, s));
    SACD_CUDA_TRY(cudaMemcpyAsync(dv, vals, (size_t)c->nnz * 4, cudaMemcpyDefault, s));
  }
  tm.mark(s, "H2D copy of the COO");
  int rc = build_layouts(*c, dc, dv);
  cudaFreeAsync(dc, s);
  cudaFreeAsync(dv, s);
  SACD_TRY(rc);
  tm.mark(s, "layouts (sort, gather)");

  // partitions (host planning over row_ptr, once)
  // nonzeros per MTTKRP work item (measured on B200, profiles/r01_item_size_sweep.txt): enough
  // items to fill every SM several times over, else the launch idles while the last long
  // items finish.  1024 for the 1e8-nonzero c4 and for R > 64 (c5 R=256: 256-item runs lose
  // 2%); 256 for mid-size tensors (c2 0.25 -> 0.08 ms, c3 1.21 -> 1.08, c5 R=8/16 -14..16%)
  // and for a sharded rank (c4, 8 emulated ranks: 17.2 -> 13.2 ms summed); 64 under 1e5
  // nonzeros (c1 0.095 -> 0.041 ms).
  // T follows the nonzeros ONE rank processes (nnz / G): a sharded rank's launch then has
  // enough items to fill the GPU (c4 over 8 ranks: 256, 1.25e7 nonzeros each), and a one-rank
  // sharded run uses exactly the unsharded items, so it sums every row of M in the unsharded
  // order (bitwise equal results, test_sharded_nccl_world1_matches_unsharded).
  const long long nnz_rank = c->nnz / std::max(1, c->G);
  long long T = 1024;
  if (c->opt.nnz_per_item > 0) T = c->opt.nnz_per_item;
  else if (c->pitch >= 128 || nnz_rank >= 50000000LL) T = 1024;
  else if (nnz_rank < 100000) T = 64;
  else T = 256;
  long long max_slots = 1, maxI = 1, max_chunks = 1;
  std::vector<long long> rps[3];
  for (int n = 0; n < 3; ++n) {
    ModeData &md = c->m[n];
    rps[n].resize((size_t)md.I + 1);
    SACD_CUDA_TRY(cudaMemcpyAsync(rps[n].data(), md.row_ptr, rps[n].size() * 8, cudaMemcpyDeviceToHost, s));
    maxI = std::max(maxI, md.I);
  }
  SACD_CUDA_TRY(cudaStreamSynchronize(s));
  if (!c->sharded) {
    for (int n = 0; n < 3; ++n) {
      ModeData &md = c->m[n];
      std::vector<WorkItem> items;
      std::vector<SplitRow> splits;
      long long nslots = 0;
      // a-blocked execution order (opt.reserved[1] > 0: blocks of that many a-rows).  Off by
      // default: on c4's W mode (F_a = 512 MB, 1e4-nnz slices) it cut the launch's DRAM
      // reads from 13.7 to 10.8 GB but not its time (5.38 vs 5.40 ms): the per-nonzero
      // b-row gathers dominate there.
      long long ablk = 0;
      if (c->opt.reserved[1] > 0) ablk = c->opt.reserved[1];
      if (ablk > 0 && ablk < c->dims[md.a] && c->nnz > 0 && mttkrp_reads_nzm(*c)) {
        std::vector<long long> seg_start;
        std::vector<int> seg_row;
        SACD_TRY(build_blocked_order(*c, n, ablk, seg_start, seg_row));
        build_items_segments(seg_start, seg_row, c->nnz, md.I, T, items, splits, nslots);
        md.ablk_rows = ablk;
      } else {
        build_items(rps[n], md.I, 0, c->nnz, T, 32, items, splits, nslots);
      }
      md.n_items = (long long)items.size();
      md.n_splits = (long long)splits.size();
      md.n_slots = nslots;
      std::vector<FixChunk> chunks;
      plan_fixup(splits, chunks);
      md.n_chunks = (long long)chunks.size();
      max_chunks = std::max(max_chunks, md.n_chunks);
      SACD_TRY(upload(&md.items, items));
      SACD_TRY(upload(&md.splits, splits));
      SACD_TRY(upload(&md.chunks, chunks));
      max_slots = std::max(max_slots, nslots);
      c->device_bytes += (long long)(items.size() * sizeof(WorkItem) + splits.size() * sizeof(SplitRow));
    }
  } else {
    // sharded engine: plans of every rank, items of the local shard(s)
    for (int n = 0; n < 3; ++n) {
      c->all_plans[n].resize(c->G);
      for (int q = 0; q < c->G; ++q) c->all_plans[n][q] = plan_shard(rps[n].data(), c->m[n].I, c->G, q);
    }
    const int first = c->opt.emulate_ranks > 1 ? 0 : c->me;
    const int count = c->opt.emulate_ranks > 1 ? c->G : 1;
    c->shards.resize(count);
    for (int k = 0; k < count; ++k) {
      Shard &sh = c->shards[k];
      sh.rank = first + k;
      long long slots_k = 1;
      for (int n = 0; n < 3; ++n) {
        sh.plan[n] = c->all_plans[n][sh.rank];
        std::vector<WorkItem> items;
        std::vector<SplitRow> splits;
        long long nslots = 0;
        build_items(rps[n], c->m[n].I, sh.plan[n].lo, sh.plan[n].hi, T, 32, items, splits, nslots);
        sh.n_items[n] = (long long)items.size();
        sh.n_splits[n] = (long long)splits.size();
        std::vector<FixChunk> chunks;
        plan_fixup(splits, chunks);
        sh.n_chunks[n] = (long long)chunks.size();
        max_chunks = std::max(max_chunks, sh.n_chunks[n]);
        SACD_TRY(upload(&sh.items[n], items));
        SACD_TRY(upload(&sh.splits[n], splits));
        SACD_TRY(upload(&sh.chunks[n], chunks));
        slots_k = std::max(slots_k, nslots);
        c->m[n].n_items += sh.n_items[n];
        c->m[n].n_splits += sh.n_splits[n];
      }
      SACD_CUDA_TRY(cudaMalloc(&sh.M, (size_t)((maxI + 31) / 32 * 32) * c->pitch * rs));
      SACD_CUDA_TRY(cudaMalloc(&sh.partial, (size_t)slots_k * c->pitch * rs));
      c->max_slots = std::max(c->max_slots, slots_k);
      c->device_bytes += (long long)((size_t)maxI * c->pitch * rs + (size_t)slots_k * c->pitch * rs);
    }
    // NCCL communicator (one rank per process; emulated ranks need none)
    if (c->opt.emulate_ranks <= 1) {
      ncclUniqueId id;
      if (c->world > 1) {
        if (!c->opt.nccl_unique_id) {
          set_error("sacd_init: world_size > 1 needs opt.nccl_unique_id (sacd_nccl_unique_id on rank 0)");
          return SACD_EINVAL;
        }
        memcpy(&id, c->opt.nccl_unique_id, sizeof(id));
      } else {
        const ncclResult_t r = ncclGetUniqueId(&id);
        if (r != ncclSuccess) {
          set_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
          return SACD_ENCCL;
        }
      }
      ncclComm_t comm;
      const ncclResult_t r = ncclCommInitRank(&comm, c->world, id, c->me);
      if (r != ncclSuccess) {
        set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        return SACD_ENCCL;
      }
      c->comm = comm;
    }
  }
  // factors, z_prev, Grams, scratch
  const int P = c->pitch, R = c->R;
  for (int n = 0; n < 3; ++n) {
    ModeData &md = c->m[n];
    SACD_CUDA_TRY(cudaMalloc(&md.F, (size_t)md.I * P * rs));
    const size_t zrows = (size_t)((md.I + 31) / 32 * 32);
    SACD_CUDA_TRY(pool_alloc(&md.Z, zrows * P * rs, c->device, s));
    SACD_CUDA_TRY(cudaMemsetAsync(md.Z, 0, zrows * P * rs, s));
    SACD_CUDA_TRY(cudaMalloc(&md.G, (size_t)R * R * 8));
    SACD_CUDA_TRY(cudaMalloc(&md.cmask, (size_t)std::max(1LL, md.I) * 4));
    SACD_CUDA_TRY(cudaMemsetAsync(md.cmask, 0, (size_t)std::max(1LL, md.I) * 4, s));
    c->device_bytes += (long long)(2 * (size_t)md.I * P * rs + (size_t)R * R * 8);
  }
  c->max_row_blocks = (maxI + 31) / 32 + 1;  // >= ceil(I / rows_per_block) for every pitch
  // delta exchange buffers: list slot q holds up to rank q's owned elements
  c->delta = c->sharded && c->opt.reserved[3] == 1 && (double)maxI * P < 4294967295.0;
  c->p2p = c->sharded && c->opt.reserved[3] == 2;
  if (c->p2p && !c->Fold) {  // pass-start snapshot of the owned rows (change detection)
    SACD_CUDA_TRY(cudaMalloc(&c->Fold, (size_t)maxI * P * rs));
    c->device_bytes += (long long)((size_t)maxI * P * rs);
  }
  if (c->delta) {
    c->doff.assign(c->G, 0);
    c->dcap.assign(c->G, 0);
    long long tot = 0;
    for (int q = 0; q < c->G; ++q) {
      long long cap = 1;
      for (int n = 0; n < 3; ++n)
        cap = std::max(cap, (c->all_plans[n][q].rhi - c->all_plans[n][q].rlo) * (long long)P);
      c->doff[q] = tot;
      c->dcap[q] = cap;
      tot += cap;
    }
    SACD_CUDA_TRY(cudaMalloc(&c->Fold, (size_t)maxI * P * rs));
    SACD_CUDA_TRY(cudaMalloc(&c->didx, (size_t)tot * 4));
    SACD_CUDA_TRY(cudaMalloc(&c->dval, (size_t)tot * rs));
    SACD_CUDA_TRY(cudaMalloc(&c->dcnt, (size_t)c->G * 8));
    SACD_CUDA_TRY(cudaMalloc(&c->dblk, (size_t)kDeltaBlocks * 4));
    SACD_CUDA_TRY(cudaMemset(c->dcnt, 0, (size_t)c->G * 8));
    c->device_bytes += (long long)((size_t)maxI * P * rs + (size_t)tot * (4 + rs));
  }
  // row ranges of the Gram partials: at most 148 for the DMMA kernel (one per SM per panel
  // pair; the fixed-order reduce then reads half as many partials: c4 0.73 -> 0.57 ms per
  // sweep in eager timing vs 296) and 296 for the FMA kernel; at least 64 rows each, and at
  // least 2048 for fp64 R > 64 (36 / 10 panel pairs already fill the GPU: c5 R=256 Gram
  // 0.35 -> 0.22 ms, R=128 0.19 -> 0.16)
  const long long gcap = (c->opt.precision == SACD_F64 && c->pitch >= 32) ? 148 : 296;
  const long long grows = (c->opt.precision == SACD_F64 && c->pitch >= 128) ? 2048 : 64;
  c->gram_blocks = (int)std::min<long long>(gcap, std::max<long long>(1, (maxI + grows - 1) / grows));
  if (getenv("SACD_GRAM_BLOCKS")) c->gram_blocks = std::max(1, atoi(getenv("SACD_GRAM_BLOCKS")));  // tuning
  SACD_CUDA_TRY(pool_alloc(&c->M, (size_t)((maxI + 31) / 32 * 32) * P * rs, c->device, s));
  SACD_CUDA_TRY(cudaMalloc(&c->item_ctr, 2 * sizeof(unsigned long long)));  // MTTKRP items, row blocks
  SACD_CUDA_TRY(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  if (c->opt.variant == SACD_VARIANT_SNAPSHOT) {  // snapshot importances of one pass (TT layout)
    SACD_CUDA_TRY(pool_alloc(&c->Zs, (size_t)((maxI + 31) / 32 * 32) * P * rs, c->device, s));
    c->device_bytes += (long long)((size_t)((maxI + 31) / 32 * 32) * P * rs);
  }
  SACD_CUDA_TRY(pool_alloc(&c->partial, (size_t)max_slots * P * rs, c->device, s));
  SACD_CUDA_TRY(pool_alloc(&c->fixbuf, (size_t)max_chunks * P * rs, c->device, s));
  // sharded ranks write their own partial buffers (>= their slots); c->max_slots keeps the
  // smallest buffer any launch may index (debug bounds)
  c->max_slots = c->sharded ? c->max_slots : max_slots;
  c->max_chunks = max_chunks;
  c->device_bytes += (long long)((size_t)max_chunks * P * rs);
  SACD_CUDA_TRY(cudaMalloc(&c->Hr, (size_t)P * P * rs));
  SACD_CUDA_TRY(cudaMalloc(&c->Hd, (size_t)R * R * 8));
  SACD_CUDA_TRY(cudaMalloc(&c->row_part, (size_t)c->max_row_blocks * 2 * 8));
  SACD_CUDA_TRY(cudaMalloc(&c->cnt_part, (size_t)c->max_row_blocks * 2 * 8));
  // Gram partials: the separate Gram kernel's row ranges, or one per CTA of the row update
  // with the fused Gram (at most 4 resident CTAs per SM)
  c->gram_cap = (c->opt.precision == SACD_F64 && c->pitch <= 64) ? std::max(c->gram_blocks, 4 * std::max(1, c->num_sms))
                                                                 : c->gram_blocks;
  SACD_CUDA_TRY(cudaMalloc(&c->gram_part, (size_t)c->gram_cap * R * R * 8));
  c->device_bytes += (long long)((size_t)maxI * P * rs + (size_t)max_slots * P * rs + (size_t)P * P * rs +
                                 (size_t)c->max_row_blocks * 32 + (size_t)c->gram_cap * R * R * 8 +
                                 sizeof(DevState));
  if (c->sharded) {
    for (Shard &sh : c->shards) {
      SACD_CUDA_TRY(cudaMalloc(&sh.row_part, (size_t)c->max_row_blocks * 2 * 8));
      SACD_CUDA_TRY(cudaMalloc(&sh.cnt_part, (size_t)c->max_row_blocks * 2 * 8));
      SACD_CUDA_TRY(cudaMalloc(&sh.gram_part, (size_t)c->gram_cap * R * R * 8));
    }
    SACD_CUDA_TRY(cudaMalloc(&c->xid, (size_t)c->G * 8));
    SACD_CUDA_TRY(cudaMalloc(&c->xrow, (size_t)c->G * P * rs));
    SACD_CUDA_TRY(cudaMalloc(&c->xstats, (size_t)c->G * (4 + (size_t)R * R) * 8));
  }
  tm.mark(s, "work items, buffers");
  SACD_TRY(launch_setup(*c));
  SACD_TRY(launch_init_factors(*c, seed));
  if (c->p2p) SACD_TRY(setup_p2p(c));
  for (int n = 0; n < 3; ++n) SACD_TRY(launch_gram(*c, n));
  SACD_TRY(c->sharded ? launch_sharded_initial_fit(*c) : launch_initial_fit(*c));
  SACD_CUDA_TRY(cudaStreamSynchronize(s));
  tm.mark(s, "init factors, Grams, f^0");
  SACD_TRY(capture_graph(*c));
  SACD_CUDA_TRY(cudaStreamSynchronize(s));
  tm.mark(s, "graph capture");
  return SACD_OK;
}

template <typename T>
static int dev_read(Context *c, T *dst, const void *src, size_t bytes) {
  SACD_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  SACD_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SACD_OK;
}

// Host copy of `rows` rows of R doubles (src dense, row stride R) into dst (row stride ld),
// split over up to 8 threads: the destination is usually fresh pageable memory whose page
// faults dominate a single-threaded copy.
static void host_rows_copy(double *dst, long long ld, const double *src, long long rows, int R) {
  const size_t bytes = (size_t)rows * R * 8;
  const int nt = (int)std::max<size_t>(1, std::min<size_t>(8, bytes >> 22));  // >= 4 MB per thread
  auto part = [&](int t) {
    const long long r0 = rows * t / nt, r1 = rows * (t + 1) / nt;
    if (ld == R) {
      memcpy(dst + r0 * ld, src + r0 * R, (size_t)(r1 - r0) * R * 8);
    } else {
      for (long long r = r0; r < r1; ++r) memcpy(dst + r * ld, src + r * R, (size_t)R * 8);
    }
  };
  if (nt == 1) {
    part(0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(part, t);
  part(0);
  for (auto &x : th) x.join();
}

static bool is_pinned_host(const void *p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// factor-like matrix (Real, pitch) -> host fp64 with leading dimension ld.  Pinned `out`:
// one 2D copy.  Pageable `out`: through the context's pinned ring of two chunks, the D2H copy
// of chunk i + 1 overlapping the multi-threaded host copy of chunk i (the copy engine then
// runs at pinned bandwidth instead of the driver's single staging path for pageable memory).
static int read_matrix(Context *c, const void *src, long long rows, double *out, long long ld, bool ttl = false) {
  double *tmp = nullptr;
  cudaStream_t s = c->stream;
  SACD_CUDA_TRY(pool_alloc(&tmp, (size_t)std::max(1LL, rows) * c->R * 8, c->device, s));
  int rc = launch_convert_out(*c, src, rows, tmp, ttl);
  const size_t row_bytes = (size_t)c->R * 8;
  const size_t total = (size_t)rows * row_bytes;
  auto fail = [&](cudaError_t e) {
    set_error(std::string("read_matrix: ") + cudaGetErrorString(e));
    rc = SACD_ECUDA;
  };
  if (rc == SACD_OK && (total < (8u << 20) || is_pinned_host(out))) {
    cudaError_t e = cudaMemcpy2DAsync(out, (size_t)ld * 8, tmp, row_bytes, row_bytes, (size_t)rows,
                                      cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) fail(e);
  } else if (rc == SACD_OK) {
    if (!c->pin) {
      c->pin_chunk = (size_t)32 << 20;
      cudaError_t e = cudaHostAlloc(&c->pin, 2 * c->pin_chunk, cudaHostAllocDefault);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->pin_ev[0], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->pin_ev[1], cudaEventDisableTiming);
      if (e != cudaSuccess) {
        fail(e);
        c->pin = nullptr;
      }
    }
    const long long crow = std::max<long long>(1, (long long)(c->pin_chunk / row_bytes));
    const long long nch = (rows + crow - 1) / crow;
    auto issue = [&](long long k) {
      const long long r0 = k * crow, r1 = std::min(rows, r0 + crow);
      char *buf = reinterpret_cast<char *>(c->pin) + (size_t)(k & 1) * c->pin_chunk;
      cudaError_t e = cudaMemcpyAsync(buf, tmp + r0 * c->R, (size_t)(r1 - r0) * row_bytes, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaEventRecord(c->pin_ev[k & 1], s);
      if (e != cudaSuccess) fail(e);
    };
    if (rc == SACD_OK && nch > 0) issue(0);
    for (long long k = 0; rc == SACD_OK && k < nch; ++k) {
      cudaError_t e = cudaEventSynchronize(c->pin_ev[k & 1]);
      if (e != cudaSuccess) {
        fail(e);
        break;
      }
      if (k + 1 < nch) issue(k + 1);  // into the other half, while this one is copied out
      const long long r0 = k * crow, r1 = std::min(rows, r0 + crow);
      host_rows_copy(out + r0 * ld, ld, reinterpret_cast<const double *>(reinterpret_cast<char *>(c->pin) +
                                                                          (size_t)(k & 1) * c->pin_chunk),
                     r1 - r0, c->R);
    }
  }
  cudaFreeAsync(tmp, s);
  if (rc == SACD_OK) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) fail(e);
  }
  return rc;
}

static int write_matrix(Context *c, void *dst, long long rows, const double *in, long long ld, bool ttl = false) {
  double *tmp = nullptr;
  cudaStream_t s = c->stream;
  SACD_CUDA_TRY(pool_alloc(&tmp, (size_t)std::max(1LL, rows) * c->R * 8, c->device, s));
  cudaError_t e = cudaMemcpy2DAsync(tmp, (size_t)c->R * 8, in, (size_t)ld * 8, (size_t)c->R * 8, (size_t)rows,
                                    cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) {
    set_error(std::string("write_matrix: ") + cudaGetErrorString(e));
    return SACD_ECUDA;
  }
  int rc = launch_convert_in(*c, tmp, rows, dst, ttl);
  cudaFreeAsync(tmp, s);
  if (rc == SACD_OK) {
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      set_error(std::string("write_matrix: ") + cudaGetErrorString(e));
      rc = SACD_ECUDA;
    }
  }
  return rc;
}

}  // namespace sacd

using namespace sacd;

extern "C" {

const char *sacd_last_error(void) { return g_err.c_str(); }

void sacd_default_options(sacd_options *o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(sacd_options);
  o->precision = SACD_F64;
  o->l_mode = SACD_L_DIAG;
  o->variant = SACD_VARIANT_GS_LAGGED;
  o->device = -1;
  o->world_size = 1;
  o->rank = 0;
  o->use_graph = 1;
}

int sacd_init(sacd_ctx **out, const uint32_t *coords, const float *vals, int64_t nnz, const int64_t dims[3],
              int32_t rank, uint64_t seed, const sacd_options *opt) {
  if (!out || !dims) {
    set_error("sacd_init: null argument");
    return SACD_EINVAL;
  }
  *out = nullptr;
  sacd_options o;
  sacd_default_options(&o);
  if (opt) {
    if (opt->struct_size != sizeof(sacd_options)) {
      set_error("sacd_init: options struct_size mismatch");
      return SACD_EINVAL;
    }
    o = *opt;
  }
  if (nnz < 0 || nnz > 2000000000LL || rank < 1 || rank > 256 || (nnz > 0 && (!coords || !vals))) {
    set_error("sacd_init: bad nnz/rank/pointers");
    return SACD_EINVAL;
  }
  for (int n = 0; n < 3; ++n)
    if (dims[n] < 1 || dims[n] >= (1LL << 30)) {
      set_error("sacd_init: dims must be in [1, 2^30)");
      return SACD_EINVAL;
    }
  if ((double)dims[0] * (double)dims[1] * (double)dims[2] >= 1.8e19) {
    set_error("sacd_init: Q*P*S must fit in 64 bits");
    return SACD_EINVAL;
  }
  if ((o.precision != SACD_F64 && o.precision != SACD_F32) || (o.l_mode != SACD_L_DIAG && o.l_mode != SACD_L_FROB) ||
      o.variant < SACD_VARIANT_GS_LAGGED || o.variant > SACD_VARIANT_SNAPSHOT) {
    set_error("sacd_init: bad option value");
    return SACD_EINVAL;
  }
  if (o.variant >= SACD_VARIANT_JACOBI && (o.world_size > 1 || o.emulate_ranks > 1 || o.force_sharded)) {
    set_error("sacd_init: the JACOBI / SNAPSHOT variants run unsharded only");
    return SACD_EINVAL;
  }
#ifndef SACD_TUNING
  if (o.mttkrp_variant != 0) {
    set_error("sacd_init: mttkrp_variant != 0 needs the tuning build (libsacd_tuning.so, -DSACD_TUNING)");
    return SACD_EINVAL;
  }
#else
  {
    // every tuning variant that has a kernel for this precision / pitch (others would launch
    // no MTTKRP at all and leave M stale)
    const int v = o.mttkrp_variant;
    int p = 8;
    while (p < rank) p <<= 1;
    const bool f64 = o.precision == SACD_F64;
    const bool ok = v == 0 || (p >= 32 && (v == 1 || (v >= 10 && v <= 15) || (v >= 20 && v <= 49 && (v != 39 || f64)) ||
                                           (v >= 50 && v <= 69 && f64 && p == 64)));
    if (!ok) {
      set_error("sacd_init: mttkrp_variant has no kernel for this precision / rank");
      return SACD_EINVAL;
    }
  }
#endif
  if (o.reserved[3] < 0 || o.reserved[3] > 2) {
    set_error("sacd_init: exchange (reserved[3]) must be 0 (rows), 1 (delta lists) or 2 (peer memory)");
    return SACD_EINVAL;
  }
  if (o.world_size < 1 || o.rank < 0 || o.rank >= o.world_size || o.emulate_ranks < 0 ||
      (o.emulate_ranks > 1 && o.world_size != 1)) {
    set_error("sacd_init: bad world_size / rank / emulate_ranks");
    return SACD_EINVAL;
  }
  sacd_ctx *c = new (std::nothrow) sacd_ctx();
  if (!c) {
    set_error("sacd_init: host allocation failed");
    return SACD_ENOMEM;
  }
  c->opt = o;
  if (o.device >= 0) {
    c->device = o.device;
  } else if (cudaGetDevice(&c->device) != cudaSuccess) {
    set_error("sacd_init: no CUDA device");
    delete c;
    return SACD_ECUDA;
  }
  if (cudaSetDevice(c->device) != cudaSuccess) {
    set_error("sacd_init: cudaSetDevice failed");
    delete c;
    return SACD_ECUDA;
  }
  for (int n = 0; n < 3; ++n) c->dims[n] = dims[n];
  c->nnz = nnz;
  c->world = o.world_size;
  c->me = o.rank;
  c->sharded = o.world_size > 1 || o.force_sharded || o.emulate_ranks > 1;
  c->G = o.emulate_ranks > 1 ? o.emulate_ranks : o.world_size;
  c->R = rank;
  int p = 8;
  while (p < rank) p <<= 1;
  c->pitch = p;
  if (o.stream) {
    c->stream = (cudaStream_t)o.stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      set_error("sacd_init: stream creation failed");
      delete c;
      return SACD_ECUDA;
    }
    c->own_stream = true;
  }
  const int rc = init_impl(c, coords, vals, seed);
  if (rc != SACD_OK) {
    destroy(c);
    return rc;
  }
  *out = c;
  return SACD_OK;
}

int sacd_iterate(sacd_ctx *c, int32_t n) {
  CTX_CHECK(c);
  if (n < 0) {
    set_error("sacd_iterate: n < 0");
    return SACD_EINVAL;
  }
  for (int i = 0; i < n; ++i) {
    if (c->graph_exec && !c->opt.profile) {
      cudaError_t e = cudaGraphLaunch(c->graph_exec, c->stream);
      if (e != cudaSuccess) {
        set_error(std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
        return sticky(c, SACD_ECUDA);
      }
    } else {
      const int rc = sweep_eager(*c);
      if (rc != SACD_OK) return sticky(c, rc);
    }
  }
  return SACD_OK;
}

int sacd_sync(sacd_ctx *c) {
  CTX_CHECK(c);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    set_error(std::string("sacd_sync: ") + cudaGetErrorString(e));
    return sticky(c, SACD_ECUDA);
  }
  return SACD_OK;
}

int sacd_fit(sacd_ctx *c, double *objective, double *fit) {
  CTX_CHECK(c);
  double v[2];
  const int rc = dev_read(c, v, reinterpret_cast<const char *>(c->st) + offsetof(DevState, f), sizeof(v));
  if (rc != SACD_OK) return sticky(c, rc);
  if (objective) *objective = v[0];
  if (fit) *fit = v[1];
  return SACD_OK;
}

int sacd_factors(sacd_ctx *c, int32_t mode, double *out, int64_t ld) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2 || ld < c->R || !out) {
    set_error("sacd_factors: bad mode/ld/out");
    return SACD_ESTATE;
  }
  return sticky(c, read_matrix(c, c->m[mode].F, c->m[mode].I, out, ld));
}

int sacd_replica_factors(sacd_ctx *c, int32_t shard, int32_t mode, double *out, int64_t ld) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2 || ld < c->R || !out || shard < 0 || shard >= (int)c->shards.size()) {
    set_error("sacd_replica_factors: bad shard/mode/ld/out");
    return SACD_ESTATE;
  }
  const Shard &sh = c->shards[(size_t)shard];
  const void *src = (c->p2p && sh.Frep[mode]) ? sh.Frep[mode] : c->m[mode].F;
  return sticky(c, read_matrix(c, src, c->m[mode].I, out, ld));
}

int sacd_get_zprev(sacd_ctx *c, int32_t mode, double *out, int64_t ld) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2 || ld < c->R || !out) {
    set_error("sacd_get_zprev: bad mode/ld/out");
    return SACD_ESTATE;
  }
  return sticky(c, read_matrix(c, c->m[mode].Z, c->m[mode].I, out, ld, true));
}

int sacd_set_zprev(sacd_ctx *c, int32_t mode, const double *in, int64_t ld) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2 || ld < c->R || !in) {
    set_error("sacd_set_zprev: bad mode/ld/in");
    return SACD_ESTATE;
  }
  return sticky(c, write_matrix(c, c->m[mode].Z, c->m[mode].I, in, ld, true));
}

int sacd_set_factors(sacd_ctx *c, int32_t mode, const double *in, int64_t ld) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2 || ld < c->R || !in) {
    set_error("sacd_set_factors: bad mode/ld/in");
    return SACD_ESTATE;
  }
  int rc = write_matrix(c, c->m[mode].F, c->m[mode].I, in, ld);
  if (rc == SACD_OK) rc = sync_replicas(c, mode);
  if (rc == SACD_OK) rc = launch_gram(*c, mode);
  if (rc == SACD_OK && cudaStreamSynchronize(c->stream) != cudaSuccess) rc = SACD_ECUDA;
  return sticky(c, rc);
}

// held-out evaluation: predictions (out) and / or RMSE at n coordinates (host or device)
static int eval_impl(Context *c, const uint32_t *coords, const float *vals, long long n, double *out,
                     double *rmse) {
  cudaStream_t s = c->stream;
  const size_t nn = (size_t)std::max(1LL, n), nb = (size_t)std::max(1LL, (n + 7) / 8);
  uint32_t *dc = nullptr;
  float *dv = nullptr;
  double *dout = nullptr, *part = nullptr, *sse = nullptr;
  int *flag = nullptr;
  int rc = sync_if_device(coords, vals), hflag = 0;
  if (rc != SACD_OK) return rc;
  double hsse = 0.0;
  auto ck = [&](cudaError_t e) {
    if (e != cudaSuccess && rc == SACD_OK) {
      set_error(std::string("sacd_predict/rmse: ") + cudaGetErrorString(e));
      rc = e == cudaErrorMemoryAllocation ? SACD_ENOMEM : SACD_ECUDA;
    }
    return rc == SACD_OK;
  };
  if (ck(pool_alloc(&dc, nn * 12, c->device, s)) && ck(pool_alloc(&dout, nn * 8, c->device, s)) &&
      ck(pool_alloc(&part, nb * 8, c->device, s)) && ck(pool_alloc(&sse, 8, c->device, s)) && ck(pool_alloc(&flag, 4, c->device, s)) &&
      (!vals || ck(pool_alloc(&dv, nn * 4, c->device, s))) && ck(cudaMemsetAsync(flag, 0, 4, s)) &&
      (n == 0 || ck(cudaMemcpyAsync(dc, coords, (size_t)n * 12, cudaMemcpyDefault, s))) &&
      (!vals || n == 0 || ck(cudaMemcpyAsync(dv, vals, (size_t)n * 4, cudaMemcpyDefault, s)))) {
    rc = launch_range_check(*c, dc, n, flag);
    if (rc == SACD_OK && ck(cudaMemcpyAsync(&hflag, flag, 4, cudaMemcpyDeviceToHost, s)) &&
        ck(cudaStreamSynchronize(s))) {
      if (hflag) {
        set_error("sacd_predict/rmse: coordinate index out of range");
        rc = SACD_ERANGE;
      } else {
        rc = launch_predict(*c, dc, n, dv, out ? dout : nullptr, part, rmse ? sse : nullptr);
        if (rc == SACD_OK && out && n > 0) ck(cudaMemcpyAsync(out, dout, (size_t)n * 8, cudaMemcpyDefault, s));
        if (rc == SACD_OK && rmse) ck(cudaMemcpyAsync(&hsse, sse, 8, cudaMemcpyDeviceToHost, s));
        if (rc == SACD_OK) ck(cudaStreamSynchronize(s));
        if (rc == SACD_OK && rmse) *rmse = n > 0 ? sqrt(hsse / (double)n) : 0.0;
      }
    }
  }
  cudaFreeAsync(dc, s);
  cudaFreeAsync(dv, s);
  cudaFreeAsync(dout, s);
  cudaFreeAsync(part, s);
  cudaFreeAsync(sse, s);
  cudaFreeAsync(flag, s);
  cudaStreamSynchronize(s);
  return rc;
}

int sacd_predict(sacd_ctx *c, const uint32_t *coords, int64_t n, double *out) {
  CTX_CHECK(c);
  if (n < 0 || (n > 0 && (!coords || !out))) {
    set_error("sacd_predict: bad n / null pointer");
    return SACD_EINVAL;
  }
  const int rc = eval_impl(c, coords, nullptr, n, out, nullptr);
  return rc == SACD_ERANGE ? rc : sticky(c, rc);
}

int sacd_rmse(sacd_ctx *c, const uint32_t *coords, const float *vals, int64_t n, double *rmse) {
  CTX_CHECK(c);
  if (n < 0 || !rmse || (n > 0 && (!coords || !vals))) {
    set_error("sacd_rmse: bad n / null pointer");
    return SACD_EINVAL;
  }
  const int rc = eval_impl(c, coords, vals, n, nullptr, rmse);
  return rc == SACD_ERANGE ? rc : sticky(c, rc);
}

int sacd_mttkrp(sacd_ctx *c, int32_t mode, double *out, int64_t ld) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2 || ld < c->R || !out) {
    set_error("sacd_mttkrp: bad mode/ld/out");
    return SACD_ESTATE;
  }
  // empty slices are not written by the MTTKRP kernel: clear M first for this entry point
  cudaError_t e =
      cudaMemsetAsync(c->M, 0, (size_t)((c->m[mode].I + 31) / 32 * 32) * c->pitch * real_size(*c), c->stream);
  if (e != cudaSuccess) {
    set_error(std::string("sacd_mttkrp: ") + cudaGetErrorString(e));
    return sticky(c, SACD_ECUDA);
  }
  int rc = c->sharded ? launch_sharded_mttkrp(*c, mode) : launch_mttkrp(*c, mode, c->M);
  if (rc == SACD_OK) rc = read_matrix(c, c->M, c->m[mode].I, out, ld, false);
  return sticky(c, rc);
}

int sacd_time_mttkrp(sacd_ctx *c, int32_t mode, int32_t reps, double *ms) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2 || reps < 1 || !ms) {
    set_error("sacd_time_mttkrp: bad args");
    return SACD_EINVAL;
  }
  const int saved = c->opt.profile;
  c->opt.profile = 0;
  cudaEvent_t e0, e1;
  SACD_CUDA_TRY(cudaEventCreate(&e0));
  SACD_CUDA_TRY(cudaEventCreate(&e1));
  auto one = [&]() { return c->sharded ? launch_sharded_mttkrp(*c, mode) : launch_mttkrp(*c, mode, c->M); };
  int rc = one();  // warm-up
  SACD_CUDA_TRY(cudaEventRecord(e0, c->stream));
  for (int i = 0; i < reps && rc == SACD_OK; ++i) rc = one();
  SACD_CUDA_TRY(cudaEventRecord(e1, c->stream));
  SACD_CUDA_TRY(cudaEventSynchronize(e1));
  float t = 0.f;
  SACD_CUDA_TRY(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  c->opt.profile = saved;
  *ms = (double)t / reps;
  return sticky(c, rc);
}

int sacd_gram(sacd_ctx *c, int32_t mode, double *out) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2 || !out) {
    set_error("sacd_gram: bad mode/out");
    return SACD_ESTATE;
  }
  return sticky(c, dev_read(c, out, c->m[mode].G, (size_t)c->R * c->R * 8));
}

int sacd_hessian(sacd_ctx *c, int32_t mode, double *out) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2 || !out) {
    set_error("sacd_hessian: bad mode/out");
    return SACD_ESTATE;
  }
  int rc = launch_hessian_only(*c, mode);
  if (rc == SACD_OK) rc = dev_read(c, out, c->Hd, (size_t)c->R * c->R * 8);
  return sticky(c, rc);
}

int sacd_mode_update(sacd_ctx *c, int32_t mode, int32_t branch, uint8_t *decisions, double *ti, int64_t *E,
                     int64_t *Ech) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2 || branch < -1 || branch > 2) {
    set_error("sacd_mode_update: bad mode/branch");
    return SACD_ESTATE;
  }
  const size_t nd = (size_t)c->m[mode].I * c->R;
  uint8_t *dd = nullptr;
  if (decisions) {
    SACD_CUDA_TRY(pool_alloc(&dd, std::max<size_t>(1, nd), c->device, c->stream));
  }
  if (dd) SACD_CUDA_TRY(cudaMemsetAsync(dd, 0, std::max<size_t>(1, nd), c->stream));
  int rc = c->sharded ? launch_sharded_mode_update(*c, mode, branch, false, false, dd)
                      : launch_mode_update(*c, mode, branch, false, false, dd);
  if (rc == SACD_OK && decisions) rc = dev_read(c, decisions, dd, nd);
  if (dd) cudaFreeAsync(dd, c->stream);
  if (rc == SACD_OK) {
    double t;
    long long e[2];
    rc = dev_read(c, &t, reinterpret_cast<const char *>(c->st) + offsetof(DevState, ti_cur) + mode * 8, 8);
    if (rc == SACD_OK) rc = dev_read(c, &e[0], reinterpret_cast<const char *>(c->st) + offsetof(DevState, E) + mode * 8, 8);
    if (rc == SACD_OK)
      rc = dev_read(c, &e[1], reinterpret_cast<const char *>(c->st) + offsetof(DevState, Ech) + mode * 8, 8);
    if (rc == SACD_OK) {
      if (ti) *ti = t;
      if (E) *E = e[0];
      if (Ech) *Ech = e[1];
    }
  }
  return sticky(c, rc);
}

int sacd_layout(sacd_ctx *c, int32_t mode, uint32_t *idx_a, uint32_t *idx_b, float *val, int64_t *row_ptr) {
  CTX_CHECK(c);
  if (mode < 0 || mode > 2) {
    set_error("sacd_layout: bad mode");
    return SACD_ESTATE;
  }
  ModeData &md = c->m[mode];
  int rc = SACD_OK;
  uint32_t *tmp = nullptr;
  if (!md.idx_a && c->nnz) {  // no SoA copies: unpack the canonical 16-byte records
    if (cudaMalloc(&tmp, (size_t)c->nnz * 12) != cudaSuccess) {
      cudaGetLastError();
      set_error("sacd_layout: out of device memory");
      return SACD_ENOMEM;
    }
    rc = launch_unpack_nzm(*c, md.nzm, c->nnz, tmp, tmp + c->nnz, reinterpret_cast<float *>(tmp + 2 * c->nnz));
  }
  const uint32_t *sa = md.idx_a ? md.idx_a : tmp, *sb = md.idx_b ? md.idx_b : (tmp ? tmp + c->nnz : nullptr);
  const float *sv = md.val ? md.val : (tmp ? reinterpret_cast<const float *>(tmp + 2 * c->nnz) : nullptr);
  if (rc == SACD_OK && idx_a && c->nnz) {
    rc = dev_read(c, idx_a, sa, (size_t)c->nnz * 4);
    for (long long e = 0; rc == SACD_OK && e < c->nnz; ++e) idx_a[e] &= kIdxMask;  // strip the flag bits
  }
  if (rc == SACD_OK && idx_b && c->nnz) {
    rc = dev_read(c, idx_b, sb, (size_t)c->nnz * 4);
    for (long long e = 0; rc == SACD_OK && e < c->nnz; ++e) idx_b[e] &= kIdxMask;
  }
  if (rc == SACD_OK && val && c->nnz) rc = dev_read(c, val, sv, (size_t)c->nnz * 4);
  if (rc == SACD_OK && row_ptr) rc = dev_read(c, row_ptr, md.row_ptr, (size_t)(md.I + 1) * 8);
  if (tmp) cudaFree(tmp);
  return sticky(c, rc);
}

int sacd_stats(sacd_ctx *c, sacd_iter_stats *out, int32_t cap, int32_t *n_out) {
  CTX_CHECK(c);
  int cnt = 0;
  int rc = dev_read(c, &cnt, reinterpret_cast<const char *>(c->st) + offsetof(DevState, ring_count), sizeof(int));
  if (rc != SACD_OK) return sticky(c, rc);
  const int avail = std::min(cnt, kRing);
  const int n = std::min(avail, std::max(0, (int)cap));
  const int first = cnt - avail;  // oldest retained record
  for (int i = 0; i < n && out; ++i) {
    const int slot = (first + i) % kRing;
    rc = dev_read(c, out + i, reinterpret_cast<const char *>(c->st) + offsetof(DevState, ring) +
                                  (size_t)slot * sizeof(sacd_iter_stats),
                  sizeof(sacd_iter_stats));
    if (rc != SACD_OK) return sticky(c, rc);
  }
  if (n_out) *n_out = out ? n : avail;
  return SACD_OK;
}

int sacd_get_info(sacd_ctx *c, sacd_info *o) {
  CTX_CHECK(c);
  if (!o) return SACD_EINVAL;
  memset(o, 0, sizeof(*o));
  for (int n = 0; n < 3; ++n) {
    o->dims[n] = c->dims[n];
    o->mode_a[n] = c->m[n].a;
    o->mode_b[n] = c->m[n].b;
    o->items[n] = c->m[n].n_items;
    o->split_rows[n] = c->m[n].n_splits;
  }
  o->nnz = c->nnz;
  o->rank = c->R;
  o->pitch = c->pitch;
  o->precision = c->opt.precision;
  o->l_mode = c->opt.l_mode;
  o->variant = c->opt.variant;
  o->device_bytes = c->device_bytes;
  o->kernels_per_sweep = c->kernels_per_sweep;
  o->world_size = c->world;
  o->world_rank = c->me;
  o->sharded_ranks = c->sharded ? c->G : 1;
  o->delta_exchange = c->delta ? 1 : 0;
  o->delta_elems_sent = c->delta_sent;
  o->full_elems_equiv = c->full_equiv;
  for (int n = 0; n < 3; ++n) o->fibers[n] = c->m[n].n_fibers;
  o->uniform_values = c->uniform_x ? 1 : 0;
  o->uniform_value = c->uniform_x ? c->xu : 0.0;
  int k = 0;
  int rc = dev_read(c, &k, reinterpret_cast<const char *>(c->st) + offsetof(DevState, k), sizeof(int));
  if (rc == SACD_OK)
    rc = dev_read(c, &o->xnorm2, reinterpret_cast<const char *>(c->st) + offsetof(DevState, xnorm2), 8);
  o->k = k;
  return sticky(c, rc);
}

int sacd_profile_read(sacd_ctx *c, double ms[SACD_NUM_KCLASS], int64_t launches[SACD_NUM_KCLASS]) {
  CTX_CHECK(c);
  const int rc = prof_flush(*c);
  if (rc != SACD_OK) return sticky(c, rc);
  for (int i = 0; i < SACD_NUM_KCLASS; ++i) {
    if (ms) ms[i] = c->prof_ms[i];
    if (launches) launches[i] = c->prof_n[i];
  }
  return SACD_OK;
}

int sacd_set_profile(sacd_ctx *c, int32_t on) {
  CTX_CHECK(c);
  c->opt.profile = on ? 1 : 0;
  return SACD_OK;
}

int sacd_profile_reset(sacd_ctx *c) {
  CTX_CHECK(c);
  const int rc = prof_flush(*c);
  for (int i = 0; i < SACD_NUM_KCLASS; ++i) {
    c->prof_ms[i] = 0;
    c->prof_n[i] = 0;
  }
  return sticky(c, rc);
}

int sacd_shard_plan(const int64_t *row_ptr, int64_t I, int32_t world, int32_t rank, int64_t out[5]) {
  if (!row_ptr || !out || I < 1 || world < 1 || rank < 0 || rank >= world) {
    set_error("sacd_shard_plan: bad arguments");
    return SACD_EINVAL;
  }
  ShardPlan p = plan_shard(reinterpret_cast<const long long *>(row_ptr), I, world, rank);
  out[0] = p.lo;
  out[1] = p.hi;
  out[2] = p.rlo;
  out[3] = p.rhi;
  out[4] = p.head;
  return SACD_OK;
}

int sacd_abi_sizes(int32_t out[4]) {
  if (!out) return SACD_EINVAL;
  out[0] = SACD_ABI_VERSION;
  out[1] = (int32_t)sizeof(sacd_options);
  out[2] = (int32_t)sizeof(sacd_iter_stats);
  out[3] = (int32_t)sizeof(sacd_info);
  return SACD_OK;
}

int sacd_nccl_unique_id(void *out128) {
  if (!out128) return SACD_EINVAL;
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    set_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    return SACD_ENCCL;
  }
  memcpy(out128, &id, sizeof(id));
  return SACD_OK;
}

void sacd_free(sacd_ctx *c) { destroy(c); }

}  // extern "C"
