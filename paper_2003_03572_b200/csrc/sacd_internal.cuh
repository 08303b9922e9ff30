// sacd_internal.cuh -- internal declarations of libsacd (B200 / sm_100a).
// The public ABI is include/sacd.h; nothing here crosses it.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/sacd.h"

namespace sacd {

// ------------------------------------------------------------------ errors
void set_error(const std::string &msg);

struct Status {
  int code;
};

#define SACD_CUDA_TRY(call)                                                                    \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      ::sacd::set_error(std::string(#call) + ": " + cudaGetErrorString(e_) + " @" + __FILE__ + \
                        ":" + std::to_string(__LINE__));                                       \
      return (e_ == cudaErrorMemoryAllocation) ? SACD_ENOMEM : SACD_ECUDA;                     \
    }                                                                                          \
  } while (0)

#define SACD_TRY(call)          \
  do {                          \
    int rc_ = (call);           \
    if (rc_ != SACD_OK) return rc_; \
  } while (0)

// ------------------------------------------------------------------ device memory pool
// The library's stream-ordered allocations (the uploaded COO, the layout build's multi-GB
// sort scratch, the per-mode nonzero records, M, z_prev, the split-row partials, per-call
// temporaries) come from ONE pool per device that the library owns (cudaMemPoolCreate), not
// from the device's default pool.  Freed memory stays mapped in it up to a release threshold
// (a quarter of the device's memory; SACD_POOL_RELEASE_MB overrides), so the layout of mode 2
// reuses mode 1's scratch, and a later sacd_init in the same process (the next tensor, the
// next repetition) finds its buffers mapped instead of paying the page-mapping cost of fresh
// device memory again, which dominated sacd_init (c4: ~80 ms of ~180).  Buffers shared with
// peers through CUDA IPC (factor replicas, flags, exchange slots) stay on cudaMalloc.
cudaMemPool_t device_pool(int device);
template <typename T>
inline cudaError_t pool_alloc(T **p, size_t bytes, int device, cudaStream_t s) {
  return cudaMallocFromPoolAsync(reinterpret_cast<void **>(p), bytes, device_pool(device), s);
}

// SACD_INIT_TIMING=1 prints the wall time of each sacd_init phase to stderr (diagnostics)
struct InitTimer {
  bool on = getenv("SACD_INIT_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(cudaStream_t s, const char *what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[sacd_init] %-32s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// ------------------------------------------------------------------ device structures
// One MTTKRP work item: either whole rows [row0,row1) whose nonzeros are [nz0,nz1), or
// (slot >= 0) one segment [nz0,nz1) of a heavy row row0 whose partial goes to `slot`.
struct WorkItem {
  long long nz0, nz1;
  int row0, row1;
  long long slot;
};

struct SplitRow {
  long long slot0, nslots;
  int row, chunk0;  // chunk0: first FixChunk of this row (ceil(nslots / kFixChunk) chunks)
};

// Fix-up of split rows in two levels: chunk c sums slots [slot0, slot0 + nslots) (at most
// kFixChunk) in slot order into M[row] directly (out < 0: row = -out - 1, single-chunk
// rows) or into the level-2 buffer row `out`; level 2 sums a row's chunk rows in order.
constexpr int kFixChunk = 64;
struct FixChunk {
  long long slot0;
  int nslots, out;
};

constexpr int kRing = 4096;

// idx_a carries two flag bits set by the layout builder (mode lengths are < 2^30):
// bit 31 = first nonzero of a fiber (new (i_n, i_a)), bit 30 = first nonzero of a row.
// SACD_DEBUG builds (libsacd_debug.so) check indices and slots inside the kernels with
// device-side asserts (a failed assert traps and the context reports ECUDA).
#ifdef SACD_DEBUG
#include <cassert>
#define SACD_DASSERT(cond) assert(cond)
#else
#define SACD_DASSERT(cond) ((void)0)
#endif

// Bounds of the MTTKRP launch that follows (set by k_set_dbg in SACD_DEBUG builds only).
struct DebugBounds {
  long long nnz, Ia, Ib, In, nslots, nchunk_rows;
};

constexpr uint32_t kFiberStart = 1u << 31;
constexpr uint32_t kRowStart = 1u << 30;
constexpr uint32_t kIdxMask = (1u << 30) - 1u;

// Device-resident control state: everything the sweep graph needs to decide on device.
struct DevState {
  int k;                 // completed/started sweeps
  int nhist[3];          // number of ti values recorded per mode
  double ti1[3], ti2[3]; // ti^{k-1}, ti^{k-2} per mode (reading C10)
  int branch[3];         // branch used by the latest pass of each mode
  double Lfrob[3];       // ||H||_F of the latest pass of each mode
  double ti_cur[3];
  long long E[3], Ech[3];
  double xnorm2;
  double f, fit;
  double mdot;           // sum_i sum_r w_ir m^W_ir of the latest W pass
  int ring_count;
  unsigned long long t_begin;  // %globaltimer (ns) at the start of the current sweep
  sacd_iter_stats ring[kRing];
};

struct ModeData {
  long long I = 0;
  int a = 0, b = 0;               // the other modes ("a" = the longer, L1)
  uint32_t *idx_a = nullptr, *idx_b = nullptr, *idx_n = nullptr;  // idx_a has flag bits
  float *val = nullptr;
  uint4 *nzm = nullptr;           // per nonzero {idx_a|flags, idx_b|flags, bits(val), row}: one 16-byte load
  long long *row_ptr = nullptr;   // I+1
  WorkItem *items = nullptr;
  long long n_items = 0;
  SplitRow *splits = nullptr;
  long long n_splits = 0, n_slots = 0;
  FixChunk *chunks = nullptr;
  long long n_chunks = 0;
  long long ablk_rows = 0;        // > 0: nzm / items follow the a-blocked execution order
  long long n_fibers = 0;         // distinct (i_n, i_a) in the layout (MTTKRP kernel choice)
  void *F = nullptr;              // Real[I * pitch]
  void *Z = nullptr;              // Real[ceil32(I) * pitch]  (z_prev, TT layout)
  double *G = nullptr;            // fp64 R x R Gram of F
  uint32_t *cmask = nullptr;      // [I] 16-byte chunk support mask of each row of F (k_chunk_mask)
};

// slice sharding plan of one mode (capi.cu; see sacd_shard_plan in include/sacd.h)
struct ShardPlan {
  long long lo = 0, hi = 0, rlo = 0, rhi = 0, head = -1;
};

// One rank's share of the sharded engine: its nonzero ranges, MTTKRP work
// items over them, and its private scratch.  A process holds one shard (NCCL) or all of
// them (emulated ranks on one GPU).
struct Shard {
  int rank = 0;
  ShardPlan plan[3];
  WorkItem *items[3] = {nullptr, nullptr, nullptr};
  long long n_items[3] = {0, 0, 0};
  SplitRow *splits[3] = {nullptr, nullptr, nullptr};
  long long n_splits[3] = {0, 0, 0};
  FixChunk *chunks[3] = {nullptr, nullptr, nullptr};
  long long n_chunks[3] = {0, 0, 0};
  void *M = nullptr;             // Real [maxI * pitch]
  void *partial = nullptr;       // Real [slots * pitch]
  double *row_part = nullptr;    // 2 * max row blocks
  long long *cnt_part = nullptr; // 2 * max row blocks
  double *gram_part = nullptr;   // gram blocks * R * R
  // peer-memory exchange (opt.reserved[3] = 2): this rank's factor replicas (its own device
  // memory; with emulated ranks every shard has separate replicas), device arrays of the G
  // ranks' replica base pointers per mode (IPC-mapped peers across processes), the flags the
  // peers raise in this rank's memory after pushing, and this rank's pass counter
  void *Frep[3] = {nullptr, nullptr, nullptr};
  void **d_peerF[3] = {nullptr, nullptr, nullptr};
  unsigned long long *flags = nullptr;      // [G]
  unsigned long long **d_peer_flags = nullptr;
  unsigned long long *epoch = nullptr;
  bool own_rep = false;                     // Frep allocated by this shard (emulation, q > 0)
  // this rank's exchange arrays (G slots each: head ids, head rows, stats) and device tables
  // of every rank's arrays (p2p; shard 0 / a process's own shard uses the context's arrays)
  long long *xid_r = nullptr;
  void *xrow_r = nullptr;
  double *xstats_r = nullptr;
  long long **d_px = nullptr;
  void **d_pr = nullptr;
  double **d_ps = nullptr;
  std::vector<void *> ipc_opened;
};

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool dead = false;
  sacd_options opt{};
  long long dims[3]{};
  long long nnz = 0;
  int R = 0, pitch = 0;           // pitch = kernel tile RT (8..256)
  ModeData m[3];
  DevState *st = nullptr;         // device
  // scratch
  void *M = nullptr;              // Real[ceil32(maxI) * pitch] (TT layout)
  void *Zs = nullptr;             // Real[ceil32(maxI) * pitch] snapshot z of a pass (SNAPSHOT variant)
  unsigned long long *item_ctr = nullptr;  // work counter of the dynamically scheduled MTTKRP
  int num_sms = 0;
  void *partial = nullptr;        // Real[max slots * pitch]
  void *fixbuf = nullptr;         // Real[max chunks * pitch] (level-2 fix-up rows)
  void *Hr = nullptr;             // Real[pitch * pitch]
  double *Hd = nullptr;           // R x R
  double *row_part = nullptr;     // 4 * max row blocks (ti, mdot) as doubles
  long long *cnt_part = nullptr;  // 2 * max row blocks (E, Ech)
  double *gram_part = nullptr;    // gram blocks * R * R
  uint8_t *decisions = nullptr;   // teacher-forced only
  long long max_row_blocks = 0;
  long long max_slots = 1, max_chunks = 1;  // rows of the partial / fix-up buffers (debug bounds)
  bool uniform_x = false;  // every value of the tensor equals xu (bitwise), e.g. a binary tensor
  double xu = 0.0;
  int gram_blocks = 0;
  int gram_cap = 0;               // Gram partials the gram_part buffers hold (>= gram_blocks)
  long long device_bytes = 0;
  // graph
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  int kernels_per_sweep = 0;
  // profiling
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_pending;  // (class, pool index of start)
  size_t ev_next = 0;
  double prof_ms[SACD_NUM_KCLASS]{};
  long long prof_n[SACD_NUM_KCLASS]{};
  // sharded engine (world > 1, forced, or emulated ranks)
  bool sharded = false;
  int G = 1;                      // total ranks
  int world = 1, me = 0;          // NCCL process group
  void *comm = nullptr;           // ncclComm_t
  std::vector<ShardPlan> all_plans[3];
  std::vector<Shard> shards;
  long long *xid = nullptr;       // [G] head row ids
  void *xrow = nullptr;           // [G * pitch] head partial rows (Real)
  double *xstats = nullptr;       // [G * (4 + R*R)] (ti, md, E, Ech, Gram partial)
  // delta exchange (opt.reserved[3] = 1): per mode pass each owner sends only the
  // elements of its rows that changed, as (element index, value) lists
  bool delta = false;
  bool p2p = false;               // opt.reserved[3] = 2: changed 16-byte chunks pushed to peers'
                                  // replicas by a kernel, device-side flags (graph-capturable)
  void *const *rows_peers = nullptr;  // set around a shard's fused row-update launch (p2p)
  int rows_me = 0;
  bool capturing = false;         // inside capture_graph (no host synchronisation allowed)
  void *Fold = nullptr;           // Real [maxI * pitch]: owned rows before the pass
  uint32_t *didx = nullptr;       // [sum_q cap_q] list of rank q at doff[q]
  void *dval = nullptr;           // Real [sum_q cap_q]
  long long *dcnt = nullptr;      // [G] list lengths (device)
  int *dblk = nullptr;            // [kDeltaBlocks] per-block change counts
  std::vector<long long> doff, dcap;  // host: slot offsets / capacities (elements)
  long long delta_sent = 0, full_equiv = 0;  // host: elements exchanged as deltas / as full rows
  // pinned staging ring for device -> pageable-host reads (sacd_factors & co.): two chunks,
  // the D2H copy of one overlapping the multi-threaded host copy of the other
  void *pin = nullptr;
  size_t pin_chunk = 0;
  cudaEvent_t pin_ev[2] = {nullptr, nullptr};
};

constexpr int kDeltaBlocks = 296;

size_t real_size(const Context &c);

// The per-mode SoA copies of the layout (idx_a, idx_b, idx_n, val) are read only by the R <= 16
// MTTKRP kernel, the warp fiber kernel (variant 1) and the a-blocked order builder; every
// other path reads the 16-byte records (nzm), which also serve the canonical readback.
inline bool layout_needs_soa(const Context &c) {
  return c.pitch < 32 || c.opt.mttkrp_variant == 1 || c.opt.reserved[1] > 0;
}

ShardPlan plan_shard(const long long *row_ptr, long long I, int world, int rank);

// layout.cu
int build_layouts(Context &c, const uint32_t *coords_dev, const float *vals_dev);
// rewrite md.nzm of mode n in the a-blocked order (block = i_a / ablk_rows); returns the
// (blk, row) segments in execution order: start offsets and row ids
int build_blocked_order(Context &c, int n, long long ablk_rows, std::vector<long long> &seg_start,
                        std::vector<int> &seg_row);

// kernels.cu
int launch_init_factors(Context &c, uint64_t seed);
int launch_mttkrp(Context &c, int mode, void *out_M);
int launch_mode_update(Context &c, int mode, int branch_override, bool begin_sweep, bool end_sweep,
                       uint8_t *decisions_dev);
int launch_gram(Context &c, int mode);
int launch_initial_fit(Context &c);
int launch_unpack_nzm(Context &c, const uint4 *nzm, long long nnz, uint32_t *ia, uint32_t *ib, float *v);
int launch_range_check(Context &c, const uint32_t *coords_dev, long long n, int *flag_dev);
int launch_predict(Context &c, const uint32_t *coords_dev, long long n, const float *vals_dev, double *out_dev,
                   double *part_dev, double *sse_dev);  // vals/out/sse may be null
int launch_convert_in(Context &c, const double *src_dev, long long rows, void *dst, bool tt_layout);
int launch_convert_out(Context &c, const void *src, long long rows, double *dst_dev, bool tt_layout);
int launch_hessian_only(Context &c, int mode);
int launch_setup(Context &c);
int launch_sharded_mode_update(Context &c, int mode, int branch_override, bool begin_sweep, bool end_sweep,
                               uint8_t *decisions_dev);
int launch_sharded_mttkrp(Context &c, int mode);   // merged M of the owned rows -> c.M
int launch_sharded_initial_fit(Context &c);
int nccl_allgather_inplace(Context &c, void *buf, size_t count_per_rank, int dtype);  // dtype 0 f64, 1 f32, 2 i64
int nccl_broadcast_rows(Context &c, int mode);
long long rows_block_for(const Context &c);

// profiling helpers (kernels.cu uses them around launches)
int prof_begin(Context &c, int kclass);
int prof_end(Context &c, int kclass, int start_idx);

}  // namespace sacd
