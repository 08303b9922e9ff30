/*
 * sacd.h -- C ABI of the B200-native SaCD hot path (libsacd.so).
 *
 * Saturating Coordinate Descent for sparse nonnegative CP tensor factorization,
 * arXiv 2003.03572 ("the paper"; line numbers "P:n" refer to PAPER.md).  The problem the
 * library solves is the paper's problem statement: given a sparse 3-way tensor X as the
 * set Omega of observed cells (q,p,s) with values x_qps (Table 2) and a rank R
 * (P:171), find nonnegative U (Q x R), V (P x R), W (S x R) minimising
 *     f(U,V,W) = || X - [[U,V,W]] ||^2                    (eq:ntf; Eq 6-7)
 * by `maxiters` sweeps of Algorithm 1 from a random initialisation.  The
 * readings of ambiguous passages are listed in DESIGN.md section 3 (C1-C19).
 *
 * Conventions for every entry point
 *   - Every call returns an int status (sacd_status); no C++ exception crosses the ABI.
 *     A thread-local message for the last failure is available from sacd_last_error().
 *   - SACD_ECUDA / SACD_ENCCL are sticky: after one, only sacd_free() is valid.
 *   - Matrices are row-major.  "Host" pointers are ordinary CPU memory; arguments marked
 *     "host or device" may be either (detected with cudaPointerGetAttributes).
 *   - A context is used from one host thread at a time.  All device memory, streams,
 *     events and graphs are owned by the context and released by sacd_free().
 *   - Calls are stream-ordered on the context's stream; calls that return data to the
 *     host synchronise that stream before returning.
 */
#ifndef SACD_H
#define SACD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SACD_ABI_VERSION 2

typedef struct sacd_ctx sacd_ctx; /* opaque; owned by the library until sacd_free */

typedef enum {
  SACD_OK = 0,
  SACD_EINVAL = -1,     /* bad argument: dims not in [1,2^30), rank not in [1,256], nnz < 0     */
  SACD_ERANGE = -2,     /* a coordinate index >= its mode length                              */
  SACD_EDUP = -3,       /* duplicate (q,p,s) (Omega is a set, Table 2)           */
  SACD_ENONFINITE = -4, /* NaN or Inf value                                                   */
  SACD_ENOMEM = -5,     /* device or host allocation failed                                   */
  SACD_ECUDA = -6,      /* CUDA error (sticky)                                                */
  SACD_ENCCL = -7,      /* NCCL error (sticky)                                                */
  SACD_ESTATE = -8      /* bad mode / ld / call order                                         */
} sacd_status;

/* Lipschitz constant used in the importance (Eq 20). */
enum {
  SACD_L_DIAG = 0, /* L_r = h_rr, the Gram-Hadamard diagonal (Eq 15): default (C5)    */
  SACD_L_FROB = 1  /* L = ||H||_F, Alg 1 line "L = ||H||" literally (Lemma 1)    */
};

/* Element selection. */
enum {
  SACD_VARIANT_GS_LAGGED = 0, /* Alg 1 selection with the lagged ti branch (C10) */
  SACD_VARIANT_SELECT_OFF = 1, /* the k==1 rule (z > 0) every sweep: projected GS CD           */
  SACD_VARIANT_JACOBI = 2,     /* Lemma 2 literally: every gradient of a pass from   */
                               /* the rows at pass start (not monotone: reading C9, pin P12)     */
  SACD_VARIANT_SNAPSHOT = 3    /* exact-timing ti (reading C10'): Alg 1's z from G at */
                               /* pass start give ti^k, which picks Eq 24 / Eq 27 for   */
                               /* the SAME pass; those z gate Gauss-Seidel updates; */
                               /* z_prev <- them.  Costs one extra read of M, F, z_prev per mode */
};

/* Arithmetic precision of factors, z_prev, MTTKRP and the row update (Grams, H and all
 * reductions are fp64 in both). */
enum { SACD_F64 = 0, SACD_F32 = 1 };

/* Branch of the selection rule for one mode pass (C10). */
enum { SACD_BR_AUTO = -1, SACD_BR_FIRST = 0, SACD_BR_EQ24 = 1, SACD_BR_EQ27 = 2 };

typedef struct {
  uint32_t struct_size;       /* = sizeof(sacd_options) (ABI versioning)                    */
  int32_t precision;          /* SACD_F64 (default) | SACD_F32                              */
  int32_t l_mode;             /* SACD_L_DIAG (default) | SACD_L_FROB                        */
  int32_t variant;            /* SACD_VARIANT_* (default GS_LAGGED); JACOBI and SNAPSHOT run  */
                              /* unsharded only (EINVAL with world_size > 1 / emulate_ranks)  */
  int32_t device;             /* CUDA ordinal; -1 = the calling thread's current device      */
  int32_t world_size, rank;   /* slice sharding across GPUs (1, 0 = single GPU)             */
  const void *nccl_unique_id; /* 128 bytes from sacd_nccl_unique_id() on rank 0 (G > 1)     */
  void *stream;               /* cudaStream_t to run on, or NULL = library-owned stream     */
  int32_t use_graph;          /* 1 (default): sacd_iterate replays a captured CUDA graph    */
  int32_t profile;            /* 1: time every kernel class with CUDA events (no graph)     */
  int32_t nnz_per_item;       /* MTTKRP work-item size in nonzeros (0 = by problem size:    */
                              /* 1024 for >= 5e7 nonzeros or R > 64, 256 for sharded ranks   */
                              /* and mid-size tensors, 64 under 1e5 nonzeros)                */
  int32_t mttkrp_variant;     /* MTTKRP tuning variant (0 = default; tools/mttkrp_tune.py)  */
  int32_t force_sharded;      /* 1: run the sharded (NCCL) engine also when world_size == 1 */
  int32_t emulate_ranks;      /* G >= 2 (with world_size 1): emulate the G ranks of the     */
                              /* sharded engine on this GPU, exchanges as local copies      */
  int32_t reserved[4];        /* [0]: row-update variant (0 = default: fp64 runs the DMMA     */
                              /* out-of-block gradient kernels (R <= 64: row blocks from a     */
                              /* work counter), fp32 the FMA kernel; 1 = FMA kernel with H     */
                              /* from global/L1; 2 = FMA kernel with H in shared memory;      */
                              /* 6 = the R <= 64 DMMA kernel on a static grid);               */
                              /* [1]: MTTKRP a-blocked order: > 0 = blocks of that many      */
                              /* a-rows, <= 0 = canonical order (default);                  */
                              /* [2]: Gram kernel (0 = default: fp64 tensor cores (DMMA): for */
                              /* pitch <= 64 fused into the row update while max I_n x R <=    */
                              /* 2^20, else a streaming kernel after it; for pitch >= 128 panel */
                              /* pairs; 1 = the FMA kernel; 2 = always fused; 3 = panel pairs  */
                              /* also for pitch <= 64; 4 = always the streaming kernel)        */
                              /* [3]: sharded exchange (0 = full owned rows, graph-captured;   */
                              /* 1 = delta: only the changed elements as (index, value) lists, */
                              /* full rows when those are smaller; NCCL sweeps then run eagerly */
                              /* because the list lengths are read on the host; 2 = peer      */
                              /* memory: a kernel stores every changed 16-byte chunk of the   */
                              /* owned rows straight into the peers' replicas (CUDA IPC over  */
                              /* NVLink), the head partials and stats slots likewise, and     */
                              /* device-side flags order the passes: no NCCL call and no host */
                              /* round trip per sweep, graph-captured)                        */
} sacd_options;

/* Per-sweep statistics (device-side ring, read by sacd_stats). */
typedef struct {
  int32_t k;             /* sweep index, 1-based                                            */
  int32_t branch[3];     /* SACD_BR_* used for U, V, W                                      */
  double objective;      /* f^k after the W pass (Eq 6-7 via the Gram identity, C1)          */
  double fit;            /* 1 - sqrt(f)/||X|| (C16)                                          */
  double ti[3];          /* total importance ti^k per mode (Eq 25)                    */
  int64_t E[3];          /* #elements selected (Lemma 4)                              */
  int64_t E_changed[3];  /* #selected with a nonzero step (C14)                              */
  double ms;             /* device time of the sweep: %globaltimer at its first kernel to the   */
                         /* end of its objective kernel (FitReport per-sweep time)  */
} sacd_iter_stats;

typedef struct {
  int64_t dims[3];
  int64_t nnz;      /* this rank's nonzeros (all of them for G = 1)                         */
  int32_t rank;     /* R                                                                    */
  int32_t pitch;    /* factor row pitch on device (R rounded up to the kernel tile)          */
  int32_t precision;
  int32_t l_mode, variant;
  int32_t k;        /* completed sweeps                                                      */
  int32_t mode_a[3], mode_b[3]; /* the "a" (longer) and "b" other modes of each layout      */
  double xnorm2;    /* ||X||^2 in fp64                                                       */
  int64_t items[3]; /* MTTKRP work items per mode                                            */
  int64_t split_rows[3];
  int64_t device_bytes;
  int32_t kernels_per_sweep; /* libsacd kernels launched per sweep (from the captured graph)   */
  int32_t world_size, world_rank, sharded_ranks; /* sharded engine: G ranks (1 = unsharded)    */
  int32_t delta_exchange;   /* 1: sharded passes exchange changed elements          */
  int64_t delta_elems_sent; /* NCCL delta exchange so far: elements sent as (index, value) ...  */
  int64_t full_elems_equiv; /* ... and the elements the full-row exchange would have sent       */
  int64_t fibers[3];        /* distinct (i_n, i_a) per layout: the MTTKRP's per-fiber gathers    */
  int32_t uniform_values;   /* 1: every value equals the first (bitwise), e.g. a binary tensor:  */
                            /* the MTTKRP then needs no per-nonzero value (exact)                */
  double uniform_value;     /* that value (0 unless uniform_values)                              */
} sacd_info;

void sacd_default_options(sacd_options *opt);

/* Build a context: validate the COO tensor, copy it to the device, build the three
 * mode-sorted layouts (Table 2 slices Omega^U_q, Omega^V_p, Omega^W_s; key (i_n, i_a, i_b)
 * with a the longer other mode, reading L1), compute ||X||^2 (fp64), initialise the factors
 * uniformly in [0,1) from `seed` (Alg 1 input; reading C12) and their Grams, and
 * capture the sweep graph.
 *   coords : host or device, nnz x 3 uint32 (q,p,s), 0-based.   vals : host or device, fp32.
 *   dims   : host, {Q, P, S}, each >= 1 and < 2^30.              rank : 1..256.
 * Errors: EINVAL, ERANGE, EDUP, ENONFINITE, ENOMEM, ECUDA.  nnz == 0 is legal.
 * The caller keeps ownership of coords/vals and may free them when the call returns.
 * Device inputs may come from any stream: the call synchronises the device before reading
 * them (so e.g. tensors just produced on PyTorch's current stream are complete). */
int sacd_init(sacd_ctx **out, const uint32_t *coords, const float *vals, int64_t nnz, const int64_t dims[3],
              int32_t rank, uint64_t seed, const sacd_options *opt);

/* Run n_sweeps sweeps of Alg 1 (each: U, V, W mode updates, then the objective),
 * asynchronously on the context stream; k += n_sweeps. */
int sacd_iterate(sacd_ctx *ctx, int32_t n_sweeps);

/* Block until all queued work of the context has finished. */
int sacd_sync(sacd_ctx *ctx);

/* Objective f (Eq 6-7, all cells, C1) and fit = 1 - sqrt(f)/||X|| after the last completed
 * sweep (k = 0: the initial factors).  Synchronous. */
int sacd_fit(sacd_ctx *ctx, double *objective, double *fit);

/* Copy factor `mode` (0=U, 1=V, 2=W) into host memory `out` (I_mode rows, leading
 * dimension ld >= rank, fp64).  Errors: ESTATE for a bad mode or ld. */
int sacd_factors(sacd_ctx *ctx, int32_t mode, double *out, int64_t ld);

/* Copy up to `cap` per-sweep records, oldest first, into host `out`; *n_out = count. */
int sacd_stats(sacd_ctx *ctx, sacd_iter_stats *out, int32_t cap, int32_t *n_out);

int sacd_get_info(sacd_ctx *ctx, sacd_info *out);

void sacd_free(sacd_ctx *ctx);

const char *sacd_last_error(void);

/* --------------------------------------------------------------------------------------
 * Held-out evaluation (the paper's 80/20 protocol).
 * ------------------------------------------------------------------------------------ */

/* Predictions of the current CP model at n coordinates (Eq 8):
 *   out[e] = sum_{r<R} u_(q_e, r) v_(p_e, r) w_(s_e, r)
 *   coords : host or device, n x 3 uint32 (q,p,s), each index < dims[mode].
 *   out    : host or device, n fp64 (written).  n == 0 is legal.
 * Errors: EINVAL (n < 0 or null pointers with n > 0), ERANGE (index out of range; nothing
 * written), ENOMEM, ECUDA.  Synchronous; the caller owns both buffers.  Device inputs are
 * read after a device synchronisation, as in sacd_init. */
int sacd_predict(sacd_ctx *ctx, const uint32_t *coords, int64_t n, double *out);

/* Root mean squared error of the current model on n held-out entries (Eq 30,
 * P:886-890): sqrt( sum_e (x_e - xhat_e)^2 / n ), the squared errors summed in fp64 in a
 * fixed order (deterministic).  coords as sacd_predict; vals: host or device, n fp32.
 * n == 0 gives *rmse = 0.  Errors as sacd_predict.  Synchronous. */
int sacd_rmse(sacd_ctx *ctx, const uint32_t *coords, const float *vals, int64_t n, double *rmse);

/* --------------------------------------------------------------------------------------
 * Component entry points (teacher forcing, parity tests and kernel timing).  Each runs the
 * same kernels the sweep runs.
 * ------------------------------------------------------------------------------------ */

/* Overwrite factor `mode` from host fp64 `in` (ld >= rank; columns >= rank ignored) and
 * refresh its Gram.  Values are rounded to the context precision. */
int sacd_set_factors(sacd_ctx *ctx, int32_t mode, const double *in, int64_t ld);

/* Factor `mode` as held by shard `shard`'s replica (host fp64, ld >= rank).  Shards are the
 * ranks this context runs (one per process, or all G with emulated ranks); with the
 * peer-memory exchange and emulated ranks every shard has its own replicas, which must stay
 * bitwise identical.  Otherwise this is sacd_factors.  Errors: ESTATE. */
int sacd_replica_factors(sacd_ctx *ctx, int32_t shard, int32_t mode, double *out, int64_t ld);

/* Read / overwrite the previous importances z^{k-1} of `mode` (Alg 1). */
int sacd_get_zprev(sacd_ctx *ctx, int32_t mode, double *out, int64_t ld);
int sacd_set_zprev(sacd_ctx *ctx, int32_t mode, const double *in, int64_t ld);

/* Sparse MTTKRP for `mode` with the current factors:
 *   M_(i,r) = sum_{e in Omega^(mode)_i} x_e a_(e,r) b_(e,r)   (Eq 9 first term, P:340;
 *   column form P:623-625, 655, 682), written to host `out` (I_mode x ld, fp64). */
int sacd_mttkrp(sacd_ctx *ctx, int32_t mode, double *out, int64_t ld);

/* Time `reps` back-to-back launches of the MTTKRP of `mode` with CUDA events on the context
 * stream; *ms = mean milliseconds per launch. */
int sacd_time_mttkrp(sacd_ctx *ctx, int32_t mode, int32_t reps, double *ms);

/* Gram G_mode = F^T F (fp64, R x R, host `out`), and H = G_a * G_b for `mode` (Eq 10 /
 * ppdei / ppdet: the Hadamard product of the OTHER factors' Grams). */
int sacd_gram(sacd_ctx *ctx, int32_t mode, double *out);
int sacd_hessian(sacd_ctx *ctx, int32_t mode, double *out);

/* One mode update (MTTKRP, H, the column-wise SaCD step, Gram refresh) with the selection
 * branch `branch` (SACD_BR_AUTO = the device rule C10, which also advances the history).
 * Optional host outputs: decisions (I_mode x rank bytes, 1 = element selected), ti, E,
 * E_changed.  Synchronous. */
int sacd_mode_update(sacd_ctx *ctx, int32_t mode, int32_t branch, uint8_t *decisions, double *ti, int64_t *E,
                     int64_t *E_changed);

/* Copy the mode-sorted layout of `mode` to host: idx_a/idx_b/val have nnz entries (the
 * indices in modes mode_a/mode_b of sacd_info), row_ptr has I_mode + 1 (int64). */
int sacd_layout(sacd_ctx *ctx, int32_t mode, uint32_t *idx_a, uint32_t *idx_b, float *val, int64_t *row_ptr);

/* Profiling (opt.profile = 1): per kernel class, total milliseconds and launch count
 * accumulated by sacd_iterate since the last reset.  Classes: 0 mttkrp, 1 split-row
 * fix-up, 2 hessian/branch, 3 SaCD row update, 4 Gram, 5 finalize/fit.  Synchronous. */
#define SACD_NUM_KCLASS 6
int sacd_profile_read(sacd_ctx *ctx, double ms[SACD_NUM_KCLASS], int64_t launches[SACD_NUM_KCLASS]);
int sacd_profile_reset(sacd_ctx *ctx);
/* Switch profiling on (sacd_iterate launches eagerly with per-class CUDA events) or off
 * (sacd_iterate replays the captured sweep graph, if opt.use_graph).  Never fails on a
 * live context. */
int sacd_set_profile(sacd_ctx *ctx, int32_t on);

/* Slice-sharding plan of one mode for `world` ranks; a pure host function
 * (no GPU).  row_ptr: host, I + 1 entries of the mode-sorted layout (sacd_layout).
 * Output for `rank` (0 <= rank < world):
 *   out[0], out[1] : its nonzero range [lo, hi), lo = floor(rank * nnz / world)
 *   out[2], out[3] : its owned rows [rlo, rhi): the rows whose first nonzero index
 *                    row_ptr[r] lies in [lo, hi); the last rank also owns the trailing
 *                    empty rows (row_ptr[r] == nnz)
 *   out[4]         : its head row, the row owned by a lower rank to which the nonzeros
 *                    [lo, min(hi, row_ptr[rlo])) belong, or -1 if there are none
 * Every row is owned by exactly one rank; a row's MTTKRP is its owner's local part plus
 * the head partials of the higher ranks whose head row it is.  Errors: EINVAL. */
int sacd_shard_plan(const int64_t *row_ptr, int64_t I, int32_t world, int32_t rank, int64_t out[5]);

/* ABI self-description for bindings: out = {SACD_ABI_VERSION, sizeof(sacd_options),
 * sizeof(sacd_iter_stats), sizeof(sacd_info)}.  Needs no GPU. */
int sacd_abi_sizes(int32_t out[4]);

/* Multi-GPU: a fresh 128-byte NCCL unique id (rank 0), to be broadcast by the caller. */
int sacd_nccl_unique_id(void *out128);

/* Sharded engine (world_size > 1, force_sharded or emulate_ranks): per mode, every rank
 * computes the MTTKRP of its nnz-balanced range of the mode-sorted nonzeros (plan:
 * sacd_shard_plan); head partials of rows cut by a range boundary are all-gathered and
 * added by the row owner in rank order; owners run the SaCD row update on their rows; the
 * updated rows are broadcast by their owners (NCCL all-gather-v over NVLink) into every
 * rank's replicated factor; (ti, md, E, E_changed, Gram partial) are all-gathered and
 * summed in rank order, so every rank holds the same state and takes the same branch.
 * Every rank passes the same full COO to sacd_init.  sacd_factors returns the full
 * replicated factor; sacd_get_zprev / sacd_mttkrp / decisions are valid on owned rows. */

#ifdef __cplusplus
}
#endif
#endif /* SACD_H */
