/*
 * sacd_oracle.c -- plain, slow, fp64 CPU ORACLE for Saturating Coordinate Descent (SaCD)
 * for sparse nonnegative CP tensor factorization (arXiv 2003.03572, "PAPER.md").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2003_03572_b200/), and neither
 * imports the other.
 *
 * Every function follows the paper's definitions in the paper's order and notation,
 * with no blocking, fusion or reordering.  Citations "P:n" are PAPER.md line numbers;
 * readings "Cn" are the ones listed in DESIGN.md section 3 (= SURVEY.md section 8(c)).
 *
 *   layout          Table 2: Omega^U_q, Omega^V_p, Omega^W_s as mode-sorted slices
 *   init            Alg 1 input "Randomly Initialized", reading C12 (SplitMix64)
 *   gram / H        Eq 10, ppdei, ppdet:  H = A^T A * B^T B
 *   mttkrp          Eq 9 first term X_(1)(W (.) V), column form P:623-625
 *   gradient        Eq 14:  g_qr = -m_qr + (U H)_qr,  read column-sequentially (C9)
 *   step            Eq 11-13: u <- max(0, u - g/h_rr)
 *   importance      Eq 20: z = -g*uhat - (L/2)*uhat^2, uhat the constrained step (C6)
 *   selection       Alg 1: k==1: z>0; else sp>0 with sp from Eq 24
 *                   or Eq 27 chosen by total importance Eq 25-26,
 *                   lagged by one sweep (C10)
 *   objective       Eq 6-7 over all cells (C1), via the Gram identity
 *   predict / RMSE  Eq 8 at held-out coordinates; Eq 30
 *
 * Parity status: pinned by tests/test_oracle_pins.py (P1-P12 in DESIGN.md section 3).
 * The selection dynamics end to end (E, ti trajectories) are "parity unpinned": the paper
 * prints no trace of them.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORA_OK 0
#define ORA_EINVAL -1
#define ORA_ERANGE -2
#define ORA_EDUP -3
#define ORA_ENONFINITE -4
#define ORA_ENOMEM -5

#define BR_FIRST 0 /* Alg 1 line "if z_qr > 0" at k == 1            */
#define BR_EQ24 1  /* sp = z^k - z^{k-1}            (Eq 24)            */
#define BR_EQ27 2  /* sp = z^{k-1} - z^k            (Eq 27)            */

#define VAR_GS_LAGGED 0  /* default reading (C9, C10)                          */
#define VAR_SELECT_OFF 1 /* the k==1 rule every sweep: plain projected GS CD   */
#define VAR_JACOBI 2     /* Lemma 2 literal: g from the row at pass start (C9) */
#define VAR_SNAPSHOT 3   /* exact-timing ti: Alg 1's z from G at pass start, */
                         /* ti^k from those z, updates Gauss-Seidel (reading C10')        */

void ora_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int ora_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ random numbers
 * Reading C12: mix64 = SplitMix64 finaliser; rand(seed, tag, ctr) =
 * mix64(mix64(seed ^ tag) + (ctr+1) * 0x9E3779B97F4A7C15); unit24(x) = (x >> 40) 2^-24. */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t ora_rand(uint64_t seed, uint64_t tag, uint64_t ctr) {
  return mix64(mix64(seed ^ tag) + (ctr + 1ULL) * 0x9E3779B97F4A7C15ULL);
}

/* Alg 1 input "Randomly Initialized factor matrices": uniform [0,1) (C12).
 * F_n[i][r] = unit24(rand(seed, INIT=1, off_n + i*R + r)), off_0 = 0, off_1 = I_0 R,
 * off_2 = (I_0 + I_1) R.  Each F_n is row-major I_n x R. */
void ora_init_factors(const int64_t dims[3], int R, uint64_t seed, double *U, double *V, double *W) {
  double *F[3] = {U, V, W};
  uint64_t off = 0;
  for (int n = 0; n < 3; n++) {
    for (int64_t i = 0; i < dims[n]; i++)
      for (int r = 0; r < R; r++) {
        uint64_t x = ora_rand(seed, 1, off + (uint64_t)i * (uint64_t)R + (uint64_t)r);
        F[n][i * R + r] = (double)(x >> 40) * (1.0 / 16777216.0);
      }
    off += (uint64_t)dims[n] * (uint64_t)R;
  }
}

/* ------------------------------------------------------------------ layout
 * Table 2: Omega^(n)_i = the nonzeros whose mode-n index is i.  Entries are
 * ordered by the key (i_n, i_a, i_b) with a = the other mode of LARGER length (ties ->
 * lower mode id) and b = the remaining one (reading L1); keys are unique so the
 * order is unique. */
void ora_other_modes(const int64_t dims[3], int n, int *a, int *b) {
  int o1 = (n + 1) % 3, o2 = (n + 2) % 3;
  int lo = o1 < o2 ? o1 : o2, hi = o1 < o2 ? o2 : o1;
  if (dims[hi] > dims[lo]) { *a = hi; *b = lo; }
  else { *a = lo; *b = hi; }
}

typedef struct { uint64_t key; int64_t pos; } ora_kv;

static int kv_cmp(const void *x, const void *y) {
  uint64_t a = ((const ora_kv *)x)->key, b = ((const ora_kv *)y)->key;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* Validates (in-range, finite, no duplicates) and builds the mode-n layout.
 * Outputs: idx_a[nnz], idx_b[nnz] (indices in modes a and b), val[nnz], row_ptr[I_n+1]. */
int ora_layout(int64_t nnz, const uint32_t *coords, const float *vals, const int64_t dims[3], int n,
               uint32_t *idx_a, uint32_t *idx_b, float *val, int64_t *row_ptr) {
  if (nnz < 0 || n < 0 || n > 2) return ORA_EINVAL;
  for (int m = 0; m < 3; m++)
    if (dims[m] < 1) return ORA_EINVAL;
  int a, b;
  ora_other_modes(dims, n, &a, &b);
  for (int64_t e = 0; e < nnz; e++) {
    for (int m = 0; m < 3; m++)
      if ((int64_t)coords[3 * e + m] >= dims[m]) return ORA_ERANGE;
    if (!isfinite(vals[e])) return ORA_ENONFINITE;
  }
  ora_kv *kv = (ora_kv *)malloc(sizeof(ora_kv) * (size_t)(nnz > 0 ? nnz : 1));
  if (!kv) return ORA_ENOMEM;
  for (int64_t e = 0; e < nnz; e++) {
    uint64_t in = coords[3 * e + n], ia = coords[3 * e + a], ib = coords[3 * e + b];
    kv[e].key = (in * (uint64_t)dims[a] + ia) * (uint64_t)dims[b] + ib;
    kv[e].pos = e;
  }
  qsort(kv, (size_t)nnz, sizeof(ora_kv), kv_cmp);
  for (int64_t e = 1; e < nnz; e++)
    if (kv[e].key == kv[e - 1].key) { free(kv); return ORA_EDUP; }
  for (int64_t i = 0; i <= dims[n]; i++) row_ptr[i] = 0;
  for (int64_t e = 0; e < nnz; e++) {
    int64_t p = kv[e].pos;
    idx_a[e] = coords[3 * p + a];
    idx_b[e] = coords[3 * p + b];
    val[e] = vals[p];
    row_ptr[coords[3 * p + n] + 1] += 1;
  }
  for (int64_t i = 0; i < dims[n]; i++) row_ptr[i + 1] += row_ptr[i];
  free(kv);
  return ORA_OK;
}

/* ------------------------------------------------------------------ dense algebra */
/* G = F^T F for F row-major I x R; each entry a sequential sum over rows (Eq 10 factors). */
void ora_gram(const double *F, int64_t I, int R, double *G) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < R; r++)
    for (int t = r; t < R; t++) {
      double s = 0.0;
      for (int64_t i = 0; i < I; i++) s += F[i * R + r] * F[i * R + t];
      G[r * R + t] = s;
      G[t * R + r] = s;
    }
}

/* Eq 4: Hadamard product; here H = G_a * G_b (Eq 10, ppdei, ppdet). */
void ora_hadamard(const double *X, const double *Y, int64_t count, double *Z) {
  for (int64_t i = 0; i < count; i++) Z[i] = X[i] * Y[i];
}

/* Alg 1 "L = ||H||" with Table 2's Frobenius norm. */
double ora_frobenius(const double *H, int R) {
  double s = 0.0;
  for (int64_t i = 0; i < (int64_t)R * R; i++) s += H[i] * H[i];
  return sqrt(s);
}

/* ------------------------------------------------------------------ MTTKRP
 * m_{i,r} = sum_{e in Omega^(n)_i} x_e * a_{e,r} * b_{e,r}   (Eq 9 first term P:340;
 * column form P:623-625, 655, 682), summed sequentially in layout order. */
void ora_mttkrp(int64_t I, int R, const int64_t *row_ptr, const uint32_t *idx_a, const uint32_t *idx_b,
                const float *val, const double *A, const double *B, double *M) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < I; i++) {
    for (int r = 0; r < R; r++) {
      double s = 0.0;
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; e++)
        s += ((double)val[e] * A[(int64_t)idx_a[e] * R + r]) * B[(int64_t)idx_b[e] * R + r];
      M[i * R + r] = s;
    }
  }
}

/* ------------------------------------------------------------------ one SaCD mode pass
 * For each row i (rows independent), columns r = 0..R-1 in order (C9):
 *   if h_rr == 0: z = 0, no update, not counted (C11)
 *   g    = -m_ir + sum_j u_ij h_jr                     Eq 14, current row (C9)
 *   uhat = max(0, u_ir - g/h_rr) - u_ir                Eq 11-12
 *   z    = -g*uhat - (L_r/2)*uhat^2                    Eq 20
 *   sel  = FIRST: z > 0; EQ24: z - zprev > 0; EQ27: zprev - z > 0
 *   if sel: u_ir <- u_ir + uhat  (computed as max(0, u - g/h), C17)   Eq 13
 *   zprev_ir <- z  (always, C8)
 * Outputs: ti = sum of z (Eq 25) in row-major order, E = #selected (Lemma 4),
 * E_changed = #selected with uhat != 0 (C14), mdot = sum_i sum_r u_ir(new) m_ir.
 * decisions (optional, one byte per element, row-major) = sel. */
int ora_mode_pass(int64_t I, int R, const double *M, const double *H, double *F, double *zprev, int branch,
                  int l_mode, int jacobi, uint8_t *decisions, double *ti_out, int64_t *E_out,
                  int64_t *Ech_out, double *mdot_out) {
  if (R < 1 || branch < 0 || branch > 2) return ORA_EINVAL;
  const double Lfrob = ora_frobenius(H, R);
  int64_t E = 0, Ech = 0;
  int fail = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : E, Ech)
  for (int64_t i = 0; i < I; i++) {
    double *u = F + i * R;
    double *zp = zprev + i * R;
    const double *m = M + i * R;
    double *u0 = NULL;
    if (jacobi) {
      u0 = (double *)malloc(sizeof(double) * (size_t)R);
      if (!u0) { fail = 1; continue; }
      memcpy(u0, u, sizeof(double) * (size_t)R);
    }
    for (int r = 0; r < R; r++) {
      const double h = H[r * R + r];
      double z = 0.0;
      int sel = 0;
      if (h != 0.0) {
        double s = 0.0;
        for (int j = 0; j < R; j++) s += (jacobi ? u0[j] : u[j]) * H[j * R + r];
        const double g = -m[r] + s;
        const double unew = fmax(0.0, u[r] - g / h);
        const double uhat = unew - u[r];
        const double L = (l_mode == 0) ? h : Lfrob;
        z = -g * uhat - (L / 2.0) * uhat * uhat;
        if (branch == BR_FIRST) sel = z > 0.0;
        else if (branch == BR_EQ24) sel = (z - zp[r]) > 0.0;
        else sel = (zp[r] - z) > 0.0;
        if (sel) {
          E += 1;
          if (uhat != 0.0) Ech += 1;
          u[r] = unew;
        }
      }
      zp[r] = z;
      if (decisions) decisions[i * R + r] = (uint8_t)sel;
    }
    free(u0);
  }
  if (fail) return ORA_ENOMEM;
  /* Eq 25: ti^k = sum_q sum_r z^k_qr, sequential row-major order */
  double ti = 0.0, mdot = 0.0;
  for (int64_t x = 0; x < I * R; x++) ti += zprev[x];
  for (int64_t x = 0; x < I * R; x++) mdot += F[x] * M[x];
  *ti_out = ti;
  *E_out = E;
  *Ech_out = Ech;
  if (mdot_out) *mdot_out = mdot;
  return ORA_OK;
}

/* ------------------------------------------------------------------ snapshot-scored pass
 * SURVEY 8(f) f4 / DESIGN.md reading C10': the exact-timing alternative to the lagged ti.
 * Alg 1 computes G (hence every gradient) once per mode pass, so every z^k_qr of
 * Eq 20 is known before any selection and ti^k (Eq 25) can gate the same pass
 * (Eq 27 if ti^k > ti^{k-1}; else Eq 24; k == 1: z > 0):
 *   (1) snapshot  zs_qr = -g0*d0 - (L/2)*d0^2 with g0 = -m_qr + sum_j u0_qj h_jr from the
 *       rows at pass start (u0) and d0 = max(0, u0_qr - g0/h_rr) - u0_qr; zs = 0 if h_rr == 0;
 *   (2) ti^k = sum of zs in row-major order; branch from (first, ti^k, ti_prev);
 *   (3) for each row, r = 0..R-1 in order: sel by the branch on (zs_qr, zprev_qr); a
 *       selected element takes the Gauss-Seidel step of the CURRENT row (Eq 14 with
 *       columns < r updated, Eq 11-13), so each applied update is an exact coordinate
 *       minimisation and f stays non-increasing; zprev_qr <- zs_qr.
 * Outputs as ora_mode_pass, plus the branch it chose. */
int ora_mode_pass_snapshot(int64_t I, int R, const double *M, const double *H, double *F, double *zprev,
                           int first, double ti_prev, int branch_override, int l_mode, uint8_t *decisions,
                           double *ti_out, int64_t *E_out, int64_t *Ech_out, double *mdot_out, int *branch_out) {
  if (R < 1) return ORA_EINVAL;
  const double Lfrob = ora_frobenius(H, R);
  double *zs = (double *)malloc(sizeof(double) * (size_t)(I > 0 ? I * R : 1));
  if (!zs) return ORA_ENOMEM;
  /* (1) snapshot importance from the rows at pass start (no update in this loop) */
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < I; i++) {
    const double *u = F + i * R;
    const double *m = M + i * R;
    for (int r = 0; r < R; r++) {
      const double h = H[r * R + r];
      double z = 0.0;
      if (h != 0.0) {
        double s = 0.0;
        for (int j = 0; j < R; j++) s += u[j] * H[j * R + r];
        const double g = -m[r] + s;
        const double uhat = fmax(0.0, u[r] - g / h) - u[r];
        const double L = (l_mode == 0) ? h : Lfrob;
        z = -g * uhat - (L / 2.0) * uhat * uhat;
      }
      zs[i * R + r] = z;
    }
  }
  /* (2) exact-timing total importance and branch */
  double ti = 0.0;
  for (int64_t x = 0; x < I * R; x++) ti += zs[x];
  const int branch = branch_override >= 0 ? branch_override : (first ? BR_FIRST : (ti > ti_prev ? BR_EQ27 : BR_EQ24));
  if (branch < 0 || branch > 2) { free(zs); return ORA_EINVAL; }
  /* (3) Gauss-Seidel pass gated by the snapshot */
  int64_t E = 0, Ech = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : E, Ech)
  for (int64_t i = 0; i < I; i++) {
    double *u = F + i * R;
    double *zp = zprev + i * R;
    const double *m = M + i * R;
    for (int r = 0; r < R; r++) {
      const double h = H[r * R + r];
      const double z = zs[i * R + r];
      int sel = 0;
      if (h != 0.0) {
        if (branch == BR_FIRST) sel = z > 0.0;
        else if (branch == BR_EQ24) sel = (z - zp[r]) > 0.0;
        else sel = (zp[r] - z) > 0.0;
        if (sel) {
          double s = 0.0;
          for (int j = 0; j < R; j++) s += u[j] * H[j * R + r];
          const double g = -m[r] + s;
          const double unew = fmax(0.0, u[r] - g / h);
          E += 1;
          if (unew != u[r]) Ech += 1;
          u[r] = unew;
        }
      }
      zp[r] = z;
      if (decisions) decisions[i * R + r] = (uint8_t)sel;
    }
  }
  double mdot = 0.0;
  for (int64_t x = 0; x < I * R; x++) mdot += F[x] * M[x];
  free(zs);
  *ti_out = ti;
  *E_out = E;
  *Ech_out = Ech;
  if (mdot_out) *mdot_out = mdot;
  if (branch_out) *branch_out = branch;
  return ORA_OK;
}

/* Reading C10: branch at sweep k (1-based) for a mode whose total-importance history is
 * ti_hist[0..k-2] (ti^1 .. ti^{k-1}). */
int ora_branch(int k, const double *ti_hist, int variant) {
  if (variant == VAR_SELECT_OFF || k == 1) return BR_FIRST;
  if (k == 2) return BR_EQ24;
  return (ti_hist[k - 2] > ti_hist[k - 3]) ? BR_EQ27 : BR_EQ24;
}

/* ------------------------------------------------------------------ objective
 * Eq 6-7 over ALL cells (C1), absent cells = 0, by brute force.  Tiny only. */
int ora_objective_dense(const int64_t dims[3], int64_t nnz, const uint32_t *coords, const float *vals,
                        const double *U, const double *V, const double *W, int R, double *f_out) {
  const int64_t Q = dims[0], P = dims[1], S = dims[2];
  double *X = (double *)calloc((size_t)(Q * P * S), sizeof(double));
  if (!X) return ORA_ENOMEM;
  for (int64_t e = 0; e < nnz; e++)
    X[((int64_t)coords[3 * e] * P + coords[3 * e + 1]) * S + coords[3 * e + 2]] = (double)vals[e];
  double f = 0.0;
  for (int64_t q = 0; q < Q; q++)
    for (int64_t p = 0; p < P; p++)
      for (int64_t s = 0; s < S; s++) {
        double xh = 0.0; /* Eq 8 */
        for (int r = 0; r < R; r++) xh += U[q * R + r] * V[p * R + r] * W[s * R + r];
        const double d = X[(q * P + p) * S + s] - xh;
        f += d * d;
      }
  free(X);
  *f_out = f;
  return ORA_OK;
}

/* sum_{r,t} (G_U * G_V * G_W)_{rt} = ||[[U,V,W]]||^2 */
static double model_norm2(const double *GU, const double *GV, const double *GW, int R) {
  double s = 0.0;
  for (int64_t x = 0; x < (int64_t)R * R; x++) s += GU[x] * GV[x] * GW[x];
  return s;
}

/* Sparse-explicit form: sum_Omega (x - xhat)^2 + (||[[U,V,W]]||^2 - sum_Omega xhat^2). */
int ora_objective_sparse(const int64_t dims[3], int64_t nnz, const uint32_t *coords, const float *vals,
                         const double *U, const double *V, const double *W, int R, double *f_out) {
  double *G[3];
  const double *F[3] = {U, V, W};
  for (int n = 0; n < 3; n++) {
    G[n] = (double *)malloc(sizeof(double) * (size_t)R * R);
    if (!G[n]) return ORA_ENOMEM;
    ora_gram(F[n], dims[n], R, G[n]);
  }
  /* sum over Omega in 64 fixed, contiguous chunks (each sequential), then the chunks in
     order: the result does not depend on the thread count */
  enum { NCH = 64 };
  double cse[NCH], csx[NCH];
#pragma omp parallel for schedule(static)
  for (int ch = 0; ch < NCH; ch++) {
    const int64_t e0 = nnz * ch / NCH, e1 = nnz * (ch + 1) / NCH;
    double a = 0.0, b = 0.0;
    for (int64_t e = e0; e < e1; e++) {
      double xh = 0.0;
      for (int r = 0; r < R; r++)
        xh += U[(int64_t)coords[3 * e] * R + r] * V[(int64_t)coords[3 * e + 1] * R + r] *
              W[(int64_t)coords[3 * e + 2] * R + r];
      const double d = (double)vals[e] - xh;
      a += d * d;
      b += xh * xh;
    }
    cse[ch] = a;
    csx[ch] = b;
  }
  double se = 0.0, sx2 = 0.0;
  for (int ch = 0; ch < NCH; ch++) {
    se += cse[ch];
    sx2 += csx[ch];
  }
  *f_out = se + (model_norm2(G[0], G[1], G[2], R) - sx2);
  for (int n = 0; n < 3; n++) free(G[n]);
  return ORA_OK;
}

/* ------------------------------------------------------------------ held-out evaluation
 * Eq 8: xhat_qps = sum_{r=1}^R u_qr v_pr w_sr, summed over r in order.
 * out[e] for the n test coordinates (u32 [n][3]); each index must be in range. */
int ora_predict(int64_t n, const uint32_t *coords, const int64_t dims[3], const double *U, const double *V,
                const double *W, int R, double *out) {
  for (int64_t e = 0; e < n; e++)
    for (int m = 0; m < 3; m++)
      if ((int64_t)coords[3 * e + m] >= dims[m]) return ORA_ERANGE;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < n; e++) {
    double xh = 0.0;
    for (int r = 0; r < R; r++)
      xh += U[(int64_t)coords[3 * e] * R + r] * V[(int64_t)coords[3 * e + 1] * R + r] *
            W[(int64_t)coords[3 * e + 2] * R + r];
    out[e] = xh;
  }
  return ORA_OK;
}

/* Eq 30: RMSE = sqrt( sum (x_test - xhat_test)^2 / n ), the squared errors summed
 * sequentially in test-entry order.  n = 0 gives 0. */
int ora_rmse(int64_t n, const uint32_t *coords, const float *vals, const int64_t dims[3], const double *U,
             const double *V, const double *W, int R, double *rmse_out) {
  double *xh = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (!xh) return ORA_ENOMEM;
  int rc = ora_predict(n, coords, dims, U, V, W, R, xh);
  if (rc != ORA_OK) {
    free(xh);
    return rc;
  }
  double se = 0.0;
  for (int64_t e = 0; e < n; e++) {
    const double d = (double)vals[e] - xh[e];
    se += d * d;
  }
  *rmse_out = n > 0 ? sqrt(se / (double)n) : 0.0;
  free(xh);
  return ORA_OK;
}

/* ------------------------------------------------------------------ full SaCD run
 * Alg 1 under readings C1-C17: K sweeps, each updating U, V, W in turn.
 * In:  tensor (coords u32 [nnz][3], vals f32), dims, R, seed (init), K, l_mode, variant.
 *      If init != NULL it holds the initial factors (U | V | W concatenated, row-major)
 *      instead of the seeded init.
 * Out: U, V, W (row-major I_n x R), f[K+1] (objective after sweep k, k=0 initial),
 *      E, Ech, ti, branch: [K][3].  zprev_out (optional): final z_prev, concatenated.
 *      xnorm2_out: ||X||^2 (mode-0 layout order). */
int ora_sacd_run(int64_t nnz, const uint32_t *coords, const float *vals, const int64_t dims[3], int R,
                 uint64_t seed, int K, int l_mode, int variant, const double *init, double *U, double *V,
                 double *W, double *f, int64_t *E, int64_t *Ech, double *ti, int *branch, double *zprev_out,
                 double *xnorm2_out) {
  if (R < 1 || K < 0) return ORA_EINVAL;
  int rc = ORA_OK;
  double *F[3] = {U, V, W};
  uint32_t *ia[3] = {0}, *ib[3] = {0};
  float *vv[3] = {0};
  int64_t *rp[3] = {0};
  double *zp[3] = {0}, *M[3] = {0}, *G[3] = {0};
  double *H = (double *)malloc(sizeof(double) * (size_t)R * R);
  double *tih = (double *)malloc(sizeof(double) * (size_t)(3 * (K + 1)));
  if (!H || !tih) { rc = ORA_ENOMEM; goto done; }
  for (int n = 0; n < 3; n++) {
    size_t ne = (size_t)(nnz > 0 ? nnz : 1);
    ia[n] = (uint32_t *)malloc(sizeof(uint32_t) * ne);
    ib[n] = (uint32_t *)malloc(sizeof(uint32_t) * ne);
    vv[n] = (float *)malloc(sizeof(float) * ne);
    rp[n] = (int64_t *)malloc(sizeof(int64_t) * (size_t)(dims[n] + 1));
    zp[n] = (double *)calloc((size_t)(dims[n] * R), sizeof(double));
    M[n] = (double *)malloc(sizeof(double) * (size_t)(dims[n] * R));
    G[n] = (double *)malloc(sizeof(double) * (size_t)R * R);
    if (!ia[n] || !ib[n] || !vv[n] || !rp[n] || !zp[n] || !M[n] || !G[n]) { rc = ORA_ENOMEM; goto done; }
    rc = ora_layout(nnz, coords, vals, dims, n, ia[n], ib[n], vv[n], rp[n]);
    if (rc) goto done;
  }
  if (init) {
    const double *p = init;
    for (int n = 0; n < 3; n++) {
      memcpy(F[n], p, sizeof(double) * (size_t)(dims[n] * R));
      p += dims[n] * R;
    }
  } else {
    ora_init_factors(dims, R, seed, U, V, W);
  }
  double xn2 = 0.0;
  for (int64_t e = 0; e < nnz; e++) xn2 += (double)vv[0][e] * (double)vv[0][e];
  if (xnorm2_out) *xnorm2_out = xn2;
  /* f^0 */
  for (int n = 0; n < 3; n++) ora_gram(F[n], dims[n], R, G[n]);
  {
    int a, b;
    ora_other_modes(dims, 2, &a, &b);
    ora_mttkrp(dims[2], R, rp[2], ia[2], ib[2], vv[2], F[a], F[b], M[2]);
    double ip = 0.0;
    for (int64_t x = 0; x < dims[2] * R; x++) ip += W[x] * M[2][x];
    f[0] = xn2 - 2.0 * ip + model_norm2(G[0], G[1], G[2], R);
  }
  for (int k = 1; k <= K; k++) {
    double mdot = 0.0;
    for (int n = 0; n < 3; n++) {
      int a, b;
      ora_other_modes(dims, n, &a, &b);
      /* Grams of the CURRENT other factors (U^k, V^k already updated this sweep) */
      ora_gram(F[a], dims[a], R, G[a]);
      ora_gram(F[b], dims[b], R, G[b]);
      ora_hadamard(G[a], G[b], (int64_t)R * R, H);
      ora_mttkrp(dims[n], R, rp[n], ia[n], ib[n], vv[n], F[a], F[b], M[n]);
      int br;
      double tk;
      int64_t e1, e2;
      if (variant == VAR_SNAPSHOT) {
        rc = ora_mode_pass_snapshot(dims[n], R, M[n], H, F[n], zp[n], k == 1, k > 1 ? tih[n * (K + 1) + (k - 2)] : 0.0,
                                    -1, l_mode, NULL, &tk, &e1, &e2, &mdot, &br);
      } else {
        br = ora_branch(k, tih + n * (K + 1), variant);
        rc = ora_mode_pass(dims[n], R, M[n], H, F[n], zp[n], br, l_mode, variant == VAR_JACOBI, NULL, &tk, &e1,
                           &e2, &mdot);
      }
      if (rc) goto done;
      tih[n * (K + 1) + (k - 1)] = tk;
      ti[(k - 1) * 3 + n] = tk;
      E[(k - 1) * 3 + n] = e1;
      Ech[(k - 1) * 3 + n] = e2;
      branch[(k - 1) * 3 + n] = br;
    }
    /* objective after the W pass: m^W depends only on U^k, V^k, so <X, Xhat> = sum w . m^W */
    for (int n = 0; n < 3; n++) ora_gram(F[n], dims[n], R, G[n]);
    f[k] = xn2 - 2.0 * mdot + model_norm2(G[0], G[1], G[2], R);
  }
  if (zprev_out) {
    double *p = zprev_out;
    for (int n = 0; n < 3; n++) {
      memcpy(p, zp[n], sizeof(double) * (size_t)(dims[n] * R));
      p += dims[n] * R;
    }
  }
done:
  for (int n = 0; n < 3; n++) {
    free(ia[n]); free(ib[n]); free(vv[n]); free(rp[n]); free(zp[n]); free(M[n]); free(G[n]);
  }
  free(H);
  free(tih);
  return rc;
}
