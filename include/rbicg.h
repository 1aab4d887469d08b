/*
 * rbicg.h -- C ABI of the B200-native recycling BiCG (RBiCG) hot path.
 *
 * Method: Ahuja, de Sturler, Gugercin, Chang, "Recycling BiCG" (arXiv
 * 1010.0762); citations "P:n" are lines of that paper's PAPER.md.
 *
 *   * Problem: a sequence of dual systems A x = b, A^* x~ = b~.
 *   * Iteration: Algorithm 2 with the augmented bi-Lanczos
 *     relations and the oblique projections against C, C~.
 *   * Recycle space: harmonic Ritz vectors, first-system cases
 *     (P:614-684), bi-orthogonal C, C~ by SVD.
 *   * Bilinear form u^*A^{-1}w.
 *
 * Conventions shared by every entry point
 *   - Scalars: RBICG_F64 = IEEE double; RBICG_C128 = interleaved (re, im)
 *     doubles.  Inner product (u, v) = u^* v (reading Q1).
 *   - Vectors are contiguous arrays of n scalars.  n x k blocks (U, Ũ) are
 *     COLUMN-major with leading dimension n in this ABI (the library keeps its
 *     own row-major device copies).
 *   - Pointers are host or device memory according to the `on_device` flag of
 *     the call (device pointers must be from the ctx's device).  The caller
 *     owns every array it passes; the library reads/writes them on the ctx
 *     stream and every call returns only once its outputs are host-visible
 *     (the call synchronises the ctx stream before returning).
 *   - Handles (ctx, mat, rec) are owned by the library until the matching
 *     *_free / rbicg_finalize.  One ctx per host thread.
 *   - Errors: no exception crosses the ABI.  Return value 0 = success,
 *     > 0 = numerical outcome with valid outputs, < 0 = error (outputs
 *     undefined, recycle state unchanged where possible).  rbicg_strerror()
 *     gives a static message.
 *   - Every step of the solve runs in this library's sm_100a kernels; the only
 *     host arithmetic is the small dense cycle-end control work (the
 *     generalised eigenproblem of order k+s and the k x k SVD, LAPACK via
 *     dlopen of the OpenBLAS shipped with scipy; path from $RBICG_LAPACK).
 */
#ifndef RBICG_H
#define RBICG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  RBICG_OK = 0,
  RBICG_MAXITER = 1,            /* max_itn reached; outputs = last iterate   */
  RBICG_BREAKDOWN_SERIOUS = 2,  /* (r~_i, r_i) = 0                    */
  RBICG_BREAKDOWN_SECOND = 3,   /* (p~_i, q_i) = 0                */
  RBICG_RECYCLE_EMPTY = 4,      /* p = 0 after truncation (P:702 footnote);  */
                                /* solve valid, returned basis has k = 0     */
  RBICG_EINVAL = -1,
  RBICG_ENOMEM = -2,
  RBICG_ECUDA = -3,
  RBICG_ENCCL = -4,
  RBICG_ELAPACK = -5,
  RBICG_ESTATE = -6
};

typedef enum { RBICG_F64 = 0, RBICG_C128 = 1 } rbicg_dtype;

typedef struct rbicg_ctx rbicg_ctx;
typedef struct rbicg_mat rbicg_mat;
typedef struct rbicg_rec rbicg_rec;

/* Multi-GPU row partition.  NULL or nranks == 1 = one GPU.
 *   mode 0: one process per GPU; NCCL communicator from nccl_id (the
 *           ncclUniqueId of rbicg_nccl_unique_id on rank 0, broadcast by the
 *           caller); this process is `rank`.  Collectives are stream-ordered
 *           and captured in the loop's CUDA graph.
 *   mode 1: "virtual ranks" -- nranks contexts in ONE process, one host
 *           thread each (normally all on one GPU), meeting at host barriers;
 *           nccl_id is any 128-byte token shared by the group.  Every
 *           collective synchronises its stream (no graph, no kernel ever
 *           waits on another); sums are taken in rank order.  For testing the
 *           partitioned path where fewer GPUs than ranks exist.
 * Rows are split evenly: rank q owns [floor(q n/P), floor((q+1) n/P)).
 * Partitioned calls are collective: every rank makes the same calls in the
 * same order.  rbicg_matrix_csr takes ONLY the rank's block of rows (local
 * rowptr, GLOBAL column indices, local values; blocks are contiguous and in
 * rank order, of any sizes -- the library gathers the sizes): the rows of A^*
 * in the block are assembled on the device from the rank's entries plus the
 * entries of A in its columns held by other ranks, exchanged over the
 * communicator; the ghost/send plan is cached per context while the block's
 * sparsity pattern (hashed on the device) repeats.  Vectors (b, x, u, w, ...)
 * and recycle blocks are the rank's own rows; scalar results are replicated.
 * The dbg_project and dbg_time_kernels hooks are single-GPU only
 * (RBICG_EINVAL).  row_begin/row_end are informative. */
typedef struct {
  int32_t rank, nranks;
  uint8_t nccl_id[128];
  int64_t row_begin, row_end;
  int32_t mode;
  int32_t force_partition; /* 1: the partitioned code path even with nranks == 1
                              (one-rank NCCL communicator: the collective plumbing,
                              graph capture and split reductions on one GPU) */
} rbicg_dist;

typedef struct {
  int32_t k;              /* recycle width (0 = plain BiCG, Algorithm 1)      */
  int32_t s;              /* cycle length, >= 2                        */
  int32_t max_itn;        /* iteration cap                             */
  double tol;             /* relative: ||r|| <= tol ||b|| and ||r~|| <= tol ||b~|| (Q2) */
  double trunc_tol;       /* keep sigma_i >= trunc_tol of the column-normalised
                             Gram C~^*C (reading Q13)                   */
  uint64_t seed;          /* unused by the library (random draws are inputs)  */
  int32_t update_recycle; /* build U_j, Ũ_j at cycle ends (§4)                 */
  int32_t record_history; /* fill `hist` when non-NULL                         */
  int32_t force_iters;    /* > 0: run exactly this many iterations, stop test
                             off (parity protocol Q27); 0 = normal            */
  int32_t pencil;         /* cycle-end pencil assembly with a recycle space:
                             0 = explicit Grams Ψ~^*Ψ, Ψ~^*Φ of the stored
                             vectors (plain, reading Q15); 1 = the §4.4
                             recurrences: carried small blocks,
                             only Ῡ_j^*U_{j-1} and, once per system,
                             C~^*U are O(n) products                       */
} rbicg_opts;

typedef struct {
  int32_t status, iterations, cycles, k_in, k_out;
  double relres_rec, relres_dual_rec;    /* recursive ||r||/||b||, ||r~||/||b~|| */
  double relres_true, relres_dual_true;  /* after step 7            */
  double t_loop_ms, t_cycle_dev_ms, t_host_eig_ms, t_refresh_ms, t_total_ms;
  double alg_bytes;                       /* algorithmic HBM bytes of the loop */
  int32_t kernel_launches;                /* kernels launched by this call     */
  int32_t lookahead_cancellations;        /* fused iteration: iterations whose look-ahead
                                             ρ_i expansion cancelled to < 1e3 eps of its
                                             terms (β_i inexact)    */
} rbicg_result;

/* Create a context on `device`, adopting `cuda_stream` (a cudaStream_t, NULL
 * = the legacy default stream).  dist may be NULL.  Returns RBICG_ECUDA if the
 * device cannot be used. */
int rbicg_init(rbicg_ctx **ctx, int device, void *cuda_stream,
               const rbicg_dist *dist);
int rbicg_finalize(rbicg_ctx *ctx);

/* Build the device matrix store of A (SELL-32 layout, rebuilt per system,
 * P:44-52) and its explicit conjugate transpose A^* (BASELINE.json (1)).
 * rowptr[n+1], colind[nnz] are int32 CSR (columns need not be sorted; n and
 * nnz < 2^31), val[nnz] of `dtype`.  on_device selects where the three
 * arrays live.  The matrix is immutable once built.  On a partitioned
 * context n and nnz count the rank's block of rows only and colind holds
 * global column indices (see rbicg_dist); the global order is the sum of the
 * blocks (< 2^31).  Collective there. */
int rbicg_matrix_csr(rbicg_ctx *ctx, int64_t n, int64_t nnz,
                     const int32_t *rowptr, const int32_t *colind,
                     const void *val, rbicg_dtype dtype, int on_device,
                     rbicg_mat **A);
int rbicg_matrix_free(rbicg_mat *A);

/* Recycle space handle (U, Ũ) with room for k_max columns; starts empty. */
int rbicg_recycle_new(rbicg_ctx *ctx, int64_t n, int32_t k_max,
                      rbicg_dtype dtype, rbicg_rec **R);
/* Copy out the current basis (k columns, column-major n x k each). */
int rbicg_recycle_export(const rbicg_rec *R, int32_t *k, void *U, void *Ut,
                         int on_device);
/* Replace the basis by (U, Ũ) (column-major n x k, k <= k_max). */
int rbicg_recycle_import(rbicg_rec *R, int32_t k, const void *U,
                         const void *Ut, int on_device);
int rbicg_recycle_free(rbicg_rec *R);

/* Solve the dual pair A x = b, A^* x~ = b~ with RBiCG (Algorithm 2) using the
 * recycle space in R (refreshed for this A: C = AU, C~ = A^*Ũ, SVD),
 * and (if opts->update_recycle) replace R by the recycle space built during
 * this solve (the last full cycle's U_j, Ũ_j, reading Q18).
 *   x, xt   in: x_{-1}, x~_{-1}; out: solution after step 7.
 *   xt_redraw  nullable; the random x~_{-1} used once if (r_0, r~_0) = 0
 *           (Algorithm 2 step 3; reading Q4).
 *   hist    nullable [max_itn][6] doubles: ||r_i||/||b||, ||r~_i||/||b~||,
 *           Re a_i, Im a_i, Re b_i, Im b_i.
 * All of b, bt, x, xt, xt_redraw, hist live on host or device per on_device. */
int rbicg_solve_dual(rbicg_ctx *ctx, const rbicg_mat *A, const void *b,
                     const void *bt, void *x, void *xt, const void *xt_redraw,
                     rbicg_rec *R, const rbicg_opts *opts, int on_device,
                     rbicg_result *res, double *hist);

/* Split preconditioning (the paper's experiments,
 * PAPER.md:1330-1333, :1406-1409).  rbicg_prec_ilut factors the n x n CSR
 * (host or device arrays; same conventions as rbicg_matrix_csr) by Crout ILU
 * with threshold droptol (ILUC, no pivoting; drop rule of the paper's Matlab:
 * off-diagonal U(k, j) kept if |u| >= droptol ||A(:, j)||, L(i, k) kept if
 * |l| >= droptol ||A(:, k)|| before the division by the pivot; droptol = 0 is
 * the exact LU).  Host factorisation (per-system setup), device factors L, U
 * and their conjugate transposes.  RBICG_EINVAL on a zero pivot or on a
 * partitioned context.  rbicg_prec_export copies L (which = 0: strictly lower
 * part, unit diagonal implied) or U (which = 1) to host CSR; two-call (NULL
 * arrays: *nnz only).
 * rbicg_solve_dual_pc runs Algorithm 2 on the split-preconditioned pair
 *   (L^{-1} A U^{-1}) x̂ = L^{-1} b,   (L^{-1} A U^{-1})^* x̂~ = U^{-*} b~,
 * x_{-1}, x~_{-1} mapped to x̂ = U x, x̂~ = L^* x~ and back after step 7; the
 * recycle space in R, the stop test and the true residuals belong to the
 * preconditioned pair (readings Q33, Q34).  Same arguments as
 * rbicg_solve_dual; P = NULL is rbicg_solve_dual.  One GPU only. */
typedef struct rbicg_prec rbicg_prec;
int rbicg_prec_ilut(rbicg_ctx *ctx, int64_t n, int64_t nnz, const int32_t *rowptr,
                    const int32_t *colind, const void *val, rbicg_dtype dtype,
                    double droptol, int on_device, rbicg_prec **P);
int rbicg_prec_free(rbicg_prec *P);
int rbicg_prec_export(const rbicg_prec *P, int which, int32_t *rowptr,
                      int32_t *colind, void *val, int64_t *nnz);
int rbicg_solve_dual_pc(rbicg_ctx *ctx, const rbicg_mat *A, const rbicg_prec *P,
                        const void *b, const void *bt, void *x, void *xt,
                        const void *xt_redraw, rbicg_rec *R,
                        const rbicg_opts *opts, int on_device,
                        rbicg_result *res, double *hist);

/* u^* A^{-1} w from the dual pair A x = w, A^* x~ = u, estimator
 * u^*x + x~^*(w - Ax) (reading Q19).  value: one scalar of A's dtype (host).
 * x, xt: nullable outputs (initial guesses are zero). */
int rbicg_bilinear(rbicg_ctx *ctx, const rbicg_mat *A, const void *u,
                   const void *w, rbicg_rec *R, const rbicg_opts *opts,
                   int on_device, void *value, rbicg_result *res);

/* IRKA support (Algorithm 3; the model
 * G(s) = c^*(sI - A)^{-1} b with E = I).
 * rbicg_matrix_shifted_csr builds the store of sigma I - A directly from the
 * CSR of A (the shifted system of one IRKA shift): the same
 * arguments as rbicg_matrix_csr plus sigma = (sigma_re, sigma_im); every
 * entry is negated and sigma added on the diagonal, on the device, before the
 * SELL build.  Every row must hold its diagonal entry once (RBICG_EINVAL
 * otherwise); sigma_im must be 0 for RBICG_F64.  One GPU only.
 * rbicg_reduced_model forms the projected model of step 2d:
 *   Ar = W^* A V,  Er = W^* V (E = I, reading Q20),  br = W^* b,  cr = V^* c
 * with V = [v_1 .. v_r], W = [w_1 .. w_r] the primal and dual solutions of
 * the r shifted pairs (each column contiguous: column i at V + i n), b, c of
 * length n, all of A's dtype on the device (on_device = 1) or host.  A v_i
 * runs the library's SpMV, the products its Gram kernel.  Outputs are host
 * arrays of A's dtype: Ar, Er row-major r x r, br, cr of length r.
 * 1 <= r <= 32.  One GPU only (RBICG_EINVAL on a partitioned context). */
int rbicg_matrix_shifted_csr(rbicg_ctx *ctx, int64_t n, int64_t nnz,
                             const int32_t *rowptr, const int32_t *colind,
                             const void *val, rbicg_dtype dtype,
                             double sigma_re, double sigma_im, int on_device,
                             rbicg_mat **A);
int rbicg_reduced_model(rbicg_ctx *ctx, const rbicg_mat *A, int32_t r,
                        const void *V, const void *W, const void *b,
                        const void *c, int on_device, void *Ar, void *Er,
                        void *br, void *cr);

/* Parity hooks (per-call checks, BASELINE.json: 1e-12 relative).
 * spmv_pair: z = A p, zt = A^* pt.
 * project: given R's refreshed basis for A, zeta = D_c^{-1} C~^* z and
 *   zetat = D_c^{-1} C^* zt; also returns the refreshed basis
 *   (column-major) in U, Ut, C, Ct (nullable) and D_c in d (nullable). */
int rbicg_dbg_spmv_pair(rbicg_ctx *ctx, const rbicg_mat *A, const void *p,
                        const void *pt, void *z, void *zt, int on_device);
int rbicg_dbg_project(rbicg_ctx *ctx, const rbicg_mat *A, rbicg_rec *R,
                      double trunc_tol, const void *z, const void *zt,
                      void *zeta, void *zetat, int32_t *k_out, void *U,
                      void *Ut, void *C, void *Ct, double *d, int on_device);

/* Per-kernel CUDA-event timing of `iters` hot-loop iterations (stop test off)
 * on a fresh state for this matrix and R's recycle space (bench roofline).
 * ms[13] out: [0] average duration (ms) of the SpMV-pair + coefficient kernel,
 * [1] of the update kernel, [2] 0 if every timed launch did full work,
 * [3] active recycle width k, [4] 1 if x is rebuilt lazily (the update kernel
 * does not touch x, p), [5] 1 if pass 1 stages matrix tiles via TMA,
 * [6] ms per iteration when the same `iters` iterations (restarted from the
 * initial state) run as one captured CUDA graph with no events between the
 * kernels, the way the solver runs its cycles, [7] 0 if that graph run did
 * full work, [8], [9] unused (-1), [10] ms per launch of the SpMV-pair
 * kernel alone as `iters` back-to-back launches in one graph (its duration
 * inside the solver's graph, without host launch gaps), [11] the same for the
 * update kernel, [12] 0 if those launches all did full work, [13] 1 if A and
 * A^* share one SELL column array (structurally symmetric A: pass 1 streams
 * one pattern and two value arrays), [14] ms per launch of the fused
 * iteration kernel (one kernel per iteration while no recycle space is
 * active; -1 when that form does not apply) as `iters` launches in one graph,
 * [15] 0 if those launches all did full work, [16] 1 if the fused kernel
 * streams int16 column deltas (banded A with a shared column array).  ms must
 * hold 17 doubles. */
int rbicg_dbg_time_kernels(rbicg_ctx *ctx, const rbicg_mat *A, rbicg_rec *R,
                           const rbicg_opts *opts, int iters, double *ms);

/* Host-only partition plan (no GPU needed): for `rank` of `nranks` even row
 * blocks of the n x n CSR (global column indices), the ghost columns of the
 * SpMV pair (columns of local rows of A and A^* owned elsewhere, sorted), the
 * owners they are received from and the own rows sent to each neighbour.
 * Two-call pattern: counts[6] = {row_begin, row_end, nghost, nrecv_nbr,
 * nsend_nbr, nsend_idx}; array outputs may be NULL.  send_idx holds local
 * row indices, concatenated per send neighbour in that neighbour's ghost
 * order. */
int rbicg_plan_partition(int64_t n, const int32_t *rowptr, const int32_t *colind,
                         int32_t nranks, int32_t rank, int64_t *counts, int64_t *ghost,
                         int32_t *recv_nbr, int64_t *recv_cnt, int32_t *send_nbr,
                         int64_t *send_cnt, int32_t *send_idx);

/* 128-byte ncclUniqueId for a mode-0 group (call on rank 0, broadcast it).
 * RBICG_ENCCL if NCCL cannot be loaded ($RBICG_NCCL or libnccl.so.2). */
int rbicg_nccl_unique_id(uint8_t *id);

const char *rbicg_strerror(int status);
/* Kernel launches issued through this library since load (driver evidence). */
int64_t rbicg_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* RBICG_H */
