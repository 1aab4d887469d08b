// internal.h -- library-internal types shared by the RBiCG translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <complex>
#include <vector>
#include <string>
#include <memory>

#include "common.cuh"
#include "comm.h"

namespace rbicg {

constexpr int KMAX = 32;   // maximum recycle width supported by the kernels
constexpr int BS = 256;    // threads per block of the streaming kernels
constexpr int TRH = BS / 2;  // rows per tile of the split form of pass 1
// number of pass-1 sums: C~^*z, C^*z~, C^*p~ (k each), p~^*z, and the Q32
// sums C~^*r_{i-1}, C^*r~_{i-1} (k each)
__host__ __device__ __forceinline__ int p1_nsums(int k) { return 5 * k + 1; }

// SELL-32 matrix (slices of 32 consecutive rows, column-major inside a slice,
// zero-padded to the slice's longest row; sigma = 1, i.e. no row sorting, so
// vectors keep their natural order).
struct DevMat {
  int64_t n = 0, nslices = 0, padded = 0;
  int tile_max = 0;         // max elements in one 256-row tile (8 slices)
  int tile_max_h = 0;       // max elements in one 128-row tile (4 slices)
  int max_w = 0;            // widest slice (padded row length)
  int64_t *sptr = nullptr;  // nslices + 1 element offsets (multiples of 32)
  int32_t *cols = nullptr;
  void *vals = nullptr;
  int64_t bandwidth = -1;   // max |col - row| of A (-1: unknown, e.g. a row partition)
  int16_t *dcols = nullptr; // col - row as int16 (banded A with one shared column array;
                            // the fused kernel streams these instead of cols)
  int cols_shared = 0;      // cols aliases the other matrix's (A^* of a structurally
                            // symmetric A: same SELL column array, build_t)
};

// Device-resident iteration state (one per solve; scalars of Algorithm 2).
template <typename T>
struct DevState {
  int iter;      // completed iterations i
  int kidx;      // fused form: k_fused launches that did work (K(i), i = kidx + 1 next)
  int la_cancel; // fused form: iterations whose look-ahead ρ_i expansion cancelled (|ρ_ext| <
                 //   1e3 eps (|ρ_{i-1}| + |α||(r~,z)| + |α||(z~,r)| + |α|²|(z~,z)|)): β_i inexact
  int done;      // 0 running, 1 finished, 2 paused at a cycle boundary
  int status;    // RBICG_* of the finished iteration
  int max_itn;
  int force;     // stop test disabled (Q27 protocol)
  int stop_at;   // pause after this iteration (cycle boundary)
  int k;
  int seg_start;   // lazy x: first iteration index of the open segment
  unsigned cnt[4];
  int g1;        // halo overlap: blocks of the interior launch (LoopArgs::phase)
  T rho, beta, alpha, sigma;   // ρ_{i}, β_{i}, α_i, σ_i
  double rnorm, rtnorm;        // ||r_i||, ||r~_i||
  double tolb, tolbt;          // tol ||b||, tol ||b~||
  double bn2, btn2, rn2, rtn2; // squared norms from the residual kernel
  T gam[KMAX], gamt[KMAX];     // γ_i = α_iζ_i - g_{i-1}, γ~_i = ᾱ_iζ~_i - g~_{i-1} (pass 2:
                               //   r_i = r_{i-1} - α_i z_i + C γ_i; Q32, hot.cuh)
  T zc[KMAX], ztc[KMAX];       // ζ_c, ζ~_c
  T g[KMAX], gt[KMAX];         // Ĉ^*r_{-1}, Č^*r~_{-1} (minusXR)
  double dinv[KMAX];           // D_c^{-1}
};

template <typename T>
struct IterRec {   // per-iteration record (index i; record 0 = init)
  T alpha, beta, rho, sigma;
  double rnorm, rtnorm;
};

template <typename T>
struct LoopArgs {
  int64_t n;
  int k, ring, G;
  int64_t ldr;             // ring column stride (n rounded up to 32)
  int staged, tile_max;    // pass 1 stages SELL tiles in smem via TMA
  int split, tile_max_h;   // pass 1 in the split form: 128-row tiles, one thread per row and matrix
  int p1_stages;           // TMA stages of SELL tiles in pass 1 (1 or 2)
  int stage_v;             // pass-1 stages also carry the tile's rows of r, p, r~, p~
  int stage_c;             // pass 1 also bulk-copies the C, C~ rows of each tile
  int l2ef;                // matrix tiles loaded with an L2 evict-first policy
  int pf;                  // pass 1 prefetches the next tile's vector rows into L2
  int abl;                 // timing ablations (RBICG_ABL, never set in a solve): 1 no gathers
  int pass2_tma;           // pass 2 streams its tiles through smem via TMA
  int shared_cols;         // A and A^* share one SELL column array (structurally symmetric A)
  int tile_contig;         // fused form: contiguous tile runs per CTA instead of grid-strided
  const int16_t *dcols;    // fused form: int16 column deltas (null: int32 columns)
  int lazy_x;              // x, x~ rebuilt per segment from the Lanczos ring
  T *pseg[2], *ptseg[2];   // p_a, p~_a at the start of the open segment, by segment parity
  int cyc;                 // cycle length s (segment parity = (seg_start / s) & 1)
  int nsm;
  DevMat A, AH;
  T *rring, *rtring;       // ring of residual columns (r_m in column m % ring)
  T *p[2], *pt[2];         // ping-pong search directions
  T *z, *zt;
  T *zp[2], *ztp[2];       // fused form: per-row nodes {z_i, p_i} by iteration parity, one
                           //   gather per column (128-bit real, 256-bit complex)
  T *x, *xt;
  const T *C, *Ct;         // row-major n x k
  const T *AC, *AHCt;      // fused form with k > 0: A C and A^* C~ (row-major n x k, per system)
  DevState<T> *st;
  IterRec<T> *hist;        // [max_itn + 1]
  T *zhist, *zthist;       // [max_itn + 1][k]
  T *part;                 // block partials [outputs][G]
  int dist;                // row-partitioned: reduction tails write local sums to red
  T *red;                  //   (allreduced, then a one-block leader kernel runs the scalar step)
  // halo overlap (row partition): the tiles of the SpMV kernels are visited in
  // torder (256-row tiles) / torder_h (128-row tiles, split pass 1) -- interior
  // tiles (no ghost column) first -- and one iteration's kernel runs as two
  // launches: [0, nint) while the halo is in flight, [nint, ntiles) after it.
  // ordered = 0: every tile in natural order (one GPU).  phase 1 (interior
  // launch) writes its block partials at part[o * pstride + b] and records its
  // grid size in st->g1; phase 2 (boundary launch, issued after phase 1 has
  // completed) writes at slots g1 + b and its last block reduces all g1 + G2.
  int ordered;
  const int32_t *torder, *torder_h;
  int64_t tbase, tcount;
  int phase, pstride;
};

struct ColDesc {           // one column of an n-row panel: p[row * stride]
  const void *p;
  int64_t stride;
};

}  // namespace rbicg

using cplx = std::complex<double>;

struct rbicg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;       // library stream (non-blocking)
  cudaStream_t user_stream = nullptr;  // caller's stream (may be legacy NULL)
  cudaEvent_t order_ev = nullptr;
  int prio_lo = 0, prio_hi = 0;
  int nsm = 148;
  int grid_stream = 296;  // persistent grid of the streaming kernels
  // reusable device workspace
  void *work = nullptr;
  size_t work_bytes = 0;
  void *host_pinned = nullptr;
  size_t host_bytes = 0;
  // row partition: nranks > 1 -> comm (main loop) and
  // comm_side (cycle-end worker) are set
  int rank = 0, nranks = 1;
  std::unique_ptr<rbicg::Comm> comm, comm_side;
  bool partitioned = false;   // nranks > 1, or forced (rbicg_dist.force_partition)
  bool dist() const { return partitioned; }
  // device buffers of the last solve (bytes, pointer), reused by the next
  std::vector<std::pair<size_t, void *>> arena;
  cudaStream_t side = nullptr;   // cycle-end stream (low priority), kept across solves
  // row partition: the halo exchange runs on halo_stream (fork / join events)
  // while the interior tiles of the iteration's SpMV kernel run
  cudaStream_t halo_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  uint64_t async_key = 0;        // (n, k, s, dtype) of the last device-memory query
  size_t async_avail = 0;        // free + this ctx's idle arena bytes at that query
};

struct rbicg_mat {
  rbicg_ctx *ctx = nullptr;
  int64_t n = 0, nnz = 0;          // rows held here (the row block when partitioned)
  int64_t n_global = 0, row_begin = 0;
  rbicg_dtype dtype = RBICG_F64;
  rbicg::DevMat A, AH;             // partitioned: columns local (own, then ghosts)
  rbicg::HaloPlan halo;            // partitioned: ghost rows / send lists
  // partitioned: tile visiting orders for the halo overlap (LoopArgs::torder):
  // 256-row (ord) and 128-row (ord_h) tiles, interior tiles (no ghost column
  // in A or A^*) first; nint / nint_h interior tiles of ntl / ntl_h
  int32_t *ord = nullptr, *ord_h = nullptr;
  int64_t nint = 0, ntl = 0, nint_h = 0, ntl_h = 0;
};

namespace rbicg {
// one triangular factor of the split preconditioner, device CSR (precond.cu)
struct TriCSR {
  int64_t n = 0, nnz = 0;
  int32_t *rp = nullptr, *ci = nullptr;
  void *v = nullptr;
  int unit = 0;     // unit diagonal (not stored)
  int upper = 0;    // solve backward (rows n-1 .. 0)
  int32_t *order = nullptr;   // rows sorted by dependency level (the solve's claim order)
  int levels = 0;
};
// scratch of the preconditioned operator (one per stream that applies it)
struct PcWork {
  int *flags = nullptr;
  unsigned long long *counter = nullptr;
  void *y = nullptr, *yt = nullptr, *q = nullptr, *qt = nullptr, *v = nullptr, *u = nullptr;
};
}  // namespace rbicg

struct rbicg_prec {   // split preconditioner M = L U ≈ A (NEXT-4, precond.cu)
  rbicg_ctx *ctx = nullptr;
  int64_t n = 0;
  rbicg_dtype dtype = RBICG_F64;
  double droptol = 0;
  rbicg::TriCSR L, U, LH, UH;   // L unit lower, U upper, L^* unit upper, U^* lower
  int64_t nnzL = 0, nnzU = 0;
};

struct rbicg_rec {
  rbicg_ctx *ctx = nullptr;
  int64_t n = 0;
  int32_t kmax = 0, k = 0;
  rbicg_dtype dtype = RBICG_F64;
  void *U = nullptr, *Ut = nullptr;   // device row-major n x k (compact)
};

namespace rbicg {

// ---- matrix.cu
void build_matrix(rbicg_ctx *ctx, int64_t n, int64_t nnz, const int32_t *rowptr_d,
                  const int32_t *col_d, const void *val_d, rbicg_dtype dt, rbicg_mat *M);
void free_devmat(DevMat &m);
// val <- sigma I - A on a device CSR (every row holds its diagonal once, else EINVAL)
void shift_csr_values(rbicg_ctx *ctx, int64_t n, const int32_t *rowptr_d, const int32_t *col_d,
                      void *val_d, rbicg_dtype dt, double sigma_re, double sigma_im);
// partitioned store: local rows of A and of A^* given as CSR (device arrays,
// local column indices in [0, nloc + nghost))
void build_matrix_local(rbicg_ctx *ctx, int64_t nloc, const int32_t *rpA, const int32_t *ciA,
                        const void *vA, const int32_t *rpH, const int32_t *ciH, const void *vH,
                        rbicg_dtype dt, rbicg_mat *M);

// ---- partition.cu: the row-block store of a partitioned context (the block's
// rows of A with GLOBAL columns in; A^* rows by the value halo; halo plan)
void build_partitioned(rbicg_ctx *ctx, int64_t nloc, int64_t nnz, const int32_t *rowptr_d,
                       const int32_t *colind_global_d, const void *val_d, rbicg_dtype dt, rbicg_mat *M);
void forget_partition_plan(const rbicg_ctx *ctx);

// ---- precond.cu (split preconditioning, NEXT-4): Â = L^{-1} A U^{-1}
void pc_build(rbicg_prec *P, const int32_t *rowptr_h, const int32_t *colind_h, const void *val_h);
void pc_free(rbicg_prec *P);
void pc_export(const rbicg_prec *P, int which, int32_t *rp, int32_t *ci, void *v, int64_t *nnz);
void pc_work_alloc(const rbicg_prec *P, PcWork &w);
void pc_work_free(PcWork &w);
// z = Â p and z~ = Â^* p~ (either side may be null); `done`: skip when the
// solver's loop state says finished/paused (nullable)
template <typename T>
void pc_apply_pair(const rbicg_prec *P, const rbicg_mat *M, const T *p, const T *pt, T *z, T *zt, PcWork &w,
                   cudaStream_t s, const int *done);
template <typename T>   // Y = Â X (adj: Â^* X), row-major n x k blocks
void pc_apply_block(const rbicg_prec *P, const rbicg_mat *M, bool adj, const T *X, T *Y, int k, PcWork &w,
                    cudaStream_t s);
template <typename T>   // x = F^{-1} b, F = L, U, L^*, U^* for which = 0..3
void pc_solve_factor(const rbicg_prec *P, int which, const T *b, T *x, PcWork &w, cudaStream_t s);
template <typename T>   // y = F x
void pc_mul_factor(const rbicg_prec *P, int which, const T *x, T *y, cudaStream_t s);

// ---- kernels.cu (launch wrappers; all on ctx->stream)
void prepare_kernels();        // one-time function attributes (not capturable)
void prepare_block_kernels();
int stream_blocks_per_sm();    // occupancy of the streaming kernels
template <typename T> void launch_pass1(const LoopArgs<T> &a, cudaStream_t s);
template <typename T> void launch_pass2(const LoopArgs<T> &a, cudaStream_t s);
template <typename T> void launch_fused(const LoopArgs<T> &a, cudaStream_t s);
template <typename T> void launch_leader_fused(const LoopArgs<T> &a, cudaStream_t s);
template <typename T> void launch_fusedk(const LoopArgs<T> &a, cudaStream_t s);
template <typename T> void launch_pc_pupdate(const LoopArgs<T> &a, T *pfix, T *ptfix, cudaStream_t s);
template <typename T> void launch_pc_proj(const LoopArgs<T> &a, cudaStream_t s);
template <typename T>
void launch_halo_fused(const LoopArgs<T> &a, const int32_t *idx, int64_t nsend, T *sendbuf,
                       const T *recvbuf, int64_t nghost, int pack, cudaStream_t s);
template <typename T>
void launch_resid(const LoopArgs<T> &a, const T *b, const T *bt, const T *x, const T *xt,
                  T *r, T *rt, int with_coef, cudaStream_t s);
template <typename T>
void launch_init2(const LoopArgs<T> &a, const T *U, const T *Ut, cudaStream_t s);
template <typename T>
void launch_step7(const LoopArgs<T> &a, const T *U, const T *Ut, T *xo, T *xto, cudaStream_t s);
// Allow a kernel all the dynamic shared memory an SM offers beside its
// static shared memory (227 KB per block on sm_100a).
template <typename F> inline void allow_max_dyn_smem(F *f) {
  cudaFuncAttributes fa{};
  RB_CUDA(cudaFuncGetAttributes(&fa, (const void *)f));
  RB_CUDA(cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(227 * 1024 - fa.sharedSizeBytes)));
}
// row-partitioned form (kernels.cu)
template <typename T> void launch_leader1(const LoopArgs<T> &a, cudaStream_t s);
template <typename T> void launch_leader2(const LoopArgs<T> &a, cudaStream_t s);
template <typename T> void launch_leader_resid(const LoopArgs<T> &a, int coef, cudaStream_t s);
template <typename T> void launch_leader_init2(const LoopArgs<T> &a, cudaStream_t s);
template <typename T>
void launch_halo_pack_loop(const LoopArgs<T> &a, const int32_t *idx, int64_t nsend, T *buf, cudaStream_t s);
template <typename T>
void launch_halo_unpack_loop(const LoopArgs<T> &a, const T *buf, int64_t nghost, cudaStream_t s);
template <typename T>
void launch_pack_rows(const T *X, int k, const int32_t *idx, int64_t cnt, T *out, cudaStream_t s);
template <typename T>
void launch_spmv_pair(const DevMat &A, const DevMat &AH, const T *p, const T *pt, T *z, T *zt,
                      cudaStream_t s);

// ---- blocks.cu
template <typename T>
void launch_spmm(const DevMat &A, const T *X, T *Y, int k, cudaStream_t s);
template <typename T>
void gram(const std::vector<ColDesc> &X, const std::vector<ColDesc> &Y, int64_t n,
          std::vector<cplx> &G, rbicg_ctx *ctx, cudaStream_t s);   // G = X^H Y (row-major mX x mY)
template <typename T>
void gram_cc(const T *C, const T *Ct, int k, int64_t n, std::vector<cplx> &out, rbicg_ctx *ctx,
             cudaStream_t strm);
template <typename T>
void gemm_panels(const std::vector<ColDesc> &X, const std::vector<cplx> &M, int p, int64_t n,
                 T *out, rbicg_ctx *ctx, cudaStream_t s, bool sync = true,
                 T *out_last = nullptr);   // out (row-major n x p) = X M; with out_last, M has
                                           // p + 1 columns and the last one goes to out_last[n]

template <typename T>
void gemm_multi(const std::vector<ColDesc> &X, const std::vector<cplx> &M,
                const std::vector<std::pair<T *, int>> &outs, int64_t n, rbicg_ctx *ctx,
                cudaStream_t s);   // [out_0 | out_1 | ...] = X M (M row-major mX x Σ widths)

// ---- workspace helpers (api.cu)
void *ws_alloc(size_t bytes);
void ws_free(void *p);

// ---- control.cpp (host LAPACK shim)
int lapack_ggev(bool real, int m, std::vector<cplx> P, std::vector<cplx> Q,
                std::vector<cplx> &alpha, std::vector<cplx> &beta, std::vector<cplx> &VL,
                std::vector<cplx> &VR, std::vector<int> &pair_first);
int lapack_geev(bool real, int m, const std::vector<cplx> &P, std::vector<cplx> &alpha,
                std::vector<cplx> &beta, std::vector<cplx> &VL, std::vector<cplx> &VR);
int lapack_gesvd(bool real, int m, std::vector<cplx> G, std::vector<double> &S,
                 std::vector<cplx> &Mleft, std::vector<cplx> &Nright);

}  // namespace rbicg
