// internal.h -- library-internal types shared by the RBiCG translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <complex>
#include <vector>
#include <string>

#include "common.cuh"

namespace rbicg {

constexpr int KMAX = 32;   // maximum recycle width supported by the kernels
constexpr int BS = 256;    // threads per block of the streaming kernels

// SELL-32 matrix (slices of 32 consecutive rows, column-major inside a slice,
// zero-padded to the slice's longest row; sigma = 1, i.e. no row sorting, so
// vectors keep their natural order).
struct DevMat {
  int64_t n = 0, nslices = 0, padded = 0;
  int tile_max = 0;         // max elements in one 256-row tile (8 slices)
  int max_w = 0;            // widest slice (padded row length)
  int64_t *sptr = nullptr;  // nslices + 1 element offsets (multiples of 32)
  int32_t *cols = nullptr;
  void *vals = nullptr;
};

// Device-resident iteration state (one per solve; scalars of Algorithm 2).
template <typename T>
struct DevState {
  int iter;      // completed iterations i
  int done;      // 0 running, 1 finished, 2 paused at a cycle boundary
  int status;    // RBICG_* of the finished iteration
  int max_itn;
  int force;     // stop test disabled (Q27 protocol)
  int stop_at;   // pause after this iteration (cycle boundary)
  int k;
  int seg_start;   // lazy x: first iteration index of the open segment
  unsigned cnt[4];
  T rho, beta, alpha, sigma;   // ρ_{i}, β_{i}, α_i, σ_i
  double rnorm, rtnorm;        // ||r_i||, ||r~_i||
  double tolb, tolbt;          // tol ||b||, tol ||b~||
  double bn2, btn2, rn2, rtn2; // squared norms from the residual kernel
  T zeta[KMAX], zetat[KMAX];   // ζ_i, ζ~_i
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
  int staged, tile_max;    // pass 1 stages SELL tiles in smem via TMA
  int pass2_tma;           // pass 2 streams its tiles through smem via TMA
  int lazy_x;              // x, x~ rebuilt per segment from the Lanczos ring
  T *pseg, *ptseg;         // p_a, p~_a at the start of the open segment
  int nsm;
  DevMat A, AH;
  T *rring, *rtring;       // ring of residual columns (r_m in column m % ring)
  T *p[2], *pt[2];         // ping-pong search directions
  T *z, *zt;
  T *x, *xt;
  const T *C, *Ct;         // row-major n x k
  DevState<T> *st;
  IterRec<T> *hist;        // [max_itn + 1]
  T *zhist, *zthist;       // [max_itn + 1][k]
  T *part;                 // block partials [outputs][G]
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
  int prio_lo = 0;
  int nsm = 148;
  int grid_stream = 296;  // persistent grid of the streaming kernels
  // reusable device workspace
  void *work = nullptr;
  size_t work_bytes = 0;
  void *host_pinned = nullptr;
  size_t host_bytes = 0;
  // pass timings from rbicg_dbg_time_kernels
};

struct rbicg_mat {
  rbicg_ctx *ctx = nullptr;
  int64_t n = 0, nnz = 0;
  rbicg_dtype dtype = RBICG_F64;
  rbicg::DevMat A, AH;
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

// ---- kernels.cu (launch wrappers; all on ctx->stream)
void prepare_kernels();        // one-time function attributes (not capturable)
void prepare_block_kernels();
int stream_blocks_per_sm();    // occupancy of the streaming kernels
template <typename T> void launch_pass1(const LoopArgs<T> &a, cudaStream_t s);
template <typename T> void launch_pass2(const LoopArgs<T> &a, cudaStream_t s);
template <typename T>
void launch_resid(const LoopArgs<T> &a, const T *b, const T *bt, const T *x, const T *xt,
                  T *r, T *rt, int with_coef, cudaStream_t s);
template <typename T>
void launch_init2(const LoopArgs<T> &a, const T *U, const T *Ut, cudaStream_t s);
template <typename T>
void launch_step7(const LoopArgs<T> &a, const T *U, const T *Ut, T *xo, T *xto, cudaStream_t s);
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
void gram_pairs(const std::vector<const T *> &panels, const std::vector<int> &ncols,
                const std::vector<std::pair<int, int>> &pairs, int64_t n, std::vector<cplx> &out,
                rbicg_ctx *ctx, cudaStream_t s);   // out[i] = x_{a_i}^H x_{b_i}, compact panels
template <typename T>
void gemm_panels(const std::vector<ColDesc> &X, const std::vector<cplx> &M, int p, int64_t n,
                 T *out, rbicg_ctx *ctx, cudaStream_t s, bool sync = true);   // out (row-major n x p) = X M

// ---- workspace helpers (api.cu)
void *ws_alloc(size_t bytes);
void ws_free(void *p);

// ---- control.cpp (host LAPACK shim)
int lapack_ggev(bool real, int m, std::vector<cplx> P, std::vector<cplx> Q,
                std::vector<cplx> &alpha, std::vector<cplx> &beta, std::vector<cplx> &VL,
                std::vector<cplx> &VR, std::vector<int> &pair_first);
int lapack_gesvd(bool real, int m, std::vector<cplx> G, std::vector<double> &S,
                 std::vector<cplx> &Mleft, std::vector<cplx> &Nright);

}  // namespace rbicg
