// matrix.cu -- device matrix store: CSR -> SELL-32 for A and for the explicit
// conjugate transpose A^* (BASELINE.json north star (1); the operator pair of
// Algorithm 2 lines z = A p, z~ = A^* p~).
//
// The transpose is a stable counting sort by column (CUB radix sort of the
// column keys, a library sort primitive), so each row of A^* lists its
// entries in ascending column order, like scipy's A.conj().T.tocsr().
#include <cub/cub.cuh>

#include "internal.h"
#include <cstdlib>

namespace rbicg {

__global__ void k_row_index(const int32_t *rowptr, int64_t n, int32_t *rowidx) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    for (int32_t e = rowptr[r]; e < rowptr[r + 1]; ++e) rowidx[e] = (int32_t)r;
}

__global__ void k_iota(int32_t *v, int64_t m) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

__global__ void k_count_cols(const int32_t *col, int64_t nnz, int32_t *counts) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(counts + col[e], 1);
}

template <typename T>
__global__ void k_gather_t(const int32_t *perm, const int32_t *rowidx, const T *val, int64_t nnz,
                           int32_t *colT, T *valT) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = perm[t];
    colT[t] = rowidx[e];
    valT[t] = conj(val[e]);
  }
}

__global__ void k_slice_width(const int32_t *rowptr, int64_t n, int64_t nslices, int64_t *w32) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nslices;
       s += (int64_t)gridDim.x * blockDim.x) {
    int32_t w = 0;
    for (int l = 0; l < 32; ++l) {
      const int64_t r = s * 32 + l;
      if (r < n) w = max(w, rowptr[r + 1] - rowptr[r]);
    }
    w32[s] = (int64_t)w * 32;
  }
}

template <typename T>
__global__ void k_sell_fill(const int32_t *rowptr, const int32_t *col, const T *val, int64_t n,
                            int64_t nslices, const int64_t *sptr, int32_t *scol, T *sval) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nslices * 32;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = g >> 5;
    const int lane = (int)(g & 31);
    const int64_t off = sptr[s];
    const int w = (int)((sptr[s + 1] - off) >> 5);
    const int64_t r = g;   // row = slice*32 + lane
    int32_t b = 0, len = 0;
    if (r < n) {
      b = rowptr[r];
      len = rowptr[r + 1] - b;
    }
    for (int jj = 0; jj < w; ++jj) {
      const int64_t idx = off + (int64_t)jj * 32 + lane;
      if (jj < len) {
        scol[idx] = col[b + jj];
        sval[idx] = val[b + jj];
      } else {
        scol[idx] = r < n ? (int32_t)r : 0;   // padding: a valid address, zero value
        sval[idx] = zero<T>();
      }
    }
  }
}

template <typename I>
__global__ void k_differ(const I *a, const I *b, int64_t m, int *flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    if (a[i] != b[i]) *flag = 1;
}

// max |col - row| over the stored entries (the SpMV's reach in rows)
__global__ void k_bandwidth(const int32_t *rowptr, const int32_t *col, int64_t n, int *bw) {
  int m = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    for (int32_t e = rowptr[r]; e < rowptr[r + 1]; ++e) m = max(m, abs(col[e] - (int)r));
  atomicMax(bw, m);
}

// SELL column deltas col - row (row = slice * 32 + lane), int16
__global__ void k_make_dcols(const int32_t *cols, const int64_t *sptr, int64_t nslices, int16_t *dc) {
  for (int64_t sl = blockIdx.x; sl < nslices; sl += gridDim.x) {
    const int64_t o = sptr[sl], e = sptr[sl + 1];
    for (int64_t q = o + threadIdx.x; q < e; q += blockDim.x) {
      const int64_t row = sl * 32 + ((q - o) & 31);
      dc[q] = (int16_t)(cols[q] - row);
    }
  }
}

static int grid1d(int64_t m) { return (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 148 * 32)); }

template <typename T>
static void csr_to_sell(rbicg_ctx *ctx, int64_t n, const int32_t *rowptr, const int32_t *col,
                        const T *val, DevMat &out) {
  cudaStream_t st = ctx->stream;
  out.n = n;
  out.nslices = (n + 31) / 32;
  int64_t *w32 = (int64_t *)ws_alloc(sizeof(int64_t) * (out.nslices + 1));
  out.sptr = (int64_t *)ws_alloc(sizeof(int64_t) * (out.nslices + 1));
  k_slice_width<<<grid1d(out.nslices), 256, 0, st>>>(rowptr, n, out.nslices, w32);
  RB_CUDA(cudaMemsetAsync(w32 + out.nslices, 0, sizeof(int64_t), st));
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, w32, out.sptr, out.nslices + 1, st);
  void *dtmp = ws_alloc(tmp + 16);
  cub::DeviceScan::ExclusiveSum(dtmp, tmp, w32, out.sptr, out.nslices + 1, st);
  std::vector<int64_t> hs(out.nslices + 1);
  RB_CUDA(cudaMemcpyAsync(hs.data(), out.sptr, sizeof(int64_t) * (out.nslices + 1),
                          cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  out.padded = hs[out.nslices];
  int64_t tm = 0;
  for (int64_t s0 = 0; s0 < out.nslices; s0 += BS / 32)
    tm = std::max(tm, hs[std::min(s0 + BS / 32, out.nslices)] - hs[s0]);
  out.tile_max = (int)std::min<int64_t>(tm, INT32_MAX);
  int64_t tmh = 0;
  for (int64_t s0 = 0; s0 < out.nslices; s0 += BS / 64)
    tmh = std::max(tmh, hs[std::min(s0 + BS / 64, out.nslices)] - hs[s0]);
  out.tile_max_h = (int)std::min<int64_t>(tmh, INT32_MAX);
  int64_t mw = 0;
  for (int64_t s0 = 0; s0 < out.nslices; ++s0) mw = std::max(mw, (hs[s0 + 1] - hs[s0]) / 32);
  out.max_w = (int)std::min<int64_t>(mw, INT32_MAX);
  ws_free(dtmp);
  ws_free(w32);
  out.cols = (int32_t *)ws_alloc(sizeof(int32_t) * std::max<int64_t>(out.padded, 1));
  out.vals = ws_alloc(sizeof(T) * std::max<int64_t>(out.padded, 1));
  k_sell_fill<T><<<grid1d(out.nslices * 32), 256, 0, st>>>(rowptr, col, val, n, out.nslices, out.sptr,
                                                           out.cols, (T *)out.vals);
  count_launch(2);
}

// A structurally symmetric A (every stencil discretisation) has the same
// sorted column list in row i of A and of A^*: the SELL column arrays are then
// identical and A^* keeps only its values -- pass 1 streams 4 bytes less per
// nonzero of A^* (DESIGN §6).  Decided by comparing the built arrays.
static void make_dcols(rbicg_ctx *ctx, rbicg_mat *M) {
  DevMat &A = M->A;
  if (getenv("RBICG_NO_DCOLS") || !M->AH.cols_shared || A.bandwidth < 0 || A.bandwidth > 32767) return;
  A.dcols = (int16_t *)ws_alloc(sizeof(int16_t) * std::max<int64_t>(A.padded, 1));
  k_make_dcols<<<(int)std::min<int64_t>(std::max<int64_t>(A.nslices, 1), 4096), 256, 0, ctx->stream>>>(
      A.cols, A.sptr, A.nslices, A.dcols);
  count_launch();
}

static void share_cols(rbicg_ctx *ctx, rbicg_mat *M) {
  if (getenv("RBICG_NO_SHARED_COLS")) return;
  DevMat &A = M->A, &H = M->AH;
  if (A.n != H.n || A.nslices != H.nslices || A.padded != H.padded) return;
  cudaStream_t st = ctx->stream;
  int *flag = (int *)ws_alloc(sizeof(int));
  RB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  k_differ<int64_t><<<grid1d(A.nslices + 1), 256, 0, st>>>(A.sptr, H.sptr, A.nslices + 1, flag);
  k_differ<int32_t><<<grid1d(A.padded), 256, 0, st>>>(A.cols, H.cols, A.padded, flag);
  count_launch(2);
  int h = 1;
  RB_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  ws_free(flag);
  if (h) return;
  ws_free(H.cols);
  H.cols = A.cols;
  H.cols_shared = 1;
}

// Structurally symmetric A with sorted rows: A^*'s pattern is A's, and the
// value of A^*[j][i] = conj(A[i][j]) sits at the position of column i in row j
// (binary search) -- no sort.  flag = 1 if a row is unsorted or has a
// duplicate, or an (i, j) has no (j, i): the caller then takes the sort path.
template <typename T>
__global__ void k_sym_transpose(const int32_t *rowptr, const int32_t *col, const T *val, int64_t n,
                                T *valT, int *flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = rowptr[i], e = rowptr[i + 1];
    for (int32_t q = b; q < e; ++q) {
      const int32_t j = col[q];
      if (q > b && col[q - 1] >= j) {
        *flag = 1;
        return;
      }
      int32_t lo = rowptr[j], hi = rowptr[j + 1] - 1;
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (col[mid] < (int32_t)i) lo = mid + 1;
        else hi = mid;
      }
      if (lo > hi || col[lo] != (int32_t)i) {
        *flag = 1;
        return;
      }
      valT[lo] = conj(val[q]);
    }
  }
}

template <typename T>
static void build_t(rbicg_ctx *ctx, int64_t n, int64_t nnz, const int32_t *rowptr,
                    const int32_t *col, const T *val, rbicg_mat *M) {
  cudaStream_t st = ctx->stream;
  csr_to_sell<T>(ctx, n, rowptr, col, val, M->A);
  {
    int *bw = (int *)ws_alloc(sizeof(int));
    RB_CUDA(cudaMemsetAsync(bw, 0, sizeof(int), st));
    k_bandwidth<<<grid1d(n), 256, 0, st>>>(rowptr, col, n, bw);
    count_launch();
    int h = 0;
    RB_CUDA(cudaMemcpyAsync(&h, bw, sizeof(int), cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    ws_free(bw);
    M->A.bandwidth = h;
  }
  if (!getenv("RBICG_NO_SYM_T") && nnz > 0) {   // structurally symmetric fast path
    T *valT = (T *)ws_alloc(sizeof(T) * nnz);
    int *flag = (int *)ws_alloc(sizeof(int));
    RB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    k_sym_transpose<T><<<grid1d(n), 256, 0, st>>>(rowptr, col, val, n, valT, flag);
    count_launch();
    int h = 1;
    RB_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    ws_free(flag);
    if (!h) {
      csr_to_sell<T>(ctx, n, rowptr, col, valT, M->AH);
      share_cols(ctx, M);
      if (sizeof(T) == 8) make_dcols(ctx, M);
      RB_CUDA(cudaStreamSynchronize(st));
      ws_free(valT);
      return;
    }
    ws_free(valT);
  }
  // ---- conjugate transpose
  int32_t *rowidx = (int32_t *)ws_alloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  int32_t *iota = (int32_t *)ws_alloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  int32_t *keys_out = (int32_t *)ws_alloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  int32_t *perm = (int32_t *)ws_alloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  int32_t *cnt = (int32_t *)ws_alloc(sizeof(int32_t) * (n + 1));
  int32_t *rowptrT = (int32_t *)ws_alloc(sizeof(int32_t) * (n + 1));
  int32_t *colT = (int32_t *)ws_alloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  T *valT = (T *)ws_alloc(sizeof(T) * std::max<int64_t>(nnz, 1));
  k_row_index<<<grid1d(n), 256, 0, st>>>(rowptr, n, rowidx);
  k_iota<<<grid1d(nnz), 256, 0, st>>>(iota, nnz);
  RB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), st));
  k_count_cols<<<grid1d(nnz), 256, 0, st>>>(col, nnz, cnt);
  count_launch(3);
  int bits = 1;
  while (bits < 31 && ((int64_t)1 << bits) < n) ++bits;
  size_t t1 = 0, t2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, col, keys_out, iota, perm, (int)nnz, 0, bits, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, cnt, rowptrT, (int)(n + 1), st);
  void *tmp = ws_alloc(std::max(t1, t2) + 16);
  cub::DeviceRadixSort::SortPairs(tmp, t1, col, keys_out, iota, perm, (int)nnz, 0, bits, st);
  cub::DeviceScan::ExclusiveSum(tmp, t2, cnt, rowptrT, (int)(n + 1), st);
  k_gather_t<T><<<grid1d(nnz), 256, 0, st>>>(perm, rowidx, val, nnz, colT, valT);
  count_launch(3);
  csr_to_sell<T>(ctx, n, rowptrT, colT, valT, M->AH);
  share_cols(ctx, M);
  if (sizeof(T) == 8) make_dcols(ctx, M);   // int16 deltas: real data only (la.dcols)
  RB_CUDA(cudaStreamSynchronize(st));
  for (void *p : {(void *)rowidx, (void *)iota, (void *)keys_out, (void *)perm, (void *)cnt,
                  (void *)rowptrT, (void *)colT, (void *)valT, tmp})
    ws_free(p);
}

void build_matrix(rbicg_ctx *ctx, int64_t n, int64_t nnz, const int32_t *rowptr_d,
                  const int32_t *col_d, const void *val_d, rbicg_dtype dt, rbicg_mat *M) {
  M->n = n;
  M->nnz = nnz;
  M->dtype = dt;
  if (dt == RBICG_F64)
    build_t<double>(ctx, n, nnz, rowptr_d, col_d, (const double *)val_d, M);
  else
    build_t<zc>(ctx, n, nnz, rowptr_d, col_d, (const zc *)val_d, M);
}

// rows that reference a ghost column (>= nloc) in A or A^*: flag their
// 256-row and 128-row tiles
__global__ void k_ghost_tiles(const int32_t *rpA, const int32_t *ciA, const int32_t *rpH,
                              const int32_t *ciH, int64_t nloc, int *f256, int *f128) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nloc;
       r += (int64_t)gridDim.x * blockDim.x) {
    bool g = false;
    for (int32_t e = rpA[r]; e < rpA[r + 1] && !g; ++e) g = ciA[e] >= nloc;
    for (int32_t e = rpH[r]; e < rpH[r + 1] && !g; ++e) g = ciH[e] >= nloc;
    if (g) {
      f256[r / BS] = 1;
      f128[r / TRH] = 1;
    }
  }
}

static int32_t *tile_order(const std::vector<int> &flag, int64_t &nint) {
  std::vector<int32_t> ord;
  ord.reserve(flag.size());
  for (size_t t = 0; t < flag.size(); ++t)
    if (!flag[t]) ord.push_back((int32_t)t);
  nint = (int64_t)ord.size();
  for (size_t t = 0; t < flag.size(); ++t)
    if (flag[t]) ord.push_back((int32_t)t);
  int32_t *d = (int32_t *)ws_alloc(sizeof(int32_t) * std::max<size_t>(ord.size(), 1));
  RB_CUDA(cudaMemcpy(d, ord.data(), sizeof(int32_t) * ord.size(), cudaMemcpyHostToDevice));
  return d;
}

void build_matrix_local(rbicg_ctx *ctx, int64_t nloc, const int32_t *rpA, const int32_t *ciA,
                        const void *vA, const int32_t *rpH, const int32_t *ciH, const void *vH,
                        rbicg_dtype dt, rbicg_mat *M) {
  M->n = nloc;
  M->dtype = dt;
  {   // halo-overlap tile orders (interior tiles first)
    const int64_t t256 = (nloc + BS - 1) / BS, t128 = (nloc + TRH - 1) / TRH;
    int *f = (int *)ws_alloc(sizeof(int) * (t256 + t128));
    RB_CUDA(cudaMemsetAsync(f, 0, sizeof(int) * (t256 + t128), ctx->stream));
    k_ghost_tiles<<<grid1d(nloc), 256, 0, ctx->stream>>>(rpA, ciA, rpH, ciH, nloc, f, f + t256);
    count_launch();
    std::vector<int> h(t256 + t128);
    RB_CUDA(cudaMemcpyAsync(h.data(), f, sizeof(int) * h.size(), cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
    ws_free(f);
    // RBICG_FORCE_HALO_SPLIT=1 (tests): the last eighth of the tiles counts as
    // boundary even without ghosts, so a one-rank NCCL context runs the overlap
    // (fork/join + two launches) inside its captured graph
    if (getenv("RBICG_FORCE_HALO_SPLIT")) {
      for (int64_t t = t256 - std::max<int64_t>(1, t256 / 8); t < t256; ++t) h[t] = 1;
      for (int64_t t = t128 - std::max<int64_t>(1, t128 / 8); t < t128; ++t) h[t256 + t] = 1;
    }
    M->ord = tile_order(std::vector<int>(h.begin(), h.begin() + t256), M->nint);
    M->ord_h = tile_order(std::vector<int>(h.begin() + t256, h.end()), M->nint_h);
    M->ntl = t256;
    M->ntl_h = t128;
  }
  if (dt == RBICG_F64) {
    csr_to_sell<double>(ctx, nloc, rpA, ciA, (const double *)vA, M->A);
    csr_to_sell<double>(ctx, nloc, rpH, ciH, (const double *)vH, M->AH);
  } else {
    csr_to_sell<zc>(ctx, nloc, rpA, ciA, (const zc *)vA, M->A);
    csr_to_sell<zc>(ctx, nloc, rpH, ciH, (const zc *)vH, M->AH);
  }
  share_cols(ctx, M);
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
}

// sigma I - A in place on a device CSR value array (IRKA's shifted systems,
// P:1100-1101): one thread per row negates its entries and adds sigma to the
// diagonal; a row without exactly one diagonal entry sets *bad.
template <typename T>
__global__ void k_shift_rows(const int32_t *rowptr, const int32_t *col, T *val, int64_t n, T sigma,
                             int *bad) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int diag = 0;
    for (int32_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
      T v = neg(val[e]);
      if (col[e] == r) {
        v = add(v, sigma);
        ++diag;
      }
      val[e] = v;
    }
    if (diag != 1) atomicOr(bad, 1);
  }
}

void shift_csr_values(rbicg_ctx *ctx, int64_t n, const int32_t *rowptr_d, const int32_t *col_d,
                      void *val_d, rbicg_dtype dt, double sre, double sim) {
  int *bad = (int *)ws_alloc(sizeof(int));
  RB_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
  if (dt == RBICG_F64)
    k_shift_rows<double><<<grid1d(n), 256, 0, ctx->stream>>>(rowptr_d, col_d, (double *)val_d, n, sre, bad);
  else
    k_shift_rows<zc><<<grid1d(n), 256, 0, ctx->stream>>>(rowptr_d, col_d, (zc *)val_d, n, mk(sre, sim), bad);
  count_launch();
  int h = 0;
  RB_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  ws_free(bad);
  RB_CHECK(h == 0, RBICG_EINVAL);
}

void free_devmat(DevMat &m) {
  // pooled device memory (reused by the next system's store); no device sync
  ws_free(m.sptr);
  if (!m.cols_shared) ws_free(m.cols);
  if (m.dcols) ws_free(m.dcols);
  ws_free(m.vals);
  m = DevMat();
}

}  // namespace rbicg
