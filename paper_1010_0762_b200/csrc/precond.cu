// precond.cu -- split preconditioning for RBiCG.
//
// The paper's experiments split-precondition every system with a Crout ILUT
// (drop tolerance 0.05 for convection-diffusion) and the
// recycle spaces belong to the preconditioned operator.
// With M = L U ≈ A the solver runs Algorithm 2 on
//     Â = L^{-1} A U^{-1},   Â^* = U^{-*} A^* L^{-*},
// primal right-hand side L^{-1} b, dual U^{-*} b~, and maps back
// x = U^{-1} x̂, x~ = L^{-*} x̂~ (readings Q33/Q34).
//
//   * factorisation: Crout ILU with threshold (ILUC), host C++ -- per-system
//     setup like the pencil's LAPACK, not the hot loop -- with the drop rule the
//     paper's Matlab documents: off-diagonal U(k, j) kept if |u| >= t ||A(:, j)||,
//     L(i, k) kept if |l| >= t ||A(:, k)|| before the scaling by the pivot;
//   * device: L (unit lower), U (upper), L^* (unit upper), U^* (lower) as CSR;
//     triangular solves are sync-free: one warp per row, rows claimed in
//     dependency order from an atomic counter (a row only ever waits for rows
//     claimed before it, by warps already running -- no deadlock), each
//     dependency awaited on a per-row ready flag (acquire/release);
//   * Â p = L^{-1}(A(U^{-1} p)) and Â^* p~ = U^{-*}(A^*(L^{-*} p~)) in one
//     "apply pair" (two solves, the SpMV pair, two solves).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "hot.cuh"

namespace rbicg {

// ------------------------------------------------------------------ host ILUC
namespace {

template <typename C> double mag(const C &v) { return std::abs(v); }
inline double cj(double v) { return v; }
inline std::complex<double> cj(const std::complex<double> &v) { return std::conj(v); }

template <typename C>
void iluc_host(int64_t n, const int32_t *rp, const int32_t *ci, const C *va, double t,
               std::vector<std::vector<std::pair<int32_t, C>>> &Lrows,
               std::vector<std::vector<std::pair<int32_t, C>>> &Urows) {
  // column norms of A and A by column (for w = A(k+1:, k))
  std::vector<double> cn(n, 0.0);
  std::vector<std::vector<std::pair<int32_t, C>>> Acols(n);
  for (int64_t i = 0; i < n; ++i)
    for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
      cn[ci[e]] += std::norm(va[e]);
      Acols[ci[e]].emplace_back((int32_t)i, va[e]);
    }
  for (auto &v : cn) v = std::sqrt(v);
  Lrows.assign(n, {});
  Urows.assign(n, {});
  std::vector<std::vector<std::pair<int32_t, C>>> Lcols(n), Ucols(n);
  std::vector<C> z(n, C(0)), w(n, C(0));
  std::vector<char> zin(n, 0), win(n, 0);
  std::vector<int32_t> zl, wl;
  for (int64_t k = 0; k < n; ++k) {
    zl.clear();
    wl.clear();
    auto zadd = [&](int32_t j, C v) {
      if (!zin[j]) {
        zin[j] = 1;
        zl.push_back(j);
      }
      z[j] += v;
    };
    auto wadd = [&](int32_t i, C v) {
      if (!win[i]) {
        win[i] = 1;
        wl.push_back(i);
      }
      w[i] += v;
    };
    for (int32_t e = rp[k]; e < rp[k + 1]; ++e)   // z = A(k, k:)
      if (ci[e] >= k) zadd(ci[e], va[e]);
    for (auto &li : Lrows[k])                       // z -= L(k, i) U(i, k:)
      for (auto &uj : Urows[li.first])
        if (uj.first >= k) zadd(uj.first, -li.second * uj.second);
    for (auto &ai : Acols[k])                       // w = A(k+1:, k)
      if (ai.first > k) wadd(ai.first, ai.second);
    for (auto &ui : Ucols[k])                       // w -= U(i, k) L(k+1:, i), i < k
      if (ui.first < k)
        for (auto &lr : Lcols[ui.first])
          if (lr.first > k) wadd(lr.first, -ui.second * lr.second);
    const C piv = zin[k] ? z[k] : C(0);
    RB_CHECK(mag(piv) != 0.0 && std::isfinite(mag(piv)), RBICG_EINVAL);   // zero pivot
    std::sort(zl.begin(), zl.end());
    std::sort(wl.begin(), wl.end());
    for (int32_t j : zl) {
      if (j == k || mag(z[j]) >= t * cn[j]) {
        Urows[k].emplace_back(j, z[j]);
        Ucols[j].emplace_back((int32_t)k, z[j]);
      }
      z[j] = C(0);
      zin[j] = 0;
    }
    for (int32_t i : wl) {
      if (mag(w[i]) >= t * cn[k]) {
        const C l = w[i] / piv;
        Lrows[i].emplace_back((int32_t)k, l);
        Lcols[k].emplace_back(i, l);
      }
      w[i] = C(0);
      win[i] = 0;
    }
  }
}

}  // namespace

}  // namespace rbicg

namespace rbicg {

// ------------------------------------------------------------------ device
__device__ __forceinline__ double shfl_idx(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ zc shfl_idx(zc v, int src) {
  return mk(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// x = T^{-1} b for one triangular factor; flags[n] zero and *counter zero on
// entry; `done` (nullable): the solver's state -- a finished/paused loop
// skips the solve (its graph still holds the launch).  One thread per row;
// a warp claims 32 consecutive rows of the level order (rows sorted by
// dependency level, computed at factorisation), so the rows a warp holds are
// mostly independent and every dependency of a claimed row was claimed
// earlier by a running thread (deadlock-free); dependencies are awaited on
// per-row ready flags (acquire/release) with a short back-off.
template <typename T>
__global__ void __launch_bounds__(256) k_trsv(const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                              const T *__restrict__ v, const int32_t *__restrict__ order,
                                              int64_t n, int unit, const T *__restrict__ b, T *x, int *flags,
                                              unsigned long long *counter, const int *done) {
  if (done && __ldcg(done)) return;
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(counter, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= (unsigned long long)n) return;
    const int64_t idx = (int64_t)base + lane;
    if (idx < n) {
      const int64_t row = order[idx];
      T acc = zero<T>(), diag = mk_re<T>(1.0);
      for (int32_t e = rp[row]; e < rp[row + 1]; ++e) {
        const int32_t c = ci[e];
        const T a = v[e];
        if (c == row) {
          diag = a;
        } else {
          while (ld_acquire(&flags[c]) == 0) {
          }
          acc = mad(a, ldcg(x + c), acc);
        }
      }
      T val = sub(b[row], acc);
      if (!unit) val = divd(val, diag);
      x[row] = val;
      st_release(&flags[row], 1);
    }
  }
}

// y = T x (CSR, stored entries, unit diagonal added when `unit`)
template <typename T>
__global__ void k_csr_mv(const int32_t *rp, const int32_t *ci, const T *v, int64_t n, int unit, const T *x,
                         T *y) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    T acc = unit ? x[r] : zero<T>();
    for (int32_t e = rp[r]; e < rp[r + 1]; ++e) acc = mad(v[e], x[ci[e]], acc);
    y[r] = acc;
  }
}

// strided column <-> contiguous vector (row-major n x k blocks)
template <typename T>
__global__ void k_col_get(const T *X, int k, int c, int64_t n, T *v) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    v[r] = X[r * k + c];
}
template <typename T>
__global__ void k_col_put(const T *v, int k, int c, int64_t n, T *X) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    X[r * k + c] = v[r];
}

static int gsz(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 2368)); }

// ------------------------------------------------------------------ host API
template <typename T>
void pc_trsv(const rbicg_prec *P, const TriCSR &F, const T *b, T *x, PcWork &w, cudaStream_t s,
             const int *done) {
  RB_CUDA(cudaMemsetAsync(w.flags, 0, sizeof(int) * P->n, s));
  RB_CUDA(cudaMemsetAsync(w.counter, 0, sizeof(unsigned long long), s));
  // threads in flight: a few levels' worth of rows (more only spin on flags)
  static const int blocks_env = getenv("RBICG_TRSV_BLOCKS") ? atoi(getenv("RBICG_TRSV_BLOCKS")) : 0;
  const int blocks = blocks_env > 0 ? blocks_env : P->ctx->nsm;
  k_trsv<T><<<blocks, 256, 0, s>>>(F.rp, F.ci, (const T *)F.v, F.order, P->n, F.unit, b, x, w.flags,
                                   w.counter, done);
  count_launch();
}

template <typename T>
void pc_apply_pair(const rbicg_prec *P, const rbicg_mat *M, const T *p, const T *pt, T *z, T *zt, PcWork &w,
                   cudaStream_t s, const int *done) {
  T *y = (T *)w.y, *yt = (T *)w.yt, *q = (T *)w.q, *qt = (T *)w.qt;
  if (p) pc_trsv<T>(P, P->U, p, y, w, s, done);       // y = U^{-1} p
  if (pt) pc_trsv<T>(P, P->LH, pt, yt, w, s, done);   // y~ = L^{-*} p~
  launch_spmv_pair<T>(M->A, M->AH, p ? y : yt, pt ? yt : y, q, qt, s);
  if (p) pc_trsv<T>(P, P->L, q, z, w, s, done);       // z = L^{-1} A y
  if (pt) pc_trsv<T>(P, P->UH, qt, zt, w, s, done);   // z~ = U^{-*} A^* y~
}

template <typename T>
void pc_apply_block(const rbicg_prec *P, const rbicg_mat *M, bool adj, const T *X, T *Y, int k, PcWork &w,
                    cudaStream_t s) {
  const int64_t n = P->n;
  for (int c = 0; c < k; ++c) {
    k_col_get<T><<<gsz(n), 256, 0, s>>>(X, k, c, n, (T *)w.v);
    count_launch();
    if (!adj) pc_apply_pair<T>(P, M, (const T *)w.v, nullptr, (T *)w.u, nullptr, w, s, nullptr);
    else pc_apply_pair<T>(P, M, nullptr, (const T *)w.v, nullptr, (T *)w.u, w, s, nullptr);
    k_col_put<T><<<gsz(n), 256, 0, s>>>((const T *)w.u, k, c, n, Y);
    count_launch();
  }
}

template <typename T> void pc_solve_factor(const rbicg_prec *P, int which, const T *b, T *x, PcWork &w,
                                           cudaStream_t s) {
  const TriCSR &F = which == 0 ? P->L : which == 1 ? P->U : which == 2 ? P->LH : P->UH;
  pc_trsv<T>(P, F, b, x, w, s, nullptr);
}

template <typename T> void pc_mul_factor(const rbicg_prec *P, int which, const T *x, T *y, cudaStream_t s) {
  const TriCSR &F = which == 0 ? P->L : which == 1 ? P->U : which == 2 ? P->LH : P->UH;
  k_csr_mv<T><<<gsz(P->n), 256, 0, s>>>(F.rp, F.ci, (const T *)F.v, P->n, F.unit, x, y);
  count_launch();
}

void pc_work_alloc(const rbicg_prec *P, PcWork &w) {
  const size_t vb = (P->dtype == RBICG_F64 ? 8 : 16) * (size_t)std::max<int64_t>(P->n, 1);
  w.flags = (int *)ws_alloc(sizeof(int) * std::max<int64_t>(P->n, 1));
  w.counter = (unsigned long long *)ws_alloc(sizeof(unsigned long long));
  for (void **q : {&w.y, &w.yt, &w.q, &w.qt, &w.v, &w.u}) *q = ws_alloc(vb);
}
void pc_work_free(PcWork &w) {
  ws_free(w.flags);
  ws_free(w.counter);
  for (void *q : {w.y, w.yt, w.q, w.qt, w.v, w.u}) ws_free(q);
  w = PcWork();
}

#define RB_PC_INST(T)                                                                                         \
  template void pc_apply_pair<T>(const rbicg_prec *, const rbicg_mat *, const T *, const T *, T *, T *,       \
                                 PcWork &, cudaStream_t, const int *);                                       \
  template void pc_apply_block<T>(const rbicg_prec *, const rbicg_mat *, bool, const T *, T *, int, PcWork &, \
                                  cudaStream_t);                                                              \
  template void pc_solve_factor<T>(const rbicg_prec *, int, const T *, T *, PcWork &, cudaStream_t);          \
  template void pc_mul_factor<T>(const rbicg_prec *, int, const T *, T *, cudaStream_t);
RB_PC_INST(double)
RB_PC_INST(zc)

// upload one factor (host rows -> device CSR); conj_t: the conjugate transpose
template <typename C>
static TriCSR upload_factor(rbicg_ctx *ctx, int64_t n, const std::vector<std::vector<std::pair<int32_t, C>>> &rows,
                            bool conj_t, bool store_unit_diag, int unit, int upper) {
  std::vector<std::vector<std::pair<int32_t, C>>> tr;
  const auto *src = &rows;
  if (conj_t) {
    tr.assign(n, {});
    for (int64_t i = 0; i < n; ++i)
      for (auto &e : rows[i]) tr[e.first].emplace_back((int32_t)i, cj(e.second));
    src = &tr;
  }
  std::vector<int32_t> rp(n + 1, 0), ci;
  std::vector<C> v;
  for (int64_t i = 0; i < n; ++i) {
    for (auto &e : (*src)[i]) {
      if (e.first == i && !store_unit_diag && unit) continue;
      ci.push_back(e.first);
      v.push_back(e.second);
    }
    rp[i + 1] = (int32_t)ci.size();
  }
  // dependency levels (forward for lower, backward for upper factors) and
  // the rows sorted by (level, row): the solve's claim order
  std::vector<int32_t> lev(n, 0), order(n);
  for (int64_t q = 0; q < n; ++q) {
    const int64_t i = upper ? n - 1 - q : q;
    int32_t l = 0;
    for (int32_t e = rp[i]; e < rp[i + 1]; ++e)
      if (ci[e] != i) l = std::max(l, lev[ci[e]] + 1);
    lev[i] = l;
  }
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b2) { return lev[a] < lev[b2]; });
  TriCSR F;
  F.n = n;
  F.nnz = (int64_t)ci.size();
  F.unit = unit;
  F.upper = upper;
  F.levels = n ? *std::max_element(lev.begin(), lev.end()) + 1 : 0;
  F.order = (int32_t *)ws_alloc(4 * std::max<int64_t>(n, 1));
  RB_CUDA(cudaMemcpyAsync(F.order, order.data(), 4 * n, cudaMemcpyHostToDevice, ctx->stream));
  F.rp = (int32_t *)ws_alloc(4 * (n + 1));
  F.ci = (int32_t *)ws_alloc(4 * std::max<size_t>(ci.size(), 1));
  F.v = ws_alloc(sizeof(C) * std::max<size_t>(v.size(), 1));
  RB_CUDA(cudaMemcpyAsync(F.rp, rp.data(), 4 * (n + 1), cudaMemcpyHostToDevice, ctx->stream));
  if (!ci.empty()) {
    RB_CUDA(cudaMemcpyAsync(F.ci, ci.data(), 4 * ci.size(), cudaMemcpyHostToDevice, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(F.v, v.data(), sizeof(C) * v.size(), cudaMemcpyHostToDevice, ctx->stream));
  }
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  return F;
}

template <typename C>
static void build_prec(rbicg_prec *P, const int32_t *rp, const int32_t *ci, const C *va) {
  std::vector<std::vector<std::pair<int32_t, C>>> Lr, Ur;
  iluc_host<C>(P->n, rp, ci, va, P->droptol, Lr, Ur);
  // L stored with its unit diagonal omitted; rows of L hold (col < row) entries
  P->L = upload_factor<C>(P->ctx, P->n, Lr, false, false, 1, 0);
  P->U = upload_factor<C>(P->ctx, P->n, Ur, false, true, 0, 1);
  P->LH = upload_factor<C>(P->ctx, P->n, Lr, true, false, 1, 1);
  P->UH = upload_factor<C>(P->ctx, P->n, Ur, true, true, 0, 0);
  P->nnzL = P->L.nnz + P->n;
  P->nnzU = P->U.nnz;
}

void pc_build(rbicg_prec *P, const int32_t *rp, const int32_t *ci, const void *va) {
  if (P->dtype == RBICG_F64) build_prec<double>(P, rp, ci, (const double *)va);
  else build_prec<std::complex<double>>(P, rp, ci, (const std::complex<double> *)va);
}

static void free_factor(TriCSR &F) {
  ws_free(F.order);
  ws_free(F.rp);
  ws_free(F.ci);
  ws_free(F.v);
  F = TriCSR();
}
void pc_free(rbicg_prec *P) {
  free_factor(P->L);
  free_factor(P->U);
  free_factor(P->LH);
  free_factor(P->UH);
}

// export of the factors (host CSR; tests compare them with the oracle's ILUC)
void pc_export(const rbicg_prec *P, int which, int32_t *rp, int32_t *ci, void *v, int64_t *nnz) {
  const TriCSR &F = which == 0 ? P->L : P->U;
  *nnz = F.nnz;
  if (!rp) return;
  const size_t w = P->dtype == RBICG_F64 ? 8 : 16;
  RB_CUDA(cudaMemcpy(rp, F.rp, 4 * (P->n + 1), cudaMemcpyDeviceToHost));
  if (F.nnz) {
    RB_CUDA(cudaMemcpy(ci, F.ci, 4 * F.nnz, cudaMemcpyDeviceToHost));
    RB_CUDA(cudaMemcpy(v, F.v, w * F.nnz, cudaMemcpyDeviceToHost));
  }
}

}  // namespace rbicg
