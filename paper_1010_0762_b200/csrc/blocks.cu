// blocks.cu -- cycle-end / per-system block kernels.
//
//   spmm         C = A U, C~ = A^* Ũ (k columns, row-major n x k)
//   gram         G = X^H Y for column lists X, Y (the pencil Grams
//                Ψ~^*Ψ, Ψ~^*Φ of finalGenEigValue, and C~^*C)
//   gemm_panels  out = [columns] M (U_j = Φ_j W_j N_j etc.)
//
// The Gram is a two-stage deterministic reduction: blocks own a 32 x 32
// output tile and a chunk of rows; the per-chunk partials are summed in chunk
// order by a second kernel.
#include "hot.cuh"
#include <cstdlib>

namespace rbicg {

template <typename T> __device__ __forceinline__ T ldp(const void *p, int64_t i) {
  return reinterpret_cast<const T *>(p)[i];
}

// cp.async (LDGSTS) element copies with zero fill, for software pipelining of
// the row sub-tiles of the Gram kernels (the columns are arbitrary strided
// descriptors, so per-element async copies rather than bulk tensor copies).
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
template <typename T>
__device__ __forceinline__ void cp_async_el(T *dst, const T *src, bool pred) {
  const int sz = pred ? (int)sizeof(T) : 0;
  if (sizeof(T) == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "r"(sz)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "r"(sz)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ------------------------------------------------------------------ SpMM
// One block per SELL slice (32 rows) x k columns: the slice's column indices
// and values are loaded once, coalesced, into shared memory; thread
// (row lr, column j), j fastest, then gathers X rows (k contiguous values).
template <typename T>
__global__ void __launch_bounds__(1024) k_spmm(DevMat A, const T *__restrict__ X, T *__restrict__ Y,
                                               int k) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const int64_t sl = blockIdx.x;
  const int64_t off = A.sptr[sl];
  const int w = (int)((A.sptr[sl + 1] - off) >> 5);
  T *sv = reinterpret_cast<T *>(sm_raw);
  int32_t *sc = reinterpret_cast<int32_t *>(sv + 32 * w);
  for (int e = threadIdx.x; e < 32 * w; e += blockDim.x) {
    sc[e] = A.cols[off + e];
    sv[e] = reinterpret_cast<const T *>(A.vals)[off + e];
  }
  __syncthreads();
  const int lr = threadIdx.x / k, j = threadIdx.x - lr * k;
  const int64_t row = sl * 32 + lr;
  if (lr >= 32 || row >= A.n) return;
  T acc = zero<T>();
#pragma unroll 4
  for (int jj = 0; jj < w; ++jj) acc = mad(sv[jj * 32 + lr], X[(int64_t)sc[jj * 32 + lr] * k + j], acc);
  Y[row * k + j] = acc;
}

// generic fallback for very wide slices: thread per (row, column)
template <typename T>
__global__ void __launch_bounds__(256) k_spmm_wide(DevMat A, const T *__restrict__ X,
                                                   T *__restrict__ Y, int k) {
  const int64_t total = A.n * k;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / k;
    const int j = (int)(idx - row * k);
    const int64_t sl = row >> 5;
    const int lane = (int)(row & 31);
    const int64_t off = A.sptr[sl];
    const int w = (int)((A.sptr[sl + 1] - off) >> 5);
    T acc = zero<T>();
    for (int jj = 0; jj < w; ++jj)
      acc = mad(reinterpret_cast<const T *>(A.vals)[off + jj * 32 + lane],
                X[(int64_t)A.cols[off + jj * 32 + lane] * k + j], acc);
    Y[idx] = acc;
  }
}

// One thread per row computing all k outputs (KB >= k accumulators): the
// row's SELL entries are read once (coalesced across the warp) and each
// nonzero gathers one contiguous k-row of X.  k_spmm_rows0 (round 1, one
// nonzero at a time, RBICG_SPMM_V=0) was latency-bound (C3 cycle end 0.65 ms
// per SpMM, 2.9 TB/s); k_spmm_rows hoists a chunk of the row's SELL entries
// and keeps that chunk's X rows in flight (16-byte loads and stores for even
// k): 0.50 ms.  (Staging the output tile in shared memory for coalesced
// stores measured 0.66 ms.)
template <typename T, int KB>
__global__ void __launch_bounds__(256) k_spmm_rows0(DevMat A, const T *__restrict__ X,
                                                    T *__restrict__ Y, int k) {
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < A.n;
       row += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sl = row >> 5;
    const int lane = (int)(row & 31);
    const int64_t off = A.sptr[sl];
    const int w = (int)((A.sptr[sl + 1] - off) >> 5);
    T acc[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) acc[j] = zero<T>();
    for (int jj = 0; jj < w; ++jj) {
      const int c = __ldcs(A.cols + off + jj * 32 + lane);
      const T v = reinterpret_cast<const T *>(A.vals)[off + jj * 32 + lane];
      const T *xr = X + (int64_t)c * k;
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < k) acc[j] = mad(v, xr[j], acc[j]);
    }
    T *yr = Y + row * k;
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < k) yr[j] = acc[j];
  }
}
template <typename T, int KB, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_spmm_rows(DevMat A, const T *__restrict__ X,
                                                    T *__restrict__ Y, int k) {
  constexpr int NQ0 = (192 / (KB * (int)sizeof(T))) < 1 ? 1 : ((192 / (KB * (int)sizeof(T))) > 4 ? 4 : (192 / (KB * (int)sizeof(T))));
  constexpr int NQ = MINB >= 3 && KB >= 8 ? 1 : NQ0;
  const bool vec = sizeof(T) == 8 && (k % 2) == 0 && ((uintptr_t)X % 16) == 0 && ((uintptr_t)Y % 16) == 0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < A.n;
       row += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sl = row >> 5;
    const int lane = (int)(row & 31);
    const int64_t off = A.sptr[sl];
    const int w = (int)((A.sptr[sl + 1] - off) >> 5);
    T acc[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) acc[j] = zero<T>();
    for (int j0 = 0; j0 < w; j0 += NQ) {
      int c[NQ];
      T v[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const bool in = j0 + q < w;
        c[q] = in ? __ldcs(A.cols + off + (j0 + q) * 32 + lane) : (int)row;
        v[q] = in ? reinterpret_cast<const T *>(A.vals)[off + (j0 + q) * 32 + lane] : zero<T>();
      }
      T xv[NQ][KB];
      if constexpr (sizeof(T) == 8 && KB % 2 == 0) {
        if (vec) {
#pragma unroll
          for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int j = 0; j < KB; j += 2) {
              double2 t = j < k ? reinterpret_cast<const double2 *>(X + (int64_t)c[q] * k)[j / 2]
                                : make_double2(0.0, 0.0);
              xv[q][j] = t.x;
              xv[q][j + 1] = t.y;
            }
        } else {
#pragma unroll
          for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int j = 0; j < KB; ++j) xv[q][j] = j < k ? X[(int64_t)c[q] * k + j] : zero<T>();
        }
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
          for (int j = 0; j < KB; ++j) xv[q][j] = j < k ? X[(int64_t)c[q] * k + j] : zero<T>();
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int j = 0; j < KB; ++j) acc[j] = mad(v[q], xv[q][j], acc[j]);
    }
    T *yr = Y + row * k;
    if constexpr (sizeof(T) == 8 && KB % 2 == 0) {
      if (vec) {
#pragma unroll
        for (int j = 0; j < KB; j += 2)
          if (j < k) reinterpret_cast<double2 *>(yr)[j / 2] = make_double2(acc[j], acc[j + 1]);
        continue;
      }
    }
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < k) yr[j] = acc[j];
  }
}

template <typename T, int KB>
static void spmm_rows_launch(const DevMat &A, const T *X, T *Y, int k, cudaStream_t s, int nsm) {
  static const bool v0 = getenv("RBICG_SPMM_V") && atoi(getenv("RBICG_SPMM_V")) == 0;
  // resident blocks per SM the kernel is compiled for (register cap; the
  // gathers are latency-bound: ncu long-scoreboard stalls dominate at 2 blocks
  // of 94 registers).  3 (64 registers, one nonzero's X row per step for
  // k >= 8): C3 k = 10 SpMM 503 -> 435 us (profiles/r02_spmm_minb.txt);
  // RBICG_SPMM_MINB=1 restores the uncapped form (same FMA order, same bits)
  static const int minb = getenv("RBICG_SPMM_MINB") ? atoi(getenv("RBICG_SPMM_MINB")) : 3;
  auto fn = v0 ? k_spmm_rows0<T, KB>
               : (minb >= 4 ? k_spmm_rows<T, KB, 4>
                            : (minb == 3 ? k_spmm_rows<T, KB, 3> : (minb == 2 ? k_spmm_rows<T, KB, 2> : k_spmm_rows<T, KB>)));
  int per = 1;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, 0));
  const int64_t blocks = (A.n + 255) / 256;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)std::max(1, per) * nsm));
  fn<<<grid, 256, 0, s>>>(A, X, Y, k);
  RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
}

template <typename T> void launch_spmm(const DevMat &A, const T *X, T *Y, int k, cudaStream_t s) {
  if (k <= 0) return;
  RB_CHECK(k <= KMAX, RBICG_EINVAL);
  // real data: the row form (C3 cycle end 0.50 vs 0.65 ms for the slice form);
  // complex: the slice form (thread per (row, column): a warp's gathers cover
  // 32 / k whole 16k-byte X rows) -- C4 0.104 vs 0.25 ms
  static const bool rows_form = !getenv("RBICG_SPMM_SLICE");
  if (rows_form && sizeof(T) == 8 && A.max_w <= 64) {
    int dev = 0, nsm = 148;
    RB_CUDA(cudaGetDevice(&dev));
    RB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (k <= 4) spmm_rows_launch<T, 4>(A, X, Y, k, s, sm_budget(nsm));
    else if (k <= 8) spmm_rows_launch<T, 8>(A, X, Y, k, s, sm_budget(nsm));
    else if (k <= 12) spmm_rows_launch<T, 12>(A, X, Y, k, s, sm_budget(nsm));
    else if (k <= 16) spmm_rows_launch<T, 16>(A, X, Y, k, s, sm_budget(nsm));
    else if (k <= 24) spmm_rows_launch<T, 24>(A, X, Y, k, s, sm_budget(nsm));
    else spmm_rows_launch<T, 32>(A, X, Y, k, s, sm_budget(nsm));
    count_launch();
    return;
  }
  const size_t sm = (size_t)32 * std::max(1, A.max_w) * (sizeof(T) + 4);
  if (sm <= 48 * 1024) {
    k_spmm<T><<<(int)A.nslices, 32 * k, sm, s>>>(A, X, Y, k);
    RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
  } else {
    const int grid = (int)std::min<int64_t>((A.n * k + 255) / 256, 148 * 16);
    k_spmm_wide<T><<<grid, 256, 0, s>>>(A, X, Y, k);
    RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
  }
  count_launch();
}

// ------------------------------------------------------------------ Gram
// one warp per output entry: lanes sum chunks strided by 32, fixed shuffle tree
template <typename T>
__global__ void k_gram_reduce(const T *__restrict__ part, int nchunks, int mXY, T *__restrict__ G) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, l = threadIdx.x & 31;
  if (w >= mXY) return;
  T s = zero<T>();
  for (int c = l; c < nchunks; c += 32) s = add(s, part[(int64_t)c * mXY + w]);
  s = warp_sum(s);
  if (l == 0) G[w] = s;
}

// Register-tiled Gram (the pencil Grams of a cycle end: X = Ψ~ with 42..92
// columns, Y = [Ψ, X0]): each thread owns an MX x MY micro-tile of the
// block's output tile (up to 256 micro-tiles; the rest of the threads form
// further row groups over the same tile); the tile's X and Y rows pass
// through shared memory in double-buffered stages of G2R rows (cp.async, row
// index fastest so a warp reads 32 consecutive rows of a column).  Every
// column is read once per output tile -- one tile whenever the micro-tiles
// fit (every cycle end of the BASELINE configs) -- and the inner loop does
// MX*MY FMAs per MX + MY shared loads (fp64: 8 x 8, 64 FMAs per 16 loads).
constexpr int G2R = 32;   // rows per stage

template <typename T, int MX, int MY>
__global__ void __launch_bounds__(256, (sizeof(T) * MX * MY > 256 ? 1 : 2)) k_gram2(const ColDesc *__restrict__ X, int mX,
                                                  const ColDesc *__restrict__ Y, int mY, int tX,
                                                  int tY, int64_t n, int64_t chunk,
                                                  T *__restrict__ part) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const int tXp = (tX + MX - 1) / MX * MX, tYp = (tY + MY - 1) / MY * MY;
  const int ntx = tXp / MX, nty = tYp / MY, nmt = ntx * nty;
  const int ng = max(1, 256 / nmt);
  const int ncol = tXp + tYp;
  ColDesc *sd = reinterpret_cast<ColDesc *>(sm_raw);
  T *sbase = reinterpret_cast<T *>(sm_raw + ((sizeof(ColDesc) * ncol + 15) / 16) * 16);
  // [row][col]: X columns then Y columns; an odd row stride keeps the
  // row-fast cp.async stores of a warp (32 rows of one column) on distinct banks
  const int lds = ncol | 1;
  const int stage = G2R * lds;
  const int tilesY = (mY + tY - 1) / tY;
  const int bx = blockIdx.x / tilesY, by = blockIdx.x % tilesY;
  const int x0 = bx * tX, y0 = by * tY;
  const int tid = threadIdx.x;
  for (int c = tid; c < ncol; c += 256) {
    ColDesc d{nullptr, 0};
    if (c < tXp) {
      if (c < tX && x0 + c < mX) d = X[x0 + c];
    } else if (c - tXp < tY && y0 + c - tXp < mY) {
      d = Y[y0 + c - tXp];
    }
    sd[c] = d;
  }
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.y * chunk, r1 = min(n, r0 + chunk);
  const int mt = tid % nmt, g = tid / nmt;
  const bool active = g < ng;
  const int ix = mt / nty, iy = mt % nty;
  T acc[MX][MY];
#pragma unroll
  for (int u = 0; u < MX; ++u)
#pragma unroll
    for (int v = 0; v < MY; ++v) acc[u][v] = zero<T>();
  const int nel = G2R * ncol;
  auto load = [&](int64_t rb, int buf) {
    T *st = sbase + buf * stage;
    for (int e = tid; e < nel; e += 256) {
      const int c = e / G2R, r = e % G2R;
      const ColDesc d = sd[c];
      const int64_t row = rb + r;
      const bool ok = d.p != nullptr && row < r1;
      const T *src = reinterpret_cast<const T *>(ok ? d.p : (const void *)part);
      cp_async_el(st + r * lds + c, ok ? src + row * d.stride : src, ok);
    }
    cp_async_commit();
  };
  if (r0 < r1) load(r0, 0);
  int buf = 0;
  for (int64_t rb = r0; rb < r1; rb += G2R, buf ^= 1) {
    if (rb + G2R < r1) load(rb + G2R, buf ^ 1);
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (active) {
      const T *st = sbase + buf * stage;
      for (int r = g; r < G2R; r += ng) {
        const T *row = st + r * lds;
        T xv[MX], yv[MY];
        // micro-tile columns strided by the tile's micro-tile counts: the
        // threads of a warp (consecutive iy) read consecutive words, no bank
        // conflicts (contiguous 8-column micro-tiles put 9 threads on 2 banks);
        // (explicitly loading the next row's operands first: 3.93 vs 3.70 ms)
#pragma unroll
        for (int u = 0; u < MX; ++u) xv[u] = conj(row[u * ntx + ix]);
#pragma unroll
        for (int v = 0; v < MY; ++v) yv[v] = row[tXp + v * nty + iy];
#pragma unroll
        for (int u = 0; u < MX; ++u)
#pragma unroll
          for (int v = 0; v < MY; ++v) acc[u][v] = mad(xv[u], yv[v], acc[u][v]);
      }
    }
    __syncthreads();
  }
  if (!active) return;
  // partial (chunk, row group) -> part[((chunk * ng + g) * mX + a) * mY + b]
  const int64_t pc = (int64_t)blockIdx.y * ng + g;
#pragma unroll
  for (int u = 0; u < MX; ++u)
#pragma unroll
    for (int v = 0; v < MY; ++v) {
      const int a = u * ntx + ix, bb = v * nty + iy;
      if (a < tX && bb < tY && x0 + a < mX && y0 + bb < mY)
        part[(pc * mX + x0 + a) * mY + y0 + bb] = acc[u][v];
    }
}

// fp64 tensor-core Gram: the same stages as k_gram2, stored column-major
// ([col][row], column stride GMS = GR + 4 doubles, so the fragment loads of a
// half-warp -- 4 rows x 4 columns -- hit distinct banks); the TM x TN grid of
// 8 x 8 output tiles is computed by mma.sync m8n8k4 f64 (DMMA, the only fp64
// tensor-core form on sm_100a).  Work split: the tiles in column-major order
// (tm fastest) are cut into 8 contiguous ranges of ceil(TM*TN / 8) tiles, one
// per warp, so every SM sub-partition (warps w, w + 4) gets the same number of
// DMMAs.  (Round 2's first form gave warp w whole column tiles w, w + 8, ...:
// with TN = 9 (C3: 61 x 71) warp 0 did twice the work and its sub-partition's
// DMMA pipe bounded the kernel -- ncu: tensor pipe 62 % active, 3.19 ms.)
// Within a range the B fragment of a column is reused by its consecutive row
// tiles.  Partials per chunk as k_gram2 (ng = 1).  Complex: four real MMAs per
// tile (conj(x) y).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
template <typename T, int NTW, int GR, int NST>
__global__ void __launch_bounds__(256) k_gram_mma(const ColDesc *__restrict__ X, int mX,
                                                  const ColDesc *__restrict__ Y, int mY, int64_t n,
                                                  int64_t chunk, T *__restrict__ part) {
  // column stride: = 4 mod 16 doubles (real), = 4 mod 8 complex elements (the
  // 16-byte fragment loads of a quarter-warp then hit distinct banks)
  constexpr int GMS = GR + 4;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const int tXp = (mX + 7) / 8 * 8, tYp = (mY + 7) / 8 * 8;
  const int ncol = tXp + tYp;
  ColDesc *sd = reinterpret_cast<ColDesc *>(sm_raw);
  T *sbase = reinterpret_cast<T *>(sm_raw + ((sizeof(ColDesc) * ncol + 15) / 16) * 16);
  const int stage = ncol * GMS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = tid; c < ncol; c += 256) {
    ColDesc d{nullptr, 0};
    if (c < tXp) {
      if (c < mX) d = X[c];
    } else if (c - tXp < mY) {
      d = Y[c - tXp];
    }
    sd[c] = d;
  }
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  // thread -> (row lr = tid % GR of the stage, columns tid / GR + i 256 / GR):
  // no per-element index arithmetic (the loader dominated the instruction count)
  const int lr = tid % GR, cstep = 256 / GR;
  auto load = [&](int64_t rb, int buf) {
    T *st = sbase + buf * stage + lr;
    const int64_t row = rb + lr;
    const bool rok = row < r1;
    for (int c = tid / GR; c < ncol; c += cstep) {
      const ColDesc d = sd[c];
      const bool ok = rok && d.p != nullptr;
      const T *src = reinterpret_cast<const T *>(ok ? d.p : (const void *)part);
      cp_async_el(st + c * GMS, ok ? src + row * d.stride : src, ok);
    }
    cp_async_commit();
  };
  // this warp's tiles: linear indices [t0, t0 + nt) of the column-major grid
  const int TM = tXp / 8, TN = tYp / 8, NT = TM * TN;
  const int per = (NT + 7) / 8;
  const int t0 = min(NT, warp * per), nt = min(NT, t0 + per) - t0;
  const int tm0 = t0 % TM, tn0 = t0 / TM;
  constexpr bool CPLX = sizeof(T) == 16;
  double acc[NTW][2], aci[NTW][2];   // real parts; imaginary parts (complex)
#pragma unroll
  for (int t = 0; t < NTW; ++t) acc[t][0] = acc[t][1] = aci[t][0] = aci[t][1] = 0.0;
  // fragment offsets of the warp's tiles, fixed for the whole kernel (slots
  // t >= nt repeat the last tile: their loads stay in the stage, their MMAs
  // are skipped); with them the inner loop has no index arithmetic and its
  // loads can all be issued ahead of the MMAs
  int oa[NTW], ob[NTW];
  {
    int tm = tm0, tn = min(tn0, TN - 1);
#pragma unroll
    for (int t = 0; t < NTW; ++t) {
      oa[t] = tm * 8 * GMS;
      ob[t] = tn * 8 * GMS;
      if (t + 1 < nt) {
        if (++tm == TM) {
          tm = 0;
          ++tn;
        }
      }
    }
  }
  const int fr = lane & 3, fc = lane >> 2;   // fragment row (k) and column (m or n)
  // NST-stage ring: NST - 1 stages in flight while one is consumed
#pragma unroll
  for (int q = 0; q < NST - 1; ++q) {
    if (r0 + q * GR < r1) load(r0 + q * GR, q);
    else cp_async_commit();
  }
  int buf = 0;
  for (int64_t rb = r0; rb < r1; rb += GR, buf = (buf + 1) % NST) {
    {
      const int64_t rn = rb + (int64_t)(NST - 1) * GR;
      if (rn < r1) load(rn, (buf + NST - 1) % NST);
      else cp_async_commit();
    }
    cp_async_wait<NST - 1>();
    __syncthreads();
    const T *st = sbase + buf * stage;
    const T *sa = st + fc * GMS + fr;                 // A fragments: X column tm * 8 + fc
    const T *sb = st + (tXp + fc) * GMS + fr;         // B fragments: Y column tn * 8 + fc
#pragma unroll 2   // (4: same 1.23 ms for C4's complex pencil, with spills)
    for (int k0 = 0; k0 < GR; k0 += 4) {
      T b = sb[ob[0] + k0];
#pragma unroll
      for (int t = 0; t < NTW; ++t) {
        if (t > 0 && ob[t] != ob[t - 1]) b = sb[ob[t] + k0];   // a new column tile
        const T a = sa[oa[t] + k0];
        if (t < nt) {
          if constexpr (!CPLX) {
            dmma(acc[t], re(a), re(b));
          } else {   // conj(x) y = (xr yr + xi yi) + i (xr yi - xi yr)
            dmma(acc[t], re(a), re(b));
            dmma(acc[t], im(a), im(b));
            dmma(aci[t], re(a), im(b));
            dmma(aci[t], -im(a), re(b));
          }
        }
      }
    }
    __syncthreads();
  }
  // D fragment: row fc (of the 8 x 8 tile), columns 2 fr, 2 fr + 1
  int tm = tm0, tn = tn0;
#pragma unroll
  for (int t = 0; t < NTW; ++t) {
    if (t < nt) {
      const int a = tm * 8 + fc;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int bb = tn * 8 + 2 * fr + q;
        if (a < mX && bb < mY) {
          T v;
          if constexpr (CPLX) v = mk(acc[t][q], aci[t][q]);
          else v = acc[t][q];
          part[((int64_t)blockIdx.x * mX + a) * mY + bb] = v;
        }
      }
      if (++tm == TM) {
        tm = 0;
        ++tn;
      }
    }
  }
}

// Real data, the default: the same stages with a 2-D warp grid (WR x WC = 8
// warps, warp w = (w / WC, w % WC)), each warp owning an RM x RN rectangle of
// output tiles whose RM A fragments and RN B fragments it loads once per
// k-step: RM + RN fragment loads feed RM * RN MMAs.  The flat per-warp tile
// ranges above re-load an A fragment per tile and were bound by shared-memory
// wavefronts (ncu, C3 7 x 8 tiles: 76 % of the smem peak, DMMA pipe 57 %);
// the host picks (WR, RM, RN) for the shape by a cost model of the busiest
// SM sub-partition's MMAs against the stage's shared-memory wavefronts.
template <typename T, int RMX, int RNX, int GR, int NST>
__global__ void __launch_bounds__(256) k_gram_mma2(const ColDesc *__restrict__ X, int mX,
                                                   const ColDesc *__restrict__ Y, int mY, int64_t n,
                                                   int64_t chunk, T *__restrict__ part, int WC, int RM,
                                                   int RN) {
  constexpr int GMS = GR + 4;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const int tXp = (mX + 7) / 8 * 8, tYp = (mY + 7) / 8 * 8;
  const int ncol = tXp + tYp;
  ColDesc *sd = reinterpret_cast<ColDesc *>(sm_raw);
  T *sbase = reinterpret_cast<T *>(sm_raw + ((sizeof(ColDesc) * ncol + 15) / 16) * 16);
  const int stage = ncol * GMS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = tid; c < ncol; c += 256) {
    ColDesc d{nullptr, 0};
    if (c < tXp) {
      if (c < mX) d = X[c];
    } else if (c - tXp < mY) {
      d = Y[c - tXp];
    }
    sd[c] = d;
  }
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  const int lr = tid % GR, cstep = 256 / GR;
  auto load = [&](int64_t rb, int buf) {
    T *st = sbase + buf * stage + lr;
    const int64_t row = rb + lr;
    const bool rok = row < r1;
    for (int c = tid / GR; c < ncol; c += cstep) {
      const ColDesc d = sd[c];
      const bool ok = rok && d.p != nullptr;
      const T *src = reinterpret_cast<const T *>(ok ? d.p : (const void *)part);
      cp_async_el(st + c * GMS, ok ? src + row * d.stride : src, ok);
    }
    cp_async_commit();
  };
  const int TM = tXp / 8, TN = tYp / 8;
  const int tm0 = (warp / WC) * RM, tn0 = (warp % WC) * RN;
  const int rm = max(0, min(RM, TM - tm0)), rn = max(0, min(RN, TN - tn0));
  double acc[RMX][RNX][2];
#pragma unroll
  for (int i = 0; i < RMX; ++i)
#pragma unroll
    for (int j = 0; j < RNX; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int fr = lane & 3, fc = lane >> 2;
#pragma unroll
  for (int q = 0; q < NST - 1; ++q) {
    if (r0 + q * GR < r1) load(r0 + q * GR, q);
    else cp_async_commit();
  }
  int buf = 0;
  for (int64_t rb = r0; rb < r1; rb += GR, buf = (buf + 1) % NST) {
    {
      const int64_t rn_ = rb + (int64_t)(NST - 1) * GR;
      if (rn_ < r1) load(rn_, (buf + NST - 1) % NST);
      else cp_async_commit();
    }
    cp_async_wait<NST - 1>();
    __syncthreads();
    if (rm > 0 && rn > 0) {
      const T *st = sbase + buf * stage;
      const T *sa = st + (tm0 * 8 + fc) * GMS + fr;
      const T *sb = st + (tXp + tn0 * 8 + fc) * GMS + fr;
      // the stage's 8 k-steps fully unrolled (vs 2: C3 pencils 2.87 / 2.49 ->
      // 2.82 / 2.33 ms, profiles/r02_gram_forms.txt)
#pragma unroll
      for (int k0 = 0; k0 < GR; k0 += 4) {
        double a[RMX], b[RNX];
#pragma unroll
        for (int i = 0; i < RMX; ++i) a[i] = i < rm ? re(sa[i * 8 * GMS + k0]) : 0.0;
#pragma unroll
        for (int j = 0; j < RNX; ++j) b[j] = j < rn ? re(sb[j * 8 * GMS + k0]) : 0.0;
#pragma unroll
        for (int j = 0; j < RNX; ++j)
          if (j < rn)
#pragma unroll
            for (int i = 0; i < RMX; ++i)
              if (i < rm) dmma(acc[i][j], a[i], b[j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < RMX; ++i)
#pragma unroll
    for (int j = 0; j < RNX; ++j)
      if (i < rm && j < rn) {
        const int a = (tm0 + i) * 8 + fc;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int bb = (tn0 + j) * 8 + 2 * fr + q;
          if (a < mX && bb < mY) part[((int64_t)blockIdx.x * mX + a) * mY + bb] = T(acc[i][j][q]);
        }
      }
}

// warp-grid choice for k_gram_mma2: (WR, RM, RN) minimising
// max(16 x MMAs of the busiest sub-partition, 2 x fragment loads + stage
// writes) per k-step -- cycles of the DMMA pipe (16 per m8n8k4 f64, measured
// 37 TFLOP/s) against shared-memory wavefronts (256-byte fragment loads)
struct WarpGrid {
  int WR, WC, RM, RN, cost;
};
static WarpGrid pick_warp_grid(int TM, int TN, int ncol, const int (*shapes)[2], int nshapes) {
  WarpGrid best{0, 0, 0, 0, 1 << 30};
  for (int WR : {1, 2, 4, 8}) {
    const int WC = 8 / WR, RM = (TM + WR - 1) / WR, RN = (TN + WC - 1) / WC;
    bool fits = false;
    for (int q = 0; q < nshapes; ++q) fits |= RM <= shapes[q][0] && RN <= shapes[q][1];
    if (!fits) continue;
    int D[4] = {0, 0, 0, 0}, L = 0;
    for (int w = 0; w < 8; ++w) {
      const int r = std::max(0, std::min(RM, TM - (w / WC) * RM));
      const int c = std::max(0, std::min(RN, TN - (w % WC) * RN));
      D[w % 4] += r * c;
      if (r > 0 && c > 0) L += r + c;
    }
    const int maxD = std::max(std::max(D[0], D[1]), std::max(D[2], D[3]));
    // primary: the bound; ties (common: equal MMA balance) to fewer loads
    const int cost = 4 * std::max(16 * maxD, 2 * L + ncol / 3) + (2 * L + ncol / 3) / 8;
    if (cost < best.cost) best = WarpGrid{WR, WC, RM, RN, cost};
  }
  return best;
}

// real: up to 10 x 16 tiles (X up to 80 columns, Y up to 128: every BASELINE
// pencil, C2/C3 51..61 x 61..71, C5 71 x 91), NTW = 20 tiles per warp;
// complex: up to 8 x 8 tiles (64 x 64 per launch: C4's 49 x 57), four real
// MMAs per tile; false when it does not apply
template <typename T, int GR, int NST>
static bool gram_mma_run(const std::vector<ColDesc> &X, const std::vector<ColDesc> &Y, int64_t n,
                         std::vector<cplx> &G, rbicg_ctx *ctx, cudaStream_t strm) {
  constexpr bool CPLX = sizeof(T) == 16;
  constexpr int MAXM = CPLX ? 64 : 80, MAXN = CPLX ? 64 : 128;
  constexpr int GMS = GR + 4;
  const int mX = (int)X.size(), mY = (int)Y.size();
  if (mX > MAXM || mY > MAXN) return false;
  // tiles per warp: the smallest instantiated NTW >= ceil(TM TN / 8)
  const int per = ((mX + 7) / 8 * ((mY + 7) / 8) + 7) / 8;
  void (*kern)(const ColDesc *, int, const ColDesc *, int, int64_t, int64_t, T *) = nullptr;
  if constexpr (CPLX) {
    if (per <= 2) kern = k_gram_mma<T, 2, GR, NST>;
    else if (per <= 4) kern = k_gram_mma<T, 4, GR, NST>;
    else if (per <= 6) kern = k_gram_mma<T, 6, GR, NST>;
    else kern = k_gram_mma<T, 8, GR, NST>;
  } else {
    if (per <= 2) kern = k_gram_mma<T, 2, GR, NST>;
    else if (per <= 4) kern = k_gram_mma<T, 4, GR, NST>;
    else if (per <= 6) kern = k_gram_mma<T, 6, GR, NST>;
    else if (per <= 7) kern = k_gram_mma<T, 7, GR, NST>;
    else if (per <= 8) kern = k_gram_mma<T, 8, GR, NST>;
    else if (per <= 9) kern = k_gram_mma<T, 9, GR, NST>;
    else if (per <= 10) kern = k_gram_mma<T, 10, GR, NST>;
    else if (per <= 12) kern = k_gram_mma<T, 12, GR, NST>;
    else if (per <= 14) kern = k_gram_mma<T, 14, GR, NST>;
    else if (per <= 16) kern = k_gram_mma<T, 16, GR, NST>;
    else kern = k_gram_mma<T, 20, GR, NST>;
  }
  const int ncol = (mX + 7) / 8 * 8 + (mY + 7) / 8 * 8;
  const size_t smem = ((sizeof(ColDesc) * ncol + 15) / 16) * 16 + sizeof(T) * NST * (size_t)ncol * GMS;
  // real data: the 2-D warp grid (RBICG_GRAM_FLAT=1: the flat tile ranges)
  static const bool flat = getenv("RBICG_GRAM_FLAT") != nullptr;
  void (*kern2)(const ColDesc *, int, const ColDesc *, int, int64_t, int64_t, T *, int, int, int) = nullptr;
  WarpGrid wg{};
  if constexpr (!CPLX) {
    if (!flat) {
      // instantiated rectangles (RMX, RNX)
      static const int shapes[][2] = {{2, 1}, {4, 1}, {7, 1}, {8, 1}, {10, 2}, {2, 2}, {3, 2}, {4, 2}, {4, 3},
                                      {5, 2}, {5, 3}, {5, 4}, {2, 3}, {2, 4}, {2, 5}, {3, 4}, {3, 6}, {3, 8}};
      const int nsh = (int)(sizeof(shapes) / sizeof(shapes[0]));
      const int TM = (mX + 7) / 8, TN = (mY + 7) / 8;
      wg = pick_warp_grid(TM, TN, 8 * (TM + TN), shapes, nsh);
      // the smallest instantiated rectangle holding (RM, RN).  Measured on the
      // C3 probe's two pencils (profiles/r02_gram_forms.txt): 7 x 8 tiles
      // 2.49 ms (flat 2.45), 8 x 9 tiles 2.86 ms (flat 3.66) -- the grid is the
      // default wherever it fits (the cost model picks its shape only)
      int bq = -1;
      for (int q = 0; q < nsh; ++q)
        if (wg.RM <= shapes[q][0] && wg.RN <= shapes[q][1] &&
            (bq < 0 || shapes[q][0] * shapes[q][1] < shapes[bq][0] * shapes[bq][1]))
          bq = q;
      switch (bq) {
        case 0: kern2 = k_gram_mma2<T, 2, 1, GR, NST>; break;
        case 1: kern2 = k_gram_mma2<T, 4, 1, GR, NST>; break;
        case 2: kern2 = k_gram_mma2<T, 7, 1, GR, NST>; break;
        case 3: kern2 = k_gram_mma2<T, 8, 1, GR, NST>; break;
        case 4: kern2 = k_gram_mma2<T, 10, 2, GR, NST>; break;
        case 5: kern2 = k_gram_mma2<T, 2, 2, GR, NST>; break;
        case 6: kern2 = k_gram_mma2<T, 3, 2, GR, NST>; break;
        case 7: kern2 = k_gram_mma2<T, 4, 2, GR, NST>; break;
        case 8: kern2 = k_gram_mma2<T, 4, 3, GR, NST>; break;
        case 9: kern2 = k_gram_mma2<T, 5, 2, GR, NST>; break;
        case 10: kern2 = k_gram_mma2<T, 5, 3, GR, NST>; break;
        case 11: kern2 = k_gram_mma2<T, 5, 4, GR, NST>; break;
        case 12: kern2 = k_gram_mma2<T, 2, 3, GR, NST>; break;
        case 13: kern2 = k_gram_mma2<T, 2, 4, GR, NST>; break;
        case 14: kern2 = k_gram_mma2<T, 2, 5, GR, NST>; break;
        case 15: kern2 = k_gram_mma2<T, 3, 4, GR, NST>; break;
        case 16: kern2 = k_gram_mma2<T, 3, 6, GR, NST>; break;
        case 17: kern2 = k_gram_mma2<T, 3, 8, GR, NST>; break;
        default: break;
      }
    }
  }
  const void *kv = kern2 ? (const void *)kern2 : (const void *)kern;   // (attributes: prepare_block_kernels)
  if (smem > 200 * 1024) return false;
  int occ = 1;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kv, 256, smem));
  const int64_t slots = (int64_t)std::max(1, occ) * sm_budget(ctx->nsm);
  int nchunks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 4 * GR - 1) / (4 * GR), slots));
  const int64_t chunk = ((n + nchunks - 1) / nchunks + GR - 1) / GR * GR;
  nchunks = (int)((n + chunk - 1) / chunk);
  const size_t desc_bytes = sizeof(ColDesc) * (mX + mY);
  const size_t part_bytes = sizeof(T) * (size_t)nchunks * mX * mY;
  const size_t g_bytes = sizeof(T) * (size_t)mX * mY;
  char *buf = (char *)ws_alloc(desc_bytes + part_bytes + g_bytes + 64);
  ColDesc *dX = (ColDesc *)buf;
  T *dpart = (T *)(buf + ((desc_bytes + 15) / 16) * 16);
  T *dG = dpart + (size_t)nchunks * mX * mY;
  std::vector<ColDesc> both(X);
  both.insert(both.end(), Y.begin(), Y.end());
  RB_CUDA(cudaMemcpyAsync(dX, both.data(), desc_bytes, cudaMemcpyHostToDevice, strm));
  if (kern2) kern2<<<nchunks, 256, smem, strm>>>(dX, mX, dX + mX, mY, n, chunk, dpart, wg.WC, wg.RM, wg.RN);
  else kern<<<nchunks, 256, smem, strm>>>(dX, mX, dX + mX, mY, n, chunk, dpart);
  k_gram_reduce<T><<<(mX * mY * 32 + 255) / 256, 256, 0, strm>>>(dpart, nchunks, mX * mY, dG);
  RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
  count_launch(2);
  std::vector<T> h((size_t)mX * mY);
  RB_CUDA(cudaMemcpyAsync(h.data(), dG, g_bytes, cudaMemcpyDeviceToHost, strm));
  RB_CUDA(cudaStreamSynchronize(strm));
  ws_free(buf);
  for (size_t i = 0; i < h.size(); ++i) G[i] = cplx(re(h[i]), im(h[i]));
  return true;
}

template <typename T, int MX, int MY>
static void gram2_run(const std::vector<ColDesc> &X, const std::vector<ColDesc> &Y, int64_t n,
                      std::vector<cplx> &G, rbicg_ctx *ctx, cudaStream_t strm) {
  const int mX = (int)X.size(), mY = (int)Y.size();
  // output tile: all of X x Y when its micro-tiles fit 256 threads, else
  // split Y (then X) into tiles that do
  int ntxA = (mX + MX - 1) / MX, ntyA = (mY + MY - 1) / MY;
  int ntx = std::min(ntxA, 16), nty = std::max(1, std::min(ntyA, 256 / ntx));
  if (ntxA * ntyA <= 256) {
    ntx = ntxA;
    nty = ntyA;
  }
  const int tX = std::min(mX, ntx * MX), tY = std::min(mY, nty * MY);
  const int tiles = ((mX + tX - 1) / tX) * ((mY + tY - 1) / tY);
  const int nmt = ((tX + MX - 1) / MX) * ((tY + MY - 1) / MY);
  const int ng = std::max(1, 256 / nmt);
  const int ncol = (tX + MX - 1) / MX * MX + (tY + MY - 1) / MY * MY;
  const size_t smem = ((sizeof(ColDesc) * ncol + 15) / 16) * 16 + sizeof(T) * 2 * G2R * (ncol | 1);
  static bool attr = false;
  if (!attr) {
    RB_CUDA(cudaFuncSetAttribute((const void *)k_gram2<T, MX, MY>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  RB_CHECK(smem <= 200 * 1024, RBICG_EINVAL);
  // resident blocks per SM (1 for the 8 x 8 fp64 micro-tiles: 64 accumulators
  // per thread), whole waves of (tile, chunk) blocks
  const int64_t slots = (int64_t)(sizeof(T) * MX * MY > 256 ? 2 : 4) * sm_budget(ctx->nsm);
  int nchunks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 4 * G2R - 1) / (4 * G2R),
                                                            (slots + tiles - 1) / tiles));
  const int64_t chunk = ((n + nchunks - 1) / nchunks + G2R - 1) / G2R * G2R;
  nchunks = (int)((n + chunk - 1) / chunk);
  const size_t desc_bytes = sizeof(ColDesc) * (mX + mY);
  const size_t part_bytes = sizeof(T) * (size_t)nchunks * ng * mX * mY;
  const size_t g_bytes = sizeof(T) * (size_t)mX * mY;
  char *buf = (char *)ws_alloc(desc_bytes + part_bytes + g_bytes + 64);
  ColDesc *dX = (ColDesc *)buf;
  T *dpart = (T *)(buf + ((desc_bytes + 15) / 16) * 16);
  T *dG = dpart + (size_t)nchunks * ng * mX * mY;
  std::vector<ColDesc> both(X);
  both.insert(both.end(), Y.begin(), Y.end());
  RB_CUDA(cudaMemcpyAsync(dX, both.data(), desc_bytes, cudaMemcpyHostToDevice, strm));
  dim3 grid(tiles, nchunks);
  k_gram2<T, MX, MY><<<grid, 256, smem, strm>>>(dX, mX, dX + mX, mY, tX, tY, n, chunk, dpart);
  k_gram_reduce<T><<<(mX * mY * 32 + 255) / 256, 256, 0, strm>>>(dpart, ng * nchunks, mX * mY, dG);
  RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
  count_launch(2);
  std::vector<T> h((size_t)mX * mY);
  RB_CUDA(cudaMemcpyAsync(h.data(), dG, g_bytes, cudaMemcpyDeviceToHost, strm));
  RB_CUDA(cudaStreamSynchronize(strm));
  ws_free(buf);
  for (size_t i = 0; i < h.size(); ++i) G[i] = cplx(re(h[i]), im(h[i]));
}

template <typename T>
void gram(const std::vector<ColDesc> &X, const std::vector<ColDesc> &Y, int64_t n,
          std::vector<cplx> &G, rbicg_ctx *ctx, cudaStream_t strm) {
  const int mX = (int)X.size(), mY = (int)Y.size();
  G.assign((size_t)mX * mY, cplx(0, 0));
  if (mX == 0 || mY == 0) return;
  static const int var = getenv("RBICG_GRAM2") ? atoi(getenv("RBICG_GRAM2")) : 0;
  if constexpr (sizeof(T) == 16) {
    // complex: four real fp64 tensor-core MMAs per tile (RBICG_GRAM2=44: FFMA)
    // (up to 64 x 64 per launch; a wider Y is split into 64-column pieces --
    // two column tiles per warp need 188 registers and measured slower than the
    // FFMA form, 2.07 vs 1.95 ms at C4)
    if (var == 0 && X.size() <= 64) {
      const int mX = (int)X.size(), mY = (int)Y.size();
      bool ok = true;
      for (int y0 = 0; y0 < mY && ok; y0 += 64) {
        const int w = std::min(64, mY - y0);
        std::vector<ColDesc> Yp(Y.begin() + y0, Y.begin() + y0 + w);
        std::vector<cplx> Gp;
        Gp.assign((size_t)mX * w, cplx(0, 0));
        ok = gram_mma_run<T, 32, 2>(X, Yp, n, Gp, ctx, strm);
        if (ok)
          for (int a = 0; a < mX; ++a)
            for (int b = 0; b < w; ++b) G[(size_t)a * mY + y0 + b] = Gp[(size_t)a * w + b];
      }
      if (ok) return;
    }
    gram2_run<T, 4, 4>(X, Y, n, G, ctx, strm);
  } else {
    // fp64 tensor cores (RBICG_GRAM2=88 / 48 / 44: the FFMA micro-tile forms)
    // (16-row stages, 3-4 stages, TMA bulk staging per column segment and a
    // 2 x 4 warp grid measured slower: 3.4-5.4 ms)
    if (var == 0 && gram_mma_run<T, 32, 2>(X, Y, n, G, ctx, strm)) return;
    if (var == 48) return gram2_run<T, 4, 8>(X, Y, n, G, ctx, strm);
    if (var == 44) return gram2_run<T, 4, 4>(X, Y, n, G, ctx, strm);
    gram2_run<T, 8, 8>(X, Y, n, G, ctx, strm);   // RBICG_GRAM2=88
  }
}

// ------------------------------------------------------------------ C~^*C Gram
// The bi-orthogonalisation Gram of two row-major n x k blocks (C, C~): the
// column norms of both and C~^*C, register-tiled -- each thread owns a 4 x 4
// tile of C~^*C (or 4 norms) over a strided subset of the staged rows, so a
// shared-memory load feeds 2 (not 0.5) FMAs.  Rows arrive in 64-row
// sub-tiles by cp.async, double buffered (both blocks' sub-tiles are single
// contiguous ranges).  Output order: |c_j|^2, |c~_j|^2, then c~_a^* c_b (a-major).
// GCR rows per sub-tile (64; 288-row sub-tiles measured no faster at k = 10:
// 93 vs 87 us on C2)
static int gcr_rows(int) {
  static const int r = getenv("RBICG_GCR_ROWS") ? atoi(getenv("RBICG_GCR_ROWS")) : 128;
  return r;
}
template <typename T>
__global__ void __launch_bounds__(256) k_gram_cc(const T *__restrict__ C, const T *__restrict__ Ct, int k,
                                                 int64_t n, int64_t chunk, int GCR, T *__restrict__ part) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T *sbase = reinterpret_cast<T *>(sm_raw);   // 2 stages x [C rows | C~ rows], GCR * k each
  const int stage = 2 * GCR * k;
  const int tid = threadIdx.x;
  const int kb = (k + 3) / 4, W = kb * kb + 2 * kb, R = max(1, 256 / W);
  const int item = tid % W, grp = tid / W;
  const bool act = grp < R;
  const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  auto load = [&](int64_t rb, int buf) {
    T *st = sbase + buf * stage;
    const int rows = (int)min((int64_t)GCR, r1 - rb);
    const int ne = GCR * k, nv = rows * k;
    constexpr int PER = 16 / sizeof(T);
    for (int q = 0; q < 2; ++q) {
      const T *src = (q ? Ct : C) + rb * k;
      T *dst = st + q * GCR * k;
      for (int e = tid * PER; e < ne; e += 256 * PER) {
        const int valid = max(0, min(PER, nv - e)) * (int)sizeof(T);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst + e)),
                     "l"(valid ? src + e : src), "r"(valid)
                     : "memory");
      }
    }
    cp_async_commit();
  };
  // item -> (kind, A, B): tiles first, then the C norms, then the C~ norms
  const bool tile = item < kb * kb;
  const int A = tile ? item / kb : 0, B = tile ? item % kb : (item - kb * kb) % kb;
  const int side = tile ? 0 : (item - kb * kb) / kb;   // norms: 0 C, 1 C~
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = zero<T>();
  if (r0 < r1) load(r0, 0);
  int buf = 0;
  for (int64_t rb = r0; rb < r1; rb += GCR, buf ^= 1) {
    if (rb + GCR < r1) load(rb + GCR, buf ^ 1);
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const T *sc = sbase + buf * stage;
    const T *sct = sc + GCR * k;
    const int rows = (int)min((int64_t)GCR, r1 - rb);
    if (act) {
      if (tile) {
        for (int rr = grp; rr < rows; rr += R) {
          T a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int ca = 4 * A + i, cb = 4 * B + i;
            a[i] = ca < k ? sct[rr * k + ca] : zero<T>();
            b[i] = cb < k ? sc[rr * k + cb] : zero<T>();
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = cmad(a[i], b[j], acc[i][j]);
        }
      } else {
        const T *sx = side ? sct : sc;
        for (int rr = grp; rr < rows; rr += R) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int cj = 4 * B + j;
            const T v = cj < k ? sx[rr * k + cj] : zero<T>();
            acc[0][j] = cmad(v, v, acc[0][j]);
          }
        }
      }
    }
    __syncthreads();
  }
  // reduce over the row groups: red[grp][item][16], then one sum per output
  T *red = sbase;   // reuses the stages (>= 256 * 16 elements: checked by the host)
  if (act)
#pragma unroll
    for (int e = 0; e < 16; ++e) red[((size_t)grp * W + item) * 16 + e] = acc[e / 4][e % 4];
  __syncthreads();
  const int np = 2 * k + k * k;
  for (int o = tid; o < np; o += 256) {
    int it, e;
    if (o < k) {   // |c_o|^2
      it = kb * kb + o / 4;
      e = o % 4;
    } else if (o < 2 * k) {
      it = kb * kb + kb + (o - k) / 4;
      e = (o - k) % 4;
    } else {
      const int a2 = (o - 2 * k) / k, b2 = (o - 2 * k) % k;
      it = (a2 / 4) * kb + b2 / 4;
      e = (a2 % 4) * 4 + b2 % 4;
    }
    T sum = zero<T>();
    for (int g = 0; g < R; ++g) sum = add(sum, red[((size_t)g * W + it) * 16 + e]);
    part[(int64_t)blockIdx.x * np + o] = sum;
  }
}

// fp64 tensor-core form (real data, the default): the register-tiled FFMA
// kernel above is shared-memory bound (ncu, C3 k = 10: smem wavefronts 80 %
// of peak, 0.50 ms for 1.13 GB, 0.35 of the HBM peak) -- every 4 x 4 tile
// re-reads its operands.  Here each warp takes 4-row k-steps of the staged
// rows and one fragment load per 8-column tile of C~ and of C feeds all
// KT^2 tiles of C~^*C (mma.sync m8n8k4 f64); the column norms are plain FMAs
// on the fragment registers (lane = (row k0 + (lane & 3), column lane >> 2)
// of the tile), summed over the 4 row lanes at the end -- as diagonal MMA
// tiles they doubled the MMA count (ncu: 0.29 ms, MMA-bound).
// Stages: 128 rows of C and of C~ (contiguous), 3-deep cp.async ring.  Same
// partial layout as k_gram_cc (|c_j|^2, |c~_j|^2, c~_a^*c_b).
template <int KT>
__global__ void __launch_bounds__(256) k_gram_cc_mma(const double *__restrict__ C,
                                                     const double *__restrict__ Ct, int k, int64_t n,
                                                     int64_t chunk, double *__restrict__ part) {
  constexpr int GCR = 128, NST = 3, NTL = KT * KT + 2 * KT;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double *sbase = reinterpret_cast<double *>(sm_raw);   // NST x [C rows | C~ rows]
  double nt_[KT], nc_[KT];                              // per-lane column-norm partials
  const int stage = 2 * GCR * k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane & 3, fc = lane >> 2;
  const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  auto load = [&](int64_t rb, int buf) {
    double *st = sbase + buf * stage;
    const int rows = (int)min((int64_t)GCR, r1 - rb);
    const int ne = GCR * k, nv = rows * k;
    for (int q = 0; q < 2; ++q) {
      const double *src = (q ? Ct : C) + rb * k;
      double *dst = st + q * GCR * k;
      for (int e = tid * 2; e < ne; e += 256 * 2) {
        const int valid = max(0, min(2, nv - e)) * 8;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst + e)),
                     "l"(valid ? src + e : src), "r"(valid)
                     : "memory");
      }
    }
    cp_async_commit();
  };
  double acc[KT * KT][2];   // C~^*C tiles (i-major)
#pragma unroll
  for (int t = 0; t < KT * KT; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
  for (int i = 0; i < KT; ++i) nt_[i] = nc_[i] = 0.0;
#pragma unroll
  for (int q = 0; q < NST - 1; ++q) {
    if (r0 + q * GCR < r1) load(r0 + q * GCR, q);
    else cp_async_commit();
  }
  int buf = 0;
  for (int64_t rb = r0; rb < r1; rb += GCR, buf = (buf + 1) % NST) {
    {
      const int64_t rn = rb + (int64_t)(NST - 1) * GCR;
      if (rn < r1) load(rn, (buf + NST - 1) % NST);
      else cp_async_commit();
    }
    cp_async_wait<NST - 1>();
    __syncthreads();
    const double *sc = sbase + buf * stage, *sct = sc + GCR * k;
#pragma unroll 2
    for (int ks = warp; ks < GCR / 4; ks += 8) {
      const int ro = (ks * 4 + fr) * k;
      double at[KT], bc[KT];
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        const int col = i * 8 + fc;
        at[i] = col < k ? sct[ro + col] : 0.0;
        bc[i] = col < k ? sc[ro + col] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j) dmma(acc[i * KT + j], at[i], bc[j]);
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        nt_[i] = fma(at[i], at[i], nt_[i]);
        nc_[i] = fma(bc[i], bc[i], nc_[i]);
      }
    }
    __syncthreads();
  }
  // warp partials -> shared memory (reusing the stages), summed in warp order
  double *red = sbase;   // [warp][tile][64]
#pragma unroll
  for (int t = 0; t < KT * KT; ++t) {
    red[((size_t)warp * NTL + t) * 64 + fc * 8 + 2 * fr] = acc[t][0];
    red[((size_t)warp * NTL + t) * 64 + fc * 8 + 2 * fr + 1] = acc[t][1];
  }
  // norms: sum the 4 row lanes (fr) of each column, store on the diagonal
  // slots of the norm "tiles" (the layout the output loop reads)
#pragma unroll
  for (int i = 0; i < KT; ++i) {
    double a = nt_[i], c = nc_[i];
    a += __shfl_xor_sync(0xffffffffu, a, 1);
    a += __shfl_xor_sync(0xffffffffu, a, 2);
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    if (fr == 0) {
      red[((size_t)warp * NTL + KT * KT + i) * 64 + fc * 9] = a;
      red[((size_t)warp * NTL + KT * KT + KT + i) * 64 + fc * 9] = c;
    }
  }
  __syncthreads();
  const int np = 2 * k + k * k;
  for (int o = tid; o < np; o += 256) {
    int t, e;
    if (o < k) {   // |c_o|^2
      t = KT * KT + KT + o / 8;
      e = (o % 8) * 9;
    } else if (o < 2 * k) {   // |c~_o|^2
      t = KT * KT + (o - k) / 8;
      e = ((o - k) % 8) * 9;
    } else {   // c~_a^* c_b
      const int a2 = (o - 2 * k) / k, b2 = (o - 2 * k) % k;
      t = (a2 / 8) * KT + b2 / 8;
      e = (a2 % 8) * 8 + b2 % 8;
    }
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) sum += red[((size_t)w * NTL + t) * 64 + e];
    part[(int64_t)blockIdx.x * np + o] = sum;
  }
}

template <int KT>
static void gram_cc_mma_launch(const double *C, const double *Ct, int k, int64_t n, int &nb_out,
                               rbicg_ctx *ctx, cudaStream_t strm, double **buf_out) {
  constexpr int GCR = 128, NST = 3, NTL = KT * KT + 2 * KT;
  const size_t sm = std::max(sizeof(double) * NST * 2 * GCR * (size_t)k, sizeof(double) * 8 * NTL * 64);
  RB_CHECK(sm <= 200 * 1024, RBICG_EINVAL);   // (attributes: prepare_block_kernels)
  int per = 1;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_gram_cc_mma<KT>, 256, sm));
  const int np = 2 * k + k * k;
  int nchunks = (int)std::max<int64_t>(
      1, std::min<int64_t>((n + 4 * GCR - 1) / (4 * GCR), (int64_t)std::max(1, per) * sm_budget(ctx->nsm)));
  const int64_t chunk = ((n + nchunks - 1) / nchunks + GCR - 1) / GCR * GCR;
  const int nb = (int)((n + chunk - 1) / chunk);
  double *buf = (double *)ws_alloc(sizeof(double) * ((size_t)nb * np + np) + 64);
  k_gram_cc_mma<KT><<<nb, 256, sm, strm>>>(C, Ct, k, n, chunk, buf);
  RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
  nb_out = nb;
  *buf_out = buf;
}

template <typename T>
void gram_cc(const T *C, const T *Ct, int k, int64_t n, std::vector<cplx> &out, rbicg_ctx *ctx,
             cudaStream_t strm) {
  const int np = 2 * k + k * k;
  out.assign(np, cplx(0, 0));
  if (k == 0) return;
  const int kb = (k + 3) / 4, W = kb * kb + 2 * kb;
  RB_CHECK(W <= 256, RBICG_EINVAL);
  static const bool ffma = getenv("RBICG_GRAM_CC_FFMA") != nullptr;
  if constexpr (sizeof(T) == 8) {
    // fp64 tensor cores (rows 16-byte aligned: C, C~ of the recycle blocks)
    if (!ffma && ((uintptr_t)C % 16) == 0 && ((uintptr_t)Ct % 16) == 0) {
      int nb = 0;
      double *buf = nullptr;
      if (k <= 8) gram_cc_mma_launch<1>(C, Ct, k, n, nb, ctx, strm, &buf);
      else if (k <= 16) gram_cc_mma_launch<2>(C, Ct, k, n, nb, ctx, strm, &buf);
      else if (k <= 24) gram_cc_mma_launch<3>(C, Ct, k, n, nb, ctx, strm, &buf);
      else gram_cc_mma_launch<4>(C, Ct, k, n, nb, ctx, strm, &buf);
      double *dG = buf + (size_t)nb * np;
      k_gram_reduce<double><<<(np * 32 + 255) / 256, 256, 0, strm>>>(buf, nb, np, dG);
      RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
      count_launch(2);
      std::vector<double> h(np);
      RB_CUDA(cudaMemcpyAsync(h.data(), dG, sizeof(double) * np, cudaMemcpyDeviceToHost, strm));
      RB_CUDA(cudaStreamSynchronize(strm));
      ws_free(buf);
      for (int i = 0; i < np; ++i) out[i] = cplx(h[i], 0.0);
      return;
    }
  }
  // rows per stage: halved until two stages of both blocks fit (complex k > 19
  // overflowed the 160 KB stage budget at 128 rows: EINVAL, caught by
  // test_projection_parity_widths)
  int GCR = gcr_rows(k);
  while (GCR > 16 && sizeof(T) * 2 * 2 * GCR * (size_t)k > 160 * 1024) GCR /= 2;
  const size_t sm = std::max(sizeof(T) * 2 * 2 * GCR * (size_t)k,
                             sizeof(T) * 16 * (size_t)W * std::max(1, 256 / W));
  RB_CHECK(sm <= 160 * 1024, RBICG_EINVAL);
  // one full wave of resident blocks (a partial second wave left SMs idle)
  int per = 1;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_gram_cc<T>, 256, sm));
  static const int cps = getenv("RBICG_GCR_CPS") ? atoi(getenv("RBICG_GCR_CPS")) : 0;
  const int nchunks = (int)std::max<int64_t>(
      1, std::min<int64_t>((n + 1023) / 1024, (cps ? cps : std::max(1, per)) * sm_budget(ctx->nsm)));
  const int64_t chunk = ((n + nchunks - 1) / nchunks + GCR - 1) / GCR * GCR;
  const int nb = (int)((n + chunk - 1) / chunk);
  char *buf = (char *)ws_alloc(sizeof(T) * ((size_t)nb * np + np) + 64);
  T *dpart = (T *)buf;
  T *dG = dpart + (size_t)nb * np;
  k_gram_cc<T><<<nb, 256, sm, strm>>>(C, Ct, k, n, chunk, GCR, dpart);
  k_gram_reduce<T><<<(np * 32 + 255) / 256, 256, 0, strm>>>(dpart, nb, np, dG);
  RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
  count_launch(2);
  std::vector<T> h(np);
  RB_CUDA(cudaMemcpyAsync(h.data(), dG, sizeof(T) * np, cudaMemcpyDeviceToHost, strm));
  RB_CUDA(cudaStreamSynchronize(strm));
  ws_free(buf);
  for (int i = 0; i < np; ++i) out[i] = cplx(re(h[i]), im(h[i]));
}

// ------------------------------------------------------------------ panels x M
// out[row, c] = Σ_a X_a[row] M[a, c]; one thread per row keeps the whole output
// row in registers (PB >= p accumulators), so out may alias an input panel
// with the same layout.  Column loads are coalesced across the warp for
// vector columns; M lives in shared memory.
template <typename T, int PB>
__global__ void __launch_bounds__(256) k_gemm_panels(const ColDesc *__restrict__ X, int mX,
                                                     const T *__restrict__ M, int p, int64_t n,
                                                     T *out, T *out_last) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T *sM = reinterpret_cast<T *>(sm_raw);                 // [mX][PB], zero padded
  ColDesc *sX = reinterpret_cast<ColDesc *>(sM + (size_t)mX * PB);
  for (int e = threadIdx.x; e < mX * PB; e += blockDim.x) {
    const int a = e / PB, c = e % PB;
    sM[e] = c < p ? M[a * p + c] : zero<T>();
  }
  for (int e = threadIdx.x; e < mX; e += blockDim.x) sX[e] = X[e];
  __syncthreads();
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    T acc[PB];
#pragma unroll
    for (int c = 0; c < PB; ++c) acc[c] = zero<T>();
#pragma unroll 4
    for (int a = 0; a < mX; ++a) {
      const T xv = ldp<T>(sX[a].p, row * sX[a].stride);
#pragma unroll
      for (int c = 0; c < PB; ++c) acc[c] = mad(xv, sM[a * PB + c], acc[c]);
    }
    // with out_last the last of the p columns goes to its own vector
    const int po = out_last ? p - 1 : p;
#pragma unroll
    for (int c = 0; c < PB; ++c) {
      if (c < po) out[row * po + c] = acc[c];
      else if (c == po && out_last) out_last[row] = acc[c];
    }
  }
}

// out (row-major n x p) = X (row-major n x m, ONE contiguous block) M: the
// biorthogonalisation's U F, C F and the candidate's C_j N_p.
// 256-row tiles of X (contiguous 256 m values) stream into shared memory by
// cp.async, double buffered; thread = row (PB accumulators, M broadcast from
// shared memory); the tile's output (contiguous 256 p values) is staged and
// stored with 16-byte coalesced stores.  The strided-column form
// (k_gemm_panels) ran these at 3.3 TB/s (C3, 0.33 ms per 10 -> 10 GEMM).
template <typename T, int PB>
__global__ void __launch_bounds__(256) k_gemm_rm(const T *__restrict__ X, int m, const T *__restrict__ M,
                                                 int p, int64_t n, T *__restrict__ out) {
  // complex: the tile is staged TRANSPOSED ([a][row], row stride 257): the
  // row-major form put a thread's 16-byte elements 16 m bytes apart, an 8-way
  // bank conflict for m = 8 on every read (ncu: C4 8 -> 8 GEMM 96 us, 0.41 of
  // the HBM peak); the output tile likewise ([c][row])
  constexpr bool TR = sizeof(T) == 16;
  constexpr int LD = TR ? 257 : 256;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T *sM = reinterpret_cast<T *>(sm_raw);     // [m][PB]
  T *sX = sM + (size_t)m * PB;               // 2 x [256 m] (complex: 2 x [m][257])
  T *sO = sX + (size_t)2 * LD * m;           // [256 p] (complex: [p][257])
  const int tid = threadIdx.x;
  for (int e = tid; e < m * PB; e += 256) {
    const int a = e / PB, c = e % PB;
    sM[e] = c < p ? M[a * p + c] : zero<T>();
  }
  const int64_t ntiles = (n + 255) / 256;
  constexpr int PER = 16 / sizeof(T);
  auto load = [&](int64_t tile, int buf) {
    const int64_t base = tile * 256 * m;
    const int ne = (int)min((int64_t)256, n - tile * 256) * m;
    T *dst = sX + (size_t)buf * LD * m;
    for (int e = tid * PER; e < ne; e += 256 * PER) {
      const int valid = max(0, min(PER, ne - e)) * (int)sizeof(T);
      T *d = dst + e;
      if constexpr (TR) d = dst + (e % m) * LD + e / m;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(d)),
                   "l"(X + base + e), "r"(valid)
                   : "memory");
    }
    cp_async_commit();
  };
  int buf = 0;
  if ((int64_t)blockIdx.x < ntiles) load(blockIdx.x, 0);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    if (tile + gridDim.x < ntiles) load(tile + gridDim.x, buf ^ 1);
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const int rows = (int)min((int64_t)256, n - tile * 256);
    if (tid < rows) {
      const T *xr = sX + (size_t)buf * LD * m + (TR ? (size_t)tid : (size_t)tid * m);
      T acc[PB];
#pragma unroll
      for (int c = 0; c < PB; ++c) acc[c] = zero<T>();
      for (int a = 0; a < m; ++a) {
        const T xv = xr[TR ? a * LD : a];
#pragma unroll
        for (int c = 0; c < PB; ++c) acc[c] = mad(xv, sM[a * PB + c], acc[c]);
      }
#pragma unroll
      for (int c = 0; c < PB; ++c)
        if (c < p) sO[TR ? c * LD + tid : tid * p + c] = acc[c];
    }
    __syncthreads();
    const int64_t ob = tile * 256 * p;
    const int ne = rows * p;
    if constexpr (TR) {
      for (int e = tid; e < ne; e += 256) out[ob + e] = sO[(e % p) * LD + e / p];
    } else if ((ob % PER) == 0) {
      const int nv = ne / PER;
      for (int e = tid; e < nv; e += 256)
        reinterpret_cast<double2 *>(out + ob)[e] = reinterpret_cast<const double2 *>(sO)[e];
      for (int e = nv * PER + tid; e < ne; e += 256) out[ob + e] = sO[e];
    } else {
      for (int e = tid; e < ne; e += 256) out[ob + e] = sO[e];
    }
    // (the next iteration's __syncthreads orders these sO reads before its writes)
  }
}

template <typename T, int PB>
static void gemm_rm_launch(const T *X, int m, const T *dM, int p, int64_t n, T *out, rbicg_ctx *ctx,
                           cudaStream_t strm) {
  const size_t LD = sizeof(T) == 16 ? 257 : 256;   // (complex: transposed tiles, k_gemm_rm)
  const size_t sm = sizeof(T) * ((size_t)m * PB + 2 * LD * m + LD * p);
  RB_CHECK(sm <= 200 * 1024, RBICG_EINVAL);
  int per = 1;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_gemm_rm<T, PB>, 256, sm));
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((n + 255) / 256, (int64_t)std::max(1, per) * sm_budget(ctx->nsm)));
  k_gemm_rm<T, PB><<<grid, 256, sm, strm>>>(X, m, dM, p, n, out);
  RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
  count_launch();
}

template <typename T, int PB>
static void gemm_launch(const ColDesc *dX, int mX, const T *dM, int p, int64_t n, T *out,
                        T *out_last, rbicg_ctx *ctx, cudaStream_t strm) {
  const size_t sm = sizeof(T) * (size_t)mX * PB + sizeof(ColDesc) * mX;
  RB_CHECK(sm <= 200 * 1024, RBICG_EINVAL);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_budget(ctx->nsm) * 8);
  k_gemm_panels<T, PB><<<grid, 256, sm, strm>>>(dX, mX, dM, p, n, out, out_last);
  RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
  count_launch();
}

template <typename T>
void gemm_panels(const std::vector<ColDesc> &X, const std::vector<cplx> &M, int pin, int64_t n,
                 T *out, rbicg_ctx *ctx, cudaStream_t strm, bool sync, T *out_last) {
  const int mX = (int)X.size();
  const int p = pin + (out_last ? 1 : 0);   // columns of M
  if (p <= 0) return;
  RB_CHECK(p <= KMAX, RBICG_EINVAL);
  // the register-tiled multi-output GEMM (8 columns' loads in flight, two rows
  // per thread): C3 cycle-end U_j = Φ_j W_j (41 -> 10 columns) 1.27 ms at
  // 2.7 TB/s with the panel kernel below (RBICG_GEMM_PANELS_V1=1)
  static const bool v1 = getenv("RBICG_GEMM_PANELS_V1") != nullptr;
  if (!v1 && mX > 16) {   // (10 -> 10 columns: 0.33 ms here vs 0.41 ms multi-output)
    std::vector<std::pair<T *, int>> outs{{out, pin}};
    if (out_last) outs.emplace_back(out_last, 1);
    gemm_multi<T>(X, M, outs, n, ctx, strm);
    RB_CUDA(cudaStreamSynchronize(strm));
    return;
  }
  std::vector<T> hM((size_t)mX * p);
  for (size_t i = 0; i < hM.size(); ++i) {
    T v = zero<T>();
    reinterpret_cast<double *>(&v)[0] = M[i].real();
    if (sizeof(T) == 16) reinterpret_cast<double *>(&v)[1] = M[i].imag();
    hM[i] = v;
  }
  const size_t desc_bytes = sizeof(ColDesc) * std::max(mX, 1);
  const size_t m_bytes = sizeof(T) * std::max<size_t>(hM.size(), 1);
  char *buf = (char *)ws_alloc(desc_bytes + m_bytes + 32);
  ColDesc *dX = (ColDesc *)buf;
  T *dM = (T *)(buf + ((desc_bytes + 15) / 16) * 16);
  if (mX) {
    RB_CUDA(cudaMemcpyAsync(dX, X.data(), sizeof(ColDesc) * mX, cudaMemcpyHostToDevice, strm));
    RB_CUDA(cudaMemcpyAsync(dM, hM.data(), sizeof(T) * hM.size(), cudaMemcpyHostToDevice, strm));
  }
  // the columns of ONE row-major n x mX block (U, C of a basis): staged tiles
  bool rm = !out_last && mX > 0 && X[0].stride == mX && ((uintptr_t)X[0].p % 16) == 0 && !v1;
  for (int a = 1; rm && a < mX; ++a)
    rm = X[a].stride == mX && (const char *)X[a].p == (const char *)X[0].p + (size_t)a * sizeof(T);
  static const bool rm_off = getenv("RBICG_GEMM_RM") && atoi(getenv("RBICG_GEMM_RM")) == 0;
  {   // the staged form only when its tiles fit (complex k > 16: the panel kernel)
    const int PB = p <= 4 ? 4 : p <= 8 ? 8 : p <= 12 ? 12 : p <= 16 ? 16 : p <= 24 ? 24 : 32;
    const size_t LD = sizeof(T) == 16 ? 257 : 256;
    if (sizeof(T) * ((size_t)mX * PB + 2 * LD * mX + LD * p) > 200 * 1024) rm = false;
  }
  if (rm && !rm_off) {
    const T *X0 = reinterpret_cast<const T *>(X[0].p);
    if (p <= 4) gemm_rm_launch<T, 4>(X0, mX, dM, p, n, out, ctx, strm);
    else if (p <= 8) gemm_rm_launch<T, 8>(X0, mX, dM, p, n, out, ctx, strm);
    else if (p <= 12) gemm_rm_launch<T, 12>(X0, mX, dM, p, n, out, ctx, strm);
    else if (p <= 16) gemm_rm_launch<T, 16>(X0, mX, dM, p, n, out, ctx, strm);
    else if (p <= 24) gemm_rm_launch<T, 24>(X0, mX, dM, p, n, out, ctx, strm);
    else gemm_rm_launch<T, 32>(X0, mX, dM, p, n, out, ctx, strm);
  } else if (p <= 4) gemm_launch<T, 4>(dX, mX, dM, p, n, out, out_last, ctx, strm);
  else if (p <= 8) gemm_launch<T, 8>(dX, mX, dM, p, n, out, out_last, ctx, strm);
  else if (p <= 12) gemm_launch<T, 12>(dX, mX, dM, p, n, out, out_last, ctx, strm);
  else if (p <= 16) gemm_launch<T, 16>(dX, mX, dM, p, n, out, out_last, ctx, strm);
  else if (p <= 24) gemm_launch<T, 24>(dX, mX, dM, p, n, out, out_last, ctx, strm);
  else gemm_launch<T, 32>(dX, mX, dM, p, n, out, out_last, ctx, strm);
  // the pinned-free staging below is host memory: synchronous copies above
  // completed before return only if we sync; otherwise keep hM alive by
  // syncing lazily through the stream-ordered free below
  if (sync) {
    RB_CUDA(cudaStreamSynchronize(strm));
    ws_free(buf);
  } else {
    RB_CUDA(cudaStreamSynchronize(strm));   // hM (pageable) must outlive its copy
    ws_free(buf);
  }
}

// Several outputs from one pass over the panel columns: output segment q takes
// columns [c0_q, c0_q + nc_q) of X M into its own row-major n x nc_q array
// (U_j, C_j and the lazy-x flush of a cycle end, api.cu).
struct OutSegs {
  void *p[4];
  int nc[4];
  int ns;
};
// Two rows per thread (rows q*256 + tid of a 512-row tile, coalesced per
// column) so each shared-memory read of M feeds two FMAs, and M is read in
// 16-byte pairs: the broadcast LDS, not the FMAs or HBM, bounded the
// one-row-per-thread form (281 us for 44 -> 21 columns at n = 1M).
template <typename T> struct MPair { T a, b; };
template <typename T, int PB, int RX>
constexpr int gm_rpt() { return RX ? RX : ((sizeof(T) == 8 && PB <= 24) ? 2 : 1); }
template <typename T, int PB, int RX>
constexpr int gm_minb() { return sizeof(T) == 8 && gm_rpt<T, PB, RX>() == 1 && PB <= 12 ? 4 : 2; }   // (complex at 3 blocks/SM: C4 282 -> 312 us, stack frame)
template <typename T, int PB, int RX = 0>
__global__ void __launch_bounds__(256, (gm_minb<T, PB, RX>())) k_gemm_multi(const ColDesc *__restrict__ X, int mX,
                                                       const T *__restrict__ M, int p, int64_t n,
                                                       OutSegs O) {
  constexpr int RPT = gm_rpt<T, PB, RX>();   // rows per thread (registers; complex: 1)
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T *sM = reinterpret_cast<T *>(sm_raw);   // [mX][PB], zero padded (PB even)
  ColDesc *sX = reinterpret_cast<ColDesc *>(sM + (size_t)mX * PB);
  for (int e = threadIdx.x; e < mX * PB; e += blockDim.x) {
    const int a = e / PB, c = e % PB;
    sM[e] = c < p ? M[a * p + c] : zero<T>();
  }
  for (int e = threadIdx.x; e < mX; e += blockDim.x) sX[e] = X[e];
  __syncthreads();
  const int64_t ntiles = (n + 256 * RPT - 1) / (256 * RPT);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int64_t row[RPT];
    bool ok[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      row[q] = tile * 256 * RPT + q * 256 + threadIdx.x;
      ok[q] = row[q] < n;
    }
    T acc[RPT][PB];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
      for (int c = 0; c < PB; ++c) acc[q][c] = zero<T>();
    // AU columns' loads are issued before their FMAs: AU x RPT loads per
    // thread in flight (the kernel is bound by HBM latency x bytes in flight)
    constexpr int AU = PB <= 12 ? 8 : 4;   // (PB 24 with 1 row and 8 ahead: C5 12.4 vs 11.3 ms)
    int a = 0;
    for (; a + AU <= mX; a += AU) {
      T xv[AU][RPT];
#pragma unroll
      for (int u = 0; u < AU; ++u)
#pragma unroll
        for (int q = 0; q < RPT; ++q)
          xv[u][q] = ok[q] ? ldp<T>(sX[a + u].p, row[q] * sX[a + u].stride) : zero<T>();
#pragma unroll
      for (int u = 0; u < AU; ++u) {
        const MPair<T> *mp = reinterpret_cast<const MPair<T> *>(sM + (a + u) * PB);
#pragma unroll
        for (int c2 = 0; c2 < PB / 2; ++c2) {
          const MPair<T> m = mp[c2];
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            acc[q][2 * c2] = mad(xv[u][q], m.a, acc[q][2 * c2]);
            acc[q][2 * c2 + 1] = mad(xv[u][q], m.b, acc[q][2 * c2 + 1]);
          }
        }
      }
    }
    for (; a < mX; ++a) {
      T xv[RPT];
#pragma unroll
      for (int q = 0; q < RPT; ++q) xv[q] = ok[q] ? ldp<T>(sX[a].p, row[q] * sX[a].stride) : zero<T>();
      const MPair<T> *mp = reinterpret_cast<const MPair<T> *>(sM + a * PB);
#pragma unroll
      for (int c2 = 0; c2 < PB / 2; ++c2) {
        const MPair<T> m = mp[c2];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          acc[q][2 * c2] = mad(xv[q], m.a, acc[q][2 * c2]);
          acc[q][2 * c2 + 1] = mad(xv[q], m.b, acc[q][2 * c2 + 1]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      if (!ok[q]) continue;
      int c0 = 0;
      for (int sg = 0; sg < O.ns; ++sg) {
        T *out = reinterpret_cast<T *>(O.p[sg]);
        const int nc = O.nc[sg];
#pragma unroll
        for (int c = 0; c < PB; ++c)
          if (c >= c0 && c < c0 + nc) out[row[q] * nc + (c - c0)] = acc[q][c];
        c0 += nc;
      }
    }
  }
}

// TMA-staged form for unit-stride, 16-byte aligned columns (the Lanczos ring
// columns, the direction segment and x of the relation GEMM): one persistent
// CTA per SM, 128 threads, 256-row tiles (two rows per thread for real,
// 128-row tiles for complex); a tile's mX column segments land in shared
// memory by 1-D bulk copies (cp.async.bulk + mbarrier), double buffered, so
// HBM requests stay in flight while the FMAs of the previous tile run.  The
// ragged last tile is filled by ordinary loads.
template <typename T>
void gemm_multi(const std::vector<ColDesc> &X, const std::vector<cplx> &M,
                const std::vector<std::pair<T *, int>> &outs, int64_t n, rbicg_ctx *ctx,
                cudaStream_t strm) {
  const int mX = (int)X.size();
  int p = 0;
  OutSegs O{};
  RB_CHECK(outs.size() <= 4, RBICG_EINVAL);
  for (size_t q = 0; q < outs.size(); ++q) {
    O.p[q] = outs[q].first;
    O.nc[q] = outs[q].second;
    p += outs[q].second;
  }
  O.ns = (int)outs.size();
  if (p <= 0 || mX == 0) return;
  RB_CHECK((int)M.size() == mX * p, RBICG_EINVAL);
  if (p > 32) {
    // wider than one launch's register tile: split the output segments into
    // groups of <= 32 columns, one launch per group (X is read once per group)
    size_t q0 = 0;
    int c0 = 0;
    while (q0 < outs.size()) {
      size_t q1 = q0;
      int w = 0;
      while (q1 < outs.size() && w + outs[q1].second <= 32) w += outs[q1++].second;
      RB_CHECK(q1 > q0, RBICG_EINVAL);   // one segment wider than 32
      std::vector<cplx> Mg((size_t)mX * w);
      for (int a = 0; a < mX; ++a)
        for (int c = 0; c < w; ++c) Mg[(size_t)a * w + c] = M[(size_t)a * p + c0 + c];
      gemm_multi<T>(X, Mg, std::vector<std::pair<T *, int>>(outs.begin() + q0, outs.begin() + q1),
                    n, ctx, strm);
      q0 = q1;
      c0 += w;
    }
    return;
  }
  std::vector<T> hM((size_t)mX * p);
  for (size_t i = 0; i < hM.size(); ++i) {
    T v = zero<T>();
    reinterpret_cast<double *>(&v)[0] = M[i].real();
    if (sizeof(T) == 16) reinterpret_cast<double *>(&v)[1] = M[i].imag();
    hM[i] = v;
  }
  const size_t desc_bytes = sizeof(ColDesc) * mX;
  char *buf = (char *)ws_alloc(desc_bytes + sizeof(T) * hM.size() + 32);
  ColDesc *dX = (ColDesc *)buf;
  T *dM = (T *)(buf + ((desc_bytes + 15) / 16) * 16);
  RB_CUDA(cudaMemcpyAsync(dX, X.data(), desc_bytes, cudaMemcpyHostToDevice, strm));
  RB_CUDA(cudaMemcpyAsync(dM, hM.data(), sizeof(T) * hM.size(), cudaMemcpyHostToDevice, strm));
  auto go = [&](auto kern, int PB, int rpt) {
    const size_t sm = sizeof(T) * (size_t)mX * PB + sizeof(ColDesc) * mX;
    RB_CHECK(sm <= 200 * 1024, RBICG_EINVAL);
    int per = 1;
    RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, sm));
    const int rows_per_block = 256 * rpt;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((n + rows_per_block - 1) / rows_per_block, (int64_t)std::max(1, per) * sm_budget(ctx->nsm)));
    kern<<<grid, 256, sm, strm>>>(dX, mX, dM, p, n, O);
    RB_CUDA(cudaGetLastError());   // a launch that could not start (config) fails here
  };
  static const int rx = getenv("RBICG_GEMM_RPT") ? atoi(getenv("RBICG_GEMM_RPT")) : 0;
  const int r2 = sizeof(T) == 8 ? 2 : 1;
  if (p <= 12) {
    if (rx == 1) go(k_gemm_multi<T, 12, 1>, 12, 1);
    else go(k_gemm_multi<T, 12>, 12, r2);
  } else if (p <= 24) {
    go(k_gemm_multi<T, 24>, 24, r2);
  } else {
    go(k_gemm_multi<T, 32>, 32, 1);
  }
  count_launch();
  RB_CUDA(cudaStreamSynchronize(strm));   // hM (pageable) must outlive its copy
  ws_free(buf);
}

void prepare_block_kernels() {
  RB_CUDA(cudaFuncSetAttribute(k_gram_cc<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  RB_CUDA(cudaFuncSetAttribute(k_gram_cc<zc>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  RB_CUDA(cudaFuncSetAttribute(k_spmm<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  RB_CUDA(cudaFuncSetAttribute(k_spmm<zc>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
#define RB_SATTR(T, KB)                                                                      \
  RB_CUDA(cudaFuncSetAttribute(k_gemm_rm<T, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               200 * 1024));
  RB_SATTR(double, 4) RB_SATTR(double, 8) RB_SATTR(double, 12) RB_SATTR(double, 16)
  RB_SATTR(double, 24) RB_SATTR(double, 32)
  RB_SATTR(zc, 4) RB_SATTR(zc, 8) RB_SATTR(zc, 12) RB_SATTR(zc, 16) RB_SATTR(zc, 24)
  RB_SATTR(zc, 32)
#undef RB_SATTR
#define RB_GATTR(T, PB)                                                                      \
  RB_CUDA(cudaFuncSetAttribute(k_gemm_panels<T, PB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               200 * 1024));
  RB_GATTR(double, 4) RB_GATTR(double, 8) RB_GATTR(double, 12) RB_GATTR(double, 16)
  RB_GATTR(double, 24) RB_GATTR(double, 32)
  RB_GATTR(zc, 4) RB_GATTR(zc, 8) RB_GATTR(zc, 12) RB_GATTR(zc, 16) RB_GATTR(zc, 24)
  RB_GATTR(zc, 32)
#undef RB_GATTR
  // every Gram / SpMM instantiation the cycle end can pick, loaded and given
  // its shared-memory limit here: under lazy module loading a first launch in
  // the middle of a sequence loads the kernel then (measured: C4 systems that
  // met a new pencil shape took 37-110 ms instead of 11-21 ms)
#define RB_G2(R, C) (const void *)k_gram_mma2<double, R, C, 32, 2>,
  for (auto f : {RB_G2(2, 1) RB_G2(4, 1) RB_G2(7, 1) RB_G2(8, 1) RB_G2(10, 2) RB_G2(2, 2) RB_G2(3, 2)
                     RB_G2(4, 2) RB_G2(4, 3) RB_G2(5, 2) RB_G2(5, 3) RB_G2(5, 4) RB_G2(2, 3) RB_G2(2, 4)
                         RB_G2(2, 5) RB_G2(3, 4) RB_G2(3, 6) RB_G2(3, 8)(const void *)k_gram_mma<double, 2, 32, 2>,
                 (const void *)k_gram_mma<double, 4, 32, 2>, (const void *)k_gram_mma<double, 6, 32, 2>,
                 (const void *)k_gram_mma<double, 7, 32, 2>, (const void *)k_gram_mma<double, 8, 32, 2>,
                 (const void *)k_gram_mma<double, 9, 32, 2>, (const void *)k_gram_mma<double, 10, 32, 2>,
                 (const void *)k_gram_mma<double, 12, 32, 2>, (const void *)k_gram_mma<double, 14, 32, 2>,
                 (const void *)k_gram_mma<double, 16, 32, 2>, (const void *)k_gram_mma<double, 20, 32, 2>,
                 (const void *)k_gram_mma<zc, 2, 32, 2>, (const void *)k_gram_mma<zc, 4, 32, 2>,
                 (const void *)k_gram_mma<zc, 6, 32, 2>, (const void *)k_gram_mma<zc, 8, 32, 2>,
                 (const void *)k_gram_cc_mma<1>, (const void *)k_gram_cc_mma<2>, (const void *)k_gram_cc_mma<3>,
                 (const void *)k_gram_cc_mma<4>, (const void *)k_gram2<double, 8, 8>,
                 (const void *)k_gram2<double, 4, 8>, (const void *)k_gram2<double, 4, 4>,
                 (const void *)k_gram2<zc, 4, 4>})
    RB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
#undef RB_G2
#define RB_SP(T, KB)                                                                                   (const void *)k_spmm_rows<T, KB>, (const void *)k_spmm_rows<T, KB, 2>, (const void *)k_spmm_rows<T, KB, 3>,       (const void *)k_spmm_rows<T, KB, 4>, (const void *)k_spmm_rows0<T, KB>,
  for (auto f : {RB_SP(double, 4) RB_SP(double, 8) RB_SP(double, 12) RB_SP(double, 16) RB_SP(double, 24)
                     RB_SP(double, 32)(const void *)k_spmm_wide<double>, (const void *)k_spmm_wide<zc>}) {
    cudaFuncAttributes fa;
    RB_CUDA(cudaFuncGetAttributes(&fa, f));
  }
#undef RB_SP
  for (auto f : {(const void *)k_gemm_multi<double, 12>, (const void *)k_gemm_multi<double, 24>,
                 (const void *)k_gemm_multi<double, 32>, (const void *)k_gemm_multi<zc, 12>,
                 (const void *)k_gemm_multi<zc, 24>, (const void *)k_gemm_multi<zc, 32>,
                 (const void *)k_gemm_multi<double, 12, 1>, (const void *)k_gemm_multi<zc, 12, 1>})
    RB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
}

#define RB_BINST(T)                                                                        \
  template void gram_cc<T>(const T *, const T *, int, int64_t, std::vector<cplx> &, rbicg_ctx *, \
                           cudaStream_t);                                                     \
  template void launch_spmm<T>(const DevMat &, const T *, T *, int, cudaStream_t);         \
  template void gram<T>(const std::vector<ColDesc> &, const std::vector<ColDesc> &, int64_t, \
                        std::vector<cplx> &, rbicg_ctx *, cudaStream_t);                   \
  template void gemm_panels<T>(const std::vector<ColDesc> &, const std::vector<cplx> &, int, \
                               int64_t, T *, rbicg_ctx *, cudaStream_t, bool, T *);       \
  template void gemm_multi<T>(const std::vector<ColDesc> &, const std::vector<cplx> &,       \
                              const std::vector<std::pair<T *, int>> &, int64_t, rbicg_ctx *, \
                              cudaStream_t);
RB_BINST(double)
RB_BINST(zc)

}  // namespace rbicg
