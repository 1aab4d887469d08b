// kernels.cu -- the RBiCG hot loop on sm_100a (Algorithm 2).
//
// One iteration = two persistent streaming kernels, each ending in a
// deterministic grid reduction done by the last block to finish:
//
//   pass 1  p_i = r_{i-1} + β_{i-1} p_{i-1},  p~_i = r~_{i-1} + β̄ p~_{i-1}
//           z_i = A p_i,  z~_i = A^* p~_i          (SELL-32 SpMV pair, the
//           direction update fused into the gather)
//           partial sums of C~^*z, C^*z~, C^*p~, p~^*z  (oblique-projection
//           coefficients; σ_i via reading Q23)
//           last block: ζ = D_c^{-1}C~^*z, ζ~ = D_c^{-1}C^*z~,
//                       σ = p~^*z - (C^*p~)^*ζ, α = ρ/σ, ζ_c += αζ, ...
//   pass 2  q = z - Cζ, q~ = z~ - C~ζ~; x += αp; x~ += ᾱp~;
//           r_i = r_{i-1} - αq (written straight into the Lanczos ring
//           column i), r~_i likewise; partial ρ_i, ||r||², ||r~||²
//           last block: β_i = ρ_i/ρ_{i-1}, stop test (Q2), breakdown (Q3),
//           iteration record for the cycle-end control.
//
// Kernels read the iteration index from the device state, so one captured
// CUDA graph of s iterations is replayed for every cycle; once the state says
// done/paused every kernel is a no-op (exact iteration counts, no host poll).
#include "internal.h"
#include <cstdlib>

namespace rbicg {

std::atomic<int64_t> g_launches{0};
static const bool g_pdl = getenv("RBICG_PDL") != nullptr;   // measured: no gain

template <typename T> __device__ __forceinline__ T ldg(const T *p);
template <> __device__ __forceinline__ double ldg<double>(const double *p) { return __ldg(p); }
template <> __device__ __forceinline__ zc ldg<zc>(const zc *p) {
  double2 v = __ldg(reinterpret_cast<const double2 *>(p));
  return mk(v.x, v.y);
}
// streaming (evict-first) loads for data touched once per pass
template <typename T> __device__ __forceinline__ T ldcs(const T *p);
template <> __device__ __forceinline__ double ldcs<double>(const double *p) { return __ldcs(p); }
template <> __device__ __forceinline__ zc ldcs<zc>(const zc *p) {
  double2 v = __ldcs(reinterpret_cast<const double2 *>(p));
  return mk(v.x, v.y);
}


// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: the next kernel of the loop is launched while
// this one drains; it may run its independent prologue (TMA of matrix tiles)
// and then waits here for the full completion of its predecessor.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- TMA / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion via mbarrier tx count
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra "
      "WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// y_row = Σ_j a_{row,j} (r_j + β p_j)   (FUSE)   or   Σ_j a_{row,j} p_j
template <typename T, bool FUSE>
__device__ __forceinline__ T sell_row(const DevMat &M, int64_t row, const T *__restrict__ r,
                                      const T *__restrict__ p, T beta) {
  const int64_t sl = row >> 5;
  const int lane = (int)(row & 31);
  const int64_t off = M.sptr[sl];
  const int w = (int)((M.sptr[sl + 1] - off) >> 5);
  const int32_t *__restrict__ cols = M.cols + off + lane;
  const T *__restrict__ vals = reinterpret_cast<const T *>(M.vals) + off + lane;
  T acc = zero<T>();
#pragma unroll 4
  for (int jj = 0; jj < w; ++jj) {
    const int c = __ldcs(cols + jj * 32);
    const T v = ldcs(vals + jj * 32);
    T pj;
    if (FUSE) pj = mad(beta, ldg(p + c), ldg(r + c));
    else pj = ldg(p + c);
    acc = mad(v, pj, acc);
  }
  return acc;
}


// One row of the SpMV pair from TMA-staged SELL tiles (column-major slices in
// shared memory).  Both matrices' gathers are issued together in chunks of 4
// so up to 16 independent loads per thread are in flight.
template <typename T>
__device__ __forceinline__ void sell_pair_smem(const int32_t *__restrict__ cA, const T *__restrict__ vA,
                                               int wA, const int32_t *__restrict__ cH,
                                               const T *__restrict__ vH, int wH,
                                               const T *__restrict__ r, const T *__restrict__ p,
                                               const T *__restrict__ rt, const T *__restrict__ pt,
                                               T beta, T cb, T &z, T &zt) {
  z = zero<T>();
  zt = zero<T>();
  const int wm = max(wA, wH);
  for (int j0 = 0; j0 < wm; j0 += 4) {
    int ca[4], ch[4];
    T va[4], vh[4], ra[4], pa[4], rh[4], ph[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int jj = j0 + q;
      const bool ia = jj < wA, ih = jj < wH;
      ca[q] = ia ? cA[jj * 32] : 0;
      va[q] = ia ? vA[jj * 32] : zero<T>();
      ch[q] = ih ? cH[jj * 32] : 0;
      vh[q] = ih ? vH[jj * 32] : zero<T>();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ra[q] = ldg(r + ca[q]);
      pa[q] = ldg(p + ca[q]);
      rh[q] = ldg(rt + ch[q]);
      ph[q] = ldg(pt + ch[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      z = mad(va[q], mad(beta, pa[q], ra[q]), z);
      zt = mad(vh[q], mad(cb, ph[q], rh[q]), zt);
    }
  }
}

// Deterministic block sum (fixed shuffle tree + fixed warp order). Valid in
// thread 0.  sbuf needs BS/32 entries.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T *sbuf) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sbuf[w] = v;
  __syncthreads();
  T r = zero<T>();
  if (threadIdx.x == 0)
    for (int i = 0; i < BS / 32; ++i) r = add(r, sbuf[i]);
  return r;
}

// Last-block election; returns true in every thread of the last block.
__device__ __forceinline__ bool last_block(unsigned *cnt, int *s_flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned v = atomicAdd(cnt, 1u);
    *s_flag = (v == gridDim.x - 1);
  }
  __syncthreads();
  return *s_flag != 0;
}

// Final fixed-order reduction of `nout` outputs stored as part[o*G + b].
// All partial loads of a lane are issued before any add (they are L2 hits;
// a dependent chain of G/32 loads would cost microseconds at the kernel tail).
constexpr int RED_PER_LANE = 40;   // supports G <= 1280 blocks
template <typename T>
__device__ __forceinline__ void final_reduce(const T *part, int nout, int G, T *s_fin) {
  __threadfence();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int o = w; o < nout; o += BS / 32) {
    const T *src = part + (int64_t)o * G;
    T v[RED_PER_LANE];
#pragma unroll
    for (int q = 0; q < RED_PER_LANE; ++q) {
      const int b = l + 32 * q;
      v[q] = b < G ? ldcg(src + b) : zero<T>();
    }
    T acc = zero<T>();
#pragma unroll
    for (int q = 0; q < RED_PER_LANE; ++q) acc = add(acc, v[q]);
    acc = warp_sum(acc);
    if (l == 0) s_fin[o] = acc;
  }
  __syncthreads();
}

// ============================================================== pass 1
template <typename T>
__global__ void __launch_bounds__(BS, 4) k_pass1(LoopArgs<T> a) {
  __shared__ T s_z[BS], s_zt[BS], s_pt[BS];
  __shared__ T s_red[3 * BS];
  __shared__ T s_fin[3 * KMAX + 1];
  __shared__ T s_w[BS / 32];
  __shared__ int s_last;
  DevState<T> *st = a.st;
  const int tid = threadIdx.x;
  const int64_t n = a.n;
  const int64_t ntiles = (n + BS - 1) / BS;
  // TMA staging of the SELL tiles of A and A^* (one tile = 8 slices = BS rows)
  extern __shared__ __align__(128) unsigned char p1_smem[];
  __shared__ uint64_t bar;
  const int TM = a.tile_max;   // elements per tile per matrix (multiple of 32)
  int32_t *scA = reinterpret_cast<int32_t *>(p1_smem);
  int32_t *scH = scA + TM;
  T *svA = reinterpret_cast<T *>(scH + TM);
  T *svH = svA + TM;
  const int64_t ns = a.A.nslices;
  auto issue = [&](int64_t t) {
    const int64_t s0 = t * (BS / 32), s1 = min(s0 + BS / 32, ns);
    const int64_t oA = a.A.sptr[s0], eA = a.A.sptr[s1];
    const int64_t oH = a.AH.sptr[s0], eH = a.AH.sptr[s1];
    const uint32_t nA = (uint32_t)(eA - oA), nH = (uint32_t)(eH - oH);
    mbar_expect_tx(&bar, (nA + nH) * (4u + (uint32_t)sizeof(T)));
    if (nA) {
      tma_load_1d(scA, a.A.cols + oA, nA * 4u, &bar);
      tma_load_1d(svA, reinterpret_cast<const T *>(a.A.vals) + oA, nA * (uint32_t)sizeof(T), &bar);
    }
    if (nH) {
      tma_load_1d(scH, a.AH.cols + oH, nH * 4u, &bar);
      tma_load_1d(svH, reinterpret_cast<const T *>(a.AH.vals) + oH, nH * (uint32_t)sizeof(T), &bar);
    }
  };
  // prologue independent of the previous kernel: first matrix tile
  if (a.staged) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0 && (int64_t)blockIdx.x < ntiles) issue(blockIdx.x);
  }
  pdl_wait();
  if (st->done) {
    if (a.staged && (int64_t)blockIdx.x < ntiles) mbar_wait(&bar, 0);   // drain the copy
    return;
  }
  const int it = st->iter;
  const bool segcopy = a.lazy_x && it == st->seg_start;
  const T beta = st->beta;
  const T cb = conj(beta);
  const T *__restrict__ r = a.rring + (int64_t)(it % a.ring) * n;
  const T *__restrict__ rt = a.rtring + (int64_t)(it % a.ring) * n;
  const T *__restrict__ pold = a.p[it & 1];
  const T *__restrict__ ptold = a.pt[it & 1];
  T *__restrict__ pnew = a.p[(it + 1) & 1];
  T *__restrict__ ptnew = a.pt[(it + 1) & 1];
  const int k = a.k;
  const int rstep = k > 0 ? BS / k : 0;
  const int kt = rstep * k;
  T a1 = zero<T>(), a2 = zero<T>(), a3 = zero<T>(), aptz = zero<T>();
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * BS;
    const int rows = (int)min((int64_t)BS, n - row0);
    if (a.staged) {
      // slice geometry (global loads overlap the bulk copy)
      const int64_t sl = (row0 >> 5) + (tid >> 5);
      const int64_t slc = min(sl, ns - 1);
      const int64_t bA = a.A.sptr[tile * (BS / 32)], bH = a.AH.sptr[tile * (BS / 32)];
      const int64_t oA = a.A.sptr[slc], oH = a.AH.sptr[slc];
      const int wA = (int)((a.A.sptr[slc + 1] - oA) >> 5), wH = (int)((a.AH.sptr[slc + 1] - oH) >> 5);
      const int lane = tid & 31;
      mbar_wait(&bar, phase);
      phase ^= 1u;
      if (tid < rows) {
        const int64_t row = row0 + tid;
        T z, zt;
        sell_pair_smem<T>(scA + (oA - bA) + lane, svA + (oA - bA) + lane, wA,
                          scH + (oH - bH) + lane, svH + (oH - bH) + lane, wH, r, pold, rt, ptold,
                          beta, cb, z, zt);
        const T po = ldg(pold + row), pto = ldg(ptold + row);
        const T pn = mad(beta, po, ldg(r + row));
        const T ptn = mad(cb, pto, ldg(rt + row));
        if (segcopy) {   // lazy x: keep p_a, p~_a of the new segment
          a.pseg[row] = po;
          a.ptseg[row] = pto;
        }
        pnew[row] = pn;
        ptnew[row] = ptn;
        a.z[row] = z;
        a.zt[row] = zt;
        aptz = cmad(ptn, z, aptz);
        s_z[tid] = z;
        s_zt[tid] = zt;
        s_pt[tid] = ptn;
      }
      __syncthreads();   // staged tile consumed -> refill
      if (tid == 0 && tile + gridDim.x < ntiles) issue(tile + gridDim.x);
    } else if (tid < rows) {
      const int64_t row = row0 + tid;
      const T z = sell_row<T, true>(a.A, row, r, pold, beta);
      const T zt = sell_row<T, true>(a.AH, row, rt, ptold, cb);
      const T po = ldg(pold + row), pto = ldg(ptold + row);
      const T pn = mad(beta, po, ldg(r + row));
      const T ptn = mad(cb, pto, ldg(rt + row));
      if (segcopy) {
        a.pseg[row] = po;
        a.ptseg[row] = pto;
      }
      pnew[row] = pn;
      ptnew[row] = ptn;
      a.z[row] = z;
      a.zt[row] = zt;
      aptz = cmad(ptn, z, aptz);
      s_z[tid] = z;
      s_zt[tid] = zt;
      s_pt[tid] = ptn;
    }
    if (k > 0) {
      __syncthreads();
      if (tid < kt) {
        // thread tid always meets column tid % k because kt is a multiple of k
        const int nel = rows * k;
        const T *__restrict__ Ct = a.Ct + row0 * k;
        const T *__restrict__ C = a.C + row0 * k;
        int lr = tid / k;
        for (int e = tid; e < nel; e += kt, lr += rstep) {
          const T ct = ldcs(Ct + e), c = ldcs(C + e);
          a1 = cmad(ct, s_z[lr], a1);   // conj(c~_{row,j}) z_row
          a2 = cmad(c, s_zt[lr], a2);   // conj(c_{row,j}) z~_row
          a3 = cmad(c, s_pt[lr], a3);   // conj(c_{row,j}) p~_row
        }
      }
      __syncthreads();
    }
  }
  pdl_trigger();
  // ---- block reduction, fixed order
  const int G = gridDim.x;
  const int nout = 3 * k + 1;
  if (k > 0) {
    s_red[tid] = tid < kt ? a1 : zero<T>();
    s_red[BS + tid] = tid < kt ? a2 : zero<T>();
    s_red[2 * BS + tid] = tid < kt ? a3 : zero<T>();
  }
  const T bptz = block_sum(aptz, s_w);   // contains __syncthreads
  if (tid < 3 * k) {
    const int ty = tid / k, j = tid % k;
    T s = zero<T>();
    for (int m = 0; m < rstep; ++m) s = add(s, s_red[ty * BS + j + m * k]);
    a.part[(int64_t)tid * G + blockIdx.x] = s;
  }
  if (tid == 0) a.part[(int64_t)(3 * k) * G + blockIdx.x] = bptz;
  if (!last_block(&st->cnt[0], &s_last)) return;
  final_reduce(a.part, nout, G, s_fin);
  if (tid == 0) {
    st->cnt[0] = 0;
    const int i = it + 1;
    T sigma = s_fin[3 * k];
    for (int j = 0; j < k; ++j) {
      const T zj = scal(st->dinv[j], s_fin[j]);   // ζ_i = D_c^{-1} C~^* z_i
      s_fin[j] = zj;
      s_fin[k + j] = scal(st->dinv[j], s_fin[k + j]);   // ζ~_i = D_c^{-1} C^* z~_i
      sigma = sub(sigma, cmul(s_fin[2 * k + j], zj));   // (p~, z - Cζ)  (Q23)
    }
    const T alpha = divd(st->rho, sigma);
    if (iszero(sigma) || !finite(alpha)) {   // breakdown of the second kind
      st->status = RBICG_BREAKDOWN_SECOND;
      st->done = 1;
      return;
    }
    st->alpha = alpha;
    st->sigma = sigma;
    const T ca = conj(alpha);
    for (int j = 0; j < k; ++j) {
      const T zj = s_fin[j], ztj = s_fin[k + j];
      st->zeta[j] = zj;
      st->zetat[j] = ztj;
      st->zc[j] = mad(alpha, zj, st->zc[j]);
      st->ztc[j] = mad(ca, ztj, st->ztc[j]);
      a.zhist[(int64_t)i * k + j] = zj;
      a.zthist[(int64_t)i * k + j] = ztj;
    }
  }
}

// ============================================================== pass 2
template <typename T>
__global__ void __launch_bounds__(BS, 3) k_pass2(LoopArgs<T> a, int staged) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ T s_zeta[KMAX], s_zetat[KMAX];
  __shared__ T s_w[BS / 32];
  __shared__ T s_fin[3];
  __shared__ int s_last;
  DevState<T> *st = a.st;
  pdl_wait();
  if (st->done) return;
  const int tid = threadIdx.x;
  const int it = st->iter;
  const int k = a.k;
  const T alpha = st->alpha;
  const T ca = conj(alpha);
  if (tid < k) {
    s_zeta[tid] = st->zeta[tid];
    s_zetat[tid] = st->zetat[tid];
  }
  __syncthreads();
  const int64_t n = a.n;
  const T *__restrict__ rold = a.rring + (int64_t)(it % a.ring) * n;
  const T *__restrict__ rtold = a.rtring + (int64_t)(it % a.ring) * n;
  T *__restrict__ rnew = a.rring + (int64_t)((it + 1) % a.ring) * n;
  T *__restrict__ rtnew = a.rtring + (int64_t)((it + 1) % a.ring) * n;
  const T *__restrict__ pn = a.p[(it + 1) & 1];
  const T *__restrict__ ptn = a.pt[(it + 1) & 1];
  T arho = zero<T>();
  double an = 0.0, ant = 0.0;
  const int64_t ntiles = (n + BS - 1) / BS;
  const int64_t nfull = n / BS;
  const bool lazy = a.lazy_x != 0;
  // row update shared by the staged and the direct path
  auto update_row = [&](int64_t row, T q, T qt, T ro, T rto, T pv, T ptv, T xv, T xtv,
                        const T *cr, const T *ctr) {
    if (k > 0) {
      T d = zero<T>(), dt = zero<T>();
      for (int j = 0; j < k; ++j) {
        d = mad(cr[j], s_zeta[j], d);
        dt = mad(ctr[j], s_zetat[j], dt);
      }
      q = sub(q, d);     // q_i = z_i - C ζ_i
      qt = sub(qt, dt);  // q~_i = z~_i - C~ ζ~_i
    }
    const T rn = sub(ro, mul(alpha, q));
    const T rtn = sub(rto, mul(ca, qt));
    if (!lazy) {
      a.x[row] = mad(alpha, pv, xv);
      a.xt[row] = mad(ca, ptv, xtv);
    }
    rnew[row] = rn;
    rtnew[row] = rtn;
    arho = cmad(rtn, rn, arho);
    an += abs2(rn);
    ant += abs2(rtn);
  };
  if (staged) {
    // TMA double buffering: each full 256-row tile of the ten input streams
    // (z, z~, r, r~, p, p~, x, x~ and the C, C~ tiles) is bulk-copied into
    // shared memory while the previous tile is being processed.
    __shared__ uint64_t bars[2];
    const int64_t stage = (int64_t)8 * BS + (int64_t)2 * BS * k;
    T *sb = reinterpret_cast<T *>(smem_raw);
    auto issue = [&](int64_t t, int si) {
      T *b = sb + si * stage;
      const int64_t r0 = t * BS;
      const uint32_t vb = BS * (uint32_t)sizeof(T);
      const uint32_t cb = (uint32_t)(BS * k * sizeof(T));
      mbar_expect_tx(&bars[si], (lazy ? 4u : 8u) * vb + 2u * cb);
      tma_load_1d(b + 0 * BS, a.z + r0, vb, &bars[si]);
      tma_load_1d(b + 1 * BS, a.zt + r0, vb, &bars[si]);
      tma_load_1d(b + 2 * BS, rold + r0, vb, &bars[si]);
      tma_load_1d(b + 3 * BS, rtold + r0, vb, &bars[si]);
      if (!lazy) {
        tma_load_1d(b + 4 * BS, pn + r0, vb, &bars[si]);
        tma_load_1d(b + 5 * BS, ptn + r0, vb, &bars[si]);
        tma_load_1d(b + 6 * BS, a.x + r0, vb, &bars[si]);
        tma_load_1d(b + 7 * BS, a.xt + r0, vb, &bars[si]);
      }
      if (k > 0) {
        tma_load_1d(b + 8 * BS, a.C + r0 * k, cb, &bars[si]);
        tma_load_1d(b + 8 * BS + BS * k, a.Ct + r0 * k, cb, &bars[si]);
      }
    };
    if (tid == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0 && (int64_t)blockIdx.x < nfull) issue(blockIdx.x, 0);
    uint32_t ph[2] = {0u, 0u};
    int i = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
      const int si = i & 1;
      const int64_t nxt = tile + gridDim.x;
      if (tid == 0 && nxt < nfull) issue(nxt, si ^ 1);
      const int64_t row0 = tile * BS;
      if (tile < nfull) {
        mbar_wait(&bars[si], ph[si]);
        ph[si] ^= 1u;
        const T *b = sb + si * stage;
        update_row(row0 + tid, b[tid], b[BS + tid], b[2 * BS + tid], b[3 * BS + tid],
                   b[4 * BS + tid], b[5 * BS + tid], b[6 * BS + tid], b[7 * BS + tid],
                   b + 8 * BS + tid * k, b + 8 * BS + BS * k + tid * k);
      } else if (tid < (int)(n - row0)) {
        const int64_t row = row0 + tid;
        update_row(row, a.z[row], a.zt[row], rold[row], rtold[row],
                   lazy ? zero<T>() : pn[row], lazy ? zero<T>() : ptn[row],
                   lazy ? zero<T>() : a.x[row], lazy ? zero<T>() : a.xt[row], a.C + row * k,
                   a.Ct + row * k);
      }
      __syncthreads();   // stage si consumed before it is refilled
    }
  } else {
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t row0 = tile * BS;
      const int rows = (int)min((int64_t)BS, n - row0);
      if (tid < rows) {
        const int64_t row = row0 + tid;
        // all independent loads first (no aliasing stalls behind the stores)
        const T q = ldcs(a.z + row), qt = ldcs(a.zt + row);
        const T ro = ldcs(rold + row), rto = ldcs(rtold + row);
        T pv = zero<T>(), ptv = zero<T>(), xv = zero<T>(), xtv = zero<T>();
        if (!lazy) {
          pv = ldg(pn + row);
          ptv = ldg(ptn + row);
          xv = ldcs(a.x + row);
          xtv = ldcs(a.xt + row);
        }
        update_row(row, q, qt, ro, rto, pv, ptv, xv, xtv, a.C + row * k, a.Ct + row * k);
      }
    }
  }
  pdl_trigger();
  const int G = gridDim.x;
  const T b0 = block_sum(arho, s_w);
  double b1 = block_sum(an, reinterpret_cast<double *>(s_w));
  double b2 = block_sum(ant, reinterpret_cast<double *>(s_w));
  if (tid == 0) {
    a.part[blockIdx.x] = b0;
    T t1 = zero<T>(), t2 = zero<T>();
    reinterpret_cast<double *>(&t1)[0] = b1;
    reinterpret_cast<double *>(&t2)[0] = b2;
    a.part[G + blockIdx.x] = t1;
    a.part[2 * G + blockIdx.x] = t2;
  }
  if (!last_block(&st->cnt[1], &s_last)) return;
  final_reduce(a.part, 3, G, s_fin);
  if (tid == 0) {
    st->cnt[1] = 0;
    const int i = it + 1;
    const T rho = s_fin[0];
    const double rn = sqrt(re(s_fin[1])), rtn = sqrt(re(s_fin[2]));
    const T beta = divd(rho, st->rho);   // β_i = ρ_i / ρ_{i-1}
    IterRec<T> rec;
    rec.alpha = alpha;
    rec.beta = beta;
    rec.rho = rho;
    rec.sigma = st->sigma;
    rec.rnorm = rn;
    rec.rtnorm = rtn;
    a.hist[i] = rec;
    st->iter = i;
    st->rnorm = rn;
    st->rtnorm = rtn;
    const bool conv = !st->force && rn <= st->tolb && rtn <= st->tolbt;
    if (conv) {
      st->done = 1;
      st->status = RBICG_OK;
    } else if (iszero(rho) || !finite(beta)) {
      st->done = 1;
      st->status = RBICG_BREAKDOWN_SERIOUS;
    } else if (i >= st->max_itn) {
      st->done = 1;
      st->status = st->force ? RBICG_OK : RBICG_MAXITER;
    } else if (i == st->stop_at) {
      st->done = 2;   // paused at a cycle boundary for the recycle update
    }
    st->rho = rho;
    st->beta = beta;
  }
}

// ============================================================== init / finish
// r = b - A x, r~ = b~ - A^* x~; partial ||b||², ||b~||², ||r||², ||r~||² and,
// with coef, C~^*r and C^*r~ (minusXR).
template <typename T>
__global__ void __launch_bounds__(BS, 4) k_resid(LoopArgs<T> a, const T *b, const T *bt, const T *x,
                                              const T *xt, T *r, T *rt, int coef) {
  __shared__ T s_r[BS], s_rt[BS];
  __shared__ T s_red[2 * BS];
  __shared__ T s_w[BS / 32];
  __shared__ T s_fin[4 + 2 * KMAX];
  __shared__ int s_last;
  DevState<T> *st = a.st;
  const int tid = threadIdx.x;
  const int64_t n = a.n;
  const int k = coef ? a.k : 0;
  const int rstep = k > 0 ? BS / k : 0;
  const int kt = rstep * k;
  double nb = 0, nbt = 0, nr = 0, nrt = 0;
  T a1 = zero<T>(), a2 = zero<T>();
  const int64_t ntiles = (n + BS - 1) / BS;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * BS;
    const int rows = (int)min((int64_t)BS, n - row0);
    if (tid < rows) {
      const int64_t row = row0 + tid;
      const T bv = b[row], btv = bt[row];
      const T rv = sub(bv, sell_row<T, false>(a.A, row, nullptr, x, zero<T>()));
      const T rtv = sub(btv, sell_row<T, false>(a.AH, row, nullptr, xt, zero<T>()));
      r[row] = rv;
      rt[row] = rtv;
      nb += abs2(bv);
      nbt += abs2(btv);
      nr += abs2(rv);
      nrt += abs2(rtv);
      s_r[tid] = rv;
      s_rt[tid] = rtv;
    }
    if (k > 0) {
      __syncthreads();
      if (tid < kt) {
        const int nel = rows * k;
        const T *Ct = a.Ct + row0 * k;
        const T *C = a.C + row0 * k;
        int lr = tid / k;
        for (int e = tid; e < nel; e += kt, lr += rstep) {
          a1 = cmad(Ct[e], s_r[lr], a1);
          a2 = cmad(C[e], s_rt[lr], a2);
        }
      }
      __syncthreads();
    }
  }
  const int G = gridDim.x;
  if (k > 0) {
    s_red[tid] = tid < kt ? a1 : zero<T>();
    s_red[BS + tid] = tid < kt ? a2 : zero<T>();
  }
  double sums[4] = {nb, nbt, nr, nrt};
  for (int q = 0; q < 4; ++q) {
    double v = block_sum(sums[q], reinterpret_cast<double *>(s_w));
    if (tid == 0) {
      T t = zero<T>();
      reinterpret_cast<double *>(&t)[0] = v;
      a.part[(int64_t)q * G + blockIdx.x] = t;
    }
  }
  if (tid < 2 * k) {
    const int ty = tid / k, j = tid % k;
    T s = zero<T>();
    for (int m = 0; m < rstep; ++m) s = add(s, s_red[ty * BS + j + m * k]);
    a.part[(int64_t)(4 + tid) * G + blockIdx.x] = s;
  }
  if (!last_block(&st->cnt[2], &s_last)) return;
  final_reduce(a.part, 4 + 2 * k, G, s_fin);
  if (tid == 0) {
    st->cnt[2] = 0;
    st->bn2 = re(s_fin[0]);
    st->btn2 = re(s_fin[1]);
    st->rn2 = re(s_fin[2]);
    st->rtn2 = re(s_fin[3]);
    for (int j = 0; j < k; ++j) {
      st->g[j] = scal(st->dinv[j], s_fin[4 + j]);       // Ĉ^* r_{-1}
      st->gt[j] = scal(st->dinv[j], s_fin[4 + k + j]);  // Č^* r~_{-1}
    }
  }
}

// x_0 = x_{-1} + U g, r_0 = r_{-1} - C g (and duals); ρ_0, norms; state reset.
template <typename T>
__global__ void __launch_bounds__(BS, 4) k_init2(LoopArgs<T> a, const T *U, const T *Ut) {
  __shared__ T s_g[KMAX], s_gt[KMAX];
  __shared__ T s_w[BS / 32];
  __shared__ T s_fin[3];
  __shared__ int s_last;
  DevState<T> *st = a.st;
  const int tid = threadIdx.x;
  const int k = a.k;
  if (tid < k) {
    s_g[tid] = st->g[tid];
    s_gt[tid] = st->gt[tid];
  }
  __syncthreads();
  const int64_t n = a.n;
  T *r = a.rring;   // ring column 0 holds r_{-1} -> r_0
  T *rt = a.rtring;
  T arho = zero<T>();
  double an = 0, ant = 0;
  for (int64_t row = (int64_t)blockIdx.x * BS + tid; row < n; row += (int64_t)gridDim.x * BS) {
    T rv = r[row], rtv = rt[row], xv = a.x[row], xtv = a.xt[row];
    if (k > 0) {
      T du = zero<T>(), dc = zero<T>(), dut = zero<T>(), dct = zero<T>();
      for (int j = 0; j < k; ++j) {
        du = mad(U[row * k + j], s_g[j], du);
        dc = mad(a.C[row * k + j], s_g[j], dc);
        dut = mad(Ut[row * k + j], s_gt[j], dut);
        dct = mad(a.Ct[row * k + j], s_gt[j], dct);
      }
      xv = add(xv, du);
      rv = sub(rv, dc);
      xtv = add(xtv, dut);
      rtv = sub(rtv, dct);
      a.x[row] = xv;
      a.xt[row] = xtv;
      r[row] = rv;
      rt[row] = rtv;
    }
    arho = cmad(rtv, rv, arho);
    an += abs2(rv);
    ant += abs2(rtv);
  }
  const int G = gridDim.x;
  const T b0 = block_sum(arho, s_w);
  double b1 = block_sum(an, reinterpret_cast<double *>(s_w));
  double b2 = block_sum(ant, reinterpret_cast<double *>(s_w));
  if (tid == 0) {
    a.part[blockIdx.x] = b0;
    T t1 = zero<T>(), t2 = zero<T>();
    reinterpret_cast<double *>(&t1)[0] = b1;
    reinterpret_cast<double *>(&t2)[0] = b2;
    a.part[G + blockIdx.x] = t1;
    a.part[2 * G + blockIdx.x] = t2;
  }
  if (!last_block(&st->cnt[3], &s_last)) return;
  final_reduce(a.part, 3, G, s_fin);
  if (tid == 0) {
    st->cnt[3] = 0;
    const T rho = s_fin[0];
    const double rn = sqrt(re(s_fin[1])), rtn = sqrt(re(s_fin[2]));
    st->rho = rho;
    st->beta = zero<T>();
    st->alpha = zero<T>();
    st->sigma = zero<T>();
    st->iter = 0;
    st->rnorm = rn;
    st->rtnorm = rtn;
    for (int j = 0; j < KMAX; ++j) {
      st->zc[j] = zero<T>();
      st->ztc[j] = zero<T>();
    }
    IterRec<T> rec;
    rec.alpha = zero<T>();
    rec.beta = zero<T>();
    rec.rho = rho;
    rec.sigma = zero<T>();
    rec.rnorm = rn;
    rec.rtnorm = rtn;
    a.hist[0] = rec;
    st->status = RBICG_OK;
    st->done = 0;
    if (!st->force && rn <= st->tolb && rtn <= st->tolbt) {
      st->done = 1;
    } else if (iszero(rho) || !finite(rho)) {
      st->done = 1;
      st->status = RBICG_BREAKDOWN_SERIOUS;
    } else if (st->max_itn <= 0) {
      st->done = 1;
      st->status = RBICG_MAXITER;
    }
  }
}

// Step 7: x = x_i - U ζ_c, x~ = x~_i - Ũ ζ~_c.
template <typename T>
__global__ void __launch_bounds__(BS) k_step7(LoopArgs<T> a, const T *U, const T *Ut, T *xo, T *xto) {
  __shared__ T s_c[KMAX], s_ct[KMAX];
  const DevState<T> *st = a.st;
  const int k = a.k;
  if (threadIdx.x < k) {
    s_c[threadIdx.x] = st->zc[threadIdx.x];
    s_ct[threadIdx.x] = st->ztc[threadIdx.x];
  }
  __syncthreads();
  for (int64_t row = (int64_t)blockIdx.x * BS + threadIdx.x; row < a.n;
       row += (int64_t)gridDim.x * BS) {
    T du = zero<T>(), dut = zero<T>();
    for (int j = 0; j < k; ++j) {
      du = mad(U[row * k + j], s_c[j], du);
      dut = mad(Ut[row * k + j], s_ct[j], dut);
    }
    xo[row] = sub(a.x[row], du);
    xto[row] = sub(a.xt[row], dut);
  }
}

template <typename T>
__global__ void __launch_bounds__(BS) k_spmv_pair(DevMat A, DevMat AH, const T *p, const T *pt, T *z,
                                                  T *zt) {
  for (int64_t row = (int64_t)blockIdx.x * BS + threadIdx.x; row < A.n;
       row += (int64_t)gridDim.x * BS) {
    z[row] = sell_row<T, false>(A, row, nullptr, p, zero<T>());
    zt[row] = sell_row<T, false>(AH, row, nullptr, pt, zero<T>());
  }
}

// ============================================================== launchers
static int grid_for(int64_t n, int G) {
  const int64_t tiles = (n + BS - 1) / BS;
  return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, G));
}

template <typename T> size_t pass1_smem(int tile_max) {
  return (size_t)2 * tile_max * (4 + sizeof(T));
}
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), int grid, size_t sm, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(BS);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RB_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <typename T> void launch_pass1(const LoopArgs<T> &a, cudaStream_t s) {
  const size_t sm = a.staged ? pass1_smem<T>(a.tile_max) : 0;
  int per_sm = 1;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pass1<T>, BS, sm));
  const int G = std::min(a.G, std::max(1, per_sm) * a.nsm);
  launch_pdl(k_pass1<T>, grid_for(a.n, G), sm, s, a);
  count_launch();
}

// two stages of (8 vector tiles + C, C~ tiles)
template <typename T> size_t pass2_smem(int k) {
  return (size_t)2 * (8 * BS + 2 * BS * k) * sizeof(T);
}

template <typename T> void launch_pass2(const LoopArgs<T> &a, cudaStream_t s) {
  size_t sm = pass2_smem<T>(a.k);
  const int staged = (sm <= 200 * 1024 && a.pass2_tma) ? 1 : 0;
  if (!staged) sm = 0;
  int per_sm = 1;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pass2<T>, BS, sm));
  const int G = std::min(a.G, std::max(1, per_sm) * a.nsm);
  launch_pdl(k_pass2<T>, grid_for(a.n, G), sm, s, a, staged);
  count_launch();
}

template <typename T>
void launch_resid(const LoopArgs<T> &a, const T *b, const T *bt, const T *x, const T *xt, T *r,
                  T *rt, int with_coef, cudaStream_t s) {
  k_resid<T><<<grid_for(a.n, a.G), BS, 0, s>>>(a, b, bt, x, xt, r, rt, with_coef);
  count_launch();
}

template <typename T> void launch_init2(const LoopArgs<T> &a, const T *U, const T *Ut, cudaStream_t s) {
  k_init2<T><<<grid_for(a.n, a.G), BS, 0, s>>>(a, U, Ut);
  count_launch();
}

template <typename T>
void launch_step7(const LoopArgs<T> &a, const T *U, const T *Ut, T *xo, T *xto, cudaStream_t s) {
  k_step7<T><<<grid_for(a.n, a.G), BS, 0, s>>>(a, U, Ut, xo, xto);
  count_launch();
}

template <typename T>
void launch_spmv_pair(const DevMat &A, const DevMat &AH, const T *p, const T *pt, T *z, T *zt,
                      cudaStream_t s) {
  k_spmv_pair<T><<<grid_for(A.n, 1184), BS, 0, s>>>(A, AH, p, pt, z, zt);
  count_launch();
}

int stream_blocks_per_sm() {
  int b1 = 0, b2 = 0;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_pass1<double>, BS, 0));
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_pass1<zc>, BS, 0));
  return std::max(1, std::min(b1, b2));
}

void prepare_kernels() {
  RB_CUDA(cudaFuncSetAttribute(k_pass1<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  RB_CUDA(cudaFuncSetAttribute(k_pass1<zc>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  RB_CUDA(cudaFuncSetAttribute(k_pass2<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  RB_CUDA(cudaFuncSetAttribute(k_pass2<zc>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  prepare_block_kernels();
}

#define RB_INST(T)                                                                          \
  template void launch_pass1<T>(const LoopArgs<T> &, cudaStream_t);                          \
  template void launch_pass2<T>(const LoopArgs<T> &, cudaStream_t);                          \
  template void launch_resid<T>(const LoopArgs<T> &, const T *, const T *, const T *,        \
                                const T *, T *, T *, int, cudaStream_t);                     \
  template void launch_init2<T>(const LoopArgs<T> &, const T *, const T *, cudaStream_t);    \
  template void launch_step7<T>(const LoopArgs<T> &, const T *, const T *, T *, T *,         \
                                cudaStream_t);                                               \
  template void launch_spmv_pair<T>(const DevMat &, const DevMat &, const T *, const T *, T *, \
                                    T *, cudaStream_t);
RB_INST(double)
RB_INST(zc)

}  // namespace rbicg
