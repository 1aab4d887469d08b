// hot.cuh -- device building blocks of the RBiCG hot loop (Algorithm 2,
// PAPER.md:453-473) in its two-kernel form (kernels.cu: k_pass1/k_pass1s,
// k_pass2, one launch each per iteration).
//
//   phase 1  p_i = r_{i-1} + β_{i-1} p_{i-1},  p~_i = r~_{i-1} + β̄ p~_{i-1}
//            z_i = A p_i,  z~_i = A^* p~_i          (SELL-32 SpMV pair, the
//            direction update fused into the gather)
//            partial sums of C~^*z, C^*z~, C^*p~, p~^*z  (oblique-projection
//            coefficients; σ_i via reading Q23) and of C~^*r_{i-1},
//            C^*r~_{i-1} (Petrov-Galerkin maintenance, reading Q32)
//            reduction leader: ζ = D_c^{-1}C~^*z, ζ~ = D_c^{-1}C^*z~,
//                              σ = p~^*z - (C^*p~)^*ζ, α = ρ/σ,
//                              g = D_c^{-1}C~^*r_{i-1}, g~ = D_c^{-1}C^*r~_{i-1},
//                              γ = αζ - g, γ~ = ᾱζ~ - g~, ζ_c += γ, ζ~_c += γ~
//   phase 2  r_i = r_{i-1} - αz + Cγ  (= r_{i-1} - α q_i - C g, q = z - Cζ,
//            P:461, :470 with Q32), r~_i = r~_{i-1} - ᾱz~ + C~γ~ (written
//            straight into the Lanczos ring column i);
//            (x += αp; x~ += ᾱp~ unless lazy x); partial ρ_i, ||r||², ||r~||²
//            reduction leader: β_i = ρ_i/ρ_{i-1}, stop test (Q2), breakdown
//            (Q3), iteration record for the cycle-end control.
#pragma once
#include "internal.h"

namespace rbicg {

// ---------------------------------------------------------------- loads
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
// COH = true: load of a vector another block may have rewritten earlier in
// the same launch (L2 only, never a stale L1 / read-only-cache line);
// COH = false -> read-only path.
template <bool COH, typename T> __device__ __forceinline__ T ldv(const T *p) {
  if (COH) return ldcg(p);
  return ldg(p);
}

// Direction p_j / p~_j (ring column or ping-pong buffer).
template <typename T> __device__ __forceinline__ T *pcol(const LoopArgs<T> &a, int j) {
  return a.p[j & 1];
}
template <typename T> __device__ __forceinline__ T *ptcol(const LoopArgs<T> &a, int j) {
  return a.pt[j & 1];
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
__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// same, with an L2 eviction-priority policy (createpolicy) for streamed data
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_1d_hint(void *dst, const void *src, uint32_t bytes,
                                                 uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra "
      "WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// generic-proxy writes of this thread -> later bulk (async-proxy) reads
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---------------------------------------------------------------- SpMV rows
// y_row = Σ_j a_{row,j} (r_j + β p_j)   (FUSE)   or   Σ_j a_{row,j} p_j
template <typename T, bool FUSE, bool COH = false>
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
    if (FUSE) pj = mad(beta, ldv<COH>(p + c), ldg(r + c));
    else pj = ldv<COH>(p + c);
    acc = mad(v, pj, acc);
  }
  return acc;
}

// One row of the SpMV pair from TMA-staged SELL tiles (column-major slices in
// shared memory).  Both matrices' gathers are issued together in chunks of 4
// so up to 16 independent loads per thread are in flight.  r, r~ are Lanczos
// ring columns (never rewritten within a launch: read-only path); p, p~ go
// through ldv<COH>.
template <typename T, bool COH>
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
      pa[q] = ldv<COH>(p + ca[q]);
      rh[q] = ldg(rt + ch[q]);
      ph[q] = ldv<COH>(pt + ch[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      z = mad(va[q], mad(beta, pa[q], ra[q]), z);
      zt = mad(vh[q], mad(cb, ph[q], rh[q]), zt);
    }
  }
}

// ---------------------------------------------------------------- reductions
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

// Release-ordered arrival (MEMBAR without the L1 invalidation __threadfence
// adds, which would also discard the L1 lines of the other blocks still
// working on this SM).
__device__ __forceinline__ unsigned atom_add_release(unsigned *p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_release() { asm volatile("fence.release.gpu;" ::: "memory"); }
// acquire side: invalidates this SM's L1 (CCTL.IVALL) -- issued only once
// every block of the grid has arrived
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acquire.gpu;" ::: "memory"); }

// Last-block election; returns true in every thread of the last block.
__device__ __forceinline__ bool last_block(unsigned *cnt, int *s_flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned v = atom_add_release(cnt, 1u);
    *s_flag = (v == gridDim.x - 1);
    if (*s_flag) fence_acquire();
  }
  __syncthreads();
  return *s_flag != 0;
}

// Tile visiting order of the SpMV kernels (LoopArgs::torder): the number of
// tiles this launch visits, the tile of visit index ix, and the reduction's
// block count / this block's slot.
template <typename T> __device__ __forceinline__ int64_t launch_tiles(const LoopArgs<T> &a, int64_t ntiles) {
  return a.ordered ? a.tcount : ntiles;
}
template <typename T>
__device__ __forceinline__ int64_t tile_at(const LoopArgs<T> &a, const int32_t *ord, int64_t ix) {
  return a.ordered ? (int64_t)ord[a.tbase + ix] : ix;
}
// the reduction of one iteration's SpMV kernel: stride of the partials,
// this block's slot, and (phase 2 / single launch) the number of partials
template <typename T> __device__ __forceinline__ int red_stride(const LoopArgs<T> &a) {
  return a.phase ? a.pstride : (int)gridDim.x;
}
template <typename T> __device__ __forceinline__ int red_slot(const LoopArgs<T> &a) {
  return (a.phase == 2 ? __ldcg(&a.st->g1) : 0) + (int)blockIdx.x;
}
template <typename T> __device__ __forceinline__ int red_count(const LoopArgs<T> &a) {
  return (a.phase == 2 ? __ldcg(&a.st->g1) : 0) + (int)gridDim.x;
}
// phase 1: record the grid and stop after the partials (true = return)
template <typename T> __device__ __forceinline__ bool interior_done(const LoopArgs<T> &a) {
  if (a.phase != 1) return false;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.st->g1 = (int)gridDim.x;
  return true;
}

// Final fixed-order reduction of `nout` outputs stored as part[o*G + b].
// All partial loads of a lane are issued before any add (they are L2 hits;
// a dependent chain of G/32 loads would cost microseconds at the kernel tail).
constexpr int RED_PER_LANE = 20;   // one round of loads for G <= 640 blocks
template <typename T>
__device__ __forceinline__ void final_reduce(const T *part, int nout, int G, T *s_fin, int stride = 0) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int o = w; o < nout; o += BS / 32) {
    const T *src = part + (int64_t)o * (stride ? stride : G);
    T acc = zero<T>();
    for (int q0 = 0; q0 < G; q0 += 32 * RED_PER_LANE) {
      T v[RED_PER_LANE];
#pragma unroll
      for (int q = 0; q < RED_PER_LANE; ++q) {
        const int b = q0 + l + 32 * q;
        v[q] = b < G ? ldcg(src + b) : zero<T>();
      }
#pragma unroll
      for (int q = 0; q < RED_PER_LANE; ++q) acc = add(acc, v[q]);
    }
    acc = warp_sum(acc);
    if (l == 0) s_fin[o] = acc;
  }
  __syncthreads();
}

// ---------------------------------------------------------------- state snapshot
// The device-state fields a phase needs, loaded in parallel at the phase start
// through L2 (the leader of the previous reduction wrote them; a dependent
// chain of L2 loads in one thread at the tail cost microseconds per launch).
template <typename T>
struct Snap {
  T beta, alpha, rho, sigma;
  double tolb, tolbt;
  int iter, done, seg_start, force, max_itn, stop_at;
  double dinv[KMAX];
  T gam[KMAX], gamt[KMAX], zc[KMAX], ztc[KMAX];
};
template <typename T>
__device__ __forceinline__ void snap_load(const DevState<T> *st, int k, Snap<T> &s) {
  const int tid = threadIdx.x;
  if (tid < k) {
    s.dinv[tid] = __ldcg(&st->dinv[tid]);
    s.gam[tid] = ldcg(&st->gam[tid]);
    s.gamt[tid] = ldcg(&st->gamt[tid]);
    s.zc[tid] = ldcg(&st->zc[tid]);
    s.ztc[tid] = ldcg(&st->ztc[tid]);
  }
  if (tid == 32) {
    s.beta = ldcg(&st->beta);
    s.alpha = ldcg(&st->alpha);
    s.rho = ldcg(&st->rho);
    s.sigma = ldcg(&st->sigma);
    s.tolb = __ldcg(&st->tolb);
    s.tolbt = __ldcg(&st->tolbt);
    s.iter = __ldcg(&st->iter);
    s.done = __ldcg(&st->done);
    s.seg_start = __ldcg(&st->seg_start);
    s.force = __ldcg(&st->force);
    s.max_itn = __ldcg(&st->max_itn);
    s.stop_at = __ldcg(&st->stop_at);
  }
  __syncthreads();
}

// ---------------------------------------------------------------- leaders
// Phase-1 reduction leader (whole block; s_fin holds the reduced sums).
// Returns false (in every thread) on a breakdown of the second kind.
template <typename T>
__device__ __forceinline__ bool p1_leader(const LoopArgs<T> &a, DevState<T> *st, const Snap<T> &sn,
                                          int it, T *s_fin, T *s_alpha, int *s_ok) {
  const int tid = threadIdx.x;
  const int k = a.k;
  if (tid < k) {   // ζ_i = D_c^{-1} C~^* z_i, ζ~_i = D_c^{-1} C^* z~_i
    s_fin[tid] = scal(sn.dinv[tid], s_fin[tid]);
    s_fin[k + tid] = scal(sn.dinv[tid], s_fin[k + tid]);
    // Q32: g_{i-1} = D_c^{-1} C~^* r_{i-1}, g~_{i-1} = D_c^{-1} C^* r~_{i-1}
    s_fin[3 * k + 1 + tid] = scal(sn.dinv[tid], s_fin[3 * k + 1 + tid]);
    s_fin[4 * k + 1 + tid] = scal(sn.dinv[tid], s_fin[4 * k + 1 + tid]);
  }
  __syncthreads();
  if (tid == 0) {
    T sigma = s_fin[3 * k];
    for (int j = 0; j < k; ++j) sigma = sub(sigma, cmul(s_fin[2 * k + j], s_fin[j]));   // (p~, z - Cζ)  (Q23)
    const T alpha = divd(sn.rho, sigma);
    *s_ok = !(iszero(sigma) || !finite(alpha));
    if (!*s_ok) {   // breakdown of the second kind
      st->status = RBICG_BREAKDOWN_SECOND;
      st->done = 1;
    } else {
      st->alpha = alpha;
      st->sigma = sigma;
    }
    *s_alpha = alpha;
  }
  __syncthreads();
  if (!*s_ok) return false;
  if (tid < k) {
    const int i = it + 1, j = tid;
    const T alpha = *s_alpha, ca = conj(alpha);
    const T zj = s_fin[j], ztj = s_fin[k + j];
    // γ = αζ - g: pass 2 forms r_i = r_{i-1} - α q_i - C g_{i-1} as
    // r_{i-1} - α z_i + C γ, and ζ_c += γ keeps b - A(x_i - Uζ_c) = r_i (Q32)
    const T gj = sub(mul(alpha, zj), s_fin[3 * k + 1 + j]);
    const T gtj = sub(mul(ca, ztj), s_fin[4 * k + 1 + j]);
    st->gam[j] = gj;
    st->gamt[j] = gtj;
    st->zc[j] = add(sn.zc[j], gj);
    st->ztc[j] = add(sn.ztc[j], gtj);
    a.zhist[(int64_t)i * k + j] = zj;
    a.zthist[(int64_t)i * k + j] = ztj;
    fence_release();
  }
  return true;
}

// Phase-2 reduction leader (thread 0): β, iteration record, stop test.
template <typename T>
__device__ __forceinline__ void p2_leader(const LoopArgs<T> &a, DevState<T> *st, const Snap<T> &sn,
                                          int it, const T *s_fin) {
  if (threadIdx.x != 0) return;
  const int i = it + 1;
  const T rho = s_fin[0];
  const double rn = sqrt(re(s_fin[1])), rtn = sqrt(re(s_fin[2]));
  const T beta = divd(rho, sn.rho);   // β_i = ρ_i / ρ_{i-1}
  IterRec<T> rec;
  rec.alpha = sn.alpha;
  rec.beta = beta;
  rec.rho = rho;
  rec.sigma = sn.sigma;
  rec.rnorm = rn;
  rec.rtnorm = rtn;
  a.hist[i] = rec;
  int done = 0, status = RBICG_OK;
  const bool conv = !sn.force && rn <= sn.tolb && rtn <= sn.tolbt;
  if (conv) {
    done = 1;
  } else if (iszero(rho) || !finite(beta)) {
    done = 1;
    status = RBICG_BREAKDOWN_SERIOUS;
  } else if (i >= sn.max_itn) {
    done = 1;
    status = sn.force ? RBICG_OK : RBICG_MAXITER;
  } else if (i == sn.stop_at) {
    done = 2;   // paused at a cycle boundary for the recycle update
  }
  st->iter = i;
  st->rnorm = rn;
  st->rtnorm = rtn;
  st->rho = rho;
  st->beta = beta;
  if (done) {
    st->status = status;
    st->done = done;
  }
}

// ---------------------------------------------------------------- phase bodies
// Phase-1 shared-memory scratch (static part).
// s_red (block partials of the projection coefficients) reuses the storage of
// s_z, s_zt, s_pt: it is written only after the last tile's projection.
template <typename T>
struct P1Scratch {
  T buf[3 * BS];
  __device__ T *s_z() { return buf; }
  __device__ T *s_zt() { return buf + BS; }
  __device__ T *s_pt() { return buf + 2 * BS; }
  __device__ T *s_red() { return buf; }
};

// Phase-1 stage: [cols A | cols A^* | vals A | vals A^*] (tile_max each) and,
// with stage_v, the tile's own rows of r, p, r~, p~ (BS each).  The stage's
// mbarrier expects two arrivals when stage_v (matrix part, vector part: the
// vector part depends on the previous phase, the matrix part does not).
// [cols A | cols A^* (unless shared) | vals A | vals A^*]
template <typename T> __host__ __device__ __forceinline__ int p1_ncols(const LoopArgs<T> &a) {
  return a.shared_cols ? 1 : 2;
}
template <typename T> __host__ __device__ __forceinline__ size_t p1_mat_bytes(const LoopArgs<T> &a) {
  return (size_t)a.tile_max * (4 * p1_ncols(a) + 2 * sizeof(T));
}
template <typename T> __host__ __device__ __forceinline__ size_t p1_stage_bytes(const LoopArgs<T> &a) {
  return p1_mat_bytes<T>(a) + (a.stage_v ? (size_t)4 * BS * sizeof(T) : 0);
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Vector part of a phase-1 stage for tile t of iteration it (full tiles; a
// partial tile only arrives and reads its rows from global memory).
template <typename T>
__device__ __forceinline__ void p1_issue_vec(const LoopArgs<T> &a, unsigned char *stage,
                                             uint64_t *bar, int64_t t, int it) {
  if ((t + 1) * BS > a.n) {
    mbar_arrive(bar);
    return;
  }
  T *v = reinterpret_cast<T *>(stage + p1_mat_bytes<T>(a));
  const uint32_t vb = BS * (uint32_t)sizeof(T);
  const int64_t r0 = t * BS;
  mbar_expect_tx(bar, 4u * vb);
  tma_load_1d(v, a.rring + (int64_t)(it % a.ring) * a.ldr + r0, vb, bar);
  tma_load_1d(v + BS, pcol(a, it) + r0, vb, bar);
  tma_load_1d(v + 2 * BS, a.rtring + (int64_t)(it % a.ring) * a.ldr + r0, vb, bar);
  tma_load_1d(v + 3 * BS, ptcol(a, it) + r0, vb, bar);
}

// Matrix-tile TMA for phase 1 into one stage, tile t.
template <typename T>
__device__ __forceinline__ void p1_issue(const LoopArgs<T> &a, unsigned char *stages,
                                         size_t stage_bytes, uint64_t *bar, int64_t t) {
  const int TM = a.tile_max;
  int32_t *cA = reinterpret_cast<int32_t *>(stages);
  int32_t *cH = cA + TM;
  T *vA = reinterpret_cast<T *>(cA + p1_ncols(a) * TM);
  T *vH = vA + TM;
  const int64_t ns = a.A.nslices;
  const int64_t s0 = t * (BS / 32), s1 = min(s0 + BS / 32, ns);
  const int64_t oA = a.A.sptr[s0], eA = a.A.sptr[s1];
  const int64_t oH = a.AH.sptr[s0], eH = a.AH.sptr[s1];
  const uint32_t nA = (uint32_t)(eA - oA), nH = (uint32_t)(eH - oH);
  const uint32_t nHc = a.shared_cols ? 0u : nH;   // A^*'s columns: A's (structurally symmetric)
  mbar_expect_tx(bar, (nA + nH) * (uint32_t)sizeof(T) + (nA + nHc) * 4u);
  if (a.l2ef) {   // the matrix pair is streamed once per pass: evict it first
    const uint64_t pol = policy_evict_first();
    if (nA) {
      tma_load_1d_hint(cA, a.A.cols + oA, nA * 4u, bar, pol);
      tma_load_1d_hint(vA, reinterpret_cast<const T *>(a.A.vals) + oA, nA * (uint32_t)sizeof(T), bar, pol);
    }
    if (nH) {
      if (nHc) tma_load_1d_hint(cH, a.AH.cols + oH, nH * 4u, bar, pol);
      tma_load_1d_hint(vH, reinterpret_cast<const T *>(a.AH.vals) + oH, nH * (uint32_t)sizeof(T), bar, pol);
    }
    return;
  }
  if (nA) {
    tma_load_1d(cA, a.A.cols + oA, nA * 4u, bar);
    tma_load_1d(vA, reinterpret_cast<const T *>(a.A.vals) + oA, nA * (uint32_t)sizeof(T), bar);
  }
  if (nH) {
    if (nHc) tma_load_1d(cH, a.AH.cols + oH, nH * 4u, bar);
    tma_load_1d(vH, reinterpret_cast<const T *>(a.AH.vals) + oH, nH * (uint32_t)sizeof(T), bar);
  }
}

// Phase 1 over this block's tiles (blockIdx.x, +G, ...).  With a.staged the
// matrix tiles come through `nst` TMA stages (bars[0..nst-1]); the caller has
// already issued the first min(nst, #tiles) tiles.  par holds the parity bit
// of each mbarrier (bit j for bars[j]).  On return the four partial
// accumulators are in a1..aptz.
template <typename T, bool COH>
__device__ __forceinline__ void p1_tiles(const LoopArgs<T> &a, unsigned char *dsm, uint64_t *bars,
                                         uint32_t &par, P1Scratch<T> &sc, int it, T beta,
                                         bool segcopy, T &a1, T &a2, T &a3, T &a4, T &a5,
                                         T &aptz) {
  const int tid = threadIdx.x;
  const int64_t n = a.n;
  const int64_t ntiles = (n + BS - 1) / BS;
  const int64_t G64 = gridDim.x;
  const int TM = a.tile_max;
  const int nst = a.p1_stages;
  const size_t stage_bytes = p1_stage_bytes<T>(a);
  const bool stage_v = a.staged && a.stage_v;
  const int k = a.k;
  T *sC = reinterpret_cast<T *>(dsm + nst * stage_bytes);   // [C tile | C~ tile]
  const bool stage_c = a.staged && a.stage_c && k > 0;
  const int64_t ns = a.A.nslices;
  const T cb = conj(beta);
  const T *__restrict__ r = a.rring + (int64_t)(it % a.ring) * a.ldr;
  const T *__restrict__ rt = a.rtring + (int64_t)(it % a.ring) * a.ldr;
  const T *__restrict__ pold = pcol(a, it);
  const T *__restrict__ ptold = ptcol(a, it);
  T *__restrict__ pnew = pcol(a, it + 1);
  T *__restrict__ ptnew = ptcol(a, it + 1);
  const int rstep = k > 0 ? BS / k : 0;
  const int kt = rstep * k;
  const int64_t nvis = launch_tiles(a, ntiles);
  int i = 0;
  for (int64_t ix = blockIdx.x; ix < nvis; ix += G64, ++i) {
    const int64_t tile = tile_at(a, a.torder, ix);
    const int64_t row0 = tile * BS;
    const int rows = (int)min((int64_t)BS, n - row0);
    const bool cst = stage_c && rows == BS;
    if (cst && tid == 0) {   // C buffer is free (trailing barrier below)
      const uint32_t cbytes = (uint32_t)(BS * k * sizeof(T));
      mbar_expect_tx(&bars[2], 2u * cbytes);
      tma_load_1d(sC, a.C + tile * BS * k, cbytes, &bars[2]);
      tma_load_1d(sC + BS * k, a.Ct + tile * BS * k, cbytes, &bars[2]);
    }
    if (a.pf && tid == 32 && ix + G64 < nvis && (tile_at(a, a.torder, ix + G64) + 1) * BS <= n) {
      // the vector rows of this block's next tile: first touched by the
      // gathers of nearby tiles, so pull them into L2 ahead of the wave
      const int64_t r1 = tile_at(a, a.torder, ix + G64) * BS;
      const uint32_t vb = BS * (uint32_t)sizeof(T);
      prefetch_l2(r + r1, vb);
      prefetch_l2(rt + r1, vb);
      prefetch_l2(pold + r1, vb);
      prefetch_l2(ptold + r1, vb);
    }
    auto finish_row = [&](int64_t row, T z, T zt, T rr, T po, T rtr, T pto) {
      const T pn = mad(beta, po, rr);
      const T ptn = mad(cb, pto, rtr);
      if (segcopy) {   // lazy x: keep p_a, p~_a of the new segment
        a.pseg[(it / a.cyc) & 1][row] = po;
        a.ptseg[(it / a.cyc) & 1][row] = pto;
      }
      if (!(a.abl & 2)) {   // (timing ablation 2: no stores)
        pnew[row] = pn;
        ptnew[row] = ptn;
        a.z[row] = z;
        a.zt[row] = zt;
      }
      aptz = cmad(ptn, z, aptz);
      sc.s_z()[tid] = z;
      sc.s_zt()[tid] = zt;
      sc.s_pt()[tid] = ptn;
    };
    if (a.staged) {
      const int si = nst == 2 ? (i & 1) : 0;
      const unsigned char *base = dsm + si * stage_bytes;
      const int32_t *scA = reinterpret_cast<const int32_t *>(base);
      const int32_t *scH = a.shared_cols ? scA : scA + TM;
      const T *svA = reinterpret_cast<const T *>(scA + p1_ncols(a) * TM);
      const T *svH = svA + TM;
      // slice geometry (global loads overlap the bulk copy)
      const int64_t sl = (row0 >> 5) + (tid >> 5);
      const int64_t slc = min(sl, ns - 1);
      const int64_t bA = a.A.sptr[tile * (BS / 32)], bH = a.AH.sptr[tile * (BS / 32)];
      const int64_t oA = a.A.sptr[slc], oH = a.AH.sptr[slc];
      const int wA = (int)((a.A.sptr[slc + 1] - oA) >> 5), wH = (int)((a.AH.sptr[slc + 1] - oH) >> 5);
      const int lane = tid & 31;
      mbar_wait(&bars[si], (par >> si) & 1u);
      par ^= 1u << si;
      if (tid < rows) {
        T z, zt;
        if (a.abl & 1) {   // timing ablation: no gathers (row-local operands)
          const int64_t row = row0 + tid;
          const T *sv = reinterpret_cast<const T *>(base + p1_mat_bytes<T>(a));
          const bool vs = stage_v && rows == BS;
          const T xr = vs ? mad(beta, sv[BS + tid], sv[tid]) : mad(beta, ldg(pold + row), ldg(r + row));
          const T xrt = vs ? mad(cb, sv[3 * BS + tid], sv[2 * BS + tid]) : mad(cb, ldg(ptold + row), ldg(rt + row));
          z = zero<T>();
          zt = zero<T>();
          for (int j = 0; j < wA; ++j) z = mad(svA[(oA - bA) + lane + j * 32], xr, z);
          for (int j = 0; j < wH; ++j) zt = mad(svH[(oH - bH) + lane + j * 32], xrt, zt);
        } else {
          sell_pair_smem<T, COH>(scA + (oA - bA) + lane, svA + (oA - bA) + lane, wA,
                                 scH + (oH - bH) + lane, svH + (oH - bH) + lane, wH, r, pold, rt,
                                 ptold, beta, cb, z, zt);
        }
        const int64_t row = row0 + tid;
        if (stage_v && rows == BS) {
          const T *sv = reinterpret_cast<const T *>(base + p1_mat_bytes<T>(a));
          finish_row(row, z, zt, sv[tid], sv[BS + tid], sv[2 * BS + tid], sv[3 * BS + tid]);
        } else {
          finish_row(row, z, zt, ldg(r + row), ldv<COH>(pold + row), ldg(rt + row),
                     ldv<COH>(ptold + row));
        }
      }
      __syncthreads();   // stage si consumed -> refill with visit ix + nst G
      if (tid == 0 && ix + nst * G64 < nvis) {
        const int64_t tn = tile_at(a, a.torder, ix + nst * G64);
        p1_issue<T>(a, dsm + si * stage_bytes, stage_bytes, &bars[si], tn);
        if (stage_v) p1_issue_vec<T>(a, dsm + si * stage_bytes, &bars[si], tn, it);
      }
    } else if (tid < rows) {
      const int64_t row = row0 + tid;
      const T z = sell_row<T, true, COH>(a.A, row, r, pold, beta);
      const T zt = sell_row<T, true, COH>(a.AH, row, rt, ptold, cb);
      finish_row(row, z, zt, ldg(r + row), ldv<COH>(pold + row), ldg(rt + row),
                 ldv<COH>(ptold + row));
    }
    if (k > 0) {
      __syncthreads();
      if (tid < kt) {
        // thread tid always meets column tid % k because kt is a multiple of k
        const int nel = rows * k;
        int lr = tid / k;
        if (cst) {
          mbar_wait(&bars[2], (par >> 2) & 1u);
          const T *__restrict__ Ct = sC + BS * k;
          const T *__restrict__ C = sC;
          for (int e = tid; e < nel; e += kt, lr += rstep) {
            const T ct = Ct[e], c = C[e];
            a1 = cmad(ct, sc.s_z()[lr], a1);   // conj(c~_{row,j}) z_row
            a2 = cmad(c, sc.s_zt()[lr], a2);   // conj(c_{row,j}) z~_row
            a3 = cmad(c, sc.s_pt()[lr], a3);   // conj(c_{row,j}) p~_row
            a4 = cmad(ct, ldg(r + row0 + lr), a4);    // conj(c~_{row,j}) r_row (Q32)
            a5 = cmad(c, ldg(rt + row0 + lr), a5);    // conj(c_{row,j}) r~_row
          }
        } else {
          const T *__restrict__ Ct = a.Ct + row0 * k;
          const T *__restrict__ C = a.C + row0 * k;
#pragma unroll 4
          for (int e = tid; e < nel; e += kt, lr += rstep) {
            const T ct = ldcs(Ct + e), c = ldcs(C + e);
            a1 = cmad(ct, sc.s_z()[lr], a1);
            a2 = cmad(c, sc.s_zt()[lr], a2);
            a3 = cmad(c, sc.s_pt()[lr], a3);
            a4 = cmad(ct, ldg(r + row0 + lr), a4);
            a5 = cmad(c, ldg(rt + row0 + lr), a5);
          }
        }
      } else if (cst) {
        mbar_wait(&bars[2], (par >> 2) & 1u);   // keep every thread's parity in step
      }
      if (cst) par ^= 1u << 2;
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- phase 1, split form
// 128-row tiles; threads 0..127 compute the rows of z = A p (gathering r, p),
// threads 128..255 the rows of z~ = A^* p~ (gathering r~, p~), so each thread
// has one row of one matrix and issues all of its gathers in one round (CH
// nonzeros at a time).  Stage: [cols A | cols A^* | vals A | vals A^*]
// (tile_max_h each) [r | p | r~ | p~ rows, 128 each].

template <typename T> __host__ __device__ __forceinline__ size_t p1s_mat_bytes(int tmh) {
  return (size_t)2 * tmh * (4 + sizeof(T));
}
template <typename T> __host__ __device__ __forceinline__ size_t p1s_stage_bytes(const LoopArgs<T> &a) {
  return p1s_mat_bytes<T>(a.tile_max_h) + (a.stage_v ? (size_t)4 * TRH * sizeof(T) : 0);
}
template <typename T>
__device__ __forceinline__ void p1s_issue(const LoopArgs<T> &a, unsigned char *stage, uint64_t *bar,
                                          int64_t t) {
  const int TM = a.tile_max_h;
  int32_t *cA = reinterpret_cast<int32_t *>(stage);
  int32_t *cH = cA + TM;
  T *vA = reinterpret_cast<T *>(cH + TM);
  T *vH = vA + TM;
  const int64_t ns = a.A.nslices;
  const int64_t s0 = t * (TRH / 32), s1 = min(s0 + TRH / 32, ns);
  const int64_t oA = a.A.sptr[s0], eA = a.A.sptr[s1];
  const int64_t oH = a.AH.sptr[s0], eH = a.AH.sptr[s1];
  const uint32_t nA = (uint32_t)(eA - oA), nH = (uint32_t)(eH - oH);
  const uint32_t nHc = a.shared_cols ? 0u : nH;
  mbar_expect_tx(bar, (nA + nH) * (uint32_t)sizeof(T) + (nA + nHc) * 4u);
  const uint64_t pol = policy_evict_first();   // streamed once per pass
  if (nA) {
    tma_load_1d_hint(cA, a.A.cols + oA, nA * 4u, bar, pol);
    tma_load_1d_hint(vA, reinterpret_cast<const T *>(a.A.vals) + oA, nA * (uint32_t)sizeof(T), bar, pol);
  }
  if (nH) {
    if (nHc) tma_load_1d_hint(cH, a.AH.cols + oH, nH * 4u, bar, pol);
    tma_load_1d_hint(vH, reinterpret_cast<const T *>(a.AH.vals) + oH, nH * (uint32_t)sizeof(T), bar, pol);
  }
}
template <typename T>
__device__ __forceinline__ void p1s_issue_vec(const LoopArgs<T> &a, unsigned char *stage,
                                              uint64_t *bar, int64_t t, int it) {
  if ((t + 1) * TRH > a.n) {
    mbar_arrive(bar);
    return;
  }
  T *v = reinterpret_cast<T *>(stage + p1s_mat_bytes<T>(a.tile_max_h));
  const uint32_t vb = TRH * (uint32_t)sizeof(T);
  const int64_t r0 = t * TRH;
  mbar_expect_tx(bar, 4u * vb);
  tma_load_1d(v, a.rring + (int64_t)(it % a.ring) * a.ldr + r0, vb, bar);
  tma_load_1d(v + TRH, pcol(a, it) + r0, vb, bar);
  tma_load_1d(v + 2 * TRH, a.rtring + (int64_t)(it % a.ring) * a.ldr + r0, vb, bar);
  tma_load_1d(v + 3 * TRH, ptcol(a, it) + r0, vb, bar);
}

// One row of one matrix from its staged SELL slice: Σ_j a_j (r_{c_j} + β p_{c_j}),
// CH nonzeros' gathers in flight at a time.
template <typename T, bool COH, int CH>
__device__ __forceinline__ T sell_row_smem(const int32_t *__restrict__ c, const T *__restrict__ v, int w,
                                           const T *__restrict__ r, const T *__restrict__ p, T beta) {
  T acc = zero<T>();
  for (int j0 = 0; j0 < w; j0 += CH) {
    int cc[CH];
    T vv[CH], rr[CH], pp[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const int jj = j0 + q;
      const bool in = jj < w;
      cc[q] = in ? c[jj * 32] : 0;
      vv[q] = in ? v[jj * 32] : zero<T>();
    }
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      rr[q] = ldg(r + cc[q]);
      pp[q] = ldv<COH>(p + cc[q]);
    }
#pragma unroll
    for (int q = 0; q < CH; ++q) acc = mad(vv[q], mad(beta, pp[q], rr[q]), acc);
  }
  return acc;
}

template <typename T, bool COH, int CH>
__device__ __forceinline__ void p1_tiles_split(const LoopArgs<T> &a, unsigned char *dsm, uint64_t *bars,
                                               uint32_t &par, P1Scratch<T> &sc, int it, T beta,
                                               bool segcopy, T &a1, T &a2, T &a3, T &a4, T &a5,
                                               T &aptz) {
  const int tid = threadIdx.x;
  const int side = tid >> 7;          // 0: A, 1: A^*
  const int lr = tid & (TRH - 1);
  const int lane = tid & 31;
  const int64_t n = a.n;
  const int64_t ntiles = (n + TRH - 1) / TRH;
  const int64_t G64 = gridDim.x;
  const int TM = a.tile_max_h;
  const int nst = a.p1_stages;
  const size_t stage_bytes = p1s_stage_bytes<T>(a);
  const bool stage_v = a.stage_v != 0;
  const int k = a.k;
  T *sC = reinterpret_cast<T *>(dsm + nst * stage_bytes);   // [C tile | C~ tile]
  const bool stage_c = a.stage_c && k > 0;
  const int64_t ns = a.A.nslices;
  const T bet = side ? conj(beta) : beta;
  const DevMat &M = side ? a.AH : a.A;
  const T *__restrict__ rv = a.rring + (int64_t)(it % a.ring) * a.ldr;
  const T *__restrict__ rtv = a.rtring + (int64_t)(it % a.ring) * a.ldr;
  const T *__restrict__ r = side ? rtv : rv;
  const T *__restrict__ pold = side ? ptcol(a, it) : pcol(a, it);
  T *__restrict__ pnew = side ? ptcol(a, it + 1) : pcol(a, it + 1);
  T *__restrict__ zout = side ? a.zt : a.z;
  T *__restrict__ pseg = side ? a.ptseg[(it / a.cyc) & 1] : a.pseg[(it / a.cyc) & 1];
  T *s_z = sc.s_z(), *s_zt = s_z + TRH, *s_pt2 = s_z + 2 * TRH;   // s_pt double-buffered
  T *s_r = s_z + 4 * TRH, *s_rt = s_z + 5 * TRH;   // r_{i-1}, r~_{i-1} rows (Q32)
  const int rstep = k > 0 ? BS / k : 0;
  const int kt = rstep * k;
  const int64_t nvis = launch_tiles(a, ntiles);
  int i = 0;
  for (int64_t ix = blockIdx.x; ix < nvis; ix += G64, ++i) {
    const int64_t tile = tile_at(a, a.torder_h, ix);
    const int64_t row0 = tile * TRH;
    const int rows = (int)min((int64_t)TRH, n - row0);
    const bool cst = stage_c && rows == TRH;
    if (cst && tid == 0) {   // C buffer is free (trailing barrier below)
      const uint32_t cbytes = (uint32_t)(TRH * k * sizeof(T));
      mbar_expect_tx(&bars[2], 2u * cbytes);
      tma_load_1d(sC, a.C + tile * TRH * k, cbytes, &bars[2]);
      tma_load_1d(sC + TRH * k, a.Ct + tile * TRH * k, cbytes, &bars[2]);
    }
    const int si = nst == 2 ? (i & 1) : 0;
    const unsigned char *base = dsm + si * stage_bytes;
    const int32_t *sc0 = reinterpret_cast<const int32_t *>(base) + (side && !a.shared_cols ? TM : 0);
    const T *sv0 = reinterpret_cast<const T *>(base + (size_t)2 * TM * 4) + (side ? TM : 0);
    const int64_t slc = min((row0 >> 5) + (lr >> 5), ns - 1);
    const int64_t bM = M.sptr[tile * (TRH / 32)];
    const int64_t oM = M.sptr[slc];
    const int wM = (int)((M.sptr[slc + 1] - oM) >> 5);
    T *s_pt = s_pt2 + (i & 1) * TRH;
    mbar_wait(&bars[si], (par >> si) & 1u);
    par ^= 1u << si;
    if (lr < rows) {
      const int64_t row = row0 + lr;
      const T acc = sell_row_smem<T, COH, CH>(sc0 + (oM - bM) + lane, sv0 + (oM - bM) + lane, wM, r,
                                              pold, bet);
      T rr, pp;
      if (stage_v && rows == TRH) {
        const T *sv = reinterpret_cast<const T *>(base + p1s_mat_bytes<T>(TM)) + side * 2 * TRH;
        rr = sv[lr];
        pp = sv[TRH + lr];
      } else {
        rr = ldg(r + row);
        pp = ldv<COH>(pold + row);
      }
      const T pn = mad(bet, pp, rr);
      if (segcopy) pseg[row] = pp;   // lazy x: keep p_a, p~_a of the new segment
      pnew[row] = pn;
      zout[row] = acc;
      if (side) {
        s_zt[lr] = acc;
        s_pt[lr] = pn;
        s_rt[lr] = rr;
      } else {
        s_z[lr] = acc;
        s_r[lr] = rr;
      }
    }
    __syncthreads();   // stage si consumed -> refill with tile + nst G
    if (tid == 0 && ix + nst * G64 < nvis) {
      const int64_t tn = tile_at(a, a.torder_h, ix + nst * G64);
      p1s_issue<T>(a, dsm + si * stage_bytes, &bars[si], tn);
      if (stage_v) p1s_issue_vec<T>(a, dsm + si * stage_bytes, &bars[si], tn, it);
    }
    if (!side && lr < rows) aptz = cmad(s_pt[lr], s_z[lr], aptz);   // p~^* z
    if (k > 0) {
      if (tid < kt) {
        const int nel = rows * k;
        int lq = tid / k;
        if (cst) {
          mbar_wait(&bars[2], (par >> 2) & 1u);
          const T *__restrict__ Ct = sC + TRH * k;
          const T *__restrict__ C = sC;
          for (int e = tid; e < nel; e += kt, lq += rstep) {
            const T ct = Ct[e], c = C[e];
            a1 = cmad(ct, s_z[lq], a1);    // conj(c~_{row,j}) z_row
            a2 = cmad(c, s_zt[lq], a2);    // conj(c_{row,j}) z~_row
            a3 = cmad(c, s_pt[lq], a3);    // conj(c_{row,j}) p~_row
            a4 = cmad(ct, s_r[lq], a4);    // conj(c~_{row,j}) r_row   (Q32)
            a5 = cmad(c, s_rt[lq], a5);    // conj(c_{row,j}) r~_row
          }
        } else {
          const T *__restrict__ Ct = a.Ct + row0 * k;
          const T *__restrict__ C = a.C + row0 * k;
#pragma unroll 4
          for (int e = tid; e < nel; e += kt, lq += rstep) {
            const T ct = ldcs(Ct + e), c = ldcs(C + e);
            a1 = cmad(ct, s_z[lq], a1);
            a2 = cmad(c, s_zt[lq], a2);
            a3 = cmad(c, s_pt[lq], a3);
            a4 = cmad(ct, s_r[lq], a4);
            a5 = cmad(c, s_rt[lq], a5);
          }
        }
      } else if (cst) {
        mbar_wait(&bars[2], (par >> 2) & 1u);
      }
      if (cst) par ^= 1u << 2;
      __syncthreads();
    }
  }
}

// Phase-1 block partials -> a.part[o*G + b] (fixed order): o in [0, 3k) the
// coefficient sums a1..a3, 3k p~^*z, [3k+1, 5k+1) the Q32 sums a4, a5.
template <typename T>
__device__ __forceinline__ void p1_partials(const LoopArgs<T> &a, P1Scratch<T> &sc, T *s_w, T a1,
                                            T a2, T a3, T a4, T a5, T aptz) {
  const int tid = threadIdx.x;
  const int k = a.k;
  const int G = red_stride(a), b = red_slot(a);
  const int rstep = k > 0 ? BS / k : 0;
  const int kt = rstep * k;
  if (k > 0) {
    sc.s_red()[tid] = tid < kt ? a1 : zero<T>();
    sc.s_red()[BS + tid] = tid < kt ? a2 : zero<T>();
    sc.s_red()[2 * BS + tid] = tid < kt ? a3 : zero<T>();
  }
  const T bptz = block_sum(aptz, s_w);   // contains __syncthreads
  if (tid < 3 * k) {
    const int ty = tid / k, j = tid % k;
    T s = zero<T>();
    for (int m = 0; m < rstep; ++m) s = add(s, sc.s_red()[ty * BS + j + m * k]);
    a.part[(int64_t)tid * G + b] = s;
  }
  if (tid == 0) a.part[(int64_t)(3 * k) * G + b] = bptz;
  if (k > 0) {   // second round through the same scratch
    __syncthreads();
    sc.s_red()[tid] = tid < kt ? a4 : zero<T>();
    sc.s_red()[BS + tid] = tid < kt ? a5 : zero<T>();
    __syncthreads();
    if (tid < 2 * k) {
      const int ty = tid / k, j = tid % k;
      T s = zero<T>();
      for (int m = 0; m < rstep; ++m) s = add(s, sc.s_red()[ty * BS + j + m * k]);
      a.part[(int64_t)(3 * k + 1 + tid) * G + b] = s;
    }
  }
}

// Phase-2 TMA of one full 256-row tile of the input streams into stage `b`,
// in two parts that arrive separately on the stage's mbarrier (count 2):
//   A: r, r~ (+ x, x~ when x is eager) and the C, C~ rows -- written before
//      the preceding pass 1 started, so pass 2 may issue them before its
//      programmatic-launch wait;
//   B: z, z~ (+ p, p~ when x is eager) -- written by that pass 1.
template <typename T>
__device__ __forceinline__ void p2_issue_a(const LoopArgs<T> &a, T *b, uint64_t *bar, int64_t t,
                                           const T *rold, const T *rtold) {
  const int k = a.k;
  const bool lazy = a.lazy_x != 0;
  const int64_t r0 = t * BS;
  const uint32_t vb = BS * (uint32_t)sizeof(T);
  const uint32_t cbytes = (uint32_t)(BS * k * sizeof(T));
  mbar_expect_tx(bar, (lazy ? 2u : 4u) * vb + 2u * cbytes);
  tma_load_1d(b + 2 * BS, rold + r0, vb, bar);
  tma_load_1d(b + 3 * BS, rtold + r0, vb, bar);
  if (!lazy) {
    tma_load_1d(b + 6 * BS, a.x + r0, vb, bar);
    tma_load_1d(b + 7 * BS, a.xt + r0, vb, bar);
  }
  const int nv = lazy ? 4 : 8;
  if (k > 0) {
    tma_load_1d(b + nv * BS, a.C + r0 * k, cbytes, bar);
    tma_load_1d(b + nv * BS + BS * k, a.Ct + r0 * k, cbytes, bar);
  }
}
template <typename T>
__device__ __forceinline__ void p2_issue_b(const LoopArgs<T> &a, T *b, uint64_t *bar, int64_t t,
                                           const T *pn, const T *ptn) {
  const bool lazy = a.lazy_x != 0;
  const int64_t r0 = t * BS;
  const uint32_t vb = BS * (uint32_t)sizeof(T);
  mbar_expect_tx(bar, (lazy ? 2u : 4u) * vb);
  tma_load_1d(b + 0 * BS, a.z + r0, vb, bar);
  tma_load_1d(b + 1 * BS, a.zt + r0, vb, bar);
  if (!lazy) {
    tma_load_1d(b + 4 * BS, pn + r0, vb, bar);
    tma_load_1d(b + 5 * BS, ptn + r0, vb, bar);
  }
}
template <typename T>
__device__ __forceinline__ void p2_issue(const LoopArgs<T> &a, T *b, uint64_t *bar, int64_t t,
                                         const T *rold, const T *rtold, const T *pn, const T *ptn) {
  p2_issue_a<T>(a, b, bar, t, rold, rtold);
  p2_issue_b<T>(a, b, bar, t, pn, ptn);
}
// elements of one phase-2 stage: 4 (lazy x) or 8 vector tiles + C, C~ tiles
template <typename T> __host__ __device__ __forceinline__ int64_t p2_stage_elems(int k, int lazy) {
  return (int64_t)(lazy ? 4 : 8) * BS + (int64_t)2 * BS * k;
}

// Phase 2 over this block's tiles.  With `staged` the full tiles come through
// two TMA stages at sb (bars2[0..1], each expecting two arrivals, parity bits
// 0..1 of par2); `first` = 0: nothing of the block's first full tile issued
// yet, 1: all of it issued into stage 0, 2: its part A issued.
// Accumulates ρ, ||r||², ||r~||² partials.
template <typename T>
__device__ __forceinline__ void p2_tiles(const LoopArgs<T> &a, bool staged, T *sb, uint64_t *bars2,
                                         uint32_t &par2, int first, int it, T alpha,
                                         const T *s_gam, const T *s_gamt, T &arho, double &an,
                                         double &ant) {
  const int tid = threadIdx.x;
  const int k = a.k;
  const T ca = conj(alpha);
  const int64_t n = a.n;
  const T *__restrict__ rold = a.rring + (int64_t)(it % a.ring) * a.ldr;
  const T *__restrict__ rtold = a.rtring + (int64_t)(it % a.ring) * a.ldr;
  T *__restrict__ rnew = a.rring + (int64_t)((it + 1) % a.ring) * a.ldr;
  T *__restrict__ rtnew = a.rtring + (int64_t)((it + 1) % a.ring) * a.ldr;
  const T *__restrict__ pn = pcol(a, it + 1);
  const T *__restrict__ ptn = ptcol(a, it + 1);
  const int64_t ntiles = (n + BS - 1) / BS;
  const int64_t nfull = n / BS;
  const int64_t G64 = gridDim.x;
  const bool lazy = a.lazy_x != 0;
  auto update_row = [&](int64_t row, T q, T qt, T ro, T rto, T pv, T ptv, T xv, T xtv,
                        const T *cr, const T *ctr) {
    // r_i = r_{i-1} - α_i q_i - C g_{i-1} = r_{i-1} - α_i z_i + C γ_i with
    // q_i = z_i - C ζ_i and the Q32 term; the duals likewise
    T rn = sub(ro, mul(alpha, q));
    T rtn = sub(rto, mul(ca, qt));
    if (k > 0) {
      T d = zero<T>(), dt = zero<T>();
      for (int j = 0; j < k; ++j) {
        d = mad(cr[j], s_gam[j], d);
        dt = mad(ctr[j], s_gamt[j], dt);
      }
      rn = add(rn, d);
      rtn = add(rtn, dt);
    }
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
    // TMA double buffering: each full 256-row tile of the input streams is
    // bulk-copied into shared memory while the previous tile is processed.
    const int64_t stage = p2_stage_elems<T>(k, lazy);
    const int nv = lazy ? 4 : 8;
    if (tid == 0 && (int64_t)blockIdx.x < nfull) {
      if (first == 0) p2_issue<T>(a, sb, &bars2[0], blockIdx.x, rold, rtold, pn, ptn);
      else if (first == 2) p2_issue_b<T>(a, sb, &bars2[0], blockIdx.x, pn, ptn);
    }
    int i = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += G64, ++i) {
      const int si = i & 1;
      const int64_t nxt = tile + G64;
      if (tid == 0 && nxt < nfull)
        p2_issue<T>(a, sb + (si ^ 1) * stage, &bars2[si ^ 1], nxt, rold, rtold, pn, ptn);
      const int64_t row0 = tile * BS;
      if (tile < nfull) {
        mbar_wait(&bars2[si], (par2 >> si) & 1u);
        par2 ^= 1u << si;
        const T *b = sb + si * stage;
        if (lazy)
          update_row(row0 + tid, b[tid], b[BS + tid], b[2 * BS + tid], b[3 * BS + tid], zero<T>(),
                     zero<T>(), zero<T>(), zero<T>(), b + nv * BS + tid * k,
                     b + nv * BS + BS * k + tid * k);
        else
          update_row(row0 + tid, b[tid], b[BS + tid], b[2 * BS + tid], b[3 * BS + tid],
                     b[4 * BS + tid], b[5 * BS + tid], b[6 * BS + tid], b[7 * BS + tid],
                     b + nv * BS + tid * k, b + nv * BS + BS * k + tid * k);
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
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += G64) {
      const int64_t row0 = tile * BS;
      const int rows = (int)min((int64_t)BS, n - row0);
      if (tid < rows) {
        const int64_t row = row0 + tid;
        // all independent loads first (no aliasing stalls behind the stores)
        const T q = ldcs(a.z + row), qt = ldcs(a.zt + row);
        const T ro = ldcs(rold + row), rto = ldcs(rtold + row);
        T pv = zero<T>(), ptv = zero<T>(), xv = zero<T>(), xtv = zero<T>();
        if (!lazy) {
          pv = ldcg(pn + row);
          ptv = ldcg(ptn + row);
          xv = ldcs(a.x + row);
          xtv = ldcs(a.xt + row);
        }
        update_row(row, q, qt, ro, rto, pv, ptv, xv, xtv, a.C + row * k, a.Ct + row * k);
      }
    }
  }
}

// Phase-2 block partials -> a.part[o*G + b], o = 0 (ρ), 1 (||r||²), 2 (||r~||²).
template <typename T>
__device__ __forceinline__ void p2_partials(const LoopArgs<T> &a, T *s_w, T arho, double an,
                                            double ant) {
  const int G = gridDim.x;
  const T b0 = block_sum(arho, s_w);
  double b1 = block_sum(an, reinterpret_cast<double *>(s_w));
  double b2 = block_sum(ant, reinterpret_cast<double *>(s_w));
  if (threadIdx.x == 0) {
    a.part[blockIdx.x] = b0;
    T t1 = zero<T>(), t2 = zero<T>();
    reinterpret_cast<double *>(&t1)[0] = b1;
    reinterpret_cast<double *>(&t2)[0] = b2;
    a.part[G + blockIdx.x] = t1;
    a.part[2 * G + blockIdx.x] = t2;
  }
}

}  // namespace rbicg
