// kernels.cu -- the RBiCG hot loop on sm_100a (Algorithm 2),
// two-kernel form: one launch per reduction point of an iteration, each ending
// in a deterministic grid reduction done by the last block to finish (the
// phase bodies and the reduction leaders are in hot.cuh).
//
// Kernels read the iteration index from the device state, so one captured
// CUDA graph of s iterations is replayed for every cycle; once the state says
// done/paused every kernel is a no-op (exact iteration counts, no host poll).
#include "hot.cuh"
#include <cstdlib>

namespace rbicg {

std::atomic<int64_t> g_launches{0};
thread_local int g_sm_cap = 0;
template <typename T> __device__ void resid_leader(DevState<T> *st, const T *s_fin, int k);
template <typename T> __device__ void init2_leader(const LoopArgs<T> &a, DevState<T> *st, const T *s_fin);
static const bool g_pdl = getenv("RBICG_PDL") ? atoi(getenv("RBICG_PDL")) != 0 : true;


// ============================================================== pass 1
template <typename T, int MINB = 4>
__global__ void __launch_bounds__(BS, MINB) k_pass1(LoopArgs<T> a) {
  __shared__ P1Scratch<T> sc;
  __shared__ Snap<T> sn;
  __shared__ T s_fin[5 * KMAX + 1];
  __shared__ T s_w[BS / 32];
  __shared__ T s_alpha;
  __shared__ int s_last, s_ok;
  __shared__ uint64_t bars[3];
  extern __shared__ __align__(128) unsigned char p1_smem[];
  DevState<T> *st = a.st;
  const int tid = threadIdx.x;
  const int64_t nvis = launch_tiles(a, (a.n + BS - 1) / BS);
  const int64_t G64 = gridDim.x;
  const size_t stage_bytes = p1_stage_bytes<T>(a);
  const int nst = a.p1_stages;
  const bool stage_v = a.staged && a.stage_v;
  // prologue independent of the previous kernel: the first matrix tiles
  if (a.staged) {
    if (tid == 0) {
      mbar_init(&bars[0], stage_v ? 2 : 1);
      mbar_init(&bars[1], stage_v ? 2 : 1);
      mbar_init(&bars[2], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
      for (int q = 0; q < nst; ++q)
        if ((int64_t)blockIdx.x + q * G64 < nvis)
          p1_issue<T>(a, p1_smem + q * stage_bytes, stage_bytes, &bars[q],
                      tile_at(a, a.torder, blockIdx.x + q * G64));
  }
  pdl_wait();
  snap_load(st, a.k, sn);
  if (tid == 0 && stage_v)   // the vector rows depend on the previous kernel
    for (int q = 0; q < nst; ++q)
      if ((int64_t)blockIdx.x + q * G64 < nvis) {
        if (sn.done) mbar_arrive(&bars[q]);
        else p1_issue_vec<T>(a, p1_smem + q * stage_bytes, &bars[q], tile_at(a, a.torder, blockIdx.x + q * G64),
                             sn.iter);
      }
  if (sn.done) {
    if (a.staged)   // drain the copies in flight
      for (int q = 0; q < nst; ++q)
        if ((int64_t)blockIdx.x + q * G64 < nvis) mbar_wait(&bars[q], 0);
    return;
  }
  uint32_t par = 0;
  T a1 = zero<T>(), a2 = zero<T>(), a3 = zero<T>(), a4 = zero<T>(), a5 = zero<T>(), aptz = zero<T>();
  p1_tiles<T, false>(a, p1_smem, bars, par, sc, sn.iter, sn.beta,
                     a.lazy_x && sn.iter == sn.seg_start, a1, a2, a3, a4, a5, aptz);
  pdl_trigger();
  p1_partials<T>(a, sc, s_w, a1, a2, a3, a4, a5, aptz);
  if (interior_done(a) || !last_block(&st->cnt[0], &s_last)) return;
  final_reduce(a.part, p1_nsums(a.k), red_count(a), s_fin, red_stride(a));
  if (tid == 0) st->cnt[0] = 0;
  if (a.dist) {   // local sums -> allreduce -> k_leader1
    for (int o = tid; o < p1_nsums(a.k); o += BS) a.red[o] = s_fin[o];
    return;
  }
  p1_leader<T>(a, st, sn, sn.iter, s_fin, &s_alpha, &s_ok);
}

// pass 1, split form (hot.cuh p1_tiles_split): one thread per row and matrix
template <typename T, int CH>
__global__ void __launch_bounds__(BS, 4) k_pass1s(LoopArgs<T> a) {
  __shared__ P1Scratch<T> sc;
  __shared__ Snap<T> sn;
  __shared__ T s_fin[5 * KMAX + 1];
  __shared__ T s_w[BS / 32];
  __shared__ T s_alpha;
  __shared__ int s_last, s_ok;
  __shared__ uint64_t bars[3];
  extern __shared__ __align__(128) unsigned char p1_smem[];
  DevState<T> *st = a.st;
  const int tid = threadIdx.x;
  const int64_t nvis = launch_tiles(a, (a.n + TRH - 1) / TRH);
  const int64_t G64 = gridDim.x;
  const size_t stage_bytes = p1s_stage_bytes<T>(a);
  const int nst = a.p1_stages;
  const bool stage_v = a.stage_v != 0;
  if (tid == 0) {
    mbar_init(&bars[0], stage_v ? 2 : 1);
    mbar_init(&bars[1], stage_v ? 2 : 1);
    mbar_init(&bars[2], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)   // prologue independent of the previous kernel: first matrix tiles
    for (int q = 0; q < nst; ++q)
      if ((int64_t)blockIdx.x + q * G64 < nvis)
        p1s_issue<T>(a, p1_smem + q * stage_bytes, &bars[q], tile_at(a, a.torder_h, blockIdx.x + q * G64));
  pdl_wait();
  snap_load(st, a.k, sn);
  if (tid == 0 && stage_v)   // the vector rows depend on the previous kernel
    for (int q = 0; q < nst; ++q)
      if ((int64_t)blockIdx.x + q * G64 < nvis) {
        if (sn.done) mbar_arrive(&bars[q]);
        else p1s_issue_vec<T>(a, p1_smem + q * stage_bytes, &bars[q], tile_at(a, a.torder_h, blockIdx.x + q * G64),
                              sn.iter);
      }
  if (sn.done) {
    for (int q = 0; q < nst; ++q)
      if ((int64_t)blockIdx.x + q * G64 < nvis) mbar_wait(&bars[q], 0);
    return;
  }
  uint32_t par = 0;
  T a1 = zero<T>(), a2 = zero<T>(), a3 = zero<T>(), a4 = zero<T>(), a5 = zero<T>(), aptz = zero<T>();
  p1_tiles_split<T, false, CH>(a, p1_smem, bars, par, sc, sn.iter, sn.beta,
                               a.lazy_x && sn.iter == sn.seg_start, a1, a2, a3, a4, a5, aptz);
  pdl_trigger();
  p1_partials<T>(a, sc, s_w, a1, a2, a3, a4, a5, aptz);
  if (interior_done(a) || !last_block(&st->cnt[0], &s_last)) return;
  final_reduce(a.part, p1_nsums(a.k), red_count(a), s_fin, red_stride(a));
  if (tid == 0) st->cnt[0] = 0;
  if (a.dist) {   // local sums -> allreduce -> k_leader1
    for (int o = tid; o < p1_nsums(a.k); o += BS) a.red[o] = s_fin[o];
    return;
  }
  p1_leader<T>(a, st, sn, sn.iter, s_fin, &s_alpha, &s_ok);
}

// ============================================================== pass 2
template <typename T, int MINB = 3>
__global__ void __launch_bounds__(BS, MINB) k_pass2(LoopArgs<T> a, int staged) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ Snap<T> sn;
  __shared__ T s_w[BS / 32];
  __shared__ T s_fin[3];
  __shared__ int s_last;
  __shared__ uint64_t bars2[2];
  DevState<T> *st = a.st;
  const int tid = threadIdx.x;
  T *sb = reinterpret_cast<T *>(smem_raw);
  const bool pre = staged && (int64_t)blockIdx.x < a.n / BS;
  if (staged) {
    if (tid == 0) {
      mbar_init(&bars2[0], 2);
      mbar_init(&bars2[1], 2);
      fence_mbar_init();
    }
    __syncthreads();
    // Part A of the first tile before the programmatic-launch wait: r_{i-1},
    // r~_{i-1} and C, C~ were written before the preceding pass 1 started
    // (it waited for the previous pass 2), so they are complete here.
    if (pre && tid == 0) {
      const int it0 = __ldcg(&st->iter);
      p2_issue_a<T>(a, sb, &bars2[0], blockIdx.x, a.rring + (int64_t)(it0 % a.ring) * a.ldr,
                    a.rtring + (int64_t)(it0 % a.ring) * a.ldr);
    }
  }
  pdl_wait();
  snap_load(st, a.k, sn);
  if (sn.done) {
    if (pre) {   // complete the stage's second arrival and drain the copy
      if (tid == 0) mbar_arrive(&bars2[0]);
      mbar_wait(&bars2[0], 0);
    }
    return;
  }
  uint32_t par2 = 0;
  T arho = zero<T>();
  double an = 0.0, ant = 0.0;
  p2_tiles<T>(a, staged != 0, sb, bars2, par2, pre ? 2 : 0, sn.iter, sn.alpha, sn.gam, sn.gamt,
              arho, an, ant);
  pdl_trigger();
  p2_partials<T>(a, s_w, arho, an, ant);
  if (!last_block(&st->cnt[1], &s_last)) return;
  final_reduce(a.part, 3, gridDim.x, s_fin);
  if (tid == 0) st->cnt[1] = 0;
  if (a.dist) {   // local sums -> allreduce -> k_leader2
    for (int o = tid; o < 3; o += BS) a.red[o] = s_fin[o];
    return;
  }
  p2_leader<T>(a, st, sn, sn.iter, s_fin);
}

// ============================================================== split-preconditioned form (NEXT-4)
// Â = L^{-1} A U^{-1} is not a SELL matrix, so with a preconditioner the
// iteration's first phase is split: k_pc_pupdate (p_i = r_{i-1} + β p_{i-1},
// duals; also into fixed buffers for the captured operator launches), then
// z_i = Â p_i, z~_i = Â^* p~_i (precond.cu: triangular solves and the SpMV
// pair), then k_pc_proj (the pass-1 reduction without the SpMV: C~^*z, C^*z~,
// C^*p~, p~^*z and the Q32 sums, the same leader), then pass 2 unchanged.
template <typename T>
__global__ void __launch_bounds__(BS) k_pc_pupdate(LoopArgs<T> a, T *pfix, T *ptfix) {
  __shared__ Snap<T> sn;
  snap_load(a.st, a.k, sn);
  if (sn.done) return;
  const int it = sn.iter;
  const T beta = sn.beta, cb = conj(sn.beta);
  const T *r = a.rring + (int64_t)(it % a.ring) * a.ldr;
  const T *rt = a.rtring + (int64_t)(it % a.ring) * a.ldr;
  const T *po = pcol(a, it), *pto = ptcol(a, it);
  T *pn = pcol(a, it + 1), *ptn = ptcol(a, it + 1);
  for (int64_t row = blockIdx.x * (int64_t)BS + threadIdx.x; row < a.n; row += (int64_t)gridDim.x * BS) {
    const T v = mad(beta, po[row], r[row]);
    const T vt = mad(cb, pto[row], rt[row]);
    pn[row] = v;
    ptn[row] = vt;
    pfix[row] = v;
    ptfix[row] = vt;
  }
}

template <typename T>
__global__ void __launch_bounds__(BS) k_pc_proj(LoopArgs<T> a) {
  __shared__ P1Scratch<T> sc;
  __shared__ Snap<T> sn;
  __shared__ T s_v[5 * BS];   // z, z~, p~, r, r~ rows of the tile
  __shared__ T s_fin[5 * KMAX + 1];
  __shared__ T s_w[BS / 32];
  __shared__ T s_alpha;
  __shared__ int s_last, s_ok;
  DevState<T> *st = a.st;
  snap_load(st, a.k, sn);
  if (sn.done) return;
  const int tid = threadIdx.x, k = a.k, it = sn.iter;
  const int64_t n = a.n;
  const T *r = a.rring + (int64_t)(it % a.ring) * a.ldr;
  const T *rt = a.rtring + (int64_t)(it % a.ring) * a.ldr;
  const T *ptn = ptcol(a, it + 1);
  const int rstep = k > 0 ? BS / k : 0;
  const int kt = rstep * k;
  T a1 = zero<T>(), a2 = zero<T>(), a3 = zero<T>(), a4 = zero<T>(), a5 = zero<T>(), aptz = zero<T>();
  const int64_t ntiles = (n + BS - 1) / BS;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * BS;
    const int rows = (int)min((int64_t)BS, n - row0);
    if (tid < rows) {
      const int64_t row = row0 + tid;
      const T z = a.z[row], zt = a.zt[row], pt = ptn[row];
      s_v[tid] = z;
      s_v[BS + tid] = zt;
      s_v[2 * BS + tid] = pt;
      s_v[3 * BS + tid] = r[row];
      s_v[4 * BS + tid] = rt[row];
      aptz = cmad(pt, z, aptz);   // (p~_i, z_i)
    }
    if (k > 0) {
      __syncthreads();
      if (tid < kt) {
        const int nel = rows * k;
        const T *__restrict__ Ct = a.Ct + row0 * k;
        const T *__restrict__ C = a.C + row0 * k;
        int lr = tid / k;
        for (int e = tid; e < nel; e += kt, lr += rstep) {
          const T ct = Ct[e], c = C[e];
          a1 = cmad(ct, s_v[lr], a1);            // C~^* z
          a2 = cmad(c, s_v[BS + lr], a2);        // C^* z~
          a3 = cmad(c, s_v[2 * BS + lr], a3);    // C^* p~
          a4 = cmad(ct, s_v[3 * BS + lr], a4);   // C~^* r   (Q32)
          a5 = cmad(c, s_v[4 * BS + lr], a5);    // C^* r~
        }
      }
      __syncthreads();
    }
  }
  p1_partials<T>(a, sc, s_w, a1, a2, a3, a4, a5, aptz);
  if (!last_block(&st->cnt[0], &s_last)) return;
  final_reduce(a.part, p1_nsums(k), gridDim.x, s_fin);
  if (tid == 0) st->cnt[0] = 0;
  p1_leader<T>(a, st, sn, it, s_fin, &s_alpha, &s_ok);
}

// ============================================================== row-partitioned form
// The scalar steps after the allreduce of the block sums (one block each);
// every rank runs them on identical global sums, so the scalars stay
// replicated.
template <typename T>
__global__ void __launch_bounds__(BS) k_leader1(LoopArgs<T> a) {
  __shared__ Snap<T> sn;
  __shared__ T s_fin[5 * KMAX + 1];
  __shared__ T s_alpha;
  __shared__ int s_ok;
  snap_load(a.st, a.k, sn);
  if (sn.done) return;
  for (int o = threadIdx.x; o < p1_nsums(a.k); o += BS) s_fin[o] = ldcg(a.red + o);
  __syncthreads();
  p1_leader<T>(a, a.st, sn, sn.iter, s_fin, &s_alpha, &s_ok);
}
template <typename T>
__global__ void __launch_bounds__(BS) k_leader2(LoopArgs<T> a) {
  __shared__ Snap<T> sn;
  __shared__ T s_fin[3];
  snap_load(a.st, a.k, sn);
  if (sn.done) return;
  if (threadIdx.x < 3) s_fin[threadIdx.x] = ldcg(a.red + threadIdx.x);
  __syncthreads();
  p2_leader<T>(a, a.st, sn, sn.iter, s_fin);
}
template <typename T>
__global__ void __launch_bounds__(BS) k_leader_resid(LoopArgs<T> a, int coef) {
  __shared__ T s_fin[4 + 2 * KMAX];
  const int k = coef ? a.k : 0;
  for (int o = threadIdx.x; o < 4 + 2 * k; o += BS) s_fin[o] = ldcg(a.red + o);
  __syncthreads();
  resid_leader<T>(a.st, s_fin, k);
}
template <typename T>
__global__ void __launch_bounds__(BS) k_leader_init2(LoopArgs<T> a) {
  __shared__ T s_fin[3];
  if (threadIdx.x < 3) s_fin[threadIdx.x] = ldcg(a.red + threadIdx.x);
  __syncthreads();
  init2_leader<T>(a, a.st, s_fin);
}

// Halo of the gathered vectors of iteration `it` (state): r_it, p_it, r~_it,
// p~_it (own rows send_idx -> sendbuf; received ghosts -> the ghost rows
// [n, n + nghost) of the same columns).  Fixed buffer addresses, so the
// exchange between them can be captured in the cycle's graph.
template <typename T>
__global__ void k_halo_pack_loop(LoopArgs<T> a, const int32_t *idx, int64_t nsend, T *sendbuf) {
  const int it = __ldcg(&a.st->iter);
  const T *v[4] = {a.rring + (int64_t)(it % a.ring) * a.ldr, pcol(a, it),
                   a.rtring + (int64_t)(it % a.ring) * a.ldr, ptcol(a, it)};
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nsend;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = idx[j];
#pragma unroll
    for (int q = 0; q < 4; ++q) sendbuf[q * nsend + j] = v[q][r];
  }
}
template <typename T>
__global__ void k_halo_unpack_loop(LoopArgs<T> a, const T *recvbuf, int64_t nghost) {
  const int it = __ldcg(&a.st->iter);
  T *v[4] = {a.rring + (int64_t)(it % a.ring) * a.ldr, pcol(a, it),
             a.rtring + (int64_t)(it % a.ring) * a.ldr, ptcol(a, it)};
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nghost;
       g += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q][a.n + g] = recvbuf[q * nghost + g];
  }
}
// rows idx of an n x k row-major block -> out (k values per row)
template <typename T>
__global__ void k_pack_rows(const T *X, int k, const int32_t *idx, int64_t cnt, T *out) {
  const int64_t tot = cnt * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = X[(int64_t)idx[e / k] * k + e % k];
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
  if (tid == 0) st->cnt[2] = 0;
  if (a.dist) {   // local sums -> allreduce -> k_leader_resid
    for (int o = tid; o < 4 + 2 * k; o += BS) a.red[o] = s_fin[o];
    return;
  }
  resid_leader<T>(st, s_fin, k);
}

template <typename T>
__device__ void resid_leader(DevState<T> *st, const T *s_fin, int k) {
  if (threadIdx.x == 0) {
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
  if (tid == 0) st->cnt[3] = 0;
  if (a.dist) {
    for (int o = tid; o < 3; o += BS) a.red[o] = s_fin[o];
    return;
  }
  init2_leader<T>(a, st, s_fin);
}

template <typename T>
__device__ void init2_leader(const LoopArgs<T> &a, DevState<T> *st, const T *s_fin) {
  if (threadIdx.x == 0) {
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

// ============================================================== fused form
// One kernel per iteration while no recycle space is active (k = 0; DESIGN §6
// "fused iteration"; oracle variant "lookahead").  K(i) completes iteration
// i-1 and runs the SpMV pair of iteration i:
//   r_{i-1} = r_{i-2} - α_{i-1} z_{i-1},   p_i = r_{i-1} + β_{i-1} p_{i-1},
//   z_i = A p_i   (r_{i-1}, p_i formed on the fly in the gather from the stored
//                  r_{i-2}, z_{i-1}, p_{i-1} of the neighbour columns)
// and the duals; one reduction gives ρ_{i-1} (exact), ||r_{i-1}||, ||r~_{i-1}||
// (the stop test of iteration i-1), σ_i = (p~_i, z_i), and (r~_{i-1}, z_i),
// (z~_i, r_{i-1}), (z~_i, z_i) for ρ_i's one-step expansion, which gives β_i
// with α_i = ρ_{i-1}/σ_i.  r_{i-1} lands in ring column i-1 (K(1) reads r_0
// from column 0 and writes nothing there).
constexpr int NFUSED = 7;
// The gathered (z, p) of column c in one load: 16 bytes for real data
// (LDG.128), 32 bytes for complex (a 256-bit LDG); r comes from the ring
// column.  (Real nodes {r, z, p, pad} read as one 256-bit load measured
// slower: C2 59.8 vs 46.4 us per iteration.)
template <typename T> struct RZP { T r, z, p; };
__device__ __forceinline__ void ld256(const void *p, double &a, double &b, double &c, double &d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}
__device__ __forceinline__ void st256(void *p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
__device__ __forceinline__ RZP<double> ld_node(const double *nodes, const double *ring, int64_t c) {
  const double2 v = __ldg(reinterpret_cast<const double2 *>(nodes) + c);
  return RZP<double>{ldg(ring + c), v.x, v.y};
}
// (all four words are consumed by every caller: ptxas masks a 256-bit load
// whose words are not all used, and masks finer than 128 bits faulted on B200
// with cudaErrorInvalidAddressSpace)
__device__ __forceinline__ RZP<zc> ld_node(const zc *nodes, const zc *ring, int64_t c) {
  double zx, zy, px, py;
  ld256(nodes + 2 * c, zx, zy, px, py);
  return RZP<zc>{ldg(ring + c), mk(zx, zy), mk(px, py)};
}
__device__ __forceinline__ void st_node(double *nodes, int64_t c, double, double z, double p) {
  reinterpret_cast<double2 *>(nodes)[c] = make_double2(z, p);
}
__device__ __forceinline__ void st_node(zc *nodes, int64_t c, zc, zc z, zc p) {
  st256(nodes + 2 * c, z.x, z.y, p.x, p.y);
}
// staged copy of the tile's (r, {z, p}) rows [lo, lo + cnt) (fused form,
// VS): columns inside come from shared memory, the others from global memory
template <typename T> struct VStage {
  const T *r, *nd, *rt, *ndt;
  int lo, cnt;
};
template <typename T>
__device__ __forceinline__ RZP<T> node_at(const T *__restrict__ nd, const T *__restrict__ r,
                                          const T *__restrict__ snd, const T *__restrict__ sr, int lo,
                                          int cnt, int c) {
  const int q = c - lo;
  if ((unsigned)q < (unsigned)cnt) return RZP<T>{sr[q], snd[2 * q], snd[2 * q + 1]};
  return ld_node(nd, r, c);
}
template <typename T, bool VS>
__device__ __forceinline__ void fused_pair_smem(const int32_t *__restrict__ cA, const T *__restrict__ vA,
                                                int wA, const int32_t *__restrict__ cH,
                                                const T *__restrict__ vH, int wH,
                                                const T *__restrict__ r, const T *__restrict__ nd,
                                                const T *__restrict__ rt, const T *__restrict__ ndt,
                                                const VStage<T> &vs,
                                                T malpha, T beta, T cmalpha, T cb, T &zo, T &zto) {
  zo = zero<T>();
  zto = zero<T>();
  const int wm = max(wA, wH);
  for (int j0 = 0; j0 < wm; j0 += 4) {
    int ca[4], ch[4];
    T va[4], vh[4];
    RZP<T> xa[4], xh[4];
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
      if (VS) {
        xa[q] = node_at(nd, r, vs.nd, vs.r, vs.lo, vs.cnt, ca[q]);
        xh[q] = node_at(ndt, rt, vs.ndt, vs.rt, vs.lo, vs.cnt, ch[q]);
      } else {
        xa[q] = ld_node(nd, r, ca[q]);
        xh[q] = ld_node(ndt, rt, ch[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      zo = mad(va[q], mad(beta, xa[q].p, mad(malpha, xa[q].z, xa[q].r)), zo);
      zto = mad(vh[q], mad(cb, xh[q].p, mad(cmalpha, xh[q].z, xh[q].r)), zto);
    }
  }
}

// The scalar step of K(i) (one thread): completes iteration i-1 (record,
// stop test, breakdowns, cycle pause) and prepares α_i, β_i (look-ahead ρ_i).
// The device-state fields the fused leader reads, loaded at kernel start (in
// parallel, off the tail: a dependent chain of L2 loads in the one leader
// thread sat on the critical path of every iteration)
template <typename T> struct FSnap {
  T sigma, rho;
  double tolb, tolbt;
  int force, max_itn, stop_at;
};
template <typename T>
__device__ __forceinline__ void fsnap_load(const DevState<T> *st, FSnap<T> &f) {
  f.sigma = ldcg(&st->sigma);
  f.rho = ldcg(&st->rho);
  f.tolb = __ldcg(&st->tolb);
  f.tolbt = __ldcg(&st->tolbt);
  f.force = __ldcg(&st->force);
  f.max_itn = __ldcg(&st->max_itn);
  f.stop_at = __ldcg(&st->stop_at);
}
template <typename T>
__device__ __forceinline__ void fused_leader(const LoopArgs<T> &a, DevState<T> *st, const T *s_fin, int i,
                                             T alpha, T beta, const FSnap<T> &fs) {
  const T rho_prev = s_fin[0];
  const double rn = sqrt(re(s_fin[1])), rtn = sqrt(re(s_fin[2]));
  const T sigma = s_fin[3];
  int done = 0, status = RBICG_OK;
  if (i >= 2) {   // iteration i-1 completes here
    const int m = i - 1;
    IterRec<T> rec;
    rec.alpha = alpha;
    rec.beta = beta;
    rec.rho = rho_prev;
    rec.sigma = fs.sigma;
    rec.rnorm = rn;
    rec.rtnorm = rtn;
    a.hist[m] = rec;
    const int force = fs.force;
    const bool conv = !force && rn <= fs.tolb && rtn <= fs.tolbt;
    if (conv) {
      done = 1;
    } else if (iszero(rho_prev) || !finite(divd(rho_prev, fs.rho))) {
      done = 1;
      status = RBICG_BREAKDOWN_SERIOUS;
    } else if (m >= fs.max_itn) {
      done = 1;
      status = force ? RBICG_OK : RBICG_MAXITER;
    } else if (m == fs.stop_at) {
      done = 2;
    }
    st->iter = m;
    st->rnorm = rn;
    st->rtnorm = rtn;
    st->rho = rho_prev;
  }
  // iteration i's scalars (kept also when finishing: a retry resumes with them)
  const T alpha_i = divd(rho_prev, sigma);
  if (!done && (iszero(sigma) || !finite(alpha_i))) {
    done = 1;
    status = RBICG_BREAKDOWN_SECOND;
  }
  // ρ_i ≈ ρ_{i-1} - α_i (r~, z) - α_i (z~, r) + α_i² (z~, z)
  const T rho_ext = add(sub(sub(rho_prev, mul(alpha_i, s_fin[4])), mul(alpha_i, s_fin[5])),
                        mul(mul(alpha_i, alpha_i), s_fin[6]));
  {   // flag a cancelling expansion (near-breakdown regime): β_i is then inexact
    const double aa = sqrt(abs2(alpha_i));
    const double mag = sqrt(abs2(rho_prev)) + aa * (sqrt(abs2(s_fin[4])) + sqrt(abs2(s_fin[5]))) +
                       aa * aa * sqrt(abs2(s_fin[6]));
    if (sqrt(abs2(rho_ext)) < 1e3 * 2.220446049250313e-16 * mag) st->la_cancel += 1;
  }
  st->alpha = alpha_i;
  st->beta = divd(rho_ext, rho_prev);
  st->sigma = sigma;
  st->kidx = i;
  if (done) {
    st->status = status;
    st->done = done;
  }
}

// Banded A with one shared column array (DC): the tile's columns arrive as
// int16 deltas col - row (2 bytes per nonzero instead of 4); A and A^* share
// them, so one delta serves both gathers of a nonzero slot.
template <typename T> __host__ __device__ __forceinline__ size_t dc_mat_bytes(const LoopArgs<T> &a) {
  return (size_t)a.tile_max * (2 + 2 * sizeof(T));
}
template <typename T>
__device__ __forceinline__ void fused_issue_dc(const LoopArgs<T> &a, unsigned char *stage, uint64_t *bar,
                                               int64_t t) {
  const int TM = a.tile_max;
  int16_t *dA = reinterpret_cast<int16_t *>(stage);
  T *vA = reinterpret_cast<T *>(stage + (size_t)TM * 2);
  T *vH = vA + TM;
  const int64_t ns = a.A.nslices;
  const int64_t s0 = t * (BS / 32), s1 = min(s0 + BS / 32, ns);
  const int64_t oA = a.A.sptr[s0], eA = a.A.sptr[s1];
  const uint32_t nA = (uint32_t)(eA - oA);
  mbar_expect_tx(bar, nA * (2u + 2u * (uint32_t)sizeof(T)));
  if (!nA) return;
  const uint64_t pol = policy_evict_first();
  tma_load_1d_hint(dA, a.dcols + oA, nA * 2u, bar, pol);
  tma_load_1d_hint(vA, reinterpret_cast<const T *>(a.A.vals) + oA, nA * (uint32_t)sizeof(T), bar, pol);
  tma_load_1d_hint(vH, reinterpret_cast<const T *>(a.AH.vals) + oA, nA * (uint32_t)sizeof(T), bar, pol);
}
template <typename T>
__device__ __forceinline__ void fused_pair_dc(const int16_t *__restrict__ dA, const T *__restrict__ vA,
                                              const T *__restrict__ vH, int w, int row,
                                              const T *__restrict__ r, const T *__restrict__ nd,
                                              const T *__restrict__ rt, const T *__restrict__ ndt,
                                              T malpha, T beta, T cmalpha, T cb, T &zo, T &zto) {
  zo = zero<T>();
  zto = zero<T>();
  for (int j0 = 0; j0 < w; j0 += 4) {
    int cc[4];
    T va[4], vh[4];
    RZP<T> xa[4], xh[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int jj = j0 + q;
      const bool in = jj < w;
      cc[q] = in ? row + (int)dA[jj * 32] : 0;
      va[q] = in ? vA[jj * 32] : zero<T>();
      vh[q] = in ? vH[jj * 32] : zero<T>();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      xa[q] = ld_node(nd, r, cc[q]);
      xh[q] = ld_node(ndt, rt, cc[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      zo = mad(va[q], mad(beta, xa[q].p, mad(malpha, xa[q].z, xa[q].r)), zo);
      zto = mad(vh[q], mad(cb, xh[q].p, mad(cmalpha, xh[q].z, xh[q].r)), zto);
    }
  }
}

constexpr int TRV = BS + 4;   // staged vector rows per tile: the tile and 2 rows each side
template <typename T> __host__ __device__ __forceinline__ size_t fused_vec_bytes() {
  return (size_t)6 * TRV * sizeof(T);   // r, {z, p} (2), r~, {z~, p~} (2)
}
// vector part of stage `stage` for tile t: the ranges [lo, lo + cnt) of
// r_{i-2} and of the {z, p} nodes (both sides); cnt even so every copy is a
// multiple of 16 bytes
__device__ __forceinline__ void fused_vrange(int64_t t, int64_t n, int &lo, int &cnt) {
  const int64_t a0 = max((int64_t)0, t * BS - 2), a1 = min(n, t * BS + BS + 2);
  lo = (int)a0;
  cnt = (int)((a1 - a0) & ~(int64_t)1);
}
template <typename T>
__device__ __forceinline__ void fused_issue_vec(unsigned char *vb, uint64_t *bar, int64_t t, int64_t n,
                                                const T *r, const T *nd, const T *rt, const T *ndt) {
  int lo, cnt;
  fused_vrange(t, n, lo, cnt);
  T *d = reinterpret_cast<T *>(vb);
  const uint32_t rb = (uint32_t)(cnt * sizeof(T)), nb = 2 * rb;
  mbar_expect_tx(bar, 2 * (rb + nb));
  tma_load_1d(d, r + lo, rb, bar);
  tma_load_1d(d + TRV, nd + 2 * (int64_t)lo, nb, bar);
  tma_load_1d(d + 3 * TRV, rt + lo, rb, bar);
  tma_load_1d(d + 4 * TRV, ndt + 2 * (int64_t)lo, nb, bar);
}

template <typename T, int MINB, bool VS = false, bool DC = false>
__global__ void __launch_bounds__(BS, MINB) k_fused(LoopArgs<T> a) {
  __shared__ T s_fin[NFUSED + 1];
  __shared__ T s_w[NFUSED][BS / 32];
  __shared__ int s_last;
  __shared__ uint64_t bars[2];
  __shared__ T s_ab[2];
  __shared__ int s_i[5];   // kidx, done, seg_start, iter, stop_at
  __shared__ FSnap<T> s_fs;
  extern __shared__ __align__(128) unsigned char f_smem[];
  DevState<T> *st = a.st;
  const int tid = threadIdx.x;
  const int64_t n = a.n;
  const int64_t ntiles = launch_tiles(a, (n + BS - 1) / BS);   // visits of this launch
  const int64_t G64 = gridDim.x;
  // this CTA's visits: grid-strided (b, b + G, ...) or one contiguous run
  // (a.tile_contig: neighbouring tiles' vector rows stay in this SM's L1);
  // visit ix is tile tile_at(ix) (natural order on one GPU)
  const int64_t t0 = a.tile_contig ? (ntiles * blockIdx.x) / G64 : blockIdx.x;
  const int64_t t1 = a.tile_contig ? (ntiles * (blockIdx.x + 1)) / G64 : ntiles;
  const int64_t tstep = a.tile_contig ? 1 : G64;
  const size_t mat_bytes = DC ? dc_mat_bytes<T>(a) : p1_mat_bytes<T>(a);
  const size_t stage_bytes = mat_bytes + (VS ? fused_vec_bytes<T>() : 0);
  const int nst = a.p1_stages;
  if (tid == 0) {   // VS: two arrivals per stage (matrix part, vector part)
    mbar_init(&bars[0], VS ? 2 : 1);
    mbar_init(&bars[1], VS ? 2 : 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < nst; ++q)
      if (t0 + q * tstep < t1) {
        const int64_t tq = tile_at(a, a.torder, t0 + q * tstep);
        if (DC) fused_issue_dc<T>(a, f_smem + q * stage_bytes, &bars[q], tq);
        else p1_issue<T>(a, f_smem + q * stage_bytes, stage_bytes, &bars[q], tq);
      }
  pdl_wait();
  if (tid == 0) {
    s_i[0] = __ldcg(&st->kidx);
    s_i[1] = __ldcg(&st->done);
    s_i[2] = __ldcg(&st->seg_start);
    s_ab[0] = ldcg(&st->alpha);
    s_ab[1] = ldcg(&st->beta);
  }
  if (tid == 32) fsnap_load(st, s_fs);
  __syncthreads();
  if (s_i[1]) {   // finished or paused: drain the copies in flight
    for (int q = 0; q < nst; ++q)
      if (t0 + q * tstep < t1) {
        if (VS && tid == 0) mbar_arrive(&bars[q]);   // the vector part never comes
        mbar_wait(&bars[q], 0);
      }
    return;
  }
  const int i = s_i[0] + 1;
  const T alpha = s_ab[0], beta = s_ab[1];
  const T malpha = neg(alpha), cmalpha = conj(malpha), cb = conj(beta);
  const T *__restrict__ r = a.rring + (int64_t)(max(i - 2, 0) % a.ring) * a.ldr;
  const T *__restrict__ rt = a.rtring + (int64_t)(max(i - 2, 0) % a.ring) * a.ldr;
  T *__restrict__ rw = a.rring + (int64_t)((i - 1) % a.ring) * a.ldr;
  T *__restrict__ rtw = a.rtring + (int64_t)((i - 1) % a.ring) * a.ldr;
  const T *__restrict__ zpo = a.zp[(i - 1) & 1];
  const T *__restrict__ ztpo = a.ztp[(i - 1) & 1];
  T *__restrict__ zpn = a.zp[i & 1];
  T *__restrict__ ztpn = a.ztp[i & 1];
  const bool wr = i >= 2;   // K(1): r_0 is already in column 0
  const bool segcopy = a.lazy_x && i - 2 == s_i[2];
  T *__restrict__ pseg = a.pseg[(s_i[2] / a.cyc) & 1];
  T *__restrict__ ptseg = a.ptseg[(s_i[2] / a.cyc) & 1];
  if (VS && tid == 0)   // the vector parts of the first tiles (written by the previous kernel)
    for (int q = 0; q < nst; ++q)
      if (t0 + q * tstep < t1)
        fused_issue_vec<T>(f_smem + q * stage_bytes + mat_bytes, &bars[q], tile_at(a, a.torder, t0 + q * tstep),
                           n, r, zpo, rt, ztpo);
  T acc[NFUSED];
#pragma unroll
  for (int o = 0; o < NFUSED; ++o) acc[o] = zero<T>();
  const int TM = a.tile_max;
  const int64_t ns = a.A.nslices;
  uint32_t par = 0;
  int it = 0;
  for (int64_t ix = t0; ix < t1; ix += tstep, ++it) {
    const int64_t tile = tile_at(a, a.torder, ix);
    const int64_t row0 = tile * BS;
    const int rows = (int)min((int64_t)BS, n - row0);
    const int si = nst == 2 ? (it & 1) : 0;
    const unsigned char *base = f_smem + si * stage_bytes;
    const int32_t *scA = reinterpret_cast<const int32_t *>(base);
    const int32_t *scH = a.shared_cols ? scA : scA + TM;
    const T *svA = reinterpret_cast<const T *>(scA + p1_ncols(a) * TM);
    const T *svH = svA + TM;
    const int64_t sl = (row0 >> 5) + (tid >> 5);
    const int64_t slc = min(sl, ns - 1);
    const int64_t bA = a.A.sptr[tile * (BS / 32)], bH = a.AH.sptr[tile * (BS / 32)];
    const int64_t oA = a.A.sptr[slc], oH = a.AH.sptr[slc];
    const int wA = (int)((a.A.sptr[slc + 1] - oA) >> 5), wH = (int)((a.AH.sptr[slc + 1] - oH) >> 5);
    const int lane = tid & 31;
    mbar_wait(&bars[si], (par >> si) & 1u);
    par ^= 1u << si;
    VStage<T> vs{};
    if (VS) {
      const T *vb = reinterpret_cast<const T *>(base + mat_bytes);
      vs.r = vb;
      vs.nd = vb + TRV;
      vs.rt = vb + 3 * TRV;
      vs.ndt = vb + 4 * TRV;
      fused_vrange(tile, n, vs.lo, vs.cnt);
    }
    if (tid < rows) {
      const int64_t row = row0 + tid;
      T z, zt;
      if (DC) {
        const int16_t *sdc = reinterpret_cast<const int16_t *>(base);
        const T *dvA = reinterpret_cast<const T *>(base + (size_t)TM * 2);
        fused_pair_dc<T>(sdc + (oA - bA) + lane, dvA + (oA - bA) + lane, dvA + TM + (oA - bA) + lane, wA,
                         (int)row, r, zpo, rt, ztpo, malpha, beta, cmalpha, cb, z, zt);
      } else {
        fused_pair_smem<T, VS>(scA + (oA - bA) + lane, svA + (oA - bA) + lane, wA,
                               scH + (oH - bH) + lane, svH + (oH - bH) + lane, wH, r, zpo, rt, ztpo, vs,
                               malpha, beta, cmalpha, cb, z, zt);
      }
      const RZP<T> o = VS ? node_at(zpo, r, vs.nd, vs.r, vs.lo, vs.cnt, (int)row) : ld_node(zpo, r, row);
      const RZP<T> ot = VS ? node_at(ztpo, rt, vs.ndt, vs.rt, vs.lo, vs.cnt, (int)row) : ld_node(ztpo, rt, row);
      const T rr = mad(malpha, o.z, o.r);
      const T rtr = mad(cmalpha, ot.z, ot.r);
      const T pr = mad(beta, o.p, rr);
      const T ptr = mad(cb, ot.p, rtr);
      if (segcopy) {   // lazy x: p_a of the open segment (a = i - 2), before it is overwritten
        const RZP<T> q = ld_node(zpn, r, row), qt = ld_node(ztpn, rt, row);
        const T z0 = zero<T>();   // (z consumed too: a whole-node load, see ld_node)
        pseg[row] = mad(z0, q.z, q.p);
        ptseg[row] = mad(z0, qt.z, qt.p);
      }
      if (wr) {
        rw[row] = rr;
        rtw[row] = rtr;
      }
      st_node(zpn, row, rr, z, pr);
      st_node(ztpn, row, rtr, zt, ptr);
      acc[0] = cmad(rtr, rr, acc[0]);      // ρ_{i-1}
      acc[1] = add(acc[1], mk_re<T>(abs2(rr)));
      acc[2] = add(acc[2], mk_re<T>(abs2(rtr)));
      acc[3] = cmad(ptr, z, acc[3]);       // σ_i
      acc[4] = cmad(rtr, z, acc[4]);       // (r~_{i-1}, z_i)
      acc[5] = cmad(zt, rr, acc[5]);       // (z~_i, r_{i-1})
      acc[6] = cmad(zt, z, acc[6]);        // (z~_i, z_i)
    }
    __syncthreads();   // stage si consumed
    if (tid == 0 && ix + nst * tstep < t1) {
      const int64_t tn = tile_at(a, a.torder, ix + nst * tstep);
      if (DC) fused_issue_dc<T>(a, f_smem + si * stage_bytes, &bars[si], tn);
      else p1_issue<T>(a, f_smem + si * stage_bytes, stage_bytes, &bars[si], tn);
      if (VS) fused_issue_vec<T>(f_smem + si * stage_bytes + mat_bytes, &bars[si], tn, n, r, zpo, rt, ztpo);
    }
  }
  pdl_trigger();
  // block partials (fixed order) -> part[o * G + b]
  const int w = tid >> 5, l = tid & 31;
#pragma unroll
  for (int o = 0; o < NFUSED; ++o) {
    const T v = warp_sum(acc[o]);
    if (l == 0) s_w[o][w] = v;
  }
  __syncthreads();
  if (tid < NFUSED) {
    T sum = zero<T>();
    for (int q = 0; q < BS / 32; ++q) sum = add(sum, s_w[tid][q]);
    a.part[(int64_t)tid * red_stride(a) + red_slot(a)] = sum;
  }
  if (interior_done(a) || !last_block(&st->cnt[0], &s_last)) return;
  final_reduce(a.part, NFUSED, red_count(a), s_fin, red_stride(a));
  if (tid == 0) st->cnt[0] = 0;
  if (a.dist) {   // local sums -> allreduce -> k_leader_fused
    if (tid < NFUSED) a.red[tid] = s_fin[tid];
    return;
  }
  if (tid == 0) fused_leader<T>(a, st, s_fin, i, alpha, beta, s_fs);
}

// partitioned form: the scalar step after the allreduce of the block sums
template <typename T>
__global__ void __launch_bounds__(32) k_leader_fused(LoopArgs<T> a) {
  DevState<T> *st = a.st;
  if (threadIdx.x != 0 || __ldcg(&st->done)) return;
  T s_fin[NFUSED];
  for (int o = 0; o < NFUSED; ++o) s_fin[o] = ldcg(a.red + o);
  FSnap<T> fs;
  fsnap_load(st, fs);
  fused_leader<T>(a, st, s_fin, __ldcg(&st->kidx) + 1, ldcg(&st->alpha), ldcg(&st->beta), fs);
}

// halo of the fused form: the own rows of r_{i-2}, z_{i-1}, p_{i-1} and the
// duals that the neighbours gather, into ghost rows [n, nx)
template <typename T>
__global__ void k_halo_pack_fused(LoopArgs<T> a, const int32_t *idx, int64_t nsend, T *sendbuf) {
  const int i = __ldcg(&a.st->kidx) + 1;
  if (__ldcg(&a.st->done)) return;
  const T *r = a.rring + (int64_t)(max(i - 2, 0) % a.ring) * a.ldr;
  const T *rt = a.rtring + (int64_t)(max(i - 2, 0) % a.ring) * a.ldr;
  const T *nd = a.zp[(i - 1) & 1], *ndt = a.ztp[(i - 1) & 1];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nsend;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx[j];
    sendbuf[0 * nsend + j] = r[row];
    sendbuf[1 * nsend + j] = nd[2 * row];
    sendbuf[2 * nsend + j] = nd[2 * row + 1];
    sendbuf[3 * nsend + j] = rt[row];
    sendbuf[4 * nsend + j] = ndt[2 * row];
    sendbuf[5 * nsend + j] = ndt[2 * row + 1];
  }
}
template <typename T>
__global__ void k_halo_unpack_fused(LoopArgs<T> a, const T *recvbuf, int64_t nghost) {
  const int i = __ldcg(&a.st->kidx) + 1;
  if (__ldcg(&a.st->done)) return;
  T *r = a.rring + (int64_t)(max(i - 2, 0) % a.ring) * a.ldr;
  T *rt = a.rtring + (int64_t)(max(i - 2, 0) % a.ring) * a.ldr;
  T *nd = a.zp[(i - 1) & 1], *ndt = a.ztp[(i - 1) & 1];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nghost;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = a.n + g;
    r[row] = recvbuf[0 * nghost + g];
    nd[2 * row] = recvbuf[1 * nghost + g];
    nd[2 * row + 1] = recvbuf[2 * nghost + g];
    rt[row] = recvbuf[3 * nghost + g];
    ndt[2 * row] = recvbuf[4 * nghost + g];
    ndt[2 * row + 1] = recvbuf[5 * nghost + g];
  }
}

// ------------------------------------------------------------------ fused form, k > 0
// K(i) with a recycle space (the oracle's "lookahead" variant with the
// projections and Q32): K(i) completes iteration i-1 and starts iteration i,
//   r_{i-1} = r_{i-2} - α_{i-1} z_{i-1} + C γ_{i-1}   (γ = αζ - g, Q32; own rows)
//   x_{i-1} = x_{i-2} + α_{i-1} p_{i-1}                 (eager x, own rows)
//   p_i = r_{i-1} + β_{i-1} p_{i-1},
//   z_i = A p_i = Σ_c a_rc (r_{i-2} - α z_{i-1} + β p_{i-1})_c + (A C)_r γ_{i-1}
// (the neighbours' C γ term through A C, formed once per system at the
// refresh), and the duals with C~, A^* C~, γ~, ᾱ, β̄.  ONE reduction per
// iteration: the 7 scalars of k_fused and the k-vectors C~^*z_i, C^*z~_i,
// C^*p~_i, C^*r~_{i-1}, C~^*r_{i-1} -- ζ_i, ζ~_i, σ_i, the Q32 g_{i-1}, g~_{i-1}
// and β_i from the expansion of ρ_i = (r~_i, r_i).  Two n x k reads per side
// (C, A C) instead of the two-kernel form's two C passes, and 16 instead of
// 22 n-vectors per iteration.
constexpr int NFK = 7;
template <typename T>
__device__ __forceinline__ void fusedk_leader(const LoopArgs<T> &a, DevState<T> *st, const T *s_fin, int i,
                                              T alpha, T beta, const T *gam_o, const T *gamt_o) {
  const int k = a.k;
  const T *b1 = s_fin + NFK, *b2 = b1 + k, *b3 = b2 + k, *b4 = b3 + k, *b5 = b4 + k;
  const T rho_prev = s_fin[0];   // ρ_{i-1}, exact
  const double rn = sqrt(re(s_fin[1])), rtn = sqrt(re(s_fin[2]));
  int done = 0, status = RBICG_OK;
  if (i >= 2) {   // iteration i-1 completes here: record, ζ_c, stop test
    const int m = i - 1;
    IterRec<T> rec;
    rec.alpha = alpha;
    rec.beta = beta;
    rec.rho = rho_prev;
    rec.sigma = ldcg(&st->sigma);
    rec.rnorm = rn;
    rec.rtnorm = rtn;
    a.hist[m] = rec;
    for (int j = 0; j < k; ++j) {   // ζ_c += γ_{i-1} (Q32 form of P:465)
      st->zc[j] = add(ldcg(&st->zc[j]), gam_o[j]);
      st->ztc[j] = add(ldcg(&st->ztc[j]), gamt_o[j]);
    }
    const int force = __ldcg(&st->force);
    const bool conv = !force && rn <= __ldcg(&st->tolb) && rtn <= __ldcg(&st->tolbt);
    if (conv) {
      done = 1;
    } else if (iszero(rho_prev) || !finite(divd(rho_prev, ldcg(&st->rho)))) {
      done = 1;
      status = RBICG_BREAKDOWN_SERIOUS;
    } else if (m >= __ldcg(&st->max_itn)) {
      done = 1;
      status = force ? RBICG_OK : RBICG_MAXITER;
    } else if (m == __ldcg(&st->stop_at)) {
      done = 2;
    }
    st->iter = m;
    st->rnorm = rn;
    st->rtnorm = rtn;
    st->rho = rho_prev;
  }
  // iteration i: ζ_i = D^{-1} C~^*z_i, ζ~_i = D^{-1} C^*z~_i, σ_i, α_i
  T zeta[KMAX], zetat[KMAX];
  T sigma = s_fin[3];
  for (int j = 0; j < k; ++j) {
    const double di = __ldcg(&st->dinv[j]);
    zeta[j] = scal(di, b1[j]);
    zetat[j] = scal(di, b2[j]);
    sigma = sub(sigma, cmul(b3[j], zeta[j]));   // (p~, z - Cζ)  (Q23)
  }
  const T alpha_i = divd(rho_prev, sigma);
  if (!done && (iszero(sigma) || !finite(alpha_i))) {
    done = 1;
    status = RBICG_BREAKDOWN_SECOND;
  }
  // ρ_i ≈ ρ_{i-1} - α (r~, q) - α (q~, r) + α² (q~, q) - (r~, C g) - (C~ g~, r)
  //       + (C~ g~, C g),  q = z - Cζ, q~ = z~ - C~ζ~, g = D^{-1}C~^*r, g~ = D^{-1}C^*r~
  T rq = s_fin[4], qr = s_fin[5], qq = s_fin[6], gterm = zero<T>();
  const T ca = conj(alpha_i);
  for (int j = 0; j < k; ++j) {
    const double di = __ldcg(&st->dinv[j]), d = 1.0 / di;
    const T g = scal(di, b5[j]), gt = scal(di, b4[j]);
    rq = sub(rq, cmul(b4[j], zeta[j]));                       // (C^*r~)^* ζ
    qr = sub(qr, cmul(zetat[j], b5[j]));                      // ζ~^* (C~^*r)
    qq = sub(qq, cmul(b2[j], zeta[j]));                       // (C^*z~)^* ζ
    qq = sub(qq, cmul(zetat[j], b1[j]));                      // ζ~^* (C~^*z)
    qq = add(qq, scal(d, cmul(zetat[j], zeta[j])));           // ζ~^* D ζ
    gterm = add(gterm, cmul(b4[j], g));                       // (r~, C g)
    gterm = add(gterm, cmul(gt, b5[j]));                      // (C~ g~, r)
    gterm = sub(gterm, scal(d, cmul(gt, g)));                 // -(C~ g~, C g)
    // γ_i = α_i ζ_i - g_{i-1}, γ~_i = ᾱ_i ζ~_i - g~_{i-1}  (Q32)
    st->gam[j] = sub(mul(alpha_i, zeta[j]), g);
    st->gamt[j] = sub(mul(ca, zetat[j]), gt);
    a.zhist[(int64_t)i * k + j] = zeta[j];
    a.zthist[(int64_t)i * k + j] = zetat[j];
  }
  const T rho_ext = sub(add(sub(sub(rho_prev, mul(alpha_i, rq)), mul(alpha_i, qr)),
                            mul(mul(alpha_i, alpha_i), qq)), gterm);
  {   // flag a cancelling expansion (β_i inexact)
    const double aa = sqrt(abs2(alpha_i));
    const double mag = sqrt(abs2(rho_prev)) + aa * (sqrt(abs2(rq)) + sqrt(abs2(qr))) + aa * aa * sqrt(abs2(qq));
    if (sqrt(abs2(rho_ext)) < 1e3 * 2.220446049250313e-16 * mag) st->la_cancel += 1;
  }
  st->alpha = alpha_i;
  st->beta = divd(rho_ext, rho_prev);
  st->sigma = sigma;
  st->kidx = i;
  if (done) {
    st->status = status;
    st->done = done;
  }
}

template <typename T, int MINB>
__global__ void __launch_bounds__(BS, MINB) k_fusedk(LoopArgs<T> a) {
  __shared__ T s_fin[NFK + 5 * KMAX];
  __shared__ T s_w[NFK][BS / 32];
  __shared__ T s_gam[KMAX], s_gamt[KMAX];
  __shared__ T s_row[5][BS];   // z, z~, p~, r~, r of the tile (the k-dots), then block partials
  __shared__ int s_last;
  __shared__ uint64_t bars[2];
  __shared__ T s_ab[2];
  __shared__ int s_i[2];
  extern __shared__ __align__(128) unsigned char f_smem[];
  DevState<T> *st = a.st;
  const int tid = threadIdx.x;
  const int k = a.k;
  const int64_t n = a.n;
  const int64_t ntiles = (n + BS - 1) / BS;
  const int64_t G64 = gridDim.x;
  const int64_t t0 = a.tile_contig ? (ntiles * blockIdx.x) / G64 : blockIdx.x;
  const int64_t t1 = a.tile_contig ? (ntiles * (blockIdx.x + 1)) / G64 : ntiles;
  const int64_t tstep = a.tile_contig ? 1 : G64;
  const size_t stage_bytes = p1_mat_bytes<T>(a);
  const int nst = a.p1_stages;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < nst; ++q)
      if (t0 + q * tstep < t1) p1_issue<T>(a, f_smem + q * stage_bytes, stage_bytes, &bars[q], t0 + q * tstep);
  pdl_wait();
  if (tid == 0) {
    s_i[0] = __ldcg(&st->kidx);
    s_i[1] = __ldcg(&st->done);
    s_ab[0] = ldcg(&st->alpha);
    s_ab[1] = ldcg(&st->beta);
  }
  if (tid < k) {
    s_gam[tid] = ldcg(&st->gam[tid]);
    s_gamt[tid] = ldcg(&st->gamt[tid]);
  }
  __syncthreads();
  if (s_i[1]) {
    for (int q = 0; q < nst; ++q)
      if (t0 + q * tstep < t1) mbar_wait(&bars[q], 0);
    return;
  }
  const int i = s_i[0] + 1;
  const T alpha = s_ab[0], beta = s_ab[1];
  const T malpha = neg(alpha), cmalpha = conj(malpha), cb = conj(beta), ca = conj(alpha);
  const T *__restrict__ r = a.rring + (int64_t)(max(i - 2, 0) % a.ring) * a.ldr;
  const T *__restrict__ rt = a.rtring + (int64_t)(max(i - 2, 0) % a.ring) * a.ldr;
  T *__restrict__ rw = a.rring + (int64_t)((i - 1) % a.ring) * a.ldr;
  T *__restrict__ rtw = a.rtring + (int64_t)((i - 1) % a.ring) * a.ldr;
  const T *__restrict__ zpo = a.zp[(i - 1) & 1];
  const T *__restrict__ ztpo = a.ztp[(i - 1) & 1];
  T *__restrict__ zpn = a.zp[i & 1];
  T *__restrict__ ztpn = a.ztp[i & 1];
  const bool wr = i >= 2;
  const T *__restrict__ C = a.C;
  const T *__restrict__ Ct = a.Ct;
  const T *__restrict__ AC = a.AC;
  const T *__restrict__ AHCt = a.AHCt;
  T acc[NFK];
#pragma unroll
  for (int o = 0; o < NFK; ++o) acc[o] = zero<T>();
  T b1 = zero<T>(), b2 = zero<T>(), b3 = zero<T>(), b4 = zero<T>(), b5 = zero<T>();
  const int rstep = BS / k, kt = rstep * k;   // k-dots: thread tid < kt owns column tid % k
  const int TM = a.tile_max;
  const int64_t ns = a.A.nslices;
  VStage<T> vs{};
  uint32_t par = 0;
  int it = 0;
  for (int64_t tile = t0; tile < t1; tile += tstep, ++it) {
    const int64_t row0 = tile * BS;
    const int rows = (int)min((int64_t)BS, n - row0);
    const int si = nst == 2 ? (it & 1) : 0;
    const unsigned char *base = f_smem + si * stage_bytes;
    const int32_t *scA = reinterpret_cast<const int32_t *>(base);
    const int32_t *scH = a.shared_cols ? scA : scA + TM;
    const T *svA = reinterpret_cast<const T *>(scA + p1_ncols(a) * TM);
    const T *svH = svA + TM;
    const int64_t sl = (row0 >> 5) + (tid >> 5);
    const int64_t slc = min(sl, ns - 1);
    const int64_t bA = a.A.sptr[tile * (BS / 32)], bH = a.AH.sptr[tile * (BS / 32)];
    const int64_t oA = a.A.sptr[slc], oH = a.AH.sptr[slc];
    const int wA = (int)((a.A.sptr[slc + 1] - oA) >> 5), wH = (int)((a.AH.sptr[slc + 1] - oH) >> 5);
    const int lane = tid & 31;
    mbar_wait(&bars[si], (par >> si) & 1u);
    par ^= 1u << si;
    if (tid < rows) {
      const int64_t row = row0 + tid;
      T z, zt;
      fused_pair_smem<T, false>(scA + (oA - bA) + lane, svA + (oA - bA) + lane, wA,
                                scH + (oH - bH) + lane, svH + (oH - bH) + lane, wH, r, zpo, rt, ztpo, vs,
                                malpha, beta, cmalpha, cb, z, zt);
      T cg = zero<T>(), cgt = zero<T>(), acg = zero<T>(), acgt = zero<T>();
      for (int j = 0; j < k; ++j) {
        const int64_t e = row * k + j;
        cg = mad(ldg(C + e), s_gam[j], cg);
        cgt = mad(ldg(Ct + e), s_gamt[j], cgt);
        acg = mad(ldg(AC + e), s_gam[j], acg);
        acgt = mad(ldg(AHCt + e), s_gamt[j], acgt);
      }
      z = add(z, acg);      // + (A C)_row γ_{i-1}
      zt = add(zt, acgt);
      const RZP<T> o = ld_node(zpo, r, row), ot = ld_node(ztpo, rt, row);
      const T rr = add(mad(malpha, o.z, o.r), cg);          // r_{i-1} = r_{i-2} - α z_{i-1} + C γ_{i-1}
      const T rtr = add(mad(cmalpha, ot.z, ot.r), cgt);
      const T pr = mad(beta, o.p, rr);
      const T ptr = mad(cb, ot.p, rtr);
      if (wr) {
        rw[row] = rr;
        rtw[row] = rtr;
        a.x[row] = mad(alpha, o.p, a.x[row]);               // x_{i-1} = x_{i-2} + α p_{i-1}
        a.xt[row] = mad(ca, ot.p, a.xt[row]);
      }
      st_node(zpn, row, rr, z, pr);
      st_node(ztpn, row, rtr, zt, ptr);
      acc[0] = cmad(rtr, rr, acc[0]);
      acc[1] = add(acc[1], mk_re<T>(abs2(rr)));
      acc[2] = add(acc[2], mk_re<T>(abs2(rtr)));
      acc[3] = cmad(ptr, z, acc[3]);
      acc[4] = cmad(rtr, z, acc[4]);
      acc[5] = cmad(zt, rr, acc[5]);
      acc[6] = cmad(zt, z, acc[6]);
      s_row[0][tid] = z;
      s_row[1][tid] = zt;
      s_row[2][tid] = ptr;
      s_row[3][tid] = rtr;
      s_row[4][tid] = rr;
    }
    __syncthreads();   // stage si consumed; the tile's rows staged for the k-dots
    if (tid == 0 && tile + nst * tstep < t1)
      p1_issue<T>(a, f_smem + si * stage_bytes, stage_bytes, &bars[si], tile + nst * tstep);
    if (tid < kt) {
      const int nel = rows * k;
      int lr = tid / k;
      const T *__restrict__ Cb = C + row0 * k;
      const T *__restrict__ Ctb = Ct + row0 * k;
      for (int e = tid; e < nel; e += kt, lr += rstep) {
        const T c = ldg(Cb + e), ct = ldg(Ctb + e);
        b1 = cmad(ct, s_row[0][lr], b1);   // C~^* z_i
        b2 = cmad(c, s_row[1][lr], b2);    // C^* z~_i
        b3 = cmad(c, s_row[2][lr], b3);    // C^* p~_i
        b4 = cmad(c, s_row[3][lr], b4);    // C^* r~_{i-1}
        b5 = cmad(ct, s_row[4][lr], b5);   // C~^* r_{i-1}
      }
    }
    __syncthreads();
  }
  pdl_trigger();
  const int w = tid >> 5, l = tid & 31;
#pragma unroll
  for (int o = 0; o < NFK; ++o) {
    const T v = warp_sum(acc[o]);
    if (l == 0) s_w[o][w] = v;
  }
  s_row[0][tid] = tid < kt ? b1 : zero<T>();
  s_row[1][tid] = tid < kt ? b2 : zero<T>();
  s_row[2][tid] = tid < kt ? b3 : zero<T>();
  s_row[3][tid] = tid < kt ? b4 : zero<T>();
  s_row[4][tid] = tid < kt ? b5 : zero<T>();
  __syncthreads();
  const int G = gridDim.x;
  if (tid < NFK) {
    T sum = zero<T>();
    for (int q = 0; q < BS / 32; ++q) sum = add(sum, s_w[tid][q]);
    a.part[(int64_t)tid * G + blockIdx.x] = sum;
  }
  if (tid < 5 * k) {
    const int ty = tid / k, j = tid % k;
    T sum = zero<T>();
    for (int m = 0; m < rstep; ++m) sum = add(sum, s_row[ty][j + m * k]);
    a.part[(int64_t)(NFK + tid) * G + blockIdx.x] = sum;
  }
  if (!last_block(&st->cnt[0], &s_last)) return;
  final_reduce(a.part, NFK + 5 * k, G, s_fin);
  if (tid == 0) {
    st->cnt[0] = 0;
    fusedk_leader<T>(a, st, s_fin, i, alpha, beta, s_gam, s_gamt);
  }
}

template <typename T> size_t fused_smem(const LoopArgs<T> &a, bool vs) {
  const size_t mat = (a.dcols && !vs) ? dc_mat_bytes<T>(a) : p1_mat_bytes<T>(a);
  return (size_t)a.p1_stages * (mat + (vs ? fused_vec_bytes<T>() : 0));
}

// ============================================================== launchers
static int grid_for(int64_t n, int G) {
  const int64_t tiles = (n + BS - 1) / BS;
  return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, G));
}
// grid of an SpMV-kernel launch: its visits (halo-overlap ranges) or all tiles
template <typename T> static int grid_visits(const LoopArgs<T> &a, int G) {
  return a.ordered ? (int)std::max<int64_t>(1, std::min<int64_t>(a.tcount, G)) : grid_for(a.n, G);
}
// the boundary launch of the halo overlap follows an event join: plain launch
thread_local bool g_pdl_off = false;

template <typename T> size_t pass1_smem(const LoopArgs<T> &a) {
  return (size_t)a.p1_stages * p1_stage_bytes<T>(a) +
         (a.stage_c && a.k > 0 ? (size_t)2 * BS * a.k * sizeof(T) : 0);
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
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl && !g_pdl_off ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RB_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <typename T> size_t pass1s_smem(const LoopArgs<T> &a) {
  return (size_t)a.p1_stages * p1s_stage_bytes<T>(a) +
         (a.stage_c && a.k > 0 ? (size_t)2 * TRH * a.k * sizeof(T) : 0);
}
static int p1s_chunk() {
  static const int ch = getenv("RBICG_P1S_CH") ? atoi(getenv("RBICG_P1S_CH")) : 8;
  return ch;
}
template <typename T> static void *pass1s_fn() {
  switch (p1s_chunk()) {
    case 4: return (void *)k_pass1s<T, 4>;
    case 6: return (void *)k_pass1s<T, 6>;
    default: return (void *)k_pass1s<T, 8>;
  }
}

template <typename T> void launch_pass1(const LoopArgs<T> &a, cudaStream_t s) {
  if (a.split) {
    const size_t sm = pass1s_smem<T>(a);
    int per_sm = 1;
    RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pass1s_fn<T>(), BS, sm));
    const int G = std::min(a.G, std::max(1, per_sm) * a.nsm);
    const int64_t tiles = a.ordered ? a.tcount : (a.n + TRH - 1) / TRH;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, G)));
    cfg.blockDim = dim3(BS);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl && !g_pdl_off ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void *args[] = {(void *)&a};
    RB_CUDA(cudaLaunchKernelExC(&cfg, pass1s_fn<T>(), args));
    count_launch();
    return;
  }
  const size_t sm = a.staged ? pass1_smem<T>(a) : 0;
  int per_sm = 1;
  // register bound of the k = 0 form: RBICG_P1_MINB (4 = 64 regs, 5, 6)
  static const int minb = getenv("RBICG_P1_MINB") ? atoi(getenv("RBICG_P1_MINB")) : 4;
  auto fn = minb >= 6 ? k_pass1<T, 6> : (minb == 5 ? k_pass1<T, 5> : k_pass1<T, 4>);
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, BS, sm));
  const int G = std::min(a.G, std::max(1, per_sm) * a.nsm);
  launch_pdl(fn, grid_visits(a, G), sm, s, a);
  count_launch();
}

// two stages of (8 vector tiles + C, C~ tiles)
template <typename T> size_t pass2_smem(int k, int lazy) {
  return (size_t)2 * p2_stage_elems<T>(k, lazy) * sizeof(T);
}

// fused iteration (k = 0, staged SELL tiles): RBICG_FUSED_MINB = 3/4 (registers)
template <typename T> void launch_fused(const LoopArgs<T> &a0, cudaStream_t s) {
  // one TMA stage of matrix tiles (RBICG_FUSED_STAGES=2 measured C2 50.5 vs
  // 46.5 us per iteration at 4 CTAs/SM)
  LoopArgs<T> a = a0;
  static const int fst = getenv("RBICG_FUSED_STAGES") ? atoi(getenv("RBICG_FUSED_STAGES")) : 1;
  a.p1_stages = std::min(2, std::max(1, fst));
  // vector rows of each tile staged by TMA too, in-tile gathers from shared
  // memory (opt-in: measured slower, C2 50.8 vs 46.8 us, C3 296 vs 278 us --
  // those gathers were L1 hits already)
  static const int vse = getenv("RBICG_FUSED_VS") ? atoi(getenv("RBICG_FUSED_VS")) : 0;
  const bool vs = vse != 0;
  const size_t sm = fused_smem<T>(a, vs);
  // 4 CTAs/SM at 64 registers (C2: 46.3 us per iteration; 3 CTAs at 80: 56.3 us)
  // (complex: 3 CTAs/SM, 80 registers -- 64 spill with the 256-bit node loads)
  static const int minb_env = getenv("RBICG_FUSED_MINB") ? atoi(getenv("RBICG_FUSED_MINB")) : 0;
  const int minb = minb_env ? minb_env : (sizeof(T) == 8 ? 4 : 3);
  const bool dc = a.dcols != nullptr && !vs;
  auto fn = dc ? (minb >= 4 ? k_fused<T, 4, false, true> : k_fused<T, 3, false, true>)
          : vs ? (minb >= 4 ? k_fused<T, 4, true> : k_fused<T, 3, true>)
               : (minb >= 6 ? k_fused<T, 6> : minb == 5 ? k_fused<T, 5> : minb == 4 ? k_fused<T, 4> : k_fused<T, 3>);
  static const int carve = getenv("RBICG_FUSED_CARVEOUT") ? atoi(getenv("RBICG_FUSED_CARVEOUT")) : -1;
  if (carve >= 0) RB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
  int per_sm = 1;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, BS, sm));
  const int G = std::min(a.G, std::max(1, per_sm) * a.nsm);
  launch_pdl(fn, grid_visits(a, G), sm, s, a);
  count_launch();
}

template <typename T> void launch_fusedk(const LoopArgs<T> &a0, cudaStream_t s) {
  LoopArgs<T> a = a0;
  a.p1_stages = 1;
  const size_t sm = (size_t)p1_mat_bytes<T>(a);
  static const int minb_env = getenv("RBICG_FUSEDK_MINB") ? atoi(getenv("RBICG_FUSEDK_MINB")) : 0;
  const int minb = minb_env ? minb_env : (sizeof(T) == 8 ? 4 : 3);
  auto fn = minb >= 4 ? k_fusedk<T, 4> : k_fusedk<T, 3>;
  int per_sm = 1;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, BS, sm));
  const int G = std::min(a.G, std::max(1, per_sm) * a.nsm);
  launch_pdl(fn, grid_for(a.n, G), sm, s, a);
  count_launch();
}
template <typename T> void launch_pc_pupdate(const LoopArgs<T> &a, T *pfix, T *ptfix, cudaStream_t s) {
  k_pc_pupdate<T><<<grid_for(a.n, a.G), BS, 0, s>>>(a, pfix, ptfix);
  count_launch();
}
template <typename T> void launch_pc_proj(const LoopArgs<T> &a, cudaStream_t s) {
  k_pc_proj<T><<<grid_for(a.n, a.G), BS, 0, s>>>(a);
  count_launch();
}
template <typename T> void launch_leader_fused(const LoopArgs<T> &a, cudaStream_t s) {
  k_leader_fused<T><<<1, 32, 0, s>>>(a);
  count_launch();
}
template <typename T>
void launch_halo_fused(const LoopArgs<T> &a, const int32_t *idx, int64_t nsend, T *sendbuf,
                       const T *recvbuf, int64_t nghost, int pack, cudaStream_t s) {
  if (pack && nsend > 0) {
    k_halo_pack_fused<T><<<(int)std::min<int64_t>((nsend + 255) / 256, 1184), 256, 0, s>>>(a, idx, nsend, sendbuf);
    count_launch();
  }
  if (!pack && nghost > 0) {
    k_halo_unpack_fused<T><<<(int)std::min<int64_t>((nghost + 255) / 256, 1184), 256, 0, s>>>(a, recvbuf, nghost);
    count_launch();
  }
}

template <typename T> void launch_pass2(const LoopArgs<T> &a, cudaStream_t s) {
  size_t sm = pass2_smem<T>(a.k, a.lazy_x);
  const int staged = (sm <= 200 * 1024 && a.pass2_tma) ? 1 : 0;
  if (!staged) sm = 0;
  int per_sm = 1;
  // register bound: RBICG_P2_MINB (4 = 64 regs, measured C3 pass 2 63.4 -> 58.5 us; 3 = 80)
  static const int minb = getenv("RBICG_P2_MINB") ? atoi(getenv("RBICG_P2_MINB")) : 4;
  auto fn = minb >= 4 ? k_pass2<T, 4> : k_pass2<T, 3>;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, BS, sm));
  const int G = std::min(a.G, std::max(1, per_sm) * a.nsm);
  launch_pdl(fn, grid_for(a.n, G), sm, s, a, staged);
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

static int g_small(int64_t m) { return (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 1184)); }
template <typename T> void launch_leader1(const LoopArgs<T> &a, cudaStream_t s) {
  k_leader1<T><<<1, BS, 0, s>>>(a);
  count_launch();
}
template <typename T> void launch_leader2(const LoopArgs<T> &a, cudaStream_t s) {
  k_leader2<T><<<1, BS, 0, s>>>(a);
  count_launch();
}
template <typename T> void launch_leader_resid(const LoopArgs<T> &a, int coef, cudaStream_t s) {
  k_leader_resid<T><<<1, BS, 0, s>>>(a, coef);
  count_launch();
}
template <typename T> void launch_leader_init2(const LoopArgs<T> &a, cudaStream_t s) {
  k_leader_init2<T><<<1, BS, 0, s>>>(a);
  count_launch();
}
template <typename T>
void launch_halo_pack_loop(const LoopArgs<T> &a, const int32_t *idx, int64_t nsend, T *buf,
                           cudaStream_t s) {
  if (nsend <= 0) return;
  k_halo_pack_loop<T><<<g_small(nsend), 256, 0, s>>>(a, idx, nsend, buf);
  count_launch();
}
template <typename T>
void launch_halo_unpack_loop(const LoopArgs<T> &a, const T *buf, int64_t nghost, cudaStream_t s) {
  if (nghost <= 0) return;
  k_halo_unpack_loop<T><<<g_small(nghost), 256, 0, s>>>(a, buf, nghost);
  count_launch();
}
template <typename T>
void launch_pack_rows(const T *X, int k, const int32_t *idx, int64_t cnt, T *out, cudaStream_t s) {
  if (cnt <= 0 || k <= 0) return;
  k_pack_rows<T><<<g_small(cnt * k), 256, 0, s>>>(X, k, idx, cnt, out);
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
  allow_max_dyn_smem(k_pass1s<double, 4>);
  allow_max_dyn_smem(k_pass1s<double, 6>);
  allow_max_dyn_smem(k_pass1s<double, 8>);
  allow_max_dyn_smem(k_pass1s<zc, 4>);
  allow_max_dyn_smem(k_pass1s<zc, 6>);
  allow_max_dyn_smem(k_pass1s<zc, 8>);
  allow_max_dyn_smem(k_pass1<double, 4>);
  allow_max_dyn_smem(k_pass1<double, 5>);
  allow_max_dyn_smem(k_pass1<double, 6>);
  allow_max_dyn_smem(k_pass1<zc, 4>);
  allow_max_dyn_smem(k_pass1<zc, 5>);
  allow_max_dyn_smem(k_pass1<zc, 6>);
  allow_max_dyn_smem(k_pass2<double, 3>);
  allow_max_dyn_smem(k_pass2<double, 4>);
  allow_max_dyn_smem(k_pass2<zc, 3>);
  allow_max_dyn_smem(k_pass2<zc, 4>);
  allow_max_dyn_smem(k_fused<double, 3>);
  allow_max_dyn_smem(k_fused<double, 4>);
  allow_max_dyn_smem(k_fusedk<double, 4>);
  allow_max_dyn_smem(k_fusedk<double, 3>);
  allow_max_dyn_smem(k_fusedk<zc, 4>);
  allow_max_dyn_smem(k_fusedk<zc, 3>);
  allow_max_dyn_smem(k_fused<double, 4, false, true>);
  allow_max_dyn_smem(k_fused<double, 3, false, true>);
  allow_max_dyn_smem(k_fused<zc, 4, false, true>);
  allow_max_dyn_smem(k_fused<zc, 3, false, true>);
  allow_max_dyn_smem(k_fused<double, 4, true>);
  allow_max_dyn_smem(k_fused<double, 3, true>);
  allow_max_dyn_smem(k_fused<zc, 4, true>);
  allow_max_dyn_smem(k_fused<zc, 3, true>);
  allow_max_dyn_smem(k_fused<double, 5>);
  allow_max_dyn_smem(k_fused<double, 6>);
  allow_max_dyn_smem(k_fused<zc, 5>);
  allow_max_dyn_smem(k_fused<zc, 6>);
  allow_max_dyn_smem(k_fused<zc, 3>);
  allow_max_dyn_smem(k_fused<zc, 4>);
  prepare_block_kernels();
}

#define RB_INST(T)                                                                          \
  template void launch_pass1<T>(const LoopArgs<T> &, cudaStream_t);                          \
  template void launch_pass2<T>(const LoopArgs<T> &, cudaStream_t);                          \
  template void launch_fused<T>(const LoopArgs<T> &, cudaStream_t);                          \
  template void launch_leader_fused<T>(const LoopArgs<T> &, cudaStream_t);                   \
  template void launch_fusedk<T>(const LoopArgs<T> &, cudaStream_t);                         \
  template void launch_pc_pupdate<T>(const LoopArgs<T> &, T *, T *, cudaStream_t);           \
  template void launch_pc_proj<T>(const LoopArgs<T> &, cudaStream_t);                         \
  template void launch_halo_fused<T>(const LoopArgs<T> &, const int32_t *, int64_t, T *,      \
                                     const T *, int64_t, int, cudaStream_t);                 \
  template void launch_resid<T>(const LoopArgs<T> &, const T *, const T *, const T *,        \
                                const T *, T *, T *, int, cudaStream_t);                     \
  template void launch_init2<T>(const LoopArgs<T> &, const T *, const T *, cudaStream_t);    \
  template void launch_step7<T>(const LoopArgs<T> &, const T *, const T *, T *, T *,         \
                                cudaStream_t);                                               \
  template void launch_spmv_pair<T>(const DevMat &, const DevMat &, const T *, const T *, T *, \
                                    T *, cudaStream_t);                                       \
  template void launch_leader1<T>(const LoopArgs<T> &, cudaStream_t);                        \
  template void launch_leader2<T>(const LoopArgs<T> &, cudaStream_t);                        \
  template void launch_leader_resid<T>(const LoopArgs<T> &, int, cudaStream_t);              \
  template void launch_leader_init2<T>(const LoopArgs<T> &, cudaStream_t);                   \
  template void launch_halo_pack_loop<T>(const LoopArgs<T> &, const int32_t *, int64_t, T *, \
                                         cudaStream_t);                                       \
  template void launch_halo_unpack_loop<T>(const LoopArgs<T> &, const T *, int64_t,          \
                                           cudaStream_t);                                     \
  template void launch_pack_rows<T>(const T *, int, const int32_t *, int64_t, T *, cudaStream_t);
RB_INST(double)
RB_INST(zc)

}  // namespace rbicg
