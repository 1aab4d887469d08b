// persist.cu -- the RBiCG hot loop as ONE persistent cooperative kernel per
// cycle (Algorithm 2; phase bodies in hot.cuh).
//
// An iteration has two global reduction points (σ_i before α_i, ρ_i before
// β_i).  The two-kernel form (kernels.cu) pays a kernel
// boundary at each: launch, ramp-up of the first TMA tiles and the gathers,
// and the drain of the slowest block.  Here every block stays resident for
// the whole cycle and the reduction points are grid barriers whose last
// arriving block is the reduction leader (the same fixed-order final sum and
// scalar step as the last block of the two-kernel form, so both forms give
// bitwise-identical iterates for the same grid).  Before each barrier a block
// already issues the bulk copies of its first tile of the next phase (the
// matrix tiles are constant; the phase-2 inputs are the block's own rows), so
// the barrier latency overlaps data movement.
//
// Coherence inside one launch: the gathered directions p, p~ are rewritten
// every other iteration by other blocks, so they are read through L2 only
// (ld.global.cg); the residuals r, r~ are Lanczos ring columns written once
// per launch before they are read (ring >= s + 2, columns 256-byte aligned),
// so the read-only path is safe.  Own rows written with generic stores and
// read back by the TMA engine are ordered by fence.proxy.async.
#include "hot.cuh"
#include <cstdlib>
#include <algorithm>

namespace rbicg {

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Arrive at the grid barrier (release-ordered, no L1 invalidation while other
// blocks of this SM still work); true in every thread of the last block to
// arrive, which acquires (every block has arrived by then).
__device__ __forceinline__ bool grid_arrive(unsigned *cnt, int *s_flag) {
  return last_block(cnt, s_flag);
}
// Leader: open the barrier (generation `next`) after its scalar step.
__device__ __forceinline__ void grid_release(unsigned *cnt, unsigned *gen, unsigned next) {
  __syncthreads();
  if (threadIdx.x == 0) {
    *cnt = 0;
    st_release_u32(gen, next);
  }
}
// Others: poll the generation with relaxed loads (no L1 invalidation per
// poll), then acquire once.
__device__ __forceinline__ void grid_wait(const unsigned *gen, unsigned next) {
  if (threadIdx.x == 0) {
    while (ld_relaxed_u32(gen) != next) __nanosleep(32);
    fence_acquire();
  }
  __syncthreads();
}

template <typename T> __host__ __device__ __forceinline__ size_t loop_p1_bytes(const LoopArgs<T> &a) {
  return (size_t)a.p1_stages * p1_stage_bytes<T>(a) +
         (a.stage_c && a.k > 0 ? (size_t)2 * BS * a.k * sizeof(T) : 0);
}
template <typename T> __host__ __device__ __forceinline__ size_t loop_p2_bytes(const LoopArgs<T> &a) {
  return (size_t)2 * p2_stage_elems<T>(a.k, a.lazy_x) * sizeof(T);
}

template <typename T, bool COH, int MINB>
__global__ void __launch_bounds__(BS, MINB) k_loop(LoopArgs<T> a, int p2_staged) {
  __shared__ P1Scratch<T> sc;
  __shared__ Snap<T> sn;
  __shared__ T s_fin[3 * KMAX + 1];
  __shared__ T s_w[BS / 32];
  __shared__ T s_alpha;
  __shared__ int s_last, s_ok;
  __shared__ unsigned s_gen;
  __shared__ uint64_t bars[3], bars2[2];
  // phase-1 and phase-2 buffers share the dynamic shared memory: each phase's
  // first tile is issued only after the other phase has consumed its buffers
  extern __shared__ __align__(128) unsigned char dsm[];
  T *sb2 = reinterpret_cast<T *>(dsm);
  DevState<T> *st = a.st;
  const int tid = threadIdx.x;
  const int k = a.k;
  const int64_t ntiles = (a.n + BS - 1) / BS;
  const int64_t nfull = a.n / BS;
  const int64_t G64 = gridDim.x;
  const size_t stage_bytes = p1_stage_bytes<T>(a);
  const int nst = a.p1_stages;
  const bool stage_v = a.staged && a.stage_v;
  if (tid == 0) {
    mbar_init(&bars[0], stage_v ? 2 : 1);
    mbar_init(&bars[1], stage_v ? 2 : 1);
    mbar_init(&bars[2], 1);
    mbar_init(&bars2[0], 2);   // phase-2 stages: two arrivals (p2_issue_a/_b)
    mbar_init(&bars2[1], 2);
    fence_mbar_init();
    s_gen = ld_relaxed_u32(&st->gen);
  }
  __syncthreads();
  // first tiles of phase 1 of iteration `it` (own vector rows: written by
  // this block with generic stores -> proxy fence before the bulk copies)
  auto issue_p1_first = [&](int it_next) {
    if (stage_v) {
      fence_proxy_async();
      __syncthreads();
    }
    if (a.staged && tid == 0)
      for (int q = 0; q < nst; ++q)
        if ((int64_t)blockIdx.x + q * G64 < ntiles) {
          p1_issue<T>(a, dsm + q * stage_bytes, stage_bytes, &bars[q], blockIdx.x + q * G64);
          if (stage_v) p1_issue_vec<T>(a, dsm + q * stage_bytes, &bars[q], blockIdx.x + q * G64, it_next);
        }
  };
  uint32_t par = 0, par2 = 0;
  auto drain_p1_first = [&]() {
    if (!a.staged) return;
    for (int q = 0; q < nst; ++q)
      if ((int64_t)blockIdx.x + q * G64 < ntiles) {
        mbar_wait(&bars[q], (par >> q) & 1u);
        par ^= 1u << q;
      }
  };
  snap_load(st, k, sn);
  issue_p1_first(sn.iter);
  const unsigned gen0 = s_gen;
  unsigned nb = 0;
  for (;;) {
    snap_load(st, k, sn);
    if (sn.done) {
      drain_p1_first();
      break;
    }
    const int it = sn.iter;
    // ---------------- phase 1: SpMV pair + projection coefficients
    T a1 = zero<T>(), a2 = zero<T>(), a3 = zero<T>(), aptz = zero<T>();
    p1_tiles<T, COH>(a, dsm, bars, par, sc, it, sn.beta, a.lazy_x && it == sn.seg_start, a1, a2,
                      a3, aptz);
    p1_partials<T>(a, sc, s_w, a1, a2, a3, aptz);
    // own rows of z, z~ (and r_{i-1}) are read back by the TMA engine
    const bool pre2 = p2_staged && (int64_t)blockIdx.x < nfull;
    if (p2_staged) {
      fence_proxy_async();
      __syncthreads();
      if (pre2 && tid == 0)
        p2_issue<T>(a, sb2, &bars2[0], blockIdx.x, a.rring + (int64_t)(it % a.ring) * a.ldr,
                    a.rtring + (int64_t)(it % a.ring) * a.ldr, pcol(a, it + 1), ptcol(a, it + 1));
    }
    ++nb;
    if (grid_arrive(&st->cnt[0], &s_last)) {
      final_reduce(a.part, 3 * k + 1, gridDim.x, s_fin);
      p1_leader<T>(a, st, sn, it, s_fin, &s_alpha, &s_ok);
      grid_release(&st->cnt[0], &st->gen, gen0 + nb);
    } else {
      grid_wait(&st->gen, gen0 + nb);
    }
    snap_load(st, k, sn);   // α_i, ζ_i, ζ~_i (or a breakdown)
    if (sn.done) {
      if (pre2) mbar_wait(&bars2[0], par2 & 1u);
      break;
    }
    // ---------------- phase 2: corrections, updates, ρ_i
    T arho = zero<T>();
    double an = 0.0, ant = 0.0;
    p2_tiles<T>(a, p2_staged != 0, sb2, bars2, par2, pre2 ? 1 : 0, it, sn.alpha, sn.zeta, sn.zetat, arho,
                an, ant);
    p2_partials<T>(a, s_w, arho, an, ant);
    __syncthreads();     // phase-2 buffers consumed
    issue_p1_first(it + 1);   // next iteration's first tiles
    ++nb;
    if (grid_arrive(&st->cnt[0], &s_last)) {
      final_reduce(a.part, 3, gridDim.x, s_fin);
      p2_leader<T>(a, st, sn, it, s_fin);
      grid_release(&st->cnt[0], &st->gen, gen0 + nb);
    } else {
      grid_wait(&st->gen, gen0 + nb);
    }
  }
}

template <typename T> size_t loop_smem(const LoopArgs<T> &a, int p2_staged) {
  const size_t p1 = a.staged ? loop_p1_bytes<T>(a) : 0;
  const size_t p2 = p2_staged ? loop_p2_bytes<T>(a) : 0;
  return std::max(p1, p2);
}

// The instantiation for these arguments: COH when the directions are
// ping-pong buffers (L2-only gathers), MINB = blocks per SM the registers are
// bounded for (RBICG_LOOP_MINB, default 4).
template <typename T> static void *loop_fn(const LoopArgs<T> &a) {
  static const int minb = getenv("RBICG_LOOP_MINB") ? atoi(getenv("RBICG_LOOP_MINB")) : 4;
  if (minb == 3) return a.pring_len ? (void *)k_loop<T, false, 3> : (void *)k_loop<T, true, 3>;
  return a.pring_len ? (void *)k_loop<T, false, 4> : (void *)k_loop<T, true, 4>;
}

// Grid of the cooperative loop kernel for these arguments (0: not possible).
template <typename T> int loop_grid(const LoopArgs<T> &a, int *p2_staged_out) {
  int p2_staged = a.pass2_tma ? 1 : 0;
  if (p2_staged && loop_p2_bytes<T>(a) > 200 * 1024) p2_staged = 0;
  const size_t sm = loop_smem<T>(a, p2_staged);
  int per_sm = 0;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, loop_fn<T>(a), BS, sm));
  if (const char *e = getenv("RBICG_LOOP_BPS")) per_sm = std::min(per_sm, std::max(1, atoi(e)));
  *p2_staged_out = p2_staged;
  const int64_t tiles = (a.n + BS - 1) / BS;
  return (int)std::min<int64_t>({(int64_t)per_sm * a.nsm, tiles, (int64_t)a.G});
}

template <typename T> bool launch_loop(const LoopArgs<T> &a, cudaStream_t s) {
  int p2_staged = 0;
  const int G = loop_grid<T>(a, &p2_staged);
  if (G <= 0) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(BS);
  cfg.dynamicSmemBytes = loop_smem<T>(a, p2_staged);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void *args[] = {(void *)&a, (void *)&p2_staged};
  RB_CUDA(cudaLaunchKernelExC(&cfg, loop_fn<T>(a), args));
  count_launch();
  return true;
}

void prepare_loop_kernels() {
  allow_max_dyn_smem(k_loop<double, true, 3>);
  allow_max_dyn_smem(k_loop<double, false, 3>);
  allow_max_dyn_smem(k_loop<zc, true, 3>);
  allow_max_dyn_smem(k_loop<zc, false, 3>);
  allow_max_dyn_smem(k_loop<double, true, 4>);
  allow_max_dyn_smem(k_loop<double, false, 4>);
  allow_max_dyn_smem(k_loop<zc, true, 4>);
  allow_max_dyn_smem(k_loop<zc, false, 4>);
}

template bool launch_loop<double>(const LoopArgs<double> &, cudaStream_t);
template bool launch_loop<zc>(const LoopArgs<zc> &, cudaStream_t);
template int loop_grid<double>(const LoopArgs<double> &, int *);
template int loop_grid<zc>(const LoopArgs<zc> &, int *);

}  // namespace rbicg
