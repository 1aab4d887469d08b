// Micro-benchmark: cost of one grid barrier (arrive + leader release + wait)
// in a cooperative kernel on this GPU, flat vs two-level arrival counting.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier barrier.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned atom_add_release(unsigned *p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// mode 0: flat counter; mode 1: groups of GS blocks, last of a group arrives at the top
template <int MODE>
__global__ void kbar(unsigned *cnt, unsigned *gen, int iters, int GS, unsigned long long *t) {
  __shared__ int flag;
  unsigned g0 = 0;
  if (threadIdx.x == 0) g0 = ld_relaxed(gen);
  const int G = gridDim.x;
  const int ngroups = (G + GS - 1) / GS;
  const int grp = blockIdx.x / GS;
  const int gsize = min(GS, G - grp * GS);
  unsigned long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int b = 1; b <= iters; ++b) {
    __syncthreads();
    if (threadIdx.x == 0) {
      bool last;
      if (MODE == 0) {
        last = atom_add_release(&cnt[0], 1u) == (unsigned)G - 1;
      } else {
        last = atom_add_release(&cnt[1 + grp * 32], 1u) == (unsigned)gsize - 1;
        if (last) {
          cnt[1 + grp * 32] = 0;
          last = atom_add_release(&cnt[0], 1u) == (unsigned)ngroups - 1;
        }
      }
      flag = last;
      if (last) {
        asm volatile("fence.acquire.gpu;" ::: "memory");
        cnt[0] = 0;
        st_release(gen, g0 + b);
      } else {
        while (ld_relaxed(gen) != g0 + b) __nanosleep(32);
        asm volatile("fence.acquire.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *t = t1 - t0;
  }
}

int main() {
  unsigned *cnt, *gen;
  unsigned long long *t, ht;
  cudaMalloc(&cnt, 4096 * 4);
  cudaMalloc(&gen, 4);
  cudaMalloc(&t, 8);
  cudaMemset(cnt, 0, 4096 * 4);
  cudaMemset(gen, 0, 4);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2000;
  for (int bps : {1, 2, 3, 4}) {
    for (int mode = 0; mode < 2; ++mode) {
      for (int GS : {8, 16, 37}) {
        if (mode == 0 && GS != 8) continue;
        int G = nsm * bps;
        void *args[] = {&cnt, &gen, (void *)&iters, &GS, &t};
        cudaLaunchCooperativeKernel(mode ? (void *)kbar<1> : (void *)kbar<0>, G, 256, args, 0, 0);
        cudaLaunchCooperativeKernel(mode ? (void *)kbar<1> : (void *)kbar<0>, G, 256, args, 0, 0);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&ht, t, 8, cudaMemcpyDeviceToHost);
        printf("G=%d mode=%d GS=%d: %.3f us per barrier (%s)\n", G, mode, GS, ht / 1e3 / iters,
               cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
