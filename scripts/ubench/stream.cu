// Micro-benchmark: read-only streaming of a buffer through 1-D TMA bulk
// copies (cp.async.bulk + mbarrier) into shared memory, as the SpMV-pair
// kernel streams its SELL tiles: tile bytes x stages x blocks/SM, sized like
// C2 (201 MB) and C3 (1.69 GB).  Prints GB/s per configuration, timed over
// back-to-back launches in a CUDA graph.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)));
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk(void *d, const void *s, uint32_t n, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
                   su32(b)), "r"(ph) : "memory");
}

__global__ void kstream(const char *src, size_t bytes, int tile, int nst, double *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bars[8];
  const int64_t ntiles = (int64_t)(bytes / tile);
  const int64_t G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int q = 0; q < nst; ++q) mbar_init(&bars[q]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < nst; ++q) {
      const int64_t t = blockIdx.x + q * G;
      if (t < ntiles) {
        expect_tx(&bars[q], tile);
        bulk(sm + q * tile, src + t * tile, tile, &bars[q]);
      }
    }
  double acc = 0;
  int i = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += G, ++i) {
    const int si = i % nst;
    wait(&bars[si], (i / nst) & 1);
    const double *d = reinterpret_cast<const double *>(sm + si * tile);
    for (int e = threadIdx.x; e < tile / 8; e += blockDim.x) acc += d[e];
    __syncthreads();
    const int64_t nx = t + nst * G;
    if (threadIdx.x == 0 && nx < ntiles) {
      expect_tx(&bars[si], tile);
      bulk(sm + si * tile, src + nx * tile, tile, &bars[si]);
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

// plain vectorised loads for comparison
__global__ void kldg(const double2 *src, size_t n2, double *out) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(src + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(kstream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  char *buf;
  double *out;
  const size_t maxb = (size_t)1700 << 20;
  cudaMalloc(&buf, maxb);
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, maxb);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t bytes : {(size_t)201 << 20, (size_t)1690 << 20}) {
    const int reps = bytes < ((size_t)500 << 20) ? 40 : 8;
    for (int tile : {8192, 16384, 32768, 65536}) {
      for (int nst : {1, 2, 3}) {
        for (int bps : {1, 2, 3, 4, 6, 8}) {
          const size_t smem = (size_t)tile * nst;
          int occ = 0;
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kstream, 256, smem);
          if (occ < bps) continue;
          const int G = nsm * bps;
          cudaGraph_t g;
          cudaGraphExec_t ge;
          cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
          for (int r = 0; r < reps; ++r) kstream<<<G, 256, smem, s>>>(buf, bytes, tile, nst, out);
          cudaStreamEndCapture(s, &g);
          cudaGraphInstantiate(&ge, g, 0);
          cudaGraphLaunch(ge, s);
          cudaEventRecord(e0, s);
          cudaGraphLaunch(ge, s);
          cudaEventRecord(e1, s);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          const double us = ms * 1e3 / reps;
          printf("bytes=%zuMB tile=%d nst=%d bps=%d: %.1f us  %.0f GB/s\n", bytes >> 20, tile, nst, bps, us,
                 bytes / us / 1e3);
          cudaGraphExecDestroy(ge);
          cudaGraphDestroy(g);
        }
      }
    }
    for (int bps : {2, 4, 8}) {
      const int G = nsm * bps;
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int r = 0; r < reps; ++r) kldg<<<G, 256, 0, s>>>((const double2 *)buf, bytes / 16, out);
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e0, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / reps;
      printf("bytes=%zuMB LDG.128 bps=%d: %.1f us  %.0f GB/s\n", bytes >> 20, bps, us, bytes / us / 1e3);
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
