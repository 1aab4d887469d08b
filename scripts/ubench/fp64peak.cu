// Micro-benchmark: fp64 throughput of this B200 -- mma.sync m8n8k4 f64 (DMMA,
// the only fp64 tensor-core form on sm_100a) and plain FFMA (DFMA) -- the
// compute ceiling of the cycle-end pencil Gram (blocks.cu k_gram_mma).
// Each warp runs ACC independent accumulator chains; one CTA of 256 threads
// per SM slot, 1..4 CTAs per SM.  Prints TFLOP/s (2 flops per FMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64peak fp64peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void __launch_bounds__(256) kdmma(int iters, double *out) {
  double d[ACC][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < ACC; ++i) d[i][0] = d[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int ACC>
__global__ void __launch_bounds__(256) kdfma(int iters, double *out) {
  double d[ACC];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < ACC; ++i) d[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) d[i] = fma(d[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += d[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int per = 1; per <= 4; per *= 2) {
    const int grid = nsm * per;
    for (int rep = 0; rep < 2; ++rep) {
      kdmma<8><<<grid, 256>>>(iters, out);
      cudaEventRecord(e0);
      kdmma<8><<<grid, 256>>>(iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = (double)grid * 8 /*warps*/ * iters * 8 /*ACC*/ * 512.0;
      if (rep) printf("dmma m8n8k4 f64: %d CTAs/SM x 8 warps, 8 chains: %.2f TFLOP/s (%.3f ms)\n", per,
                      flops / ms / 1e9, ms);
      kdfma<16><<<grid, 256>>>(iters, out);
      cudaEventRecord(e0);
      kdfma<16><<<grid, 256>>>(iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double f2 = (double)grid * 256 * iters * 16 * 2.0;
      if (rep) printf("dfma: %d CTAs/SM x 256 threads, 16 chains: %.2f TFLOP/s (%.3f ms)\n", per,
                      f2 / ms / 1e9, ms);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
