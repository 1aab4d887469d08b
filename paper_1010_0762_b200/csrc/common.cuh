// common.cuh -- scalar traits, error handling and small device helpers for
// the RBiCG sm_100a kernels.  Real (double) and complex (zc) arithmetic share
// one template code path; the conjugations follow the inner product
// (u, v) = u^* v of reading Q1.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <atomic>

#include "../../include/rbicg.h"

namespace rbicg {

struct __align__(16) zc {
  double x, y;
};

__host__ __device__ __forceinline__ zc mk(double a, double b) { zc r; r.x = a; r.y = b; return r; }

// ---------------------------------------------------------------- arithmetic
__host__ __device__ __forceinline__ double conj(double a) { return a; }
__host__ __device__ __forceinline__ zc conj(zc a) { return mk(a.x, -a.y); }
__host__ __device__ __forceinline__ double add(double a, double b) { return a + b; }
__host__ __device__ __forceinline__ zc add(zc a, zc b) { return mk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double sub(double a, double b) { return a - b; }
__host__ __device__ __forceinline__ zc sub(zc a, zc b) { return mk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double mul(double a, double b) { return a * b; }
__host__ __device__ __forceinline__ zc mul(zc a, zc b) {
  return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__host__ __device__ __forceinline__ double cmul(double a, double b) { return a * b; }
__host__ __device__ __forceinline__ zc cmul(zc a, zc b) {
  return mk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
// acc + a*b
__host__ __device__ __forceinline__ double mad(double a, double b, double c) { return fma(a, b, c); }
__host__ __device__ __forceinline__ zc mad(zc a, zc b, zc c) {
  return mk(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// acc + conj(a)*b
__host__ __device__ __forceinline__ double cmad(double a, double b, double c) { return fma(a, b, c); }
__host__ __device__ __forceinline__ zc cmad(zc a, zc b, zc c) {
  return mk(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
}
__host__ __device__ __forceinline__ double scal(double s, double a) { return s * a; }
__host__ __device__ __forceinline__ zc scal(double s, zc a) { return mk(s * a.x, s * a.y); }
__host__ __device__ __forceinline__ double abs2(double a) { return a * a; }
__host__ __device__ __forceinline__ double abs2(zc a) { return a.x * a.x + a.y * a.y; }
__host__ __device__ __forceinline__ double divd(double a, double b) { return a / b; }
__host__ __device__ __forceinline__ zc divd(zc a, zc b) {
  // Smith's algorithm is not needed at these magnitudes; plain formula as
  // numpy uses for complex128 division is NOT guaranteed identical -- parity
  // is judged to tolerance, not bitwise.
  double den = b.x * b.x + b.y * b.y;
  return mk((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}
template <typename T> __host__ __device__ __forceinline__ T zero();
template <> __host__ __device__ __forceinline__ double zero<double>() { return 0.0; }
template <> __host__ __device__ __forceinline__ zc zero<zc>() { return mk(0.0, 0.0); }
template <typename T> __host__ __device__ __forceinline__ T mk_re(double a);
template <> __host__ __device__ __forceinline__ double mk_re<double>(double a) { return a; }
template <> __host__ __device__ __forceinline__ zc mk_re<zc>(double a) { return mk(a, 0.0); }
__host__ __device__ __forceinline__ double neg(double a) { return -a; }
__host__ __device__ __forceinline__ zc neg(zc a) { return mk(-a.x, -a.y); }
__host__ __device__ __forceinline__ bool finite(double a) { return isfinite(a); }
__host__ __device__ __forceinline__ bool finite(zc a) { return isfinite(a.x) && isfinite(a.y); }
__host__ __device__ __forceinline__ bool iszero(double a) { return a == 0.0; }
__host__ __device__ __forceinline__ bool iszero(zc a) { return a.x == 0.0 && a.y == 0.0; }
__host__ __device__ __forceinline__ double re(double a) { return a; }
__host__ __device__ __forceinline__ double re(zc a) { return a.x; }
__host__ __device__ __forceinline__ double im(double) { return 0.0; }
__host__ __device__ __forceinline__ double im(zc a) { return a.y; }

// ---------------------------------------------------------------- warp/block
__device__ __forceinline__ double shfl_down(double v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
__device__ __forceinline__ zc shfl_down(zc v, int o) {
  return mk(__shfl_down_sync(0xffffffffu, v.x, o), __shfl_down_sync(0xffffffffu, v.y, o));
}
// Deterministic warp sum (fixed shuffle tree); result valid in lane 0.
template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = add(v, shfl_down(v, o));
  return v;
}
__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }
__device__ __forceinline__ zc ldcg(const zc *p) {
  double2 v = __ldcg(reinterpret_cast<const double2 *>(p));
  return mk(v.x, v.y);
}

// ---------------------------------------------------------------- launch count
extern std::atomic<int64_t> g_launches;
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// SM budget for the grids of the blocked kernels launched by this host thread
// (0: all SMs).  The overlapped cycle end runs its kernels under a cap so the
// loop's kernels keep SMs to dispatch onto (RBICG_SIDE_SMS).
extern thread_local int g_sm_cap;
extern thread_local bool g_pdl_off;   // launch without programmatic dependent launch
inline int sm_budget(int nsm) { return g_sm_cap > 0 && g_sm_cap < nsm ? g_sm_cap : nsm; }

// ---------------------------------------------------------------- errors
struct Err {
  int code;
};
#define RB_CUDA(call)                                                             \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess) {                                                      \
      fprintf(stderr, "rbicg: CUDA error %s at %s:%d: %s\n", cudaGetErrorName(_e), \
              __FILE__, __LINE__, cudaGetErrorString(_e));                        \
      throw ::rbicg::Err{RBICG_ECUDA};                                            \
    }                                                                             \
  } while (0)
#define RB_CHECK(cond, code)            \
  do {                                  \
    if (!(cond)) throw ::rbicg::Err{code}; \
  } while (0)

inline size_t wbytes(rbicg_dtype t) { return t == RBICG_C128 ? 16 : 8; }

}  // namespace rbicg
