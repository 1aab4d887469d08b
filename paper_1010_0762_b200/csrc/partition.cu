// partition.cu -- the row-block matrix store of the partitioned path
// (the sequence's matrices A^{(j)}).
//
// Every rank passes ITS contiguous block of rows of A: a local rowptr and
// GLOBAL column indices (rank order = row order; blocks need not be even).
// Nothing global is ever assembled:
//   * row ranges: one host allreduce of the P block sizes;
//   * rows of A^* in the block, A^*[i, j] = conj(a_ji) for own i: the rank's
//     own entries with an own column, plus the entries of A in its columns
//     that other ranks hold -- those arrive as (column, row, value) triplets
//     over the communicator (the value halo, SURVEY C-8), exchanged per system
//     because the values change; assembled and sorted on the device (CUB);
//   * ghost columns (columns of the block's rows of A and A^* owned elsewhere),
//     the per-neighbour receive ranges and the send lists: the ghost ids are
//     requested from their owners through the communicator.  This plan depends
//     only on the sparsity pattern, which a sequence keeps, so it is cached per
//     context under a hash of the block's pattern (device-computed) and
//     rebuilt only when the hash, the block or the partition changes.
// Local column indices: own column c -> c - r0; ghost g -> nloc + position in
// the sorted ghost list (the ghosts of one owner are contiguous), which is the
// layout the halo kernels and the SpMV gathers expect (internal.h HaloPlan).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <numeric>

#include "internal.h"

namespace rbicg {

namespace {

template <typename T> struct Trip {   // one entry a_jc of A sent to the owner of column c
  int64_t c, j;
  T v;
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {   // splitmix64 finaliser
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

// pattern hash: a sum (mod 2^64) of per-entry mixes -- order independent, so
// the atomics make it deterministic
__global__ void k_pattern_hash(const int32_t *rp, const int32_t *ci, int64_t nloc,
                               unsigned long long *h) {
  uint64_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nloc;
       i += (int64_t)gridDim.x * blockDim.x) {
    acc += mix64(((uint64_t)i << 1) ^ (uint64_t)rp[i + 1]);
    for (int32_t e = rp[i]; e < rp[i + 1]; ++e)
      acc += mix64(((uint64_t)i << 32) ^ (uint64_t)(uint32_t)ci[e] ^ 0x9e3779b97f4a7c15ull);
  }
  atomicAdd(h, (unsigned long long)acc);
}

__global__ void k_row_of(const int32_t *rp, int64_t nloc, int32_t *row) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nloc;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int32_t e = rp[i]; e < rp[i + 1]; ++e) row[e] = (int32_t)i;
}

__device__ __forceinline__ int owner_dev(const int64_t *rbeg, int P, int64_t c) {
  int lo = 0, hi = P - 1;   // largest q with rbeg[q] <= c
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (rbeg[mid] <= c) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

struct ForeignCol {
  const int32_t *ci;
  int64_t r0, r1;
  __device__ bool operator()(const int64_t &e) const {
    const int64_t c = ci[e];
    return c < r0 || c >= r1;
  }
};

// export triplets of the foreign-column entries (positions pos[0..m)) and
// their destination ranks (the radix-sort keys)
template <typename T>
__global__ void k_pack_exports(const int64_t *pos, int64_t m, const int32_t *row, const int32_t *ci,
                               const T *v, int64_t r0, const int64_t *rbeg, int P, Trip<T> *out,
                               int32_t *dest, unsigned *cnt) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = pos[t];
    Trip<T> tr;
    tr.c = ci[e];
    tr.j = r0 + row[e];
    tr.v = v[e];
    out[t] = tr;
    const int d = owner_dev(rbeg, P, tr.c);
    dest[t] = d;
    atomicAdd(&cnt[d], 1u);
  }
}

template <typename T>
__global__ void k_permute_trips(const Trip<T> *in, const int32_t *perm, int64_t m, Trip<T> *out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = in[perm[t]];
}

// A^* COO of the block: own entries with an own column (row = c - r0, column
// = global row j) and the imported triplets; key = row * nglob + column
template <typename T>
__global__ void k_adj_coo(const int32_t *row, const int32_t *ci, const T *v, int64_t nnz, int64_t r0,
                          int64_t r1, const Trip<T> *imp, int64_t nimp, int64_t nglob,
                          unsigned long long *key, T *val, int64_t *cursor) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz + nimp;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rr, cc;
    T a;
    if (e < nnz) {
      const int64_t c = ci[e];
      if (c < r0 || c >= r1) continue;
      rr = c - r0;
      cc = r0 + row[e];
      a = v[e];
    } else {
      const Trip<T> t = imp[e - nnz];
      rr = t.c - r0;
      cc = t.j;
      a = t.v;
    }
    const int64_t slot = atomicAdd((unsigned long long *)cursor, 1ull);
    key[slot] = (unsigned long long)rr * (unsigned long long)nglob + (unsigned long long)cc;
    val[slot] = conj(a);
  }
}

template <typename T>
__global__ void k_adj_split(const unsigned long long *key, const int32_t *perm, const T *val_in,
                            int64_t m, int64_t nglob, int64_t *colg, T *val, int32_t *rowcnt) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = key[t];
    const int64_t r = (int64_t)(k / (unsigned long long)nglob);
    colg[t] = (int64_t)(k % (unsigned long long)nglob);
    val[t] = val_in[perm[t]];
    atomicAdd(&rowcnt[r], 1);
  }
}

// global column -> local: own c - r0, ghost nloc + lower_bound(ghost, c)
template <typename I>
__global__ void k_local_cols(const I *cg, int64_t m, int64_t r0, int64_t r1, int64_t nloc,
                             const int64_t *ghost, int64_t ng, int32_t *cl) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cg[t];
    if (c >= r0 && c < r1) {
      cl[t] = (int32_t)(c - r0);
    } else {
      int64_t lo = 0, hi = ng;
      while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (ghost[mid] < c) lo = mid + 1;
        else hi = mid;
      }
      cl[t] = (int32_t)(nloc + lo);
    }
  }
}

__global__ void k_iota(int32_t *v, int64_t m) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x)
    v[t] = (int32_t)t;
}

int grid_of(int64_t m) { return (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 4096)); }

// A HaloPlan-shaped exchange plan from a P x P count matrix (cnt[src * P + dst]):
// this rank sends cnt[q][d] units to every d, receives cnt[s][q] from every s.
HaloPlan xplan_from(const std::vector<double> &cnt, int P, int q) {
  HaloPlan h;
  int64_t off = 0;
  for (int d = 0; d < P; ++d) {
    const int64_t c = (int64_t)cnt[(size_t)q * P + d];
    if (d == q || c == 0) continue;
    h.send_nbr.push_back(d);
    h.send_off.push_back(off);
    h.send_cnt.push_back(c);
    off += c;
  }
  h.nsend = off;
  off = 0;
  for (int src = 0; src < P; ++src) {
    const int64_t c = (int64_t)cnt[(size_t)src * P + q];
    if (src == q || c == 0) continue;
    h.recv_nbr.push_back(src);
    h.recv_off.push_back(off);
    h.recv_cnt.push_back(c);
    off += c;
  }
  h.nghost = off;
  return h;
}

struct CachedPlan {
  uint64_t hash = 0;
  int64_t nloc = -1, nnz = -1, r0 = -1, nglob = -1;
  std::vector<int64_t> ghost;
  HaloPlan halo;                 // send_idx kept host-side here
  std::vector<int32_t> send_idx;
};
std::mutex g_plan_mu;
std::map<const rbicg_ctx *, CachedPlan> g_plans;

template <typename T>
void build_block(rbicg_ctx *ctx, int64_t nloc, int64_t nnz, const int32_t *rp, const int32_t *ci,
                 const T *v, rbicg_dtype dt, rbicg_mat *M) {
  Comm *cm = ctx->comm.get();
  const int P = ctx->nranks, q = ctx->rank;
  cudaStream_t s = ctx->stream;
  std::vector<void *> tmp;
  auto dalloc = [&](size_t bytes) {
    void *p = ws_alloc(std::max<size_t>(bytes, 16));
    tmp.push_back(p);
    return p;
  };
  struct Free {
    std::vector<void *> &t;
    ~Free() {
      for (void *p : t) ws_free(p);
    }
  } fr{tmp};
  // ---- row ranges (rank order) and the pattern hash
  std::vector<double> sz(P, 0.0);
  sz[q] = (double)nloc;
  cm->allreduce_host(sz.data(), P);
  std::vector<int64_t> rbeg(P + 1, 0);
  for (int p = 0; p < P; ++p) rbeg[p + 1] = rbeg[p] + (int64_t)sz[p];
  const int64_t r0 = rbeg[q], r1 = rbeg[q + 1], nglob = rbeg[P];
  RB_CHECK(nglob < INT32_MAX, RBICG_EINVAL);
  int64_t *d_rbeg = (int64_t *)dalloc(sizeof(int64_t) * (P + 1));
  RB_CUDA(cudaMemcpyAsync(d_rbeg, rbeg.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, s));
  unsigned long long *d_h = (unsigned long long *)dalloc(8);
  RB_CUDA(cudaMemsetAsync(d_h, 0, 8, s));
  k_pattern_hash<<<grid_of(nloc), 256, 0, s>>>(rp, ci, nloc, d_h);
  int32_t *row = (int32_t *)dalloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  k_row_of<<<grid_of(nloc), 256, 0, s>>>(rp, nloc, row);
  count_launch(2);
  uint64_t hash = 0;
  RB_CUDA(cudaMemcpyAsync(&hash, d_h, 8, cudaMemcpyDeviceToHost, s));
  // ---- export triplets: own-row entries with a foreign column, by owner
  int64_t *pos = (int64_t *)dalloc(sizeof(int64_t) * std::max<int64_t>(nnz, 1));
  int64_t *d_nsel = (int64_t *)dalloc(sizeof(int64_t));
  {
    thrust::counting_iterator<int64_t> it(0);
    size_t tb = 0;
    cub::DeviceSelect::If(nullptr, tb, it, pos, d_nsel, nnz, ForeignCol{ci, r0, r1}, s);
    void *t = dalloc(tb);
    cub::DeviceSelect::If(t, tb, it, pos, d_nsel, nnz, ForeignCol{ci, r0, r1}, s);
  }
  int64_t nexp = 0;
  RB_CUDA(cudaMemcpyAsync(&nexp, d_nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  RB_CUDA(cudaStreamSynchronize(s));
  Trip<T> *exp0 = (Trip<T> *)dalloc(sizeof(Trip<T>) * std::max<int64_t>(nexp, 1));
  Trip<T> *expo = (Trip<T> *)dalloc(sizeof(Trip<T>) * std::max<int64_t>(nexp, 1));
  int32_t *dest = (int32_t *)dalloc(sizeof(int32_t) * std::max<int64_t>(nexp, 1));
  int32_t *dest2 = (int32_t *)dalloc(sizeof(int32_t) * std::max<int64_t>(nexp, 1));
  int32_t *iota = (int32_t *)dalloc(sizeof(int32_t) * std::max<int64_t>(nexp, 1));
  int32_t *perm = (int32_t *)dalloc(sizeof(int32_t) * std::max<int64_t>(nexp, 1));
  unsigned *d_cnt = (unsigned *)dalloc(sizeof(unsigned) * P);
  RB_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned) * P, s));
  std::vector<unsigned> cnt(P, 0);
  if (nexp) {
    k_pack_exports<T><<<grid_of(nexp), 256, 0, s>>>(pos, nexp, row, ci, v, r0, d_rbeg, P, exp0, dest, d_cnt);
    k_iota<<<grid_of(nexp), 256, 0, s>>>(iota, nexp);
    int bits = 1;
    while ((1 << bits) < P) ++bits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, dest, dest2, iota, perm, (int)nexp, 0, bits, s);
    void *t = dalloc(tb);
    cub::DeviceRadixSort::SortPairs(t, tb, dest, dest2, iota, perm, (int)nexp, 0, bits, s);   // stable
    k_permute_trips<T><<<grid_of(nexp), 256, 0, s>>>(exp0, perm, nexp, expo);
    count_launch(2);
    RB_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(unsigned) * P, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
  }
  std::vector<double> cmat((size_t)P * P, 0.0);
  for (int d = 0; d < P; ++d) cmat[(size_t)q * P + d] = (double)cnt[d];
  cm->allreduce_host(cmat.data(), (int64_t)P * P);
  const HaloPlan xp = xplan_from(cmat, P, q);
  RB_CHECK(xp.nsend == nexp, RBICG_ESTATE);
  const int64_t nimp = xp.nghost;
  Trip<T> *imp = (Trip<T> *)dalloc(sizeof(Trip<T>) * std::max<int64_t>(nimp, 1));
  cm->exchange(xp, expo, imp, 0, sizeof(Trip<T>), 1, s);
  // ---- halo plan (cached while the pattern and the partition repeat)
  CachedPlan pl;
  bool hit = false;
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_plans.find(ctx);
    hit = it != g_plans.end() && it->second.hash == hash && it->second.nloc == nloc &&
          it->second.nnz == nnz && it->second.r0 == r0 && it->second.nglob == nglob;
    if (hit) pl = it->second;
  }
  {   // every rank must agree to reuse
    std::vector<double> agree(1, hit ? 1.0 : 0.0);
    cm->allreduce_host(agree.data(), 1);
    hit = agree[0] == (double)P;
  }
  if (!hit) {
    // ghosts: foreign columns of the block's rows of A (export c) and of A^*
    // (import j), sorted and unique
    std::vector<Trip<T>> he(nexp), hi(nimp);
    if (nexp) RB_CUDA(cudaMemcpyAsync(he.data(), expo, sizeof(Trip<T>) * nexp, cudaMemcpyDeviceToHost, s));
    if (nimp) RB_CUDA(cudaMemcpyAsync(hi.data(), imp, sizeof(Trip<T>) * nimp, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> g;
    g.reserve(nexp + nimp);
    for (auto &t : he) g.push_back(t.c);
    for (auto &t : hi) g.push_back(t.j);
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    pl.ghost = g;
    HaloPlan &h = pl.halo;
    h.nloc = nloc;
    h.nghost = (int64_t)g.size();
    std::vector<double> req((size_t)P * P, 0.0);   // req[q][o]: ghosts q needs from o
    for (size_t i = 0; i < g.size(); ++i) {
      int o = (int)(std::upper_bound(rbeg.begin(), rbeg.end(), g[i]) - rbeg.begin()) - 1;
      if (h.recv_nbr.empty() || h.recv_nbr.back() != o) {
        h.recv_nbr.push_back(o);
        h.recv_off.push_back((int64_t)i);
        h.recv_cnt.push_back(0);
      }
      h.recv_cnt.back()++;
      req[(size_t)q * P + o] += 1.0;
    }
    cm->allreduce_host(req.data(), (int64_t)P * P);
    // ask the owners: my ghost ids go out grouped by owner, the ids other
    // ranks need from me come back -- in their ghost order
    const HaloPlan rq = xplan_from(req, P, q);
    int64_t *d_g = (int64_t *)dalloc(sizeof(int64_t) * std::max<size_t>(g.size(), 1));
    if (!g.empty())
      RB_CUDA(cudaMemcpyAsync(d_g, g.data(), sizeof(int64_t) * g.size(), cudaMemcpyHostToDevice, s));
    int64_t *d_want = (int64_t *)dalloc(sizeof(int64_t) * std::max<int64_t>(rq.nghost, 1));
    cm->exchange(rq, d_g, d_want, 0, sizeof(int64_t), 1, s);
    std::vector<int64_t> want(rq.nghost);
    if (rq.nghost)
      RB_CUDA(cudaMemcpyAsync(want.data(), d_want, sizeof(int64_t) * rq.nghost, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
    h.send_nbr = rq.recv_nbr;
    h.send_off = rq.recv_off;
    h.send_cnt = rq.recv_cnt;
    h.nsend = rq.nghost;
    pl.send_idx.resize(want.size());
    for (size_t i = 0; i < want.size(); ++i) {
      RB_CHECK(want[i] >= r0 && want[i] < r1, RBICG_ESTATE);
      pl.send_idx[i] = (int32_t)(want[i] - r0);
    }
    pl.hash = hash;
    pl.nloc = nloc;
    pl.nnz = nnz;
    pl.r0 = r0;
    pl.nglob = nglob;
    std::lock_guard<std::mutex> lk(g_plan_mu);
    g_plans[ctx] = pl;
  }
  const int64_t ng = (int64_t)pl.ghost.size();
  int64_t *d_ghost = (int64_t *)dalloc(sizeof(int64_t) * std::max<int64_t>(ng, 1));
  if (ng) RB_CUDA(cudaMemcpyAsync(d_ghost, pl.ghost.data(), sizeof(int64_t) * ng, cudaMemcpyHostToDevice, s));
  // ---- local columns of A
  int32_t *ciA = (int32_t *)dalloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  if (nnz) k_local_cols<int32_t><<<grid_of(nnz), 256, 0, s>>>(ci, nnz, r0, r1, nloc, d_ghost, ng, ciA);
  // ---- A^* rows of the block: COO -> sorted -> CSR with local columns
  const int64_t mH = (nnz - nexp) + nimp;
  unsigned long long *key = (unsigned long long *)dalloc(8 * std::max<int64_t>(mH, 1));
  unsigned long long *key2 = (unsigned long long *)dalloc(8 * std::max<int64_t>(mH, 1));
  T *valc = (T *)dalloc(sizeof(T) * std::max<int64_t>(mH, 1));
  T *valH = (T *)dalloc(sizeof(T) * std::max<int64_t>(mH, 1));
  int64_t *colg = (int64_t *)dalloc(sizeof(int64_t) * std::max<int64_t>(mH, 1));
  int32_t *ciH = (int32_t *)dalloc(sizeof(int32_t) * std::max<int64_t>(mH, 1));
  int32_t *io2 = (int32_t *)dalloc(sizeof(int32_t) * std::max<int64_t>(mH, 1));
  int32_t *pm2 = (int32_t *)dalloc(sizeof(int32_t) * std::max<int64_t>(mH, 1));
  int32_t *rcnt = (int32_t *)dalloc(sizeof(int32_t) * (nloc + 1));
  int32_t *rpH = (int32_t *)dalloc(sizeof(int32_t) * (nloc + 1));
  int64_t *cursor = (int64_t *)dalloc(sizeof(int64_t));
  RB_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int64_t), s));
  RB_CUDA(cudaMemsetAsync(rcnt, 0, sizeof(int32_t) * (nloc + 1), s));
  k_adj_coo<T><<<grid_of(nnz + nimp), 256, 0, s>>>(row, ci, v, nnz, r0, r1, imp, nimp, nglob, key, valc,
                                                   cursor);
  {
    if (mH) k_iota<<<grid_of(mH), 256, 0, s>>>(io2, mH);
    int bits = 1;
    while (bits < 64 && (1ull << bits) < (unsigned long long)nloc * (unsigned long long)nglob) ++bits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, io2, pm2, (int)mH, 0, bits, s);
    void *t = dalloc(tb);
    cub::DeviceRadixSort::SortPairs(t, tb, key, key2, io2, pm2, (int)mH, 0, bits, s);
    // (row, column) keys are unique, so the order -- and the values' order
    // after the atomic-slot assembly -- is deterministic
    k_adj_split<T><<<grid_of(mH), 256, 0, s>>>(key2, pm2, valc, mH, nglob, colg, valH, rcnt);
    size_t tb2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb2, rcnt, rpH, (int)(nloc + 1), s);
    void *t2 = dalloc(tb2);
    cub::DeviceScan::ExclusiveSum(t2, tb2, rcnt, rpH, (int)(nloc + 1), s);
    if (mH) k_local_cols<int64_t><<<grid_of(mH), 256, 0, s>>>(colg, mH, r0, r1, nloc, d_ghost, ng, ciH);
    count_launch(4);
  }
  build_matrix_local(ctx, nloc, rp, ciA, v, rpH, ciH, valH, dt, M);
  M->nnz = nnz;
  M->row_begin = r0;
  M->n_global = nglob;
  HaloPlan &h = M->halo;
  h = pl.halo;
  h.send_idx = (int32_t *)ws_alloc(4 * std::max<int64_t>(h.nsend, 1));
  if (h.nsend)
    RB_CUDA(cudaMemcpyAsync(h.send_idx, pl.send_idx.data(), 4 * h.nsend, cudaMemcpyHostToDevice, s));
  RB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

void build_partitioned(rbicg_ctx *ctx, int64_t nloc, int64_t nnz, const int32_t *rp, const int32_t *ci,
                       const void *v, rbicg_dtype dt, rbicg_mat *M) {
  if (dt == RBICG_F64) build_block<double>(ctx, nloc, nnz, rp, ci, (const double *)v, dt, M);
  else build_block<zc>(ctx, nloc, nnz, rp, ci, (const zc *)v, dt, M);
}

void forget_partition_plan(const rbicg_ctx *ctx) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  g_plans.erase(ctx);
}

}  // namespace rbicg
