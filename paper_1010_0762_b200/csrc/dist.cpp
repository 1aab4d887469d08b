// dist.cpp -- host-side row-partition planning for the multi-GPU path
// (SURVEY.md §8(e)): contiguous row blocks, ghost columns of the SpMV pair,
// per-neighbour receive ranges and send lists.  Pure host code (no CUDA), so
// the planning is testable on CPU (tests/test_dist_plan.py, gloo).
//
// Conventions (shared with the device halo kernels):
//   * rank q owns global rows [r0(q), r1(q)), r0(q) = floor(q n / P).
//   * local column index of an own column c is c - r0; ghost columns (those
//     referenced by the local rows of A or of A^* but owned elsewhere) are
//     sorted by global index and appended after the own block, so the ghosts
//     received from one neighbour are contiguous.
//   * send list to neighbour q': the own rows (local indices, ascending) that
//     appear in q''s ghost set, in q''s ghost order.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/rbicg.h"
#include "dist_plan.h"

namespace rbicg {

int64_t part_begin(int64_t n, int P, int q) { return (int64_t)((__int128)n * q / P); }

int owner_of(int64_t n, int P, int64_t c) {
  // smallest q with part_begin(q+1) > c
  int lo = 0, hi = P - 1;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (part_begin(n, P, mid + 1) > c) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// Columns of A^* rows [r0, r1) = rows i of A with a nonzero in a column of
// [r0, r1): computed from the global CSR by a scan (no transpose needed for
// the ghost set).
static void transpose_rows(int64_t n, const int32_t *rowptr, const int32_t *col, int64_t r0,
                           int64_t r1, std::vector<std::vector<int64_t>> &rows_of_col) {
  rows_of_col.assign(r1 - r0, {});
  for (int64_t i = 0; i < n; ++i)
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int64_t c = col[e];
      if (c >= r0 && c < r1) rows_of_col[c - r0].push_back(i);
    }
}

std::vector<int64_t> ghost_set(int64_t n, const int32_t *rowptr, const int32_t *col, int P,
                               int q) {
  const int64_t r0 = part_begin(n, P, q), r1 = part_begin(n, P, q + 1);
  std::vector<int64_t> g;
  for (int64_t i = r0; i < r1; ++i)
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
      if (col[e] < r0 || col[e] >= r1) g.push_back(col[e]);
  std::vector<std::vector<int64_t>> roc;
  transpose_rows(n, rowptr, col, r0, r1, roc);
  for (auto &v : roc)
    for (int64_t i : v)
      if (i < r0 || i >= r1) g.push_back(i);
  std::sort(g.begin(), g.end());
  g.erase(std::unique(g.begin(), g.end()), g.end());
  return g;
}

Plan make_plan(int64_t n, const int32_t *rowptr, const int32_t *col, int P, int q) {
  Plan pl;
  pl.P = P;
  pl.q = q;
  pl.r0 = part_begin(n, P, q);
  pl.r1 = part_begin(n, P, q + 1);
  pl.nloc = pl.r1 - pl.r0;
  pl.ghost = ghost_set(n, rowptr, col, P, q);
  // receive plan: ghosts grouped by owner (ascending = contiguous)
  for (size_t g = 0; g < pl.ghost.size(); ++g) {
    const int o = owner_of(n, P, pl.ghost[g]);
    if (pl.recv_nbr.empty() || pl.recv_nbr.back() != o) {
      pl.recv_nbr.push_back(o);
      pl.recv_off.push_back((int64_t)g);
      pl.recv_cnt.push_back(0);
    }
    pl.recv_cnt.back()++;
  }
  // send plan: for every other rank, which of my rows are in its ghost set
  for (int o = 0; o < P; ++o) {
    if (o == q) continue;
    const std::vector<int64_t> go = ghost_set(n, rowptr, col, P, o);
    std::vector<int32_t> idx;
    for (int64_t c : go)
      if (c >= pl.r0 && c < pl.r1) idx.push_back((int32_t)(c - pl.r0));
    if (!idx.empty()) {
      pl.send_nbr.push_back(o);
      pl.send_off.push_back((int64_t)pl.send_idx.size());
      pl.send_cnt.push_back((int64_t)idx.size());
      pl.send_idx.insert(pl.send_idx.end(), idx.begin(), idx.end());
    }
  }
  return pl;
}

int64_t local_col(const Plan &pl, int64_t c) {
  if (c >= pl.r0 && c < pl.r1) return c - pl.r0;
  auto it = std::lower_bound(pl.ghost.begin(), pl.ghost.end(), c);
  return pl.nloc + (int64_t)(it - pl.ghost.begin());
}

// Local CSR of rows [r0, r1) of A (and of A^*, built from the global CSR)
// with local column indices.  vals of w bytes each; A^* values conjugated
// when cplx.
void local_csr(const Plan &pl, int64_t n, const int32_t *rowptr, const int32_t *col,
               const void *val, size_t w, bool cplx, bool adjoint, std::vector<int32_t> &rp,
               std::vector<int32_t> &cl, std::vector<unsigned char> &vv) {
  rp.assign(pl.nloc + 1, 0);
  cl.clear();
  vv.clear();
  const unsigned char *V = (const unsigned char *)val;
  if (!adjoint) {
    for (int64_t i = pl.r0; i < pl.r1; ++i) {
      for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
        cl.push_back((int32_t)local_col(pl, col[e]));
        vv.insert(vv.end(), V + (size_t)e * w, V + (size_t)(e + 1) * w);
      }
      rp[i - pl.r0 + 1] = (int32_t)cl.size();
    }
    return;
  }
  // rows of A^* = columns of A, entries in ascending row order of A
  std::vector<std::vector<std::pair<int64_t, int64_t>>> rows(pl.nloc);
  for (int64_t i = 0; i < n; ++i)
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int64_t c = col[e];
      if (c >= pl.r0 && c < pl.r1) rows[c - pl.r0].emplace_back(i, e);
    }
  for (int64_t r = 0; r < pl.nloc; ++r) {
    for (auto &ie : rows[r]) {
      cl.push_back((int32_t)local_col(pl, ie.first));
      const unsigned char *src = V + (size_t)ie.second * w;
      size_t at = vv.size();
      vv.insert(vv.end(), src, src + w);
      if (cplx) {   // conjugate: negate the imaginary double
        double im;
        memcpy(&im, &vv[at + 8], 8);
        im = -im;
        memcpy(&vv[at + 8], &im, 8);
      }
    }
    rp[r + 1] = (int32_t)cl.size();
  }
}

}  // namespace rbicg

using namespace rbicg;

// C ABI: partition plan of `rank` (see include/rbicg.h).
int rbicg_plan_partition(int64_t n, const int32_t *rowptr, const int32_t *colind, int32_t nranks,
                         int32_t rank, int64_t *counts, int64_t *ghost, int32_t *recv_nbr,
                         int64_t *recv_cnt, int32_t *send_nbr, int64_t *send_cnt,
                         int32_t *send_idx) {
  if (n <= 0 || !rowptr || !colind || nranks < 1 || rank < 0 || rank >= nranks || !counts)
    return RBICG_EINVAL;
  try {
    const Plan pl = make_plan(n, rowptr, colind, nranks, rank);
    counts[0] = pl.r0;
    counts[1] = pl.r1;
    counts[2] = (int64_t)pl.ghost.size();
    counts[3] = (int64_t)pl.recv_nbr.size();
    counts[4] = (int64_t)pl.send_nbr.size();
    counts[5] = (int64_t)pl.send_idx.size();
    if (ghost) std::copy(pl.ghost.begin(), pl.ghost.end(), ghost);
    if (recv_nbr) std::copy(pl.recv_nbr.begin(), pl.recv_nbr.end(), recv_nbr);
    if (recv_cnt) std::copy(pl.recv_cnt.begin(), pl.recv_cnt.end(), recv_cnt);
    if (send_nbr) std::copy(pl.send_nbr.begin(), pl.send_nbr.end(), send_nbr);
    if (send_cnt) std::copy(pl.send_cnt.begin(), pl.send_cnt.end(), send_cnt);
    if (send_idx) std::copy(pl.send_idx.begin(), pl.send_idx.end(), send_idx);
  } catch (...) {
    return RBICG_ENOMEM;
  }
  return 0;
}
