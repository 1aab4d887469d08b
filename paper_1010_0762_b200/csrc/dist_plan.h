// dist_plan.h -- row-partition plan (host), see dist.cpp.
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

namespace rbicg {

struct Plan {
  int P = 1, q = 0;
  int64_t r0 = 0, r1 = 0, nloc = 0;
  std::vector<int64_t> ghost;                 // sorted global ids
  std::vector<int> recv_nbr;                  // owner ranks, ascending
  std::vector<int64_t> recv_off, recv_cnt;    // ranges inside the ghost block
  std::vector<int> send_nbr;
  std::vector<int64_t> send_off, send_cnt;    // ranges inside send_idx
  std::vector<int32_t> send_idx;              // local own indices
  int64_t next() const { return nloc + (int64_t)ghost.size(); }
};

int64_t part_begin(int64_t n, int P, int q);
int owner_of(int64_t n, int P, int64_t c);
std::vector<int64_t> ghost_set(int64_t n, const int32_t *rowptr, const int32_t *col, int P, int q);
Plan make_plan(int64_t n, const int32_t *rowptr, const int32_t *col, int P, int q);
int64_t local_col(const Plan &pl, int64_t c);
void local_csr(const Plan &pl, int64_t n, const int32_t *rowptr, const int32_t *col,
               const void *val, size_t w, bool cplx, bool adjoint, std::vector<int32_t> &rp,
               std::vector<int32_t> &cl, std::vector<unsigned char> &vv);

}  // namespace rbicg
