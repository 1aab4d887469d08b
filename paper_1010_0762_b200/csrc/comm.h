// comm.h -- the collectives of the row-partitioned (multi-GPU) hot path
// (SURVEY.md §8(e)): the halo exchange before each SpMV pair (C-1), the sum
// of the per-iteration scalar batches (C-2, C-3), the Gram sums and the
// broadcast of the small host results of the cycle end (C-4, C-5).
//
// Two implementations of one interface, so the solver code is the same:
//   * CommNccl     one process per GPU; NCCL (dlopen'd) on the caller's
//                  stream -- stream-ordered and CUDA-graph capturable.
//   * CommThreads  "virtual ranks": P contexts in one process (one host thread
//                  each, normally all on one GPU) meeting at host barriers;
//                  every collective synchronises its stream, so the loop is
//                  not graph-captured.  Sums are taken in rank order.
// A context holds two channels (main loop, cycle-end worker) so collectives
// of the two host threads of a rank never interleave.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <memory>
#include <vector>

namespace rbicg {

struct HaloPlan {   // one matrix's neighbour lists (dist_plan.h Plan, device send list)
  int64_t nloc = 0, nghost = 0, nsend = 0;
  std::vector<int> send_nbr, recv_nbr;
  std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;
  int32_t *send_idx = nullptr;   // device, local row indices, per send neighbour
};

struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() {}
  // collectives may be captured into a CUDA graph
  virtual bool capturable() const = 0;
  // in-place sum over ranks of `count` doubles at device pointer p
  virtual void allreduce_dev(double *p, int64_t count, cudaStream_t s) = 0;
  // halo: `m` arrays; array v sends sendbuf[v][send_off[i] .. +send_cnt[i]) (units
  // of `unit` bytes, per send neighbour i) and receives recvbuf[v][recv_off[i] ..
  // +recv_cnt[i]); sendbuf[v] = send + v * nsend * unit, recvbuf[v] = recv + v * rstride
  virtual void exchange(const HaloPlan &h, const void *send, void *recv, int64_t rstride_bytes,
                        size_t unit, int m, cudaStream_t s) = 0;
  // blocking, host memory
  virtual void allreduce_host(double *v, int64_t count) = 0;
  virtual void bcast_host(void *v, size_t bytes, int root) = 0;
};

// key: 128 bytes identifying the group (ncclUniqueId for NCCL; any agreed
// token for virtual ranks).  channel 0 / 1.
std::unique_ptr<Comm> make_comm_nccl(int rank, int nranks, const uint8_t key[128], int device);
std::unique_ptr<Comm> split_comm_nccl(Comm *parent);   // second channel of the same group
std::unique_ptr<Comm> make_comm_threads(int rank, int nranks, const uint8_t key[128], int channel);
int nccl_unique_id(uint8_t out[128]);

}  // namespace rbicg
