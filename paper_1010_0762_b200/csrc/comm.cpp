// comm.cpp -- NCCL and virtual-rank implementations of comm.h.
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/rbicg.h"
#include "common.cuh"

namespace rbicg {

// ================================================================= NCCL
// dlopen'd so the library loads without NCCL; path from $RBICG_NCCL (the
// Python binding points it at the NCCL that ships with torch).
static struct {
  std::once_flag once;
  void *h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommSplit) commSplit = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
} N;

static void nccl_load() {
  std::call_once(N.once, [] {
    const char *p = getenv("RBICG_NCCL");
    if (p) N.h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!N.h) N.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!N.h) return;
#define LD(f, nm) N.f = (decltype(N.f))dlsym(N.h, nm)
    LD(getUniqueId, "ncclGetUniqueId");
    LD(commInitRank, "ncclCommInitRank");
    LD(commSplit, "ncclCommSplit");
    LD(commDestroy, "ncclCommDestroy");
    LD(allReduce, "ncclAllReduce");
    LD(broadcast, "ncclBroadcast");
    LD(send, "ncclSend");
    LD(recv, "ncclRecv");
    LD(groupStart, "ncclGroupStart");
    LD(groupEnd, "ncclGroupEnd");
#undef LD
  });
  RB_CHECK(N.getUniqueId && N.commInitRank && N.commSplit && N.allReduce && N.broadcast &&
               N.send && N.recv && N.groupStart && N.groupEnd,
           RBICG_ENCCL);
}
#define RB_NCCL(call)                                                           \
  do {                                                                          \
    ncclResult_t _r = (call);                                                   \
    if (_r != ncclSuccess) {                                                    \
      fprintf(stderr, "rbicg: NCCL error %d at %s:%d\n", (int)_r, __FILE__, __LINE__); \
      throw ::rbicg::Err{RBICG_ENCCL};                                          \
    }                                                                           \
  } while (0)

int nccl_unique_id(uint8_t out[128]) {
  nccl_load();
  ncclUniqueId id;
  RB_NCCL(N.getUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
  return 0;
}

struct CommNccl : Comm {
  ncclComm_t comm = nullptr;
  double *scratch = nullptr;
  size_t scratch_n = 0;
  cudaStream_t hs = nullptr;   // stream of the blocking host collectives
  ~CommNccl() override {
    if (scratch) cudaFree(scratch);
    if (hs) cudaStreamDestroy(hs);
    if (comm && N.commDestroy) N.commDestroy(comm);
  }
  bool capturable() const override { return true; }
  void allreduce_dev(double *p, int64_t count, cudaStream_t s) override {
    RB_NCCL(N.allReduce(p, p, (size_t)count, ncclFloat64, ncclSum, comm, s));
  }
  void exchange(const HaloPlan &h, const void *send, void *recv, int64_t rstride, size_t unit, int m,
                cudaStream_t s) override {
    RB_NCCL(N.groupStart());
    for (int v = 0; v < m; ++v) {
      const char *sb = (const char *)send + (size_t)v * h.nsend * unit;
      char *rb = (char *)recv + (size_t)v * rstride;
      for (size_t i = 0; i < h.send_nbr.size(); ++i)
        RB_NCCL(N.send(sb + h.send_off[i] * unit, h.send_cnt[i] * unit, ncclUint8, h.send_nbr[i], comm, s));
      for (size_t i = 0; i < h.recv_nbr.size(); ++i)
        RB_NCCL(N.recv(rb + h.recv_off[i] * unit, h.recv_cnt[i] * unit, ncclUint8, h.recv_nbr[i], comm, s));
    }
    RB_NCCL(N.groupEnd());
  }
  void grow(size_t n) {
    if (n <= scratch_n) return;
    if (scratch) cudaFree(scratch);
    RB_CUDA(cudaMalloc(&scratch, n * sizeof(double)));
    scratch_n = n;
  }
  void allreduce_host(double *v, int64_t count) override {
    if (count <= 0) return;
    grow((size_t)count);
    RB_CUDA(cudaMemcpyAsync(scratch, v, count * sizeof(double), cudaMemcpyHostToDevice, hs));
    RB_NCCL(N.allReduce(scratch, scratch, (size_t)count, ncclFloat64, ncclSum, comm, hs));
    RB_CUDA(cudaMemcpyAsync(v, scratch, count * sizeof(double), cudaMemcpyDeviceToHost, hs));
    RB_CUDA(cudaStreamSynchronize(hs));
  }
  void bcast_host(void *v, size_t bytes, int root) override {
    if (!bytes) return;
    grow((bytes + 7) / 8);
    RB_CUDA(cudaMemcpyAsync(scratch, v, bytes, cudaMemcpyHostToDevice, hs));
    RB_NCCL(N.broadcast(scratch, scratch, bytes, ncclUint8, root, comm, hs));
    RB_CUDA(cudaMemcpyAsync(v, scratch, bytes, cudaMemcpyDeviceToHost, hs));
    RB_CUDA(cudaStreamSynchronize(hs));
  }
};

std::unique_ptr<Comm> make_comm_nccl(int rank, int nranks, const uint8_t key[128], int device) {
  nccl_load();
  auto c = std::make_unique<CommNccl>();
  c->rank = rank;
  c->nranks = nranks;
  ncclUniqueId id;
  memcpy(&id, key, 128);
  RB_CUDA(cudaSetDevice(device));
  RB_NCCL(N.commInitRank(&c->comm, nranks, id, rank));
  RB_CUDA(cudaStreamCreateWithFlags(&c->hs, cudaStreamNonBlocking));
  return c;
}

std::unique_ptr<Comm> split_comm_nccl(Comm *parent) {
  auto *p = dynamic_cast<CommNccl *>(parent);
  RB_CHECK(p != nullptr, RBICG_ESTATE);
  auto c = std::make_unique<CommNccl>();
  c->rank = p->rank;
  c->nranks = p->nranks;
  RB_NCCL(N.commSplit(p->comm, 0, p->rank, &c->comm, nullptr));
  RB_CUDA(cudaStreamCreateWithFlags(&c->hs, cudaStreamNonBlocking));
  return c;
}

// ================================================================= virtual ranks
// One group per (key, channel): a generation barrier and slots where each rank
// publishes what the others read between two barriers.
struct VGroup {
  int P = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void *> ptr;        // published pointers
  std::vector<const HaloPlan *> plan;   // published halo plans
};
static std::mutex g_vmu;
static std::map<std::string, std::shared_ptr<VGroup>> g_vgroups;

struct CommThreads : Comm {
  std::shared_ptr<VGroup> g;
  std::vector<double> tmp;
  bool capturable() const override { return false; }
  void barrier() {
    std::unique_lock<std::mutex> lk(g->mu);
    const uint64_t my = g->gen;
    if (++g->arrived == g->P) {
      g->arrived = 0;
      ++g->gen;
      g->cv.notify_all();
      return;
    }
    // a rank that never arrives means the ranks diverged: fail instead of hanging
    if (!g->cv.wait_for(lk, std::chrono::seconds(120), [&] { return g->gen != my; }))
      throw Err{RBICG_ESTATE};
  }
  void allreduce_dev(double *p, int64_t count, cudaStream_t s) override {
    if (count <= 0) return;
    RB_CUDA(cudaStreamSynchronize(s));
    g->ptr[rank] = p;
    barrier();
    std::vector<double> acc((size_t)count, 0.0), part((size_t)count);
    for (int q = 0; q < nranks; ++q) {   // rank order
      RB_CUDA(cudaMemcpy(part.data(), g->ptr[q], count * sizeof(double), cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < count; ++i) acc[i] += part[i];
    }
    barrier();   // every rank has read every buffer
    RB_CUDA(cudaMemcpyAsync(p, acc.data(), count * sizeof(double), cudaMemcpyHostToDevice, s));
    RB_CUDA(cudaStreamSynchronize(s));
  }
  void exchange(const HaloPlan &h, const void *send, void *recv, int64_t rstride, size_t unit, int m,
                cudaStream_t s) override {
    RB_CUDA(cudaStreamSynchronize(s));
    g->ptr[rank] = send;
    g->plan[rank] = &h;
    barrier();
    for (size_t i = 0; i < h.recv_nbr.size(); ++i) {
      const int o = h.recv_nbr[i];
      const HaloPlan &ho = *g->plan[o];
      size_t j = 0;
      while (j < ho.send_nbr.size() && ho.send_nbr[j] != rank) ++j;
      RB_CHECK(j < ho.send_nbr.size() && ho.send_cnt[j] == h.recv_cnt[i], RBICG_ESTATE);
      for (int v = 0; v < m; ++v) {
        const char *src = (const char *)g->ptr[o] + (size_t)v * ho.nsend * unit + ho.send_off[j] * unit;
        char *dst = (char *)recv + (size_t)v * rstride + h.recv_off[i] * unit;
        RB_CUDA(cudaMemcpyAsync(dst, src, h.recv_cnt[i] * unit, cudaMemcpyDeviceToDevice, s));
      }
    }
    RB_CUDA(cudaStreamSynchronize(s));
    barrier();   // senders may reuse their buffers
  }
  void allreduce_host(double *v, int64_t count) override {
    g->ptr[rank] = v;
    barrier();
    tmp.assign((size_t)count, 0.0);
    for (int q = 0; q < nranks; ++q) {
      const double *src = (const double *)g->ptr[q];
      for (int64_t i = 0; i < count; ++i) tmp[i] += src[i];
    }
    barrier();
    memcpy(v, tmp.data(), count * sizeof(double));
  }
  void bcast_host(void *v, size_t bytes, int root) override {
    g->ptr[rank] = v;
    barrier();
    if (rank != root) memcpy(v, g->ptr[root], bytes);
    barrier();
  }
};

std::unique_ptr<Comm> make_comm_threads(int rank, int nranks, const uint8_t key[128], int channel) {
  auto c = std::make_unique<CommThreads>();
  c->rank = rank;
  c->nranks = nranks;
  std::string k((const char *)key, 128);
  k += (char)('0' + channel);
  std::lock_guard<std::mutex> lk(g_vmu);
  auto &slot = g_vgroups[k];
  if (!slot || slot->P != nranks) {
    slot = std::make_shared<VGroup>();
    slot->P = nranks;
    slot->ptr.assign(nranks, nullptr);
    slot->plan.assign(nranks, nullptr);
  }
  c->g = slot;
  return c;
}

}  // namespace rbicg
