// comm.cu -- communication backends of the slab-partitioned solve
// (SURVEY §8(e)): halo exchange of slab-axis ghost planes, allreduce of the
// FGMRES dot products, allgather of the first replicated coarse level.
//
//   NCCL  : one process per GPU; libnccl is dlopen'ed (the copy torch already
//           loaded, else the system one), ncclSend/Recv in a group for halos,
//           ncclAllReduce (sum, fp64) for dots, grouped ncclBroadcast for the
//           allgather.  Stream-ordered, no host synchronisation.
//   LOCAL : k virtual ranks on ONE GPU, one host thread per rank, each with
//           its own stream.  Data moves by stream-ordered device-to-device
//           copies that wait on the peers' events; the ranks meet at host
//           barriers.  No kernel ever waits on another (the host orders
//           everything), so this is safe on a single device.  Reductions sum
//           the per-rank contributions in rank order on every rank, so all
//           ranks see bit-identical dot products and take identical branches.
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "runtime.cuh"

namespace hmg {

// ------------------------------------------------------------------ LOCAL
struct LocalGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int waiting = 0;
  long long gen = 0;
  std::vector<const void *> pa, pb;   // per-rank registered pointers
  std::vector<cudaEvent_t> ev, ev2;   // per-rank "data ready" / "copies done"
  double *stage = nullptr;            // n x 512 doubles (allreduce staging)
  explicit LocalGroup(int n_) : n(n_), pa(n_), pb(n_), ev(n_), ev2(n_) {
    CK(cudaMalloc(&stage, sizeof(double) * 512 * n));
  }
  ~LocalGroup() { cudaFree(stage); }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++waiting == n) {
      waiting = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

__global__ void k_sum_stage(const double *__restrict__ stage, int nranks, int n, double *__restrict__ out) {
  HMG_PDL_PROLOGUE();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = 0;
  for (int r = 0; r < nranks; ++r) a += stage[(size_t)r * 512 + i];   // rank order on every rank
  out[i] = a;
}

struct LocalComm : Comm {
  std::shared_ptr<LocalGroup> g;
  cudaEvent_t e1 = nullptr, e2 = nullptr;
  LocalComm(std::shared_ptr<LocalGroup> g_, int r) : g(std::move(g_)) {
    rank = r;
    size = g->n;
    CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
  }
  ~LocalComm() override {
    if (e1) cudaEventDestroy(e1);
    if (e2) cudaEventDestroy(e2);
  }
  void publish(const void *a, const void *b, cudaStream_t s) {
    g->pa[rank] = a;
    g->pb[rank] = b;
    CK(cudaEventRecord(e1, s));
    g->ev[rank] = e1;
    g->barrier();
  }
  void finish(cudaStream_t s, const std::vector<int> &readers) {
    CK(cudaEventRecord(e2, s));
    g->ev2[rank] = e2;
    g->barrier();
    // the peers that read my buffers must be done before my stream moves on
    for (int q : readers) CK(cudaStreamWaitEvent(s, g->ev2[q], 0));
    g->barrier();
  }
  void halo(const void *send_lo, void *recv_lo, const void *send_hi, void *recv_hi, size_t bytes,
            cudaStream_t s) override {
    publish(send_lo, send_hi, s);
    std::vector<int> peers;
    if (rank > 0) peers.push_back(rank - 1);
    if (rank < size - 1) peers.push_back(rank + 1);
    if (rank > 0 && recv_lo && g->pb[rank - 1]) {
      CK(cudaStreamWaitEvent(s, g->ev[rank - 1], 0));
      CK(cudaMemcpyAsync(recv_lo, g->pb[rank - 1], bytes, cudaMemcpyDeviceToDevice, s));
    }
    if (rank < size - 1 && recv_hi && g->pa[rank + 1]) {
      CK(cudaStreamWaitEvent(s, g->ev[rank + 1], 0));
      CK(cudaMemcpyAsync(recv_hi, g->pa[rank + 1], bytes, cudaMemcpyDeviceToDevice, s));
    }
    finish(s, peers);
  }
  void allreduce_sum(double *d, int n, cudaStream_t s) override {
    if (n > 512) throw HmgError(HMG_EINVAL, "allreduce: too many values");
    CK(cudaMemcpyAsync(g->stage + (size_t)rank * 512, d, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    publish(nullptr, nullptr, s);
    std::vector<int> all;
    for (int q = 0; q < size; ++q)
      if (q != rank) {
        CK(cudaStreamWaitEvent(s, g->ev[q], 0));
        all.push_back(q);
      }
    launch(k_sum_stage, dim3((n + 127) / 128), dim3(128), 0, s, (const double *)g->stage, size, n, d);
    finish(s, all);
  }
  void allgatherv(void *buf, const std::vector<size_t> &off, const std::vector<size_t> &len,
                  cudaStream_t s) override {
    publish(buf, nullptr, s);
    std::vector<int> all;
    for (int q = 0; q < size; ++q) {
      if (q == rank) continue;
      all.push_back(q);
      if (!len[q]) continue;
      CK(cudaStreamWaitEvent(s, g->ev[q], 0));
      CK(cudaMemcpyAsync((char *)buf + off[q], (const char *)g->pa[q] + off[q], len[q], cudaMemcpyDeviceToDevice,
                         s));
    }
    finish(s, all);
  }
};

// ------------------------------------------------------------------ NCCL (dlopen)
namespace nccl {
typedef struct ncclComm *comm_t;
typedef struct { char internal[128]; } uid_t;
typedef int res_t;
enum { Uint8 = 1, Float64 = 8, Sum = 0 };
struct Api {
  void *h = nullptr;
  res_t (*GetUniqueId)(uid_t *);
  res_t (*CommInitRank)(comm_t *, int, uid_t, int);
  res_t (*CommDestroy)(comm_t);
  res_t (*GroupStart)();
  res_t (*GroupEnd)();
  res_t (*Send)(const void *, size_t, int, int, comm_t, cudaStream_t);
  res_t (*Recv)(void *, size_t, int, int, comm_t, cudaStream_t);
  res_t (*AllReduce)(const void *, void *, size_t, int, int, comm_t, cudaStream_t);
  res_t (*Broadcast)(const void *, void *, size_t, int, int, comm_t, cudaStream_t);
  const char *(*GetErrorString)(res_t);
};
static Api *api() {
  static Api a;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *n : names) {
      a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);   // the copy torch loaded, if any
      if (!a.h) a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) { err = "libnccl.so.2 not found"; return; }
#define S_(f) a.f = (decltype(a.f))dlsym(a.h, "nccl" #f); if (!a.f) { err = "missing nccl" #f; a.h = nullptr; return; }
    S_(GetUniqueId) S_(CommInitRank) S_(CommDestroy) S_(GroupStart) S_(GroupEnd) S_(Send) S_(Recv) S_(AllReduce)
    S_(Broadcast) S_(GetErrorString)
#undef S_
  });
  if (!a.h) throw HmgError(HMG_ENCCL, "NCCL unavailable: " + err);
  return &a;
}
#define NC(call)                                                                                    \
  do {                                                                                              \
    nccl::res_t r_ = (call);                                                                        \
    if (r_ != 0) throw HmgError(HMG_ENCCL, std::string(#call) + ": " + nccl::api()->GetErrorString(r_)); \
  } while (0)
}  // namespace nccl

struct NcclComm : Comm {
  nccl::comm_t c = nullptr;
  NcclComm(const void *uid, int r, int n) {
    rank = r;
    size = n;
    nccl::uid_t id;
    std::memcpy(&id, uid, sizeof id);
    NC(nccl::api()->CommInitRank(&c, n, id, r));
  }
  ~NcclComm() override {
    if (c) nccl::api()->CommDestroy(c);
  }
  void halo(const void *send_lo, void *recv_lo, const void *send_hi, void *recv_hi, size_t bytes,
            cudaStream_t s) override {
    auto *a = nccl::api();
    NC(a->GroupStart());
    if (rank > 0) {
      NC(a->Send(send_lo, bytes, nccl::Uint8, rank - 1, c, s));
      NC(a->Recv(recv_lo, bytes, nccl::Uint8, rank - 1, c, s));
    }
    if (rank < size - 1) {
      NC(a->Send(send_hi, bytes, nccl::Uint8, rank + 1, c, s));
      NC(a->Recv(recv_hi, bytes, nccl::Uint8, rank + 1, c, s));
    }
    NC(a->GroupEnd());
  }
  void halo_multi(const std::vector<HaloReq> &rq, cudaStream_t s) override {
    auto *a = nccl::api();
    NC(a->GroupStart());
    for (const HaloReq &q : rq) {
      if (rank > 0) {
        NC(a->Send(q.send_lo, q.bytes, nccl::Uint8, rank - 1, c, s));
        NC(a->Recv(q.recv_lo, q.bytes, nccl::Uint8, rank - 1, c, s));
      }
      if (rank < size - 1) {
        NC(a->Send(q.send_hi, q.bytes, nccl::Uint8, rank + 1, c, s));
        NC(a->Recv(q.recv_hi, q.bytes, nccl::Uint8, rank + 1, c, s));
      }
    }
    NC(a->GroupEnd());
  }
  // NCCL point-to-point and collectives are stream-ordered and graph-capturable
  bool capturable() const override { return true; }
  void allreduce_sum(double *d, int n, cudaStream_t s) override {
    NC(nccl::api()->AllReduce(d, d, n, nccl::Float64, nccl::Sum, c, s));
  }
  void allgatherv(void *buf, const std::vector<size_t> &off, const std::vector<size_t> &len,
                  cudaStream_t s) override {
    auto *a = nccl::api();
    NC(a->GroupStart());
    for (int q = 0; q < size; ++q)
      if (len[q]) NC(a->Broadcast((char *)buf + off[q], (char *)buf + off[q], len[q], nccl::Uint8, q, c, s));
    NC(a->GroupEnd());
  }
};

std::shared_ptr<void> local_group_create(int n) { return std::make_shared<LocalGroup>(n); }
Comm *local_comm_create(const std::shared_ptr<void> &group, int rank) {
  auto g = std::static_pointer_cast<LocalGroup>(group);
  if (rank < 0 || rank >= g->n) throw HmgError(HMG_EINVAL, "rank out of range");
  return new LocalComm(g, rank);
}
void nccl_unique_id(void *out128) {
  nccl::uid_t id;
  NC(nccl::api()->GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof id);
}
Comm *nccl_comm_create(const void *uid, int rank, int n) { return new NcclComm(uid, rank, n); }

}  // namespace hmg
