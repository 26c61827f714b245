// runtime.cuh -- error type, launch helper and profiling hooks shared by the
// host-side translation units of libhmg (hmg.cu, krylov.cu).
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hmg.h"
#include "common.cuh"

namespace hmg {

struct HmgError : std::runtime_error {
  hmg_status st;
  HmgError(hmg_status s, const std::string &m) : std::runtime_error(m), st(s) {}
};

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      throw ::hmg::HmgError(e_ == cudaErrorMemoryAllocation ? HMG_ENOMEM : HMG_ECUDA,              \
                            std::string(#call) + ": " + cudaGetErrorString(e_));                   \
  } while (0)

// Tag the next launch with its kernel class, level and ALGORITHMIC bytes
// (DESIGN.md §5); consumed by launch() when profiling is on.
void tag(const char *name, int level, double bytes);
bool prof_active();
long long launch_count_now();
void add_launches(long long n);
int prof_before(cudaStream_t s);
void prof_after(cudaStream_t s, int idx);

// programmatic dependent launch on (non-legacy) streams (HMG_NO_PDL=1: plain launches)
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline void launch(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s, Args... args) {
  if (g.x == 0 || g.y == 0 || g.z == 0) return;
  const int pi = prof_before(s);
  if (s != nullptr && pdl_enabled()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
  } else {
    k<<<g, b, smem, s>>>(static_cast<KArgs>(args)...);
  }
  count_launch();
  CK(cudaGetLastError());
  prof_after(s, pi);
}

// Krylov launch dispatch (krylov.cu): nv is a runtime count in [1, 31]
// mapped onto the compile-time NV of the kernels.
// Each returns the number of blocks it launched (= partial columns written).
template <typename TV, typename TW>
int krylov_multidot(int nv, bool self, const cplx<TV> *V, int64_t vstride, const cplx<TW> *w, int64_t len,
                    double2 *partial, cudaStream_t s);
template <typename TV, typename TW>
int krylov_axpy(int nv, const cplx<TV> *V, int64_t vstride, const double2 *coef, const double *vscale, double sgn,
                cplx<TW> *w, int64_t len, double2 *partial_norm, cudaStream_t s);

// Communication of the slab-partitioned solve (comm.cu).  All calls are
// collective over the ranks and stream-ordered on `s`.
struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  // send `bytes` from send_lo to rank-1 and from send_hi to rank+1; receive
  // the matching blocks into recv_lo (from rank-1) and recv_hi (from rank+1)
  virtual void halo(const void *send_lo, void *recv_lo, const void *send_hi, void *recv_hi, size_t bytes,
                    cudaStream_t s) = 0;
  // several halo exchanges as ONE communication step (NCCL: one group; LOCAL: in turn)
  struct HaloReq {
    const void *send_lo;
    void *recv_lo;
    const void *send_hi;
    void *recv_hi;
    size_t bytes;
  };
  virtual void halo_multi(const std::vector<HaloReq> &rq, cudaStream_t s) {
    for (const HaloReq &r : rq) halo(r.send_lo, r.recv_lo, r.send_hi, r.recv_hi, r.bytes, s);
  }
  // may the calls be captured into a CUDA graph (stream-ordered device work only)?
  virtual bool capturable() const { return false; }
  virtual void allreduce_sum(double *d, int n, cudaStream_t s) = 0;   // in place, device fp64
  // rank q owns bytes [off[q], off[q] + len[q]) of buf (same layout on every
  // rank); afterwards every rank holds all of them
  virtual void allgatherv(void *buf, const std::vector<size_t> &off, const std::vector<size_t> &len,
                          cudaStream_t s) = 0;
};
std::shared_ptr<void> local_group_create(int n);
Comm *local_comm_create(const std::shared_ptr<void> &group, int rank);
void nccl_unique_id(void *out128);
Comm *nccl_comm_create(const void *uid, int rank, int n);

// c64 Arnoldi kernels use 16-byte loads (explicit specialisations in krylov.cu)
template <>
int krylov_multidot<float, float>(int nv, bool self, const float2 *V, int64_t vstride, const float2 *w, int64_t len,
                                  double2 *partial, cudaStream_t s);
template <>
int krylov_axpy<float, float>(int nv, const float2 *V, int64_t vstride, const double2 *coef, const double *vscale,
                              double sgn, float2 *w, int64_t len, double2 *partial_norm, cudaStream_t s);

}  // namespace hmg
