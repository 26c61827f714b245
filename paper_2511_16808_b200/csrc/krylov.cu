// krylov.cu -- compile-time-NV dispatch of the FGMRES BLAS-1 kernels
// (k_krylov.cuh).  Separate translation unit: ~190 instantiations.
#include "runtime.cuh"
#include "k_krylov.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <unordered_map>

namespace hmg {

// Blocks of one full wave of `kernel` (occupancy API x SM count), capped by
// the work and by the partial buffer: a grid-stride stream with no tail wave.
template <typename K> static int wave_blocks(K kernel, int64_t len) {
  static std::mutex mu;
  static std::unordered_map<const void *, int> cache;
  int per_sm;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find((const void *)kernel);
    if (it == cache.end()) {
      int nb = 0, dev = 0, sms = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, KRY_THREADS, 0));
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      it = cache.emplace((const void *)kernel, std::max(1, nb) * sms).first;
    }
    per_sm = it->second;
  }
  const int64_t need = (len + KRY_THREADS - 1) / KRY_THREADS;
  return (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)per_sm, need, (int64_t)KRY_MAXBLK}));
}

template <typename TV, typename TW>
int krylov_multidot(int nv, bool self, const cplx<TV> *V, int64_t vstride, const cplx<TW> *w, int64_t len,
                    double2 *partial, cudaStream_t s) {
  const dim3 b(KRY_THREADS);
  if (self) {
    switch (nv) {
#define C_(N) case N: { auto k = k_multidot<TV, TW, N, true>; const int nb = wave_blocks(k, len); \
                        launch(k, dim3(nb), b, 0, s, V, vstride, w, len, partial); return nb; }
      HMG_NV_CASES(C_)
#undef C_
    }
  } else {
    switch (nv) {
#define C_(N) case N: { auto k = k_multidot<TV, TW, N, false>; const int nb = wave_blocks(k, len); \
                        launch(k, dim3(nb), b, 0, s, V, vstride, w, len, partial); return nb; }
      HMG_NV_CASES(C_)
#undef C_
    }
  }
  throw HmgError(HMG_EINVAL, "multidot: vector count out of range");
  return 0;
}

template <typename TV, typename TW>
int krylov_axpy(int nv, const cplx<TV> *V, int64_t vstride, const double2 *coef, const double *vscale, double sgn,
                cplx<TW> *w, int64_t len, double2 *partial_norm, cudaStream_t s) {
  const dim3 b(KRY_THREADS);
  if (partial_norm) {
    switch (nv) {
#define C_(N) case N: { auto k = k_multi_axpy<TV, TW, N, true>; const int nb = wave_blocks(k, len); \
                        launch(k, dim3(nb), b, 0, s, V, vstride, coef, vscale, sgn, w, len, partial_norm); return nb; }
      HMG_NV_CASES(C_)
#undef C_
    }
  } else {
    switch (nv) {
#define C_(N) case N: { auto k = k_multi_axpy<TV, TW, N, false>; const int nb = wave_blocks(k, len); \
                        launch(k, dim3(nb), b, 0, s, V, vstride, coef, vscale, sgn, w, len, (double2 *)nullptr); return nb; }
      HMG_NV_CASES(C_)
#undef C_
    }
  }
  throw HmgError(HMG_EINVAL, "multi_axpy: vector count out of range");
  return 0;
}

// c64 Arnoldi kernels can process two elements per thread and trip (loads of both first) up to
// HMG_KRY_U2_MAX basis vectors; measured slower at N = 4096 (multi-AXPY 275 -> 289 ms per solve
// with 10, 337 with 20), so the default is 0 (one element per trip)
static int u2max() {
  static const int v = std::getenv("HMG_KRY_U2_MAX") ? std::atoi(std::getenv("HMG_KRY_U2_MAX")) : 0;
  return v;
}

// c64 Arnoldi: 16-byte (two complex) loads
template <>
int krylov_multidot<float, float>(int nv, bool self, const float2 *V, int64_t vstride, const float2 *w, int64_t len,
                                  double2 *partial, cudaStream_t s) {
  if ((len & 1) || (vstride & 1) || (reinterpret_cast<uintptr_t>(V) & 15) || (reinterpret_cast<uintptr_t>(w) & 15))
    throw HmgError(HMG_EINVAL, "multidot: c64 vectors must be 16-byte aligned with even lengths");
  const dim3 b(KRY_THREADS);
  const float4 *V4 = reinterpret_cast<const float4 *>(V), *w4 = reinterpret_cast<const float4 *>(w);
  const int64_t len2 = len / 2, vs2 = vstride / 2;
  if (self) {
    switch (nv) {
#define C_(N) case N: { auto k = N <= u2max() ? k_multidot_f4<N, true, 2> : k_multidot_f4<N, true, 1>; \
                        const int nb = wave_blocks(k, len2); launch(k, dim3(nb), b, 0, s, V4, vs2, w4, len2, partial); return nb; }
      HMG_NV_CASES(C_)
#undef C_
    }
  } else {
    switch (nv) {
#define C_(N) case N: { auto k = N <= u2max() ? k_multidot_f4<N, false, 2> : k_multidot_f4<N, false, 1>; \
                        const int nb = wave_blocks(k, len2); launch(k, dim3(nb), b, 0, s, V4, vs2, w4, len2, partial); return nb; }
      HMG_NV_CASES(C_)
#undef C_
    }
  }
  throw HmgError(HMG_EINVAL, "multidot: vector count out of range");
  return 0;
}

template <>
int krylov_axpy<float, float>(int nv, const float2 *V, int64_t vstride, const double2 *coef, const double *vscale,
                              double sgn, float2 *w, int64_t len, double2 *partial_norm, cudaStream_t s) {
  if ((len & 1) || (vstride & 1) || (reinterpret_cast<uintptr_t>(V) & 15) || (reinterpret_cast<uintptr_t>(w) & 15))
    throw HmgError(HMG_EINVAL, "multi_axpy: c64 vectors must be 16-byte aligned with even lengths");
  const dim3 b(KRY_THREADS);
  const float4 *V4 = reinterpret_cast<const float4 *>(V);
  float4 *w4 = reinterpret_cast<float4 *>(w);
  const int64_t len2 = len / 2, vs2 = vstride / 2;
  if (partial_norm) {
    switch (nv) {
#define C_(N) case N: { auto k = N <= u2max() ? k_multi_axpy_f4<N, true, 2> : k_multi_axpy_f4<N, true, 1>; \
                        const int nb = wave_blocks(k, len2); \
                        launch(k, dim3(nb), b, 0, s, V4, vs2, coef, vscale, sgn, w4, len2, partial_norm); return nb; }
      HMG_NV_CASES(C_)
#undef C_
    }
  } else {
    switch (nv) {
#define C_(N) case N: { auto k = N <= u2max() ? k_multi_axpy_f4<N, false, 2> : k_multi_axpy_f4<N, false, 1>; \
                        const int nb = wave_blocks(k, len2); \
                        launch(k, dim3(nb), b, 0, s, V4, vs2, coef, vscale, sgn, w4, len2, (double2 *)nullptr); return nb; }
      HMG_NV_CASES(C_)
#undef C_
    }
  }
  throw HmgError(HMG_EINVAL, "multi_axpy: vector count out of range");
  return 0;
}

template int krylov_multidot<double, double>(int, bool, const double2 *, int64_t, const double2 *, int64_t, double2 *, cudaStream_t);
template int krylov_axpy<double, double>(int, const double2 *, int64_t, const double2 *, const double *, double, double2 *, int64_t, double2 *, cudaStream_t);
template int krylov_axpy<float, double>(int, const float2 *, int64_t, const double2 *, const double *, double, double2 *, int64_t, double2 *, cudaStream_t);

}  // namespace hmg
