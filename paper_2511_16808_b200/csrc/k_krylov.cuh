// k_krylov.cuh -- FGMRES BLAS-1: fused multi-dot,
// multi-AXPY (+norm), scale and solution update, all over the contiguous
// interior slab of the padded vectors (ghost entries are zero and stay zero).
// Dot products accumulate in fp64 for both precisions; reductions are
// deterministic (fixed grid, per-block partials, fixed-order final pass).
#pragma once
#include "common.cuh"

namespace hmg {

constexpr int KRY_THREADS = 256;
constexpr int KRY_MAXV = 32;  // vectors per multi-dot / multi-axpy pass

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// partial[i * nblk + block] = sum_e conj(V_i[e]) w[e],  i < nv
template <typename TV, typename TW = TV>
__global__ void __launch_bounds__(KRY_THREADS) k_multidot(const cplx<TV> *__restrict__ V, int64_t vstride, int nv,
                                                          const cplx<TW> *__restrict__ w, int64_t len,
                                                          double2 *__restrict__ partial) {
  double ar[KRY_MAXV], ai[KRY_MAXV];
#pragma unroll
  for (int i = 0; i < KRY_MAXV; ++i) ar[i] = ai[i] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += stride) {
    const cplx<TW> wv = w[e];
    const double wx = wv.x, wy = wv.y;
#pragma unroll
    for (int i = 0; i < KRY_MAXV; ++i) {
      if (i < nv) {
        const cplx<TV> v = V[(int64_t)i * vstride + e];
        ar[i] = fma((double)v.x, wx, fma((double)v.y, wy, ar[i]));
        ai[i] = fma((double)v.x, wy, fma(-(double)v.y, wx, ai[i]));
      }
    }
  }
  __shared__ double sr[KRY_THREADS / 32][KRY_MAXV], si[KRY_THREADS / 32][KRY_MAXV];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < KRY_MAXV; ++i) {
    if (i < nv) {
      const double a = warp_sum(ar[i]), b = warp_sum(ai[i]);
      if (lane == 0) { sr[wid][i] = a; si[wid][i] = b; }
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double a = 0, b = 0;
    for (int k = 0; k < KRY_THREADS / 32; ++k) { a += sr[k][threadIdx.x]; b += si[k][threadIdx.x]; }
    partial[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = make_double2(a, b);
  }
}

// out[i] = sum_b partial[i * nblk + b]  (one warp per i, fixed order)
__global__ void k_reduce_partials(const double2 *__restrict__ partial, int nblk, int nv, double2 *__restrict__ out) {
  const int i = blockIdx.x;
  if (i >= nv) return;
  double a = 0, b = 0;
  for (int k = threadIdx.x; k < nblk; k += 32) {
    a += partial[(int64_t)i * nblk + k].x;
    b += partial[(int64_t)i * nblk + k].y;
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if (threadIdx.x == 0) out[i] = make_double2(a, b);
}

// w <- w + sgn * sum_i coef[i] V_i  (coef on the device, fp64); if partial != nullptr
// also partial[block] = sum |w_new|^2 (fp64)
template <typename TV, typename TW = TV>
__global__ void __launch_bounds__(KRY_THREADS) k_multi_axpy(const cplx<TV> *__restrict__ V, int64_t vstride, int nv,
                                                            const double2 *__restrict__ coef, double sgn,
                                                            cplx<TW> *__restrict__ w, int64_t len,
                                                            double2 *__restrict__ partial) {
  __shared__ double2 sc[KRY_MAXV];
  if (threadIdx.x < nv) sc[threadIdx.x] = make_double2(sgn * coef[threadIdx.x].x, sgn * coef[threadIdx.x].y);
  __syncthreads();
  double nrm = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += stride) {
    const cplx<TW> wv = w[e];
    double x = wv.x, y = wv.y;
#pragma unroll
    for (int i = 0; i < KRY_MAXV; ++i) {
      if (i < nv) {
        const cplx<TV> v = V[(int64_t)i * vstride + e];
        const double2 c = sc[i];
        x = fma(c.x, (double)v.x, fma(-c.y, (double)v.y, x));
        y = fma(c.x, (double)v.y, fma(c.y, (double)v.x, y));
      }
    }
    const cplx<TW> o = mkc<TW>((TW)x, (TW)y);
    w[e] = o;
    nrm = fma((double)o.x, (double)o.x, fma((double)o.y, (double)o.y, nrm));
  }
  if (partial) {
    __shared__ double sn[KRY_THREADS / 32];
    nrm = warp_sum(nrm);
    if ((threadIdx.x & 31) == 0) sn[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0;
      for (int k = 0; k < KRY_THREADS / 32; ++k) a += sn[k];
      partial[blockIdx.x] = make_double2(a, 0.0);
    }
  }
}

// v <- s * w   (s real; optional precision conversion)
template <typename TI, typename TO = TI>
__global__ void k_scale(const cplx<TI> *__restrict__ w, cplx<TO> *__restrict__ v, double s, int64_t len) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += stride) {
    const cplx<TI> a = w[e];
    v[e] = mkc<TO>((TO)(s * (double)a.x), (TO)(s * (double)a.y));
  }
}

}  // namespace hmg
