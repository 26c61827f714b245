// k_krylov.cuh -- FGMRES BLAS-1: fused multi-dot
// (+ self norm), multi-AXPY (+ norm), scale, all over the contiguous interior
// slab of the padded vectors (ghost entries are zero and stay zero).
// Dot products accumulate in fp64 for both precisions; reductions are
// deterministic (fixed grid, per-block partials, fixed-order final pass).
// The number of basis vectors NV is a compile-time parameter (dispatch in
// hmg.cu), so each thread issues all NV loads of an element back to back:
// the kernels are pure streams at HBM speed.
#pragma once
#include "common.cuh"

namespace hmg {

constexpr int KRY_THREADS = 256;
constexpr int KRY_MAXV = 32;      // partial-buffer rows: NV dots + 1 self norm
constexpr int KRY_MAXBLK = 2048;  // partial-buffer columns (>= one full wave of blocks)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// partial[i * nblk + block] = sum_e conj(V_i[e]) w[e]   (i < NV)
// partial[NV * nblk + block] = sum_e |w[e]|^2           (if SELF)
template <typename TV, typename TW, int NV, bool SELF>
__global__ void __launch_bounds__(KRY_THREADS) k_multidot(const cplx<TV> *__restrict__ V, int64_t vstride,
                                                          const cplx<TW> *__restrict__ w, int64_t len,
                                                          double2 *__restrict__ partial) {
  HMG_PDL_PROLOGUE();
  constexpr int NA = NV + (SELF ? 1 : 0);
  constexpr int U = NV <= 2 ? 4 : NV <= 5 ? 2 : 1;   // elements per thread per pass: >= ~8 loads in flight
  double ar[NA], ai[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) ar[i] = ai[i] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < len; e0 += stride * U) {
    cplx<TV> v[U][NV];
    cplx<TW> wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      if (e < len) {
#pragma unroll
        for (int i = 0; i < NV; ++i) v[u][i] = V[(int64_t)i * vstride + e];
        wv[u] = w[e];
      } else {
#pragma unroll
        for (int i = 0; i < NV; ++i) v[u][i] = mkc<TV>(0, 0);
        wv[u] = mkc<TW>(0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double wx = wv[u].x, wy = wv[u].y;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        ar[i] = fma((double)v[u][i].x, wx, fma((double)v[u][i].y, wy, ar[i]));
        ai[i] = fma((double)v[u][i].x, wy, fma(-(double)v[u][i].y, wx, ai[i]));
      }
      if (SELF) ar[NV] = fma(wx, wx, fma(wy, wy, ar[NV]));
    }
  }
  __shared__ double sr[KRY_THREADS / 32][NA], si[KRY_THREADS / 32][NA];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    const double a = warp_sum(ar[i]), b = warp_sum(ai[i]);
    if (lane == 0) { sr[wid][i] = a; si[wid][i] = b; }
  }
  __syncthreads();
  if (threadIdx.x < NA) {
    double a = 0, b = 0;
#pragma unroll
    for (int k = 0; k < KRY_THREADS / 32; ++k) { a += sr[k][threadIdx.x]; b += si[k][threadIdx.x]; }
    partial[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = make_double2(a, b);
  }
}

// out[i] = sum_b partial[i * nblk + b]  (one warp per i, fixed order)
static __global__ void k_reduce_partials(const double2 *__restrict__ partial, int nblk, int nv, double2 *__restrict__ out) {
  HMG_PDL_PROLOGUE();
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

// w <- w + sgn * sum_i coef[i] V_i  (coef on the device, fp64); if NORM also
// partial[block] = sum |w_new|^2 (fp64, of the stored value)
// (vscale != nullptr: coefficient i is further multiplied by vscale[i] -- the
// 1/beta_i^2 of FGMRES's lazily normalised basis)
template <typename TV, typename TW, int NV, bool NORM>
__global__ void __launch_bounds__(KRY_THREADS) k_multi_axpy(const cplx<TV> *__restrict__ V, int64_t vstride,
                                                            const double2 *__restrict__ coef, const double *vscale,
                                                            double sgn, cplx<TW> *__restrict__ w, int64_t len,
                                                            double2 *__restrict__ partial) {
  HMG_PDL_PROLOGUE();
  __shared__ double2 sc[NV];
  if (threadIdx.x < NV) {
    const double f = sgn * (vscale ? vscale[threadIdx.x] : 1.0);
    sc[threadIdx.x] = make_double2(f * coef[threadIdx.x].x, f * coef[threadIdx.x].y);
  }
  __syncthreads();
  double nrm = 0.0;
  constexpr int U = NV <= 2 ? 4 : NV <= 5 ? 2 : 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < len; e0 += stride * U) {
    cplx<TV> v[U][NV];
    cplx<TW> wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      if (e < len) {
#pragma unroll
        for (int i = 0; i < NV; ++i) v[u][i] = V[(int64_t)i * vstride + e];
        wv[u] = w[e];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      if (e >= len) continue;
      double x = wv[u].x, y = wv[u].y;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const double2 c = sc[i];
        x = fma(c.x, (double)v[u][i].x, fma(-c.y, (double)v[u][i].y, x));
        y = fma(c.x, (double)v[u][i].y, fma(c.y, (double)v[u][i].x, y));
      }
      const cplx<TW> o = mkc<TW>((TW)x, (TW)y);
      w[e] = o;
      if (NORM) nrm = fma((double)o.x, (double)o.x, fma((double)o.y, (double)o.y, nrm));
    }
  }
  if (NORM) {
    __shared__ double sn[KRY_THREADS / 32];
    nrm = warp_sum(nrm);
    if ((threadIdx.x & 31) == 0) sn[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0;
#pragma unroll
      for (int k = 0; k < KRY_THREADS / 32; ++k) a += sn[k];
      partial[blockIdx.x] = make_double2(a, 0.0);
    }
  }
}

// v <- s * w   (s real; optional precision conversion)
template <typename TI, typename TO = TI>
__global__ void __launch_bounds__(KRY_THREADS) k_scale(const cplx<TI> *__restrict__ w, cplx<TO> *__restrict__ v,
                                                       double s, int64_t len) {
  HMG_PDL_PROLOGUE();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += stride) {
    const cplx<TI> a = w[e];
    v[e] = mkc<TO>((TO)(s * (double)a.x), (TO)(s * (double)a.y));
  }
}

// c64 variants: two complex values per 16-byte load (float4).  Slab offsets,
// lengths and the vector stride are multiples of 8 elements (row pitch
// rounded to 8), so every pair is 16-byte aligned.  len2 = len / 2 pairs.
template <int NV, bool SELF, int U = 1>
__global__ void __launch_bounds__(KRY_THREADS) k_multidot_f4(const float4 *__restrict__ V, int64_t vstride2,
                                                             const float4 *__restrict__ w, int64_t len2,
                                                             double2 *__restrict__ partial) {
  HMG_PDL_PROLOGUE();
  constexpr int NA = NV + (SELF ? 1 : 0);
  double ar[NA], ai[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) ar[i] = ai[i] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // U elements per thread and trip (all their loads issued before the arithmetic); each
  // thread still accumulates its elements in increasing order: the same sums for any U
  auto acc = [&](const float4 (&v)[NV], const float4 wv) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      ar[i] = fma((double)v[i].x, (double)wv.x, fma((double)v[i].y, (double)wv.y, ar[i]));
      ai[i] = fma((double)v[i].x, (double)wv.y, fma(-(double)v[i].y, (double)wv.x, ai[i]));
      ar[i] = fma((double)v[i].z, (double)wv.z, fma((double)v[i].w, (double)wv.w, ar[i]));
      ai[i] = fma((double)v[i].z, (double)wv.w, fma(-(double)v[i].w, (double)wv.z, ai[i]));
    }
    if (SELF) {
      ar[NV] = fma((double)wv.x, (double)wv.x, fma((double)wv.y, (double)wv.y, ar[NV]));
      ar[NV] = fma((double)wv.z, (double)wv.z, fma((double)wv.w, (double)wv.w, ar[NV]));
    }
  };
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (U == 2) {
    for (; e + stride < len2; e += 2 * stride) {
      float4 v0[NV], v1[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        v0[i] = V[(int64_t)i * vstride2 + e];
        v1[i] = V[(int64_t)i * vstride2 + e + stride];
      }
      const float4 w0 = w[e], w1 = w[e + stride];
      acc(v0, w0);
      acc(v1, w1);
    }
  }
  for (; e < len2; e += stride) {
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = V[(int64_t)i * vstride2 + e];
    acc(v, w[e]);
  }
  __shared__ double sr[KRY_THREADS / 32][NA], si[KRY_THREADS / 32][NA];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    const double a = warp_sum(ar[i]), b = warp_sum(ai[i]);
    if (lane == 0) { sr[wid][i] = a; si[wid][i] = b; }
  }
  __syncthreads();
  if (threadIdx.x < NA) {
    double a = 0, b = 0;
#pragma unroll
    for (int k = 0; k < KRY_THREADS / 32; ++k) { a += sr[k][threadIdx.x]; b += si[k][threadIdx.x]; }
    partial[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = make_double2(a, b);
  }
}

template <int NV, bool NORM, int U = 1>
__global__ void __launch_bounds__(KRY_THREADS) k_multi_axpy_f4(const float4 *__restrict__ V, int64_t vstride2,
                                                               const double2 *__restrict__ coef, const double *vscale,
                                                               double sgn, float4 *__restrict__ w, int64_t len2,
                                                               double2 *__restrict__ partial) {
  HMG_PDL_PROLOGUE();
  __shared__ double2 sc[NV];
  if (threadIdx.x < NV) {
    const double f = sgn * (vscale ? vscale[threadIdx.x] : 1.0);
    sc[threadIdx.x] = make_double2(f * coef[threadIdx.x].x, f * coef[threadIdx.x].y);
  }
  __syncthreads();
  double nrm = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // U elements per thread and trip, loads first; elements still processed in increasing order
  auto upd = [&](const float4 (&v)[NV], const float4 wv, int64_t e) {
    double x0 = wv.x, y0 = wv.y, x1 = wv.z, y1 = wv.w;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double2 c = sc[i];
      x0 = fma(c.x, (double)v[i].x, fma(-c.y, (double)v[i].y, x0));
      y0 = fma(c.x, (double)v[i].y, fma(c.y, (double)v[i].x, y0));
      x1 = fma(c.x, (double)v[i].z, fma(-c.y, (double)v[i].w, x1));
      y1 = fma(c.x, (double)v[i].w, fma(c.y, (double)v[i].z, y1));
    }
    const float4 o = make_float4((float)x0, (float)y0, (float)x1, (float)y1);
    w[e] = o;
    if (NORM) {
      nrm = fma((double)o.x, (double)o.x, fma((double)o.y, (double)o.y, nrm));
      nrm = fma((double)o.z, (double)o.z, fma((double)o.w, (double)o.w, nrm));
    }
  };
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (U == 2) {
    for (; e + stride < len2; e += 2 * stride) {
      float4 v0[NV], v1[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        v0[i] = V[(int64_t)i * vstride2 + e];
        v1[i] = V[(int64_t)i * vstride2 + e + stride];
      }
      const float4 w0 = w[e], w1 = w[e + stride];
      upd(v0, w0, e);
      upd(v1, w1, e + stride);
    }
  }
  for (; e < len2; e += stride) {
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = V[(int64_t)i * vstride2 + e];
    upd(v, w[e], e);
  }
  if (NORM) {
    __shared__ double sn[KRY_THREADS / 32];
    nrm = warp_sum(nrm);
    if ((threadIdx.x & 31) == 0) sn[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0;
#pragma unroll
      for (int k = 0; k < KRY_THREADS / 32; ++k) a += sn[k];
      partial[blockIdx.x] = make_double2(a, 0.0);
    }
  }
}

#define HMG_NV_CASES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) \
  X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31)

}  // namespace hmg
