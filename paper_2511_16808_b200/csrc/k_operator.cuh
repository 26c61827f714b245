// k_operator.cuh -- fine-level matrix-free Helmholtz stencil (SURVEY §8(a) a2,
// a11) and stored-coefficient stencil of the Galerkin levels (a6).
//
//   H = L - diag(sigma) M   (Eq. 2.2; Eq. 2.3)
//   2D COMPACT4: L = (1/h^2)[-1/6 -2/3 -1/6; -2/3 10/3 -2/3; -1/6 -2/3 -1/6],
//                M = [0 1/12 0; 1/12 2/3 1/12; 0 1/12 0]
//   3D COMPACT4: L = -1/(6h^2){[0 1 0;1 2 1;0 1 0], [1 2 1;2 -24 2;1 2 1], [0 1 0;1 2 1;0 1 0]}
//                i.e. centre 4/h^2, 6 faces -1/(3h^2), 12 edges -1/(6h^2), corners 0;
//                M = centre 1/2, faces 1/12.
//   FD2: L = (1/h^2)(2d centre, -1 on the 2d faces), M = I.
// sigma multiplies row j (the row's centre node); the shifted operator uses
// sigma_s = sigma - i alpha Re(sigma)  (= w^2k^2 (1 - i(g/w + alpha)),
// readings A1/A2 of P:247-253).  Out-of-domain neighbours are the zero ghost
// layer of the padded box (truncation = homogeneous Dirichlet).
#pragma once
#include "common.cuh"
#include "k_uniform.cuh"

namespace hmg {

enum { ST_COMPACT4 = 0, ST_FD2 = 1 };

// Stencil weights of L (without 1/h^2) and M by neighbour class.
template <int DIM, int KIND> struct FineW;
template <> struct FineW<2, ST_COMPACT4> {
  static constexpr double Lc = 10.0 / 3.0, Lf = -2.0 / 3.0, Le = -1.0 / 6.0;
  static constexpr double Mc = 2.0 / 3.0, Mf = 1.0 / 12.0;
};
template <> struct FineW<3, ST_COMPACT4> {
  static constexpr double Lc = 4.0, Lf = -1.0 / 3.0, Le = -1.0 / 6.0;
  static constexpr double Mc = 0.5, Mf = 1.0 / 12.0;
};
template <> struct FineW<2, ST_FD2> {
  static constexpr double Lc = 4.0, Lf = -1.0, Le = 0.0;
  static constexpr double Mc = 1.0, Mf = 0.0;
};
template <> struct FineW<3, ST_FD2> {
  static constexpr double Lc = 6.0, Lf = -1.0, Le = 0.0;
  static constexpr double Mc = 1.0, Mf = 0.0;
};

// y = A x   (f == nullptr)   or   y = f - A x   (residual), fine level.
// sig[j] = sigma_j = (w^2k^2, -w^2k^2 g/w); alpha = shift (0 for H).
// TC = arithmetic precision (T or double); storage of x, f, y stays T;
// TS = storage precision of sigma.
// (A x)_i or (f - A x)_i at padded index i, rounded to T (shared by every kernel
// that forms the fine operator, so their results agree bit for bit)
// uni: the node lies in the level's uniform box, sigma = us (k_uniform.cuh)
template <typename T, int DIM, int KIND, typename TC, typename TS>
__device__ __forceinline__ cplx<T> fine_op_node(const Geo &g, const cplx<TS> *__restrict__ sig, TC alpha, TC ih2,
                                                const cplx<T> *__restrict__ x, const cplx<T> *__restrict__ f,
                                                int64_t i, bool uni = false, cplx<TC> us = cplx<TC>{}) {
  using W = FineW<DIM, KIND>;
  using CC = cplx<TC>;
  const int64_t px = g.px;
  auto X = [&](int64_t k) { return ccast<TC, T>(x[k]); };
  const CC xc = X(i);
  CC sf = cadd<TC>(cadd<TC>(X(i - 1), X(i + 1)), cadd<TC>(X(i - px), X(i + px)));
  CC se = mkc<TC>(0, 0);
  if (DIM == 2) {
    if (W::Le != 0.0) se = cadd<TC>(cadd<TC>(X(i - px - 1), X(i - px + 1)), cadd<TC>(X(i + px - 1), X(i + px + 1)));
  } else {
    const int64_t pz = g.pxy;
    sf = cadd<TC>(sf, cadd<TC>(X(i - pz), X(i + pz)));
    if (W::Le != 0.0) {
      se = cadd<TC>(cadd<TC>(X(i - px - 1), X(i - px + 1)), cadd<TC>(X(i + px - 1), X(i + px + 1)));
      se = cadd<TC>(se, cadd<TC>(cadd<TC>(X(i - pz - 1), X(i - pz + 1)), cadd<TC>(X(i + pz - 1), X(i + pz + 1))));
      se = cadd<TC>(se, cadd<TC>(cadd<TC>(X(i - pz - px), X(i - pz + px)), cadd<TC>(X(i + pz - px), X(i + pz + px))));
    }
  }
  // L x
  CC Lx = cscale<TC>(xc, (TC)W::Lc);
  Lx = cfmar<TC>(Lx, (TC)W::Lf, sf);
  if (W::Le != 0.0) Lx = cfmar<TC>(Lx, (TC)W::Le, se);
  Lx = cscale<TC>(Lx, ih2);
  // M x
  CC Mx = cscale<TC>(xc, (TC)W::Mc);
  if (W::Mf != 0.0) Mx = cfmar<TC>(Mx, (TC)W::Mf, sf);
  CC s = uni ? us : ccast<TC, TS>(sig[i]);   // (uniform value kept in TC: no conversion)
  s.y = fma(-alpha, s.x, s.y);
  const CC Ax = csub<TC>(Lx, cmul<TC>(s, Mx));
  return ccast<T, TC>(f ? csub<TC>(ccast<TC, T>(f[i]), Ax) : Ax);
}

template <typename T, int DIM, int KIND, typename TC = T, typename TS = T>
__global__ void __launch_bounds__(256) k_fine_op(Geo g, const cplx<TS> *__restrict__ sig, TC alpha, TC ih2,
                                                 const cplx<T> *__restrict__ x,
                                                 const cplx<T> *__restrict__ f, cplx<T> *__restrict__ y,
                                                 UBox ub, cplx<TC> us) {
  HMG_NODE_IDX(g, ix, iy, iz);
  const int64_t i = g.idx(ix, iy, iz);
  y[i] = fine_op_node<T, DIM, KIND, TC, TS>(g, sig, alpha, ih2, x, f, i, ub.in(ix, iy, iz), us);
}

// 2D c64 variant of k_fine_op: one thread per PAIR of x-adjacent nodes
// (x0 = 2p, x0 + 1), 16-byte loads of the pairs (interior x offset G and row
// pitch are even, so pairs are aligned).  Same arithmetic per node as
// k_fine_op; the second node of the last pair of an odd row is a ghost and is
// not written.  TSG = storage of sigma (float2 or double2).
template <int KIND, typename TC, typename TSG>
__global__ void __launch_bounds__(256) k_fine_op2d_pair(Geo g, const cplx<TSG> *__restrict__ sig, TC alpha, TC ih2,
                                                        const float2 *__restrict__ x, const float2 *__restrict__ f,
                                                        float2 *__restrict__ y, UBox ub, cplx<TC> us) {
  using W = FineW<2, KIND>;
  using CC = cplx<TC>;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int iy = blockIdx.y * blockDim.y + threadIdx.y;
  const int x0 = 2 * p;
  if (x0 >= g.n[0] || iy >= g.n[1]) return;
  const int64_t i = g.idx(x0, iy, 0);
  const int64_t px = g.px;
  auto row = [&](int64_t c, CC &l, CC &a, CC &b, CC &r) {   // x[c-1], x[c], x[c+1], x[c+2]
    const float4 ab = *reinterpret_cast<const float4 *>(x + c);
    const float2 lv = x[c - 1], rv = x[c + 2];
    l = mkc<TC>(lv.x, lv.y);
    a = mkc<TC>(ab.x, ab.y);
    b = mkc<TC>(ab.z, ab.w);
    r = mkc<TC>(rv.x, rv.y);
  };
  CC nl, na, nb, nr, cl, ca, cb, cr, sl, sa, sb, sr;
  row(i - px, nl, na, nb, nr);
  row(i, cl, ca, cb, cr);
  row(i + px, sl, sa, sb, sr);
  // node x0 (a) and node x0 + 1 (b)
  const CC sfa = cadd<TC>(cadd<TC>(cl, cb), cadd<TC>(na, sa));
  const CC sfb = cadd<TC>(cadd<TC>(ca, cr), cadd<TC>(nb, sb));
  CC La = cscale<TC>(ca, (TC)W::Lc), Lb = cscale<TC>(cb, (TC)W::Lc);
  La = cfmar<TC>(La, (TC)W::Lf, sfa);
  Lb = cfmar<TC>(Lb, (TC)W::Lf, sfb);
  if (W::Le != 0.0) {
    La = cfmar<TC>(La, (TC)W::Le, cadd<TC>(cadd<TC>(nl, nb), cadd<TC>(sl, sb)));
    Lb = cfmar<TC>(Lb, (TC)W::Le, cadd<TC>(cadd<TC>(na, nr), cadd<TC>(sa, sr)));
  }
  La = cscale<TC>(La, ih2);
  Lb = cscale<TC>(Lb, ih2);
  CC Ma = cscale<TC>(ca, (TC)W::Mc), Mb = cscale<TC>(cb, (TC)W::Mc);
  if (W::Mf != 0.0) {
    Ma = cfmar<TC>(Ma, (TC)W::Mf, sfa);
    Mb = cfmar<TC>(Mb, (TC)W::Mf, sfb);
  }
  const bool ua = ub.in(x0, iy, 0), ubb = ub.in(x0 + 1, iy, 0);
  CC sga = ua ? us : ccast<TC, TSG>(sig[i]), sgb = ubb ? us : ccast<TC, TSG>(sig[i + 1]);
  sga.y = fma(-alpha, sga.x, sga.y);
  sgb.y = fma(-alpha, sgb.x, sgb.y);
  CC oa = csub<TC>(La, cmul<TC>(sga, Ma)), ob = csub<TC>(Lb, cmul<TC>(sgb, Mb));
  if (f) {
    const float4 fv = *reinterpret_cast<const float4 *>(f + i);
    oa = csub<TC>(mkc<TC>(fv.x, fv.y), oa);
    ob = csub<TC>(mkc<TC>(fv.z, fv.w), ob);
  }
  if (x0 + 1 < g.n[0])
    *reinterpret_cast<float4 *>(y + i) = make_float4((float)oa.x, (float)oa.y, (float)ob.x, (float)ob.y);
  else
    y[i] = make_float2((float)oa.x, (float)oa.y);
}

// Stored stencil of radius R: coef[k][j], k = (ox+R) + (2R+1)((oy+R) + (2R+1)(oz+R)),
// multiplies x[j + o].  Coefficients towards out-of-domain nodes are zero.
// TV = vector storage/arithmetic (fp64 on Galerkin levels), TK = coefficient storage.
template <int DIM, int R> constexpr int kplanes() { return DIM == 3 ? (2 * R + 1) * (2 * R + 1) * (2 * R + 1) : (2 * R + 1) * (2 * R + 1); }

template <typename TV, typename TK, int DIM, int R, int NR = 1>
__global__ void __launch_bounds__(256) k_stored_op(Geo g, const cplx<TK> *__restrict__ coef,
                                                   const cplx<TV> *__restrict__ x,
                                                   const cplx<TV> *__restrict__ f, cplx<TV> *__restrict__ y,
                                                   int64_t bs, UBox ub, UCoef<kplanes<DIM, R>(), TV> uc) {
  // NR right-hand sides at a stride of bs elements: each coefficient is read once
  // and applied to all of them (multi-RHS batches; same per-RHS arithmetic order)
  using T = TV;
  HMG_NODE_IDX(g, ix, iy, iz);
  const int64_t i = g.idx(ix, iy, iz);
  const bool uni = ub.in(ix, iy, iz);   // coefficients from the uniform-box copy (k_uniform.cuh)
  constexpr int ZR = DIM == 3 ? R : 0;
  cplx<T> acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = mkc<T>(0, 0);
  // two copies of the unrolled loop behind a branch (not a per-coefficient select:
  // predicated-off loads and conversions would still take issue slots)
  auto run = [&](auto coef_k) {
    int k = 0;
#pragma unroll
    for (int oz = -ZR; oz <= ZR; ++oz)
#pragma unroll
      for (int oy = -R; oy <= R; ++oy)
#pragma unroll
        for (int ox = -R; ox <= R; ++ox, ++k) {
          const cplx<T> c = coef_k(k);
          const int64_t j = i + g.delta(ox, oy, oz);
#pragma unroll
          for (int r = 0; r < NR; ++r) acc[r] = cfma<T>(acc[r], c, x[r * bs + j]);
        }
  };
  if (uni) run([&](int k) { return uc.c[k]; });
  else run([&](int k) { return ccast<T, TK>(coef[(int64_t)k * g.total + i]); });
#pragma unroll
  for (int r = 0; r < NR; ++r) y[r * bs + i] = f ? csub<T>(f[r * bs + i], acc[r]) : acc[r];
}

// 2D c64 variant of k_stored_op: one thread per PAIR of x-adjacent nodes (2p,
// 2p+1): the fp32 coefficient planes load as aligned 16-byte pairs and the two
// nodes share their x-window (2R + 2 loads per row instead of 2 (2R + 1)).  Same
// per-node arithmetic and fma order as k_stored_op.
template <int R>
__global__ void __launch_bounds__(256) k_stored_op2d_pair(Geo g, const float2 *__restrict__ coef,
                                                          const double2 *__restrict__ x,
                                                          const double2 *__restrict__ f, double2 *__restrict__ y,
                                                          UBox ub, UCoef<(2 * R + 1) * (2 * R + 1), double> uc) {
  using T = double;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int iy = blockIdx.y * blockDim.y + threadIdx.y;
  const int ix = 2 * p;
  if (ix >= g.n[0] || iy >= g.n[1]) return;
  const int64_t i = g.idx(ix, iy, 0);
  const bool two = ix + 1 < g.n[0];
  const bool uni = ub.in(ix, iy, 0) && (!two || ub.in(ix + 1, iy, 0));   // both nodes in the uniform box
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  // uniform box: fp64 coefficient copies from the parameter bank, no loads, no
  // conversions -- a separate copy of the unrolled loop behind one branch
  auto run = [&](auto coef_k) {
    int k = 0;
#pragma unroll
    for (int oy = -R; oy <= R; ++oy) {
      const double2 *row = x + i + (int64_t)oy * g.px;
      double2 xw[2 * R + 2];
#pragma unroll
      for (int c = 0; c < 2 * R + 2; ++c) xw[c] = row[c - R];
#pragma unroll
      for (int ox = -R; ox <= R; ++ox, ++k) {
        double2 k0, k1;
        coef_k(k, k0, k1);
        a0 = cfma<T>(a0, k0, xw[ox + R]);
        a1 = cfma<T>(a1, k1, xw[ox + R + 1]);
      }
    }
  };
  if (uni) {
    run([&](int k, double2 &k0, double2 &k1) { k0 = k1 = uc.c[k]; });
  } else {
    run([&](int k, double2 &k0, double2 &k1) {
      const float4 c2 = *reinterpret_cast<const float4 *>(coef + (int64_t)k * g.total + i);
      k0 = mkc<T>(c2.x, c2.y);
      k1 = mkc<T>(c2.z, c2.w);
    });
  }
  y[i] = f ? csub<T>(f[i], a0) : a0;
  if (two) y[i + 1] = f ? csub<T>(f[i + 1], a1) : a1;
}

}  // namespace hmg
