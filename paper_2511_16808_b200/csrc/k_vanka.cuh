// k_vanka.cuh -- additive Vanka smoother (§3.2-3.3).
//
//   u <- u + w sum_i V_i^T W_i H_i^{-1} V_i (f - A u),  H_i = V_i A V_i^T   (Eq. 3.8)
//
// Patches: RB 2D = centre + (+-1,+-1); Element = the 2^d vertices
// of one cell (anchor = the cell's lowest corner); Plus = centre + axis
// neighbours; Jacobi = 1 node.  Non-element patches exist for every
// node and are clipped to the domain; W_i(j,j) = 1/cnt_j with cnt_j
// = number of patches containing j (reading A7 for Element).
//
// B200 design: the scatter of Eq. 3.8 is done as a conflict-free GATHER in two
// node-parallel passes: (1) every anchor c solves its patch system y_c =
// H_c^{-1} r[X_c] and stores the |X_c| local values in slot-major planes
// y[s][c]; (2) every node j sums y[s][j - o_s] over the anchors whose patch
// contains it and applies w/cnt_j (the weight depends on j only, so it factors
// out of the gather).  No atomics, deterministic order.
#pragma once
#include "common.cuh"
#include "k_operator.cuh"

namespace hmg {

enum { PK_RB = 0, PK_ELEMENT = 1, PK_JACOBI = 2, PK_PLUS = 3 };

template <int DIM, int KIND> struct Patch {
  static constexpr int K = KIND == PK_JACOBI ? 1 : KIND == PK_ELEMENT ? (1 << DIM) : KIND == PK_PLUS ? 2 * DIM + 1 : 5;
  __host__ __device__ static __forceinline__ void off(int s, int &ox, int &oy, int &oz) {
    ox = oy = oz = 0;
    if (KIND == PK_JACOBI) return;
    if (KIND == PK_ELEMENT) { ox = s & 1; oy = (s >> 1) & 1; oz = (s >> 2) & 1; return; }
    if (KIND == PK_PLUS) {
      if (s == 0) return;
      const int a = (s - 1) >> 1, sg = ((s - 1) & 1) ? 1 : -1;
      if (a == 0) ox = sg; else if (a == 1) oy = sg; else oz = sg;
      return;
    }
    // RB (2D only)
    if (s == 0) return;
    ox = ((s - 1) & 1) ? 1 : -1;
    oy = ((s - 1) & 2) ? 1 : -1;
  }
  // is c a patch anchor?
  __host__ __device__ static __forceinline__ bool anchor(const Geo &g, int x, int y, int z) {
    if (KIND == PK_ELEMENT) {
      bool ok = x >= 0 && x < g.n[0] - 1 && y >= 0 && y < g.n[1] - 1;
      if (DIM == 3) ok = ok && z >= 0 && z < g.n[2] - 1;
      return ok;
    }
    return g.inside(x, y, z);
  }
  // cnt_j = number of patches containing node j
  __host__ __device__ static __forceinline__ int count(const Geo &g, int x, int y, int z) {
    if (KIND == PK_ELEMENT) {
      int c = ((x >= 1) + (x <= g.n[0] - 2)) * ((y >= 1) + (y <= g.n[1] - 2));
      if (DIM == 3) c *= (z >= 1) + (z <= g.n[2] - 2);
      return c;
    }
    int c = 0;
    for (int s = 0; s < K; ++s) {
      int ox, oy, oz;
      off(s, ox, oy, oz);
      c += g.inside(x - ox, y - oy, z - oz);
    }
    return c;
  }
};

// (1a) generic patch solve with stored inverses: y[a][c] = sum_b Hinv[a*K+b][c] r[c + o_b]
template <typename T, int DIM, int KIND>
__global__ void __launch_bounds__(256) k_patch_apply(Geo g, const cplx<T> *__restrict__ hinv,
                                                     const cplx<T> *__restrict__ r, cplx<T> *__restrict__ y) {
  HMG_NODE_IDX(g, ix, iy, iz);
  using P = Patch<DIM, KIND>;
  if (!P::anchor(g, ix, iy, iz)) return;
  const int64_t c = g.idx(ix, iy, iz);
  cplx<T> rv[P::K];
#pragma unroll
  for (int b = 0; b < P::K; ++b) {
    int ox, oy, oz;
    P::off(b, ox, oy, oz);
    rv[b] = r[c + g.delta(ox, oy, oz)];
  }
#pragma unroll
  for (int a = 0; a < P::K; ++a) {
    cplx<T> acc = mkc<T>(0, 0);
#pragma unroll
    for (int b = 0; b < P::K; ++b) acc = cfma<T>(acc, hinv[(int64_t)(a * P::K + b) * g.total + c], rv[b]);
    y[(int64_t)a * g.total + c] = acc;
  }
}

// (1b) fine-level RB patch in closed form (2D).  With the compact stencil the
// patch matrix is an arrow: leaf-leaf entries vanish (offsets (2,0),(2,2) lie
// outside the 9-point support), centre-leaf = L's corner weight -1/(6h^2) (M
// has no corner), diagonal a_j = Lc/h^2 - Mc sigma_s,j.  Hence
//   y_c = (r_c - e sum_l r_l/a_l) / (a_c - e^2 sum_l 1/a_l),  y_l = (r_l - e y_c)/a_l.
template <typename T, int KIND>
__global__ void __launch_bounds__(256) k_patch_rb2d_fine(Geo g, const cplx<T> *__restrict__ sig, T alpha, T ih2,
                                                         const cplx<T> *__restrict__ r, cplx<T> *__restrict__ y) {
  HMG_NODE_IDX(g, ix, iy, iz);
  using W = FineW<2, KIND>;
  const int64_t c = g.idx(ix, iy, iz);
  const T e = (T)W::Le * ih2;
  auto diag = [&](int64_t j) {
    cplx<T> s = sig[j];
    s.y = fma(-alpha, s.x, s.y);
    return mkc<T>((T)W::Lc * ih2 - (T)W::Mc * s.x, -(T)W::Mc * s.y);
  };
  const cplx<T> rc = r[c];
  const cplx<T> ac = diag(c);
  cplx<T> inva[4], rl[4];
  bool present[4];
  cplx<T> sr = mkc<T>(0, 0), si = mkc<T>(0, 0);
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int ox = (s & 1) ? 1 : -1, oy = (s & 2) ? 1 : -1;
    present[s] = g.inside(ix + ox, iy + oy, 0);
    inva[s] = mkc<T>(0, 0);
    rl[s] = mkc<T>(0, 0);
    if (present[s]) {
      const int64_t j = c + g.delta(ox, oy, 0);
      inva[s] = crecip<T>(diag(j));
      rl[s] = r[j];
      sr = cadd<T>(sr, cmul<T>(rl[s], inva[s]));
      si = cadd<T>(si, inva[s]);
    }
  }
  const cplx<T> num = mkc<T>(rc.x - e * sr.x, rc.y - e * sr.y);
  const cplx<T> den = mkc<T>(ac.x - e * e * si.x, ac.y - e * e * si.y);
  const cplx<T> yc = cdiv<T>(num, den);
  y[c] = yc;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    cplx<T> v = mkc<T>(0, 0);
    if (present[s]) v = cmul<T>(mkc<T>(rl[s].x - e * yc.x, rl[s].y - e * yc.y), inva[s]);
    y[(int64_t)(s + 1) * g.total + c] = v;
  }
}

// (2) gather: u_j (+)= (w/cnt_j) sum_s y[s][j - o_s] over anchors containing j
template <typename T, int DIM, int KIND>
__global__ void __launch_bounds__(256) k_vanka_gather(Geo g, const cplx<T> *__restrict__ y, T w,
                                                      cplx<T> *__restrict__ u, int zero_init) {
  HMG_NODE_IDX(g, ix, iy, iz);
  using P = Patch<DIM, KIND>;
  const int64_t j = g.idx(ix, iy, iz);
  cplx<T> acc = mkc<T>(0, 0);
#pragma unroll
  for (int s = 0; s < P::K; ++s) {
    int ox, oy, oz;
    P::off(s, ox, oy, oz);
    if (P::anchor(g, ix - ox, iy - oy, iz - oz)) acc = cadd<T>(acc, y[(int64_t)s * g.total + j - g.delta(ox, oy, oz)]);
  }
  const T wc = w / (T)P::count(g, ix, iy, iz);
  const cplx<T> upd = cscale<T>(acc, wc);
  u[j] = zero_init ? upd : cadd<T>(u[j], upd);
}

}  // namespace hmg
