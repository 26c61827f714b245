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
// B200 design: the scatter of Eq. 3.8 is done as a conflict-free GATHER:
// every node j sums, over the anchors c whose patch contains it, the entry of
// y_c = H_c^{-1} r[X_c] that belongs to j, and applies w/cnt_j (the weight
// depends on j only, so it factors out).  No atomics, deterministic order.
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
      x += g.o[0]; y += g.o[1]; z += g.o[2];
      bool ok = x >= 0 && x < g.N[0] - 1 && y >= 0 && y < g.N[1] - 1;
      if (DIM == 3) ok = ok && z >= 0 && z < g.N[2] - 1;
      return ok;
    }
    return g.inside(x, y, z);
  }
  // cnt_j = number of patches containing node j
  __host__ __device__ static __forceinline__ int count(const Geo &g, int x, int y, int z) {
    if (KIND == PK_ELEMENT) {
      x += g.o[0]; y += g.o[1]; z += g.o[2];
      int c = ((x >= 1) + (x <= g.N[0] - 2)) * ((y >= 1) + (y <= g.N[1] - 2));
      if (DIM == 3) c *= (z >= 1) + (z <= g.N[2] - 2);
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

// 1 / cnt_j for cnt_j = 1..8 (a table instead of a per-node fp64 division)
__constant__ double kInvCount[9] = {0.0, 1.0, 0.5, 1.0 / 3.0, 0.25, 0.2, 1.0 / 6.0, 1.0 / 7.0, 0.125};

// (1a) generic sweep with stored inverses, as a direct gather (any dim/kind):
//   u_out_j = u_j + (w/cnt_j) sum_{s: anchor c = j - o_s} sum_q Hinv_c[s][q] r[c + o_q]
// (r = f - A u precomputed; r = f for a zero initial guess).  Only row s of
// each containing anchor's inverse is read, so every stored entry is read once
// per sweep and no patch solution is staged.  Each node reads/writes only its
// own u: in place is safe.  Branch-free: a position c = j - o_s that is not an
// anchor (outside the domain, or an Element corner on the far faces) holds an
// all-zero inverse (buffers are zeroed at allocation, k_patch_inverse writes
// anchors only; slab ghost rows hold the neighbour's anchors), and r is finite
// there (zero ghosts / exchanged halo), so its terms vanish exactly and every
// load of the node can be in flight at once.
template <typename T, typename TK, int DIM, int KIND>
__global__ void __launch_bounds__(256) k_vanka_direct(Geo g, const cplx<TK> *__restrict__ hinv,
                                                      const cplx<T> *__restrict__ r, const cplx<T> *u,
                                                      cplx<T> *u_out, T w, int zero) {
  HMG_NODE_IDX(g, ix, iy, iz);
  using P = Patch<DIM, KIND>;
  constexpr int K = P::K;
  cplx<T> acc = mkc<T>(0, 0);
#pragma unroll
  for (int sI = 0; sI < K; ++sI) {
    int dx, dy, dz;
    P::off(sI, dx, dy, dz);
    const int64_t c = g.idx(ix - dx, iy - dy, iz - dz);
    cplx<TK> hw[K];
#pragma unroll
    for (int q = 0; q < K; ++q) hw[q] = hinv[(int64_t)(sI * K + q) * g.total + c];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      int bx, by, bz;
      P::off(q, bx, by, bz);
      acc = cfma<T>(acc, ccast<T, TK>(hw[q]), r[c + g.delta(bx, by, bz)]);
    }
  }
  const int64_t j = g.idx(ix, iy, iz);
  const cplx<T> upd = cscale<T>(acc, w * (T)kInvCount[P::count(g, ix, iy, iz)]);
  u_out[j] = zero ? upd : cadd<T>(u[j], upd);
}

// (1b) fine-level RB smoothing sweep in ONE kernel (2D, matrix-free).
// With the compact stencil the RB patch matrix is an arrow: leaf-leaf entries
// vanish (offsets (2,0), (2,2) lie outside the 9-point support), centre-leaf =
// L's corner weight e = -1/(6h^2) (M has no corner), diagonal a_j = Lc/h^2 -
// Mc sigma_s,j.  Hence the patch solve of anchor c is
//   y_c = (r_c - e sum_l r_l/a_l) / (a_c - e^2 sum_l 1/a_l),  y_l = (r_l - e y_c)/a_l,
// and node j gathers  y_j + sum_{present diagonal anchors c} (r_j - e y_c)/a_j,
// so only the CENTRE solutions need staging.  The two sigma-only factors
// ia_j = 1/a_j and id_c = 1/(a_c - e^2 sum_l ia_l) are precomputed at setup
// (k_rb_factors, stored in TS like every other coefficient): the sweep has no
// division and all its arithmetic is fp64.  Per block: u on the tile + 3,
// r / ia on the tile + 2, y_c on the tile + 1, all in shared memory; HBM sees
// u, f, sigma, ia, id read once and u written once (6 TS per node; 4 with
// ZERO = zero initial guess, where r = f and sigma is not needed).
template <typename TS>
__global__ void k_rb_factors(Geo g, const double2 *__restrict__ sigd, double alpha, double ih2, double Lc, double Mc,
                             double e, cplx<TS> *__restrict__ ia, cplx<TS> *__restrict__ id) {
  HMG_NODE_IDX(g, ix, iy, iz);
  auto diag = [&](int x, int y) {
    double2 s = sigd[g.idx(x, y, 0)];
    s.y = fma(-alpha, s.x, s.y);
    return make_double2(Lc * ih2 - Mc * s.x, -Mc * s.y);
  };
  const double2 ac = diag(ix, iy);
  double2 si = make_double2(0, 0);
  for (int s = 0; s < 4; ++s) {
    const int dx = (s & 1) ? 1 : -1, dy = (s & 2) ? 1 : -1;
    if (g.inside(ix + dx, iy + dy, 0)) si = cadd<double>(si, crecip<double>(diag(ix + dx, iy + dy)));
  }
  const int64_t j = g.idx(ix, iy, 0);
  ia[j] = ccast<TS, double>(crecip<double>(ac));
  id[j] = ccast<TS, double>(crecip<double>(make_double2(ac.x - e * e * si.x, ac.y - e * e * si.y)));
}

// (1b') the same RB sweep as a WARP-MARCHING stencil: each warp owns a strip
// of 32 columns (26 outputs: 3 halo lanes per side, the reach of u -> r ->
// y_c -> u) and marches along y through a segment of SEG output rows, holding
// a rolling window of rows in registers; x-neighbours come from warp shuffles.
// No shared memory, no barriers; every array is streamed once per row (x 32/26).
// Pipeline at step b (row b of r):  load u(b+1), f(b), sigma(b), ia(b), id(b-1);
//   r(b) = f - H_s u (fp64) and t(b) = r ia;  y_c(b-1) = (r - e sum_diag t) id;
//   output row b-2 = u + w/cnt (y_c + (k r - e sum_diag y_c) ia).
__device__ __forceinline__ double2 shfl_up1(double2 v) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ double2 shfl_dn1(double2 v) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ float2 shfl_up1(float2 v) {
  return make_float2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ float2 shfl_dn1(float2 v) {
  return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}

constexpr int RB_STRIP = 26;
// count-dependent factors of the RB gather: k (number of present diagonal
// anchors) as a double and 1 / (1 + k)  (a table instead of I2F + a division)
__constant__ double kRbCount[5] = {0.0, 1.0, 2.0, 3.0, 4.0};
__constant__ double kRbInvCnt[5] = {1.0, 0.5, 1.0 / 3.0, 0.25, 0.2};

// Out of place: u_out = u_in + w B (f - H_s u_in) (u_in unused with ZERO).  In
// place would race: other warps still read old u in their halo rows/columns.
// TC = arithmetic precision of the patch algebra (fp64, or the storage
// precision), TR = precision of the residual f - H_s u
template <typename TS, int KIND, bool ZERO, int SEG, typename TC = double, typename TR = double, int UNR = 1,
          int MINB = 2>
__global__ void __launch_bounds__(256, MINB) k_rb2d_march(Geo g, const cplx<TS> *__restrict__ sig,
                                                    const cplx<TS> *__restrict__ ia_, const cplx<TS> *__restrict__ id_,
                                                    double alpha_d, double ih2_d, const cplx<TS> *__restrict__ f,
                                                    const cplx<TS> *__restrict__ u, cplx<TS> *__restrict__ u_out,
                                                    double w_d) {
  using W = FineW<2, KIND>;
  using D = TC;
  const D alpha = (D)alpha_d, ih2 = (D)ih2_d, w = (D)w_d;
  using CD = cplx<D>;
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nstrips = (g.n[0] + RB_STRIP - 1) / RB_STRIP;
  const int strip = wid % nstrips, seg = wid / nstrips;
  const int y0 = seg * SEG;
  if (y0 >= g.n[1]) return;
  const int y1 = min(g.n[1], y0 + SEG);
  const int x = strip * RB_STRIP - 3 + lane;
  const bool out_lane = lane >= 3 && lane < 3 + RB_STRIP && x < g.n[0];
  const D e = W::Le * ih2;
  const CD z = mkc<D>(0, 0);
  // x validity is fixed per lane; rows are checked against the global slab range
  const bool xin = x + g.o[0] >= 0 && x + g.o[0] < g.N[0];
  const int ylo = -g.o[1], yhi = g.N[1] - g.o[1];
  auto in = [&](int y) { return xin && y >= ylo && y < yhi; };
  // rolling window (u and ia stay in their storage type: converting on use is
  // exact and keeps the register count down)
  using CS = cplx<TS>;
  const CS zs = mkc<TS>(0, 0);
  CS um1 = zs, u0 = zs, up1 = zs;       // u at rows b-1, b, b+1
  CS ub1 = zs;                          // u at row b-2 (the output row)
  CD r2 = z, r1 = z, r0 = z;            // r at rows b-2, b-1, b
  CD h2 = z, h1 = z, h0 = z;            // horizontal sums t(x-1) + t(x+1) of t = r ia, rows b-2, b-1, b
  CS a2 = zs, a1 = zs, a0 = zs;         // ia at rows b-2, b-1, b
  CD c2 = z, c1 = z;                    // y_c at rows b-2, b-1
  CD g3 = z, g2 = z, g1 = z;            // horizontal sums y_c(x-1) + y_c(x+1), rows b-3, b-2, b-1
  // one-step-ahead prefetch registers, kept in the storage type so that the
  // loads of step b+1 stay in flight during step b
  // per-lane column offset; row y of array a sits at a + col + y * px
  const int64_t px = g.px;
  // running element offset of row b in this lane's column (one 64-bit add per row)
  int64_t ob = g.base + x + (int64_t)(y0 - 2) * px;
  auto lr = [&](const CS *a, int y, int64_t o) { return in(y) ? a[o] : zs; };
  if (!ZERO) {
    u0 = lr(u, y0 - 3, ob - px);
    up1 = lr(u, y0 - 2, ob);
  }
  CS pu = ZERO ? zs : lr(u, y0 - 1, ob + px), pf = lr(f, y0 - 2, ob), pa = lr(ia_, y0 - 2, ob),
     pid = lr(id_, y0 - 3, ob - px);
  CS ps = ZERO ? zs : lr(sig, y0 - 2, ob);
  // fixed trip count SEG + 4 (rows past y1 load zeros and store nothing); unrolling
  // (UNR 2-6, renaming the rolling windows) measured no faster than UNR = 1
  static_assert((SEG + 4) % UNR == 0, "unroll must divide the trip count");
#pragma unroll UNR
  for (int it = 0; it < SEG + 4; ++it, ob += px) {
    const int b = y0 - 2 + it;
    if (!ZERO) {
      ub1 = um1;
      um1 = u0; u0 = up1; up1 = pu;
      pu = lr(u, b + 2, ob + 2 * px);
    }
    const CS pf_cur = pf, ps_cur = ps;
    const CD fb = ccast<D, TS>(pf), idb = ccast<D, TS>(pid);
    const CS ab = pa;
    pf = lr(f, b + 1, ob + px);
    pa = lr(ia_, b + 1, ob + px);
    pid = lr(id_, b, ob);
    if (!ZERO) ps = lr(sig, b + 1, ob + px);
    // ---- r(b) in TR, t(b).  L u in difference form, sum w (u_nb - u_c): exact
    // algebra because Lc + 4 Lf + 4 Le = 0 (zero ghosts included), and it keeps
    // the cancellation of the compact stencil out of a low-precision sum.
    CD rb = fb;
    if (!ZERO) {
      using Q = TR;
      using CQ = cplx<Q>;
      auto sh = [](CS v, bool up) {
        return ccast<Q, TS>(up ? mkc<TS>(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1))
                               : mkc<TS>(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1)));
      };
      const CQ uc = ccast<Q, TS>(u0);
      const CQ un = ccast<Q, TS>(um1), us = ccast<Q, TS>(up1), uw = sh(u0, true), ue = sh(u0, false);
      const CQ sf = cadd<Q>(cadd<Q>(uw, ue), cadd<Q>(un, us));
      CQ dlt = cadd<Q>(cadd<Q>(csub<Q>(uw, uc), csub<Q>(ue, uc)), cadd<Q>(csub<Q>(un, uc), csub<Q>(us, uc)));
      CQ Lx = cscale<Q>(dlt, (Q)W::Lf);
      if (W::Le != 0.0) {
        const CQ d2 = cadd<Q>(cadd<Q>(csub<Q>(sh(um1, true), uc), csub<Q>(sh(um1, false), uc)),
                              cadd<Q>(csub<Q>(sh(up1, true), uc), csub<Q>(sh(up1, false), uc)));
        Lx = cfmar<Q>(Lx, (Q)W::Le, d2);
      }
      Lx = cscale<Q>(Lx, (Q)ih2_d);
      CQ Mx = cscale<Q>(uc, (Q)W::Mc);
      if (W::Mf != 0.0) Mx = cfmar<Q>(Mx, (Q)W::Mf, sf);
      CQ sq = ccast<Q, TS>(ps_cur);
      sq.y = fma(-(Q)alpha_d, sq.x, sq.y);
      rb = in(b) ? ccast<D, Q>(csub<Q>(ccast<Q, TS>(pf_cur), csub<Q>(Lx, cmul<Q>(sq, Mx)))) : z;
    }
    r2 = r1; r1 = r0; r0 = rb;
    a2 = a1; a1 = a0; a0 = ab;
    {
      // each row of t and y_c is shuffled once; its left + right sum rolls with the window
      const CD t0 = cmul<D>(rb, ccast<D, TS>(ab));
      h2 = h1; h1 = h0; h0 = cadd<D>(shfl_up1(t0), shfl_dn1(t0));
    }
    // ---- y_c(b-1): diagonal leaves at rows b-2 and b, columns x +- 1
    {
      const CD sdiag = cadd<D>(h2, h0);
      const CD num = mkc<D>(r1.x - e * sdiag.x, r1.y - e * sdiag.y);
      const CD yc = in(b - 1) ? cmul<D>(num, idb) : z;
      c2 = c1; c1 = yc;
      g3 = g2; g2 = g1; g1 = cadd<D>(shfl_up1(yc), shfl_dn1(yc));
    }
    // ---- output row b-2
    const int yo = b - 2;
    if (yo >= y0 && yo < y1) {
      if (out_lane && in(yo)) {
        // anchors j - (dx, dy) for the 4 diagonal offsets: rows yo -+ 1, columns x -+ 1;
        // y_c vanishes outside the domain, so the sums need no masking, only the count
        const CD syl = cadd<D>(g3, g1);
        const bool xm = x - 1 + g.o[0] >= 0, xp = x + 1 + g.o[0] < g.N[0];
        const bool ym = yo - 1 >= ylo, yp = yo + 1 < yhi;
        const int k = (int)(xm && ym) + (int)(xp && ym) + (int)(xm && yp) + (int)(xp && yp);
        const D kd = (D)kRbCount[k];
        const CD lv = cmul<D>(mkc<D>(kd * r2.x - e * syl.x, kd * r2.y - e * syl.y), ccast<D, TS>(a2));
        const CD upd = cscale<D>(cadd<D>(c2, lv), w * (D)kRbInvCnt[k]);
        u_out[ob - 2 * px] = ccast<TS, D>(ZERO ? upd : cadd<D>(ccast<D, TS>(ub1), upd));
      }
    }
  }
}

// Dense K x K complex solve A y = b in registers, Gaussian elimination with
// partial pivoting (row swaps by static-index selects, so A stays in
// registers); same pivoting rule as LAPACK getrf.  b is overwritten by y.
template <typename T, int K>
__device__ __forceinline__ void small_solve(cplx<T> (&A)[K][K], cplx<T> (&b)[K]) {
  cplx<T> ipiv[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    T best = cabs2<T>(A[k][k]);
    int p = k;
#pragma unroll
    for (int i = k + 1; i < K; ++i) {
      const T v = cabs2<T>(A[i][k]);
      if (v > best) { best = v; p = i; }
    }
#pragma unroll
    for (int i = k + 1; i < K; ++i) {
      const bool sw = i == p;   // branch-free select keeps A in registers
#pragma unroll
      for (int c = k; c < K; ++c) {
        const cplx<T> t = A[k][c];
        A[k][c] = cselp<T>(sw, A[i][c], t);
        A[i][c] = cselp<T>(sw, t, A[i][c]);
      }
      const cplx<T> t = b[k];
      b[k] = cselp<T>(sw, b[i], t);
      b[i] = cselp<T>(sw, t, b[i]);
    }
    ipiv[k] = crecip_fast<T>(A[k][k]);
#pragma unroll
    for (int i = k + 1; i < K; ++i) {
      const cplx<T> f = cmul<T>(A[i][k], ipiv[k]);
#pragma unroll
      for (int c = k + 1; c < K; ++c) A[i][c] = csub<T>(A[i][c], cmul<T>(f, A[k][c]));
      b[i] = csub<T>(b[i], cmul<T>(f, b[k]));
    }
  }
#pragma unroll
  for (int k = K - 1; k >= 0; --k) {
    cplx<T> acc = b[k];
#pragma unroll
    for (int c = k + 1; c < K; ++c) acc = csub<T>(acc, cmul<T>(A[k][c], b[c]));
    b[k] = cmul<T>(acc, ipiv[k]);
  }
}

// (1c) one additive-Vanka sweep on a Galerkin level in ONE kernel (2D,
// stored stencil of radius R): residual on the tile + 2 into shared memory,
// then every output node j gathers its patch values DIRECTLY,
//     u_j += w/cnt_j sum_{s: anchor c = j - o_s} sum_b Hinv_c[s][b] r[c + o_b],
// i.e. only row s of each containing anchor's inverse is needed; every
// stored inverse entry is still read exactly once per sweep and no patch
// solution is staged (reading A8: H_i = A_l[X_i, X_i], inverses formed at
// setup in fp64 by k_patch_inverse).  HBM: stencil planes (residual), inverse
// planes, u, f read once, u' written once (ZERO: inverse planes and f only).
// Out of place (u_out != u): other blocks still read old u in their halos.
// Without stored inverses (hinv == nullptr) each anchor's patch matrix is
// assembled from the stencil and solved in registers (k_smooth_stored2d_lu).
template <typename T, typename TK, int R, int KIND, int TX, int TY, bool ZERO>
__global__ void __launch_bounds__(256) k_smooth_stored2d(Geo g, const cplx<TK> *__restrict__ coef,
                                                         const cplx<TK> *__restrict__ hinv,
                                                         const cplx<T> *__restrict__ f, const cplx<T> *__restrict__ u,
                                                         cplx<T> *__restrict__ u_out, T w) {
  using P = Patch<2, KIND>;
  constexpr int K = P::K;
  constexpr int NT = 256;
  constexpr int WS = 2 * R + 1;
  constexpr int HU = 2 + R;
  constexpr int UX = TX + 2 * HU, UY = TY + 2 * HU, RX = TX + 4, RY = TY + 4;
  constexpr int NU = (UX * UY + NT - 1) / NT, NR = (RX * RY + NT - 1) / NT;
  __shared__ cplx<T> su[ZERO ? 1 : UY * UX];
  __shared__ cplx<T> sr[RY * RX];
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const cplx<T> zero = mkc<T>(0, 0);
  if (!ZERO) {
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      const int i = tid + k * NT;
      if (i < UY * UX) {
        const int gx = x0 - HU + i % UX, gy = y0 - HU + i / UX;
        su[i] = g.inside(gx, gy, 0) ? u[g.idx(gx, gy, 0)] : zero;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const int i = tid + k * NT;
    if (i < RY * RX) {
      const int gx = x0 - 2 + i % RX, gy = y0 - 2 + i / RX;
      sr[i] = g.inside(gx, gy, 0) ? f[g.idx(gx, gy, 0)] : zero;
    }
  }
  __syncthreads();
  if (!ZERO) {
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const int i = tid + k * NT;
      if (i >= RY * RX) continue;
      const int lx = i % RX, ly = i / RX;
      const int gx = x0 - 2 + lx, gy = y0 - 2 + ly;
      if (!g.inside(gx, gy, 0)) continue;
      const int64_t j = g.idx(gx, gy, 0);
      const cplx<T> *uc = su + (ly + R) * UX + (lx + R);
      cplx<T> acc = zero;
#pragma unroll
      for (int oy = -R; oy <= R; ++oy) {
        cplx<TK> cw[WS];
#pragma unroll
        for (int ox = -R; ox <= R; ++ox) cw[ox + R] = coef[(int64_t)((ox + R) + WS * (oy + R)) * g.total + j];
#pragma unroll
        for (int ox = -R; ox <= R; ++ox) acc = cfma<T>(acc, ccast<T, TK>(cw[ox + R]), uc[oy * UX + ox]);
      }
      sr[i] = csub<T>(sr[i], acc);
    }
    __syncthreads();
  }
  for (int oy = threadIdx.y; oy < TY; oy += blockDim.y) {
    for (int ox = threadIdx.x; ox < TX; ox += blockDim.x) {
      const int gx = x0 + ox, gy = y0 + oy;
      if (!g.inside(gx, gy, 0)) continue;
      cplx<T> acc = zero;
#pragma unroll
      for (int sI = 0; sI < K; ++sI) {
        int dx, dy, dz;
        P::off(sI, dx, dy, dz);
        const int cx = gx - dx, cy = gy - dy;   // anchor whose patch holds j in slot sI
        if (!P::anchor(g, cx, cy, 0)) continue;
        const int64_t c = g.idx(cx, cy, 0);
        cplx<TK> hw[K];
#pragma unroll
        for (int q = 0; q < K; ++q) hw[q] = hinv[(int64_t)(sI * K + q) * g.total + c];
#pragma unroll
        for (int q = 0; q < K; ++q) {
          int bx, by, bz;
          P::off(q, bx, by, bz);
          // members outside the domain have zero inverse columns and r = 0 there
          acc = cfma<T>(acc, ccast<T, TK>(hw[q]), sr[(oy + 2 - dy + by) * RX + (ox + 2 - dx + bx)]);
        }
      }
      const cplx<T> upd = cscale<T>(acc, w / (T)P::count(g, gx, gy, 0));
      const int64_t j = g.idx(gx, gy, 0);
      u_out[j] = ZERO ? upd : cadd<T>(su[(oy + HU) * UX + (ox + HU)], upd);
    }
  }
}

}  // namespace hmg
