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
#include <type_traits>

#include "common.cuh"
#include "k_operator.cuh"
#include "k_uniform.cuh"

namespace hmg {

enum { PK_RB = 0, PK_ELEMENT = 1, PK_JACOBI = 2, PK_PLUS = 3 };

template <int DIM, int KIND> struct Patch {
  static constexpr int K = KIND == PK_JACOBI ? 1 : KIND == PK_ELEMENT ? (1 << DIM) : KIND == PK_PLUS ? 2 * DIM + 1 : 5;
  __host__ __device__ static constexpr void off(int s, int &ox, int &oy, int &oz) {
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

__device__ __forceinline__ double __fmul_rn_t(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float __fmul_rn_t(float a, float b) { return __fmul_rn(a, b); }

// 1 / cnt_j for cnt_j = 1..8 (a table instead of a per-node fp64 division)
__constant__ double kInvCount[9] = {0.0, 1.0, 0.5, 1.0 / 3.0, 0.25, 0.2, 1.0 / 6.0, 1.0 / 7.0, 0.125};

// (1a) the additive Vanka operator ASSEMBLED as a stencil.
//   B = sum_i V_i^T W_i H_i^{-1} V_i   (Eq. 3.8; W_i(j,j) = 1/cnt_j)
// couples node j only to j + d with d = o_q - o_s for two offsets o_s, o_q of the
// patch shape, so B is a short stencil: 13 offsets for RB / Plus 2D, 9 (27) for
// Element 2D (3D), 25 for Plus 3D, 1 for Jacobi -- against K^2 = 25 (64) inverse
// entries a per-node gather over the containing patches reads.  B is assembled
// once at setup in fp64 from the fp64 patch inverses (k_vanka_assemble) and
// stored in the level's coefficient precision; a sweep is then
//   u_out = u + w B r   (r = f - A u, or r = f for a zero initial guess).
// Mathematically the same operator (only the summation order differs).
template <int DIM, int KIND> struct BStencil {
  static constexpr int K = Patch<DIM, KIND>::K;
  struct Tab {
    int n = 0;
    int d[64][3] = {};
  };
  static constexpr Tab make() {
    Tab t;
    const int zr = DIM == 3 ? 2 : 0;
    for (int dz = -zr; dz <= zr; ++dz)
      for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx) {
          bool hit = false;
          for (int a = 0; a < K; ++a)
            for (int b = 0; b < K; ++b) {
              int ax = 0, ay = 0, az = 0, bx = 0, by = 0, bz = 0;
              Patch<DIM, KIND>::off(a, ax, ay, az);
              Patch<DIM, KIND>::off(b, bx, by, bz);
              if (bx - ax == dx && by - ay == dy && bz - az == dz) hit = true;
            }
          if (hit) {
            t.d[t.n][0] = dx;
            t.d[t.n][1] = dy;
            t.d[t.n][2] = dz;
            ++t.n;
          }
        }
    return t;
  }
  static constexpr Tab tab = make();
  static constexpr int NB = tab.n;
  template <int P> static constexpr int dx = tab.d[P][0];
  template <int P> static constexpr int dy = tab.d[P][1];
  template <int P> static constexpr int dz = tab.d[P][2];
};

static_assert(BStencil<2, PK_RB>::NB == 13 && BStencil<2, PK_PLUS>::NB == 13 && BStencil<3, PK_PLUS>::NB == 25,
              "RB / Plus operator offsets");
static_assert(BStencil<2, PK_ELEMENT>::NB == 9 && BStencil<3, PK_ELEMENT>::NB == 27 && BStencil<2, PK_JACOBI>::NB == 1,
              "Element / Jacobi operator offsets");

template <int I, int N, typename F>
__device__ __forceinline__ void static_for(F &&f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

// u_out_j = u_j + w sum_p B[p][j] r[j + d_p]   (u unused when zero; in place is safe:
// every node reads and writes only its own u).  B vanishes at non-anchor /
// out-of-domain positions and r is zero (ghosts) or exchanged (halo) there.
template <typename T, typename TK, int DIM, int KIND, int NR = 1>
__global__ void __launch_bounds__(256) k_vanka_stencil(Geo g, const cplx<TK> *__restrict__ B,
                                                       const cplx<T> *__restrict__ r, const cplx<T> *u,
                                                       cplx<T> *u_out, T w, int zero, int64_t bs, UBox ub,
                                                       UCoef<BStencil<DIM, KIND>::NB, T> uc,
                                                       const unsigned short *__restrict__ cls,
                                                       const cplx<TK> *__restrict__ tab) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(g, ix, iy, iz);
  using S = BStencil<DIM, KIND>;
  const int64_t j = g.idx(ix, iy, iz);
  bool uni = ub.in(ix, iy, iz);   // B from the uniform-box copy (k_uniform.cuh)
  // a warp with lanes on both sides of the box (an x-normal sponge face) would run BOTH copies of
  // the unrolled loop; with a dictionary every lane can take its class's entry instead -- inside
  // the box that is the box's own class, bitwise the uniform copy -- so such a warp runs one
  if (cls && !__all_sync(__activemask(), uni)) uni = false;
  cplx<T> acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = mkc<T>(0, 0);
  // uniform box: B from the parameter copy (in T); a separate loop copy behind one branch
  auto run = [&](auto bcoef) {
    static_for<0, S::NB>([&](auto P) {
      constexpr int p = decltype(P)::value;
      const cplx<T> b = bcoef(p);
      const int64_t o = j + g.delta(S::template dx<p>, S::template dy<p>, S::template dz<p>);
#pragma unroll
      for (int q = 0; q < NR; ++q) acc[q] = cfma<T>(acc[q], b, r[q * bs + o]);
    });
  };
  if (uni) {
    run([&](int p) { return uc.c[p]; });
  } else if (cls) {   // coefficient dictionary (k_dict.cuh): tab[class][p]
    const cplx<TK> *cb = tab + (int64_t)cls[j] * S::NB;
    run([&](int p) { return ccast<T, TK>(cb[p]); });
  } else {
    run([&](int p) { return ccast<T, TK>(B[(int64_t)p * g.total + j]); });
  }
  // explicit fma / mul: the same rounding in every batch-width instantiation
  // (left to the compiler, u + w acc is contracted in some and not in others)
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    cplx<T> o;
    if (zero) {
      o = mkc<T>(__fmul_rn_t(acc[q].x, w), __fmul_rn_t(acc[q].y, w));
    } else {
      const cplx<T> uq = u[q * bs + j];
      o = mkc<T>(fma(acc[q].x, w, uq.x), fma(acc[q].y, w, uq.y));
    }
    u_out[q * bs + j] = o;
  }
}

// Register-blocked k_vanka_stencil (one right-hand side): each thread owns BZ consecutive
// nodes along the slowest axis (y in 2D, z in 3D) so every r value is loaded once for all
// the outputs it reaches; input rows / planes are visited in increasing order and each
// output takes its offsets p in increasing order -- the arithmetic of k_vanka_stencil.
template <typename T, typename TK, int DIM, int KIND, int BZ>
__global__ void __launch_bounds__(256) k_vanka_stencil_blk(Geo g, const cplx<TK> *__restrict__ B,
                                                           const cplx<T> *__restrict__ r, const cplx<T> *u,
                                                           cplx<T> *u_out, T w, int zero, UBox ub,
                                                           UCoef<BStencil<DIM, KIND>::NB, T> uc,
                                                           const unsigned short *__restrict__ cls,
                                                           const cplx<TK> *__restrict__ tab) {
  HMG_PDL_PROLOGUE();
  using S = BStencil<DIM, KIND>;
  // 3D, launched with a one-dimensional block: FLAT (x, y) indexing -- consecutive threads run
  // across the row ends, so rows of 2^k + 1 nodes leave no idle lanes (257 nodes: 9 warps of 32
  // with the last one holding a single node; 129 nodes: 5 warps for 4.03 warps of work)
  int ix = blockIdx.x * blockDim.x + threadIdx.x;
  int iyt = blockIdx.y * blockDim.y + threadIdx.y;
  if (DIM == 3 && blockDim.y == 1) {
    iyt = ix / g.n[0];
    ix -= iyt * g.n[0];
  }
  const int iy = DIM == 3 ? iyt : iyt * BZ;
  const int iz = DIM == 3 ? blockIdx.z * BZ : 0;
  if (ix >= g.n[0] || iy >= g.n[1] || iz >= g.n[2]) return;
  const int64_t j0 = g.idx(ix, iy, iz);
  const int64_t ps = DIM == 3 ? g.pxy : g.px;
  const int slow0 = DIM == 3 ? iz : iy, nslow = DIM == 3 ? g.n[2] : g.n[1];
  const int olast = min(slow0 + BZ, nslow) - 1 - slow0;
  bool uni = DIM == 3 ? ub.in(ix, iy, iz) && ub.in(ix, iy, iz + olast)
                      : ub.in(ix, iy, 0) && ub.in(ix, iy + olast, 0);
  // a warp with lanes on both sides of the box (an x-normal sponge face) would run BOTH copies of
  // the unrolled loop; with a dictionary every lane can take its class's entry instead -- inside
  // the box that is the box's own class, bitwise the uniform copy -- so such a warp runs one
  if (cls && !__all_sync(__activemask(), uni)) uni = false;
  constexpr int SR = 2;   // |slow offset| <= 2 for every patch kind
  cplx<T> acc[BZ];
#pragma unroll
  for (int o = 0; o < BZ; ++o) acc[o] = mkc<T>(0, 0);
  auto run = [&](auto bcoef) {
#pragma unroll
    for (int sl = -SR; sl < BZ + SR; ++sl) {
      if (sl > olast + SR) break;
#pragma unroll
      for (int o = 0; o < BZ; ++o) {
        static_for<0, S::NB>([&](auto P) {
          constexpr int p = decltype(P)::value;
          constexpr int sp = DIM == 3 ? S::template dz<p> : S::template dy<p>;
          if (sp != sl - o) return;
          const int64_t a = j0 + (int64_t)sl * ps + (DIM == 3 ? (int64_t)S::template dy<p> * g.px : 0) +
                            S::template dx<p>;
          acc[o] = cfma<T>(acc[o], bcoef(p, o), r[a]);
        });
      }
    }
  };
  if (uni) {
    run([&](int p, int) { return uc.c[p]; });
  } else if (cls) {   // coefficient dictionary (k_dict.cuh): tab[class][p]
    const cplx<TK> *cb[BZ];
#pragma unroll
    for (int o = 0; o < BZ; ++o) cb[o] = tab + (int64_t)cls[j0 + (int64_t)min(o, olast) * ps] * S::NB;
    run([&](int p, int o) { return ccast<T, TK>(cb[o][p]); });
  } else {
    run([&](int p, int o) { return ccast<T, TK>(B[(int64_t)p * g.total + j0 + (int64_t)o * ps]); });
  }
#pragma unroll
  for (int o = 0; o < BZ; ++o) {
    if (o > olast) break;
    const int64_t j = j0 + (int64_t)o * ps;
    cplx<T> v;
    if (zero) {
      v = mkc<T>(__fmul_rn_t(acc[o].x, w), __fmul_rn_t(acc[o].y, w));
    } else {
      const cplx<T> uq = u[j];
      v = mkc<T>(fma(acc[o].x, w, uq.x), fma(acc[o].y, w, uq.y));
    }
    u_out[j] = v;
  }
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
  HMG_PDL_PROLOGUE();
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
          int MINB = 2, int PD = 1>
__global__ void __launch_bounds__(256, MINB) k_rb2d_march(Geo g, const cplx<TS> *__restrict__ sig,
                                                    const cplx<TS> *__restrict__ ia_, const cplx<TS> *__restrict__ id_,
                                                    double alpha_d, double ih2_d, const cplx<TS> *__restrict__ f,
                                                    const cplx<TS> *__restrict__ u, cplx<TS> *__restrict__ u_out,
                                                    double w_d, UBox ub, cplx<TS> usg, cplx<TS> uia, cplx<TS> uid) {
  HMG_PDL_PROLOGUE();
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
  // rows are also clamped to y1 + 2, the last row the outputs need (u at yo + 3 for
  // output yo <= y1 - 1): rows past it may lie beyond this rank's ghosted box
  const int ylo = -g.o[1], yhi = min(g.N[1] - g.o[1], y1 + 3), ydom = g.N[1] - g.o[1];
  auto in = [&](int y) { return xin && y >= ylo && y < yhi; };
  // uniform box (k_uniform.cuh): sigma, ia, id of row y come from the box's copies
  const bool xuni = x >= ub.lo[0] && x < ub.hi[0];
  auto urow = [&](int y) { return xuni && y >= ub.lo[1] && y < ub.hi[1]; };
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
  // Row streaming through a per-warp shared-memory ring filled by cp.async (zero
  // fill for rows outside the domain), PD rows ahead.  Each lane copies and reads
  // only its own column, so no barrier is needed.  (Register prefetch measured
  // slower: the compiler moves each just-issued load into the loop-carried
  // register at the back edge, and that move waits for the load.)
  constexpr int NA = ZERO ? 3 : 5;   // f, ia, id (+ u, sigma)
  constexpr int NST = PD + 2;
  extern __shared__ __align__(16) unsigned char rb_smem[];
  CS *ring = reinterpret_cast<CS *>(rb_smem) + (size_t)(threadIdx.x >> 5) * (NST * NA * 32);
  const int64_t ob0 = ob;
  auto cp = [&](const CS *a, int y, int64_t o, int slot, int k) {
    const bool ok = in(y);
    const CS *gp = ok ? a + o : a;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(ring + (slot * NA + k) * 32 + lane);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(sa), "l"(gp), "n"((int)sizeof(CS)),
                 "r"(ok ? (int)sizeof(CS) : 0)
                 : "memory");
  };
  auto issue = [&](int it_) {   // the rows step it_ consumes
    const int b_ = y0 - 2 + it_, slot = it_ % NST;
    const int64_t o = ob0 + (int64_t)it_ * px;
    cp(f, b_, o, slot, 0);
    if (!urow(b_)) cp(ia_, b_, o, slot, 1);
    if (!urow(b_ - 1)) cp(id_, b_ - 1, o - px, slot, 2);
    if (!ZERO) {
      cp(u, b_ + 1, o + px, slot, 3);
      if (!urow(b_)) cp(sig, b_, o, slot, 4);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int k = 0; k < PD; ++k) issue(k);
  // fixed trip count SEG + 4 (rows past y1 load zeros and store nothing); unrolling
  // (UNR 2-6, renaming the rolling windows) measured no faster than UNR = 1
  static_assert((SEG + 4) % UNR == 0, "unroll must divide the trip count");
#pragma unroll UNR
  for (int it = 0; it < SEG + 4; ++it, ob += px) {
    const int b = y0 - 2 + it;
    issue(it + PD);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(PD) : "memory");
    const CS *sl = ring + (it % NST) * NA * 32 + lane;
    if (!ZERO) {
      ub1 = um1;
      um1 = u0; u0 = up1; up1 = sl[3 * 32];
    }
    const bool ub_ = urow(b);
    const CS pf_cur = sl[0], ps_cur = ZERO ? zs : (ub_ ? usg : sl[4 * 32]);
    const CD fb = ccast<D, TS>(pf_cur), idb = ccast<D, TS>(urow(b - 1) ? uid : sl[2 * 32]);
    const CS ab = ub_ ? uia : sl[32];
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
        const bool ym = yo - 1 >= ylo, yp = yo + 1 < ydom;
        const int k = (int)(xm && ym) + (int)(xp && ym) + (int)(xm && yp) + (int)(xp && yp);
        const D kd = (D)kRbCount[k];
        const CD lv = cmul<D>(mkc<D>(kd * r2.x - e * syl.x, kd * r2.y - e * syl.y), ccast<D, TS>(a2));
        const CD upd = cscale<D>(cadd<D>(c2, lv), w * (D)kRbInvCnt[k]);
        u_out[ob - 2 * px] = ccast<TS, D>(ZERO ? upd : cadd<D>(ccast<D, TS>(ub1), upd));
      }
    }
  }
}

// (1b'') the same sweep with TWO columns per lane (c64): a warp owns a strip of 64
// columns (56 outputs, 4 halo columns per side, x0 even so pairs load as 16 bytes).
// Per node the arithmetic is exactly that of k_rb2d_march; the per-lane work that
// does not depend on the node count (shuffles of a row, addresses, ring traffic,
// loop and predicate logic) is shared by the two nodes.
constexpr int RB2_STRIP = 56;

// MODE 0: every warp, generic.  MODE 1: only the warps whose whole footprint (columns of the
// strip, rows y0-4 .. y0+SEG+4) lies inside the uniform box and one node inside the domain,
// with sigma, ia, id, the patch count (4) and the masks as constants -- the same operations on
// the same values as the generic code, so bit-identical.  MODE 2: the remaining warps, generic.
template <int KIND, bool ZERO, int SEG, typename TR, int MINB, int PD, int UNR = 1, int MODE = 0>
__global__ void __launch_bounds__(128, MINB) k_rb2d_march2(Geo g, const float2 *__restrict__ sig,
                                                           const float2 *__restrict__ ia_,
                                                           const float2 *__restrict__ id_, double alpha_d,
                                                           double ih2_d, const float2 *__restrict__ f,
                                                           const float2 *__restrict__ u, float2 *__restrict__ u_out,
                                                           double w_d, UBox ub, float2 usg, float2 uia, float2 uid) {
  HMG_PDL_PROLOGUE();
  using W = FineW<2, KIND>;
  using D = double;
  using CD = double2;
  using CS = float2;
  const D ih2 = ih2_d, w = w_d;
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nstrips = (g.n[0] + RB2_STRIP - 1) / RB2_STRIP;
  const int strip = wid % nstrips, seg = wid / nstrips;
  const int y0 = seg * SEG;
  if (y0 >= g.n[1]) return;
  const int y1 = min(g.n[1], y0 + SEG);
  const int x0 = strip * RB2_STRIP - 4 + 2 * lane;   // this lane's columns x0 (node 0) and x0 + 1 (node 1)
  if (MODE != 0) {
    const int xa = strip * RB2_STRIP - 4, xb = strip * RB2_STRIP + 60, ya = y0 - 4, yb = y0 + SEG + 4;
    const bool inner = xa >= ub.lo[0] && xb <= ub.hi[0] && ya >= ub.lo[1] && yb <= ub.hi[1] &&
                       xa + g.o[0] >= 1 && xb + g.o[0] <= g.N[0] - 1 && ya + g.o[1] >= 1 && yb + g.o[1] <= g.N[1] - 1;
    if (inner != (MODE == 1)) return;
  }
  constexpr bool FAST = MODE == 1;
  const bool out_lane = lane >= 2 && lane < 30;
  bool outn[2], xin[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    outn[q] = out_lane && x0 + q < g.n[0];
    xin[q] = FAST || (x0 + q + g.o[0] >= 0 && x0 + q + g.o[0] < g.N[0]);
  }
  const D e = W::Le * ih2;
  const CD z = mkc<D>(0, 0);
  const CS zs = mkc<float>(0, 0);
  // rows clamped to y1 + 2 as in k_rb2d_march (beyond it: possibly past this rank's box)
  const int ylo = -g.o[1], yhi = min(g.N[1] - g.o[1], y1 + 3), ydom = g.N[1] - g.o[1];
  auto yok = [&](int y) { return FAST || (y >= ylo && y < yhi); };
  // uniform box (k_uniform.cuh): both columns inside -> sigma, ia, id of row y from the box's copies
  const bool xuni = x0 >= ub.lo[0] && x0 + 1 < ub.hi[0];
  auto urow = [&](int y) { return FAST || (xuni && y >= ub.lo[1] && y < ub.hi[1]); };
  const CD uia_d = ccast<D, float>(uia), uid_d = ccast<D, float>(uid);   // (FAST: the constants in fp64)
  const D wcnt4 = w * (D)kRbInvCnt[4];
  CS um1[2] = {zs, zs}, u0[2] = {zs, zs}, up1[2] = {zs, zs}, ub1[2] = {zs, zs};
  CD r2[2] = {z, z}, r1[2] = {z, z}, r0[2] = {z, z};
  CD h2[2] = {z, z}, h1[2] = {z, z}, h0[2] = {z, z};
  CS a2[2] = {zs, zs}, a1[2] = {zs, zs}, a0[2] = {zs, zs};
  CD c2[2] = {z, z}, c1[2] = {z, z};
  CD g3[2] = {z, z}, g2[2] = {z, z}, g1[2] = {z, z};
  const int64_t px = g.px;
  int64_t ob = g.base + x0 + (int64_t)(y0 - 2) * px;
  // valid bytes of this lane's pair in row y (the left domain edge is at an even x)
  auto nbytes = [&](int y) { return yok(y) ? (xin[1] ? 16 : (xin[0] ? 8 : 0)) : 0; };
  auto ld2 = [&](const CS *a, int y, int64_t o, CS &v0, CS &v1) {
    const int nb = nbytes(y);
    v0 = nb >= 8 ? a[o] : zs;
    v1 = nb >= 16 ? a[o + 1] : zs;
  };
  if (!ZERO) {
    ld2(u, y0 - 3, ob - px, u0[0], u0[1]);
    ld2(u, y0 - 2, ob, up1[0], up1[1]);
  }
  constexpr int NA = ZERO ? 3 : 5;   // f, ia, id (+ u, sigma)
  constexpr int NST = PD + 2;
  extern __shared__ __align__(16) unsigned char rb_smem[];
  float4 *ring = reinterpret_cast<float4 *>(rb_smem) + (size_t)(threadIdx.x >> 5) * (NST * NA * 32);
  const int64_t ob0 = ob;
  auto cp = [&](const CS *a, int y, int64_t o, int slot, int k) {
    const int nb = nbytes(y);
    const CS *gp = nb ? a + o : a;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(ring + (slot * NA + k) * 32 + lane);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gp), "r"(nb) : "memory");
  };
  auto issue = [&](int it_) {
    const int b_ = y0 - 2 + it_, slot = it_ % NST;
    const int64_t o = ob0 + (int64_t)it_ * px;
    cp(f, b_, o, slot, 0);
    if (!urow(b_)) cp(ia_, b_, o, slot, 1);
    if (!urow(b_ - 1)) cp(id_, b_ - 1, o - px, slot, 2);
    if (!ZERO) {
      cp(u, b_ + 1, o + px, slot, 3);
      if (!urow(b_)) cp(sig, b_, o, slot, 4);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto shup = [](CS v) { return mkc<float>(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1)); };
  auto shdn = [](CS v) {
    return mkc<float>(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
  };
#pragma unroll
  for (int k = 0; k < PD; ++k) issue(k);
  static_assert((SEG + 4) % UNR == 0, "unroll must divide the trip count");
#pragma unroll UNR
  for (int it = 0; it < SEG + 4; ++it, ob += px) {
    const int b = y0 - 2 + it;
    issue(it + PD);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(PD) : "memory");
    const float4 *sl = ring + (it % NST) * NA * 32 + lane;
    auto split = [](float4 v, CS &p0, CS &p1) { p0 = mkc<float>(v.x, v.y); p1 = mkc<float>(v.z, v.w); };
    CS fv[2], av[2], dv[2], sv[2] = {zs, zs};
    const bool ub_ = urow(b), ubm = urow(b - 1);
    split(sl[0], fv[0], fv[1]);
    split(ub_ ? make_float4(uia.x, uia.y, uia.x, uia.y) : sl[32], av[0], av[1]);
    split(ubm ? make_float4(uid.x, uid.y, uid.x, uid.y) : sl[64], dv[0], dv[1]);
    if (!ZERO) {
#pragma unroll
      for (int q = 0; q < 2; ++q) { ub1[q] = um1[q]; um1[q] = u0[q]; u0[q] = up1[q]; }
      split(sl[96], up1[0], up1[1]);
      split(ub_ ? make_float4(usg.x, usg.y, usg.x, usg.y) : sl[128], sv[0], sv[1]);
    }
    CD rb[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) rb[q] = ccast<D, float>(fv[q]);
    if (!ZERO) {
      using Q = TR;
      using CQ = cplx<Q>;
      // west / east neighbours of both nodes in rows b-1, b, b+1 (one shuffle pair per row)
      CS wm[2], em[2], w0[2], e0[2], wp[2], ep[2];
      wm[0] = shup(um1[1]); em[0] = um1[1]; wm[1] = um1[0]; em[1] = shdn(um1[0]);
      w0[0] = shup(u0[1]);  e0[0] = u0[1];  w0[1] = u0[0];  e0[1] = shdn(u0[0]);
      wp[0] = shup(up1[1]); ep[0] = up1[1]; wp[1] = up1[0]; ep[1] = shdn(up1[0]);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const CQ uc = ccast<Q, float>(u0[q]);
        const CQ un = ccast<Q, float>(um1[q]), us = ccast<Q, float>(up1[q]);
        const CQ uw = ccast<Q, float>(w0[q]), ue = ccast<Q, float>(e0[q]);
        const CQ sf = cadd<Q>(cadd<Q>(uw, ue), cadd<Q>(un, us));
        CQ dlt = cadd<Q>(cadd<Q>(csub<Q>(uw, uc), csub<Q>(ue, uc)), cadd<Q>(csub<Q>(un, uc), csub<Q>(us, uc)));
        CQ Lx = cscale<Q>(dlt, (Q)W::Lf);
        if (W::Le != 0.0) {
          const CQ d2 = cadd<Q>(cadd<Q>(csub<Q>(ccast<Q, float>(wm[q]), uc), csub<Q>(ccast<Q, float>(em[q]), uc)),
                                cadd<Q>(csub<Q>(ccast<Q, float>(wp[q]), uc), csub<Q>(ccast<Q, float>(ep[q]), uc)));
          Lx = cfmar<Q>(Lx, (Q)W::Le, d2);
        }
        Lx = cscale<Q>(Lx, (Q)ih2_d);
        CQ Mx = cscale<Q>(uc, (Q)W::Mc);
        if (W::Mf != 0.0) Mx = cfmar<Q>(Mx, (Q)W::Mf, sf);
        CQ sq = ccast<Q, float>(sv[q]);
        sq.y = fma(-(Q)alpha_d, sq.x, sq.y);
        rb[q] = (xin[q] && yok(b)) ? ccast<D, Q>(csub<Q>(ccast<Q, float>(fv[q]), csub<Q>(Lx, cmul<Q>(sq, Mx)))) : z;
      }
    }
    CD t0[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      r2[q] = r1[q]; r1[q] = r0[q]; r0[q] = rb[q];
      a2[q] = a1[q]; a1[q] = a0[q]; a0[q] = av[q];
      t0[q] = cmul<D>(rb[q], FAST ? uia_d : ccast<D, float>(av[q]));
      h2[q] = h1[q]; h1[q] = h0[q];
    }
    h0[0] = cadd<D>(shfl_up1(t0[1]), t0[1]);
    h0[1] = cadd<D>(t0[0], shfl_dn1(t0[0]));
    CD yc[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const CD sdiag = cadd<D>(h2[q], h0[q]);
      const CD num = mkc<D>(r1[q].x - e * sdiag.x, r1[q].y - e * sdiag.y);
      yc[q] = (xin[q] && yok(b - 1)) ? cmul<D>(num, FAST ? uid_d : ccast<D, float>(dv[q])) : z;
      c2[q] = c1[q]; c1[q] = yc[q];
      g3[q] = g2[q]; g2[q] = g1[q];
    }
    g1[0] = cadd<D>(shfl_up1(yc[1]), yc[1]);
    g1[1] = cadd<D>(yc[0], shfl_dn1(yc[0]));
    const int yo = b - 2;
    if (yo >= y0 && yo < y1 && out_lane && yok(yo)) {
      CS o[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const CD syl = cadd<D>(g3[q], g1[q]);
        D kd, wc;
        if (FAST) {   // interior: all four diagonal anchors present
          kd = 4.0;
          wc = wcnt4;
        } else {
          const int xq = x0 + q + g.o[0];
          const bool xm = xq - 1 >= 0, xp = xq + 1 < g.N[0];
          const bool ym = yo - 1 >= ylo, yp = yo + 1 < ydom;
          const int k = (int)(xm && ym) + (int)(xp && ym) + (int)(xm && yp) + (int)(xp && yp);
          kd = (D)kRbCount[k];
          wc = w * (D)kRbInvCnt[k];
        }
        const CD lv = cmul<D>(mkc<D>(kd * r2[q].x - e * syl.x, kd * r2[q].y - e * syl.y),
                              FAST ? uia_d : ccast<D, float>(a2[q]));
        const CD upd = cscale<D>(cadd<D>(c2[q], lv), wc);
        o[q] = ccast<float, D>(ZERO ? upd : cadd<D>(ccast<D, float>(ub1[q]), upd));
      }
      float2 *dst = u_out + (ob - 2 * px);
      if (outn[0] && outn[1]) *reinterpret_cast<float4 *>(dst) = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
      else if (outn[0]) dst[0] = o[0];
    }
  }
}

}  // namespace hmg
