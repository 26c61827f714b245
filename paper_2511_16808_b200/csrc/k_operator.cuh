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
  HMG_PDL_PROLOGUE();
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
  HMG_PDL_PROLOGUE();
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

// 2D c64 fine operator as a WARP-MARCHING kernel: lane l holds the column pair
// (x0, x0 + 1), x0 = 60 s - 2 + 2 l, of strip s; lanes 1..30 write (60 outputs per
// strip), lanes 0 and 31 only supply the x-neighbours, which every lane takes from
// its neighbour lanes by shuffles.  The warp marches down a segment of SEG output
// rows holding a rolling window of three rows in fp64 registers, so every input
// element is loaded (16-byte pairs through a per-warp cp.async ring, PD rows ahead)
// and converted ONCE, instead of 12 loads and conversions per node pair in
// k_fine_op2d_pair.  Same per-node grouping of the stencil sums as fine_op_node:
// bit-identical to k_fine_op / k_fine_op2d_pair (tests/test_gpu_march.py).
constexpr int FM_STRIP = 60;
// TC: arithmetic (double: the FGMRES matvec and the fp64 model; float: the fp32 cycle residual
// of DESIGN.md §4.1, fp32 sigma only)
template <int KIND, typename TSG, int SEG, int PD, typename TC = double>
__global__ void __launch_bounds__(128) k_fine_op2d_march(Geo g, const cplx<TSG> *__restrict__ sig, double alpha,
                                                         double ih2, const float2 *__restrict__ x,
                                                         const float2 *__restrict__ f, float2 *__restrict__ y, UBox ub,
                                                         double2 us) {
  HMG_PDL_PROLOGUE();
  using W = FineW<2, KIND>;
  using CC = cplx<TC>;
  static_assert(sizeof(TC) == 8 || sizeof(TSG) == 4, "fp32 arithmetic with fp32 sigma only");
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nstrips = (g.n[0] + FM_STRIP - 1) / FM_STRIP;
  const int strip = wid % nstrips, seg = wid / nstrips;
  const int y0 = seg * SEG;
  if (y0 >= g.n[1]) return;
  const int y1 = min(g.n[1], y0 + SEG);
  const int x0 = strip * FM_STRIP - 2 + 2 * lane;
  const bool out_lane = lane >= 1 && lane <= 30 && x0 < g.n[0];
  const bool two = x0 + 1 < g.n[0];
  const bool xload = x0 < g.n[0] + g.G;   // columns past the ghost layer are never used
  const bool xuni = x0 >= ub.lo[0] && x0 + 1 < ub.hi[0];
  auto urow = [&](int yy) { return xuni && yy >= ub.lo[1] && yy < ub.hi[1]; };
  constexpr int NST = PD + 2;
  constexpr int SW = sizeof(cplx<TSG>) * 2 / 16;   // 16-byte words of a sigma pair (1 or 2)
  constexpr int NW = 2 + SW;                        // x, f, sigma words per lane and row
  extern __shared__ __align__(16) unsigned char fm_smem[];
  float4 *ring = reinterpret_cast<float4 *>(fm_smem) + (size_t)(threadIdx.x >> 5) * (NST * NW * 32);
  const int64_t px = g.px;
  const int64_t ob0 = g.base + x0 + (int64_t)(y0 - 1) * px;   // row y0 - 1, column x0
  auto cp16 = [&](const void *src, int slot, int k, bool ok) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(ring + (slot * NW + k) * 32 + lane);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(ok ? src : (const void *)x),
                 "r"(ok ? 16 : 0)
                 : "memory");
  };
  const int nrows = y1 - y0 + 2;   // input rows y0-1 .. y1
  auto issue = [&](int it) {
    if (it < nrows) {
      const int b = y0 - 1 + it, slot = it % NST;
      const int64_t o = ob0 + (int64_t)it * px;
      cp16(x + o, slot, 0, xload);
      if (f) cp16(f + o, slot, 1, xload && b >= 0 && b < g.n[1]);
      if (!urow(b) && b >= 0 && b < g.n[1]) {
#pragma unroll
        for (int w = 0; w < SW; ++w)
          cp16(reinterpret_cast<const char *>(sig + o) + 16 * w, slot, 2 + w, xload);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int k = 0; k < PD; ++k) issue(k);
  const CC z = mkc<TC>(0, 0);
  const TC alp = (TC)alpha, ih2c = (TC)ih2;
  const CC usc = mkc<TC>((TC)us.x, (TC)us.y);
  // rows b-2 (a) and b-1 (b): this lane's pair and its west / east neighbours (each row is
  // shuffled once, when it arrives, and rolls with the window)
  CC a0 = z, a1 = z, b0 = z, b1 = z, aw = z, ae = z, bw = z, be = z;
  auto shl = [](auto v) { return __shfl_up_sync(0xffffffffu, v, 1); };
  auto shr = [](auto v) { return __shfl_down_sync(0xffffffffu, v, 1); };
  for (int it = 0; it < nrows; ++it) {
    issue(it + PD);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(PD) : "memory");
    const float4 *sl = ring + (it % NST) * NW * 32 + lane;
    const float4 xv = sl[0];
    const CC c0 = mkc<TC>(xv.x, xv.y), c1 = mkc<TC>(xv.z, xv.w);   // row b
    const CC cw = mkc<TC>(shl(c1.x), shl(c1.y)), ce = mkc<TC>(shr(c0.x), shr(c0.y));
    if (it >= 2) {
      // output row yo = b - 1: rows a (yo - 1), b (yo), c (yo + 1); west of node 0 and east
      // of node 1 from the neighbour lanes
      const int yo = y0 - 2 + it;
      if (out_lane) {
        const float4 *sb = ring + ((it - 1) % NST) * NW * 32 + lane;   // row yo's f and sigma
        CC sg0, sg1;
        if (urow(yo)) {
          sg0 = sg1 = usc;
        } else if (SW == 1) {
          const float4 v = sb[2 * 32];
          sg0 = mkc<TC>(v.x, v.y);
          sg1 = mkc<TC>(v.z, v.w);
        } else {
          // the pair's two fp64 sigma values are this lane's words 2 and 3 (32 float4 apart)
          const double2 d0 = *reinterpret_cast<const double2 *>(sb + 2 * 32);
          const double2 d1 = *reinterpret_cast<const double2 *>(sb + 3 * 32);
          sg0 = mkc<TC>((TC)d0.x, (TC)d0.y);
          sg1 = mkc<TC>((TC)d1.x, (TC)d1.y);
        }
        auto node = [&](CC cc, CC w_, CC e_, CC n_, CC s_, CC nw, CC ne, CC sw, CC se_, CC sgm, TC fx, TC fy) {
          const CC sf = cadd<TC>(cadd<TC>(w_, e_), cadd<TC>(n_, s_));
          CC Lx = cscale<TC>(cc, (TC)W::Lc);
          Lx = cfmar<TC>(Lx, (TC)W::Lf, sf);
          if (W::Le != 0.0) Lx = cfmar<TC>(Lx, (TC)W::Le, cadd<TC>(cadd<TC>(nw, ne), cadd<TC>(sw, se_)));
          Lx = cscale<TC>(Lx, ih2c);
          CC Mx = cscale<TC>(cc, (TC)W::Mc);
          if (W::Mf != 0.0) Mx = cfmar<TC>(Mx, (TC)W::Mf, sf);
          sgm.y = fma(-alp, sgm.x, sgm.y);
          const CC Ax = csub<TC>(Lx, cmul<TC>(sgm, Mx));
          return f ? csub<TC>(mkc<TC>(fx, fy), Ax) : Ax;
        };
        float4 fv = make_float4(0, 0, 0, 0);
        if (f) fv = sb[32];
        // node 0 (x0): west = neighbour lane's node 1, east = own node 1
        const CC o0 = node(b0, bw, b1, a0, c0, aw, a1, cw, c1, sg0, fv.x, fv.y);
        // node 1 (x0 + 1): west = own node 0, east = neighbour lane's node 0
        const CC o1 = node(b1, b0, be, a1, c1, a0, ae, c0, ce, sg1, fv.z, fv.w);
        float2 *dst = y + ob0 + (int64_t)(it - 1) * px;
        if (two) *reinterpret_cast<float4 *>(dst) = make_float4((float)o0.x, (float)o0.y, (float)o1.x, (float)o1.y);
        else dst[0] = make_float2((float)o0.x, (float)o0.y);
      }
    }
    a0 = b0; a1 = b1; aw = bw; ae = be;
    b0 = c0; b1 = c1; bw = cw; be = ce;
  }
}

// Fine-level residual AND bicubic restriction in one warp-marching kernel (2D, c64):
//   fc = R_0 (f - H_s u)      (Alg. 2.1 step 2; R = bicubic, Eq. 3.2)
// without writing r.  Strip s: lane l holds the column pair (x0, x0 + 1), x0 = 56 s - 4 + 2 l;
// the residual is formed (k_fine_op2d_march's arithmetic, rounded to fp32 as the stored r
// would be) on lanes 1..30 for rows y0 - 2 .. y1 + 1, and the lane holding 2X (lanes
// 2..29: coarse X in [28 s, 28 s + 28)) restricts it: the x-pass over fine columns 2X-2..2X+2
// (its own pair and the neighbour lanes' by shuffles), then the y-pass over fine rows
// 2I-2..2I+2 in rolling accumulators -- the summation order of k_restrict_pair, so fc is
// bit-identical to the residual kernel followed by k_restrict_pair.  Coarse rows I with
// 2I in [y0, y1) (y0 even) belong to the segment.
constexpr int RR_STRIP = 56;
// TC: arithmetic of the residual (double: k_fine_op2d_march's; float: the fp32 cycle residual of
// DESIGN.md §4.1); the restriction is fp64 either way
template <int KIND, int SEG, int PD, typename TC = double>
__global__ void __launch_bounds__(128) k_fine_resrestrict2d_march(Geo g, Geo gc, const float2 *__restrict__ sig,
                                                                  double alpha, double ih2,
                                                                  const float2 *__restrict__ x,
                                                                  const float2 *__restrict__ f,
                                                                  double2 *__restrict__ fc, UBox ub, double2 us) {
  HMG_PDL_PROLOGUE();
  using W = FineW<2, KIND>;
  using CC = double2;
  using CR = cplx<TC>;
  static_assert(SEG % 2 == 0, "segments start on even rows");
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nstrips = (g.n[0] + RR_STRIP - 1) / RR_STRIP;
  const int strip = wid % nstrips, seg = wid / nstrips;
  const int y0 = seg * SEG;
  if (y0 >= g.n[1]) return;
  const int y1 = min(g.n[1], y0 + SEG);
  const int x0 = strip * RR_STRIP - 4 + 2 * lane;
  const bool xload = x0 >= -g.G && x0 < g.n[0] + g.G;
  const bool rlane = lane >= 1 && lane <= 30;
  // residual columns in the domain (zero outside, as the zero ghost layer of a stored r)
  const bool in0 = x0 >= 0 && x0 < g.n[0], in1 = x0 + 1 >= 0 && x0 + 1 < g.n[0];
  const int X = x0 / 2;   // x0 even (x0 >= -4 -> X >= -2)
  const bool clane = lane >= 2 && lane <= 29 && x0 >= 0 && X < gc.n[0];
  const bool xuni = x0 >= ub.lo[0] && x0 + 1 < ub.hi[0];
  auto urow = [&](int yy) { return xuni && yy >= ub.lo[1] && yy < ub.hi[1]; };
  constexpr int NST = PD + 2, NW = 3;   // x, f, sigma words per lane and row
  extern __shared__ __align__(16) unsigned char rr_smem[];
  float4 *ring = reinterpret_cast<float4 *>(rr_smem) + (size_t)(threadIdx.x >> 5) * (NST * NW * 32);
  const int64_t px = g.px;
  const int ybeg = y0 - 3;                                   // first input row
  const int nrows = (y1 + 3) - ybeg;                         // input rows y0-3 .. y1+2
  const int64_t ob0 = g.base + x0 + (int64_t)ybeg * px;
  auto cp16 = [&](const void *src, int slot, int k, bool ok) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(ring + (slot * NW + k) * 32 + lane);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(ok ? src : (const void *)x),
                 "r"(ok ? 16 : 0)
                 : "memory");
  };
  // rows the outputs need: residual rows <= y1 + 1 -> input rows <= y1 + 2 (and inside the box)
  auto rowok = [&](int b) { return b >= -g.G && b < g.n[1] + g.G; };
  auto issue = [&](int it) {
    if (it < nrows) {
      const int b = ybeg + it, slot = it % NST;
      const int64_t o = ob0 + (int64_t)it * px;
      cp16(x + o, slot, 0, xload && rowok(b));
      const bool dom = b >= 0 && b < g.n[1];
      cp16(f + o, slot, 1, xload && dom);
      if (!urow(b) && dom) cp16(sig + o, slot, 2, xload);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int k = 0; k < PD; ++k) issue(k);
  const CC z = make_double2(0, 0);
  const CR zr = mkc<TC>(0, 0);
  CR a0 = zr, a1 = zr, b0 = zr, b1 = zr, aw = zr, ae = zr, bw = zr, be = zr;
  auto shl = [](auto v) { return __shfl_up_sync(0xffffffffu, v, 1); };
  auto shr = [](auto v) { return __shfl_down_sync(0xffffffffu, v, 1); };
  const TC alp = (TC)alpha, ih2c = (TC)ih2;
  const CR usr = mkc<TC>((TC)us.x, (TC)us.y);
  CC P = z, Q = z;   // y-pass accumulators of coarse rows I0 - 1 and I0 (see below)
  const double w2 = 0.0625, w1 = 0.25, w0 = 0.375;   // RW<2>::w(+-2), (+-1), 0
  for (int it = 0; it < nrows; ++it) {
    issue(it + PD);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(PD) : "memory");
    const float4 *sl = ring + (it % NST) * NW * 32 + lane;
    const float4 xv = sl[0];
    const CR c0 = mkc<TC>(xv.x, xv.y), c1 = mkc<TC>(xv.z, xv.w);
    const CR cw = mkc<TC>(shl(c1.x), shl(c1.y)), ce = mkc<TC>(shr(c0.x), shr(c0.y));
    if (it >= 2) {
      const int b = ybeg + it - 1;   // residual row (rows a = b-1, b, c = b+1)
      float2 r0 = make_float2(0, 0), r1 = make_float2(0, 0);
      if (rlane && b >= 0 && b < g.n[1]) {
        const float4 *sb = ring + ((it - 1) % NST) * NW * 32 + lane;   // row b's f and sigma
        CR sg0, sg1;
        if (urow(b)) {
          sg0 = sg1 = usr;
        } else {
          const float4 v = sb[2 * 32];
          sg0 = mkc<TC>(v.x, v.y);
          sg1 = mkc<TC>(v.z, v.w);
        }
        const float4 fv = sb[32];
        auto node = [&](CR cc, CR w_, CR e_, CR n_, CR s_, CR nw, CR ne, CR sw, CR se_, CR sgm, TC fx, TC fy) {
          const CR sf = cadd<TC>(cadd<TC>(w_, e_), cadd<TC>(n_, s_));
          CR Lx = cscale<TC>(cc, (TC)W::Lc);
          Lx = cfmar<TC>(Lx, (TC)W::Lf, sf);
          if (W::Le != 0.0) Lx = cfmar<TC>(Lx, (TC)W::Le, cadd<TC>(cadd<TC>(nw, ne), cadd<TC>(sw, se_)));
          Lx = cscale<TC>(Lx, ih2c);
          CR Mx = cscale<TC>(cc, (TC)W::Mc);
          if (W::Mf != 0.0) Mx = cfmar<TC>(Mx, (TC)W::Mf, sf);
          sgm.y = fma(-alp, sgm.x, sgm.y);
          return csub<TC>(mkc<TC>(fx, fy), csub<TC>(Lx, cmul<TC>(sgm, Mx)));
        };
        if (in0) {
          const CR o0 = node(b0, bw, b1, a0, c0, aw, a1, cw, c1, sg0, fv.x, fv.y);
          r0 = make_float2((float)o0.x, (float)o0.y);
        }
        if (in1) {
          const CR o1 = node(b1, b0, be, a1, c1, a0, ae, c0, ce, sg1, fv.z, fv.w);
          r1 = make_float2((float)o1.x, (float)o1.y);
        }
      }
      // x-pass of the restriction at coarse column X (fine 2X = x0): r at x0-2, x0-1 (left
      // lane's pair), x0, x0+1 (own), x0+2 (right lane's first)
      // the fp32-rounded residuals widened once per lane and shuffled as doubles (an
      // F2F costs four DFMA issue slots on B200, a 64-bit shuffle two SHFL)
      const CC R0 = ccast<double, float>(r0), R1 = ccast<double, float>(r1);
      const CC lm2 = make_double2(shl(R0.x), shl(R0.y));
      const CC lm1 = make_double2(shl(R1.x), shl(R1.y));
      const CC rp2 = make_double2(shr(R0.x), shr(R0.y));
      CC hx = make_double2(0, 0);
      hx = cfmar<double>(hx, w2, lm2);
      hx = cfmar<double>(hx, w1, lm1);
      hx = cfmar<double>(hx, w0, R0);
      hx = cfmar<double>(hx, w1, R1);
      hx = cfmar<double>(hx, w2, rp2);
      // y-pass: fine row b = 2 I0 + ky.  Even b: completes row I0 - 1 (ky = +2), continues
      // I0 (ky = 0), opens I0 + 1 (ky = -2).  Odd b: ky = +1 for I0, -1 for I0 + 1.
      if ((b & 1) == 0) {
        P = cfmar<double>(P, w2, hx);
        const int I = (b >> 1) - 1;
        if (clane && I >= 0 && I < gc.n[1] && 2 * I >= y0 && 2 * I < y1) fc[gc.idx(X, I, 0)] = P;
        Q = cfmar<double>(Q, w0, hx);
        P = Q;
        Q = cfmar<double>(make_double2(0, 0), w2, hx);
      } else {
        P = cfmar<double>(P, w1, hx);
        Q = cfmar<double>(Q, w1, hx);
      }
    }
    a0 = b0; a1 = b1; aw = bw; ae = be;
    b0 = c0; b1 = c1; bw = cw; be = ce;
  }
}

// Stored stencil of radius R: coef[k][j], k = (ox+R) + (2R+1)((oy+R) + (2R+1)(oz+R)),
// multiplies x[j + o].  Coefficients towards out-of-domain nodes are zero.
// TV = vector storage/arithmetic (fp64 on Galerkin levels), TK = coefficient storage.
template <int DIM, int R> constexpr int kplanes() { return DIM == 3 ? (2 * R + 1) * (2 * R + 1) * (2 * R + 1) : (2 * R + 1) * (2 * R + 1); }

template <typename TV, typename TK, int DIM, int R, int NR = 1, int BZ = 1, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_stored_op(Geo g, const cplx<TK> *__restrict__ coef,
                                                   const cplx<TV> *__restrict__ x,
                                                   const cplx<TV> *__restrict__ f, cplx<TV> *__restrict__ y,
                                                   int64_t bs, UBox ub, UCoef<kplanes<DIM, R>(), TV> uc,
                                                   const unsigned short *__restrict__ cls,
                                                   const cplx<TK> *__restrict__ tab) {
  HMG_PDL_PROLOGUE();
  // cls != null: coefficient dictionary (k_dict.cuh): node i's coefficients are
  // tab[cls[i]][0 .. K) (stored precision, converted like the planes)
  // NR right-hand sides at a stride of bs elements: each coefficient is read once
  // and applied to all of them (multi-RHS batches; same per-RHS arithmetic order).
  // BZ consecutive nodes along the slowest axis per thread (register blocking: each
  // loaded input plane / row serves every output it reaches); input planes are
  // visited in increasing order, so each output accumulates its terms in the
  // offset order k (oz, oy, ox ascending) -- the same arithmetic for any BZ.
  using T = TV;
  constexpr int W = 2 * R + 1;
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
  const int64_t i0 = g.idx(ix, iy, iz);
  const int64_t ps = DIM == 3 ? g.pxy : g.px;   // slow-axis pitch
  const int slow0 = DIM == 3 ? iz : iy, nslow = DIM == 3 ? g.n[2] : g.n[1];
  const int olast = min(slow0 + BZ, nslow) - 1 - slow0;   // last valid output of the block
  bool uni = DIM == 3 ? ub.in(ix, iy, iz) && ub.in(ix, iy, iz + olast)
                      : ub.in(ix, iy, 0) && ub.in(ix, iy + olast, 0);
  // a warp with lanes on both sides of the box (an x-normal sponge face) would run BOTH copies of
  // the unrolled loop; with a dictionary every lane can take its class's entry instead -- inside
  // the box that is the box's own class, bitwise the uniform copy -- so such a warp runs one
  if (cls && !__all_sync(__activemask(), uni)) uni = false;
  cplx<T> acc[BZ][NR];
#pragma unroll
  for (int o = 0; o < BZ; ++o)
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[o][r] = mkc<T>(0, 0);
  constexpr int YR = DIM == 3 ? R : 0;   // in-plane y reach (3D only)
  auto run = [&](auto coef_k) {
#pragma unroll
    for (int s = -R; s < BZ + R; ++s) {
      if (s > olast + R) break;   // beyond the last valid output's reach
#pragma unroll
      for (int oy = -YR; oy <= YR; ++oy)
#pragma unroll
        for (int ox = -R; ox <= R; ++ox) {
          const int64_t j = i0 + (int64_t)s * ps + (DIM == 3 ? (int64_t)oy * g.px : 0) + ox;
          cplx<T> xv[NR];
#pragma unroll
          for (int r = 0; r < NR; ++r) xv[r] = x[r * bs + j];
#pragma unroll
          for (int o = 0; o < BZ; ++o) {
            const int d = s - o;   // slow-axis offset of this input for output o
            if (d < -R || d > R) continue;
            const int k = DIM == 3 ? ((d + R) * W + oy + R) * W + ox + R : (d + R) * W + ox + R;
            const cplx<T> c = coef_k(k, o);
#pragma unroll
            for (int r = 0; r < NR; ++r) acc[o][r] = cfma<T>(acc[o][r], c, xv[r]);
          }
        }
    }
  };
  // two copies of the unrolled loop behind a branch (not a per-coefficient select:
  // predicated-off loads and conversions would still take issue slots)
  if (uni) {
    run([&](int k, int) { return uc.c[k]; });
  } else if (cls) {
    constexpr int KP = kplanes<DIM, R>();
    const cplx<TK> *cb[BZ];
#pragma unroll
    for (int o = 0; o < BZ; ++o) cb[o] = tab + (int64_t)cls[i0 + (int64_t)min(o, olast) * ps] * KP;
    run([&](int k, int o) { return ccast<T, TK>(cb[o][k]); });
  } else {
    run([&](int k, int o) { return ccast<T, TK>(coef[(int64_t)k * g.total + i0 + (int64_t)o * ps]); });
  }
#pragma unroll
  for (int o = 0; o < BZ; ++o) {
    if (o > olast) break;
    const int64_t i = i0 + (int64_t)o * ps;
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r * bs + i] = f ? csub<T>(f[r * bs + i], acc[o][r]) : acc[o][r];
  }
}

// 2D c64 variant of k_stored_op: one thread per PAIR of x-adjacent nodes (2p,
// 2p+1) and BY consecutive rows (register blocking along y): the fp32
// coefficient planes load as aligned 16-byte pairs, the two nodes share their
// x-window (2R + 2 loads per row instead of 2 (2R + 1)), and each loaded input
// row serves every one of the BY output rows it reaches (2R + BY input rows for
// BY outputs instead of (2R + 1) BY).  Input rows are visited in increasing order
// and each output accumulates its terms in the offset order of k_stored_op, so
// the per-node arithmetic (and result) is that of k_stored_op.
//
// TILE (block 32 x 8): the block's 64 x 8 BY input tile plus a halo of 2 columns / R rows is
// first copied to shared memory by cp.async (even and odd columns in separate arrays, so
// the lanes' window reads are consecutive 16-byte words: conflict-free), and the x-window
// is read from there: one global load per input element and block instead of a latency-
// bound gather per thread (the arithmetic is unchanged: bit-identical).
template <int BY, int R> struct Tile2D {
  static constexpr int TH = 8 * BY + 2 * R, TC = 34;   // rows; 16-byte words per parity (68 columns)
};
template <int BY, int R>
__device__ __forceinline__ void tile2d_load(const Geo &g, const double2 *__restrict__ x, double2 (*E)[34],
                                            double2 (*O)[34]) {
  constexpr int TH = Tile2D<BY, R>::TH;
  const int X0 = blockIdx.x * 64, Y0 = blockIdx.y * 8 * BY;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int e = tid; e < TH * 68; e += 256) {
    const int tr = e / 68, tc = e - tr * 68;
    const int gx = X0 - 2 + tc, gy = Y0 - R + tr;
    const bool ok = gx < g.n[0] + g.G && gy < g.n[1] + g.G;
    double2 *dst = (tc & 1) ? &O[tr][tc >> 1] : &E[tr][tc >> 1];
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    const double2 *src = ok ? x + g.idx(gx, gy, 0) : x;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 16 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
}
template <int R, int BY = 1, bool DICT = false, bool TILE = false>
__global__ void __launch_bounds__(256) k_stored_op2d_pair(Geo g, const float2 *__restrict__ coef,
                                                          const double2 *__restrict__ x,
                                                          const double2 *__restrict__ f, double2 *__restrict__ y,
                                                          UBox ub, UCoef<(2 * R + 1) * (2 * R + 1), double> uc,
                                                          const unsigned short *__restrict__ cls,
                                                          const float2 *__restrict__ tab) {
  HMG_PDL_PROLOGUE();
  using T = double;
  constexpr int W = 2 * R + 1;
  constexpr int TH = TILE ? Tile2D<BY, R>::TH : 1;
  __shared__ __align__(16) double2 tE[TILE ? TH : 1][34], tO[TILE ? TH : 1][34];
  if (TILE) tile2d_load<BY, R>(g, x, tE, tO);
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int iy0 = (blockIdx.y * blockDim.y + threadIdx.y) * BY;
  const int ix = 2 * p;
  if (ix >= g.n[0] || iy0 >= g.n[1]) return;
  const int64_t i0 = g.idx(ix, iy0, 0);
  const int64_t px = g.px;
  const bool two = ix + 1 < g.n[0];
  const int ylast = min(iy0 + BY, g.n[1]) - 1;
  // every node of the BY x 2 block in the uniform box
  const bool uni = ub.in(ix, iy0, 0) && ub.in(ix, ylast, 0) && (!two || ub.in(ix + 1, iy0, 0));
  double2 a0[BY], a1[BY];
#pragma unroll
  for (int o = 0; o < BY; ++o) a0[o] = a1[o] = make_double2(0, 0);
  // input rows past the last output row's reach are never needed (and may lie
  // beyond the padded box of a ragged block): they are skipped
  const int rmax = ylast - iy0 + R;
  // uniform box: fp64 coefficient copies from the parameter bank, no loads, no
  // conversions -- a separate copy of the unrolled loop behind one branch
  auto run = [&](auto coef_k) {
#pragma unroll
    for (int r = -R; r < BY + R; ++r) {
      if (r > rmax) break;
      double2 xw[2 * R + 2];
      if (TILE) {   // tile row threadIdx.y * BY + r + R; column ix - R + c = tile column 2 tx + 2 - R + c
        const int tr = threadIdx.y * BY + r + R, tx = threadIdx.x;
#pragma unroll
        for (int c = 0; c < 2 * R + 2; ++c) {
          const int tc = 2 - R + c;   // >= 0 (R <= 2)
          xw[c] = (tc & 1) ? tO[tr][tx + (tc >> 1)] : tE[tr][tx + (tc >> 1)];
        }
      } else {
        const double2 *row = x + i0 + (int64_t)r * px;
#pragma unroll
        for (int c = 0; c < 2 * R + 2; ++c) xw[c] = row[c - R];
      }
#pragma unroll
      for (int o = 0; o < BY; ++o) {
        const int oy = r - o;   // offset of this input row for output row o
        if (oy < -R || oy > R) continue;
#pragma unroll
        for (int ox = -R; ox <= R; ++ox) {
          const int k = (oy + R) * W + ox + R;
          double2 k0, k1;
          coef_k(k, o, k0, k1);
          a0[o] = cfma<T>(a0[o], k0, xw[ox + R]);
          a1[o] = cfma<T>(a1[o], k1, xw[ox + R + 1]);
        }
      }
    }
  };
  if (uni) {
    run([&](int k, int, double2 &k0, double2 &k1) { k0 = k1 = uc.c[k]; });
  } else if (DICT) {   // coefficient dictionary (k_dict.cuh): tab[class][k]
    const float2 *cb0[BY], *cb1[BY];
#pragma unroll
    for (int o = 0; o < BY; ++o) {
      const int64_t i = i0 + (int64_t)min(o, ylast - iy0) * px;
      cb0[o] = tab + (int64_t)cls[i] * (W * W);
      cb1[o] = tab + (int64_t)cls[two ? i + 1 : i] * (W * W);
    }
    run([&](int k, int o, double2 &k0, double2 &k1) {
      const float2 c0 = cb0[o][k], c1 = cb1[o][k];
      k0 = mkc<T>(c0.x, c0.y);
      k1 = mkc<T>(c1.x, c1.y);
    });
  } else {
    run([&](int k, int o, double2 &k0, double2 &k1) {
      const float4 c2 = *reinterpret_cast<const float4 *>(coef + (int64_t)k * g.total + i0 + (int64_t)o * px);
      k0 = mkc<T>(c2.x, c2.y);
      k1 = mkc<T>(c2.z, c2.w);
    });
  }
#pragma unroll
  for (int o = 0; o < BY; ++o) {
    if (iy0 + o > ylast) break;
    const int64_t i = i0 + (int64_t)o * px;
    y[i] = f ? csub<T>(f[i], a0[o]) : a0[o];
    if (two) y[i + 1] = f ? csub<T>(f[i + 1], a1[o]) : a1[o];
  }
}

// Level-l residual / apply of the stored radius-R stencil (2D, c64 path: fp32 coefficient
// planes, fp64 level vectors) as a WARP-MARCHING kernel: lane l holds the column pair
// (x0, x0 + 1), x0 = 60 s - 2 + 2 l (lanes 1..30 write, 0 and 31 supply neighbours), the
// warp marches down SEG output rows; every input row is loaded once (32 bytes per lane
// through a cp.async ring, PD rows ahead), its +-R column neighbours come from the
// neighbour lanes by shuffles, and it is added at once to the 2R + 1 output rows it
// reaches (rolling accumulators).  Each output accumulates its terms in the offset order
// k = (oy + R)(2R + 1) + ox + R ascending -- the arithmetic of k_stored_op2d_pair.
// Coefficients come from the uniform-box copy inside the box, else from the stored planes.
constexpr int SM_STRIP = 60;
template <int R, int SEG, int PD>
__global__ void __launch_bounds__(128) k_stored_op2d_march(Geo g, const float2 *__restrict__ coef,
                                                           const double2 *__restrict__ x,
                                                           const double2 *__restrict__ f, double2 *__restrict__ y,
                                                           UBox ub, UCoef<(2 * R + 1) * (2 * R + 1), double> uc) {
  HMG_PDL_PROLOGUE();
  static_assert(R == 2 || R == 1, "radius 1 or 2");
  using T = double;
  constexpr int W = 2 * R + 1, NST = PD + 2;
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nstrips = (g.n[0] + SM_STRIP - 1) / SM_STRIP;
  const int strip = wid % nstrips, seg = wid / nstrips;
  const int y0 = seg * SEG;
  if (y0 >= g.n[1]) return;
  const int y1 = min(g.n[1], y0 + SEG);
  const int x0 = strip * SM_STRIP - 2 + 2 * lane;
  const bool out_lane = lane >= 1 && lane <= 30 && x0 < g.n[0];
  const bool two = x0 + 1 < g.n[0];
  const bool xload = x0 < g.n[0] + g.G;   // columns past the ghost layer are never used
  // both nodes of the pair inside the box's columns (rows are checked per output row)
  const bool xuni = x0 >= ub.lo[0] && (two ? x0 + 1 : x0) < ub.hi[0];
  extern __shared__ __align__(16) unsigned char sm_smem[];
  double2 *ring = reinterpret_cast<double2 *>(sm_smem) + (size_t)(threadIdx.x >> 5) * (NST * 2 * 32);
  const int64_t px = g.px;
  const int64_t ob0 = g.base + x0 + (int64_t)(y0 - R) * px;   // input row y0 - R, column x0
  const int nin = y1 - y0 + 2 * R;                               // input rows y0-R .. y1-1+R
  auto issue = [&](int it) {
    if (it < nin) {
      const int slot = it % NST;
      const double2 *src = x + ob0 + (int64_t)it * px;
      for (int h = 0; h < 2; ++h) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(ring + (slot * 2 + h) * 32 + lane);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(xload ? src + h : x),
                     "r"(xload ? 16 : 0)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int k = 0; k < PD; ++k) issue(k);
  auto shl = [](double v) { return __shfl_up_sync(0xffffffffu, v, 1); };
  auto shr = [](double v) { return __shfl_down_sync(0xffffffffu, v, 1); };
  // acc[q][n]: output row (input row - R + q) ... rolling: slot 0 = the oldest output row
  double2 a0[W], a1[W];
#pragma unroll
  for (int q = 0; q < W; ++q) a0[q] = a1[q] = make_double2(0, 0);
  for (int it = 0; it < nin; ++it) {
    issue(it + PD);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(PD) : "memory");
    const double2 *sl = ring + (it % NST) * 2 * 32 + lane;
    const double2 c0 = sl[0], c1 = sl[32];
    // window of the row: columns x0-2 .. x0+3
    double2 xw[6];
    xw[2] = c0;
    xw[3] = c1;
    xw[1] = make_double2(shl(c1.x), shl(c1.y));
    xw[4] = make_double2(shr(c0.x), shr(c0.y));
    if (R == 2) {
      xw[0] = make_double2(shl(c0.x), shl(c0.y));
      xw[5] = make_double2(shr(c1.x), shr(c1.y));
    } else {
      xw[0] = xw[5] = make_double2(0, 0);
    }
    const int yin = y0 - R + it;   // this input row
    // add it to the outputs yo = yin - oy, oy = -R..R (accumulator q = R - oy ... newest last)
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int oy = R - q;           // offset of the input row for the output in accumulator q
      const int yo = yin - oy;
      if (yo < y0 || yo >= y1 || !out_lane) continue;
      const bool uni = xuni && yo >= ub.lo[1] && yo < ub.hi[1];
      const int64_t io = ob0 + (int64_t)(yo - y0 + R) * px;
#pragma unroll
      for (int ox = -R; ox <= R; ++ox) {
        const int k = (oy + R) * W + ox + R;
        double2 k0, k1;
        if (uni) {
          k0 = k1 = uc.c[k];
        } else {
          const float4 cc = *reinterpret_cast<const float4 *>(coef + (int64_t)k * g.total + io);
          k0 = mkc<T>(cc.x, cc.y);
          k1 = mkc<T>(cc.z, cc.w);
        }
        a0[q] = cfma<T>(a0[q], k0, xw[ox + 2]);
        a1[q] = cfma<T>(a1[q], k1, xw[ox + 3]);
      }
    }
    // output row yin - R (accumulator 0) is complete
    const int yo = yin - R;
    if (yo >= y0 && yo < y1 && out_lane) {
      const int64_t io = ob0 + (int64_t)(yo - y0 + R) * px;
      if (f) {
        const double2 f0 = f[io];
        y[io] = csub<T>(f0, a0[0]);
        if (two) y[io + 1] = csub<T>(f[io + 1], a1[0]);
      } else {
        y[io] = a0[0];
        if (two) y[io + 1] = a1[0];
      }
    }
#pragma unroll
    for (int q = 0; q + 1 < W; ++q) { a0[q] = a0[q + 1]; a1[q] = a1[q + 1]; }
    a0[W - 1] = a1[W - 1] = make_double2(0, 0);
  }
}

}  // namespace hmg
