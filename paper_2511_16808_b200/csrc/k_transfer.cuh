// k_transfer.cuh -- intergrid transfers (§3.1).
//
// 1D restriction weights centred at fine node 2I (coarse node I == fine 2I):
//   lin [1 2 1]/4        (Eq. 3.1; full weighting)
//   cub [1 4 6 4 1]/16   (Eq. 3.2; bicubic)
// dD operators are tensor products (Eqs. 3.5-3.6); P = 2^d R^T of
// the P-kind weights, i.e. per axis: even fine node 2J gets
// (1/8, 3/4, 1/8) of coarse (J-1, J, J+1) for cub and 1 x J for lin; odd fine
// node 2J+1 gets 1/2 of J and 1/2 of J+1 for both.  Truncation at the boundary
// comes from the zero ghost layer (reading A5).
#pragma once
#include "common.cuh"

namespace hmg {

template <int RR> struct RW;
template <> struct RW<1> {
  __device__ static constexpr double w(int k) { return k == 0 ? 0.5 : 0.25; }
};
template <> struct RW<2> {
  __device__ static constexpr double w(int k) { return k == 0 ? 0.375 : (k == 1 || k == -1) ? 0.25 : 0.0625; }
};

// fc[I] = sum_k w(k) r[2I + k]     (coarse-node parallel; fp64 arithmetic,
// TI/TO = storage of the fine input / coarse output)
template <typename TI, typename TO, int DIM, int RR>
__global__ void __launch_bounds__(256) k_restrict(Geo gf, Geo gc, const cplx<TI> *__restrict__ r,
                                                  cplx<TO> *__restrict__ fc) {
  HMG_PDL_PROLOGUE();
  using T = double;
  HMG_NODE_IDX(gc, X, Y, Z);
  const int64_t ic = gc.idx(X, Y, Z);
  // coarse node I (global) sits on fine node 2I (global); map to fine-local
  const int64_t jf = gf.idx(2 * (X + gc.o[0]) - gf.o[0], 2 * (Y + gc.o[1]) - gf.o[1],
                            DIM == 3 ? 2 * (Z + gc.o[2]) - gf.o[2] : 0);
  constexpr int ZR = DIM == 3 ? RR : 0;
  cplx<T> acc = mkc<T>(0, 0);
#pragma unroll
  for (int kz = -ZR; kz <= ZR; ++kz) {
    cplx<T> accy = mkc<T>(0, 0);
#pragma unroll
    for (int ky = -RR; ky <= RR; ++ky) {
      cplx<T> accx = mkc<T>(0, 0);
#pragma unroll
      for (int kx = -RR; kx <= RR; ++kx)
        accx = cfmar<T>(accx, (T)RW<RR>::w(kx), ccast<T, TI>(r[jf + gf.delta(kx, ky, kz)]));
      accy = cfmar<T>(accy, (T)RW<RR>::w(ky), accx);
    }
    acc = DIM == 3 ? cfmar<T>(acc, (T)RW<RR>::w(kz), accy) : accy;
  }
  fc[ic] = ccast<TO, T>(acc);
}

// c64 fine-level restriction with cubic weights (RR = 2), 2D or 3D: the 5-wide fine
// window 2X-2 .. 2X+2 starts at an even column, so each fine row loads as three aligned
// 16-byte pairs (3D: 75 loads instead of 125 per coarse node -- the scalar gather is
// load-issue-bound); same fma order as k_restrict.
template <int DIM>
__global__ void __launch_bounds__(256) k_restrict_pair(Geo gf, Geo gc, const float2 *__restrict__ r,
                                                       double2 *__restrict__ fc) {
  HMG_PDL_PROLOGUE();
  using T = double;
  HMG_NODE_IDX(gc, X, Y, Z);
  const int64_t ic = gc.idx(X, Y, Z);
  const int64_t jf = gf.idx(2 * (X + gc.o[0]) - gf.o[0], 2 * (Y + gc.o[1]) - gf.o[1],
                            DIM == 3 ? 2 * (Z + gc.o[2]) - gf.o[2] : 0);
  constexpr int ZR = DIM == 3 ? 2 : 0;
  double2 acc = make_double2(0, 0);
#pragma unroll
  for (int kz = -ZR; kz <= ZR; ++kz) {
    double2 accy = make_double2(0, 0);
#pragma unroll
    for (int ky = -2; ky <= 2; ++ky) {
      const float4 *row = reinterpret_cast<const float4 *>(r + jf + gf.delta(-2, ky, kz));
      const float4 p0 = row[0], p1 = row[1], p2 = row[2];
      const float2 v[5] = {make_float2(p0.x, p0.y), make_float2(p0.z, p0.w), make_float2(p1.x, p1.y),
                           make_float2(p1.z, p1.w), make_float2(p2.x, p2.y)};
      double2 accx = make_double2(0, 0);
#pragma unroll
      for (int kx = -2; kx <= 2; ++kx) accx = cfmar<T>(accx, RW<2>::w(kx), ccast<T, float>(v[kx + 2]));
      accy = cfmar<T>(accy, RW<2>::w(ky), accx);
    }
    acc = DIM == 3 ? cfmar<T>(acc, RW<2>::w(kz), accy) : accy;
  }
  fc[ic] = acc;
}

// 3D c64 fine-level restriction with BZ coarse planes per thread: the in-plane (x, y)
// restricted value accy(p) of a fine plane p does not depend on the coarse plane it feeds,
// so each fine plane is loaded and reduced ONCE per thread and added, with the z weight,
// to every coarse output it reaches (fine planes 2Z-2 .. 2Z+2 of output Z, in increasing
// order = kz ascending): the arithmetic of k_restrict_pair<3>, 2BZ + 3 fine planes for BZ
// outputs instead of 5 BZ.  One rank (no offsets).
template <int BZ>
__global__ void __launch_bounds__(256) k_restrict_pair3_z(Geo gf, Geo gc, const float2 *__restrict__ r,
                                                          double2 *__restrict__ fc) {
  HMG_PDL_PROLOGUE();
  using T = double;
  const int X = blockIdx.x * blockDim.x + threadIdx.x, Y = blockIdx.y * blockDim.y + threadIdx.y;
  const int Z0 = blockIdx.z * BZ;
  if (X >= gc.n[0] || Y >= gc.n[1] || Z0 >= gc.n[2]) return;
  const int zl = min(BZ, gc.n[2] - Z0);   // outputs of this thread
  double2 acc[BZ];
#pragma unroll
  for (int o = 0; o < BZ; ++o) acc[o] = make_double2(0, 0);
  const int64_t jf0 = gf.idx(2 * X, 2 * Y, 2 * Z0);
#pragma unroll
  for (int q = -2; q <= 2 * BZ; ++q) {   // fine plane 2 Z0 + q
    if (q > 2 * (zl - 1) + 2) break;
    double2 accy = make_double2(0, 0);
#pragma unroll
    for (int ky = -2; ky <= 2; ++ky) {
      const float4 *row = reinterpret_cast<const float4 *>(r + jf0 + gf.delta(-2, ky, q));
      const float4 p0 = row[0], p1 = row[1], p2 = row[2];
      const float2 v[5] = {make_float2(p0.x, p0.y), make_float2(p0.z, p0.w), make_float2(p1.x, p1.y),
                           make_float2(p1.z, p1.w), make_float2(p2.x, p2.y)};
      double2 accx = make_double2(0, 0);
#pragma unroll
      for (int kx = -2; kx <= 2; ++kx) accx = cfmar<T>(accx, RW<2>::w(kx), ccast<T, float>(v[kx + 2]));
      accy = cfmar<T>(accy, RW<2>::w(ky), accx);
    }
#pragma unroll
    for (int o = 0; o < BZ; ++o) {
      const int kz = q - 2 * o;   // offset of this plane for output Z0 + o
      if (kz < -2 || kz > 2) continue;
      acc[o] = cfmar<T>(acc[o], RW<2>::w(kz), accy);
    }
  }
#pragma unroll
  for (int o = 0; o < BZ; ++o)
    if (o < zl) fc[gc.idx(X, Y, Z0 + o)] = acc[o];
}

// 3D prolongation + correction with BZ coarse planes per thread: the 3 x 3 coarse window of a
// coarse plane is loaded once and reused by the (up to) 3 coarse planes around it; the fine
// children 2J + {0,1}^3 of each coarse node get exactly k_prolong_block's sums.  One rank.
template <typename TU, int PR, int BZ>
__global__ void __launch_bounds__(256) k_prolong3_z(Geo gf, Geo gc, const double2 *__restrict__ e,
                                                    const cplx<TU> *u, cplx<TU> *u_out) {
  HMG_PDL_PROLOGUE();
  using T = double;
  const int X = blockIdx.x * blockDim.x + threadIdx.x, Y = blockIdx.y * blockDim.y + threadIdx.y;
  const int Z0 = blockIdx.z * BZ;
  if (X >= gc.n[0] || Y >= gc.n[1] || Z0 >= gc.n[2]) return;
  auto plane = [&](int Z, cplx<T> (&c)[3][3]) {
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) c[dy][dx] = e[gc.idx(X - 1 + dx, Y - 1 + dy, Z)];
  };
  auto wt = [](int p, int k) -> double {
    if (p == 0) return PR == 2 ? (k == 1 ? 0.75 : 0.125) : (k == 1 ? 1.0 : 0.0);
    return k == 0 ? 0.0 : 0.5;
  };
  cplx<T> c[3][3][3];   // coarse planes Z-1, Z, Z+1
  plane(Z0 - 1, c[0]);
  plane(Z0, c[1]);
  for (int o = 0; o < BZ; ++o) {
    const int Z = Z0 + o;
    if (Z >= gc.n[2]) break;
    plane(Z + 1, c[2]);
#pragma unroll
    for (int pz = 0; pz < 2; ++pz)
#pragma unroll
      for (int py = 0; py < 2; ++py)
#pragma unroll
        for (int px = 0; px < 2; ++px) {
          const int fx = 2 * X + px, fy = 2 * Y + py, fz = 2 * Z + pz;
          if (fx >= gf.n[0] || fy >= gf.n[1] || fz >= gf.n[2]) continue;
          cplx<T> acc = mkc<T>(0, 0);
#pragma unroll
          for (int dz = 0; dz < 3; ++dz) {
            const double wz = wt(pz, dz);
            if (wz == 0.0) continue;
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
              const double wy = wt(py, dy);
              if (wy == 0.0) continue;
#pragma unroll
              for (int dx = 0; dx < 3; ++dx) {
                const double wx = wt(px, dx);
                if (wx == 0.0) continue;
                acc = cfmar<T>(acc, wx * wy * wz, c[dz][dy][dx]);
              }
            }
          }
          const int64_t i = gf.idx(fx, fy, fz);
          u_out[i] = ccast<TU, T>(cadd<T>(ccast<T, TU>(u[i]), acc));
        }
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        c[0][dy][dx] = c[1][dy][dx];
        c[1][dy][dx] = c[2][dy][dx];
      }
  }
}

// Prolongation + correction  u_out = u + P e  (Alg. 2.1 step 4), coarse-node parallel: the thread of coarse node J writes
// the 2^d fine nodes 2J + {0,1}^d (global parity), loading its 3^d coarse
// neighbourhood once (instead of up to 3^d loads per fine node).  Fine nodes
// outside this rank's rows / the domain are skipped.  u_out may equal u.
template <typename TE, typename TU, int DIM, int PR>
__global__ void __launch_bounds__(256) k_prolong_block(Geo gf, Geo gc, int cx0, int cy0, int cz0, int ncx, int ncy,
                                                       int ncz, const cplx<TE> *__restrict__ e, const cplx<TU> *u,
                                                       cplx<TU> *u_out) {
  HMG_PDL_PROLOGUE();
  using T = double;
  const int X = cx0 + (int)(blockIdx.x * blockDim.x + threadIdx.x);   // GLOBAL coarse coordinates
  const int Y = cy0 + (int)(blockIdx.y * blockDim.y + threadIdx.y);
  const int Z = cz0 + (int)blockIdx.z;
  if (X >= cx0 + ncx || Y >= cy0 + ncy || (DIM == 3 && Z >= cz0 + ncz)) return;
  constexpr int ZW = DIM == 3 ? 3 : 1;
  cplx<T> c[ZW][3][3];
#pragma unroll
  for (int dz = 0; dz < ZW; ++dz)
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int jx = X - 1 + dx - gc.o[0], jy = Y - 1 + dy - gc.o[1], jz = DIM == 3 ? Z - 1 + dz - gc.o[2] : 0;
        c[dz][dy][dx] = ccast<T, TE>(e[gc.idx(jx, jy, jz)]);   // coarse ghosts are zero / halo
      }
  // 1D weights of fine parity p (0 even, 1 odd) on coarse offsets -1, 0, +1
  auto wt = [](int p, int k) -> double {
    if (p == 0) return PR == 2 ? (k == 1 ? 0.75 : 0.125) : (k == 1 ? 1.0 : 0.0);
    return k == 0 ? 0.0 : 0.5;   // odd fine 2J+1: J (k=1) and J+1 (k=2)
  };
#pragma unroll
  for (int pz = 0; pz < (DIM == 3 ? 2 : 1); ++pz)
#pragma unroll
    for (int py = 0; py < 2; ++py)
#pragma unroll
      for (int px = 0; px < 2; ++px) {
        const int fx = 2 * X + px - gf.o[0], fy = 2 * Y + py - gf.o[1], fz = DIM == 3 ? 2 * Z + pz - gf.o[2] : 0;
        if (fx < 0 || fx >= gf.n[0] || fy < 0 || fy >= gf.n[1] || (DIM == 3 && (fz < 0 || fz >= gf.n[2]))) continue;
        cplx<T> acc = mkc<T>(0, 0);
#pragma unroll
        for (int dz = 0; dz < ZW; ++dz) {
          const double wz = DIM == 3 ? wt(pz, dz) : 1.0;
          if (wz == 0.0) continue;
#pragma unroll
          for (int dy = 0; dy < 3; ++dy) {
            const double wy = wt(py, dy);
            if (wy == 0.0) continue;
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
              const double wx = wt(px, dx);
              if (wx == 0.0) continue;
              acc = cfmar<T>(acc, wx * wy * wz, c[dz][dy][dx]);
            }
          }
        }
        const int64_t i = gf.idx(fx, fy, fz);
        u_out[i] = ccast<TU, T>(cadd<T>(ccast<T, TU>(u[i]), acc));
      }
}

// Level-1 operator of the Galerkin hierarchy evaluated MATRIX-FREE through the
// fine grid (2D):  A_1 u = R_0 (L - diag(sigma_s) M) P_0 u, i.e.
// y = A_1 u  or  y = f - A_1 u, with t = P u and s = H_s t formed on the fine
// tile in shared memory.  Truncation is exact: t and s vanish outside the
// domain (P and R have no rows there), L and M read those zeros.  Reads u and f
// on the coarse tile and sigma on the fine tile: 2-3 vectors + 4 sigma values
// per coarse node instead of the (2r+1)^2 stored coefficient planes.
// Both transfers are applied separably (x pass, then y pass) with 3 / 2RR+1
// branch-free taps (odd fine nodes take weight 0 on their first tap).
// Shared memory (dynamic): region A = {u tile, P_x u} then s; region B = t,
// then R_x s.  f and the tile's sigma are prefetched into registers.
template <int PR, typename T>
__device__ __forceinline__ void ptaps3(int x, int &c, int &d0, T &w0, T &w1, T &w2) {
  // fine x -> coarse taps (c + d0, c, c + 1) with weights w0..w2; every tap address
  // lies in the coarse support of x (odd x: d0 = 0 with w0 = 0), so no read leaves the tile
  c = x >> 1;   // floor
  const bool odd = x & 1;
  if (PR == 2) {
    d0 = odd ? 0 : -1;
    w0 = odd ? T(0) : T(0.125);
    w1 = odd ? T(0.5) : T(0.75);
    w2 = odd ? T(0.5) : T(0.125);
  } else {
    d0 = 0;
    w0 = T(0);
    w1 = odd ? T(0.5) : T(1);
    w2 = odd ? T(0.5) : T(0);
  }
}

template <int RR, int TX, int TY, int WB = 16>
struct MF1Tile {
  static constexpr int CX = TX + 4, CY = TY + 4;                        // coarse u (tile + 2)
  static constexpr int FX = 2 * TX + 2 * RR - 1, FY = 2 * TY + 2 * RR - 1;   // s (R support)
  static constexpr int TXF = FX + 2, TYF = FY + 2;                      // t (+1 ring)
  static constexpr int A_WORDS = (CX * CY + TXF * CY) > FX * FY ? (CX * CY + TXF * CY) : FX * FY;
  static constexpr int B_WORDS = TXF * TYF > TX * FY ? TXF * TYF : TX * FY;
  static constexpr int SMEM = (A_WORDS + B_WORDS) * WB;
  static constexpr int NS = (FX * FY + 255) / 256;
};

// TC: tile arithmetic precision (double, or float for the c64 path: the
// stored-coefficient alternative carries fp32-rounded coefficients anyway);
// u, f, y are fp64 coarse vectors, the final f - A u is formed in fp64.
template <typename TSG, int KIND, int RR, int PR, int TX, int TY, typename TC = double>
__global__ void __launch_bounds__(256) k_galerkin1_mf(Geo gf, Geo gc, const cplx<TSG> *__restrict__ sig, double alpha,
                                                      double ih2, const double2 *__restrict__ u,
                                                      const double2 *__restrict__ f, double2 *__restrict__ y) {
  HMG_PDL_PROLOGUE();
  using T = TC;
  using V = cplx<TC>;
  using W = FineW<2, KIND>;
  using Tl = MF1Tile<RR, TX, TY, sizeof(V)>;
  constexpr int NT = 256, CX = Tl::CX, CY = Tl::CY, FX = Tl::FX, FY = Tl::FY, TXF = Tl::TXF, TYF = Tl::TYF;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V *smem = reinterpret_cast<V *>(smem_raw);
  V *su = smem;                  // [CY][CX]     phase 0-1
  V *sx = su + CX * CY;          // [CY][TXF]    phase 1-2  (P_x u)
  V *ss = smem;                  // [FY][FX]     phase 3-4  (aliases su, sx)
  V *st = smem + Tl::A_WORDS;    // [TYF][TXF]   phase 2-3
  V *sr = st;                    // [FY][TX]     phase 4-5  (R_x s, aliases st)
  const int X0 = blockIdx.x * TX, Y0 = blockIdx.y * TY;   // coarse-local tile origin
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const V zero = mkc<T>(0, 0);
  const int cx0 = X0 + gc.o[0] - 2, cy0 = Y0 + gc.o[1] - 2;                   // global coarse origin of su
  const int fx0 = 2 * (X0 + gc.o[0]) - RR, fy0 = 2 * (Y0 + gc.o[1]) - RR;   // global fine origin of ss
  // prefetch: f of this thread's output node, sigma of its s nodes
  const int ox = threadIdx.x, oy = threadIdx.y;
  const bool own = X0 + ox < gc.n[0] && Y0 + oy < gc.n[1];
  const int64_t io = own ? gc.idx(X0 + ox, Y0 + oy, 0) : 0;
  double2 fv = make_double2(0, 0);
  if (f && own) fv = f[io];
  cplx<TSG> sg[Tl::NS];
#pragma unroll
  for (int k = 0; k < Tl::NS; ++k) {
    const int i = tid + k * NT;
    const int fx = fx0 + i % FX, fy = fy0 + i / FX;
    sg[k] = mkc<TSG>(0, 0);
    if (i < FX * FY && fx >= 0 && fx < gf.N[0] && fy >= 0 && fy < gf.N[1])
      sg[k] = sig[gf.idx(fx - gf.o[0], fy - gf.o[1], 0)];
  }
  for (int i = tid; i < CX * CY; i += NT) {
    const int gx = cx0 + i % CX, gy = cy0 + i / CX;
    const bool in = gx >= 0 && gx < gc.N[0] && gy >= 0 && gy < gc.N[1];
    su[i] = in ? ccast<T, double>(u[gc.idx(gx - gc.o[0], gy - gc.o[1], 0)]) : zero;
  }
  __syncthreads();
  // phase 1: sx = P_x u on coarse rows, fine columns fx0-1 .. fx0+FX
  for (int i = tid; i < CY * TXF; i += NT) {
    const int r = i / TXF, lx = i % TXF;
    int c, d0;
    T w0, w1, w2;
    ptaps3<PR>(fx0 - 1 + lx, c, d0, w0, w1, w2);
    const V *row = su + r * CX + (c - cx0);
    V acc = cscale<T>(row[d0], w0);
    acc = cfmar<T>(acc, w1, row[0]);
    acc = cfmar<T>(acc, w2, row[1]);
    sx[i] = acc;
  }
  __syncthreads();
  // phase 2: t = P_y sx, zero outside the domain
  for (int i = tid; i < TYF * TXF; i += NT) {
    const int ly = i / TXF, lx = i % TXF;
    const int fx = fx0 - 1 + lx, fy = fy0 - 1 + ly;
    int c, d0;
    T w0, w1, w2;
    ptaps3<PR>(fy, c, d0, w0, w1, w2);
    const V *col = sx + (c - cy0) * TXF + lx;
    V acc = cscale<T>(col[d0 * TXF], w0);
    acc = cfmar<T>(acc, w1, col[0]);
    acc = cfmar<T>(acc, w2, col[TXF]);
    const bool in = fx >= 0 && fx < gf.N[0] && fy >= 0 && fy < gf.N[1];
    st[i] = in ? acc : zero;
  }
  __syncthreads();
  // phase 3: s = (L - sigma_s M) t (sigma = 0 outside the domain and t = 0 there: s = 0 only
  // if also L t = 0, so mask explicitly)
#pragma unroll
  for (int k = 0; k < Tl::NS; ++k) {
    const int i = tid + k * NT;
    if (i < FX * FY) {
      const int lx = i % FX, ly = i / FX;
      const int fx = fx0 + lx, fy = fy0 + ly;
      const V *c = st + (ly + 1) * TXF + (lx + 1);
      const V sf = cadd<T>(cadd<T>(c[-1], c[1]), cadd<T>(c[-TXF], c[TXF]));
      V Lx = cscale<T>(c[0], (T)W::Lc);
      Lx = cfmar<T>(Lx, (T)W::Lf, sf);
      if (W::Le != 0.0)
        Lx = cfmar<T>(Lx, (T)W::Le, cadd<T>(cadd<T>(c[-TXF - 1], c[-TXF + 1]), cadd<T>(c[TXF - 1], c[TXF + 1])));
      Lx = cscale<T>(Lx, (T)ih2);
      V Mx = cscale<T>(c[0], (T)W::Mc);
      if (W::Mf != 0.0) Mx = cfmar<T>(Mx, (T)W::Mf, sf);
      V sv = ccast<T, TSG>(sg[k]);
      sv.y = fma((T)-alpha, sv.x, sv.y);
      const bool in = fx >= 0 && fx < gf.N[0] && fy >= 0 && fy < gf.N[1];
      ss[i] = in ? csub<T>(Lx, cmul<T>(sv, Mx)) : zero;
    }
  }
  __syncthreads();
  // phase 4: sr = R_x s  (row ly, coarse column ox)
  for (int i = tid; i < FY * TX; i += NT) {
    const int ly = i / TX, c = i % TX;
    const V *row = ss + ly * FX + 2 * c;
    V acc = zero;
#pragma unroll
    for (int k = 0; k <= 2 * RR; ++k) acc = cfmar<T>(acc, (T)RW<RR>::w(k - RR), row[k]);
    sr[i] = acc;
  }
  __syncthreads();
  // phase 5: y = R_y sr
  if (own) {
    const V *col = sr + 2 * oy * TX + ox;
    V acc = zero;
#pragma unroll
    for (int k = 0; k <= 2 * RR; ++k) acc = cfmar<T>(acc, (T)RW<RR>::w(k - RR), col[k * TX]);
    const double2 ad = ccast<double, T>(acc);
    y[io] = f ? csub<double>(fv, ad) : ad;
  }
}

}  // namespace hmg
