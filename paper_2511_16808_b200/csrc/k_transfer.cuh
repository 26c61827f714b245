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

// u[i] += sum_J P[i, J] e[J]     (fine-node parallel)
template <int PR>
__device__ __forceinline__ int prolong_taps(int i, int *J, double *w) {
  // returns number of taps along one axis for fine coordinate i
  if ((i & 1) == 0) {
    const int c = i >> 1;
    if (PR == 2) {
      J[0] = c - 1; w[0] = 0.125;
      J[1] = c;     w[1] = 0.75;
      J[2] = c + 1; w[2] = 0.125;
      return 3;
    }
    J[0] = c; w[0] = 1.0;
    return 1;
  }
  const int c = (i - 1) >> 1;
  J[0] = c;     w[0] = 0.5;
  J[1] = c + 1; w[1] = 0.5;
  return 2;
}

// u_out = u + P e (u_out may equal u: each node reads and writes only itself)
template <typename TE, typename TU, int DIM, int PR>
__global__ void __launch_bounds__(256) k_prolong_add(Geo gf, Geo gc, const cplx<TE> *__restrict__ e,
                                                     const cplx<TU> *u, cplx<TU> *u_out) {
  using T = double;
  HMG_NODE_IDX(gf, ix, iy, iz);
  int Jx[3], Jy[3], Jz[3];
  double wx[3], wy[3], wz[3];
  // taps from GLOBAL fine coordinates (parity decides), then coarse-local indices
  const int nx = prolong_taps<PR>(ix + gf.o[0], Jx, wx);
  const int ny = prolong_taps<PR>(iy + gf.o[1], Jy, wy);
  int nz = 1;
  Jz[0] = 0; wz[0] = 1.0;
  if (DIM == 3) nz = prolong_taps<PR>(iz + gf.o[2], Jz, wz);
  for (int a = 0; a < nx; ++a) Jx[a] -= gc.o[0];
  for (int b = 0; b < ny; ++b) Jy[b] -= gc.o[1];
  if (DIM == 3)
    for (int c = 0; c < nz; ++c) Jz[c] -= gc.o[2];
  cplx<T> acc = mkc<T>(0, 0);
  for (int c = 0; c < nz; ++c) {
    cplx<T> accy = mkc<T>(0, 0);
    for (int b = 0; b < ny; ++b) {
      cplx<T> accx = mkc<T>(0, 0);
      const int64_t row = gc.base + (int64_t)Jz[c] * gc.pxy + (int64_t)Jy[b] * gc.px;
      for (int a = 0; a < nx; ++a) accx = cfmar<T>(accx, (T)wx[a], ccast<T, TE>(e[row + Jx[a]]));
      accy = cfmar<T>(accy, (T)wy[b], accx);
    }
    acc = cfmar<T>(acc, (T)wz[c], accy);
  }
  const int64_t i = gf.idx(ix, iy, iz);
  u_out[i] = ccast<TU, T>(cadd<T>(ccast<T, TU>(u[i]), acc));
}

// Same operation, coarse-node parallel: the thread of coarse node J writes
// the 2^d fine nodes 2J + {0,1}^d (global parity), loading its 3^d coarse
// neighbourhood once (instead of up to 3^d loads per fine node).  Fine nodes
// outside this rank's rows / the domain are skipped.  u_out may equal u.
template <typename TE, typename TU, int DIM, int PR>
__global__ void __launch_bounds__(256) k_prolong_block(Geo gf, Geo gc, int cx0, int cy0, int cz0, int ncx, int ncy,
                                                       int ncz, const cplx<TE> *__restrict__ e, const cplx<TU> *u,
                                                       cplx<TU> *u_out) {
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

}  // namespace hmg
