// k_setup.cuh -- hierarchy setup kernels (fp64; not part of time-to-solve,
// P:1026-1027).  SURVEY §8(a) a1 (coefficients), a6 (Galerkin), a7
// (re-discretisation option), a8 (coarsest inverse), Vanka patch factors.
#pragma once
#include "common.cuh"
#include "k_operator.cuh"
#include "k_vanka.cuh"

namespace hmg {

// unpadded x-fastest (N) <-> padded box
template <typename A>
__global__ void k_pack(Geo g, const A *__restrict__ src, A *__restrict__ dst) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(g, ix, iy, iz);
  dst[g.idx(ix, iy, iz)] = src[((int64_t)iz * g.n[1] + iy) * g.n[0] + ix];
}
template <typename A>
__global__ void k_unpack(Geo g, const A *__restrict__ src, A *__restrict__ dst) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(g, ix, iy, iz);
  dst[((int64_t)iz * g.n[1] + iy) * g.n[0] + ix] = src[g.idx(ix, iy, iz)];
}

// padded box -> padded box with precision conversion (interior nodes)
template <typename TI, typename TO>
__global__ void k_pack_cvt(Geo g, const cplx<TI> *__restrict__ src, int src_padded, cplx<TO> *__restrict__ dst,
                           int dst_padded) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(g, ix, iy, iz);
  const int64_t c = ((int64_t)iz * g.n[1] + iy) * g.n[0] + ix;
  const int64_t p = g.idx(ix, iy, iz);
  const cplx<TI> v = src[src_padded ? p : c];
  dst[dst_padded ? p : c] = mkc<TO>((TO)v.x, (TO)v.y);
}

// a1: w2k2 = omega^2 kappa^2, gq = gamma/omega (Eq. 1.1); sig = (w2k2, -w2k2 gq) in T
template <typename T>
__global__ void k_sigma(Geo g, const double *__restrict__ kappa, const double *__restrict__ gamma, double omega,
                        double *__restrict__ w2k2, double *__restrict__ gq, cplx<T> *__restrict__ sig,
                        double2 *__restrict__ sigd) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(g, ix, iy, iz);
  const int64_t s = ((int64_t)iz * g.n[1] + iy) * g.n[0] + ix;
  const int64_t i = g.idx(ix, iy, iz);
  const double k = kappa[s];
  const double a = omega * omega * k * k;
  const double b = gamma[s] / omega;
  w2k2[i] = a;
  gq[i] = b;
  sig[i] = mkc<T>((T)a, (T)(-a * b));
  sigd[i] = make_double2(a, -a * b);
}

__host__ __device__ __forceinline__ int kidx(int ox, int oy, int oz, int r, int dim) {
  const int w = 2 * r + 1;
  return (ox + r) + w * ((oy + r) + (dim == 3 ? w * (oz + r) : 0));
}

// Shifted fine-type operator A = L - diag(sigma_s) M as a stored radius-1
// stencil (double), sigma_s = w2k2 (1 - i (gq + alpha)); zero towards
// out-of-domain nodes.  Used for level 0 (patch factors / Galerkin input) and
// for the REDISCRETIZE coarse levels at h_l.
template <int DIM, int KIND>
__global__ void k_materialize(Geo g, const double *__restrict__ w2k2, const double *__restrict__ gq, double alpha,
                              double ih2, double2 *__restrict__ coef) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(g, ix, iy, iz);
  using W = FineW<DIM, KIND>;
  const int64_t i = g.idx(ix, iy, iz);
  const double2 ss = make_double2(w2k2[i], -w2k2[i] * (gq[i] + alpha));
  const int ZR = DIM == 3 ? 1 : 0;
  for (int oz = -ZR; oz <= ZR; ++oz)
    for (int oy = -1; oy <= 1; ++oy)
      for (int ox = -1; ox <= 1; ++ox) {
        const int nnz = (ox != 0) + (oy != 0) + (oz != 0);
        double Lw = nnz == 0 ? W::Lc : nnz == 1 ? W::Lf : nnz == 2 ? W::Le : 0.0;
        double Mw = nnz == 0 ? W::Mc : nnz == 1 ? W::Mf : 0.0;
        double2 v = make_double2(Lw * ih2 - Mw * ss.x, -Mw * ss.y);
        if (!g.inside(ix + ox, iy + oy, iz + oz)) v = make_double2(0, 0);
        coef[(int64_t)kidx(ox, oy, oz, 1, DIM) * g.total + i] = v;
      }
}

struct TransferW {
  int rR, rP;       // radii of R and P kinds (1 = lin, 2 = cub)
  double wR[5], wP[5];  // 1D restriction weights at offsets -r..r
};

__host__ __device__ __forceinline__ int floordiv2(int a) { return a >= 0 ? a / 2 : -((-a + 1) / 2); }

// a6: Galerkin A_c = R A_f P for one coarse row per thread.
//   A_c[I, J] = sum_{i in supp R(I)} sum_{j} R[I,i] A_f[i,j] P[j,J],
//   R[I, 2I+k] = prod wR(k_a);  P[j, J] = 2^d prod wP(j_a - 2J_a)  (P = 2^d R_P^T).
// Out-of-domain fine/coarse nodes are skipped (truncated R and P, reading A5).
// Coarse and fine boxes may be windows of the global grid (partitioned setup,
// Geo::o): all index arithmetic below is in GLOBAL coordinates, converted to the
// local box only to address memory.
template <int DIM, int RC>
__global__ void k_galerkin(Geo gf, Geo gc, const double2 *__restrict__ cf, int rf, TransferW tw,
                           double2 *__restrict__ cc) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(gc, Xl, Yl, Zl);
  const int X = Xl + gc.o[0], Y = Yl + gc.o[1], Z = Zl + gc.o[2];   // global coarse node
  auto finside = [&](int x, int y, int z) {   // global fine node in the domain
    return x >= 0 && x < gf.N[0] && y >= 0 && y < gf.N[1] && z >= 0 && z < gf.N[2];
  };
  auto cinside = [&](int x, int y, int z) {
    return x >= 0 && x < gc.N[0] && y >= 0 && y < gc.N[1] && z >= 0 && z < gc.N[2];
  };
  constexpr int WC = 2 * RC + 1;
  constexpr int KC = DIM == 3 ? WC * WC * WC : WC * WC;
  double2 acc[KC];
  for (int k = 0; k < KC; ++k) acc[k] = make_double2(0, 0);
  const double pscale = DIM == 3 ? 8.0 : 4.0;
  const int kzr = DIM == 3 ? tw.rR : 0;
  const int ozr = DIM == 3 ? rf : 0;
  for (int kz = -kzr; kz <= kzr; ++kz)
    for (int ky = -tw.rR; ky <= tw.rR; ++ky)
      for (int kx = -tw.rR; kx <= tw.rR; ++kx) {
        const int ix = 2 * X + kx, iy = 2 * Y + ky, iz = DIM == 3 ? 2 * Z + kz : 0;
        if (!finside(ix, iy, iz)) continue;
        double wr = tw.wR[kx + tw.rR] * tw.wR[ky + tw.rR];
        if (DIM == 3) wr *= tw.wR[kz + tw.rR];
        const int64_t fi = gf.idx(ix - gf.o[0], iy - gf.o[1], iz - gf.o[2]);
        for (int oz = -ozr; oz <= ozr; ++oz)
          for (int oy = -rf; oy <= rf; ++oy)
            for (int ox = -rf; ox <= rf; ++ox) {
              const double2 a = cf[(int64_t)kidx(ox, oy, oz, rf, DIM) * gf.total + fi];
              if (a.x == 0.0 && a.y == 0.0) continue;
              const int jx = ix + ox, jy = iy + oy, jz = iz + oz;
              if (!finside(jx, jy, jz)) continue;
              const int jzlo = DIM == 3 ? -floordiv2(-(jz - tw.rP)) : 0;
              const int jzhi = DIM == 3 ? floordiv2(jz + tw.rP) : 0;
              const int jylo = -floordiv2(-(jy - tw.rP)), jyhi = floordiv2(jy + tw.rP);
              const int jxlo = -floordiv2(-(jx - tw.rP)), jxhi = floordiv2(jx + tw.rP);
              for (int Jz = jzlo; Jz <= jzhi; ++Jz)
                for (int Jy = jylo; Jy <= jyhi; ++Jy)
                  for (int Jx = jxlo; Jx <= jxhi; ++Jx) {
                    if (!cinside(Jx, Jy, Jz)) continue;
                    double wp = pscale * tw.wP[jx - 2 * Jx + tw.rP] * tw.wP[jy - 2 * Jy + tw.rP];
                    if (DIM == 3) wp *= tw.wP[jz - 2 * Jz + tw.rP];
                    const int dx = Jx - X, dy = Jy - Y, dz = Jz - Z;
                    if (dx < -RC || dx > RC || dy < -RC || dy > RC || dz < -RC || dz > RC) continue;  // unreachable
                    const double s = wr * wp;
                    double2 &t = acc[kidx(dx, dy, dz, RC, DIM)];
                    t.x = fma(s, a.x, t.x);
                    t.y = fma(s, a.y, t.y);
                  }
            }
      }
  const int64_t ci = gc.idx(Xl, Yl, Zl);
  for (int k = 0; k < KC; ++k) cc[(int64_t)k * gc.total + ci] = acc[k];
}

// a7 (REDISCRETIZE): full-weighting average of a per-node field, normalised
// by the in-domain weight sum (truncated lin R, reading A13).
static __global__ void k_fw_average(Geo gf, Geo gc, const double *__restrict__ ff, double *__restrict__ fc) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(gc, Xl, Yl, Zl);
  const int X = Xl + gc.o[0], Y = Yl + gc.o[1], Z = Zl + gc.o[2];   // global (windows: Geo::o)
  const double w1[3] = {0.25, 0.5, 0.25};
  const int zr = gc.dim == 3 ? 1 : 0;
  double s = 0, ws = 0;
  for (int kz = -zr; kz <= zr; ++kz)
    for (int ky = -1; ky <= 1; ++ky)
      for (int kx = -1; kx <= 1; ++kx) {
        const int ix = 2 * X + kx, iy = 2 * Y + ky, iz = gc.dim == 3 ? 2 * Z + kz : 0;
        if (ix < 0 || ix >= gf.N[0] || iy < 0 || iy >= gf.N[1] || iz < 0 || iz >= gf.N[2]) continue;
        double w = w1[kx + 1] * w1[ky + 1] * (gc.dim == 3 ? w1[kz + 1] : 1.0);
        s += w * ff[gf.idx(ix - gf.o[0], iy - gf.o[1], iz - gf.o[2])];
        ws += w;
      }
  fc[gc.idx(Xl, Yl, Zl)] = s / ws;
}

// cast a stored stencil (double) to the working precision
template <typename T>
__global__ void k_cast(const double2 *__restrict__ src, cplx<T> *__restrict__ dst, int64_t n) {
  HMG_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = mkc<T>((T)src[i].x, (T)src[i].y);
}

// stored stencil (T, padded) -> compact double [K][N] for hmg_copy_stencil
template <typename T>
__global__ void k_compact_stencil(Geo g, int K, const cplx<T> *__restrict__ src, double2 *__restrict__ dst) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(g, ix, iy, iz);
  const int64_t N = g.nodes();
  const int64_t s = ((int64_t)iz * g.n[1] + iy) * g.n[0] + ix;
  const int64_t i = g.idx(ix, iy, iz);
  for (int k = 0; k < K; ++k) {
    const cplx<T> v = src[(int64_t)k * g.total + i];
    dst[(int64_t)k * N + s] = make_double2((double)v.x, (double)v.y);
  }
}

// Small dense complex inverse by Gauss-Jordan with partial pivoting; returns
// false if a pivot is exactly zero or not finite.
template <int K>
__device__ bool small_inverse(double2 (&A)[K][K], double2 (&X)[K][K], int m) {
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b) X[a][b] = make_double2(a == b ? 1.0 : 0.0, 0.0);
  for (int k = 0; k < m; ++k) {
    int p = k;
    double best = cabs2<double>(A[k][k]);
    for (int i = k + 1; i < m; ++i) {
      const double v = cabs2<double>(A[i][k]);
      if (v > best) { best = v; p = i; }
    }
    if (!(best > 0.0) || !isfinite(best)) return false;
    if (p != k)
      for (int b = 0; b < m; ++b) {
        double2 t = A[k][b]; A[k][b] = A[p][b]; A[p][b] = t;
        t = X[k][b]; X[k][b] = X[p][b]; X[p][b] = t;
      }
    const double2 ip = crecip<double>(A[k][k]);
    for (int b = 0; b < m; ++b) {
      A[k][b] = cmul<double>(A[k][b], ip);
      X[k][b] = cmul<double>(X[k][b], ip);
    }
    for (int i = 0; i < m; ++i) {
      if (i == k) continue;
      const double2 f = A[i][k];
      if (f.x == 0.0 && f.y == 0.0) continue;
      for (int b = 0; b < m; ++b) {
        A[i][b] = csub<double>(A[i][b], cmul<double>(f, A[k][b]));
        X[i][b] = csub<double>(X[i][b], cmul<double>(f, X[k][b]));
      }
    }
  }
  return true;
}

// Patch inverses H_i^{-1} of the (clipped) patch matrices H_i = A[X_i, X_i]
// (Eq. 3.8; P:544 clipping; entries from the level's own operator, reading A8).
// Stored as hinv[a*K+b][anchor] in T; rows/columns of clipped members are 0.
template <typename T, int DIM, int KIND>
__global__ void k_patch_inverse(Geo g, const double2 *__restrict__ coef, int r, cplx<T> *__restrict__ hinv,
                                unsigned long long *__restrict__ err) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(g, ix, iy, iz);
  using P = Patch<DIM, KIND>;
  constexpr int K = P::K;
  if (!P::anchor(g, ix, iy, iz)) return;
  const int64_t c = g.idx(ix, iy, iz);
  int mem[K], ox[K], oy[K], oz[K];
  int m = 0;
  for (int s = 0; s < K; ++s) {
    int a, b, d;
    P::off(s, a, b, d);
    if (g.inside(ix + a, iy + b, iz + d)) { mem[m] = s; ox[m] = a; oy[m] = b; oz[m] = d; ++m; }
  }
  double2 A[K][K], X[K][K];
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b) {
      const int dx = ox[b] - ox[a], dy = oy[b] - oy[a], dz = oz[b] - oz[a];
      double2 v = make_double2(0, 0);
      if (dx >= -r && dx <= r && dy >= -r && dy <= r && dz >= -r && dz <= r)
        v = coef[(int64_t)kidx(dx, dy, dz, r, DIM) * g.total + c + g.delta(ox[a], oy[a], oz[a])];
      A[a][b] = v;
    }
  const bool ok = small_inverse<K>(A, X, m);
  if (!ok) {   // GLOBAL linear index of the anchor (windows / views: Geo::o)
    const unsigned long long lin =
        (unsigned long long)(((int64_t)(iz + g.o[2]) * g.N[1] + iy + g.o[1]) * g.N[0] + ix + g.o[0]);
    atomicMin(err, lin);
  }
  for (int a = 0; a < K; ++a)
    for (int b = 0; b < K; ++b) hinv[(int64_t)(a * K + b) * g.total + c] = mkc<T>(0, 0);
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b)
      hinv[(int64_t)(mem[a] * K + mem[b]) * g.total + c] = ok ? ccast<T, double>(X[a][b]) : mkc<T>(0, 0);
}

// Assemble the additive Vanka operator B (k_vanka.cuh, BStencil) from the fp64
// patch inverses: B[d][j] = (1/cnt_j) sum_{s,q: o_q - o_s = d} Hinv_{j - o_s}[s][q]
// (Eq. 3.8; non-anchor positions hold zero inverses).  fp64 sums, stored in T.
template <typename T, int DIM, int KIND>
__global__ void k_vanka_assemble(Geo g, const double2 *__restrict__ hinv, cplx<T> *__restrict__ B) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(g, ix, iy, iz);
  using P = Patch<DIM, KIND>;
  using S = BStencil<DIM, KIND>;
  constexpr int K = P::K;
  const int64_t j = g.idx(ix, iy, iz);
  const double ic = 1.0 / (double)P::count(g, ix, iy, iz);
  static_for<0, S::NB>([&](auto PI) {
    constexpr int p = decltype(PI)::value;
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int a = 0; a < K; ++a) {
#pragma unroll
      for (int b = 0; b < K; ++b) {
        int ax = 0, ay = 0, az = 0, bx = 0, by = 0, bz = 0;
        P::off(a, ax, ay, az);
        P::off(b, bx, by, bz);
        if (bx - ax != S::template dx<p> || by - ay != S::template dy<p> || bz - az != S::template dz<p>) continue;
        const double2 h = hinv[(int64_t)(a * K + b) * g.total + g.idx(ix - ax, iy - ay, iz - az)];
        acc.x += h.x;
        acc.y += h.y;
      }
    }
    B[(int64_t)p * g.total + j] = mkc<T>((T)(acc.x * ic), (T)(acc.y * ic));
  });
}

// a8: dense coarsest matrix (row-major, compact x-fastest indices)
static __global__ void k_dense_assemble(Geo g, const double2 *__restrict__ coef, int r, double2 *__restrict__ A) {
  HMG_PDL_PROLOGUE();
  HMG_NODE_IDX(g, ix, iy, iz);
  const int64_t N = g.nodes();
  const int64_t row = ((int64_t)iz * g.n[1] + iy) * g.n[0] + ix;
  const int64_t i = g.idx(ix, iy, iz);
  const int zr = g.dim == 3 ? r : 0;
  for (int oz = -zr; oz <= zr; ++oz)
    for (int oy = -r; oy <= r; ++oy)
      for (int ox = -r; ox <= r; ++ox) {
        if (!g.inside(ix + ox, iy + oy, iz + oz)) continue;
        const int64_t col = ((int64_t)(iz + oz) * g.n[1] + (iy + oy)) * g.n[0] + (ix + ox);
        A[row * N + col] = coef[(int64_t)kidx(ox, oy, oz, r, g.dim) * g.total + i];
      }
}

// Gauss-Jordan step k, part 1 (one block): partial pivot on column k, swap
// rows, scale the pivot row, save the elimination factors fcol[i] = A[i][k].
static __global__ void k_gj_pivot(int N, int k, double2 *__restrict__ A, double2 *__restrict__ Ai,
                           double2 *__restrict__ fcol, int *__restrict__ err) {
  HMG_PDL_PROLOGUE();
  __shared__ double sv[1024];
  __shared__ int si[1024];
  const int t = threadIdx.x;
  double best = -1.0;
  int bi = k;
  for (int i = k + t; i < N; i += blockDim.x) {
    const double v = cabs2<double>(A[(int64_t)i * N + k]);
    if (v > best) { best = v; bi = i; }
  }
  sv[t] = best;
  si[t] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (t < s) {
      if (sv[t + s] > sv[t] || (sv[t + s] == sv[t] && si[t + s] < si[t])) { sv[t] = sv[t + s]; si[t] = si[t + s]; }
    }
    __syncthreads();
  }
  const int p = si[0];
  if (!(sv[0] > 0.0) || !isfinite(sv[0])) {
    if (t == 0) *err = 1;
  }
  if (p != k)
    for (int b = t; b < N; b += blockDim.x) {
      double2 x = A[(int64_t)k * N + b]; A[(int64_t)k * N + b] = A[(int64_t)p * N + b]; A[(int64_t)p * N + b] = x;
      x = Ai[(int64_t)k * N + b]; Ai[(int64_t)k * N + b] = Ai[(int64_t)p * N + b]; Ai[(int64_t)p * N + b] = x;
    }
  __syncthreads();
  const double2 piv = A[(int64_t)k * N + k];
  const double2 ip = (piv.x == 0.0 && piv.y == 0.0) ? make_double2(0, 0) : crecip<double>(piv);
  __syncthreads();
  for (int b = t; b < N; b += blockDim.x) {
    A[(int64_t)k * N + b] = cmul<double>(A[(int64_t)k * N + b], ip);
    Ai[(int64_t)k * N + b] = cmul<double>(Ai[(int64_t)k * N + b], ip);
  }
  for (int i = t; i < N; i += blockDim.x) fcol[i] = i == k ? make_double2(0, 0) : A[(int64_t)i * N + k];
}

// Gauss-Jordan step k, part 2: eliminate column k from every other row.
static __global__ void k_gj_eliminate(int N, int k, double2 *__restrict__ A, double2 *__restrict__ Ai,
                               const double2 *__restrict__ fcol) {
  HMG_PDL_PROLOGUE();
  const int i = blockIdx.y;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == k || b >= N) return;
  const double2 f = fcol[i];
  if (f.x == 0.0 && f.y == 0.0) return;
  if (b >= k) A[(int64_t)i * N + b] = csub<double>(A[(int64_t)i * N + b], cmul<double>(f, A[(int64_t)k * N + b]));
  Ai[(int64_t)i * N + b] = csub<double>(Ai[(int64_t)i * N + b], cmul<double>(f, Ai[(int64_t)k * N + b]));
}

}  // namespace hmg
