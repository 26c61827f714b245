// k_tail.cuh -- the small coarse levels of the V-cycle in ONE persistent kernel
// (DESIGN.md §5.2).  Levels below a few hundred thousand nodes are launch- and
// latency-bound: at N = 4096 the levels >= 2 took 0.32 ms of a 1.19 ms V-cycle in
// graph mode although they move a few MB.  k_coarse_tail runs the V(1,1) recursion
// (Alg. 2.1) of levels l0 .. L-1 -- zero-guess pre-smoothing, residual,
// restriction down; coarsest dense solve; prolongation, residual, smoothing up --
// as grid-stride passes separated by a software grid barrier (all blocks
// co-resident: the grid is sized by the occupancy API), one launch per cycle.
// Every pass applies the per-node arithmetic of the standalone kernels
// (k_stored_op, k_vanka_stencil, k_restrict, k_prolong_block, k_coarse_gemv), so
// the result is bit-identical (tests/test_gpu_tail.py).
#pragma once
#include "common.cuh"
#include "k_krylov.cuh"
#include "k_operator.cuh"
#include "k_transfer.cuh"
#include "k_uniform.cuh"
#include "k_vanka.cuh"

namespace hmg {

struct TailLevel {
  Geo geo;
  int r;                     // stored stencil radius
  int rR, rP;                // transfer radii to the next level
  double w;                  // damping
  const void *coef;          // stored stencil planes (TK)
  const void *bop;           // assembled Vanka operator planes (TK)
  const unsigned short *ccls, *bcls;   // coefficient dictionaries (k_dict.cuh; null: the planes)
  const void *ctab, *btab;             // their class tables [class][k] (TK)
  UBox ub;                   // uniform box
  const double2 *ucoef;      // its stencil / operator copies (device, fp64)
  const double2 *ubop;
  double2 *u, *f, *r_;       // level vectors (fp64)
};

// software grid barrier: bar[0] = arrival count, bar[1] = generation
__device__ __forceinline__ void tail_sync(unsigned *bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *gen = bar + 1;
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// cluster variant: the whole tail runs as ONE thread-block cluster (gridDim = cluster size), so
// the passes are separated by the hardware cluster barrier (release / acquire at cluster
// scope orders the global-memory writes of one pass before the reads of the next) instead of
// atomics on a global word -- a few hundred ns per pass instead of microseconds
__device__ __forceinline__ void tail_sync_cluster() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <bool CLUSTER>
__device__ __forceinline__ void tail_barrier(unsigned *bar, unsigned nblocks) {
  if constexpr (CLUSTER) tail_sync_cluster();
  else tail_sync(bar, nblocks);
}

template <typename F>
__device__ __forceinline__ void tail_nodes(const Geo &g, F &&fn) {
  const int64_t n = g.nodes();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int ix = (int)(t % g.n[0]);
    const int64_t q = t / g.n[0];
    const int iy = (int)(q % g.n[1]);
    const int iz = (int)(q / g.n[1]);
    fn(ix, iy, iz);
  }
}

// y = f - A x (f != null) / y = A x at node (ix, iy, iz): k_stored_op's arithmetic (NR = 1)
template <typename TK, int DIM, int R>
__device__ __forceinline__ void tail_stored_node(const TailLevel &L, const double2 *x, const double2 *f, double2 *y,
                                                 int ix, int iy, int iz) {
  using T = double;
  const Geo &g = L.geo;
  const int64_t i = g.idx(ix, iy, iz);
  const bool uni = L.ub.in(ix, iy, iz);
  constexpr int ZR = DIM == 3 ? R : 0;
  constexpr int KP = (2 * R + 1) * (2 * R + 1) * (2 * ZR + 1);
  // stored planes (stride total) or the node's dictionary entry (stride 1): one load path
  const cplx<TK> *coef = L.ccls ? reinterpret_cast<const cplx<TK> *>(L.ctab) + (int64_t)L.ccls[i] * KP
                                : reinterpret_cast<const cplx<TK> *>(L.coef) + i;
  const int64_t cs = L.ccls ? 1 : g.total;
  cplx<T> acc = mkc<T>(0, 0);
  // two copies of the unrolled loop behind one branch, not a per-coefficient select
  auto run = [&](auto ck) {
    int k = 0;
#pragma unroll
    for (int oz = -ZR; oz <= ZR; ++oz)
#pragma unroll
      for (int oy = -R; oy <= R; ++oy)
#pragma unroll
        for (int ox = -R; ox <= R; ++ox, ++k) acc = cfma<T>(acc, ck(k), x[i + g.delta(ox, oy, oz)]);
  };
  if (uni) run([&](int k) { return L.ucoef[k]; });
  else run([&](int k) { return ccast<T, TK>(coef[(int64_t)k * cs]); });
  y[i] = f ? csub<T>(f[i], acc) : acc;
}

// u_out = u + w B r (zero: w B r): k_vanka_stencil's arithmetic (NR = 1)
template <typename TK, int DIM, int KIND>
__device__ __forceinline__ void tail_vanka_node(const TailLevel &L, const double2 *r, const double2 *u,
                                                double2 *u_out, int zero, int ix, int iy, int iz) {
  using T = double;
  using S = BStencil<DIM, KIND>;
  const Geo &g = L.geo;
  const int64_t j = g.idx(ix, iy, iz);
  const bool uni = L.ub.in(ix, iy, iz);
  const cplx<TK> *B = L.bcls ? reinterpret_cast<const cplx<TK> *>(L.btab) + (int64_t)L.bcls[j] * S::NB
                             : reinterpret_cast<const cplx<TK> *>(L.bop) + j;
  const int64_t bs = L.bcls ? 1 : g.total;
  cplx<T> acc = mkc<T>(0, 0);
  auto run = [&](auto bk) {
    static_for<0, S::NB>([&](auto P) {
      constexpr int p = decltype(P)::value;
      acc = cfma<T>(acc, bk(p), r[j + g.delta(S::template dx<p>, S::template dy<p>, S::template dz<p>)]);
    });
  };
  if (uni) run([&](int p) { return L.ubop[p]; });
  else run([&](int p) { return ccast<T, TK>(B[(int64_t)p * bs]); });
  const T w = L.w;
  cplx<T> o;
  if (zero) {
    o = mkc<T>(__fmul_rn_t(acc.x, w), __fmul_rn_t(acc.y, w));
  } else {
    const cplx<T> uq = u[j];
    o = mkc<T>(fma(acc.x, w, uq.x), fma(acc.y, w, uq.y));
  }
  u_out[j] = o;
}

// fc[I] = R r (coarse node (X, Y, Z)): k_restrict's arithmetic (one rank: no offsets)
template <int DIM, int RR>
__device__ __forceinline__ void tail_restrict_node(const Geo &gf, const Geo &gc, const double2 *r, double2 *fc,
                                                   int X, int Y, int Z) {
  using T = double;
  const int64_t ic = gc.idx(X, Y, Z);
  const int64_t jf = gf.idx(2 * X, 2 * Y, DIM == 3 ? 2 * Z : 0);
  constexpr int ZR = DIM == 3 ? RR : 0;
  cplx<T> acc = mkc<T>(0, 0);
#pragma unroll
  for (int kz = -ZR; kz <= ZR; ++kz) {
    cplx<T> accy = mkc<T>(0, 0);
#pragma unroll
    for (int ky = -RR; ky <= RR; ++ky) {
      cplx<T> accx = mkc<T>(0, 0);
#pragma unroll
      for (int kx = -RR; kx <= RR; ++kx) accx = cfmar<T>(accx, (T)RW<RR>::w(kx), r[jf + gf.delta(kx, ky, kz)]);
      accy = cfmar<T>(accy, (T)RW<RR>::w(ky), accx);
    }
    acc = DIM == 3 ? cfmar<T>(acc, (T)RW<RR>::w(kz), accy) : accy;
  }
  fc[ic] = acc;
}

// u += P e for the fine children of coarse node (X, Y, Z): k_prolong_block's arithmetic
template <int DIM, int PR>
__device__ __forceinline__ void tail_prolong_node(const Geo &gf, const Geo &gc, const double2 *e, double2 *u, int X,
                                                  int Y, int Z) {
  using T = double;
  constexpr int ZW = DIM == 3 ? 3 : 1;
  cplx<T> c[ZW][3][3];
#pragma unroll
  for (int dz = 0; dz < ZW; ++dz)
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx)
        c[dz][dy][dx] = e[gc.idx(X - 1 + dx, Y - 1 + dy, DIM == 3 ? Z - 1 + dz : 0)];
  auto wt = [](int p, int k) -> double {
    if (p == 0) return PR == 2 ? (k == 1 ? 0.75 : 0.125) : (k == 1 ? 1.0 : 0.0);
    return k == 0 ? 0.0 : 0.5;
  };
#pragma unroll
  for (int pz = 0; pz < (DIM == 3 ? 2 : 1); ++pz)
#pragma unroll
    for (int py = 0; py < 2; ++py)
#pragma unroll
      for (int px = 0; px < 2; ++px) {
        const int fx = 2 * X + px, fy = 2 * Y + py, fz = DIM == 3 ? 2 * Z + pz : 0;
        if (fx >= gf.n[0] || fy >= gf.n[1] || (DIM == 3 && fz >= gf.n[2])) continue;
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
        u[i] = cadd<T>(u[i], acc);
      }
}

template <typename TK, int DIM, int KIND>
__device__ void tail_stored_pass(const TailLevel &L, const double2 *x, const double2 *f, double2 *y) {
  if (L.r == 1) tail_nodes(L.geo, [&](int a, int b, int c) { tail_stored_node<TK, DIM, 1>(L, x, f, y, a, b, c); });
  else tail_nodes(L.geo, [&](int a, int b, int c) { tail_stored_node<TK, DIM, 2>(L, x, f, y, a, b, c); });
}

// V(1,1) on levels l0 .. L-1 (zero initial guess on l0; lv[l0].f holds the right-hand side)
template <typename TK, int DIM, int KIND, int MINB = 1, int NT = 256, bool CLUSTER = false>
__global__ void __launch_bounds__(NT, MINB) k_coarse_tail(const TailLevel *__restrict__ lv, int l0, int L,
                                                     const double2 *__restrict__ ainv, unsigned *bar) {
  HMG_PDL_PROLOGUE();
  const unsigned nb = gridDim.x;
  for (int l = l0; l < L - 1; ++l) {
    const TailLevel &A = lv[l], &B = lv[l + 1];
    // zero-guess pre-smoothing u = w B f
    tail_nodes(A.geo, [&](int a, int b, int c) { tail_vanka_node<TK, DIM, KIND>(A, A.f, nullptr, A.u, 1, a, b, c); });
    tail_barrier<CLUSTER>(bar, nb);
    tail_stored_pass<TK, DIM, KIND>(A, A.u, A.f, A.r_);   // r = f - A u
    tail_barrier<CLUSTER>(bar, nb);
    if (A.rR == 1) tail_nodes(B.geo, [&](int a, int b, int c) { tail_restrict_node<DIM, 1>(A.geo, B.geo, A.r_, B.f, a, b, c); });
    else tail_nodes(B.geo, [&](int a, int b, int c) { tail_restrict_node<DIM, 2>(A.geo, B.geo, A.r_, B.f, a, b, c); });
    tail_barrier<CLUSTER>(bar, nb);
  }
  {   // coarsest: e = A_L^{-1} f, one warp per row (k_coarse_gemv's lane order and warp sum)
    const TailLevel &C = lv[L - 1];
    const Geo &g = C.geo;
    const int N = (int)g.nodes();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < N; row += warps) {
      double ax = 0, ay = 0;
      for (int col = lane; col < N; col += 32) {
        const int cx = col % g.n[0], cy = (col / g.n[0]) % g.n[1], cz = col / (g.n[0] * g.n[1]);
        const double2 a = ainv[row * N + col];
        const double2 v = C.f[g.idx(cx, cy, cz)];
        ax = fma(a.x, v.x, fma(-a.y, v.y, ax));
        ay = fma(a.x, v.y, fma(a.y, v.x, ay));
      }
      const double sx = warp_sum(ax), sy = warp_sum(ay);
      if (lane == 0) {
        const int rx = (int)(row % g.n[0]), ry = (int)((row / g.n[0]) % g.n[1]), rz = (int)(row / ((int64_t)g.n[0] * g.n[1]));
        C.u[g.idx(rx, ry, rz)] = make_double2(sx, sy);
      }
    }
    tail_barrier<CLUSTER>(bar, nb);
  }
  for (int l = L - 2; l >= l0; --l) {
    const TailLevel &A = lv[l], &B = lv[l + 1];
    if (A.rP == 1) tail_nodes(B.geo, [&](int a, int b, int c) { tail_prolong_node<DIM, 1>(A.geo, B.geo, B.u, A.u, a, b, c); });
    else tail_nodes(B.geo, [&](int a, int b, int c) { tail_prolong_node<DIM, 2>(A.geo, B.geo, B.u, A.u, a, b, c); });
    tail_barrier<CLUSTER>(bar, nb);
    tail_stored_pass<TK, DIM, KIND>(A, A.u, A.f, A.r_);   // post-smoothing: r = f - A u
    tail_barrier<CLUSTER>(bar, nb);
    tail_nodes(A.geo, [&](int a, int b, int c) { tail_vanka_node<TK, DIM, KIND>(A, A.r_, A.u, A.u, 0, a, b, c); });
    if (l > l0) tail_barrier<CLUSTER>(bar, nb);
  }
}

// the cluster instantiations live in their own translation unit (tail_cluster.cu): the kernel
// of the given storage precision / dimension / patch kind, launched with TAIL_CL_NT threads per
// block and gridDim = cluster size (null: not instantiated)
constexpr int TAIL_CL_NT = 512;
void *tail_cluster_fn(bool fp64_storage, int dim, int kind);

}  // namespace hmg
