// k_stage3d.cuh -- z-marching 3D stencil kernels with bulk-async (TMA engine)
// plane staging (SURVEY §8(a) a2/a3/a4 in 3D).
//
// The node-parallel gathers of k_fine_op / k_vanka_stencil issue 19 / 27
// global loads per node and were load-issue bound in 3D (ncu: SM 84 %,
// mio_throttle, DRAM 27-30 %).  Here a 256-thread block owns a TX x TY = 32 x 8
// column tile and marches through ZC planes.  Each plane's tile plus a one-node
// halo (x from x0-2 for 16-byte alignment) is copied global -> shared by
// cp.async.bulk row copies completing on an mbarrier (the copy engine, no
// register staging), NS planes ahead of the compute.  Each thread reads its 3x3
// in-plane neighbourhood once per plane from shared memory and keeps per-plane
// partial sums in registers; a node's stencil is assembled from the sums of
// planes z-1, z, z+1.  The partial sums are grouped exactly as the gather
// kernels group their terms, so the results are bit-identical to them
// (tests/test_gpu_stage3d.py).
#pragma once
#include <cstdint>

#include "common.cuh"
#include "k_operator.cuh"
#include "k_uniform.cuh"
#include "k_vanka.cuh"

namespace hmg {

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "HMG_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HMG_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int S3_TX = 32, S3_TY = 8, S3_RX = S3_TX + 4, S3_RY = S3_TY + 2;

// Per-plane staging plan shared by the kernels below: slot s of the ring holds
// NA arrays of plane z: array 0 = the halo tile (S3_RY rows x S3_RX elements of
// type E0, x from x0-2, y from y0-1), arrays 1.. = interior tiles (S3_TY rows x
// S3_TX elements, x from x0, y from y0) of per-node arrays (skipped rows leave
// stale data: their nodes never read it).  Warp 0 issues: lane 0 arms the
// barrier with the plane's byte count, then lane r copies row r.  Copies are
// clamped to the padded box [0, total) so a ragged tile never reads past the
// allocation (the clamped elements only feed nodes that are not written).
struct S3Plan {
  const char *src[4];   // base pointers (nullptr = array not staged)
  int esz[4];           // element bytes
  int na;
};

template <int NS>
__device__ __forceinline__ void s3_issue(const Geo &g, const S3Plan &pl, char *ring, int slot_bytes, const int *off,
                                         uint64_t *bar, int it, int z, int x0, int y0, unsigned skip1) {
  // skip1: bit r set = row r of array 1 is not needed (it lies in the uniform box)
  const int lane = threadIdx.x & 31;
  const int slot = it % NS;
  char *base = ring + (size_t)slot * slot_bytes;
  // row task for this lane: array a, row r
  unsigned bytes = 0;
  const char *src = nullptr;
  char *dst = nullptr;
  {
    int a = 0, r = lane;
    if (r >= S3_RY) {
      r -= S3_RY;
      a = 1 + r / S3_TY;
      r = r % S3_TY;
    }
    // (selects instead of indexing the plan arrays with the lane's runtime a: no local memory)
    const char *sa = a == 0 ? pl.src[0] : a == 1 ? pl.src[1] : a == 2 ? pl.src[2] : pl.src[3];
    const int es = a == 0 ? pl.esz[0] : a == 1 ? pl.esz[1] : a == 2 ? pl.esz[2] : pl.esz[3];
    const int oa = a == 0 ? off[0] : a == 1 ? off[1] : a == 2 ? off[2] : off[3];
    if (a < pl.na && sa && !(a == 1 && ((skip1 >> r) & 1u))) {
      const int xs = a == 0 ? x0 - 2 : x0, ys = a == 0 ? y0 - 1 + r : y0 + r;
      const int w = a == 0 ? S3_RX : S3_TX;
      const int64_t e0 = g.idx(xs, ys, z);
      int64_t n = w;
      if (e0 + n > g.total) n = g.total - e0;
      if (e0 >= 0 && n > 0) {
        bytes = (unsigned)(n * es) & ~15u;
        src = sa + e0 * es;
        dst = base + oa + (size_t)r * w * es;
      }
    }
  }
  unsigned tot = bytes;
#pragma unroll
  for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if (lane == 0) {
    fence_proxy_async();
    mbar_expect_tx(bar + slot, tot);
  }
  __syncwarp();
  if (bytes) bulk_g2s(dst, src, bytes, bar + slot);
}

// ---------------------------------------------------------------- 19/7-point operator
// y = A x or y = f - A x on the 3D fine level, A = L - diag(sigma_s) M
// (Eq. 2.3; FD2 P:101-102), the arithmetic of fine_op_node (TC),
// planes z0 .. z0+ZC-1 of the block's column tile.
template <typename T, int KIND, typename TC, typename TS, int ZC, int NS>
__global__ void __launch_bounds__(256) k_fine_op3d_z(Geo g, const cplx<TS> *__restrict__ sig, TC alpha, TC ih2,
                                                     const cplx<T> *__restrict__ x, const cplx<T> *__restrict__ f,
                                                     cplx<T> *__restrict__ y, UBox ub, cplx<TC> us) {
  using W = FineW<3, KIND>;
  using E = cplx<T>;
  using CC = cplx<TC>;
  extern __shared__ __align__(128) unsigned char s3_smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(s3_smem);
  char *ring = reinterpret_cast<char *>(s3_smem) + 128;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int x0 = blockIdx.x * S3_TX, y0 = blockIdx.y * S3_TY, z0 = blockIdx.z * ZC;
  const int zend = min(g.n[2], z0 + ZC);
  const int nplanes = zend - z0 + 2;   // planes z0-1 .. zend
  S3Plan pl;
  pl.na = f ? 3 : 2;
  pl.src[0] = reinterpret_cast<const char *>(x);
  pl.esz[0] = sizeof(E);
  pl.src[1] = reinterpret_cast<const char *>(sig);
  pl.esz[1] = sizeof(cplx<TS>);
  pl.src[2] = reinterpret_cast<const char *>(f);
  pl.esz[2] = sizeof(E);
  int off[4] = {0, 0, 0, 0};
  pl.src[3] = nullptr;
  pl.esz[3] = 0;
  off[1] = S3_RY * S3_RX * (int)sizeof(E);
  off[2] = off[1] + S3_TY * S3_TX * (int)sizeof(cplx<TS>);
  const int slot_bytes = (off[2] + (f ? S3_TY * S3_TX * (int)sizeof(E) : 0) + 127) / 128 * 128;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(bar + s, 1);
    mbar_fence_init();
  }
  __syncthreads();
  // sigma rows of the tile that lie entirely in the uniform box need no copy
  auto skip_rows = [&](int z) {
    unsigned m = 0;
    if (z >= ub.lo[2] && z < ub.hi[2] && x0 >= ub.lo[0] && min(x0 + S3_TX, g.n[0]) <= ub.hi[0])
      for (int r = 0; r < S3_TY; ++r)
        if (y0 + r >= ub.lo[1] && y0 + r < ub.hi[1]) m |= 1u << r;
    return m;
  };
  auto issue = [&](int it) {
    const int z = z0 - 1 + it;
    s3_issue<NS>(g, pl, ring, slot_bytes, off, bar, it, z, x0, y0, skip_rows(z));
  };
  if (tid < 32)
    for (int it = 0; it < NS && it < nplanes; ++it) issue(it);
  const int xi = x0 + tx, yi = y0 + ty;
  const bool own = xi < g.n[0] && yi < g.n[1];
  auto X = [&](const E *p) { return ccast<TC, T>(*p); };
  const CC zc = mkc<TC>(0, 0);
  // rolling per-plane partial sums: plane q-2 (A), q-1 (B)
  CC cA = zc, fxA = zc, fyA = zc, cB = zc, fxB = zc, fyB = zc, eB = zc;
  for (int it = 0; it < nplanes; ++it) {
    const int slot = it % NS;
    mbar_wait(bar + slot, (unsigned)(it / NS) & 1u);
    const char *sb = ring + (size_t)slot * slot_bytes;
    const E *P = reinterpret_cast<const E *>(sb) + (ty + 1) * S3_RX + (tx + 2);
    const CC c = X(P);
    const CC fx = cadd<TC>(X(P - 1), X(P + 1));
    const CC fy = cadd<TC>(X(P - S3_RX), X(P + S3_RX));
    CC e = zc;
    if (W::Le != 0.0)
      e = cadd<TC>(cadd<TC>(X(P - S3_RX - 1), X(P - S3_RX + 1)), cadd<TC>(X(P + S3_RX - 1), X(P + S3_RX + 1)));
    if (it >= 2 && own) {
      const int z = z0 - 2 + it;   // output plane = plane B
      // the grouping of fine_op_node: sf = (fx + fy) + (c(z-1) + c(z+1));
      // se = (e + (fx(z-1) + fx(z+1))) + (fy(z-1) + fy(z+1))
      const CC sf = cadd<TC>(cadd<TC>(fxB, fyB), cadd<TC>(cA, c));
      CC se = zc;
      if (W::Le != 0.0) se = cadd<TC>(cadd<TC>(eB, cadd<TC>(fxA, fx)), cadd<TC>(fyA, fy));
      CC Lx = cscale<TC>(cB, (TC)W::Lc);
      Lx = cfmar<TC>(Lx, (TC)W::Lf, sf);
      if (W::Le != 0.0) Lx = cfmar<TC>(Lx, (TC)W::Le, se);
      Lx = cscale<TC>(Lx, ih2);
      CC Mx = cscale<TC>(cB, (TC)W::Mc);
      if (W::Mf != 0.0) Mx = cfmar<TC>(Mx, (TC)W::Mf, sf);
      // sigma and f of plane B were staged one step earlier (slot it-1)
      const char *pb = ring + (size_t)((it - 1) % NS) * slot_bytes;
      const bool uni = ub.in(xi, yi, z);
      CC s = uni ? us : ccast<TC, TS>(reinterpret_cast<const cplx<TS> *>(pb + off[1])[ty * S3_TX + tx]);
      s.y = fma(-alpha, s.x, s.y);
      const CC Ax = csub<TC>(Lx, cmul<TC>(s, Mx));
      const int64_t i = g.idx(xi, yi, z);
      y[i] = ccast<T, TC>(f ? csub<TC>(ccast<TC, T>(reinterpret_cast<const E *>(pb + off[2])[ty * S3_TX + tx]), Ax)
                            : Ax);
    }
    cA = cB; fxA = fxB; fyA = fyB;
    cB = c; fxB = fx; fyB = fy; eB = e;
    __syncthreads();   // every thread is done with slot (it-1) % NS (sigma / f of plane B)
    // refill the slot consumed one step ago (its sigma / f were read just now)
    if (tid < 32 && it >= 1 && it - 1 + NS < nplanes) issue(it - 1 + NS);
  }
}

}  // namespace hmg
