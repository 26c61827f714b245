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
#include <cuda.h>

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
// one TMA tensor request: the box of `map` at element coordinates (c0, c1, c2) -> shared
// memory (out-of-range parts are zero-filled); completes on `bar` with the box's bytes
__device__ __forceinline__ void tma_load3(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

constexpr int S3_TX = 32, S3_TY = 8, S3_RX = S3_TX + 4, S3_RY = S3_TY + 2;

// Shared-memory layout of the staged kernels: NS full + NS empty mbarriers
// (128 bytes), then NS ring slots.  Block = 8 compute warps (32 x 8 nodes of a
// plane) + 1 producer warp (threadIdx.y == 8) whose lane 0 issues ONE TMA
// tensor request per staged array and plane (tensor maps over the padded level
// boxes, built on the host: make_tmap): the compute warps never meet at a block
// barrier inside the march; a slot is refilled once all 8 compute warps have
// arrived on its empty barrier.  (Row-by-row cp.async.bulk copies, 10-26
// requests per plane, were measured request-rate bound.)
constexpr int S3_THREADS = 32 * 9;

template <int NS>
__device__ __forceinline__ void s3_init(uint64_t *full, uint64_t *empty) {
  if (threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, S3_TY);
    }
    mbar_fence_init();
  }
  __syncthreads();
}
// consumer side: one arrival per compute warp on the slot's empty barrier
__device__ __forceinline__ void s3_release(uint64_t *empty_slot) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty_slot)) : "memory");
}
// producer side (one lane): for every plane, wait until its slot is free, arm the
// full barrier with the plane's bytes and issue the requests (issue(it, slot, z))
template <int NS, typename Issue>
__device__ __forceinline__ void s3_produce(uint64_t *full, uint64_t *empty, int nplanes, int z0, Issue issue) {
  for (int it = 0; it < nplanes; ++it) {
    const int slot = it % NS;
    if (it >= NS) mbar_wait(empty + slot, (unsigned)((it / NS) + 1) & 1u);   // its previous use is consumed
    issue(it, slot, z0 - 1 + it);
  }
}

// ---------------------------------------------------------------- 19/7-point operator
// y = A x or y = f - A x on the 3D fine level, A = L - diag(sigma_s) M
// (Eq. 2.3; FD2 P:101-102), the arithmetic of fine_op_node (TC),
// planes z0 .. z0+ZC-1 of the block's column tile.  mx: tensor map of x with box
// S3_RX x S3_RY x 1 (halo tile); ms / mf: sigma / f with box S3_TX x S3_TY x 1.
template <typename T, int KIND, typename TC, typename TS, int ZC, int NS>
__global__ void __launch_bounds__(S3_THREADS) k_fine_op3d_z(Geo g, const __grid_constant__ CUtensorMap mx,
                                                            const __grid_constant__ CUtensorMap ms,
                                                            const __grid_constant__ CUtensorMap mf, int has_f,
                                                            TC alpha, TC ih2, cplx<T> *__restrict__ y, UBox ub,
                                                            cplx<TC> us) {
  HMG_PDL_PROLOGUE();
  using W = FineW<3, KIND>;
  using E = cplx<T>;
  using CC = cplx<TC>;
  using ES = cplx<TS>;
  extern __shared__ __align__(128) unsigned char s3_smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(s3_smem), *empty = full + NS;
  char *ring = reinterpret_cast<char *>(s3_smem) + 128;
  constexpr int BX = S3_RY * S3_RX * (int)sizeof(E), BS = S3_TY * S3_TX * (int)sizeof(ES),
                BF = S3_TY * S3_TX * (int)sizeof(E);
  constexpr int OFF_S = (BX + 127) / 128 * 128, OFF_F = OFF_S + (BS + 127) / 128 * 128;
  constexpr int SLOT = OFF_F + (BF + 127) / 128 * 128;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x0 = blockIdx.x * S3_TX, y0 = blockIdx.y * S3_TY, z0 = blockIdx.z * ZC;
  const int zend = min(g.n[2], z0 + ZC);
  const int nplanes = zend - z0 + 2;   // planes z0-1 .. zend
  s3_init<NS>(full, empty);
  if (ty == S3_TY) {   // producer warp
    if (tx == 0) {
      const int G = g.G, wx = (int)sizeof(E) / 8, ws = (int)sizeof(ES) / 8;
      // sigma is not staged for a tile-plane inside the uniform box
      const bool xyu = x0 >= ub.lo[0] && min(x0 + S3_TX, g.n[0]) <= ub.hi[0] && y0 >= ub.lo[1] &&
                       min(y0 + S3_TY, g.n[1]) <= ub.hi[1];
      s3_produce<NS>(full, empty, nplanes, z0, [&](int, int slot, int z) {
        const bool su = xyu && z >= ub.lo[2] && z < ub.hi[2];
        char *b = ring + (size_t)slot * SLOT;
        mbar_expect_tx(full + slot, BX + (su ? 0 : BS) + (has_f ? BF : 0));
        tma_load3(b, &mx, (G + x0 - 2) * wx, G + y0 - 1, G + z, full + slot);
        if (!su) tma_load3(b + OFF_S, &ms, (G + x0) * ws, G + y0, G + z, full + slot);
        if (has_f) tma_load3(b + OFF_F, &mf, (G + x0) * wx, G + y0, G + z, full + slot);
      });
    }
    return;
  }
  const int xi = x0 + tx, yi = y0 + ty;
  const bool own = xi < g.n[0] && yi < g.n[1];
  auto X = [&](const E *p) { return ccast<TC, T>(*p); };
  const CC zc = mkc<TC>(0, 0);
  // rolling per-plane partial sums: plane q-2 (A), q-1 (B)
  CC cA = zc, fxA = zc, fyA = zc, cB = zc, fxB = zc, fyB = zc, eB = zc;
  for (int it = 0; it < nplanes; ++it) {
    const int slot = it % NS;
    mbar_wait(full + slot, (unsigned)(it / NS) & 1u);
    const char *sb = ring + (size_t)slot * SLOT;
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
      // sigma and f of plane B were staged with it (slot it-1)
      const char *pb = ring + (size_t)((it - 1) % NS) * SLOT;
      const bool uni = ub.in(xi, yi, z);
      CC s = uni ? us : ccast<TC, TS>(reinterpret_cast<const ES *>(pb + OFF_S)[ty * S3_TX + tx]);
      s.y = fma(-alpha, s.x, s.y);
      const CC Ax = csub<TC>(Lx, cmul<TC>(s, Mx));
      const int64_t i = g.idx(xi, yi, z);
      y[i] = ccast<T, TC>(has_f ? csub<TC>(ccast<TC, T>(reinterpret_cast<const E *>(pb + OFF_F)[ty * S3_TX + tx]), Ax)
                                : Ax);
    }
    cA = cB; fxA = fxB; fyA = fyB;
    cB = c; fxB = fx; fyB = fy; eB = e;
    if (it >= 1) s3_release(empty + (it - 1) % NS);   // slot it-1: x read at it-1, sigma / f just now
  }
}

// ---------------------------------------------------------------- 27-point additive Vanka operator
// u_out = u + w B r (zero: u_out = w B r) with the assembled 3D element operator B
// (Eq. 3.8, 27 offsets, k_vanka_assemble), r staged plane by plane (mr: box
// S3_RX x S3_RY x 1).  At plane p a thread adds the dz = +1 terms to output p-1
// (which completes it), the dz = 0 terms to output p and the dz = -1 terms to
// output p+1: each output receives its terms in the offset order of
// k_vanka_stencil (dz, dy, dx ascending) -- the same arithmetic.  B comes from the
// uniform-box copy inside the box, else from its stored planes at the output node.
template <typename TV, typename TK, int ZC, int NS>
__global__ void __launch_bounds__(S3_THREADS) k_vanka27_z(Geo g, const __grid_constant__ CUtensorMap mr,
                                                          const cplx<TK> *__restrict__ B, const cplx<TV> *u,
                                                          cplx<TV> *u_out, TV w, int zero, UBox ub,
                                                          UCoef<27, TV> uc) {
  HMG_PDL_PROLOGUE();
  using E = cplx<TV>;
  extern __shared__ __align__(128) unsigned char s3_smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(s3_smem), *empty = full + NS;
  char *ring = reinterpret_cast<char *>(s3_smem) + 128;
  constexpr int BX = S3_RY * S3_RX * (int)sizeof(E), SLOT = (BX + 127) / 128 * 128;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x0 = blockIdx.x * S3_TX, y0 = blockIdx.y * S3_TY, z0 = blockIdx.z * ZC;
  const int zend = min(g.n[2], z0 + ZC);
  const int nplanes = zend - z0 + 2;   // r planes z0-1 .. zend
  s3_init<NS>(full, empty);
  if (ty == S3_TY) {
    if (tx == 0) {
      const int G = g.G, wx = (int)sizeof(E) / 8;
      s3_produce<NS>(full, empty, nplanes, z0, [&](int, int slot, int z) {
        mbar_expect_tx(full + slot, BX);
        tma_load3(ring + (size_t)slot * SLOT, &mr, (G + x0 - 2) * wx, G + y0 - 1, G + z, full + slot);
      });
    }
    return;
  }
  const int xi = x0 + tx, yi = y0 + ty;
  const bool own = xi < g.n[0] && yi < g.n[1];
  const E zc = mkc<TV>(0, 0);
  E aM = zc, a0 = zc;   // partial sums of outputs p-1 and p (before plane p)
  for (int it = 0; it < nplanes; ++it) {
    const int p = z0 - 1 + it;   // plane of r in the slot
    const int slot = it % NS;
    mbar_wait(full + slot, (unsigned)(it / NS) & 1u);
    const E *P = reinterpret_cast<const E *>(ring + (size_t)slot * SLOT) + (ty + 1) * S3_RX + (tx + 2);
    E rv[9];
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) rv[(dy + 1) * 3 + dx + 1] = P[dy * S3_RX + dx];
    s3_release(empty + slot);   // r of this plane is in registers
    E aP = zc;
    if (own) {
      // output node of plane q gets B(q; dx, dy, dz) r(x + dx, y + dy, p), dz = p - q
      auto add = [&](E &acc, int q, int dz, auto uni) {
        if (q < z0 || q >= zend) return;
        const int64_t iq = g.idx(xi, yi, q);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          const int pidx = (dz + 1) * 9 + k;
          const E b = decltype(uni)::value ? uc.c[pidx] : ccast<TV, TK>(B[(int64_t)pidx * g.total + iq]);
          acc = cfma<TV>(acc, b, rv[k]);
        }
      };
      using YES = std::integral_constant<bool, true>;
      using NO = std::integral_constant<bool, false>;
      // dz = +1 completes output p-1, dz = 0 continues p, dz = -1 opens p+1
      if (ub.in(xi, yi, p - 1)) add(aM, p - 1, 1, YES{}); else add(aM, p - 1, 1, NO{});
      if (ub.in(xi, yi, p)) add(a0, p, 0, YES{}); else add(a0, p, 0, NO{});
      if (ub.in(xi, yi, p + 1)) add(aP, p + 1, -1, YES{}); else add(aP, p + 1, -1, NO{});
      const int q = p - 1;
      if (q >= z0 && q < zend) {
        const int64_t iq = g.idx(xi, yi, q);
        E o;
        if (zero) {
          o = mkc<TV>(__fmul_rn_t(aM.x, w), __fmul_rn_t(aM.y, w));
        } else {
          const E uq = u[iq];
          o = mkc<TV>(fma(aM.x, w, uq.x), fma(aM.y, w, uq.y));
        }
        u_out[iq] = o;
      }
    }
    aM = a0;
    a0 = aP;
  }
}

}  // namespace hmg
