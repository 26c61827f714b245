// k_dict.cuh -- coefficient dictionary: the uniform box
// generalised to the sponge.
//
// In the sponge of a homogeneous medium (configs 0, 1, 3 and the paper's Table
// 5.2 / 5.4 experiments) a node's coefficients -- the Galerkin
// stencil A_l = R A P or the assembled additive Vanka operator B_l
// (Eq. 3.8) -- depend only on the gamma profile in its neighbourhood, i.e. on
// its distances to the nearest faces, so the nodes outside the uniform box
// carry only a few thousand DISTINCT coefficient vectors.  Setup hashes every
// node's vector (64-bit, over the raw bits), inserts the hashes into an
// open-addressing table, numbers the distinct ones densely, copies one
// representative vector per class into a table tab[class][k] and VERIFIES bit
// for bit that every node's stored vector equals its class's entry.  The
// kernels then read a 2-byte class index per node and the coefficients from
// the (L1/L2-resident) table instead of K coefficient planes.  Same values,
// same arithmetic order: bit-identical to the stored path.  Heterogeneous
// media (every node distinct: more than 65535 classes) keep the planes.
#pragma once
#include "common.cuh"

namespace hmg {

constexpr unsigned long long kDictEmpty = 0ull;
constexpr int kDictMaxProbe = 256;

__device__ __forceinline__ unsigned long long dict_mix(unsigned long long h, unsigned long long v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h ^= h >> 31;
  h *= 0xbf58476d1ce4e5b9ull;
  h ^= h >> 29;
  return h;
}

// slot[node] = table slot of the node's coefficient vector (nplanes elements of
// W 8-byte words at stride total).  keys has mask + 1 entries (a power of two),
// zero = empty; flag[1] counts the distinct vectors inserted.  flag[0] is set --
// and every thread stops early -- when a probe sequence exceeds kDictMaxProbe
// or more than maxcls distinct vectors appear (a heterogeneous medium).
static __global__ void k_dict_insert(Geo g, const unsigned long long *__restrict__ planes, int nplanes, int W,
                              unsigned long long *keys, unsigned mask, int *__restrict__ slot, int *flag,
                              int maxcls) {
  HMG_NODE_IDX(g, ix, iy, iz);
  volatile int *stop = flag;
  if (*stop) return;
  const int64_t j = g.idx(ix, iy, iz);
  const int64_t f = ((int64_t)iz * g.n[1] + iy) * g.n[0] + ix;
  unsigned long long h = 0x243f6a8885a308d3ull;
  for (int k = 0; k < nplanes; ++k)
    for (int w = 0; w < W; ++w) h = dict_mix(h, planes[((int64_t)k * g.total + j) * W + w]);
  if (h == kDictEmpty) h = 1;
  unsigned s = (unsigned)(h ^ (h >> 32)) & mask;
  for (int p = 0; p < kDictMaxProbe && !*stop; ++p) {
    const unsigned long long prev = atomicCAS(keys + s, kDictEmpty, h);
    if (prev == kDictEmpty || prev == h) {
      slot[f] = (int)s;
      if (prev == kDictEmpty && atomicAdd(flag + 1, 1) >= maxcls) atomicExch(flag, 1);
      return;
    }
    s = (s + 1) & mask;
  }
  atomicExch(flag, 1);
}

// cls[j] = remap[slot]; rep[class] = the smallest node (linear interior index) of the class
static __global__ void k_dict_assign(Geo g, const int *__restrict__ slot, const int *__restrict__ remap,
                              unsigned short *__restrict__ cls, int *__restrict__ rep) {
  HMG_NODE_IDX(g, ix, iy, iz);
  const int64_t f = ((int64_t)iz * g.n[1] + iy) * g.n[0] + ix;
  const int c = remap[slot[f]];
  cls[g.idx(ix, iy, iz)] = (unsigned short)c;
  atomicMin(rep + c, (int)f);
}

// tab[c][k] = planes[k][node rep[c]] (W 8-byte words per element)
static __global__ void k_dict_fill(Geo g, const unsigned long long *__restrict__ planes, int nplanes, int W,
                            const int *__restrict__ rep, int ncls, unsigned long long *__restrict__ tab) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)ncls * nplanes) return;
  const int c = (int)(t / nplanes), k = (int)(t % nplanes);
  const int f = rep[c];
  const int ix = f % g.n[0], iy = (f / g.n[0]) % g.n[1], iz = f / (g.n[0] * g.n[1]);
  const int64_t j = g.idx(ix, iy, iz);
  for (int w = 0; w < W; ++w) tab[((int64_t)c * nplanes + k) * W + w] = planes[((int64_t)k * g.total + j) * W + w];
}

// *bad = 1 if any node's stored vector differs (bitwise) from its class's table entry
static __global__ void k_dict_verify(Geo g, const unsigned long long *__restrict__ planes, int nplanes, int W,
                              const unsigned short *__restrict__ cls, const unsigned long long *__restrict__ tab,
                              int *bad) {
  HMG_NODE_IDX(g, ix, iy, iz);
  const int64_t j = g.idx(ix, iy, iz);
  const int64_t c = cls[j];
  bool same = true;
  for (int k = 0; k < nplanes && same; ++k)
    for (int w = 0; w < W; ++w) same = same && planes[((int64_t)k * g.total + j) * W + w] == tab[(c * nplanes + k) * W + w];
  if (!same) atomicExch(bad, 1);
}

// exact widening of a float2 class table to fp64 (the arithmetic of the consuming kernel)
static __global__ void k_dict_widen(const float2 *__restrict__ src, double2 *__restrict__ dst, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) dst[t] = make_double2((double)src[t].x, (double)src[t].y);
}

}  // namespace hmg
