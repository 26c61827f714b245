// common.cuh -- complex arithmetic, padded-grid geometry and launch plumbing
// shared by the libhmg CUDA sources (NOT by oracle/: the two share no code).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace hmg {

// ----------------------------------------------------------------- complex
template <typename T> struct CT;
template <> struct CT<float>  { using type = float2; };
template <> struct CT<double> { using type = double2; };
template <typename T> using cplx = typename CT<T>::type;

template <typename T> __host__ __device__ __forceinline__ cplx<T> mkc(T a, T b) { cplx<T> r; r.x = a; r.y = b; return r; }
template <typename T> __host__ __device__ __forceinline__ cplx<T> cadd(cplx<T> a, cplx<T> b) { return mkc<T>(a.x + b.x, a.y + b.y); }
template <typename T> __host__ __device__ __forceinline__ cplx<T> csub(cplx<T> a, cplx<T> b) { return mkc<T>(a.x - b.x, a.y - b.y); }
template <typename T> __host__ __device__ __forceinline__ cplx<T> cmul(cplx<T> a, cplx<T> b) {
  return mkc<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <typename T> __host__ __device__ __forceinline__ cplx<T> cscale(cplx<T> a, T s) { return mkc<T>(a.x * s, a.y * s); }
// acc + a*b
template <typename T> __host__ __device__ __forceinline__ cplx<T> cfma(cplx<T> acc, cplx<T> a, cplx<T> b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
  return acc;
}
// acc + s*a (s real)
template <typename T> __host__ __device__ __forceinline__ cplx<T> cfmar(cplx<T> acc, T s, cplx<T> a) {
  acc.x = fma(s, a.x, acc.x);
  acc.y = fma(s, a.y, acc.y);
  return acc;
}
template <typename T> __host__ __device__ __forceinline__ cplx<T> cdiv(cplx<T> a, cplx<T> b) {
  T d = b.x * b.x + b.y * b.y;
  return mkc<T>((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
template <typename T> __host__ __device__ __forceinline__ cplx<T> crecip(cplx<T> b) {
  T d = b.x * b.x + b.y * b.y;
  return mkc<T>(b.x / d, -b.y / d);
}
// reciprocal / division with a correctly rounded fp32 reciprocal (MUFU + fixup)
// instead of IEEE division; fp64 keeps the exact division.
__device__ __forceinline__ float frcp(float d) { return __frcp_rn(d); }
__device__ __forceinline__ double frcp(double d) { return 1.0 / d; }
template <typename T> __device__ __forceinline__ cplx<T> crecip_fast(cplx<T> b) {
  const T i = frcp(b.x * b.x + b.y * b.y);
  return mkc<T>(b.x * i, -b.y * i);
}
template <typename T> __device__ __forceinline__ cplx<T> cdiv_fast(cplx<T> a, cplx<T> b) {
  const T i = frcp(b.x * b.x + b.y * b.y);
  return mkc<T>((a.x * b.x + a.y * b.y) * i, (a.y * b.x - a.x * b.y) * i);
}
// opaque select (selp): keeps pivot row swaps as register selects instead of
// letting the optimiser rewrite them into dynamically indexed local memory
__device__ __forceinline__ float selp(bool c, float a, float b) {
  float r;
  asm("{ .reg .pred q; setp.ne.b32 q, %3, 0; selp.f32 %0, %1, %2, q; }" : "=f"(r) : "f"(a), "f"(b), "r"((int)c));
  return r;
}
__device__ __forceinline__ double selp(bool c, double a, double b) {
  double r;
  asm("{ .reg .pred q; setp.ne.b32 q, %3, 0; selp.f64 %0, %1, %2, q; }" : "=d"(r) : "d"(a), "d"(b), "r"((int)c));
  return r;
}
template <typename T> __device__ __forceinline__ cplx<T> cselp(bool c, cplx<T> a, cplx<T> b) {
  return mkc<T>(selp(c, a.x, b.x), selp(c, a.y, b.y));
}
template <typename T> __host__ __device__ __forceinline__ T cabs2(cplx<T> a) { return a.x * a.x + a.y * a.y; }

template <typename To, typename From> __host__ __device__ __forceinline__ cplx<To> ccast(cplx<From> a) {
  return mkc<To>((To)a.x, (To)a.y);
}

// ----------------------------------------------------------------- geometry
// Every level vector lives in a zero-padded box: G ghost layers on each side
// of every axis (none in z for 2D), row pitch px rounded up to 8 elements.
// Interior node (x,y,z), 0 <= x < n[0] ..., sits at index idx(x,y,z).
// Ghost entries are zero on one GPU, so truncation (homogeneous Dirichlet,
// reading A4/A5) costs no branch in the operator kernels.
struct Geo {
  int dim;
  int n[3];        // LOCAL interior nodes per axis (n[2] = 1 in 2D)
  int N[3];        // GLOBAL nodes per axis (== n on one rank)
  int o[3];        // global coordinate of local node 0 (nonzero only on the slab axis)
  int G;           // ghost width
  int64_t px;      // row pitch
  int64_t pxy;     // plane pitch
  int64_t total;   // padded box size (elements)
  int64_t base;    // index of interior node (0,0,0)
  int64_t slab_off;  // first element of the interior slab (rows/planes G .. G+n-1)
  int64_t slab_len;  // elements of the interior slab

  __host__ __device__ __forceinline__ int64_t idx(int x, int y, int z) const {
    return base + (int64_t)z * pxy + (int64_t)y * px + x;
  }
  __host__ __device__ __forceinline__ int64_t delta(int ox, int oy, int oz) const {
    return (int64_t)oz * pxy + (int64_t)oy * px + ox;
  }
  // is LOCAL node (x,y,z) inside the GLOBAL domain?  Every boundary decision
  // (truncation, patch clipping, cnt_j) is taken in global coordinates, so a
  // slab of a partitioned grid behaves exactly like the same rows of the whole.
  __host__ __device__ __forceinline__ bool inside(int x, int y, int z) const {
    x += o[0]; y += o[1]; z += o[2];
    return x >= 0 && x < N[0] && y >= 0 && y < N[1] && z >= 0 && z < N[2];
  }
  __host__ __device__ __forceinline__ int64_t nodes() const { return (int64_t)n[0] * n[1] * n[2]; }
};

inline Geo make_geo(int dim, const int64_t nodes[3], int G) {
  Geo g;
  g.dim = dim;
  g.n[0] = (int)nodes[0];
  g.n[1] = (int)nodes[1];
  g.n[2] = dim == 3 ? (int)nodes[2] : 1;
  for (int a = 0; a < 3; ++a) { g.N[a] = g.n[a]; g.o[a] = 0; }
  g.G = G;
  g.px = ((g.n[0] + 2 * G) + 7) / 8 * 8;
  g.pxy = g.px * (g.n[1] + 2 * G);
  int Gz = dim == 3 ? G : 0;
  g.total = g.pxy * (g.n[2] + 2 * Gz);
  g.base = (int64_t)Gz * g.pxy + (int64_t)G * g.px + G;
  if (dim == 3) {
    g.slab_off = (int64_t)G * g.pxy;
    g.slab_len = (int64_t)g.n[2] * g.pxy;
  } else {
    g.slab_off = (int64_t)G * g.px;
    g.slab_len = (int64_t)g.n[1] * g.px;
  }
  return g;
}

// thread -> interior node mapping used by all node-parallel kernels:
// block (32, 8, 1), grid (ceil(nx/32), ceil(ny/8), nz)
struct NodeLaunch {
  dim3 grid, block;
};
inline NodeLaunch node_launch(const Geo &g) {
  NodeLaunch L;
  L.block = dim3(32, 8, 1);
  L.grid = dim3((g.n[0] + 31) / 32, (g.n[1] + 7) / 8, g.n[2]);
  return L;
}

// launch accounting (hmg_launch_count) -- incremented by every launch
void count_launch();

// Programmatic dependent launch (runtime.cuh launch()): every kernel of the library
// starts with this prologue.  griddepcontrol.wait blocks until the grids this one
// depends on have completed and their memory is visible, so nothing is read early;
// launch_dependents lets the NEXT kernel's blocks be scheduled once every block of
// this grid has started, hiding its launch latency behind this grid's tail.  Both are
// no-ops for a normal launch.
#define HMG_PDL_PROLOGUE()                                   \
  do {                                                       \
    asm volatile("griddepcontrol.wait;" ::: "memory");       \
    asm volatile("griddepcontrol.launch_dependents;" :::);   \
  } while (0)

}  // namespace hmg

#define HMG_NODE_IDX(g, X_, Y_, Z_)                           \
  const int X_ = blockIdx.x * blockDim.x + threadIdx.x;       \
  const int Y_ = blockIdx.y * blockDim.y + threadIdx.y;       \
  const int Z_ = blockIdx.z;                                  \
  if (X_ >= (g).n[0] || Y_ >= (g).n[1]) return;
