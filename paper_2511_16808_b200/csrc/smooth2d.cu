// smooth2d.cu -- dispatch of the fused Galerkin-level Vanka sweep
// (k_smooth_stored2d, k_vanka.cuh) over stencil radius x patch kind x zero
// initial guess.  Separate translation unit to keep compile times parallel.
#include "runtime.cuh"
#include "k_vanka.cuh"

namespace hmg {

// vectors and arithmetic fp64 on every Galerkin level; coefficients TK
template <typename TK, int R, int KIND>
static void go(bool zero, const Geo &g, const cplx<TK> *coef, const cplx<TK> *hinv, const double2 *f,
               const double2 *u, double2 *uo, double w, cudaStream_t s) {
  if (!hinv) throw HmgError(HMG_EINVAL, "fused Galerkin sweep needs the stored patch inverses");
  constexpr int TX = 32, TY = 16;   // fp64 smem: u (tile + 2 + R) and r (tile + 2), < 48 KB
  const dim3 grid((g.n[0] + TX - 1) / TX, (g.n[1] + TY - 1) / TY), block(32, 8);
  if (zero) launch(k_smooth_stored2d<double, TK, R, KIND, TX, TY, true>, grid, block, 0, s, g, coef, hinv, f, u, uo, w);
  else launch(k_smooth_stored2d<double, TK, R, KIND, TX, TY, false>, grid, block, 0, s, g, coef, hinv, f, u, uo, w);
}

template <typename T, int R>
static void go_kind(int kind, bool zero, const Geo &g, const cplx<T> *coef, const cplx<T> *hinv, const double2 *f,
                    const double2 *u, double2 *uo, double w, cudaStream_t s) {
  switch (kind) {
    case HMG_VANKA_RB: go<T, R, PK_RB>(zero, g, coef, hinv, f, u, uo, w, s); return;
    case HMG_VANKA_ELEMENT: go<T, R, PK_ELEMENT>(zero, g, coef, hinv, f, u, uo, w, s); return;
    case HMG_JACOBI: go<T, R, PK_JACOBI>(zero, g, coef, hinv, f, u, uo, w, s); return;
    case HMG_VANKA_PLUS: go<T, R, PK_PLUS>(zero, g, coef, hinv, f, u, uo, w, s); return;
  }
  throw HmgError(HMG_EINVAL, "unknown smoother");
}

template <typename T>
void smooth_stored2d(int r, int kind, bool zero, const Geo &g, const cplx<T> *coef, const cplx<T> *hinv,
                     const double2 *f, const double2 *u, double2 *uo, double w, cudaStream_t s) {
  switch (r) {
    case 1: go_kind<T, 1>(kind, zero, g, coef, hinv, f, u, uo, w, s); return;
    case 2: go_kind<T, 2>(kind, zero, g, coef, hinv, f, u, uo, w, s); return;
    case 3: go_kind<T, 3>(kind, zero, g, coef, hinv, f, u, uo, w, s); return;
  }
  throw HmgError(HMG_EINVAL, "stencil radius out of range");
}

template void smooth_stored2d<float>(int, int, bool, const Geo &, const float2 *, const float2 *, const double2 *,
                                     const double2 *, double2 *, double, cudaStream_t);
template void smooth_stored2d<double>(int, int, bool, const Geo &, const double2 *, const double2 *, const double2 *,
                                      const double2 *, double2 *, double, cudaStream_t);

}  // namespace hmg
