// tail_cluster.cu -- the cluster instantiations of k_coarse_tail (k_tail.cuh): the small coarse
// levels of a V(1,1) cycle as ONE thread-block cluster, passes separated by the hardware
// cluster barrier.  Own translation unit: built in parallel with the solver units.
#include "k_tail.cuh"

namespace hmg {

template <typename TK> static void *tail_cluster_kernel(int dim, int kind) {
  if (dim == 2) {
    switch (kind) {
      case PK_RB: return (void *)k_coarse_tail<TK, 2, PK_RB, 1, TAIL_CL_NT, true>;
      case PK_ELEMENT: return (void *)k_coarse_tail<TK, 2, PK_ELEMENT, 1, TAIL_CL_NT, true>;
      case PK_JACOBI: return (void *)k_coarse_tail<TK, 2, PK_JACOBI, 1, TAIL_CL_NT, true>;
      case PK_PLUS: return (void *)k_coarse_tail<TK, 2, PK_PLUS, 1, TAIL_CL_NT, true>;
    }
  } else {
    switch (kind) {
      case PK_ELEMENT: return (void *)k_coarse_tail<TK, 3, PK_ELEMENT, 1, TAIL_CL_NT, true>;
      case PK_JACOBI: return (void *)k_coarse_tail<TK, 3, PK_JACOBI, 1, TAIL_CL_NT, true>;
      case PK_PLUS: return (void *)k_coarse_tail<TK, 3, PK_PLUS, 1, TAIL_CL_NT, true>;
    }
  }
  return nullptr;
}

void *tail_cluster_fn(bool fp64_storage, int dim, int kind) {
  return fp64_storage ? tail_cluster_kernel<double>(dim, kind) : tail_cluster_kernel<float>(dim, kind);
}

}  // namespace hmg
