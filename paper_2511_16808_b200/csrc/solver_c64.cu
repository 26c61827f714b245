// solver_c64.cu -- instantiates the c64 solver (solver.cuh) in its own translation unit.
#include "solver.cuh"

namespace hmg {
SolverBase *make_solver_c64() { return new Solver<float>; }
}  // namespace hmg
