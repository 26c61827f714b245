// solver_c128.cu -- instantiates the c128 solver (solver.cuh) in its own translation unit.
#include "solver.cuh"

namespace hmg {
SolverBase *make_solver_c128() { return new Solver<double>; }
}  // namespace hmg
