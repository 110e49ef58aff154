// solvers, load vectors and potentials on the B200.
#pragma once

#include <vector>

#include "igb_device.hpp"

namespace igb {

struct SolverOpts {  // SolverOptions (solver.hpp:37-41)
  double tol = 1e-8;
  int max_iter = 1000;
  int restart = 30;
};
struct SolveResult {  // SolveStats (solver.hpp:43-48)
  int iterations = 0;
  double residual = 0;
  bool converged = false;
  double seconds = 0;
};
// restarted GMRES / CG of solver.hpp with device-resident vectors; b, x host
SolveResult gmres(H2Device& A, const double* b, double* x, const SolverOpts& o);
SolveResult cg(H2Device& A, const double* b, double* x, const SolverOpts& o);

// quadrature points (element-major, q = a + n b) of the load-vector rule;
// returns points per element (n^2, n = quad_order > 0 ? quad_order : P + 2)
int quad_points(const Discretization& d, int quad_order, int device, std::vector<double>& pts);
// b = load vector from data values at those points (Scalar per point, or 3
// complex components per point for Maxwell)
void assemble_rhs(const Discretization& d, int quad_order, int device, const double* gvals, double* b);
// single-layer potential of a density at points (Maxwell: 3 complex per point)
void eval_potential(const Discretization& d, int quad_order, int device, const double* density, int npts,
                    const double* pts, double* out);

}  // namespace igb
