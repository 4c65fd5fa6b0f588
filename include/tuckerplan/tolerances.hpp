// tuckerplan (B200 engine) : the two acceptance thresholds of reference tolerances.hpp that concern the engine.
// (Its corpus-statistics thresholds belong to bench.hpp, which is outside this repo's scope.)
#pragma once

namespace tuckerplan::tol {

// relative rise allowed in the reconstruction error between Gauss-Seidel sweeps (tolerances.hpp:14)
inline constexpr double kSweepMonotoneSlack = 1e-12;

// agreement of the projectors F F^T obtained through different trees in a Jacobi sweep (tolerances.hpp:17);
// the parity tests of this repo compare factor subspaces against the oracle with the same bound
inline constexpr double kProjectorTol = 1e-9;

}  // namespace tuckerplan::tol
