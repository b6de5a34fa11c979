// Host-side 1D Galerkin assembly (restates /root/reference/proj/core/src/assembly.cpp:47-149).
#pragma once

#include <functional>
#include <utility>
#include <vector>

#include "bspline.hpp"
#include "linalg.hpp"

namespace stiga {

/// Square banded matrix stored densely with its half bandwidth (assembly.hpp:18-36).
struct BandedMatrix {
    DenseMatrix m;
    int hbw = 0;
    Index rows() const { return m.rows; }
};

/// entry (i,j) = int w D^{deriv_col} b_j D^{deriv_row} b_i  (assembly.cpp:47-79).
/// element_weights (one per element) or nullptr for w = 1.
BandedMatrix assemble_univariate(const SplineSpace1D& space, const QuadratureRule& quad, int deriv_row,
                                 int deriv_col, const std::vector<double>* element_weights = nullptr);

/// assemble_univariate with a weight function of the parametric coordinate (assembly.cpp:112-116);
/// mass/stiffness (deriv_row == deriv_col) require weight > 0 at every quadrature point.
BandedMatrix assemble_univariate_fn(const SplineSpace1D& space, const QuadratureRule& quad, int deriv_row,
                                    int deriv_col, const std::function<double(double)>& weight);

/// W_t = [int b'_j b_i], M_t = T * mass on the temporal space (assembly.cpp:129-138).
std::pair<BandedMatrix, BandedMatrix> assemble_time_matrices(int p_t, int n_el_t, double T);

/// Parametric per-direction stiffness / mass (assembly.cpp:140-149), q points per element.
void assemble_spatial_parametric(int p, int n_el, int q, BandedMatrix& K, BandedMatrix& M);

} // namespace stiga
