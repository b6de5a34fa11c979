// Host-side pencil factorizations (restates /root/reference/proj/core/src/pencil.cpp:12-165).
#pragma once

#include <vector>

#include "linalg.hpp"

namespace stiga {

/// K U = M U Lambda with U^T M U = I, ascending (pencil.cpp:12-21).
void spd_generalized_eig(const DenseMatrix& K, const DenseMatrix& M, DenseMatrix& U, Vector& lambda);

struct SkewPencilEig {
    DenseMatrix U;
    std::vector<double> lambda;
    int zero_count = 0;
};
SkewPencilEig skew_pencil_eig(const DenseMatrix& W, const DenseMatrix& M);

/// pencil.hpp:40-52
struct TimeFactorization {
    DenseMatrix U;
    std::vector<double> lambda;
    int zero_count = 0;
    Vector g;
    double sigma = 0.0;
    Vector r;
    double rho = 0.0;
    Index size() const { return U.rows; }
};
TimeFactorization time_factorization(const DenseMatrix& Wt, const DenseMatrix& Mt);

} // namespace stiga
