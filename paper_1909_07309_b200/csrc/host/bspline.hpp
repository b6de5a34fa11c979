// B-spline substrate for the host-side 1D assembly.
// Restates /root/reference/proj/core/include/stiga/bspline.hpp:15-101 without Eigen.
#pragma once

#include <utility>
#include <vector>

namespace stiga {

/// Open knot vector on [0,1] with degree (bspline.hpp:15-50).
class KnotVector {
public:
    KnotVector(int degree, std::vector<double> knots);
    static KnotVector uniform_open(int degree, int n_el);

    int degree() const { return degree_; }
    const std::vector<double>& knots() const { return knots_; }
    int num_basis() const { return static_cast<int>(knots_.size()) - degree_ - 1; }
    double mesh_size() const;
    int num_elements() const { return static_cast<int>(spans_.size()); }
    std::pair<double, double> element(int e) const { return spans_[e]; }
    int find_span(double x) const;
    /// Values (deriv_order 0) or first derivatives (1) of the p+1 non-vanishing
    /// B-splines at x; returns the index of the first one (bspline.cpp:100-130).
    int eval_basis(double x, int deriv_order, double* out) const;

private:
    int degree_;
    std::vector<double> knots_;
    std::vector<std::pair<double, double>> spans_;
};

/// Spline space with optional first/last function eliminated (bspline.hpp:54-81).
class SplineSpace1D {
public:
    SplineSpace1D(KnotVector kv, bool drop_first, bool drop_last);
    static SplineSpace1D spatial(int p, int n_el);   // drops both ends
    static SplineSpace1D temporal(int p, int n_el);  // drops the first function only
    const KnotVector& knot_vector() const { return kv_; }
    int degree() const { return kv_.degree(); }
    int dim() const { return n_; }
    int eval_active(double x, int deriv_order, double* out) const;

private:
    KnotVector kv_;
    bool drop_first_, drop_last_;
    int n_;
};

/// Per-element Gauss-Legendre rule (bspline.hpp:85-97).
struct QuadratureRule {
    std::vector<double> nodes, weights;
    int points_per_element = 0;
    int num_elements = 0;
    int num_points() const { return static_cast<int>(nodes.size()); }
    int element_of(int q) const { return q / points_per_element; }
};

std::pair<std::vector<double>, std::vector<double>> gauss_legendre_reference(int q);
QuadratureRule gauss_rule(const KnotVector& kv, int points_per_element);

} // namespace stiga
