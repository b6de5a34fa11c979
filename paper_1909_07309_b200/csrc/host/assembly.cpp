// Host-side 1D Galerkin assembly; follows /root/reference/proj/core/src/assembly.cpp:47-149.
#include "assembly.hpp"

#include <algorithm>

#include <stdexcept>

namespace stiga {

namespace {
BandedMatrix assemble_impl(const SplineSpace1D& space, const QuadratureRule& quad, int deriv_row, int deriv_col,
                           const std::function<double(int, double)>& weight_at, bool check);
}

BandedMatrix assemble_univariate_fn(const SplineSpace1D& space, const QuadratureRule& quad, int deriv_row,
                                    int deriv_col, const std::function<double(double)>& weight) {
    return assemble_impl(space, quad, deriv_row, deriv_col, [&](int, double x) { return weight(x); },
                         deriv_row == deriv_col);
}

BandedMatrix assemble_univariate(const SplineSpace1D& space, const QuadratureRule& quad, int deriv_row,
                                 int deriv_col, const std::vector<double>* element_weights) {
    if (element_weights && static_cast<int>(element_weights->size()) != quad.num_elements)
        throw std::invalid_argument("assemble_univariate: one weight per element required");
    if (!element_weights)
        return assemble_impl(space, quad, deriv_row, deriv_col, [](int, double) { return 1.0; }, false);
    return assemble_impl(space, quad, deriv_row, deriv_col,
                         [&](int e, double) { return (*element_weights)[e]; }, deriv_row == deriv_col);
}

namespace {
BandedMatrix assemble_impl(const SplineSpace1D& space, const QuadratureRule& quad, int deriv_row, int deriv_col,
                           const std::function<double(int, double)>& weight_at, bool check) {
    if (deriv_row < 0 || deriv_row > 1 || deriv_col < 0 || deriv_col > 1)
        throw std::invalid_argument("assemble_univariate: derivative orders must be 0 or 1");
    if (quad.num_elements != space.knot_vector().num_elements())
        throw std::invalid_argument("assemble_univariate: quadrature built on a different knot vector");
    const int n = space.dim(), p = space.degree();
    BandedMatrix A{DenseMatrix(n, n), p};
    std::vector<double> val(p + 1), der(p + 1);
    for (int q = 0; q < quad.num_points(); ++q) {
        const double wq = weight_at(quad.element_of(q), quad.nodes[q]);
        if (check && wq <= 0.0)
            throw std::runtime_error("assemble_univariate: non-positive weight sample in a mass/stiffness integral");
        const double c = quad.weights[q] * wq;
        const int first = space.eval_active(quad.nodes[q], 0, val.data());
        space.eval_active(quad.nodes[q], 1, der.data());
        const auto& rv = deriv_row == 0 ? val : der;
        const auto& cv = deriv_col == 0 ? val : der;
        for (int a = 0; a <= p; ++a) {
            const int i = first + a;
            if (i < 0 || i >= n) continue;
            const double ri = rv[a];
            if (ri == 0.0) continue;
            for (int b = 0; b <= p; ++b) {
                const int j = first + b;
                if (j < 0 || j >= n) continue;
                A.m(i, j) += c * cv[b] * ri;
            }
        }
    }
    return A;
}
}  // namespace

std::pair<BandedMatrix, BandedMatrix> assemble_time_matrices(int p_t, int n_el_t, double T) {
    if (T <= 0.0) throw std::invalid_argument("assemble_time_matrices: T must be positive");
    const SplineSpace1D space = SplineSpace1D::temporal(p_t, n_el_t);
    const QuadratureRule quad = gauss_rule(space.knot_vector(), p_t + 1);
    BandedMatrix W = assemble_univariate(space, quad, 0, 1);
    BandedMatrix M = assemble_univariate(space, quad, 0, 0);
    for (double& v : M.m.a) v *= T;
    return {std::move(W), std::move(M)};
}

namespace {
// The spatial space on uniform open knots with both end functions dropped is mirror symmetric
// (b_i(x) = b_{n-1-i}(1-x)), so its Galerkin matrices satisfy A(i,j) = A(j,i) = A(n-1-i,n-1-j)
// exactly; quadrature reproduces that only to rounding (~1e-14 relative).  Every entry is replaced
// by the mean of its four mirror images, summed in a canonical order, so the four positions hold
// bitwise identical values: the matrices the reference's quadrature approximates, to rounding,
// and exactly centrosymmetric, which lets the setup split their eigenbasis (host/fdsetup.cpp,
// folded products).
void mirror_symmetrize(DenseMatrix& A) {
    const Index n = A.rows;
    DenseMatrix B(n, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            double v[4] = {A(i, j), A(j, i), A(n - 1 - i, n - 1 - j), A(n - 1 - j, n - 1 - i)};
            std::sort(v, v + 4);
            B(i, j) = ((v[0] + v[1]) + (v[2] + v[3])) * 0.25;
        }
    A = std::move(B);
}
}  // namespace

void assemble_spatial_parametric(int p, int n_el, int q, BandedMatrix& K, BandedMatrix& M) {
    const SplineSpace1D space = SplineSpace1D::spatial(p, n_el);
    const QuadratureRule quad = gauss_rule(space.knot_vector(), q);
    K = assemble_univariate(space, quad, 1, 1);
    M = assemble_univariate(space, quad, 0, 0);
    mirror_symmetrize(K.m);
    mirror_symmetrize(M.m);
}

} // namespace stiga
