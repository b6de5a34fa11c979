// Spline geometry map, problem catalog and the coefficient pieces of the geometry-aware
// preconditioner A^G (host side).  Restates, Eigen-free:
//   GeometryMap                         /root/reference/proj/core/src/geometry.cpp:7-97
//   fit_geometry / make_problem         /root/reference/proj/core/src/problems.cpp:59-124, 126-261
//   coefficient_diagonal_samples        /root/reference/proj/core/src/assembly.cpp:270-311
//   separate_variables                  /root/reference/proj/core/src/assembly.cpp:313-411
//   diag(A) of SpaceTimeSystem's A_     /root/reference/proj/core/src/solver.cpp:58-70, 138-142
//     (only the diagonal of the physical K_s, M_s is formed: the triplet assembly of
//      assemble_spatial_physical, assembly.cpp:151-268, would need ~131 GB at config 4)
#pragma once

#include <functional>
#include <string>
#include <vector>

#include "assembly.hpp"
#include "bspline.hpp"
#include "linalg.hpp"

namespace stiga {

/// Tensor-product spline map F : (0,1)^d -> R^d; control points over the full basis, colex rows.
class GeometryMap {
public:
    GeometryMap() = default;
    GeometryMap(std::vector<KnotVector> kvs, DenseMatrix control_points);
    static GeometryMap identity(int d);
    int dim() const { return static_cast<int>(kvs_.size()); }
    const std::vector<KnotVector>& knot_vectors() const { return kvs_; }
    const DenseMatrix& control_points() const { return cp_; }
    void value(const double* eta, double* x) const;
    /// J(r, c) = dF_r / deta_c, stored column-major d x d in J[r + d*c].
    void jacobian(const double* eta, double* J) const;

private:
    std::vector<KnotVector> kvs_;
    DenseMatrix cp_;  // prod(m_l) x d
    std::vector<Index> strides_;
};

using MapFn = std::function<void(const double* eta, double* x)>;
using FieldFn = std::function<double(const double* x)>;  // nullptr = constant 1

/// fit_geometry(map, d, p_g, n_el) (problems.cpp:59-124): least-squares spline fit on a
/// max(4m, 32)-point tensor sample grid; throws if the fitted Jacobian is not positive.
GeometryMap fit_geometry(const MapFn& map, int d, int p_g, int n_el, double* max_residual = nullptr);

/// The parts of ProblemSpec (problems.hpp:25-37) the preconditioner needs.
struct ProblemSpec {
    std::string name;
    int d = 2;
    GeometryMap geometry;
    double T = 1.0;
    FieldFn gamma_s, nu_s;                           // spatial capacity / conductivity (nullptr = 1)
    std::function<double(double)> gamma_t, nu_t;     // temporal factors (nullptr = 1)
};

/// make_problem(id) (problems.cpp:244-261) for the geometry/coefficient part of the catalog
/// ("identity-interval-1d", "identity-square-2d", "identity-cube-3d", "quarter-annulus-2d",
/// "separable-nu-2d") plus the BASELINE config-4 "deformed-cube-3d":
/// F(x^) = x^ + 0.1 sin(pi x^1) sin(pi x^2) sin(pi x^3) (1,1,1) fitted with (p_g, n_el_g) = (3, 8),
/// kappa(x) = 1 + 0.5 sin(2 pi x1) cos(2 pi x2), c(x) = 1 + 0.25 x3.
ProblemSpec make_problem(const std::string& id);

/// coefficient_diagonal_samples (assembly.cpp:270-311): element-midpoint samples, dims
/// (n_el_1..n_el_d, d+1) colex; slice l < d = (J^-1 J^-T)_{ll} |det J| nu_s, slice d = |det J| gamma_s.
std::vector<double> coefficient_diagonal_samples(const std::vector<KnotVector>& kvs, const GeometryMap& F,
                                                 const FieldFn& nu_s, const FieldFn& gamma_s);

struct SeparableCoefficients {
    std::vector<std::vector<double>> phi, Phi;
    std::vector<double> residuals;
    bool converged = true;
    int sweeps = 0;
};
/// separate_variables (assembly.cpp:313-411): ALS rank-one fit, <= 50 sweeps, tol 1e-10,
/// geometric-mean gauge on phi_2..phi_d.
SeparableCoefficients separate_variables(const std::vector<double>& samples, const std::vector<int>& nel);

/// diag(K_s) and diag(M_s) of the physical spatial matrices K = int nu_s grad B.grad B,
/// M = int gamma_s B B (assembly.cpp:151-268) by quadrature, without forming the matrices.
void physical_diagonals(const std::vector<SplineSpace1D>& spaces, const GeometryMap& F, int q, const FieldFn& nu_s,
                        const FieldFn& gamma_s, std::vector<double>& dK, std::vector<double>& dM);

/// Everything make_geometry_preconditioner (solver.cpp:127-144) feeds ExtendedFDPreconditioner::setup,
/// for uniform degree p / n_el in every direction and in time (SpaceTimeSystem, solver.cpp:34-65).
struct GeometryPreconditionerPieces {
    std::vector<DenseMatrix> Kt, Mt_s;  // K~_l, M~_l
    DenseMatrix Wt, Mt;                 // W_t and the nu_t/gamma_t-weighted M_t
    std::vector<double> D;              // diag(A) / diag(A~), N_dof
    SeparableCoefficients sep;
};
GeometryPreconditionerPieces geometry_preconditioner_pieces(const ProblemSpec& prob, int p, int n_el, bool want_D);

/// W_t and the nu_t/gamma_t-weighted M_t of SpaceTimeSystem (solver.cpp:119-125).
void time_matrices(const ProblemSpec& prob, int p, int n_el, DenseMatrix& Wt, DenseMatrix& Mt);

/// Device field kinds of a catalog problem (nu_s, gamma_s) for the in-kernel physical assembly.
void problem_field_kinds(const ProblemSpec& prob, int& nu_kind, int& gamma_kind);

/// Device kind (gpu::SourceKind) of the problem's manufactured source term / exact solution
/// (problems.cpp:131-241): 1 identity-*, 2 quarter-annulus-2d, 3 separable-nu-2d, 0 none.
int problem_source_kind(const ProblemSpec& prob);

/// The constants of A-hat (solver.cpp:82-112): gamma_mean = int gamma_s / |Omega| and
/// nu_mean = int nu_s / |Omega| * int_0^1 nu_t/gamma_t, Gauss rule with p + 1 points per element.
void system_means(const ProblemSpec& prob, int p, int n_el, double& gamma_mean, double& nu_mean);

}  // namespace stiga
