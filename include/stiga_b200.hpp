// stiga_b200.hpp -- the C++ binding a maintainer adds to the reference `stiga`:
// the same surface as ExtendedFDPreconditioner (fdsolve.hpp:41-70), KronSumOperator
// (kronop.hpp:61-79) and gmres(LinOp, LinOp*, b, GmresOptions) (gmres.hpp:12-35), over the C ABI in
// stiga_gpu.h.  Header-only, Eigen-free: matrices are dense column-major n x n buffers (the
// reference's BandedMatrix stores dense; Eigen's MatrixXd::data() can be passed as is), vectors are
// std::vector<double> on the host or raw device pointers.  Status codes are rethrown as the
// reference's exception types (std::invalid_argument / std::runtime_error).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "stiga_gpu.h"

namespace stiga {
namespace b200 {

inline void check(int st) {
    if (st == STIGA_OK) return;
    if (st == STIGA_INVALID_ARGUMENT) throw std::invalid_argument(stiga_last_error());
    throw std::runtime_error(stiga_last_error());
}

using Vector = std::vector<double>;

// A dense column-major square matrix (what the reference's BandedMatrix::matrix() holds).
struct Dense {
    int n = 0;
    std::vector<double> a;  // a[i + n * j]
    Dense() = default;
    explicit Dense(int n_) : n(n_), a(static_cast<size_t>(n_) * n_, 0.0) {}
    double& operator()(int i, int j) { return a[i + static_cast<size_t>(n) * j]; }
    double operator()(int i, int j) const { return a[i + static_cast<size_t>(n) * j]; }
};

// Eigen-free versions of the reference's 1D assembly (assembly.cpp:129-149), host side.
inline std::pair<Dense, Dense> assemble_time_matrices(int p, int n_el, double T = 1.0) {
    int n = 0;
    check(stiga_space_dim(p, n_el, 1, &n));
    Dense W(n), M(n);
    check(stiga_assemble_time_matrices(p, n_el, T, W.a.data(), M.a.data()));
    return {W, M};
}
inline std::pair<Dense, Dense> assemble_spatial_parametric(int p, int n_el) {
    int n = 0;
    check(stiga_space_dim(p, n_el, 0, &n));
    Dense K(n), M(n);
    check(stiga_assemble_spatial_parametric(p, n_el, p + 1, K.a.data(), M.a.data()));
    return {K, M};
}

// ExtendedFDPreconditioner on the B200 (fdsolve.hpp:41-70).
class Preconditioner {
public:
    static Preconditioner setup(const std::vector<Dense>& K, const std::vector<Dense>& M, const Dense& Wt,
                                const Dense& Mt, double gamma, double nu,
                                const std::optional<Vector>& D = std::nullopt, int device = 0) {
        if (K.size() != M.size() || K.empty())
            throw std::invalid_argument("ExtendedFDPreconditioner: per-direction matrices mismatch");
        std::vector<int> n;
        std::vector<const double*> Kp, Mp;
        for (size_t l = 0; l < K.size(); ++l) {
            n.push_back(K[l].n);
            Kp.push_back(K[l].a.data());
            Mp.push_back(M[l].a.data());
        }
        Preconditioner P;
        check(stiga_fd_setup(static_cast<int>(K.size()), n.data(), Kp.data(), Mp.data(), Wt.n, Wt.a.data(),
                             Mt.a.data(), gamma, nu, D ? D->data() : nullptr,
                             D ? static_cast<long long>(D->size()) : 0, device, &P.h_));
        return P;
    }
    Preconditioner() = default;
    Preconditioner(Preconditioner&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    Preconditioner& operator=(Preconditioner&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    Preconditioner(const Preconditioner&) = delete;
    Preconditioner& operator=(const Preconditioner&) = delete;
    ~Preconditioner() {
        if (h_) stiga_fd_destroy(h_);
    }

    long long size() const {
        long long n = 0;
        check(stiga_fd_size(h_, &n));
        return n;
    }
    // Host convenience (fdsolve.hpp:56): H2D, apply, D2H.
    Vector apply(const Vector& r) const {
        if (static_cast<long long>(r.size()) != size())
            throw std::invalid_argument("ExtendedFDPreconditioner::apply: vector length mismatch");
        Vector s(r.size());
        check(stiga_fd_apply_host(h_, r.data(), s.data()));
        return s;
    }
    // The hot path: device buffers, asynchronous on `st`.
    void apply_device(const double* d_r, double* d_s, cudaStream_t st = nullptr) const {
        check(stiga_fd_apply(h_, d_r, d_s, st));
    }
    stiga_fd_t handle() const { return h_; }

    // Device-side setup (stiga_fd_setup_ex): D on the device (d_D, N_dof doubles, may be
    // null), Lambda_s / S^-1 on the device, optionally cuSOLVER eigensolves.
    static Preconditioner setup_device(const std::vector<Dense>& K, const std::vector<Dense>& M, const Dense& Wt,
                                       const Dense& Mt, double gamma, double nu, const double* d_D, long long n_dof,
                                       bool cusolver = false, int device = 0) {
        std::vector<int> n;
        std::vector<const double*> Kp, Mp;
        for (size_t l = 0; l < K.size(); ++l) {
            n.push_back(K[l].n);
            Kp.push_back(K[l].a.data());
            Mp.push_back(M[l].a.data());
        }
        stiga_fd_setup_options o{STIGA_SETUP_DEVICE_SCHUR | (cusolver ? STIGA_SETUP_CUSOLVER : 0), d_D};
        Preconditioner P;
        check(stiga_fd_setup_ex(static_cast<int>(K.size()), n.data(), Kp.data(), Mp.data(), Wt.n, Wt.a.data(),
                                Mt.a.data(), gamma, nu, nullptr, d_D ? n_dof : 0, &o, device, &P.h_));
        return P;
    }

private:
    stiga_fd_t h_ = nullptr;
};

// make_problem(id) (problems.cpp:244-261): geometry, coefficients, source term / exact solution.
class Problem {
public:
    explicit Problem(const std::string& id) { check(stiga_problem_create(id.c_str(), &h_)); }
    Problem(const Problem&) = delete;
    Problem& operator=(const Problem&) = delete;
    ~Problem() {
        if (h_) stiga_problem_destroy(h_);
    }
    int dim() const {
        int d = 0;
        check(stiga_problem_dim(h_, &d));
        return d;
    }
    stiga_problem_t handle() const { return h_; }

private:
    stiga_problem_t h_ = nullptr;
};

// KronSumOperator (kronop.hpp:61-79) in the kron_sum_terms form of SpaceTimeSystem (solver.cpp:10-30).
class KronSumOperator {
public:
    static KronSumOperator spacetime(const std::vector<Dense>& K, const std::vector<Dense>& M, const Dense& Wt,
                                     const Dense& Mt, double gamma, double nu, int device = 0) {
        std::vector<int> n;
        std::vector<const double*> Kp, Mp;
        for (size_t l = 0; l < K.size(); ++l) {
            n.push_back(K[l].n);
            Kp.push_back(K[l].a.data());
            Mp.push_back(M[l].a.data());
        }
        KronSumOperator A;
        check(stiga_kronsum_create_spacetime(static_cast<int>(K.size()), n.data(), Kp.data(), Mp.data(), Wt.n,
                                             Wt.a.data(), Mt.a.data(), gamma, nu, device, &A.h_));
        return A;
    }
    // SpaceTimeSystem's A_ = M_s (x) W_t + K_s (x) M_t with the physical K_s, M_s of `prob`
    // (solver.cpp:58-70), assembled on the device.
    static KronSumOperator physical(const Problem& prob, int p, int n_el, int device = 0) {
        KronSumOperator A;
        check(stiga_kronsum_create_physical(prob.handle(), p, n_el, device, &A.h_));
        return A;
    }
    void diagonal_device(double* d_diag, cudaStream_t st = nullptr) const {
        check(stiga_kronsum_diagonal_device(h_, d_diag, st));
    }
    KronSumOperator() = default;
    KronSumOperator(KronSumOperator&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    KronSumOperator(const KronSumOperator&) = delete;
    ~KronSumOperator() {
        if (h_) stiga_kronsum_destroy(h_);
    }
    long long size() const {
        long long n = 0;
        check(stiga_kronsum_size(h_, &n));
        return n;
    }
    void apply_device(const double* d_x, double* d_y, cudaStream_t st = nullptr) const {
        check(stiga_kronsum_apply(h_, d_x, d_y, st));
    }
    stiga_kronsum_t handle() const { return h_; }

private:
    stiga_kronsum_t h_ = nullptr;
};

// gmres.hpp:15-27
struct GmresOptions {
    double tol = 1e-8;
    int max_krylov = 100;
    std::optional<int> restart;
};
struct SolveReport {
    int iterations = 0;
    std::vector<double> residual_history;
    bool converged = false;
    double wall_time_s = 0.0;
    double precond_time_fraction = 0.0;
};

// The device analogue of the reference's LinOp (gmres.hpp:12): y = Op(x) on device vectors.
using DeviceLinOp = std::function<void(const double* d_x, double* d_y, cudaStream_t st)>;

namespace detail {
inline int trampoline(void* ctx, const double* d_in, double* d_out, void* stream) {
    try {
        (*static_cast<const DeviceLinOp*>(ctx))(d_in, d_out, static_cast<cudaStream_t>(stream));
        return 0;
    } catch (...) {
        return 1;
    }
}
inline SolveReport to_report(const stiga_gmres_report& r, const std::vector<double>& hist) {
    SolveReport out;
    out.iterations = r.iterations;
    out.converged = r.converged != 0;
    out.wall_time_s = r.wall_time_s;
    out.precond_time_fraction = r.precond_time_fraction;
    out.residual_history.assign(hist.begin(), hist.begin() + std::min<size_t>(hist.size(), r.history_len));
    return out;
}
}  // namespace detail

// gmres(A, P, b, opts) (gmres.hpp:34-35) over device operators; d_b / d_x are device vectors of n.
inline SolveReport gmres(long long n, const DeviceLinOp& A, const DeviceLinOp* P, const double* d_b, double* d_x,
                         const GmresOptions& opts = {}, cudaStream_t st = nullptr) {
    stiga_gmres_options o{opts.tol, opts.max_krylov, opts.restart ? *opts.restart : 0};
    std::vector<double> hist(opts.max_krylov + 2);
    stiga_gmres_report r{0, 0, 0.0, 0.0, hist.data(), static_cast<int>(hist.size()), 0};
    check(stiga_gmres_op(n, &detail::trampoline, const_cast<DeviceLinOp*>(&A), P ? &detail::trampoline : nullptr,
                         const_cast<DeviceLinOp*>(P), nullptr, d_b, d_x, &o, &r, st));
    return detail::to_report(r, hist);
}

// gmres on the library's own handles (the device-resident SpaceTimeSystem::solve, solver.cpp:146-155).
inline SolveReport gmres(const KronSumOperator& A, const Preconditioner* P, const double* d_b, double* d_x,
                         const GmresOptions& opts = {}, cudaStream_t st = nullptr) {
    stiga_gmres_options o{opts.tol, opts.max_krylov, opts.restart ? *opts.restart : 0};
    std::vector<double> hist(opts.max_krylov + 2);
    stiga_gmres_report r{0, 0, 0.0, 0.0, hist.data(), static_cast<int>(hist.size()), 0};
    check(stiga_gmres(A.handle(), P ? P->handle() : nullptr, d_b, d_x, &o, &r, st));
    return detail::to_report(r, hist);
}

// SpaceTimeSystem pieces around the solve (solver.cpp:82-112, assembly.cpp:413-504, problems.cpp:305-402).
inline std::pair<double, double> system_means(const Problem& prob, int p, int n_el) {
    double g = 0.0, nu = 0.0;
    check(stiga_system_means(prob.handle(), p, n_el, &g, &nu));
    return {g, nu};
}
inline void assemble_rhs(const Problem& prob, int p, int n_el, double* d_b, int device = 0, cudaStream_t st = nullptr) {
    check(stiga_assemble_rhs(prob.handle(), p, n_el, p + 1, device, d_b, st));
}
struct Errors {
    double l2l2 = 0.0, x_upper = 0.0;
};
inline Errors compute_errors(const Problem& prob, int p, int n_el, const double* d_coeffs, int points_per_element,
                             int device = 0) {
    Errors e;
    check(stiga_compute_errors(prob.handle(), p, n_el, d_coeffs, points_per_element, device, &e.l2l2, &e.x_upper));
    return e;
}
// D = diag(A) / diag(A~) of make_geometry_preconditioner (solver.cpp:138-142), on the device.
inline void geometry_scaling_device(const KronSumOperator& A, const KronSumOperator& Atilde, double* d_D,
                                    cudaStream_t st = nullptr) {
    check(stiga_geometry_scaling_device(A.handle(), Atilde.handle(), d_D, st));
}

}  // namespace b200
}  // namespace stiga
