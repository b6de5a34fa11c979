// C ABI of the B200 extended-FD preconditioner / GMRES path (include/stiga_gpu.h).
//
// Host orchestration only: the host-side setup (1D assembly, pencils, Schur diagonal) runs here
// exactly where the reference runs it (fdsolve.cpp:67-153, pencil.cpp, assembly.cpp), the factors
// are uploaded once, and every apply is a fixed chain of device kernels on the caller's stream.
// There is no CPU compute fallback: without a device every compute entry point fails with
// STIGA_CUDA.
#include "stiga_gpu.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <functional>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "cuda/aux_kernels.cuh"
#include "cuda/fd_kernels.cuh"
#include "cuda/physical.cuh"
#include "cuda/setup_kernels.cuh"
#include "host/eig_device.hpp"
#include "host/assembly.hpp"
#include "host/fdsetup.hpp"
#include "host/geometry.hpp"

using namespace stiga;

#include "common.hpp"
#include "handles.hpp"

using namespace stiga;
using namespace stiga::capi;

namespace {
thread_local std::string g_last_error;
}  // namespace

namespace stiga {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace stiga

namespace {

int half_bandwidth(const DenseMatrix& F) {
    int p = 0;
    for (Index j = 0; j < F.cols; ++j)
        for (Index i = 0; i < F.rows; ++i)
            if (F(i, j) != 0.0) p = std::max(p, static_cast<int>(std::llabs(i - j)));
    return p;
}

// Band storage of coeff * F; the coefficient is folded into the band (coeff_t * kron(...)).
std::vector<double> to_band(const DenseMatrix& F, int p, double coeff) {
    const int n = static_cast<int>(F.rows), w = 2 * p + 1;
    std::vector<double> b(static_cast<size_t>(n) * w, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = std::max(0, i - p); j <= std::min(n - 1, i + p); ++j) b[i * w + (j - i + p)] = coeff * F(i, j);
    return b;
}

}  // namespace

extern "C" {

const char* stiga_last_error(void) { return g_last_error.c_str(); }

int stiga_abi_version(void) { return 101; }

int stiga_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int stiga_space_dim(int p, int n_el, int kind, int* n_out) {
    return guarded([&] {
        require(n_out != nullptr, "stiga_space_dim: null output");
        require(kind == 0 || kind == 1, "stiga_space_dim: kind must be 0 (spatial) or 1 (temporal)");
        const SplineSpace1D s = kind == 0 ? SplineSpace1D::spatial(p, n_el) : SplineSpace1D::temporal(p, n_el);
        *n_out = s.dim();
    });
}

int stiga_assemble_time_matrices(int p_t, int n_el_t, double T, double* Wt, double* Mt) {
    return guarded([&] {
        require(Wt && Mt, "stiga_assemble_time_matrices: null output");
        auto [W, M] = assemble_time_matrices(p_t, n_el_t, T);
        std::memcpy(Wt, W.m.a.data(), W.m.a.size() * sizeof(double));
        std::memcpy(Mt, M.m.a.data(), M.m.a.size() * sizeof(double));
    });
}

int stiga_assemble_spatial_parametric(int p, int n_el, int q, double* K, double* M) {
    return guarded([&] {
        require(K && M, "stiga_assemble_spatial_parametric: null output");
        BandedMatrix Kb, Mb;
        assemble_spatial_parametric(p, n_el, q, Kb, Mb);
        std::memcpy(K, Kb.m.a.data(), Kb.m.a.size() * sizeof(double));
        std::memcpy(M, Mb.m.a.data(), Mb.m.a.size() * sizeof(double));
    });
}

int stiga_assemble_univariate(int p, int n_el, int kind, int q, int deriv_row, int deriv_col,
                              const double* element_weights, double* out) {
    return guarded([&] {
        require(out != nullptr, "stiga_assemble_univariate: null output");
        require(kind == 0 || kind == 1, "stiga_assemble_univariate: kind must be 0 or 1");
        const SplineSpace1D s = kind == 0 ? SplineSpace1D::spatial(p, n_el) : SplineSpace1D::temporal(p, n_el);
        const QuadratureRule quad = gauss_rule(s.knot_vector(), q);
        std::vector<double> w;
        if (element_weights) w.assign(element_weights, element_weights + quad.num_elements);
        const BandedMatrix A = assemble_univariate(s, quad, deriv_row, deriv_col, element_weights ? &w : nullptr);
        std::memcpy(out, A.m.a.data(), A.m.a.size() * sizeof(double));
    });
}

int stiga_problem_create(const char* id, stiga_problem_t* out) {
    return guarded([&] {
        require(id && out, "make_problem: null argument");
        *out = nullptr;
        auto h = std::make_unique<stiga_problem_s>();
        h->spec = make_problem(id);
        *out = h.release();
    });
}

int stiga_problem_destroy(stiga_problem_t P) {
    return guarded([&] { delete P; });
}

int stiga_problem_dim(stiga_problem_t P, int* d) {
    return guarded([&] {
        require(P && d, "stiga_problem_dim: null argument");
        *d = P->spec.d;
    });
}

int stiga_problem_eval_geometry(stiga_problem_t P, const double* eta, double* x, double* J) {
    return guarded([&] {
        require(P && eta, "GeometryMap: null argument");
        if (x) P->spec.geometry.value(eta, x);
        if (J) P->spec.geometry.jacobian(eta, J);
    });
}

int stiga_problem_eval_fields(stiga_problem_t P, const double* x, double* nu_s, double* gamma_s) {
    return guarded([&] {
        require(P && x, "stiga_problem_eval_fields: null argument");
        if (nu_s) *nu_s = P->spec.nu_s ? P->spec.nu_s(x) : 1.0;
        if (gamma_s) *gamma_s = P->spec.gamma_s ? P->spec.gamma_s(x) : 1.0;
    });
}

int stiga_geometry_preconditioner_pieces(stiga_problem_t P, int p, int n_el, double* Kt, double* Mt_s, double* Wt,
                                         double* Mt, double* D, double* phi, double* Phi, double* residuals,
                                         int* sweeps) {
    return guarded([&] {
        require(P && Kt && Mt_s && Wt && Mt, "make_geometry_preconditioner: null argument");
        const GeometryPreconditionerPieces g = geometry_preconditioner_pieces(P->spec, p, n_el, D != nullptr);
        const int d = P->spec.d;
        const size_t nn = g.Kt[0].a.size();
        for (int l = 0; l < d; ++l) {
            std::copy(g.Kt[l].a.begin(), g.Kt[l].a.end(), Kt + l * nn);
            std::copy(g.Mt_s[l].a.begin(), g.Mt_s[l].a.end(), Mt_s + l * nn);
        }
        std::copy(g.Wt.a.begin(), g.Wt.a.end(), Wt);
        std::copy(g.Mt.a.begin(), g.Mt.a.end(), Mt);
        if (D) std::copy(g.D.begin(), g.D.end(), D);
        for (int l = 0; l < d; ++l) {
            if (phi) std::copy(g.sep.phi[l].begin(), g.sep.phi[l].end(), phi + l * n_el);
            if (Phi) std::copy(g.sep.Phi[l].begin(), g.sep.Phi[l].end(), Phi + l * n_el);
        }
        if (residuals) std::copy(g.sep.residuals.begin(), g.sep.residuals.end(), residuals);
        if (sweeps) *sweeps = g.sep.sweeps;
    });
}

}  // extern "C"

namespace {
// Dense mode-product candidates; STIGA_DENSE_KERNEL=res / stream restricts them to the resident /
// streaming kernels (tests), unset: both kinds go to the autotuner.
std::vector<gpu::Tiling> dense_candidates(int m, int n) {
    std::vector<gpu::Tiling> c = gpu::mode_tiling_candidates(m, n);
    const char* k = std::getenv("STIGA_DENSE_KERNEL");
    if (k && (std::string(k) == "res" || std::string(k) == "stream")) {
        const bool want_res = std::string(k) == "res";
        std::vector<gpu::Tiling> f;
        for (const auto& t : c)
            if ((t.res != 0) == want_res) f.push_back(t);
        if (!f.empty()) c = f;
    }
    return c;
}
}  // namespace

namespace stiga {
// Host setup (fdsolve.cpp:67-153) + device upload + autotune of an FD handle.  `prepare` (sharded
// handles, dist.cpp) runs after the host setup and before the uploads: it sets the stage spans, the
// shard state and the D^-1/2 slab.
stiga_fd_s* fd_build(int d, const int* n, const double* const* K, const double* const* M, int n_t, const double* Wt,
                     const double* Mt, double gamma, double nu, const double* scaling, long long scaling_len,
                     int device, const std::function<void(stiga_fd_s&)>& prepare, int flags,
                     const double* d_scaling) {
        require(d >= 1 && d <= gpu::kMaxDim, "ExtendedFDPreconditioner: per-direction matrices mismatch");
        require((flags & ~(STIGA_SETUP_DEVICE_SCHUR | STIGA_SETUP_CUSOLVER)) == 0, "stiga_fd_setup_ex: unknown flags");
        const bool dev_schur = (flags & STIGA_SETUP_DEVICE_SCHUR) && device >= 0;
        const bool use_cusolver = (flags & STIGA_SETUP_CUSOLVER) != 0;
        require(!use_cusolver || device >= 0, "stiga_fd_setup_ex: the cuSOLVER eigensolver needs a device");
        require(!(scaling && d_scaling), "stiga_fd_setup_ex: host and device scaling both given");
        require(!d_scaling || (device >= 0 && !prepare), "stiga_fd_setup_ex: device scaling needs an unsharded device handle");
        require(n && K && M && Wt && Mt, "stiga_fd_setup: null input");
        require(n_t >= 1, "time_factorization: shape mismatch");
        std::vector<DenseMatrix> Ks, Ms;
        long long n_s = 1;
        for (int l = 0; l < d; ++l) {
            require(n[l] >= 1 && K[l] && M[l], "spd_generalized_eig: shape mismatch");
            Ks.push_back(from_colmajor(K[l], n[l]));
            Ms.push_back(from_colmajor(M[l], n[l]));
            n_s *= n[l];
        }
        if (scaling || d_scaling)
            require(scaling_len == n_s * n_t, "ExtendedFDPreconditioner: scaling vector length mismatch");
        auto h = std::make_unique<stiga_fd_s>();
        {
            std::unique_ptr<DeviceGuard> eg;
            std::unique_ptr<ScopedSymEig> se;
            if (use_cusolver) {  // every sym_eig of this setup (pencils, split halves, time embedding)
                eg.reset(new DeviceGuard(device));
                se.reset(new ScopedSymEig(&sym_eig_cusolver));
            }
            h->F = fd_setup(Ks, Ms, from_colmajor(Wt, n_t), from_colmajor(Mt, n_t), gamma, nu, scaling, !dev_schur);
        }
        const FDFactors& F = h->F;
        h->device = device;
        h->d = d;
        h->dims.assign(F.n.begin(), F.n.end());
        h->dims.push_back(F.n_t);
        h->n_dof = F.n_dof;
        h->n_s = F.n_s_total;
        h->nt_span = F.n_t;
        h->ns_span = F.n_s_total;
        h->scratch_len = F.n_dof;
        if (device < 0) return h.release();  // host-only handle: setup + export, no device resources

        DeviceGuard dg(device);
        if (prepare) prepare(*h);
        for (int l = 0; l < d; ++l) {
            std::vector<gpu::Tiling> dense = dense_candidates(F.n[l], F.n[l]);
            if (dense.empty()) throw std::runtime_error("internal: no mode-product tiling");
            int rows = 0;
            for (const auto& t : dense) rows = std::max(rows, t.Mp);
            const DenseMatrix Ud = F.U_dev(l);  // device eigen-order (folded order for a split direction)
            h->Jt.emplace_back(new DBuf);
            h->J.emplace_back(new DBuf);
            h->Jt.back()->upload(pad_factor(Ud, true, rows, dense.front().Kp));
            h->J.back()->upload(pad_factor(Ud, false, rows, dense.front().Kp));
            h->Jft.emplace_back(new DBuf);
            h->Jfb.emplace_back(new DBuf);
            std::vector<gpu::Tiling> cands;
            // STIGA_FOLD_KERNEL=off: dense kernels only; =force: folded kernels only (split directions);
            // unset: both kinds are candidates of the setup-time autotuner
            const char* fk = std::getenv("STIGA_FOLD_KERNEL");
            const bool dense_only = fk && std::string(fk) == "off";
            const bool fold_only = fk && (std::string(fk) == "force" || std::string(fk) == "force_wm2" ||
                                          std::string(fk) == "res" || std::string(fk) == "stream");
            const bool fold_wm2 = fk && std::string(fk) == "force_wm2";  // tests: folded WM = 2 tilings only
            const bool fold_res = fk && std::string(fk) == "res";        // tests: resident-factor kernel only
            const bool fold_stream = fk && std::string(fk) == "stream";  // tests: streaming folded kernels only
            if (F.fold[l].on && !dense_only) {  // folded candidates first (half the FLOPs)
                std::vector<gpu::Tiling> fc = gpu::fold_tiling_candidates(F.n[l]);
                if (fold_wm2) fc.erase(std::remove_if(fc.begin(), fc.end(), [](const gpu::Tiling& t) { return t.WM != 2 || t.fold != 1; }),
                                       fc.end());
                if (fold_res) fc.erase(std::remove_if(fc.begin(), fc.end(), [](const gpu::Tiling& t) { return t.fold != 2; }),
                                       fc.end());
                if (fold_stream) fc.erase(std::remove_if(fc.begin(), fc.end(), [](const gpu::Tiling& t) { return t.fold != 1; }),
                                          fc.end());
                int frows = 0;
                for (const auto& t : fc) frows = std::max(frows, t.Mp);
                for (auto& t : fc) t.Mp = frows;  // both matrices padded to the largest row-block cover
                if (!fc.empty()) {
                    h->Jft.back()->upload(fold_matrices(F.fold[l], true, frows, fc.front().Kp));
                    h->Jfb.back()->upload(fold_matrices(F.fold[l], false, frows, fc.front().Kp));
                }
                cands = fc;
            }
            if (!(fold_only && !cands.empty())) cands.insert(cands.end(), dense.begin(), dense.end());
            h->cand_space.push_back(cands);
            // WM = 1 dense tiling: the fallback for the scatter / pre-scale stages when the chosen tiling
            // has no such epilogue (folded WM = 2 tilings carry their own scatter epilogue)
            gpu::Tiling tdense = dense.front();
            for (const auto& t : dense)
                if (t.WM == 1 && !t.res) {
                    tdense = t;
                    break;
                }
            h->tl_dense.push_back(tdense);
            h->tl_b.push_back(cands.front());
            h->tl.push_back(cands.front());
            h->lam.emplace_back(new DBuf);
            h->lam.back()->upload(F.lambda_dev(l));
        }
        h->cand_time = gpu::time_tiling_candidates(F.n_t);
        if (const char* tk = std::getenv("STIGA_TIME_KERNEL")) {  // tests: res / stream time-fused kernels only
            const bool want_res = std::string(tk) == "res";
            std::vector<gpu::Tiling> f;
            for (const auto& t : h->cand_time)
                if ((t.res == 2) == want_res) f.push_back(t);
            if (!f.empty()) h->cand_time = f;
        }
        h->cand_ts = dense_candidates(F.n_t, F.n_t);
        if (h->cand_ts.empty()) throw std::runtime_error("internal: no time-product tiling");
        int trows = 0;
        for (const auto& t : h->cand_time) trows = std::max(trows, t.Mp);
        for (const auto& t : h->cand_ts) trows = std::max(trows, t.Mp);
        const int tKp = h->cand_ts.front().Kp;
        h->Jt_t.upload(pad_factor(F.time.U, true, trows, tKp));
        h->J_t.upload(pad_factor(F.time.U, false, trows, tKp));
        if (dev_schur) {  // Lambda_s and S^-1 on the device, bit-identical to the host loop (fdsolve.cpp:91-136)
            gpu::SchurArgs sa;
            sa.d = d;
            for (int l = 0; l < d; ++l) {
                sa.n[l] = F.n[l];
                sa.lam[l] = h->lam[l]->p;  // device (fiber) order: S^-1 comes out in the device order
            }
            const int np = static_cast<int>(F.time.lambda.size());
            std::vector<double> pcs(4 * std::max(np, 1), 0.0);
            for (int j = 0; j < np; ++j) {
                const double lam = F.time.lambda[j];
                const double c1 = gamma / nu * lam;
                pcs[4 * j] = gamma * gamma / nu * lam * lam;
                pcs[4 * j + 1] = c1 * c1 / nu;
                pcs[4 * j + 2] = F.time.g[2 * j] * F.time.g[2 * j];
                pcs[4 * j + 3] = F.time.g[2 * j + 1] * F.time.g[2 * j + 1];
            }
            DBuf dpc;
            dpc.upload(pcs);
            sa.npairs = np;
            sa.pc = dpc.p;
            sa.gs = gamma * F.time.sigma;
            sa.nu = nu;
            sa.gg = gamma * gamma;
            if (F.time.zero_count) {
                const double gz = F.time.g[F.n_t - 2];
                sa.cz = gamma * gamma * gz * gz / nu;
                sa.zero_block = 1;
            }
            h->S_inv.alloc(static_cast<size_t>(F.n_s_total));
            int* flag = nullptr;
            ck(cudaMalloc(&flag, sizeof(int)), "cudaMalloc");
            std::unique_ptr<int, decltype(&cudaFree)> fg(flag, &cudaFree);
            ck(cudaMemset(flag, 0, sizeof(int)), "memset");
            ck(gpu::launch_schur_inv(sa, F.n_s_total, h->S_inv.p, flag, nullptr), "device Schur diagonal");
            int hf = 0;
            ck(cudaMemcpy(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost), "download");
            if (hf & 1)
                throw std::runtime_error("ExtendedFDPreconditioner: spatial eigenvalues not positive "
                                         "(stiffness pencil not positive definite)");
            if (hf & 2) throw std::runtime_error("ExtendedFDPreconditioner: singular Schur complement");
            h->schur_on_device = true;
        } else {
            h->S_inv.upload(F.S_inv_dev());
        }
        std::vector<double> pc, pc1, pc1sq, pgg;
        for (size_t j = 0; j < F.time.lambda.size(); ++j) {
            const double lam = F.time.lambda[j];
            pc.push_back(gamma * gamma / nu * lam * lam);  // fdsolve.cpp:118
            const double c1 = gamma / nu * lam;            // fdsolve.cpp:16
            pc1.push_back(c1);
            pc1sq.push_back(c1 * c1 / nu);                 // fdsolve.cpp:17 (exact only at nu = 1)
            pgg.push_back(gamma * F.time.g[2 * j]);        // fdsolve.cpp:57-58
            pgg.push_back(gamma * F.time.g[2 * j + 1]);
        }
        if (pc.empty()) {
            pc.push_back(0.0);
            pc1.push_back(0.0);
            pc1sq.push_back(0.0);
            pgg.assign(2, 0.0);
        }
        h->pair_c.upload(pc);
        h->pair_c1.upload(pc1);
        h->pair_c1sq.upload(pc1sq);
        h->pair_gg.upload(pgg);
        std::vector<double> gg(F.time.g.begin(), F.time.g.end());
        if (gg.empty()) gg.push_back(0.0);
        h->g.upload(gg);
        if (!F.d_inv_sqrt.empty()) {
            h->dinv.upload(F.d_inv_sqrt);
        } else if (d_scaling) {  // D on the device: D^-1/2 there too (fdsolve.cpp:145-151, same rounding)
            h->dinv.alloc(static_cast<size_t>(F.n_dof));
            int* flag = nullptr;
            ck(cudaMalloc(&flag, sizeof(int)), "cudaMalloc");
            std::unique_ptr<int, decltype(&cudaFree)> fg(flag, &cudaFree);
            ck(cudaMemset(flag, 0, sizeof(int)), "memset");
            ck(gpu::launch_dinv_sqrt(d_scaling, h->dinv.p, F.n_dof, flag, nullptr), "device D^-1/2");
            int hf = 0;
            ck(cudaMemcpy(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost), "download");
            if (hf) throw std::invalid_argument("ExtendedFDPreconditioner: scaling must be strictly positive");
        }
        h->scratch.alloc(static_cast<size_t>(h->scratch_len));

        gpu::ArrowParams& ap = h->ap;
        ap.d = d;
        for (int l = 0; l < d; ++l) {
            ap.n[l] = F.n[l];
            ap.lam[l] = h->lam[l]->p;
        }
        ap.S_inv = h->S_inv.p;
        ap.pair_c = h->pair_c.p;
        ap.pair_c1 = h->pair_c1.p;
        ap.pair_c1sq = h->pair_c1sq.p;
        ap.pair_gg = h->pair_gg.p;
        ap.g = h->g.p;
        ap.npairs = static_cast<int>(F.time.lambda.size());
        ap.zero_count = F.time.zero_count;
        ap.n_t = F.n_t;
        ap.gamma = gamma;
        ap.nu = nu;
        ap.inv_nu = 1.0 / nu;
        if (const char* dbg = std::getenv("STIGA_DEBUG_ARROW")) ap.debug = std::atoi(dbg);
        h->autotune();
        return h.release();
}
}  // namespace stiga

extern "C" {

int stiga_fd_setup(int d, const int* n, const double* const* K, const double* const* M, int n_t, const double* Wt,
                   const double* Mt, double gamma, double nu, const double* scaling, long long scaling_len, int device,
                   stiga_fd_t* out) {
    return guarded([&] {
        require(out != nullptr, "stiga_fd_setup: null handle output");
        *out = nullptr;
        *out = fd_build(d, n, K, M, n_t, Wt, Mt, gamma, nu, scaling, scaling_len, device, nullptr, 0, nullptr);
    });
}

int stiga_fd_setup_ex(int d, const int* n, const double* const* K, const double* const* M, int n_t, const double* Wt,
                      const double* Mt, double gamma, double nu, const double* scaling, long long scaling_len,
                      const stiga_fd_setup_options* opts, int device, stiga_fd_t* out) {
    return guarded([&] {
        require(out != nullptr, "stiga_fd_setup_ex: null handle output");
        *out = nullptr;
        const int flags = opts ? opts->flags : 0;
        const double* ds = opts ? opts->d_scaling : nullptr;
        *out = fd_build(d, n, K, M, n_t, Wt, Mt, gamma, nu, scaling, scaling_len, device, nullptr, flags, ds);
    });
}

int stiga_fd_destroy(stiga_fd_t P) {
    return guarded([&] {
        if (!P) return;
        if (P->device < 0) {
            delete P;
            return;
        }
        DeviceGuard dg(P->device);
        delete P;
    });
}

int stiga_fd_size(stiga_fd_t P, long long* n_dof) {
    return guarded([&] {
        require(P && n_dof, "stiga_fd_size: null argument");
        *n_dof = P->n_dof;
    });
}

int stiga_fd_dims(stiga_fd_t P, int* d, int* dims) {
    return guarded([&] {
        require(P && d, "stiga_fd_dims: null argument");
        *d = P->d;
        if (dims)
            for (int l = 0; l <= P->d; ++l) dims[l] = P->dims[l];
    });
}

int stiga_fd_time_info(stiga_fd_t P, int* npairs, int* zero_count, double* sigma, double* rho) {
    return guarded([&] {
        require(P != nullptr, "stiga_fd_time_info: null handle");
        if (npairs) *npairs = static_cast<int>(P->F.time.lambda.size());
        if (zero_count) *zero_count = P->F.time.zero_count;
        if (sigma) *sigma = P->F.time.sigma;
        if (rho) *rho = P->F.time.rho;
    });
}

int stiga_fd_export(stiga_fd_t P, int which, int l, double* out, long long out_len) {
    return guarded([&] {
        require(P && out, "stiga_fd_export: null argument");
        const FDFactors& F = P->F;
        const std::vector<double>* src = nullptr;
        std::vector<double> tmp;
        switch (which) {
            case 0: require(l >= 0 && l < F.d, "stiga_fd_export: direction out of range"); src = &F.U[l].a; break;
            case 1: require(l >= 0 && l < F.d, "stiga_fd_export: direction out of range"); src = &F.lambda[l]; break;
            case 2: src = &F.time.U.a; break;
            case 3: tmp = F.time.lambda; src = &tmp; break;
            case 4: src = &F.time.g; break;
            case 5:
                if (F.S_inv.empty() && P->schur_on_device) {  // device order -> the ascending (exported) order
                    DeviceGuard dg(P->device);
                    std::vector<double> dev(static_cast<size_t>(F.n_s_total));
                    ck(cudaMemcpy(dev.data(), P->S_inv.p, sizeof(double) * dev.size(), cudaMemcpyDeviceToHost),
                       "download");
                    tmp.assign(dev.size(), 0.0);
                    std::vector<Index> stride(F.d, 1);
                    for (int k = 1; k < F.d; ++k) stride[k] = stride[k - 1] * F.n[k - 1];
                    for (Index s = 0; s < static_cast<Index>(dev.size()); ++s) {
                        Index rem = s, sa = 0;
                        for (int k = 0; k < F.d; ++k) {
                            const Index f = rem % F.n[k];
                            rem /= F.n[k];
                            sa += stride[k] * (F.fold[k].on ? F.fold[k].dev_order[f] : f);
                        }
                        tmp[sa] = dev[s];
                    }
                    src = &tmp;
                } else {
                    src = &F.S_inv;
                }
                break;
            default: throw std::invalid_argument("stiga_fd_export: unknown factor id");
        }
        require(out_len >= static_cast<long long>(src->size()), "stiga_fd_export: output too small");
        std::copy(src->begin(), src->end(), out);
    });
}

int stiga_fd_apply(stiga_fd_t P, const double* d_r, double* d_s, void* stream) {
    return guarded([&] {
        require(P && d_r && d_s, "ExtendedFDPreconditioner::apply: null argument");
        require(P->device >= 0, "ExtendedFDPreconditioner::apply: host-only handle (setup with device < 0)");
        DeviceGuard dg(P->device);
        if (P->shard) fd_apply_sharded(*P, d_r, d_s, as_stream(stream), nullptr);
        else P->apply(d_r, d_s, as_stream(stream), nullptr);
    });
}

int stiga_fd_local(stiga_fd_t P, long long* t0, long long* nt_local, long long* offset, long long* len) {
    return guarded([&] {
        require(P != nullptr, "stiga_fd_local: null handle");
        const long long a = P->shard ? P->shard->t_off[P->shard->rank] : 0;
        const long long b = P->shard ? P->shard->t_len[P->shard->rank] : P->dims[P->d];
        if (t0) *t0 = a;
        if (nt_local) *nt_local = b;
        if (offset) *offset = P->n_s * a;
        if (len) *len = P->n_s * b;
    });
}

int stiga_fd_apply_profiled(stiga_fd_t P, const double* d_r, double* d_s, void* stream, float* pass_ms) {
    return guarded([&] {
        require(P && d_r && d_s && pass_ms, "stiga_fd_apply_profiled: null argument");
        require(P->device >= 0, "ExtendedFDPreconditioner::apply: host-only handle (setup with device < 0)");
        DeviceGuard dg(P->device);
        const int passes = P->launches();
        std::vector<cudaEvent_t> ev(passes + 1);
        for (auto& e : ev) ck(cudaEventCreate(&e), "cudaEventCreate");
        if (P->shard) fd_apply_sharded(*P, d_r, d_s, as_stream(stream), &ev);
        else P->apply(d_r, d_s, as_stream(stream), &ev);
        ck(cudaEventSynchronize(ev[passes]), "cudaEventSynchronize");
        for (int k = 0; k < passes; ++k) ck(cudaEventElapsedTime(&pass_ms[k], ev[k], ev[k + 1]), "elapsed");
        for (auto& e : ev) cudaEventDestroy(e);
    });
}

int stiga_fd_apply_space(stiga_fd_t P, int backward, long long t0, long long nt_local, const double* d_in,
                         double* d_out, void* stream) {
    return guarded([&] {
        require(P && d_in && d_out, "stiga_fd_apply_space: null argument");
        require(P->device >= 0, "stiga_fd_apply_space: host-only handle");
        require(!P->shard, "stiga_fd_apply_space: stage building blocks need a single-device handle");
        require(t0 >= 0 && nt_local >= 1 && t0 + nt_local <= P->dims[P->d], "stiga_fd_apply_space: time slab out of range");
        require(d_in != d_out, "stiga_fd_apply_space: input and output must not alias");
        DeviceGuard dg(P->device);
        P->apply_space(backward != 0, t0, nt_local, d_in, d_out, as_stream(stream));
    });
}

int stiga_fd_apply_time(stiga_fd_t P, long long s0, long long ns_local, const double* d_in, double* d_out,
                        void* stream) {
    return guarded([&] {
        require(P && d_in && d_out, "stiga_fd_apply_time: null argument");
        require(P->device >= 0, "stiga_fd_apply_time: host-only handle");
        require(!P->shard, "stiga_fd_apply_time: stage building blocks need a single-device handle");
        require(s0 >= 0 && ns_local >= 1 && s0 + ns_local <= P->n_s, "stiga_fd_apply_time: spatial slab out of range");
        require(d_in != d_out, "stiga_fd_apply_time: input and output must not alias");
        DeviceGuard dg(P->device);
        P->apply_time(s0, ns_local, d_in, d_out, as_stream(stream));
    });
}

namespace {
// Validates a C-ABI scatter descriptor against the stage it feeds and converts it.
gpu::Scatter to_scatter(const stiga_scatter_desc* d, bool by_time, long long a_extent, long long b_extent,
                        const char* who) {
    const std::string w(who);
    require(d != nullptr, (w + ": null scatter descriptor").c_str());
    require(d->world >= 1 && d->world <= STIGA_MAX_RANKS, (w + ": world must be 1..STIGA_MAX_RANKS").c_str());
    require((d->by_time != 0) == by_time, (w + ": scatter descriptor has the wrong owner coordinate").c_str());
    gpu::Scatter sc;
    sc.G = d->world;
    sc.by_time = by_time ? 1 : 0;
    sc.a_shift = d->a_shift;
    sc.b_shift = d->b_shift;
    require(d->offsets[0] == 0 && d->offsets[d->world] == (by_time ? b_extent : a_extent),
            (w + ": partition offsets must cover the owner coordinate exactly").c_str());
    for (int q = 0; q <= d->world; ++q) sc.off[q] = d->offsets[q];
    for (int q = 0; q < d->world; ++q) {
        require(d->offsets[q + 1] > d->offsets[q], (w + ": partition offsets must be increasing").c_str());
        require(d->dst[q] != nullptr && d->ld[q] >= 1, (w + ": null destination or bad leading dimension").c_str());
        require(d->a_shift >= 0 && d->b_shift >= 0, (w + ": negative shift").c_str());
        sc.ld[q] = d->ld[q];
        sc.ptr[q] = d->dst[q];
    }
    return sc;
}
}  // namespace

int stiga_fd_apply_space_scatter(stiga_fd_t P, long long t0, long long nt_local, const double* d_in,
                                 const stiga_scatter_desc* sc, void* stream) {
    return guarded([&] {
        require(P && d_in, "stiga_fd_apply_space_scatter: null argument");
        require(P->device >= 0, "stiga_fd_apply_space_scatter: host-only handle");
        require(!P->shard, "stiga_fd_apply_space_scatter: stage building blocks need a single-device handle");
        require(t0 >= 0 && nt_local >= 1 && t0 + nt_local <= P->dims[P->d],
                "stiga_fd_apply_space_scatter: time slab out of range");
        const gpu::Scatter s = to_scatter(sc, false, P->n_s, nt_local, "stiga_fd_apply_space_scatter");
        DeviceGuard dg(P->device);
        P->apply_space_scatter(t0, nt_local, d_in, s, as_stream(stream));
    });
}

int stiga_fd_apply_time_scatter(stiga_fd_t P, long long s0, long long ns_local, const double* d_in,
                                const stiga_scatter_desc* sc, void* stream) {
    return guarded([&] {
        require(P && d_in, "stiga_fd_apply_time_scatter: null argument");
        require(P->device >= 0, "stiga_fd_apply_time_scatter: host-only handle");
        require(!P->shard, "stiga_fd_apply_time_scatter: stage building blocks need a single-device handle");
        require(s0 >= 0 && ns_local >= 1 && s0 + ns_local <= P->n_s,
                "stiga_fd_apply_time_scatter: spatial slab out of range");
        const gpu::Scatter s = to_scatter(sc, true, ns_local, P->dims[P->d], "stiga_fd_apply_time_scatter");
        DeviceGuard dg(P->device);
        P->apply_time_scatter(s0, ns_local, d_in, s, as_stream(stream));
    });
}

int stiga_device_alloc(long long bytes, int device, void** d_ptr) {
    return guarded([&] {
        require(d_ptr != nullptr && bytes >= 0, "stiga_device_alloc: bad argument");
        *d_ptr = nullptr;
        DeviceGuard dg(device);
        if (bytes) ck(cudaMalloc(d_ptr, static_cast<size_t>(bytes)), "cudaMalloc");
    });
}

int stiga_device_free(void* d_ptr) {
    return guarded([&] {
        if (d_ptr) ck(cudaFree(d_ptr), "cudaFree");
    });
}

int stiga_ipc_handle(const void* d_ptr, void* handle_out) {
    return guarded([&] {
        require(d_ptr && handle_out, "stiga_ipc_handle: null argument");
        static_assert(sizeof(cudaIpcMemHandle_t) == STIGA_IPC_HANDLE_BYTES, "IPC handle size");
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)), "cudaIpcGetMemHandle");
        std::memcpy(handle_out, &h, sizeof(h));
    });
}

int stiga_ipc_open(const void* handle, int device, void** d_ptr) {
    return guarded([&] {
        require(handle && d_ptr, "stiga_ipc_open: null argument");
        DeviceGuard dg(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        ck(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

int stiga_ipc_close(void* d_ptr) {
    return guarded([&] {
        require(d_ptr != nullptr, "stiga_ipc_close: null argument");
        ck(cudaIpcCloseMemHandle(d_ptr), "cudaIpcCloseMemHandle");
    });
}

int stiga_copy_blocks(const double* d_src, long long src_ld, double* d_dst, long long dst_ld, long long rows,
                      long long cols, void* stream) {
    return guarded([&] {
        require(rows >= 0 && cols >= 0 && (rows == 0 || cols == 0 || (d_src && d_dst)), "stiga_copy_blocks: invalid argument");
        require(src_ld >= cols && dst_ld >= cols, "stiga_copy_blocks: leading dimension smaller than the row length");
        ck(gpu::launch_copy_blocks(d_src, src_ld, d_dst, dst_ld, rows, cols, as_stream(stream)), "copy_blocks");
    });
}

int stiga_fd_launch_info(stiga_fd_t P, int i, char* name, int name_len, double* flops) {
    return guarded([&] {
        require(P && name && name_len > 0 && flops, "stiga_fd_launch_info: null argument");
        const std::vector<std::pair<std::string, double>> L = P->launch_list();
        require(i >= 0 && i < static_cast<int>(L.size()), "stiga_fd_launch_info: launch index out of range");
        std::snprintf(name, static_cast<size_t>(name_len), "%s", L[i].first.c_str());
        *flops = L[i].second;
    });
}

int stiga_fd_launches(stiga_fd_t P, int* launches) {
    return guarded([&] {
        require(P && launches, "stiga_fd_launches: null argument");
        *launches = P->launches();
    });
}

int stiga_fd_apply_host(stiga_fd_t P, const double* h_r, double* h_s) {
    return guarded([&] {
        require(P && h_r && h_s, "ExtendedFDPreconditioner::apply: null argument");
        require(P->device >= 0, "ExtendedFDPreconditioner::apply: host-only handle (setup with device < 0)");
        DeviceGuard dg(P->device);
        // local slab for a sharded handle (collective), the whole vector otherwise
        const long long n = P->shard ? P->n_s * P->shard->t_len[P->shard->rank] : P->n_dof;
        DBuf in, out;
        in.alloc(static_cast<size_t>(n));
        out.alloc(static_cast<size_t>(n));
        ck(cudaMemcpy(in.p, h_r, sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
        if (P->shard) fd_apply_sharded(*P, in.p, out.p, nullptr, nullptr);
        else P->apply(in.p, out.p, nullptr, nullptr);
        ck(cudaMemcpy(h_s, out.p, sizeof(double) * n, cudaMemcpyDeviceToHost), "D2H");
    });
}

int stiga_kron_matvec(int D, const int* rows, const int* cols, const double* const* factors, const double* d_x,
                      double* d_y, int device, void* stream) {
    return guarded([&] {
        require(D >= 1 && rows && cols && factors && d_x && d_y, "kron_matvec: invalid argument");
        DeviceGuard dg(device);
        cudaStream_t st = as_stream(stream);
        std::vector<int> dims(cols, cols + D);
        long long n = 1;
        for (int l = 0; l < D; ++l) {
            require(rows[l] >= 1 && cols[l] >= 1, "kron_matvec: vector length does not match factor dimensions");
            n *= cols[l];
        }
        // intermediate buffers (the reference allocates a Tensor per mode product, kronop.cpp:56-59)
        DBuf tmp[2];
        const double* src = d_x;
        for (int l = 0; l < D; ++l) {
            const bool last = l == D - 1;
            long long L = 1;
            for (int k = 0; k < l; ++k) L *= dims[k];
            gpu::ModeGeom g;
            g.L = L;
            g.n = dims[l];
            g.m = rows[l];
            g.ncols = n / dims[l];
            const long long nout = g.ncols * g.m;
            double* dst = d_y;
            if (!last) {
                tmp[l % 2].alloc(static_cast<size_t>(nout));
                dst = tmp[l % 2].p;
            }
            DenseMatrix Fm(rows[l], cols[l]);
            std::memcpy(Fm.a.data(), factors[l], sizeof(double) * rows[l] * static_cast<size_t>(cols[l]));
            const gpu::Tiling t = gpu::choose_mode_tiling(rows[l], cols[l], false);
            DBuf Jp;
            Jp.upload(pad_factor(Fm, false, t.Mp, t.Kp));
            ck(gpu::launch_mode_product(t, g, src, dst, Jp.p, nullptr, st), "kron_matvec mode product");
            ck(cudaStreamSynchronize(st), "kron_matvec sync");
            dims[l] = rows[l];
            n = nout;
            src = dst;
        }
    });
}

int stiga_kronsum_create(int D, const int* dims, int nterms, const double* coeffs, const double* const* factors,
                         int device, stiga_kronsum_t* out) {
    return guarded([&] {
        require(out != nullptr, "stiga_kronsum_create: null handle output");
        *out = nullptr;
        require(D >= 1 && dims, "KronSumOperator: dimensions must be positive");
        require(nterms >= 0 && (nterms == 0 || (coeffs && factors)), "KronSumOperator: term factor count does not match dims");
        auto h = std::make_unique<stiga_kronsum_s>();
        h->device = device;
        h->D = D;
        h->n_dof = 1;
        for (int l = 0; l < D; ++l) {
            require(dims[l] >= 1, "KronSumOperator: dimensions must be positive");
            h->dims.push_back(dims[l]);
            h->n_dof *= dims[l];
        }
        DeviceGuard dg(device);
        for (int t = 0; t < nterms; ++t) {
            h->coeffs.push_back(coeffs[t]);
            h->factors.emplace_back();
            for (int l = 0; l < D; ++l) {
                require(factors[t * D + l] != nullptr, "KronSumOperator: factor shape does not match dims");
                DenseMatrix F = from_colmajor(factors[t * D + l], dims[l]);
                const int p = half_bandwidth(F);
                h->hbw.push_back(p);
                h->bands.emplace_back(new DBuf);
                h->bands.back()->upload(to_band(F, p, l == D - 1 ? coeffs[t] : 1.0));
                h->factors.back().push_back(std::move(F));
            }
        }
        *out = h.release();
    });
}

}  // extern "C"

namespace stiga {
stiga_kronsum_s* ks_build_spacetime(int d, const int* n, const double* const* K, const double* const* M, int n_t,
                                    const double* Wt, const double* Mt, double gamma, double nu, int device) {
        require(d >= 1 && n && K && M && Wt && Mt && n_t >= 1, "KronSumOperator: dimensions must be positive");
        auto h = std::make_unique<stiga_kronsum_s>();
        h->device = device;
        h->D = d + 1;
        h->spacetime = true;
        h->n_dof = 1;
        for (int l = 0; l < d; ++l) {
            require(n[l] >= 1 && K[l] && M[l], "KronSumOperator: dimensions must be positive");
            h->dims.push_back(n[l]);
            h->n_dof *= n[l];
        }
        h->dims.push_back(n_t);
        h->n_dof *= n_t;
        DeviceGuard dg(device);
        // the kron_sum_terms structure (solver.cpp:10-30): terms [gamma; M_1..M_d, W_t] and
        // [nu; M_1..K_l..M_d, M_t]; kept as dense host factors for diagonal()
        std::vector<DenseMatrix> Kd, Md;
        for (int l = 0; l < d; ++l) {
            Kd.push_back(from_colmajor(K[l], n[l]));
            Md.push_back(from_colmajor(M[l], n[l]));
        }
        const DenseMatrix Wd = from_colmajor(Wt, n_t), Mtd = from_colmajor(Mt, n_t);
        h->coeffs.push_back(gamma);
        h->factors.emplace_back(Md);
        h->factors.back().push_back(Wd);
        for (int l = 0; l < d; ++l) {
            h->coeffs.push_back(nu);
            std::vector<DenseMatrix> fs;
            for (int k = 0; k < d; ++k) fs.push_back(k == l ? Kd[k] : Md[k]);
            fs.push_back(Mtd);
            h->factors.push_back(std::move(fs));
        }
        auto push = [&](const DenseMatrix& F, double c) {
            const int p = half_bandwidth(F);
            h->hbw.push_back(p);
            h->bands.emplace_back(new DBuf);
            h->bands.back()->upload(to_band(F, p, c));
        };
        for (int l = 0; l < d; ++l) {
            push(Md[l], 1.0);
            push(Kd[l], 1.0);
        }
        push(Wd, gamma);
        push(Mtd, nu);
        // fused mat-vec: widened spatial bands and the time band columns (cuda/matvec_fused.cu)
        int fp = 0;
        for (int hb : h->hbw) fp = std::max(fp, hb);
        fp = std::max(fp, 1);
        const bool plane_ok = d < 2 || (gpu::plane2_smem_bytes(n[0], fp) <= 227 * 1024 && (n[0] + 1) / 2 <= 256);
        if (fp <= gpu::kMaxFusedP && d <= 3 && plane_ok) {
            h->fp = fp;
            const int W = 2 * fp + 1;
            auto widened = [&](const DenseMatrix& F) {
                const int m = static_cast<int>(F.rows);
                std::vector<double> b(static_cast<size_t>(m) * W, 0.0);
                for (int i = 0; i < m; ++i)
                    for (int k = 0; k < W; ++k) {
                        const int j = i + k - fp;
                        if (j >= 0 && j < m) b[static_cast<size_t>(i) * W + k] = F(i, j);
                    }
                return b;
            };
            for (int l = 0; l < d; ++l) {
                h->wband.emplace_back(new DBuf);
                h->wband.back()->upload(widened(Md[l]));
                h->wband.emplace_back(new DBuf);
                h->wband.back()->upload(widened(Kd[l]));
            }
            auto columns = [&](const DenseMatrix& F, double c) {  // col[t' * W + (dd + fp)] = c F(t' + dd, t')
                std::vector<double> col(static_cast<size_t>(n_t) * W, 0.0);
                for (int tp = 0; tp < n_t; ++tp)
                    for (int dd = -fp; dd <= fp; ++dd)
                        if (tp + dd >= 0 && tp + dd < n_t) col[static_cast<size_t>(tp) * W + dd + fp] = c * F(tp + dd, tp);
                return col;
            };
            h->tcol_w.upload(columns(Wd, gamma));
            h->tcol_m.upload(columns(Mtd, nu));
        }
        return h.release();
}
}  // namespace stiga

extern "C" {

int stiga_kronsum_create_spacetime(int d, const int* n, const double* const* K, const double* const* M, int n_t,
                                   const double* Wt, const double* Mt, double gamma, double nu, int device,
                                   stiga_kronsum_t* out) {
    return guarded([&] {
        require(out != nullptr, "stiga_kronsum_create_spacetime: null handle output");
        *out = nullptr;
        *out = ks_build_spacetime(d, n, K, M, n_t, Wt, Mt, gamma, nu, device);
    });
}

}  // extern "C"

namespace stiga {
stiga_kronsum_s* ks_build_physical(stiga_problem_s* prob, int p, int n_el, int device) {
        const ProblemSpec& spec = prob->spec;
        const int d = spec.d;
        const SplineSpace1D space = SplineSpace1D::spatial(p, n_el);
        const int n = space.dim();
        auto h = std::make_unique<stiga_kronsum_s>();
        h->device = device;
        h->D = d + 1;
        h->physical = true;
        h->n_dof = 1;
        for (int l = 0; l < d; ++l) {
            h->dims.push_back(n);
            h->n_dof *= n;
        }
        DenseMatrix Wt, Mt;
        time_matrices(spec, p, n_el, Wt, Mt);
        h->dims.push_back(static_cast<int>(Wt.rows));
        h->n_dof *= Wt.rows;
        DeviceGuard dg(device);
        // time bands (W_t, M_t) for the banded time pass
        auto push = [&](const DenseMatrix& F) {
            const int hb = half_bandwidth(F);
            h->hbw.push_back(hb);
            h->bands.emplace_back(new DBuf);
            h->bands.back()->upload(to_band(F, hb, 1.0));
        };
        push(Wt);
        push(Mt);
        for (Index i = 0; i < Wt.rows; ++i) {
            h->time_W.push_back(Wt(i, i));
            h->time_M.push_back(Mt(i, i));
        }
        // 1D quadrature tables (q = p + 1 Gauss points per element, solver.cpp:103)
        const int q = p + 1;
        const QuadratureRule quad = gauss_rule(space.knot_vector(), q);
        std::vector<double> nodes(quad.nodes), weights(quad.weights), bv, bd;
        std::vector<int> bf;
        std::vector<double> buf(p + 1);
        for (int qp = 0; qp < quad.num_points(); ++qp) {
            bf.push_back(space.eval_active(quad.nodes[qp], 0, buf.data()));
            bv.insert(bv.end(), buf.begin(), buf.end());
            space.eval_active(quad.nodes[qp], 1, buf.data());
            bd.insert(bd.end(), buf.begin(), buf.end());
        }
        h->qnode.upload(nodes);
        h->qweight.upload(weights);
        h->bval.upload(bv);
        h->bder.upload(bd);
        ck(cudaMalloc(&h->bfirst, sizeof(int) * bf.size()), "cudaMalloc");
        ck(cudaMemcpy(h->bfirst, bf.data(), sizeof(int) * bf.size(), cudaMemcpyHostToDevice), "upload");
        // geometry: uniform open knots of degree pg with neg elements, control points column-major
        const GeometryMap& F = spec.geometry;
        const KnotVector& kv0 = F.knot_vectors()[0];
        for (const KnotVector& kv : F.knot_vectors()) {
            const KnotVector u = KnotVector::uniform_open(kv.degree(), kv.num_elements());
            require(kv.knots() == u.knots(), "stiga_kronsum_create_physical: geometry needs uniform open knot vectors");
            require(kv.degree() == kv0.degree() && kv.num_elements() == kv0.num_elements(),
                    "stiga_kronsum_create_physical: geometry knot vectors must agree across directions");
        }
        h->cp.upload(F.control_points().a);
        gpu::PhysicalDesc& g = h->pdesc;
        g.d = d;
        g.p = p;
        g.q = q;
        g.n_el = n_el;
        g.n = n;
        g.pg = kv0.degree();
        g.neg = kv0.num_elements();
        g.cp = h->cp.p;
        g.ncp = F.control_points().rows;
        problem_field_kinds(spec, g.nu_kind, g.gamma_kind);
        g.qnode = h->qnode.p;
        g.qweight = h->qweight.p;
        g.bval = h->bval.p;
        g.bder = h->bder.p;
        g.bfirst = h->bfirst;
        long long S = 1;
        for (int l = 0; l < d; ++l) S *= 2 * p + 1;
        const long long Ns = h->n_dof / h->dims[d];
        h->Kst.alloc(static_cast<size_t>(Ns * S));
        h->Mst.alloc(static_cast<size_t>(Ns * S));
        ck(cudaMemset(h->Kst.p, 0, sizeof(double) * Ns * S), "memset");
        ck(cudaMemset(h->Mst.p, 0, sizeof(double) * Ns * S), "memset");
        ck(gpu::launch_physical_assembly(g, h->Kst.p, h->Mst.p, nullptr), "physical assembly");
        ck(cudaDeviceSynchronize(), "physical assembly");
        return h.release();
}
}  // namespace stiga

extern "C" {

int stiga_kronsum_create_physical(stiga_problem_t prob, int p, int n_el, int device, stiga_kronsum_t* out) {
    return guarded([&] {
        require(prob && out, "stiga_kronsum_create_physical: null argument");
        *out = nullptr;
        *out = ks_build_physical(prob, p, n_el, device);
    });
}

int stiga_kronsum_destroy(stiga_kronsum_t A) {
    return guarded([&] {
        if (!A) return;
        DeviceGuard dg(A->device);
        delete A;
    });
}

int stiga_kronsum_size(stiga_kronsum_t A, long long* n_dof) {
    return guarded([&] {
        require(A && n_dof, "stiga_kronsum_size: null argument");
        *n_dof = A->n_dof;
    });
}

int stiga_kronsum_dims(stiga_kronsum_t A, int* D, int* dims, int cap) {
    return guarded([&] {
        require(A && D && dims, "stiga_kronsum_dims: null argument");
        require(cap >= A->D, "stiga_kronsum_dims: capacity too small");
        *D = A->D;
        for (int l = 0; l < A->D; ++l) dims[l] = A->dims[l];
    });
}

int stiga_kronsum_apply(stiga_kronsum_t A, const double* d_x, double* d_y, void* stream) {
    return guarded([&] {
        require(A && d_x && d_y, "KronSumOperator::apply: vector length mismatch");
        require(d_x != d_y, "KronSumOperator::apply: input and output must not alias");
        DeviceGuard dg(A->device);
        if (A->kshard) kronsum_apply_sharded(*A, d_x, d_y, as_stream(stream));
        else A->apply(d_x, d_y, as_stream(stream));
    });
}

int stiga_kronsum_local(stiga_kronsum_t A, long long* t0, long long* nt_local, long long* offset, long long* len) {
    return guarded([&] {
        require(A != nullptr, "stiga_kronsum_local: null handle");
        const int nt = A->dims[A->D - 1];
        const long long Ns = A->n_dof / nt;
        const long long a = A->kshard ? A->kshard->t_off[A->kshard->rank] : 0;
        const long long b = A->kshard ? A->kshard->t_len[A->kshard->rank] : nt;
        if (t0) *t0 = a;
        if (nt_local) *nt_local = b;
        if (offset) *offset = Ns * a;
        if (len) *len = Ns * b;
    });
}

int stiga_kronsum_time_halfband(stiga_kronsum_t A, int* p) {
    return guarded([&] {
        require(A && p, "stiga_kronsum_time_halfband: null argument");
        require(A->physical || A->spacetime, "stiga_kronsum_time_halfband: needs a spacetime or physical operator");
        const int d = A->D - 1;
        *p = A->physical ? std::max(A->hbw[0], A->hbw[1]) : std::max(A->hbw[2 * d], A->hbw[2 * d + 1]);
    });
}

int stiga_kronsum_apply_space(stiga_kronsum_t A, long long nt_local, const double* d_x, double* d_a, double* d_b,
                              void* stream) {
    return guarded([&] {
        require(A && d_x && d_a && d_b, "stiga_kronsum_apply_space: null argument");
        require(A->physical || A->spacetime, "stiga_kronsum_apply_space: needs a spacetime or physical operator");
        const int d = A->D - 1;
        require(nt_local >= 0 && nt_local <= A->dims[d], "stiga_kronsum_apply_space: slab larger than n_t");
        require(d_x != d_a && d_x != d_b && d_a != d_b, "stiga_kronsum_apply_space: buffers must not alias");
        if (nt_local == 0) return;
        DeviceGuard dg(A->device);
        A->apply_space_slab(nt_local, d_x, d_a, d_b, as_stream(stream));
    });
}

int stiga_kronsum_apply_time(stiga_kronsum_t A, long long t0, long long nt_local, int halo_lo, int halo_hi,
                             const double* d_a, const double* d_b, double* d_y, void* stream) {
    return guarded([&] {
        require(A && d_a && d_b && d_y, "stiga_kronsum_apply_time: null argument");
        require(A->physical || A->spacetime, "stiga_kronsum_apply_time: needs a spacetime or physical operator");
        const int d = A->D - 1;
        const int nt = A->dims[d];
        require(t0 >= 0 && nt_local >= 0 && t0 + nt_local <= nt, "stiga_kronsum_apply_time: slab outside [0, n_t)");
        const int ia = A->physical ? 0 : 2 * d, ib = ia + 1;
        const int p = std::max(A->hbw[ia], A->hbw[ib]);
        require(halo_lo == std::min<long long>(p, t0) && halo_hi == std::min<long long>(p, nt - t0 - nt_local),
                "stiga_kronsum_apply_time: halo widths must be min(p, slices that exist)");
        require(d_y != d_a && d_y != d_b, "stiga_kronsum_apply_time: output must not alias the inputs");
        if (nt_local == 0) return;
        DeviceGuard dg(A->device);
        const long long Ns = A->n_dof / nt;
        ck(gpu::launch_time_band_slab(Ns, nt, t0, nt_local, halo_lo, d_a, d_b, d_y, A->band(ia), A->band(ib),
                                      as_stream(stream)),
           "time band slab");
    });
}

int stiga_vec_dot(const double* d_x, const double* d_y, long long n, double* d_result, void* stream) {
    return guarded([&] {
        require(n >= 0 && d_result && (n == 0 || (d_x && d_y)), "stiga_vec_dot: invalid argument");
        cudaStream_t st = as_stream(stream);
        if (n == 0) {
            ck(cudaMemsetAsync(d_result, 0, sizeof(double), st), "memset");
            return;
        }
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        thread_local std::vector<std::unique_ptr<DBuf>> partials;  // per device of this host thread
        if (static_cast<int>(partials.size()) <= dev) partials.resize(dev + 1);
        if (!partials[dev]) {
            partials[dev] = std::make_unique<DBuf>();
            partials[dev]->alloc(static_cast<size_t>(gpu::dot_partials_size()));
        }
        ck(gpu::launch_dot(d_x, d_y, n, partials[dev]->p, d_result, st), "dot");
    });
}

int stiga_vec_multidot(const double* const* d_V, int k, const double* d_w, long long n, double* d_out, void* stream) {
    return guarded([&] {
        require(d_V && d_w && d_out && k >= 1 && k <= 64 && n >= 1, "stiga_vec_multidot: invalid argument");
        for (int j = 0; j < k; ++j) require(d_V[j] != nullptr, "stiga_vec_multidot: null basis vector");
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        thread_local std::vector<std::unique_ptr<DBuf>> partials;  // per device of this host thread
        if (static_cast<int>(partials.size()) <= dev) partials.resize(dev + 1);
        if (!partials[dev]) {
            partials[dev] = std::make_unique<DBuf>();
            partials[dev]->alloc(static_cast<size_t>(gpu::multidot_partials_size()));
        }
        ck(gpu::launch_multidot(d_V, k, d_w, n, partials[dev]->p, d_out, as_stream(stream)), "multidot");
    });
}

int stiga_vec_multiaxpy(const double* coefs, const double* const* d_V, int k, double* d_w, long long n, void* stream) {
    return guarded([&] {
        require(coefs && d_V && d_w && k >= 1 && k <= 64 && n >= 0, "stiga_vec_multiaxpy: invalid argument");
        for (int j = 0; j < k; ++j) require(d_V[j] != nullptr, "stiga_vec_multiaxpy: null basis vector");
        ck(gpu::launch_multiaxpy(coefs, d_V, k, d_w, n, as_stream(stream)), "multiaxpy");
    });
}

int stiga_vec_axpy(double alpha, const double* d_x, double* d_y, long long n, void* stream) {
    return guarded([&] {
        require(n >= 0 && (n == 0 || (d_x && d_y)), "stiga_vec_axpy: invalid argument");
        ck(gpu::launch_axpy(alpha, d_x, d_y, n, as_stream(stream)), "axpy");
    });
}

int stiga_vec_scal(double alpha, const double* d_x, double* d_y, long long n, void* stream) {
    return guarded([&] {
        require(n >= 0 && (n == 0 || (d_x && d_y)), "stiga_vec_scal: invalid argument");
        ck(gpu::launch_scal(alpha, d_x, d_y, n, as_stream(stream)), "scal");
    });
}

int stiga_kronsum_diagonal(stiga_kronsum_t A, double* h_diag) {
    return guarded([&] {
        require(A && h_diag, "KronSumOperator::diagonal: null argument");
        std::fill(h_diag, h_diag + A->n_dof, 0.0);
        if (A->physical) {  // diag(M_s) (x) diag(W_t) + diag(K_s) (x) diag(M_t)
            DeviceGuard dg(A->device);
            const int d = A->D - 1;
            const long long Ns = A->n_dof / A->dims[d];
            DBuf dK, dM;
            dK.alloc(static_cast<size_t>(Ns));
            dM.alloc(static_cast<size_t>(Ns));
            ck(gpu::launch_stencil_diag(A->pdesc, A->Kst.p, A->Mst.p, dK.p, dM.p, nullptr), "stencil diag");
            std::vector<double> hk(Ns), hm(Ns);
            ck(cudaMemcpy(hk.data(), dK.p, sizeof(double) * Ns, cudaMemcpyDeviceToHost), "D2H");
            ck(cudaMemcpy(hm.data(), dM.p, sizeof(double) * Ns, cudaMemcpyDeviceToHost), "D2H");
            for (int t = 0; t < A->dims[d]; ++t)
                for (long long i = 0; i < Ns; ++i)
                    h_diag[t * Ns + i] = hm[i] * A->time_W[t] + hk[i] * A->time_M[t];
            return;
        }
        // kronop.cpp:117-131: acc = kron(diag(F_D), ..., diag(F_1)), first factor fastest
        for (size_t t = 0; t < A->coeffs.size(); ++t) {
            std::vector<double> acc(1, 1.0);
            for (const DenseMatrix& F : A->factors[t]) {
                std::vector<double> next(acc.size() * F.rows);
                for (Index j = 0; j < F.rows; ++j)
                    for (size_t i = 0; i < acc.size(); ++i) next[j * acc.size() + i] = F(j, j) * acc[i];
                acc.swap(next);
            }
            for (long long i = 0; i < A->n_dof; ++i) h_diag[i] += A->coeffs[t] * acc[i];
        }
    });
}

}  // extern "C"

namespace {
// diag(A) on the device (kronop.cpp:117-131 / the physical A_ of solver.cpp:67-70), or num / diag(A)
// when num is set; same per-entry operation order as stiga_kronsum_diagonal (bit-identical).
void ks_diag_device(stiga_kronsum_s* A, const double* num, double* out, cudaStream_t st) {
    require(!A->kshard, "KronSumOperator::diagonal: sharded operator (use the slab's own diagonal)");
    if (A->physical) {
        const int d = A->D - 1;
        const long long Ns = A->n_dof / A->dims[d];
        DBuf dK, dM, W, M;
        dK.alloc(static_cast<size_t>(Ns));
        dM.alloc(static_cast<size_t>(Ns));
        ck(gpu::launch_stencil_diag(A->pdesc, A->Kst.p, A->Mst.p, dK.p, dM.p, st), "stencil diag");
        W.upload(A->time_W);
        M.upload(A->time_M);
        require(num == nullptr, "internal: physical diagonal as denominator");
        ck(gpu::launch_physical_diag(dM.p, dK.p, W.p, M.p, Ns, A->dims[d], nullptr, out, st), "physical diagonal");
        ck(cudaStreamSynchronize(st), "physical diagonal");
        return;
    }
    const int D = A->D, nt = static_cast<int>(A->coeffs.size());
    std::vector<std::unique_ptr<DBuf>> bufs;
    std::vector<const double*> ptrs;
    for (int t = 0; t < nt; ++t)
        for (const DenseMatrix& F : A->factors[t]) {
            std::vector<double> dg(static_cast<size_t>(F.rows));
            for (Index j = 0; j < F.rows; ++j) dg[j] = F(j, j);
            bufs.emplace_back(new DBuf);
            bufs.back()->upload(dg);
            ptrs.push_back(bufs.back()->p);
        }
    ck(gpu::launch_kron_diag(D, A->dims.data(), nt, A->coeffs.data(), ptrs.data(), num, out, A->n_dof, st),
       "Kronecker-sum diagonal");
    ck(cudaStreamSynchronize(st), "Kronecker-sum diagonal");
}
}  // namespace

extern "C" {

int stiga_kronsum_diagonal_device(stiga_kronsum_t A, double* d_diag, void* stream) {
    return guarded([&] {
        require(A && d_diag, "KronSumOperator::diagonal: null argument");
        DeviceGuard dg(A->device);
        ks_diag_device(A, nullptr, d_diag, as_stream(stream));
    });
}

int stiga_geometry_scaling_device(stiga_kronsum_t A, stiga_kronsum_t Atilde, double* d_D, void* stream) {
    return guarded([&] {
        require(A && Atilde && d_D, "geometry scaling: null argument");
        require(A->n_dof == Atilde->n_dof && A->device == Atilde->device, "geometry scaling: operator mismatch");
        require(!Atilde->physical, "geometry scaling: A~ must be in Kronecker-sum form");
        DeviceGuard dg(A->device);
        ks_diag_device(A, nullptr, d_D, as_stream(stream));       // diag(A)
        ks_diag_device(Atilde, d_D, d_D, as_stream(stream));      // / diag(A~)
    });
}

int stiga_fp64_peak(int device, double ms, double* tflops_dmma, double* tflops_dfma) {
    return guarded([&] {
        require(tflops_dmma && tflops_dfma, "stiga_fp64_peak: null output");
        DeviceGuard dg(device);
        ck(gpu::fp64_peak_probe(ms, tflops_dmma, tflops_dfma), "fp64 peak probe");
    });
}

}  // extern "C"
