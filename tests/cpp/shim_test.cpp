// C++ consumer of the drop-in binding (include/stiga_b200.hpp over libstiga_gpu.so), as the reference's
// C++ would use it.  Built and run by tests/test_cpp_shim.py:
//   shim_test <dir>   reads <dir>/r.bin and <dir>/D.bin (c1 golden input, raw float64), writes
//                     <dir>/s.bin (unscaled apply), <dir>/s_scaled.bin (apply with D) and prints one JSON
//                     line with three GMRES solves: the library handles (stiga_gmres), the same operators
//                     as user callbacks (stiga_gmres_op), and a user-composed operator A + sigma I.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "stiga_b200.hpp"

using namespace stiga::b200;

static std::vector<double> read_bin(const std::string& path) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) throw std::runtime_error("cannot open " + path);
    const std::streamsize bytes = f.tellg();
    f.seekg(0);
    std::vector<double> v(bytes / sizeof(double));
    f.read(reinterpret_cast<char*>(v.data()), bytes);
    return v;
}
static void write_bin(const std::string& path, const std::vector<double>& v) {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(double));
}
static void cuck(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: shim_test <dir>\n");
        return 2;
    }
    const std::string dir = argv[1];
    try {
        // c1: d = 2, p = 2, n_el = 16 (BASELINE configs[0]); 1D factors on the host
        const int d = 2, p = 2, nel = 16;
        auto [Wt, Mt] = assemble_time_matrices(p, nel);
        auto [K1, M1] = assemble_spatial_parametric(p, nel);
        std::vector<Dense> K(d, K1), M(d, M1);
        const std::vector<double> r = read_bin(dir + "/r.bin");
        const std::vector<double> D = read_bin(dir + "/D.bin");

        // ExtendedFDPreconditioner::setup / apply (fdsolve.hpp:48-56), host convenience path
        Preconditioner P = Preconditioner::setup(K, M, Wt, Mt, 1.0, 1.0);
        write_bin(dir + "/s.bin", P.apply(r));
        Preconditioner PD = Preconditioner::setup(K, M, Wt, Mt, 1.0, 1.0, D);
        write_bin(dir + "/s_scaled.bin", PD.apply(r));
        bool threw = false;  // std::invalid_argument crosses the ABI as in the reference (fdsolve.cpp:156-157)
        try {
            P.apply(std::vector<double>(3, 1.0));
        } catch (const std::invalid_argument&) {
            threw = true;
        }

        // device-resident GMRES: b = r, A = kron_sum_terms(K, M, Wt, Mt, 1, 1), P = A^G with D
        const long long n = P.size();
        KronSumOperator A = KronSumOperator::spacetime(K, M, Wt, Mt, 1.0, 1.0);
        // a preconditioner for gamma = 0.4 makes the solve non-trivial (the exact one converges in 1)
        Preconditioner Pg = Preconditioner::setup(K, M, Wt, Mt, 0.4, 1.0);
        double *d_b = nullptr, *d_x = nullptr, *d_t = nullptr;
        cuck(cudaMalloc(&d_b, n * sizeof(double)));
        cuck(cudaMalloc(&d_x, n * sizeof(double)));
        cuck(cudaMalloc(&d_t, n * sizeof(double)));
        cuck(cudaMemcpy(d_b, r.data(), n * sizeof(double), cudaMemcpyHostToDevice));
        GmresOptions opts;
        opts.tol = 1e-8;
        opts.max_krylov = 200;
        opts.restart = 50;
        const SolveReport native = gmres(A, &Pg, d_b, d_x, opts);
        std::vector<double> x_native(n), x_cb(n), x_shift(n);
        cuck(cudaMemcpy(x_native.data(), d_x, n * sizeof(double), cudaMemcpyDeviceToHost));

        // the same solve with the operators as user callbacks (gmres.hpp:12 LinOp)
        DeviceLinOp Aop = [&](const double* x, double* y, cudaStream_t st) { A.apply_device(x, y, st); };
        DeviceLinOp Pop = [&](const double* x, double* y, cudaStream_t st) { Pg.apply_device(x, y, st); };
        const SolveReport cb = gmres(n, Aop, &Pop, d_b, d_x, opts);
        cuck(cudaMemcpy(x_cb.data(), d_x, n * sizeof(double), cudaMemcpyDeviceToHost));

        // a user-composed operator the library does not know: (A + sigma I) x
        const double sigma = 0.25;
        DeviceLinOp Ashift = [&](const double* x, double* y, cudaStream_t st) {
            A.apply_device(x, y, st);
            check(stiga_vec_axpy(sigma, x, y, n, st));
        };
        const SolveReport sh = gmres(n, Ashift, &Pop, d_b, d_x, opts);
        cuck(cudaMemcpy(x_shift.data(), d_x, n * sizeof(double), cudaMemcpyDeviceToHost));
        write_bin(dir + "/x_native.bin", x_native);
        write_bin(dir + "/x_cb.bin", x_cb);
        write_bin(dir + "/x_shift.bin", x_shift);
        double diff = 0.0, nrm = 0.0;
        for (long long i = 0; i < n; ++i) {
            diff += (x_native[i] - x_cb[i]) * (x_native[i] - x_cb[i]);
            nrm += x_native[i] * x_native[i];
        }
        // SpaceTimeSystem on a curved geometry (solver.cpp:34-155): the physical A_, A-hat-G with D formed on
        // the device, the device RHS, GMRES through the handles, compute_errors -- no host N_dof array
        Problem prob("quarter-annulus-2d");
        const int ps = 2, nels = 8;
        KronSumOperator Aphys = KronSumOperator::physical(prob, ps, nels);
        int nsd = 0, ntd = 0;
        check(stiga_space_dim(ps, nels, 0, &nsd));
        check(stiga_space_dim(ps, nels, 1, &ntd));
        const size_t nn = static_cast<size_t>(nsd) * nsd;
        std::vector<double> Kt(2 * nn), Mts(2 * nn);
        Dense Wg(ntd), Mg(ntd);
        check(stiga_geometry_preconditioner_pieces(prob.handle(), ps, nels, Kt.data(), Mts.data(), Wg.a.data(),
                                                   Mg.a.data(), nullptr, nullptr, nullptr, nullptr, nullptr));
        std::vector<Dense> Ks(2, Dense(nsd)), Ms(2, Dense(nsd));
        for (int l = 0; l < 2; ++l) {
            std::copy(Kt.begin() + l * nn, Kt.begin() + (l + 1) * nn, Ks[l].a.begin());
            std::copy(Mts.begin() + l * nn, Mts.begin() + (l + 1) * nn, Ms[l].a.begin());
        }
        KronSumOperator Atil = KronSumOperator::spacetime(Ks, Ms, Wg, Mg, 1.0, 1.0);
        const long long ns = Aphys.size();
        double *d_D = nullptr, *d_bs = nullptr, *d_xs = nullptr;
        cuck(cudaMalloc(&d_D, ns * sizeof(double)));
        cuck(cudaMalloc(&d_bs, ns * sizeof(double)));
        cuck(cudaMalloc(&d_xs, ns * sizeof(double)));
        geometry_scaling_device(Aphys, Atil, d_D);
        Preconditioner PG = Preconditioner::setup_device(Ks, Ms, Wg, Mg, 1.0, 1.0, d_D, ns);
        assemble_rhs(prob, ps, nels, d_bs);
        GmresOptions so;
        so.tol = 1e-10;
        so.max_krylov = 300;
        const SolveReport sys = gmres(Aphys, &PG, d_bs, d_xs, so);
        const Errors err = compute_errors(prob, ps, nels, d_xs, ps + 3);
        const auto means = system_means(prob, ps, nels);
        cudaFree(d_D);
        cudaFree(d_bs);
        cudaFree(d_xs);
        std::printf("{\"n\": %lld, \"invalid_argument\": %s, \"native_its\": %d, \"native_converged\": %s, "
                    "\"cb_its\": %d, \"cb_converged\": %s, \"cb_vs_native\": %.3e, \"shift_its\": %d, "
                    "\"shift_converged\": %s, \"sigma\": %.17g, \"sys_n\": %lld, \"sys_its\": %d, "
                    "\"sys_converged\": %s, \"err_l2l2\": %.17g, \"err_x\": %.17g, \"gamma_mean\": %.17g, "
                    "\"nu_mean\": %.17g}\n",
                    n, threw ? "true" : "false", native.iterations, native.converged ? "true" : "false",
                    cb.iterations, cb.converged ? "true" : "false", std::sqrt(diff / nrm), sh.iterations,
                    sh.converged ? "true" : "false", sigma, ns, sys.iterations, sys.converged ? "true" : "false",
                    err.l2l2, err.x_upper, means.first, means.second);
        cudaFree(d_b);
        cudaFree(d_x);
        cudaFree(d_t);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "shim_test: %s\n", e.what());
        return 1;
    }
    return 0;
}
