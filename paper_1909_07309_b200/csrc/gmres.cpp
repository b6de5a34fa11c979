// Device-resident left-preconditioned GMRES (stiga_gmres in include/stiga_gpu.h).
// Host control flow mirrors /root/reference/proj/core/src/gmres.cpp:19-132 line by line
// (MGS Arnoldi, Givens rotations, breakdown test H(k+1,k) <= 1e-14*beta0 -> converged,
// max_krylov as a TOTAL iteration cap across restarts, x0 = 0).  All N_dof-sized work (operator
// applies, dots, axpys, norms) runs on the device; only the (m+1) x m Hessenberg and the Givens
// coefficients live on the host.  Krylov vectors are allocated lazily (the reference allocates
// all m+1 columns up front, gmres.cpp:66), so a solve converging in one iteration needs O(1) vectors.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "cuda/aux_kernels.cuh"
#include "stiga_gpu.h"

namespace stiga {
void set_last_error(const std::string& msg);  // capi.cpp
}

namespace {

struct GFail : std::runtime_error {
    using std::runtime_error::runtime_error;
};
void gck(cudaError_t e, const char* w) {
    if (e != cudaSuccess) throw GFail(std::string(w) + ": " + cudaGetErrorString(e));
}
void sck(int status, const char* w) {
    if (status != STIGA_OK) throw GFail(std::string(w) + ": " + stiga_last_error());
}

// Krylov / work vectors come from a per-thread pool keyed by (device, length): large cudaMalloc /
// cudaFree pairs on every solve cost tens of milliseconds and synchronize the device.
struct Pool {
    int device = -1;
    long long n = -1;
    std::vector<double*> free_list;
    ~Pool() {
        for (double* p : free_list) cudaFree(p);
    }
};
thread_local Pool g_pool;

struct Vec {
    double* p = nullptr;
    int dev = 0;
    long long n = 0;
    explicit Vec(long long n_) : n(n_) {
        gck(cudaGetDevice(&dev), "cudaGetDevice");
        if (g_pool.device != dev || g_pool.n != n) {
            for (double* q : g_pool.free_list) cudaFree(q);
            g_pool.free_list.clear();
            g_pool.device = dev;
            g_pool.n = n;
        }
        if (!g_pool.free_list.empty()) {
            p = g_pool.free_list.back();
            g_pool.free_list.pop_back();
        } else {
            gck(cudaMalloc(&p, sizeof(double) * std::max<long long>(n, 1)), "cudaMalloc");
        }
    }
    ~Vec() {  // back to the pool only if it still serves this (device, length)
        if (!p) return;
        if (g_pool.device == dev && g_pool.n == n) g_pool.free_list.push_back(p);
        else cudaFree(p);
    }
    Vec(const Vec&) = delete;
    Vec& operator=(const Vec&) = delete;
};

struct Ctx {
    cudaStream_t st;
    long long n;
    double* partials = nullptr;
    double* result = nullptr;
    double* host = nullptr;  // pinned
    Ctx(cudaStream_t s, long long n_) : st(s), n(n_) {
        gck(cudaMalloc(&partials, sizeof(double) * stiga::gpu::dot_partials_size()), "cudaMalloc");
        gck(cudaMalloc(&result, sizeof(double)), "cudaMalloc");
        gck(cudaMallocHost(&host, sizeof(double)), "cudaMallocHost");
    }
    ~Ctx() {
        release_h();
        cudaFree(partials);
        cudaFree(result);
        cudaFreeHost(host);
    }
    double dot(const double* x, const double* y) {
        gck(stiga::gpu::launch_dot(x, y, n, partials, result, st), "dot");
        gck(cudaMemcpyAsync(host, result, sizeof(double), cudaMemcpyDeviceToHost, st), "dot D2H");
        gck(cudaStreamSynchronize(st), "dot sync");
        return *host;
    }
    double norm(const double* x) { return std::sqrt(dot(x, x)); }
    // Arnoldi column k by modified Gram-Schmidt with the coefficients kept on the device
    // (gmres.cpp:78-83): h_0 = V_0.w; for i < k: w -= h_i V_i, h_{i+1} = V_{i+1}.w; w -= h_k V_k,
    // h_{k+1} = w.w.  Same operations and order as dot/axpy pairs (bit-identical), one fused pass
    // per step and one host read-back per column instead of k+2 synchronizing round trips.
    void mgs(const std::vector<const double*>& V, double* w, int k, double* h_out) {
        if (!hdev) {
            gck(cudaMalloc(&hdev, sizeof(double) * hcap), "cudaMalloc");
            gck(cudaMallocHost(&hhost, sizeof(double) * hcap), "cudaMallocHost");
        }
        if (k + 2 > hcap) throw std::invalid_argument("gmres: Krylov column beyond the coefficient buffer");
        gck(stiga::gpu::launch_dot(V[0], w, n, partials, hdev, st), "dot");
        for (int i = 0; i <= k; ++i)
            gck(stiga::gpu::launch_axpy_dot(hdev + i, V[i], w, i < k ? V[i + 1] : nullptr, n, partials, hdev + i + 1, st),
                "axpy_dot");
        gck(cudaMemcpyAsync(hhost, hdev, sizeof(double) * (k + 2), cudaMemcpyDeviceToHost, st), "mgs D2H");
        gck(cudaStreamSynchronize(st), "mgs sync");
        for (int i = 0; i < k + 2; ++i) h_out[i] = hhost[i];
    }
    int hcap = 0;
    double* hdev = nullptr;
    double* hhost = nullptr;
    void release_h() {
        if (hdev) cudaFree(hdev);
        if (hhost) cudaFreeHost(hhost);
        hdev = hhost = nullptr;
    }
};

}  // namespace

extern "C" int stiga_gmres(stiga_kronsum_t A, stiga_fd_t P, const double* d_b, double* d_x,
                           const stiga_gmres_options* opts, stiga_gmres_report* report, void* stream) {
    try {
        if (!A || !d_b || !d_x || !opts || !report) throw std::invalid_argument("gmres: null argument");
        if (opts->tol <= 0.0) throw std::invalid_argument("gmres: tolerance must be positive");
        if (opts->max_krylov < 1) throw std::invalid_argument("gmres: max_krylov must be >= 1");
        const bool has_restart = opts->restart > 0;
        long long n = 0;
        sck(stiga_kronsum_size(A, &n), "gmres");
        if (P) {
            long long np = 0;
            sck(stiga_fd_size(P, &np), "gmres");
            if (np != n) throw std::invalid_argument("gmres: operator and preconditioner dimensions differ");
        }
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        Ctx ctx(st, n);
        ctx.hcap = (has_restart ? std::min(opts->restart, opts->max_krylov) : opts->max_krylov) + 2;
        using Clock = std::chrono::steady_clock;
        const auto t_start = Clock::now();
        double precond_ms = 0.0;
        cudaEvent_t pe0, pe1;
        gck(cudaEventCreate(&pe0), "event");
        gck(cudaEventCreate(&pe1), "event");
        auto apply_P = [&](const double* v, double* out) {  // out = P v  (or copy)
            if (!P) {
                gck(cudaMemcpyAsync(out, v, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
                return;
            }
            gck(cudaEventRecord(pe0, st), "event");
            sck(stiga_fd_apply(P, v, out, st), "gmres: preconditioner");
            gck(cudaEventRecord(pe1, st), "event");
            gck(cudaEventSynchronize(pe1), "event sync");
            float ms = 0.f;
            gck(cudaEventElapsedTime(&ms, pe0, pe1), "elapsed");
            precond_ms += ms;
        };
        auto apply_A = [&](const double* v, double* out) { sck(stiga_kronsum_apply(A, v, out, st), "gmres: operator"); };

        std::vector<double> hist;
        gck(cudaMemsetAsync(d_x, 0, sizeof(double) * n, st), "memset");
        Vec z(n), w(n), tmp(n);
        apply_P(d_b, z.p);  // z0 = P b
        const double beta0 = ctx.norm(z.p);
        hist.push_back(1.0);
        int total = 0;
        bool converged = false;
        if (beta0 == 0.0) {
            converged = true;
            hist.back() = 0.0;
        } else {
            const int cycle = has_restart ? std::min(opts->restart, opts->max_krylov) : opts->max_krylov;
            bool done = false;
            std::vector<std::unique_ptr<Vec>> V;
            while (!done && total < opts->max_krylov) {
                double beta;
                if (total == 0) {
                    beta = beta0;
                } else {  // z = P(b - A x)  (gmres.cpp:58)
                    apply_A(d_x, tmp.p);
                    gck(stiga::gpu::launch_sub(d_b, tmp.p, w.p, n, st), "sub");
                    apply_P(w.p, z.p);
                    beta = ctx.norm(z.p);
                }
                if (beta / beta0 <= opts->tol) {
                    converged = true;
                    break;
                }
                const int m = std::min(cycle, opts->max_krylov - total);
                std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0);  // column-major (m+1) x m
                auto Hk = [&](int i, int k) -> double& { return H[static_cast<size_t>(k) * (m + 1) + i]; };
                std::vector<double> cs(m), sn(m), gv(m + 1, 0.0);
                gv[0] = beta;
                if (V.empty()) V.emplace_back(new Vec(n));
                gck(stiga::gpu::launch_scal(1.0 / beta, z.p, V[0]->p, n, st), "scal");
                int k = 0;
                for (; k < m; ++k) {
                    apply_A(V[k]->p, tmp.p);
                    apply_P(tmp.p, w.p);  // w = P(A v_k)
                    std::vector<const double*> Vp(k + 1);
                    for (int i = 0; i <= k; ++i) Vp[i] = V[i]->p;
                    std::vector<double> hcol(k + 2);
                    ctx.mgs(Vp, w.p, k, hcol.data());  // modified Gram-Schmidt
                    for (int i = 0; i <= k; ++i) Hk(i, k) = hcol[i];
                    Hk(k + 1, k) = std::sqrt(hcol[k + 1]);
                    const bool tiny = Hk(k + 1, k) <= 1e-14 * beta0;
                    if (!tiny) {
                        if (static_cast<int>(V.size()) <= k + 1) V.emplace_back(new Vec(n));
                        gck(stiga::gpu::launch_scal(1.0 / Hk(k + 1, k), w.p, V[k + 1]->p, n, st), "scal");
                    }
                    for (int i = 0; i < k; ++i) {
                        const double t = cs[i] * Hk(i, k) + sn[i] * Hk(i + 1, k);
                        Hk(i + 1, k) = -sn[i] * Hk(i, k) + cs[i] * Hk(i + 1, k);
                        Hk(i, k) = t;
                    }
                    const double denom = std::hypot(Hk(k, k), Hk(k + 1, k));
                    cs[k] = Hk(k, k) / denom;
                    sn[k] = Hk(k + 1, k) / denom;
                    Hk(k, k) = denom;
                    Hk(k + 1, k) = 0.0;
                    gv[k + 1] = -sn[k] * gv[k];
                    gv[k] = cs[k] * gv[k];
                    ++total;
                    const double rel = std::abs(gv[k + 1]) / beta0;
                    hist.push_back(rel);
                    if (rel <= opts->tol || tiny) {
                        converged = true;
                        ++k;
                        done = true;
                        break;
                    }
                }
                if (k > 0) {  // y = H_k^-1 g (upper triangular), x += V y
                    std::vector<double> y(k);
                    for (int i = k - 1; i >= 0; --i) {
                        double s = gv[i];
                        for (int j = i + 1; j < k; ++j) s -= Hk(i, j) * y[j];
                        y[i] = s / Hk(i, i);
                    }
                    for (int i = 0; i < k; ++i)
                        gck(stiga::gpu::launch_axpy(y[i], V[i]->p, d_x, n, st), "axpy");
                }
                if (!has_restart && !done) break;
            }
        }
        gck(cudaStreamSynchronize(st), "gmres sync");
        cudaEventDestroy(pe0);
        cudaEventDestroy(pe1);
        const double wall = std::chrono::duration<double>(Clock::now() - t_start).count();
        report->iterations = total;
        report->converged = converged ? 1 : 0;
        report->wall_time_s = wall;
        report->precond_time_fraction = wall > 0.0 ? std::min(1.0, precond_ms * 1e-3 / wall) : 0.0;
        report->history_len = static_cast<int>(hist.size());
        if (report->residual_history)
            for (int i = 0; i < std::min(report->history_capacity, report->history_len); ++i)
                report->residual_history[i] = hist[i];
        stiga::set_last_error("");
        return STIGA_OK;
    } catch (const std::invalid_argument& e) {
        stiga::set_last_error(e.what());
        return STIGA_INVALID_ARGUMENT;
    } catch (const GFail& e) {
        stiga::set_last_error(e.what());
        return STIGA_CUDA;
    } catch (const std::exception& e) {
        stiga::set_last_error(e.what());
        return STIGA_NUMERICAL;
    }
}
