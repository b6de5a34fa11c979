// Device-resident left-preconditioned GMRES (stiga_gmres / stiga_gmres_op in include/stiga_gpu.h).
// Host control flow mirrors /root/reference/proj/core/src/gmres.cpp:19-132 line by line
// (Givens rotations, breakdown test H(k+1,k) <= 1e-14*beta0 -> converged, max_krylov as a TOTAL
// iteration cap across restarts, x0 = 0).  All N_dof-sized work (operator applies, dots, axpys,
// norms) runs on the device; only the (m+1) x m Hessenberg and the Givens coefficients live on the
// host.  Krylov vectors are allocated lazily (the reference allocates all m+1 columns up front,
// gmres.cpp:66), so a solve converging in one iteration needs O(1) vectors.
//
// Orthogonalisation: single-device solves use the reference's modified Gram-Schmidt (gmres.cpp:78-83)
// with the coefficients kept on the device; a solve over a communicator (time-sharded slabs) uses
// classical Gram-Schmidt with one reorthogonalisation (CGS2): two batched dot passes, each ONE
// all-reduce of the k+1 coefficients, instead of k+1 sequential reductions.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.hpp"
#include "cuda/aux_kernels.cuh"
#include "handles.hpp"
#include "stiga_gpu.h"

namespace stiga {
void comm_allreduce(stiga_comm_s* C, double* d_buf, long long n, cudaStream_t st);  // dist.cpp
}

using namespace stiga::capi;

namespace {

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
        ck(cudaGetDevice(&dev), "cudaGetDevice");
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
            ck(cudaMalloc(&p, sizeof(double) * std::max<long long>(n, 1)), "cudaMalloc");
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

constexpr int kMultiMax = 64;  // launch_multidot / launch_multiaxpy vectors per call

struct Ctx {
    cudaStream_t st;
    long long n;
    stiga_comm_s* comm;
    double* partials = nullptr;
    double* mpartials = nullptr;
    double* result = nullptr;
    double* host = nullptr;  // pinned
    int hcap = 0;
    double* hdev = nullptr;
    double* hhost = nullptr;
    Ctx(cudaStream_t s, long long n_, stiga_comm_s* c, int hcap_) : st(s), n(n_), comm(c), hcap(hcap_) {
        ck(cudaMalloc(&partials, sizeof(double) * stiga::gpu::dot_partials_size()), "cudaMalloc");
        ck(cudaMalloc(&result, sizeof(double)), "cudaMalloc");
        ck(cudaMallocHost(&host, sizeof(double)), "cudaMallocHost");
        ck(cudaMalloc(&hdev, sizeof(double) * hcap), "cudaMalloc");
        ck(cudaMallocHost(&hhost, sizeof(double) * hcap), "cudaMallocHost");
        if (comm) ck(cudaMalloc(&mpartials, sizeof(double) * stiga::gpu::multidot_partials_size()), "cudaMalloc");
    }
    ~Ctx() {
        cudaFree(partials);
        cudaFree(mpartials);
        cudaFree(result);
        cudaFreeHost(host);
        cudaFree(hdev);
        cudaFreeHost(hhost);
    }
    // global dot: local deterministic two-level reduction, all-reduced over the communicator
    double dot(const double* x, const double* y) {
        ck(stiga::gpu::launch_dot(x, y, n, partials, result, st), "dot");
        if (comm) stiga::comm_allreduce(comm, result, 1, st);
        ck(cudaMemcpyAsync(host, result, sizeof(double), cudaMemcpyDeviceToHost, st), "dot D2H");
        ck(cudaStreamSynchronize(st), "dot sync");
        return *host;
    }
    double norm(const double* x) { return std::sqrt(dot(x, x)); }
    // Arnoldi column k by modified Gram-Schmidt with the coefficients kept on the device
    // (gmres.cpp:78-83): h_0 = V_0.w; for i < k: w -= h_i V_i, h_{i+1} = V_{i+1}.w; w -= h_k V_k,
    // h_{k+1} = w.w.  Same operations and order as dot/axpy pairs (bit-identical), one fused pass
    // per step and one host read-back per column instead of k+2 synchronizing round trips.
    void mgs(const std::vector<const double*>& V, double* w, int k, double* h_out) {
        if (k + 2 > hcap) throw std::invalid_argument("gmres: Krylov column beyond the coefficient buffer");
        ck(stiga::gpu::launch_dot(V[0], w, n, partials, hdev, st), "dot");
        for (int i = 0; i <= k; ++i)
            ck(stiga::gpu::launch_axpy_dot(hdev + i, V[i], w, i < k ? V[i + 1] : nullptr, n, partials, hdev + i + 1, st),
               "axpy_dot");
        ck(cudaMemcpyAsync(hhost, hdev, sizeof(double) * (k + 2), cudaMemcpyDeviceToHost, st), "mgs D2H");
        ck(cudaStreamSynchronize(st), "mgs sync");
        for (int i = 0; i < k + 2; ++i) h_out[i] = hhost[i];
    }
    // h = V^T w over the communicator (chunks of 64 vectors into one device array, ONE all-reduce)
    void multidot(const std::vector<const double*>& V, const double* w, double* h) {
        const int k = static_cast<int>(V.size());
        if (k + 1 > hcap) throw std::invalid_argument("gmres: Krylov column beyond the coefficient buffer");
        for (int c0 = 0; c0 < k; c0 += kMultiMax) {
            const int kc = std::min(kMultiMax, k - c0);
            ck(stiga::gpu::launch_multidot(V.data() + c0, kc, w, n, mpartials, hdev + c0, st), "multidot");
        }
        if (comm) stiga::comm_allreduce(comm, hdev, k, st);
        ck(cudaMemcpyAsync(hhost, hdev, sizeof(double) * k, cudaMemcpyDeviceToHost, st), "multidot D2H");
        ck(cudaStreamSynchronize(st), "multidot sync");
        for (int i = 0; i < k; ++i) h[i] = hhost[i];
    }
    // w -= V h
    void multiaxpy_neg(const std::vector<const double*>& V, const std::vector<double>& h, double* w) {
        const int k = static_cast<int>(V.size());
        std::vector<double> c(k);
        for (int i = 0; i < k; ++i) c[i] = -h[i];
        for (int c0 = 0; c0 < k; c0 += kMultiMax) {
            const int kc = std::min(kMultiMax, k - c0);
            ck(stiga::gpu::launch_multiaxpy(c.data() + c0, V.data() + c0, kc, w, n, st), "multiaxpy");
        }
    }
    // Arnoldi column k by CGS2: h = V^T w, w -= V h, twice; h_out[0..k] = h1 + h2, h_out[k+1] = w.w
    void cgs2(const std::vector<const double*>& V, double* w, int k, double* h_out) {
        std::vector<double> h1(k + 1), h2(k + 1);
        multidot(V, w, h1.data());
        multiaxpy_neg(V, h1, w);
        multidot(V, w, h2.data());
        multiaxpy_neg(V, h2, w);
        for (int i = 0; i <= k; ++i) h_out[i] = h1[i] + h2[i];
        h_out[k + 1] = dot(w, w);
    }
};

// CUDA events around every preconditioner application, read once at the end of the solve (no host
// synchronization per application): precond_time_fraction of SolveReport (gmres.cpp:30-36, 127-130).
struct PrecondTimer {
    std::vector<cudaEvent_t> ev;
    size_t used = 0;
    ~PrecondTimer() {
        for (auto e : ev) cudaEventDestroy(e);
    }
    cudaEvent_t next() {
        if (used == ev.size()) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "event");
            ev.push_back(e);
        }
        return ev[used++];
    }
    double total_ms() {
        double ms = 0.0;
        for (size_t i = 0; i + 1 < used; i += 2) {
            float t = 0.f;
            ck(cudaEventElapsedTime(&t, ev[i], ev[i + 1]), "elapsed");
            ms += t;
        }
        return ms;
    }
};

using Op = std::function<void(const double*, double*)>;

void run_gmres(long long n, const Op& apply_A_raw, const Op* apply_P_raw, stiga_comm_s* comm, const double* d_b,
               double* d_x, const stiga_gmres_options* opts, stiga_gmres_report* report, cudaStream_t st) {
    if (!d_b || !d_x || !opts || !report) throw std::invalid_argument("gmres: null argument");
    if (opts->tol <= 0.0) throw std::invalid_argument("gmres: tolerance must be positive");
    if (opts->max_krylov < 1) throw std::invalid_argument("gmres: max_krylov must be >= 1");
    const bool has_restart = opts->restart > 0;
    const int cycle = has_restart ? std::min(opts->restart, opts->max_krylov) : opts->max_krylov;
    Ctx ctx(st, n, comm, cycle + 2);
    using Clock = std::chrono::steady_clock;
    const auto t_start = Clock::now();
    PrecondTimer ptimer;
    auto apply_P = [&](const double* v, double* out) {  // out = P v  (or copy)
        if (!apply_P_raw) {
            ck(cudaMemcpyAsync(out, v, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
            return;
        }
        ck(cudaEventRecord(ptimer.next(), st), "event");
        (*apply_P_raw)(v, out);
        ck(cudaEventRecord(ptimer.next(), st), "event");
    };
    const Op& apply_A = apply_A_raw;

    std::vector<double> hist;
    ck(cudaMemsetAsync(d_x, 0, sizeof(double) * n, st), "memset");
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
        bool done = false;
        std::vector<std::unique_ptr<Vec>> V;
        while (!done && total < opts->max_krylov) {
            double beta;
            if (total == 0) {
                beta = beta0;
            } else {  // z = P(b - A x)  (gmres.cpp:58)
                apply_A(d_x, tmp.p);
                ck(stiga::gpu::launch_sub(d_b, tmp.p, w.p, n, st), "sub");
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
            ck(stiga::gpu::launch_scal(1.0 / beta, z.p, V[0]->p, n, st), "scal");
            int k = 0;
            for (; k < m; ++k) {
                apply_A(V[k]->p, tmp.p);
                apply_P(tmp.p, w.p);  // w = P(A v_k)
                std::vector<const double*> Vp(k + 1);
                for (int i = 0; i <= k; ++i) Vp[i] = V[i]->p;
                std::vector<double> hcol(k + 2);
                if (comm) ctx.cgs2(Vp, w.p, k, hcol.data());
                else ctx.mgs(Vp, w.p, k, hcol.data());  // modified Gram-Schmidt (gmres.cpp:78-81)
                for (int i = 0; i <= k; ++i) Hk(i, k) = hcol[i];
                Hk(k + 1, k) = std::sqrt(std::max(hcol[k + 1], 0.0));
                const bool tiny = Hk(k + 1, k) <= 1e-14 * beta0;
                if (!tiny) {
                    if (static_cast<int>(V.size()) <= k + 1) V.emplace_back(new Vec(n));
                    ck(stiga::gpu::launch_scal(1.0 / Hk(k + 1, k), w.p, V[k + 1]->p, n, st), "scal");
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
                for (int i = 0; i < k; ++i) ck(stiga::gpu::launch_axpy(y[i], V[i]->p, d_x, n, st), "axpy");
            }
            if (!has_restart && !done) break;
        }
    }
    ck(cudaStreamSynchronize(st), "gmres sync");
    const double wall = std::chrono::duration<double>(Clock::now() - t_start).count();
    const double precond_ms = ptimer.total_ms();
    report->iterations = total;
    report->converged = converged ? 1 : 0;
    report->wall_time_s = wall;
    report->precond_time_fraction = wall > 0.0 ? std::min(1.0, precond_ms * 1e-3 / wall) : 0.0;
    report->history_len = static_cast<int>(hist.size());
    if (report->residual_history)
        for (int i = 0; i < std::min(report->history_capacity, report->history_len); ++i)
            report->residual_history[i] = hist[i];
}

void sck(int status, const char* w) {
    if (status != STIGA_OK) {
        const std::string msg = std::string(w) + ": " + stiga_last_error();
        if (status == STIGA_INVALID_ARGUMENT) throw std::invalid_argument(msg);
        if (status == STIGA_CUDA) throw CudaFailure(msg);
        throw std::runtime_error(msg);
    }
}

}  // namespace

extern "C" int stiga_gmres(stiga_kronsum_t A, stiga_fd_t P, const double* d_b, double* d_x,
                           const stiga_gmres_options* opts, stiga_gmres_report* report, void* stream) {
    return guarded([&] {
        if (!A) throw std::invalid_argument("gmres: null argument");
        long long n = A->n_local();
        stiga_comm_s* comm = A->kshard ? A->kshard->comm : nullptr;
        if (P) {
            long long np = 0, t0 = 0, ntl = 0, off = 0;
            sck(stiga_fd_local(P, &t0, &ntl, &off, &np), "gmres");
            if (np != n) throw std::invalid_argument("gmres: operator and preconditioner dimensions differ");
            stiga_comm_s* pc = P->shard ? P->shard->comm : nullptr;
            if (pc != comm) throw std::invalid_argument("gmres: operator and preconditioner are sharded differently");
        }
        cudaStream_t st = as_stream(stream);
        Op opA = [&](const double* v, double* out) { sck(stiga_kronsum_apply(A, v, out, st), "gmres: operator"); };
        Op opP = [&](const double* v, double* out) { sck(stiga_fd_apply(P, v, out, st), "gmres: preconditioner"); };
        DeviceGuard dg(A->device);
        run_gmres(n, opA, P ? &opP : nullptr, comm, d_b, d_x, opts, report, st);
    });
}

extern "C" int stiga_gmres_op(long long n, stiga_linop_fn A, void* A_ctx, stiga_linop_fn P, void* P_ctx,
                              stiga_comm_t comm, const double* d_b, double* d_x, const stiga_gmres_options* opts,
                              stiga_gmres_report* report, void* stream) {
    return guarded([&] {
        if (!A || n < 1) throw std::invalid_argument("gmres: null operator or empty system");
        Op opA = [&](const double* v, double* out) {
            const int s = A(A_ctx, v, out, stream);
            if (s != 0) throw std::runtime_error("gmres: operator callback failed (status " + std::to_string(s) + ")");
        };
        Op opP = [&](const double* v, double* out) {
            const int s = P(P_ctx, v, out, stream);
            if (s != 0)
                throw std::runtime_error("gmres: preconditioner callback failed (status " + std::to_string(s) + ")");
        };
        run_gmres(n, opA, P ? &opP : nullptr, comm, d_b, d_x, opts, report, as_stream(stream));
    });
}
