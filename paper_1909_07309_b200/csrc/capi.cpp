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
#include "host/assembly.hpp"
#include "host/fdsetup.hpp"
#include "host/geometry.hpp"

using namespace stiga;

namespace {

thread_local std::string g_last_error;

struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return STIGA_OK;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return STIGA_INVALID_ARGUMENT;
    } catch (const CudaFailure& e) {
        g_last_error = e.what();
        return STIGA_CUDA;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return STIGA_NUMERICAL;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return STIGA_NUMERICAL;
    }
}

void require(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

// Scoped device selection (restores the caller's current device).
struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        ck(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

struct DBuf {
    double* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t count) {
        if (p) cudaFree(p);
        p = nullptr;
        n = count;
        if (count) ck(cudaMalloc(&p, count * sizeof(double)), "cudaMalloc");
    }
    void upload(const std::vector<double>& h) {
        alloc(h.size());
        if (!h.empty()) ck(cudaMemcpy(p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice), "upload");
    }
};

DenseMatrix from_colmajor(const double* a, int n) {
    DenseMatrix m(n, n);
    std::memcpy(m.a.data(), a, sizeof(double) * n * static_cast<size_t>(n));
    return m;
}

// Row-major, zero-padded (Mp x Kp) copy of J, with J(i,j) = transpose ? U(j,i) : U(i,j).
std::vector<double> pad_factor(const DenseMatrix& U, bool transpose, int Mp, int Kp) {
    std::vector<double> out(static_cast<size_t>(Mp) * Kp, 0.0);
    const Index rows = transpose ? U.cols : U.rows;
    const Index cols = transpose ? U.rows : U.cols;
    if (rows > Mp || cols > Kp || Mp < 1)
        throw std::runtime_error("internal: no kernel tiling for a factor of size " + std::to_string(rows));
    for (Index i = 0; i < rows; ++i)
        for (Index j = 0; j < cols; ++j) out[i * Kp + j] = transpose ? U(j, i) : U(i, j);
    return out;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

namespace stiga {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace stiga

// ------------------------------------------------------------------------------------------
// FD preconditioner handle
// ------------------------------------------------------------------------------------------
struct stiga_fd_s {
    int device = 0;
    FDFactors F;
    int d = 0;
    std::vector<int> dims;  // n_1..n_d, n_t
    long long n_dof = 0, n_s = 0;
    std::vector<gpu::Tiling> tl;        // per spatial direction (forward products U_l^T)
    std::vector<gpu::Tiling> tl_b;      // backward products U_l (the last one tuned with the D^-1/2 post-scale)
    gpu::Tiling tl_t;
    gpu::Tiling tl_ts;                  // mode-kernel tiling of the split time products
    std::vector<std::unique_ptr<DBuf>> Jt, J;  // padded U_l^T, U_l (device eigen-order)
    std::vector<std::unique_ptr<DBuf>> Jft, Jfb;  // folded [A_e; A_o] / [A_p; A_q] (split directions)
    DBuf Jt_t, J_t;
    std::vector<std::unique_ptr<DBuf>> lam;
    DBuf S_inv, pair_c, pair_c1, pair_c1sq, pair_gg, g, dinv;
    DBuf scratch, scratch2;
    gpu::ArrowParams ap;

    gpu::ModeGeom geom(int mode) const {
        gpu::ModeGeom g;
        long long L = 1;
        for (int l = 0; l < mode; ++l) L *= dims[l];
        g.L = L;
        g.n = g.m = dims[mode];
        g.ncols = n_dof / dims[mode];
        return g;
    }
    // spatial mode m of a time slab with nt_local slices
    gpu::ModeGeom slab_geom(int mode, long long nt_local) const {
        gpu::ModeGeom g = geom(mode);
        g.ncols = n_s / dims[mode] * nt_local;
        return g;
    }
    // time mode of a spatial slab with ns_local spatial indices (ns_local x n_t, colex)
    gpu::ModeGeom time_geom(long long ns_local) const {
        gpu::ModeGeom g;
        g.L = ns_local;
        g.n = g.m = dims[d];
        g.ncols = ns_local;
        return g;
    }

    // One spatial mode product with tiling t: the folded kernel for a folded tiling (split
    // direction), the dense DMMA kernel otherwise.
    void mprod(const gpu::Tiling& t, int l, bool backward, const gpu::ModeGeom& g, const double* src, double* dst,
               const double* post, cudaStream_t st, const double* pre = nullptr, const gpu::Scatter* sc = nullptr) {
        if (t.fold) {
            if (sc && (backward || t.WM != 2)) throw std::runtime_error("internal: folded scatter needs a WM = 2 tiling");
            ck(gpu::launch_fold_product(t, g, src, dst, backward ? Jfb[l]->p : Jft[l]->p, !backward, post, st, pre, sc),
               "fd folded mode product");
        } else {
            ck(gpu::launch_mode_product(t, g, src, dst, backward ? J[l]->p : Jt[l]->p, post, st, pre, sc),
               "fd mode product");
        }
    }
    // best dense (unfolded) candidate of direction l (for stages the folded kernel cannot do)
    std::vector<gpu::Tiling> tl_dense;  // heuristic dense tiling per direction (J / Jt are padded for it)
    const gpu::Tiling& dense_tiling(int l) const { return (tl[l].fold || tl[l].WM != 1) ? tl_dense[l] : tl[l]; }

    // Distributed building blocks.
    void apply_space(bool backward, long long t0, long long nt_local, const double* in, double* out, cudaStream_t st) {
        if (!scratch2.p) scratch2.alloc(static_cast<size_t>(n_dof));
        double* bufs[2] = {scratch.p, scratch2.p};
        const double* dsl = dinv.p ? dinv.p + n_s * t0 : nullptr;
        const long long nloc = n_s * nt_local;
        const bool fused_pre = !backward && dsl && fused_prescale();
        const int nops = d + ((!backward && dsl && !fused_pre) ? 1 : 0);
        int k = 0;
        const double* src = in;
        auto next = [&]() -> double* { double* r = (k == nops - 1) ? out : bufs[k % 2]; ++k; return r; };
        if (!backward && dsl && !fused_pre) {
            double* dst = next();
            ck(gpu::launch_scale(dsl, src, dst, nloc, st), "slab pre-scale");
            src = dst;
        }
        for (int l = 0; l < d; ++l) {
            double* dst = next();
            mprod(backward ? tl_b[l] : (l == 0 ? first_tiling() : tl[l]), l, backward, slab_geom(l, nt_local), src, dst,
                  (backward && l == d - 1) ? dsl : nullptr, st, (fused_pre && l == 0) ? dsl : nullptr);
            src = dst;
        }
    }
    void apply_time(long long s0, long long ns_local, const double* in, double* out, cudaStream_t st) {
        if (!scratch2.p) scratch2.alloc(static_cast<size_t>(n_dof));
        gpu::ArrowParams a2 = ap;
        a2.s_off = s0;
        const gpu::ModeGeom g = time_geom(ns_local);
        if (time_split) {
            ck(gpu::launch_mode_product(tl_ts, g, in, scratch.p, Jt_t.p, nullptr, st), "slab time U_t^T");
            ck(gpu::launch_arrowhead(scratch.p, scratch2.p, ns_local, a2, st), "slab arrowhead");
            ck(gpu::launch_mode_product(tl_ts, g, scratch2.p, out, J_t.p, nullptr, st), "slab time U_t");
        } else {
            ck(gpu::launch_time_fused(tl_t, g, in, out, Jt_t.p, J_t.p, a2, st), "slab time fused");
        }
    }

    // Fused-exchange variants: the last product of the stage stores straight into the
    // owner ranks' receive buffers through the scatter epilogue, so no pack / all-to-all / unpack.
    void apply_space_scatter(long long t0, long long nt_local, const double* in, const gpu::Scatter& sc,
                             cudaStream_t st) {
        if (!scratch2.p) scratch2.alloc(static_cast<size_t>(n_dof));
        double* bufs[2] = {scratch.p, scratch2.p};
        const double* dsl = dinv.p ? dinv.p + n_s * t0 : nullptr;
        const long long nloc = n_s * nt_local;
        // the scattering product cannot also pre-scale: with d = 1 the pre-scale runs as its own pass
        const bool fused_pre = dsl && fused_prescale() && d > 1;
        const double* src = in;
        int k = 0;
        if (dsl && !fused_pre) {
            ck(gpu::launch_scale(dsl, src, bufs[k % 2], nloc, st), "slab pre-scale");
            src = bufs[k++ % 2];
        }
        for (int l = 0; l < d; ++l) {
            const bool last = l == d - 1;
            double* dst = last ? nullptr : bufs[k++ % 2];
            // the scattering product: the tuned tiling when it has a scatter epilogue (dense WM = 1 or
            // folded WM = 2), else the dense fallback
            const gpu::Tiling& tt = (l == 0 && fused_pre) ? first_tiling() : tl[l];
            const bool scatter_ok = !(fused_pre && l == 0) && (tt.fold ? tt.WM == 2 : tt.WM == 1);
            const gpu::Tiling& t = last ? (scatter_ok ? tt : dense_tiling(l)) : (l == 0 ? first_tiling() : tl[l]);
            mprod(t, l, false, slab_geom(l, nt_local), src, dst, nullptr, st, (fused_pre && l == 0) ? dsl : nullptr,
                  last ? &sc : nullptr);
            src = dst;
        }
    }
    void apply_time_scatter(long long s0, long long ns_local, const double* in, const gpu::Scatter& sc,
                            cudaStream_t st) {
        if (!scratch2.p) scratch2.alloc(static_cast<size_t>(n_dof));
        gpu::ArrowParams a2 = ap;
        a2.s_off = s0;
        const gpu::ModeGeom g = time_geom(ns_local);
        if (time_split) {
            ck(gpu::launch_mode_product(tl_ts, g, in, scratch.p, Jt_t.p, nullptr, st), "slab time U_t^T");
            ck(gpu::launch_arrowhead(scratch.p, scratch2.p, ns_local, a2, st), "slab arrowhead");
            gpu::Tiling tsc = tl_ts;
            if (tsc.WM != 1)
                for (const auto& t : cand_ts)
                    if (t.WM == 1) {
                        tsc = t;
                        break;
                    }
            ck(gpu::launch_mode_product(tsc, g, scratch2.p, nullptr, J_t.p, nullptr, st, nullptr, &sc),
               "slab time U_t (scatter)");
        } else {
            ck(gpu::launch_time_fused(tl_t, g, in, nullptr, Jt_t.p, J_t.p, a2, st, &sc), "slab time fused (scatter)");
        }
    }

    bool time_split = false;            // time direction as U_t^T GEMM + arrowhead + U_t GEMM

    // Setup-time autotuning: every candidate tiling of every mode (and both time-direction
    // variants) is timed once on the scratch vectors at the real tensor geometry and the fastest is
    // kept.  STIGA_TIME_VARIANT=fused|split forces the time path; STIGA_NO_AUTOTUNE=1 keeps the
    // heuristic first choices.
    std::vector<std::vector<gpu::Tiling>> cand_space;
    std::vector<gpu::Tiling> cand_time, cand_ts;

    float time_once(const std::function<void()>& f) {
        cudaEvent_t e0, e1;
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        f();  // warm (sets the smem attribute, loads the module)
        f();
        // short launches (< 0.25 ms) are timed in groups of 4 so launch gaps and event resolution do
        // not decide between candidates that differ by a few percent
        int inner = 1;
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            ck(cudaEventRecord(e0, nullptr), "event");
            for (int k = 0; k < inner; ++k) f();
            ck(cudaEventRecord(e1, nullptr), "event");
            ck(cudaEventSynchronize(e1), "event");
            float ms = 0.f;
            ck(cudaEventElapsedTime(&ms, e0, e1), "event");
            ms /= inner;
            if (rep == 0 && ms < 0.25f) {
                inner = 4;
                continue;
            }
            best = std::min(best, ms);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return best;
    }

    // STIGA_TUNE_CACHE=<file>: tuned choices (candidate indices) keyed by device + tensor shape, so a
    // profiled run (where ncu serialisation would distort the timings) replays the plain run's picks.
    std::string tune_key() const {
        cudaDeviceProp prop{};
        cudaGetDeviceProperties(&prop, device);
        std::string k = std::string(prop.name) + " d" + std::to_string(d);
        for (int l = 0; l < d; ++l) k += " " + std::to_string(dims[l]);
        return k + " t" + std::to_string(dims[d]) + (dinv.p ? " D" : "");
    }
    bool load_tuned(const char* path) {
        std::FILE* f = std::fopen(path, "r");
        if (!f) return false;
        const std::string key = tune_key() + " |";
        char line[1024];
        bool found = false;
        while (std::fgets(line, sizeof line, f)) {
            std::string ln(line);
            if (ln.compare(0, key.size(), key) != 0) continue;
            std::vector<int> v;
            const char* p = ln.c_str() + key.size();
            char* end = nullptr;
            for (long x = std::strtol(p, &end, 10); end != p; x = std::strtol(p, &end, 10)) {
                v.push_back(static_cast<int>(x));
                p = end;
            }
            if (static_cast<int>(v.size()) != d + 4 && static_cast<int>(v.size()) != 2 * d + 4) continue;
            bool ok = true;
            for (int l = 0; l < d; ++l) ok = ok && v[l] >= 0 && v[l] < static_cast<int>(cand_space[l].size());
            ok = ok && v[d] >= -1 && v[d] < static_cast<int>(cand_time.size()) && v[d + 1] >= 0 &&
                 v[d + 1] < static_cast<int>(cand_ts.size()) && (v[d + 2] == 1 || v[d] >= 0);
            if (!ok) continue;
            const bool has_b = static_cast<int>(v.size()) == 2 * d + 4;
            for (int l = 0; l < d && has_b; ++l)
                ok = ok && v[d + 4 + l] >= 0 && v[d + 4 + l] < static_cast<int>(cand_space[l].size());
            if (!ok) continue;
            for (int l = 0; l < d; ++l) {
                tl[l] = cand_space[l][v[l]];
                tl_b[l] = cand_space[l][has_b ? v[d + 4 + l] : v[l]];
            }
            tl_t = v[d] >= 0 ? cand_time[v[d]] : gpu::Tiling{};
            tl_ts = cand_ts[v[d + 1]];
            time_split = v[d + 2] == 1;
            use_fused_pre = v[d + 3] >= 0 && v[d + 3] < static_cast<int>(cand_space[0].size());
            tl_pre = use_fused_pre ? cand_space[0][v[d + 3]] : tl[0];
            found = true;
        }
        std::fclose(f);
        return found;
    }

    void autotune() {
        const char* force = std::getenv("STIGA_TIME_VARIANT");
        const bool no_tune = std::getenv("STIGA_NO_AUTOTUNE") != nullptr;
        const bool debug_tune = std::getenv("STIGA_DEBUG_TUNE") != nullptr;
        const char* cache = std::getenv("STIGA_TUNE_CACHE");
        if (cache && !no_tune && !force && load_tuned(cache)) return;
        if (!scratch2.p) scratch2.alloc(static_cast<size_t>(n_dof));
        ck(cudaMemset(scratch.p, 0, sizeof(double) * n_dof), "memset");
        const size_t kMaxCand = 8;
        std::vector<int> pick(d + 2, 0);
        for (int l = 0; l < d; ++l) {
            tl[l] = cand_space[l].front();
            if (no_tune) continue;
            float best = 1e30f;
            size_t n_fold = 0, n_dense = 0;
            for (size_t c = 0; c < cand_space[l].size(); ++c) {
                const gpu::Tiling& t = cand_space[l][c];
                if ((t.fold ? n_fold : n_dense)++ >= (t.fold ? 4 * kMaxCand : 2 * kMaxCand)) continue;
                const float ms = time_once([&] {
                    mprod(t, l, false, geom(l), scratch.p, scratch2.p, nullptr, nullptr);
                });
                if (ms < 0.985f * best) { best = ms; tl[l] = t; pick[l] = static_cast<int>(c); }  // 1.5%: above timing noise
                if (debug_tune)
                    std::fprintf(stderr, "[stiga tune] mode %d %s MI=%d WM=%d WN=%d NI=%d RB=%d ns=%d occ=%d: %.4f ms\n",
                                 l, t.fold ? "folded" : "dense", t.MI, t.WM, t.WN, t.NI, t.RB, t.nstage, t.ctas_per_sm,
                                 ms);
            }
        }
        // backward products U_l: tuned on their own (the folded backward kernel differs from the forward
        // one), the last direction with the D^-1/2 post-scale it carries in the apply
        std::vector<int> pick_b(d, 0);
        for (int l = 0; l < d; ++l) {
            tl_b[l] = tl[l];
            pick_b[l] = pick[l];
            if (no_tune) continue;
            const double* post = (l == d - 1) ? dinv.p : nullptr;
            float best = 1e30f;
            size_t n_fold = 0, n_dense = 0;
            for (size_t c = 0; c < cand_space[l].size(); ++c) {
                const gpu::Tiling& t = cand_space[l][c];
                if ((t.fold ? n_fold : n_dense)++ >= (t.fold ? 4 * kMaxCand : 2 * kMaxCand)) continue;
                const float ms = time_once([&] { mprod(t, l, true, geom(l), scratch.p, scratch2.p, post, nullptr); });
                if (ms < 0.985f * best) { best = ms; tl_b[l] = t; pick_b[l] = static_cast<int>(c); }
                if (debug_tune)
                    std::fprintf(stderr, "[stiga tune] bwd mode %d%s %s MI=%d WM=%d WN=%d RB=%d ns=%d: %.4f ms\n", l,
                                 post ? "+post" : "", t.fold ? "folded" : "dense", t.MI, t.WM, t.WN, t.RB, t.nstage, ms);
            }
        }
        use_fused_pre = false;
        tl_pre = tl[0];
        int pick_pre = -1;
        if (!no_tune && dinv.p) {
            const float sep = time_once([&] {
                ck(gpu::launch_scale(dinv.p, scratch.p, scratch2.p, n_dof, nullptr), "tune");
                mprod(tl[0], 0, false, geom(0), scratch2.p, scratch.p, nullptr, nullptr);
            });
            float best_fus = 1e30f;
            size_t n_fold = 0, n_dense = 0;
            for (size_t c = 0; c < cand_space[0].size(); ++c) {
                const gpu::Tiling& t = cand_space[0][c];
                if (!gpu::prescale_fits(t)) continue;
                if ((t.fold ? n_fold : n_dense)++ >= kMaxCand) continue;
                const float ms = time_once([&] { mprod(t, 0, false, geom(0), scratch.p, scratch2.p, nullptr, nullptr, dinv.p); });
                if (ms < best_fus) { best_fus = ms; tl_pre = t; pick_pre = static_cast<int>(c); }
            }
            use_fused_pre = pick_pre >= 0 && best_fus < sep;
            if (debug_tune)
                std::fprintf(stderr, "[stiga tune] pre-scale separate %.4f ms, fused %.4f ms (%s MI=%d RB=%d)\n", sep,
                             best_fus, tl_pre.fold ? "folded" : "dense", tl_pre.MI, tl_pre.RB);
        }
        const bool fused_ok = !cand_time.empty();
        tl_t = fused_ok ? cand_time.front() : gpu::Tiling{};
        tl_ts = cand_ts.front();
        float best_fused = 1e30f, best_split = 1e30f;
        if (!no_tune) {
            if (fused_ok && !(force && std::string(force) == "split")) {
                for (size_t c = 0; c < std::min(3 * kMaxCand, cand_time.size()); ++c) {
                    const gpu::Tiling& t = cand_time[c];
                    const float ms = time_once([&] {
                        ck(gpu::launch_time_fused(t, geom(d), scratch.p, scratch2.p, Jt_t.p, J_t.p, ap, nullptr), "tune");
                    });
                    if (ms < best_fused) { best_fused = ms; tl_t = t; pick[d] = static_cast<int>(c); }
                    if (debug_tune)
                        std::fprintf(stderr, "[stiga tune] time fused MI=%d WM=%d WN=%d ns=%d occ=%d: %.4f ms\n", t.MI,
                                     t.WM, t.WN, t.nstage, t.ctas_per_sm, ms);
                }
            }
            if (!(force && std::string(force) == "fused")) {
                float best_gemm = 1e30f;
                for (size_t c = 0; c < std::min(2 * kMaxCand, cand_ts.size()); ++c) {
                    const gpu::Tiling& t = cand_ts[c];
                    const float ms = time_once([&] {
                        ck(gpu::launch_mode_product(t, geom(d), scratch.p, scratch2.p, Jt_t.p, nullptr, nullptr), "tune");
                    });
                    if (ms < best_gemm) { best_gemm = ms; tl_ts = t; pick[d + 1] = static_cast<int>(c); }
                    if (debug_tune)
                        std::fprintf(stderr, "[stiga tune] time gemm MI=%d WN=%d RB=%d occ=%d: %.4f ms\n", t.MI, t.WN,
                                     t.RB, t.ctas_per_sm, ms);
                }
                const float arrow = time_once([&] {
                    ck(gpu::launch_arrowhead(scratch2.p, scratch.p, n_s, ap, nullptr), "tune");
                });
                best_split = 2.f * best_gemm + arrow;
                if (debug_tune) std::fprintf(stderr, "[stiga tune] arrowhead: %.4f ms\n", arrow);
            }
        }
        if (force && std::string(force) == "split") time_split = true;
        else if (force && std::string(force) == "fused" && fused_ok) time_split = false;
        else if (!fused_ok) time_split = true;
        else time_split = !no_tune && best_split < best_fused;
        if (cache && !no_tune && !force) {
            if (std::FILE* f = std::fopen(cache, "a")) {
                std::string ln = tune_key() + " |";
                for (int l = 0; l < d; ++l) ln += " " + std::to_string(pick[l]);
                ln += " " + std::to_string(fused_ok ? pick[d] : -1) + " " + std::to_string(pick[d + 1]) + " " +
                      std::to_string(time_split ? 1 : 0) + " " + std::to_string(use_fused_pre ? pick_pre : -1);
                for (int l = 0; l < d; ++l) ln += " " + std::to_string(pick_b[l]);
                ln += "\n";
                std::fputs(ln.c_str(), f);
                std::fclose(f);
            }
        }
    }

    // D^-1/2 pre-scale fused into the first forward mode product when its smem allows (the
    // separate scale pass otherwise); STIGA_NO_FUSED_PRESCALE=1 forces the separate pass.
    bool use_fused_pre = false;  // decided by the autotuner (fused vs separate, timed)
    gpu::Tiling tl_pre;          // tiling of the pre-scaled first forward pass (tuned separately: every
                                 // row block re-stages the D chunk, so it prefers fewer row blocks)
    bool fused_prescale() const {
        static const bool off = std::getenv("STIGA_NO_FUSED_PRESCALE") != nullptr;
        return dinv.p != nullptr && use_fused_pre && !off && gpu::prescale_fits(tl_pre);
    }
    const gpu::Tiling& first_tiling() const { return fused_prescale() ? tl_pre : tl[0]; }
    int launches() const { return 2 * d + (time_split ? 3 : 1) + (dinv.p && !fused_prescale() ? 1 : 0); }

    // Launch sequence (fdsolve.cpp:158-163): [D^-1/2 pre-scale], forward spatial modes U_l^T, the
    // time direction (fused U_t^T / arrowhead / U_t kernel, or the three as separate passes),
    // backward spatial modes U_l with the D^-1/2 post-scale fused into the last epilogue.  The
    // reference back transform applies U_1..U_d, U_t; Kronecker factors on distinct modes commute,
    // so applying U_t first is equal in exact arithmetic.  Intermediates ping-pong between two
    // handle-owned scratch vectors, so d_r may equal d_s.
    void apply(const double* in, double* out, cudaStream_t st, std::vector<cudaEvent_t>* ev) {
        if (!scratch2.p) scratch2.alloc(static_cast<size_t>(n_dof));
        double* bufs[2] = {scratch.p, scratch2.p};
        const bool scaled = dinv.p != nullptr;
        const int nops = launches();
        const double* src = in;
        int e = 0, k = 0;
        auto next = [&]() -> double* {
            double* dst = (k == nops - 1) ? out : bufs[k % 2];
            if (ev) ck(cudaEventRecord((*ev)[e++], st), "event");
            ++k;
            return dst;
        };
        const bool fused_pre = fused_prescale();
        if (scaled && !fused_pre) {
            double* dst = next();
            ck(gpu::launch_scale(dinv.p, src, dst, n_dof, st), "fd D^-1/2 pre-scale");
            src = dst;
        }
        for (int l = 0; l < d; ++l) {
            double* dst = next();
            mprod(l == 0 ? first_tiling() : tl[l], l, false, geom(l), src, dst, nullptr, st,
                  (l == 0 && fused_pre) ? dinv.p : nullptr);
            src = dst;
        }
        if (time_split) {
            double* dst = next();
            ck(gpu::launch_mode_product(tl_ts, geom(d), src, dst, Jt_t.p, nullptr, st), "fd time U_t^T product");
            src = dst;
            dst = next();
            ck(gpu::launch_arrowhead(src, dst, n_s, ap, st), "fd arrowhead solve");
            src = dst;
            dst = next();
            ck(gpu::launch_mode_product(tl_ts, geom(d), src, dst, J_t.p, nullptr, st), "fd time U_t product");
            src = dst;
        } else {
            double* dst = next();
            ck(gpu::launch_time_fused(tl_t, geom(d), src, dst, Jt_t.p, J_t.p, ap, st), "fd time-fused kernel");
            src = dst;
        }
        for (int l = 0; l < d; ++l) {
            double* dst = next();
            mprod(tl_b[l], l, true, geom(l), src, dst, (l == d - 1 && scaled) ? dinv.p : nullptr, st);
            src = dst;
        }
        if (ev) ck(cudaEventRecord((*ev)[e], st), "event");
    }
};

// ------------------------------------------------------------------------------------------
// KronSum handle
// ------------------------------------------------------------------------------------------
struct stiga_kronsum_s {
    int device = 0;
    int D = 0;
    std::vector<int> dims;
    long long n_dof = 0;
    bool spacetime = false;
    // generic: terms x D bands
    std::vector<double> coeffs;
    std::vector<std::vector<DenseMatrix>> factors;  // host copies (for diagonal)
    std::vector<std::unique_ptr<DBuf>> bands;       // term*D + l
    std::vector<int> hbw;
    // spacetime: per direction M_l, K_l bands, time gamma*W_t and nu*M_t bands
    DBuf t0, t1, t2, t3;  // scratch N_dof each
    // physical (geometry-mapped) system: stencil K_s, M_s on the device + time bands
    bool physical = false;
    gpu::PhysicalDesc pdesc;
    DBuf Kst, Mst, cp, qnode, qweight, bval, bder;
    int* bfirst = nullptr;
    std::vector<double> time_W, time_M;  // host copies for diagonal()
    ~stiga_kronsum_s() {
        if (bfirst) cudaFree(bfirst);
    }

    gpu::ModeGeom geom(int mode) const {
        gpu::ModeGeom g;
        long long L = 1;
        for (int l = 0; l < mode; ++l) L *= dims[l];
        g.L = L;
        g.n = g.m = dims[mode];
        g.ncols = n_dof / dims[mode];
        return g;
    }
    gpu::Band band(int idx) const { return gpu::Band{bands[idx]->p, hbw[idx]}; }

    void ensure_scratch(int count) {
        DBuf* s[4] = {&t0, &t1, &t2, &t3};
        for (int i = 0; i < count; ++i)
            if (!s[i]->p) s[i]->alloc(static_cast<size_t>(n_dof));
    }

    void apply(const double* x, double* y, cudaStream_t st) {
        const gpu::Band none{};
        if (physical) {  // y = M_s X W_t^T + K_s X M_t^T  (solver.cpp:67-70)
            // spatial stencils first, as the reference's mode order (kronop.cpp:75-89): MX = M_s X,
            // KX = K_s X on the tensor cores, then y = MX W_t^T + KX M_t^T in one banded time pass
            ensure_scratch(2);
            const int d = D - 1;
            ck(gpu::launch_stencil_apply2(pdesc, Mst.p, Kst.p, x, t0.p, t1.p, dims[d], st), "stencil apply");
            ck(gpu::launch_banded_pass(geom(d), t0.p, t1.p, y, nullptr, band(0), band(1), none, none, 0.0, st),
               "time bands");
            return;
        }
        if (spacetime) {
            // bands: [M_1, K_1, ..., M_d, K_d, gamma W_t, nu M_t]
            const int d = D - 1;
            ensure_scratch(4);
            double* a = t0.p;  // t_m  (M-chain)
            double* b = t1.p;  // k_m  (stiffness-sum chain)
            double* a2 = t2.p;
            double* b2 = t3.p;
            // mode 0: a = M_1 x, b = K_1 x
            ck(gpu::launch_banded_pass(geom(0), x, nullptr, a, b, band(0), none, band(1), none, 0.0, st), "banded");
            for (int m = 1; m < d; ++m) {
                // a2 = M_m a ; b2 = K_m a + M_m b
                ck(gpu::launch_banded_pass(geom(m), a, b, a2, b2, band(2 * m), none, band(2 * m + 1), band(2 * m), 0.0,
                                           st),
                   "banded");
                std::swap(a, a2);
                std::swap(b, b2);
            }
            // time: y = gamma W_t a + nu M_t b
            ck(gpu::launch_banded_pass(geom(d), a, b, y, nullptr, band(2 * d), band(2 * d + 1), none, none, 0.0, st),
               "banded");
            return;
        }
        // generic: per term D banded passes, the last accumulating into y
        ensure_scratch(2);
        const int nterms = static_cast<int>(coeffs.size());
        if (nterms == 0) {
            ck(cudaMemsetAsync(y, 0, sizeof(double) * n_dof, st), "memset");
            return;
        }
        for (int t = 0; t < nterms; ++t) {
            const double* src = x;
            double* ping[2] = {t0.p, t1.p};
            for (int l = 0; l < D; ++l) {
                const bool last = l == D - 1;
                double* dst = last ? y : ping[l % 2];
                gpu::Band Bd = band(t * D + l);
                ck(gpu::launch_banded_pass(geom(l), src, nullptr, dst, nullptr, Bd, none, none, none,
                                           last && t > 0 ? 1.0 : 0.0, st),
                   "banded");
                src = dst;
            }
        }
    }
};

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

struct stiga_problem_s {
    ProblemSpec spec;
};

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

int stiga_fd_setup(int d, const int* n, const double* const* K, const double* const* M, int n_t, const double* Wt,
                   const double* Mt, double gamma, double nu, const double* scaling, long long scaling_len, int device,
                   stiga_fd_t* out) {
    return guarded([&] {
        require(out != nullptr, "stiga_fd_setup: null handle output");
        *out = nullptr;
        require(d >= 1 && d <= gpu::kMaxDim, "ExtendedFDPreconditioner: per-direction matrices mismatch");
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
        if (scaling)
            require(scaling_len == n_s * n_t, "ExtendedFDPreconditioner: scaling vector length mismatch");
        auto h = std::make_unique<stiga_fd_s>();
        h->F = fd_setup(Ks, Ms, from_colmajor(Wt, n_t), from_colmajor(Mt, n_t), gamma, nu, scaling);
        const FDFactors& F = h->F;
        h->device = device;
        h->d = d;
        h->dims.assign(F.n.begin(), F.n.end());
        h->dims.push_back(F.n_t);
        h->n_dof = F.n_dof;
        h->n_s = F.n_s_total;
        if (device < 0) {  // host-only handle: setup + export, no device resources
            *out = h.release();
            return;
        }

        DeviceGuard dg(device);
        for (int l = 0; l < d; ++l) {
            std::vector<gpu::Tiling> dense = gpu::mode_tiling_candidates(F.n[l], F.n[l]);
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
            const bool fold_only = fk && (std::string(fk) == "force" || std::string(fk) == "force_wm2");
            const bool fold_wm2 = fk && std::string(fk) == "force_wm2";  // tests: folded WM = 2 tilings only
            if (F.fold[l].on && !dense_only) {  // folded candidates first (half the FLOPs)
                std::vector<gpu::Tiling> fc = gpu::fold_tiling_candidates(F.n[l]);
                if (fold_wm2) fc.erase(std::remove_if(fc.begin(), fc.end(), [](const gpu::Tiling& t) { return t.WM != 2; }),
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
                if (t.WM == 1) {
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
        h->cand_ts = gpu::mode_tiling_candidates(F.n_t, F.n_t);
        if (h->cand_ts.empty()) throw std::runtime_error("internal: no time-product tiling");
        int trows = 0;
        for (const auto& t : h->cand_time) trows = std::max(trows, t.Mp);
        for (const auto& t : h->cand_ts) trows = std::max(trows, t.Mp);
        const int tKp = h->cand_ts.front().Kp;
        h->Jt_t.upload(pad_factor(F.time.U, true, trows, tKp));
        h->J_t.upload(pad_factor(F.time.U, false, trows, tKp));
        h->S_inv.upload(F.S_inv_dev());
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
        if (!F.d_inv_sqrt.empty()) h->dinv.upload(F.d_inv_sqrt);
        h->scratch.alloc(static_cast<size_t>(h->n_dof));

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
        *out = h.release();
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
            case 5: src = &F.S_inv; break;
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
        P->apply(d_r, d_s, as_stream(stream), nullptr);
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
        P->apply(d_r, d_s, as_stream(stream), &ev);
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
        require(i >= 0 && i < P->launches(), "stiga_fd_launch_info: launch index out of range");
        std::vector<std::pair<std::string, double>> L;
        const double N = static_cast<double>(P->n_dof);
        if (P->dinv.p && !P->fused_prescale()) L.emplace_back("pre_scale", 0.0);
        // executed FP64 work: 2 n N per dense product, 4 F^2 N / n per folded one (F = ceil(n/2))
        auto prod_flops = [&](const gpu::Tiling& t, int l) {
            const double n = P->dims[l], Fh = n - std::floor(n / 2);
            return t.fold ? 4.0 * Fh * Fh * N / n : 2.0 * n * N;
        };
        auto tag = [](const gpu::Tiling& t) { return t.fold ? std::string("(folded)") : std::string(); };
        for (int l = 0; l < P->d; ++l) {
            const gpu::Tiling& t = l == 0 ? P->first_tiling() : P->tl[l];
            L.emplace_back("fwd_mode" + std::to_string(l) + tag(t) + (l == 0 && P->fused_prescale() ? "+pre_scale" : ""),
                           prod_flops(t, l));
        }
        const double nt = P->dims[P->d];
        if (P->time_split) {
            L.emplace_back("time_UtT", 2.0 * nt * N);
            L.emplace_back("arrowhead", 0.0);
            L.emplace_back("time_Ut", 2.0 * nt * N);
        } else {
            L.emplace_back("time_fused", 4.0 * nt * N);
        }
        for (int l = 0; l < P->d; ++l)
            L.emplace_back("bwd_mode" + std::to_string(l) + tag(P->tl_b[l]) +
                               (l == P->d - 1 && P->dinv.p ? "+post_scale" : ""),
                           prod_flops(P->tl_b[l], l));
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
        DBuf in, out;
        in.alloc(static_cast<size_t>(P->n_dof));
        out.alloc(static_cast<size_t>(P->n_dof));
        ck(cudaMemcpy(in.p, h_r, sizeof(double) * P->n_dof, cudaMemcpyHostToDevice), "H2D");
        P->apply(in.p, out.p, nullptr, nullptr);
        ck(cudaMemcpy(h_s, out.p, sizeof(double) * P->n_dof, cudaMemcpyDeviceToHost), "D2H");
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

int stiga_kronsum_create_spacetime(int d, const int* n, const double* const* K, const double* const* M, int n_t,
                                   const double* Wt, const double* Mt, double gamma, double nu, int device,
                                   stiga_kronsum_t* out) {
    return guarded([&] {
        require(out != nullptr, "stiga_kronsum_create_spacetime: null handle output");
        *out = nullptr;
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
        *out = h.release();
    });
}

int stiga_kronsum_create_physical(stiga_problem_t prob, int p, int n_el, int device, stiga_kronsum_t* out) {
    return guarded([&] {
        require(prob && out, "stiga_kronsum_create_physical: null argument");
        *out = nullptr;
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
        *out = h.release();
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
        A->apply(d_x, d_y, as_stream(stream));
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
        cudaStream_t st = as_stream(stream);
        if (A->physical) {
            ck(gpu::launch_stencil_apply2(A->pdesc, A->Mst.p, A->Kst.p, d_x, d_a, d_b, nt_local, st), "stencil apply");
            return;
        }
        // spatial chain of the spacetime form over dims [n_1 .. n_d, nt_local]
        const long long Ns = A->n_dof / A->dims[d];
        auto geo = [&](int m) {
            gpu::ModeGeom g;
            long long L = 1;
            for (int l = 0; l < m; ++l) L *= A->dims[l];
            g.L = L;
            g.n = g.m = A->dims[m];
            g.ncols = Ns * nt_local / A->dims[m];
            return g;
        };
        const gpu::Band none{};
        A->ensure_scratch(4);
        double* bufs[2][2] = {{A->t0.p, A->t1.p}, {A->t2.p, A->t3.p}};
        double* a = d == 1 ? d_a : bufs[0][0];
        double* b = d == 1 ? d_b : bufs[0][1];
        ck(gpu::launch_banded_pass(geo(0), d_x, nullptr, a, b, A->band(0), none, A->band(1), none, 0.0, st), "banded");
        for (int m = 1; m < d; ++m) {
            double* a2 = m == d - 1 ? d_a : bufs[m % 2][0];
            double* b2 = m == d - 1 ? d_b : bufs[m % 2][1];
            ck(gpu::launch_banded_pass(geo(m), a, b, a2, b2, A->band(2 * m), none, A->band(2 * m + 1), A->band(2 * m), 0.0,
                                       st),
               "banded");
            a = a2;
            b = b2;
        }
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

int stiga_fp64_peak(int device, double ms, double* tflops_dmma, double* tflops_dfma) {
    return guarded([&] {
        require(tflops_dmma && tflops_dfma, "stiga_fp64_peak: null output");
        DeviceGuard dg(device);
        ck(gpu::fp64_peak_probe(ms, tflops_dmma, tflops_dfma), "fp64 peak probe");
    });
}

}  // extern "C"
