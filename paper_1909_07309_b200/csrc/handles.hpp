// Handle types behind the C ABI (include/stiga_gpu.h): the FD preconditioner (stiga_fd_s) and the
// Kronecker-sum system operator (stiga_kronsum_s), shared by capi.cpp (single-device entry points),
// dist.cpp (time-sharded multi-GPU handles) and gmres.cpp.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "cuda/aux_kernels.cuh"
#include "cuda/fd_kernels.cuh"
#include "cuda/matvec_fused.cuh"
#include "cuda/physical.cuh"
#include "host/fdsetup.hpp"
#include "host/geometry.hpp"

struct stiga_comm_s;  // dist.cpp: NCCL or host-callback communicator of one rank

// make_problem(id) result behind stiga_problem_t (capi.cpp, system.cpp).
struct stiga_problem_s {
    stiga::ProblemSpec spec;
};

namespace stiga {
// Balanced contiguous partition of range(n) over `world` parts (the first n % world get +1).
inline void partition(long long n, int world, std::vector<long long>& off, std::vector<long long>& len) {
    off.assign(world, 0);
    len.assign(world, 0);
    const long long base = n / world, extra = n % world;
    long long o = 0;
    for (int q = 0; q < world; ++q) {
        off[q] = o;
        len[q] = base + (q < extra ? 1 : 0);
        o += len[q];
    }
}

// Time-sharded FD state of one rank: rank r owns time slices T_r of the colex vector;
// the time stage works on spatial slab S_r.  The two receive buffers are cudaMalloc'd here and shared
// with the peers through CUDA IPC; the scatter epilogues of the stage kernels store straight into them.
struct Shard {
    stiga_comm_s* comm = nullptr;
    int world = 1, rank = 0;
    std::vector<long long> t_off, t_len, s_off, s_len;
    capi::DBuf slab_recv;  // |S_r| x n_t: this rank's spatial slab for all time
    capi::DBuf time_recv;  // N_s x |T_r|: this rank's time slab (input of the backward stage)
    double* slab_ptr[STIGA_MAX_RANKS] = {};
    double* time_ptr[STIGA_MAX_RANKS] = {};
    std::vector<void*> opened;  // peers' buffers opened in this process
    gpu::Scatter fwd, tsc;
    ~Shard();  // dist.cpp (closes the IPC mappings)
};

// Time-sharded system operator state of one rank: halo-extended spatial halves a, b of the local
// time slab; the time neighbours push their p edge slices into the halos before the banded time pass.
struct KronShard {
    stiga_comm_s* comm = nullptr;
    int world = 1, rank = 0;
    std::vector<long long> t_off, t_len;
    int halo_lo = 0, halo_hi = 0, p = 0;
    capi::DBuf ext_a, ext_b;  // N_s x (halo_lo + |T_r| + halo_hi)
    double* prev_a = nullptr, *prev_b = nullptr, *next_a = nullptr, *next_b = nullptr;  // neighbours' ext
    int prev_lo = 0, prev_nt = 0, next_lo = 0;
    std::vector<void*> opened;
    ~KronShard();  // dist.cpp
};
}  // namespace stiga

struct stiga_fd_s;
struct stiga_kronsum_s;
namespace stiga {
// dist.cpp: the time-sharded apply of a sharded FD handle (space fwd + scatter, barrier, time + scatter,
// barrier, space bwd) and the time-sharded system mat-vec (space halves, halo push, barrier, time bands).
void fd_apply_sharded(stiga_fd_s& P, const double* in, double* out, cudaStream_t st, std::vector<cudaEvent_t>* ev);
void kronsum_apply_sharded(stiga_kronsum_s& A, const double* x, double* y, cudaStream_t st);
}  // namespace stiga

using namespace stiga;
using stiga::capi::CudaFailure;
using stiga::capi::DBuf;
using stiga::capi::DeviceGuard;
using stiga::capi::ck;
using stiga::capi::require;

// ------------------------------------------------------------------------------------------
// FD preconditioner handle
// ------------------------------------------------------------------------------------------
struct stiga_fd_s {
    int device = 0;
    FDFactors F;
    int d = 0;
    std::vector<int> dims;  // n_1..n_d, n_t
    long long n_dof = 0, n_s = 0;
    // Geometry the stage kernels (and the autotuner) run on: nt_span time slices for the spatial
    // stages, ns_span spatial indices for the time stage (n_t / N_s unsharded; the largest local slab
    // of a sharded handle).  Scratch vectors hold max(N_s nt_span, ns_span n_t) doubles.
    long long nt_span = 0, ns_span = 0, scratch_len = 0;
    long long dinv_t0 = 0;               // first time slice of the stored D^-1/2 (a sharded handle keeps its slab)
    std::unique_ptr<Shard> shard;        // null for a single-device handle
    std::vector<gpu::Tiling> tl;        // per spatial direction (forward products U_l^T)
    std::vector<gpu::Tiling> tl_b;      // backward products U_l (the last one tuned with the D^-1/2 post-scale)
    gpu::Tiling tl_t;
    gpu::Tiling tl_ts;                  // mode-kernel tiling of the split time products
    std::vector<std::unique_ptr<DBuf>> Jt, J;  // padded U_l^T, U_l (device eigen-order)
    std::vector<std::unique_ptr<DBuf>> Jft, Jfb;  // folded [A_e; A_o] / [A_p; A_q] (split directions)
    DBuf Jt_t, J_t;
    std::vector<std::unique_ptr<DBuf>> lam;
    DBuf S_inv, pair_c, pair_c1, pair_c1sq, pair_gg, g, dinv;
    bool schur_on_device = false;  // S_inv computed by the device setup (F.S_inv empty)
    DBuf scratch, scratch2;
    gpu::ArrowParams ap;

    // tuning / whole-apply geometry of mode `mode` (spatial: nt_span slices; time: ns_span indices)
    gpu::ModeGeom geom(int mode) const { return mode < d ? slab_geom(mode, nt_span) : time_geom(ns_span); }
    gpu::ModeGeom slab_geom_full(int mode) const {
        gpu::ModeGeom g;
        long long L = 1;
        for (int l = 0; l < mode; ++l) L *= dims[l];
        g.L = L;
        g.n = g.m = dims[mode];
        g.ncols = n_dof / dims[mode];
        return g;
    }
    const double* dinv_slab(long long t0) const { return dinv.p ? dinv.p + n_s * (t0 - dinv_t0) : nullptr; }
    void ensure_scratch() {
        scratch.ensure(static_cast<size_t>(scratch_len));
        scratch2.ensure(static_cast<size_t>(scratch_len));
    }
    // spatial mode m of a time slab with nt_local slices
    gpu::ModeGeom slab_geom(int mode, long long nt_local) const {
        gpu::ModeGeom g = slab_geom_full(mode);
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
            if (sc && (backward || t.WM != 2 || t.fold != 1)) throw std::runtime_error("internal: folded scatter needs a WM = 2 tiling");
            ck(gpu::launch_fold_product(t, g, src, dst, backward ? Jfb[l]->p : Jft[l]->p, !backward, post, st, pre, sc),
               "fd folded mode product");
        } else {
            ck(gpu::launch_mode_product(t, g, src, dst, backward ? J[l]->p : Jt[l]->p, post, st, pre, sc),
               "fd mode product");
        }
    }
    // best dense (unfolded) candidate of direction l (for stages the folded kernel cannot do)
    std::vector<gpu::Tiling> tl_dense;  // heuristic dense tiling per direction (J / Jt are padded for it)
    const gpu::Tiling& dense_tiling(int l) const { return (tl[l].fold || tl[l].res || tl[l].WM != 1) ? tl_dense[l] : tl[l]; }

    // Profiling hook of the stage functions: when prof_ev is set, an event is recorded before every
    // launch (stiga_fd_apply_profiled on sharded handles).
    std::vector<cudaEvent_t>* prof_ev = nullptr;
    size_t prof_i = 0;
    void mark(cudaStream_t st) {
        if (prof_ev && prof_i < prof_ev->size()) ck(cudaEventRecord((*prof_ev)[prof_i++], st), "event");
    }

    // Distributed building blocks.
    void apply_space(bool backward, long long t0, long long nt_local, const double* in, double* out, cudaStream_t st) {
        ensure_scratch();
        double* bufs[2] = {scratch.p, scratch2.p};
        const double* dsl = dinv_slab(t0);
        const long long nloc = n_s * nt_local;
        const bool fused_pre = !backward && dsl && fused_prescale();
        const int nops = d + ((!backward && dsl && !fused_pre) ? 1 : 0);
        int k = 0;
        const double* src = in;
        auto next = [&]() -> double* { double* r = (k == nops - 1) ? out : bufs[k % 2]; ++k; return r; };
        if (!backward && dsl && !fused_pre) {
            double* dst = next();
            mark(st);
            ck(gpu::launch_scale(dsl, src, dst, nloc, st), "slab pre-scale");
            src = dst;
        }
        for (int l = 0; l < d; ++l) {
            double* dst = next();
            mark(st);
            mprod(backward ? tl_b[l] : (l == 0 ? first_tiling() : tl[l]), l, backward, slab_geom(l, nt_local), src, dst,
                  (backward && l == d - 1) ? dsl : nullptr, st, (fused_pre && l == 0) ? dsl : nullptr);
            src = dst;
        }
    }
    void apply_time(long long s0, long long ns_local, const double* in, double* out, cudaStream_t st) {
        ensure_scratch();
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
        ensure_scratch();
        double* bufs[2] = {scratch.p, scratch2.p};
        const double* dsl = dinv_slab(t0);
        const long long nloc = n_s * nt_local;
        // the scattering product cannot also pre-scale: with d = 1 the pre-scale runs as its own pass
        const bool fused_pre = dsl && fused_prescale() && d > 1;
        const double* src = in;
        int k = 0;
        if (dsl && !fused_pre) {
            mark(st);
            ck(gpu::launch_scale(dsl, src, bufs[k % 2], nloc, st), "slab pre-scale");
            src = bufs[k++ % 2];
        }
        for (int l = 0; l < d; ++l) {
            const bool last = l == d - 1;
            double* dst = last ? nullptr : bufs[k++ % 2];
            // the scattering product: the tuned tiling when it has a scatter epilogue (dense WM = 1 or
            // folded WM = 2), else the dense fallback
            const gpu::Tiling& tt = (l == 0 && fused_pre) ? first_tiling() : tl[l];
            const bool scatter_ok = !(fused_pre && l == 0) && (tt.fold == 1 ? tt.WM == 2 : (tt.fold == 0 && tt.WM == 1 && !tt.res));
            const gpu::Tiling& t = last ? (scatter_ok ? tt : dense_tiling(l)) : (l == 0 ? first_tiling() : tl[l]);
            mark(st);
            mprod(t, l, false, slab_geom(l, nt_local), src, dst, nullptr, st, (fused_pre && l == 0) ? dsl : nullptr,
                  last ? &sc : nullptr);
            src = dst;
        }
    }
    void apply_time_scatter(long long s0, long long ns_local, const double* in, const gpu::Scatter& sc,
                            cudaStream_t st) {
        ensure_scratch();
        gpu::ArrowParams a2 = ap;
        a2.s_off = s0;
        const gpu::ModeGeom g = time_geom(ns_local);
        if (time_split) {
            mark(st);
            ck(gpu::launch_mode_product(tl_ts, g, in, scratch.p, Jt_t.p, nullptr, st), "slab time U_t^T");
            mark(st);
            ck(gpu::launch_arrowhead(scratch.p, scratch2.p, ns_local, a2, st), "slab arrowhead");
            mark(st);
            gpu::Tiling tsc = tl_ts;
            if (tsc.WM != 1 || tsc.res)  // a streaming WM = 1 tiling carries the scatter epilogue
                for (const auto& t : cand_ts)
                    if (t.WM == 1 && !t.res) {
                        tsc = t;
                        break;
                    }
            ck(gpu::launch_mode_product(tsc, g, scratch2.p, nullptr, J_t.p, nullptr, st, nullptr, &sc),
               "slab time U_t (scatter)");
        } else {
            mark(st);
            gpu::Tiling tf = tl_t;
            if (tf.res)  // the scatter epilogue lives in the streaming time-fused kernel
                for (const auto& t : cand_time)
                    if (!t.res) {
                        tf = t;
                        break;
                    }
            ck(gpu::launch_time_fused(tf, g, in, nullptr, Jt_t.p, J_t.p, a2, st, &sc), "slab time fused (scatter)");
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
        if (nt_span != dims[d] || ns_span != n_s) k += " span" + std::to_string(nt_span) + "x" + std::to_string(ns_span);
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
        ensure_scratch();
        ck(cudaMemset(scratch.p, 0, sizeof(double) * scratch_len), "memset");
        const size_t kMaxCand = 8;
        std::vector<int> pick(d + 2, 0);
        for (int l = 0; l < d; ++l) {
            tl[l] = cand_space[l].front();
            if (no_tune) continue;
            float best = 1e30f;
            size_t n_fold = 0, n_dense = 0;
            for (size_t c = 0; c < cand_space[l].size(); ++c) {
                const gpu::Tiling& t = cand_space[l][c];
                if ((t.fold ? n_fold : n_dense)++ >= (t.fold ? 4 * kMaxCand : 3 * kMaxCand)) continue;
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
                if ((t.fold ? n_fold : n_dense)++ >= (t.fold ? 4 * kMaxCand : 3 * kMaxCand)) continue;
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
                ck(gpu::launch_scale(dinv.p, scratch.p, scratch2.p, n_s * nt_span, nullptr), "tune");
                mprod(tl[0], 0, false, geom(0), scratch2.p, scratch.p, nullptr, nullptr);
            });
            float best_fus = 1e30f;
            size_t n_fold = 0, n_dense = 0;
            for (size_t c = 0; c < cand_space[0].size(); ++c) {
                const gpu::Tiling& t = cand_space[0][c];
                if (!gpu::prescale_fits(t)) continue;
                if ((t.fold ? n_fold : n_dense)++ >= 2 * kMaxCand) continue;
                const float ms = time_once([&] { mprod(t, 0, false, geom(0), scratch.p, scratch2.p, nullptr, nullptr, dinv.p); });
                if (ms < best_fus) { best_fus = ms; tl_pre = t; pick_pre = static_cast<int>(c); }
            }
            static const bool force_pre = std::getenv("STIGA_FUSED_PRESCALE") != nullptr;  // tests
            use_fused_pre = pick_pre >= 0 && (best_fus < sep || force_pre);
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
                for (size_t c = 0; c < std::min(3 * kMaxCand, cand_ts.size()); ++c) {
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
                    ck(gpu::launch_arrowhead(scratch2.p, scratch.p, ns_span, ap, nullptr), "tune");
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
    int launches() const { return static_cast<int>(launch_list().size()); }

    // (name, executed FP64 flops) of every timed segment of one apply, in launch order: a kernel
    // launch, or (sharded handles) an exchange barrier between the stages.  Flops: 2 n N per dense
    // product, 4 F^2 N / n per folded one (F = ceil(n/2)), 0 for elementwise passes and barriers.
    std::vector<std::pair<std::string, double>> launch_list() const {
        std::vector<std::pair<std::string, double>> L;
        const bool sharded = shard != nullptr;
        const double Nsp = static_cast<double>(sharded ? n_s * shard->t_len[shard->rank] : n_dof);
        const double Nt = static_cast<double>(sharded ? shard->s_len[shard->rank] * dims[d] : n_dof);
        // a sharded forward stage pre-scales in a separate pass when the scattering product is mode 0 (d = 1)
        const bool fused_pre = fused_prescale() && !(sharded && d == 1);
        if (dinv.p && !fused_pre) L.emplace_back("pre_scale", 0.0);
        auto prod_flops = [&](const gpu::Tiling& t, int l) {
            const double n = dims[l], Fh = n - std::floor(n / 2);
            return t.fold ? 4.0 * Fh * Fh * Nsp / n : 2.0 * n * Nsp;
        };
        auto tag = [](const gpu::Tiling& t) {
            return t.fold == 2 ? std::string("(folded,res)")
                               : (t.fold ? std::string("(folded)") : (t.res ? std::string("(res)") : std::string()));
        };
        for (int l = 0; l < d; ++l) {
            const gpu::Tiling& t = l == 0 ? (fused_pre ? tl_pre : tl[0]) : tl[l];
            L.emplace_back("fwd_mode" + std::to_string(l) + tag(t) + (l == 0 && fused_pre ? "+pre_scale" : "") +
                               (sharded && l == d - 1 ? "+scatter" : ""),
                           prod_flops(t, l));
        }
        if (sharded) L.emplace_back("exchange_barrier_1", 0.0);
        const double nt = dims[d];
        if (time_split) {
            L.emplace_back("time_UtT" + tag(tl_ts), 2.0 * nt * Nt);
            L.emplace_back("arrowhead", 0.0);
            L.emplace_back(std::string("time_Ut") + (sharded ? "+scatter" : tag(tl_ts)), 2.0 * nt * Nt);
        } else {
            L.emplace_back(std::string("time_fused") + (sharded ? "+scatter" : tag(tl_t)), 4.0 * nt * Nt);
        }
        if (sharded) L.emplace_back("exchange_barrier_2", 0.0);
        for (int l = 0; l < d; ++l)
            L.emplace_back("bwd_mode" + std::to_string(l) + tag(tl_b[l]) + (l == d - 1 && dinv.p ? "+post_scale" : ""),
                           prod_flops(tl_b[l], l));
        return L;
    }

    // Launch sequence (fdsolve.cpp:158-163): [D^-1/2 pre-scale], forward spatial modes U_l^T, the
    // time direction (fused U_t^T / arrowhead / U_t kernel, or the three as separate passes),
    // backward spatial modes U_l with the D^-1/2 post-scale fused into the last epilogue.  The
    // reference back transform applies U_1..U_d, U_t; Kronecker factors on distinct modes commute,
    // so applying U_t first is equal in exact arithmetic.  Intermediates ping-pong between two
    // handle-owned scratch vectors, so d_r may equal d_s.
    void apply(const double* in, double* out, cudaStream_t st, std::vector<cudaEvent_t>* ev) {
        ensure_scratch();
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
    std::unique_ptr<KronShard> kshard;  // time-sharded operator (dist.cpp); null for a single-device one
    long long n_local() const;           // entries of the local slab (n_dof unsharded)
    bool spacetime = false;
    // generic: terms x D bands
    std::vector<double> coeffs;
    std::vector<std::vector<DenseMatrix>> factors;  // host copies (for diagonal)
    std::vector<std::unique_ptr<DBuf>> bands;       // term*D + l
    std::vector<int> hbw;
    // spacetime: per direction M_l, K_l bands, time gamma*W_t and nu*M_t bands
    DBuf t0, t1, t2, t3;  // scratch N_dof each
    // fused mat-vec (cuda/matvec_fused.cu): bands widened to 2 fp + 1 taps per spatial direction
    // (M_l, K_l rows) and the COLUMNS of gamma W_t, nu M_t; fp = max half-bandwidth (0 = not available)
    int fp = 0;
    std::vector<std::unique_ptr<DBuf>> wband;  // [M_1, K_1, ..., M_d, K_d]
    DBuf tcol_w, tcol_m;
    bool use_fused() const {
        static const bool off = std::getenv("STIGA_MATVEC_PASSES") != nullptr;
        return spacetime && fp > 0 && !off;
    }
    // fields the fused time stage consumes for a slab of nt_local slices: d <= 2 the spatial halves
    // (a, b); d = 3 the mode-(0,1) halves a2, b2 (mode 2 runs inside the time stage)
    void fused_space(long long nt_local, const double* x, double* a, double* b, cudaStream_t st) {
        const int d = D - 1;
        const gpu::Band none{};
        if (d == 1) {
            gpu::ModeGeom g;
            g.L = 1;
            g.n = g.m = dims[0];
            g.ncols = nt_local;
            ck(gpu::launch_banded_pass(g, x, nullptr, a, b, band(0), none, band(1), none, 0.0, st), "banded");
            return;
        }
        const long long R = (d == 3 ? dims[2] : 1) * nt_local;
        ck(gpu::launch_plane2(dims[0], dims[1], R, fp, x, a, b, wband[0]->p, wband[1]->p, wband[2]->p, wband[3]->p, st),
           "fused mat-vec modes 0+1");
    }
    // y (slices [to0, to0+nto)) from the fields of the input slices [ti0, ti0+nti)
    void fused_time(int ti0, int nti, int to0, int nto, const double* a, const double* b, double* y, cudaStream_t st) {
        const int d = D - 1;
        long long Ns = 1;
        for (int l = 0; l < d; ++l) Ns *= dims[l];
        if (d == 3) {
            ck(gpu::launch_stream(true, static_cast<long long>(dims[0]) * dims[1], dims[2], dims[d], ti0, nti, to0, nto, fp, a, b, y,
                                  wband[4]->p, wband[5]->p, tcol_w.p, tcol_m.p, st),
               "fused mat-vec mode 2 + time");
        } else {
            ck(gpu::launch_stream(false, Ns, 1, dims[d], ti0, nti, to0, nto, fp, a, b, y, nullptr, nullptr, tcol_w.p, tcol_m.p, st),
               "fused mat-vec time");
        }
    }
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

    void ensure_scratch(int count) {  // local-slab sized (N_dof / world for a sharded operator)
        DBuf* s[4] = {&t0, &t1, &t2, &t3};
        for (int i = 0; i < count; ++i) s[i]->ensure(static_cast<size_t>(n_local()));
    }

    // Spatial halves of a time slab with nt_local slices (N_s x nt_local colex): d_a = a(x), d_b = b(x)
    // (spacetime: a = (M_d .. M_1) x, b = sum_l (M_d .. K_l .. M_1) x; physical: a = M_s x, b = K_s x).
    void apply_space_slab(long long nt_local, const double* d_x, double* d_a, double* d_b, cudaStream_t st) {
        const int d = D - 1;
        if (physical) {
            ck(gpu::launch_stencil_apply2(pdesc, Mst.p, Kst.p, d_x, d_a, d_b, nt_local, st), "stencil apply");
            return;
        }
        // spatial chain of the spacetime form over dims [n_1 .. n_d, nt_local]
        const long long Ns = n_dof / dims[d];
        auto geo = [&](int m) {
            gpu::ModeGeom g;
            long long L = 1;
            for (int l = 0; l < m; ++l) L *= dims[l];
            g.L = L;
            g.n = g.m = dims[m];
            g.ncols = Ns * nt_local / dims[m];
            return g;
        };
        const gpu::Band none{};
        ensure_scratch(4);
        double* bufs[2][2] = {{t0.p, t1.p}, {t2.p, t3.p}};
        double* a = d == 1 ? d_a : bufs[0][0];
        double* b = d == 1 ? d_b : bufs[0][1];
        ck(gpu::launch_banded_pass(geo(0), d_x, nullptr, a, b, band(0), none, band(1), none, 0.0, st), "banded");
        for (int m = 1; m < d; ++m) {
            double* a2 = m == d - 1 ? d_a : bufs[m % 2][0];
            double* b2 = m == d - 1 ? d_b : bufs[m % 2][1];
            ck(gpu::launch_banded_pass(geo(m), a, b, a2, b2, band(2 * m), none, band(2 * m + 1), band(2 * m), 0.0,
                                       st),
               "banded");
            a = a2;
            b = b2;
        }
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
        if (use_fused()) {  // two kernels: modes 0+1 (plane tiles), [mode 2 +] time (streamed ring)
            const int d = D - 1, nt = dims[d];
            ensure_scratch(2);
            fused_space(nt, x, t0.p, t1.p, st);
            fused_time(0, nt, 0, nt, t0.p, t1.p, y, st);
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

inline long long stiga_kronsum_s::n_local() const {
    if (!kshard) return n_dof;
    return n_dof / dims[D - 1] * kshard->t_len[kshard->rank];
}
