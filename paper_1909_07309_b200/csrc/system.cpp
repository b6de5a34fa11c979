// C ABI of the SpaceTimeSystem glue around the hot path (include/stiga_gpu.h, "space-time system"):
//   stiga_problem_info     ProblemSpec fields the caller needs (problems.hpp:25-37)
//   stiga_system_means     gamma_mean / nu_mean of A-hat (solver.cpp:82-112), host quadrature
//   stiga_assemble_rhs     b_ = assemble_rhs(f / gamma_t, ...) (solver.cpp:72-76, assembly.cpp:413-504), device
//   stiga_compute_errors   compute_errors (problems.cpp:305-402), device
// The two device entry points replace the reference's element loops by sum factorization over the
// tensor Gauss grid (cuda/spacetime.cu): the source term / exact solution is evaluated once per
// space-time quadrature point, and the banded 1D collocation matrices move between the grid and
// the spline coefficients one mode at a time, in batches of time points.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "cuda/spacetime.cuh"
#include "handles.hpp"
#include "host/bspline.hpp"
#include "host/geometry.hpp"

using namespace stiga;
using namespace stiga::capi;

namespace {

struct IBuf {
    int* p = nullptr;
    IBuf() = default;
    IBuf(const IBuf&) = delete;
    IBuf& operator=(const IBuf&) = delete;
    ~IBuf() {
        if (p) cudaFree(p);
    }
    void upload(const std::vector<int>& h) {
        if (p) cudaFree(p);
        p = nullptr;
        if (h.empty()) return;
        ck(cudaMalloc(&p, sizeof(int) * h.size()), "cudaMalloc");
        ck(cudaMemcpy(p, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice), "upload");
    }
};

// Gauss rule of one 1D space and its active-basis tables (collocation_active, problems.cpp:35-49), plus
// for every basis function i the contiguous range [tlo, thi) of quadrature points whose support
// window contains i (the transpose of the banded collocation matrix).
struct Table1D {
    int Q = 0, n = 0, p1 = 0;
    std::vector<double> node, weight;
    DBuf d_node, d_weight, d_val, d_der;
    IBuf d_first, d_tlo, d_thi;

    Table1D(const SplineSpace1D& s, int ppe) {
        const QuadratureRule quad = gauss_rule(s.knot_vector(), ppe);
        Q = quad.num_points();
        n = s.dim();
        p1 = s.degree() + 1;
        node = quad.nodes;
        weight = quad.weights;
        std::vector<double> val, der, buf(p1);
        std::vector<int> first;
        for (int q = 0; q < Q; ++q) {
            first.push_back(s.eval_active(quad.nodes[q], 0, buf.data()));
            val.insert(val.end(), buf.begin(), buf.end());
            s.eval_active(quad.nodes[q], 1, buf.data());
            der.insert(der.end(), buf.begin(), buf.end());
        }
        std::vector<int> lo(n, Q), hi(n, 0);
        for (int q = 0; q < Q; ++q)
            for (int a = 0; a < p1; ++a) {
                const int i = first[q] + a;
                if (i < 0 || i >= n) continue;
                lo[i] = std::min(lo[i], q);
                hi[i] = std::max(hi[i], q + 1);
            }
        for (int i = 0; i < n; ++i)
            if (lo[i] >= hi[i]) lo[i] = hi[i] = 0;
        d_node.upload(node);
        d_weight.upload(weight);
        d_val.upload(val);
        d_der.upload(der);
        d_first.upload(first);
        d_tlo.upload(lo);
        d_thi.upload(hi);
    }
};

// The problem's spline map as a device descriptor (uniform open knots, as the physical assembly).
void geometry_desc(const ProblemSpec& spec, DBuf& cp, gpu::PhysicalDesc& g) {
    const GeometryMap& F = spec.geometry;
    const KnotVector& kv0 = F.knot_vectors()[0];
    for (const KnotVector& kv : F.knot_vectors()) {
        const KnotVector u = KnotVector::uniform_open(kv.degree(), kv.num_elements());
        require(kv.knots() == u.knots(), "space-time grid: geometry needs uniform open knot vectors");
        require(kv.degree() == kv0.degree() && kv.num_elements() == kv0.num_elements(),
                "space-time grid: geometry knot vectors must agree across directions");
    }
    cp.upload(F.control_points().a);
    g.d = spec.d;
    g.pg = kv0.degree();
    g.neg = kv0.num_elements();
    g.cp = cp.p;
    g.ncp = F.control_points().rows;
}

// Spatial quadrature grid with its geometry (x, w det J [, J^-T]) on the device.
struct SpatialGrid {
    int d = 0;
    long long Nq = 1;
    std::vector<std::unique_ptr<Table1D>> tabs;
    DBuf cp, x, wdet, JinvT;

    SpatialGrid(const ProblemSpec& spec, int p, int n_el, int ppe, bool want_jinv, cudaStream_t st) {
        d = spec.d;
        require(d >= 1 && d <= 3, "space-time grid: d must be 1, 2 or 3");
        const SplineSpace1D s = SplineSpace1D::spatial(p, n_el);
        int Q[3] = {1, 1, 1};
        const double* nodes[3] = {};
        const double* wts[3] = {};
        for (int l = 0; l < d; ++l) {
            tabs.emplace_back(new Table1D(s, ppe));
            Q[l] = tabs[l]->Q;
            nodes[l] = tabs[l]->d_node.p;
            wts[l] = tabs[l]->d_weight.p;
            Nq *= Q[l];
        }
        gpu::PhysicalDesc g;
        geometry_desc(spec, cp, g);
        x.alloc(static_cast<size_t>(Nq) * d);
        wdet.alloc(static_cast<size_t>(Nq));
        if (want_jinv) JinvT.alloc(static_cast<size_t>(Nq) * d * d);
        int* bad = nullptr;
        ck(cudaMalloc(&bad, sizeof(int)), "cudaMalloc");
        std::unique_ptr<int, decltype(&cudaFree)> guard(bad, &cudaFree);
        ck(cudaMemsetAsync(bad, 0, sizeof(int), st), "memset");
        ck(gpu::launch_qgrid_geometry(g, nodes, wts, Q, x.p, wdet.p, want_jinv ? JinvT.p : nullptr, bad, st),
           "quadrature-grid geometry");
        int hbad = 0;
        ck(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st), "download");
        ck(cudaStreamSynchronize(st), "quadrature-grid geometry");
        if (hbad) throw std::runtime_error("non-positive Jacobian determinant at a quadrature point");
    }
};

// Time points per batch so that `fields` grid tensors of Nq x nb doubles stay within `budget` bytes.
int time_batch(long long Nq, int Qt, int fields, double budget) {
    const double per = 8.0 * static_cast<double>(Nq) * fields;
    return static_cast<int>(std::max(1.0, std::min(static_cast<double>(Qt), std::floor(budget / per))));
}

}  // namespace

extern "C" {

int stiga_problem_info(stiga_problem_t P, int* d, double* T, int* has_rhs, int* has_exact, double* gamma0,
                       double* nu0) {
    return guarded([&] {
        require(P != nullptr, "stiga_problem_info: null problem");
        const int kind = problem_source_kind(P->spec);
        if (d) *d = P->spec.d;
        if (T) *T = P->spec.T;
        if (has_rhs) *has_rhs = kind != 0;
        if (has_exact) *has_exact = kind != 0;
        if (gamma0) *gamma0 = 1.0;  // every catalog problem uses gamma0 = nu0 = 1 (problems.hpp:31)
        if (nu0) *nu0 = 1.0;
    });
}

int stiga_system_means(stiga_problem_t P, int p, int n_el, double* gamma_mean, double* nu_mean) {
    return guarded([&] {
        require(P && gamma_mean && nu_mean, "stiga_system_means: null argument");
        require(p >= 1 && n_el >= 1, "stiga_system_means: p and n_el must be >= 1");
        system_means(P->spec, p, n_el, *gamma_mean, *nu_mean);
    });
}

int stiga_assemble_rhs(stiga_problem_t P, int p, int n_el, int points_per_element, int device, double* d_b,
                       void* stream) {
    return guarded([&] {
        require(P && d_b, "assemble_rhs: null argument");
        require(p >= 1 && n_el >= 1 && points_per_element >= 1, "assemble_rhs: p, n_el, points_per_element must be >= 1");
        const ProblemSpec& spec = P->spec;
        const int kind = problem_source_kind(spec);
        require(kind != 0, "assemble_rhs: the problem has no analytic source term");
        require(!spec.gamma_t, "assemble_rhs: time-dependent capacity is not in the device catalog");
        DeviceGuard dg(device);
        const cudaStream_t st = as_stream(stream);
        const int d = spec.d;
        SpatialGrid grid(spec, p, n_el, points_per_element, false, st);
        const Table1D tt(SplineSpace1D::temporal(p, n_el), points_per_element);
        long long Ns = 1;
        for (int l = 0; l < d; ++l) Ns *= grid.tabs[l]->n;
        const long long Nq = grid.Nq;
        const int nb = time_batch(Nq, tt.Q, 2, 1.0e9);
        DBuf A, B;
        A.alloc(static_cast<size_t>(Nq) * nb);
        B.alloc(static_cast<size_t>(Nq) * nb);
        ck(cudaMemsetAsync(d_b, 0, sizeof(double) * Ns * tt.n, st), "memset");
        for (int qt0 = 0; qt0 < tt.Q; qt0 += nb) {
            const int nbk = std::min(nb, tt.Q - qt0);
            ck(gpu::launch_rhs_eval(d, kind, Nq, grid.x.p, grid.wdet.p, tt.d_node.p + qt0, tt.d_weight.p + qt0, nbk,
                                    spec.T, A.p, st),
               "rhs source on the quadrature grid");
            double* in = A.p;
            double* out = B.p;
            // spatial modes: (n_0..n_{l-1}, Q_l, Q_{l+1}..Q_{d-1}, nbk) -> n_l
            long long L = 1;
            for (int l = 0; l < d; ++l) {
                const Table1D& t = *grid.tabs[l];
                long long R = nbk;
                for (int k = l + 1; k < d; ++k) R *= grid.tabs[k]->Q;
                ck(gpu::launch_colloc(L, t.Q, R, t.n, t.d_first.p, t.d_val.p, t.p1, t.d_tlo.p, t.d_thi.p, 0, true, 0.0,
                                      in, out, st),
                   "rhs spatial contraction");
                std::swap(in, out);
                L *= t.n;
            }
            // time: accumulate the batch's points into b (N_s, n_t)
            ck(gpu::launch_colloc(Ns, nbk, 1, tt.n, tt.d_first.p, tt.d_val.p, tt.p1, tt.d_tlo.p, tt.d_thi.p, qt0, true,
                                  1.0, in, d_b, st),
               "rhs time contraction");
        }
        ck(cudaStreamSynchronize(st), "assemble_rhs");
    });
}

int stiga_compute_errors(stiga_problem_t P, int p, int n_el, const double* d_coeffs, int points_per_element,
                         int device, double* l2l2, double* x_upper) {
    return guarded([&] {
        require(P && d_coeffs && l2l2 && x_upper, "compute_errors: null argument");
        require(p >= 1 && n_el >= 1 && points_per_element >= 1, "compute_errors: p, n_el, points_per_element must be >= 1");
        const ProblemSpec& spec = P->spec;
        const int kind = problem_source_kind(spec);
        require(kind != 0, "compute_errors: problem has no exact solution");
        DeviceGuard dg(device);
        cudaStream_t st = nullptr;
        const int d = spec.d;
        const double T = spec.T, gamma = 1.0, nu = 1.0;
        const double wt_dt = gamma * gamma / nu;
        SpatialGrid grid(spec, p, n_el, points_per_element, true, st);
        const Table1D tt(SplineSpace1D::temporal(p, n_el), points_per_element);
        long long Ns = 1;
        for (int l = 0; l < d; ++l) Ns *= grid.tabs[l]->n;
        const long long Nq = grid.Nq;
        // per batch: d + 2 result grids, two ping-pong grids, two time-contracted coefficient slabs
        const int nb = time_batch(std::max(Nq, Ns), tt.Q, d + 6, 3.0e9);
        std::vector<std::unique_ptr<DBuf>> field(d + 2);
        for (auto& f : field) {
            f.reset(new DBuf);
            f->alloc(static_cast<size_t>(Nq) * nb);
        }
        DBuf A, B, T0, T1;
        A.alloc(static_cast<size_t>(std::max(Nq, Ns)) * nb);
        B.alloc(static_cast<size_t>(std::max(Nq, Ns)) * nb);
        T0.alloc(static_cast<size_t>(Ns) * nb);
        T1.alloc(static_cast<size_t>(Ns) * nb);
        const int nblocks = 148 * 4;
        DBuf part;
        part.alloc(4 * nblocks);
        std::vector<double> hpart(4 * nblocks);
        double sums[4] = {0.0, 0.0, 0.0, 0.0};
        for (int qt0 = 0; qt0 < tt.Q; qt0 += nb) {
            const int nbk = std::min(nb, tt.Q - qt0);
            // time first: (N_s, n_t) -> (N_s, nbk) with the value / derivative collocation rows
            ck(gpu::launch_colloc(Ns, tt.n, 1, nbk, tt.d_first.p, tt.d_val.p, tt.p1, nullptr, nullptr, qt0, false, 0.0,
                                  d_coeffs, T0.p, st),
               "errors time collocation");
            ck(gpu::launch_colloc(Ns, tt.n, 1, nbk, tt.d_first.p, tt.d_der.p, tt.p1, nullptr, nullptr, qt0, false, 0.0,
                                  d_coeffs, T1.p, st),
               "errors time collocation");
            // fields: V (slot -1), G_l (slot l), Vt (slot d) on the spatial grid
            for (int slot = -1; slot <= d; ++slot) {
                const double* src = slot == d ? T1.p : T0.p;
                double* dst = field[slot + 1]->p;
                double* bufs[2] = {A.p, B.p};
                long long L = 1;
                for (int l = 0; l < d; ++l) {
                    const Table1D& t = *grid.tabs[l];
                    long long R = nbk;
                    for (int k = l + 1; k < d; ++k) R *= grid.tabs[k]->n;
                    double* out = (l == d - 1) ? dst : bufs[l & 1];
                    ck(gpu::launch_colloc(L, t.n, R, t.Q, t.d_first.p, slot == l ? t.d_der.p : t.d_val.p, t.p1, nullptr,
                                          nullptr, 0, false, 0.0, src, out, st),
                       "errors spatial collocation");
                    src = out;
                    L *= t.Q;
                }
            }
            const double* G[3] = {field[1]->p, d > 1 ? field[2]->p : nullptr, d > 2 ? field[3]->p : nullptr};
            ck(gpu::launch_error_terms(d, kind, Nq, nbk, grid.x.p, grid.wdet.p, grid.JinvT.p, field[0]->p, G[0], G[1],
                                       G[2], field[d + 1]->p, tt.d_node.p + qt0, tt.d_weight.p + qt0, T, wt_dt, nu,
                                       part.p, nblocks, st),
               "error terms");
            ck(cudaMemcpyAsync(hpart.data(), part.p, sizeof(double) * 4 * nblocks, cudaMemcpyDeviceToHost, st),
               "download");
            ck(cudaStreamSynchronize(st), "compute_errors");
            for (int b = 0; b < nblocks; ++b)
                for (int c = 0; c < 4; ++c) sums[c] += hpart[4 * b + c];
        }
        if (sums[1] == 0.0 || sums[3] == 0.0)
            throw std::invalid_argument("compute_errors: exact solution has zero norm");
        *l2l2 = std::sqrt(sums[0] / sums[1]);
        *x_upper = std::sqrt(sums[2] / sums[3]);
    });
}

}  // extern "C"
