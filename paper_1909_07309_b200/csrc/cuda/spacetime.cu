// Space-time quadrature-grid kernels (RHS assembly and error norms).  See spacetime.cuh.
#include "spacetime.cuh"
#include "geom_device.cuh"

namespace stiga {
namespace gpu {

namespace {

using namespace geomdev;

// ---- manufactured solutions of the catalog (problems.cpp:131-241) ------------------------------
template <int D>
__device__ __forceinline__ double sin_prod(const double* x) {
    double v = 1.0;
    for (int l = 0; l < D; ++l) v *= sin(kPi * x[l]);
    return v;
}

__device__ __forceinline__ double annulus_P(double x1, double x2) {
    const double r2 = x1 * x1 + x2 * x2;
    return -(r2 - 1.0) * (r2 - 4.0) * x1 * x2 * x2;
}

__device__ __forceinline__ double annulus_lapP(double x1, double x2) {
    const double x13 = x1 * x1 * x1, x22 = x2 * x2;
    return -2.0 * x13 * x1 * x1 - 44.0 * x13 * x22 + 10.0 * x13 - 42.0 * x1 * x22 * x22 + 90.0 * x1 * x22 - 8.0 * x1;
}

__device__ __forceinline__ double separable_nu_t(double t) { return 1.0 + 50.0 * (1.0 + cos(t / (2.0 * kPi))); }

// f(x, t) (problems.cpp:157-159, 211-213, 229-240)
template <int D>
__device__ double source(int kind, const double* x, double t) {
    if (kind == kSrcIdentity) {
        return sin_prod<D>(x) * (kPi * cos(kPi * t) + D * kPi * kPi * sin(kPi * t));
    } else if (kind == kSrcAnnulus) {
        return annulus_P(x[0], x[1]) * cos(t) - annulus_lapP(x[0], x[1]) * sin(t);
    } else if (kind == kSrcSeparableNu) {
        const double s1 = sin(kPi * x[0]), c1 = cos(kPi * x[0]);
        const double s2 = sin(kPi * x[D > 1 ? 1 : 0]), c2 = cos(kPi * x[D > 1 ? 1 : 0]);
        const double st = sin(kPi * t), ct = cos(kPi * t);
        const double x1 = x[0], x2 = x[D > 1 ? 1 : 0];
        const double r = hypot(x1, x2);
        const double r3 = r * r * r;
        const double dnu1 = -49.5 * x1 * x2 / r3;
        const double dnu2 = 49.5 * x1 * x1 / r3;
        const double lap_u = -2.0 * kPi * kPi * s1 * s2 * st;
        const double gdot = dnu1 * kPi * c1 * s2 * st + dnu2 * kPi * s1 * c2 * st;
        return kPi * s1 * s2 * ct - separable_nu_t(t) * ((50.5 + 49.5 * x2 / r) * lap_u + gdot);
    }
    return 0.0;
}

// u, grad u, du/dt (problems.cpp:137-154, 200-209; separable-nu keeps the identity solution)
template <int D>
__device__ void exact(int kind, const double* x, double t, double& u, double* gu, double& ut) {
    if (kind == kSrcAnnulus) {
        const double x1 = x[0], x2 = x[D > 1 ? 1 : 0];
        const double P = annulus_P(x1, x2), st = sin(t);
        const double a = x1 * x1, b = x2 * x2;
        const double d1 = -5.0 * a * a * b - 6.0 * a * b * b + 15.0 * a * b - b * b * b + 5.0 * b * b - 4.0 * b;
        const double x13 = a * x1, x23 = b * x2;
        const double d2 = -2.0 * a * a * x1 * x2 - 8.0 * x13 * x23 + 10.0 * x13 * x2 - 6.0 * x1 * x23 * b +
                          20.0 * x1 * x23 - 8.0 * x1 * x2;
        u = P * st;
        ut = P * cos(t);
        gu[0] = d1 * st;
        if (D > 1) gu[D > 1 ? 1 : 0] = d2 * st;
        return;
    }
    const double sp = sin_prod<D>(x), st = sin(kPi * t);
    u = sp * st;
    ut = sp * kPi * cos(kPi * t);
    for (int l = 0; l < D; ++l) {
        double v = kPi * cos(kPi * x[l]);
        for (int k = 0; k < D; ++k)
            if (k != l) v *= sin(kPi * x[k]);
        gu[l] = v * st;
    }
}

template <int D>
__global__ void __launch_bounds__(256) qgrid_geometry_kernel(PhysicalDesc g, const double* n0, const double* n1,
                                                             const double* n2, const double* w0, const double* w1,
                                                             const double* w2, int Q0, int Q1, int Q2, double* xo,
                                                             double* wdet, double* JinvT, int* bad) {
    const double* nodes[3] = {n0, n1, n2};
    const double* wts[3] = {w0, w1, w2};
    const int Q[3] = {Q0, Q1, Q2};
    long long Nq = 1;
    for (int l = 0; l < D; ++l) Nq *= Q[l];
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < Nq;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        double eta[D], w = 1.0;
        long long rem = i;
        for (int l = 0; l < D; ++l) {
            const int jl = static_cast<int>(rem % Q[l]);
            rem /= Q[l];
            eta[l] = nodes[l][jl];
            w *= wts[l][jl];
        }
        double x[D], J[D * D], Ji[D * D];
        geometry_eval<D>(g, eta, x, J);
        const double det = det_inv<D>(J, Ji);
        if (!(det > 0.0)) atomicOr(bad, 1);
        for (int c = 0; c < D; ++c) xo[i + Nq * c] = x[c];
        wdet[i] = w * det;
        if (JinvT)
            for (int r = 0; r < D; ++r)
                for (int c = 0; c < D; ++c) JinvT[i + Nq * (r + D * c)] = Ji[c + D * r];  // (J^-1)^T
    }
}

template <int D>
__global__ void __launch_bounds__(256) rhs_eval_kernel(int kind, long long Nq, const double* __restrict__ xg,
                                                       const double* __restrict__ wdet, const double* tnode,
                                                       const double* tweight, int nb, double T, double* F) {
    const long long total = Nq * nb;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long js = i % Nq;
        const int k = static_cast<int>(i / Nq);
        double x[D];
        for (int c = 0; c < D; ++c) x[c] = xg[js + Nq * c];
        const double wx = wdet[js] * T;  // assembly.cpp:484 (w det T)
        F[i] = wx * tweight[k] * source<D>(kind, x, T * tnode[k]);
    }
}

__global__ void __launch_bounds__(256) colloc_fwd_kernel(long long L, int nin, long long R, int nout,
                                                         const int* __restrict__ first,
                                                         const double* __restrict__ tab, int p1, int qoff,
                                                         const double* __restrict__ in, double* __restrict__ out) {
    const long long total = L * nout * R;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long l = i % L, rest = i / L;
        const int q = static_cast<int>(rest % nout);
        const long long r = rest / nout;
        const int qg = qoff + q;
        const int f0 = first[qg];
        double acc = 0.0;
        for (int a = 0; a < p1; ++a) {
            const int j = f0 + a;
            if (j >= 0 && j < nin) acc += tab[static_cast<long long>(qg) * p1 + a] * in[l + L * (j + static_cast<long long>(nin) * r)];
        }
        out[i] = acc;
    }
}

__global__ void __launch_bounds__(256) colloc_tr_kernel(long long L, int nin, long long R, int nout,
                                                        const int* __restrict__ first, const double* __restrict__ tab,
                                                        int p1, const int* __restrict__ tlo,
                                                        const int* __restrict__ thi, int qoff, double beta,
                                                        const double* __restrict__ in, double* __restrict__ out) {
    const long long total = L * nout * R;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long l = i % L, rest = i / L;
        const int j = static_cast<int>(rest % nout);
        const long long r = rest / nout;
        const int lo = max(tlo[j], qoff), hi = min(thi[j], qoff + nin);
        double acc = 0.0;
        for (int qg = lo; qg < hi; ++qg) {
            const int a = j - first[qg];
            if (a >= 0 && a < p1)
                acc += tab[static_cast<long long>(qg) * p1 + a] * in[l + L * ((qg - qoff) + static_cast<long long>(nin) * r)];
        }
        out[i] = beta == 0.0 ? acc : beta * out[i] + acc;
    }
}

template <int D>
__global__ void __launch_bounds__(256) error_terms_kernel(int kind, long long Nq, int nb, const double* __restrict__ xg,
                                                          const double* __restrict__ wdet,
                                                          const double* __restrict__ JinvT,
                                                          const double* __restrict__ V, const double* G0,
                                                          const double* G1, const double* G2,
                                                          const double* __restrict__ Vt, const double* tnode,
                                                          const double* tweight, double T, double wt_dt, double nu,
                                                          double* partial) {
    const double* G[3] = {G0, G1, G2};
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    const long long total = Nq * nb;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long js = i % Nq;
        const int k = static_cast<int>(i / Nq);
        const double t = T * tnode[k];
        const double w = tweight[k] * T * wdet[js];  // problems.cpp:380-381 (wt wsp det)
        double x[D], ge[D], gh[D];
        for (int c = 0; c < D; ++c) x[c] = xg[js + Nq * c];
        double ue, dte;
        exact<D>(kind, x, t, ue, ge, dte);
        const double e = V[i] - ue;
        const double de = Vt[i] / T - dte;
        for (int l = 0; l < D; ++l) gh[l] = G[l][i];
        double gerr2 = 0.0, ge2 = 0.0;
        for (int r = 0; r < D; ++r) {
            double v = 0.0;
            for (int c = 0; c < D; ++c) v += JinvT[js + Nq * (r + D * c)] * gh[c];
            v -= ge[r];
            gerr2 += v * v;
            ge2 += ge[r] * ge[r];
        }
        s[0] += w * e * e;
        s[1] += w * ue * ue;
        s[2] += w * (wt_dt * de * de + nu * gerr2);
        s[3] += w * (wt_dt * dte * dte + nu * ge2);
    }
    __shared__ double red[4][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c = 0; c < 4; ++c) {
        double v = s[c];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) red[c][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double v = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
        partial[blockIdx.x * 4 + threadIdx.x] = v;
    }
}

int grid_for(long long total) {
    long long b = (total + 255) / 256;
    return static_cast<int>(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

cudaError_t launch_qgrid_geometry(const PhysicalDesc& g, const double* const* qnode, const double* const* qweight,
                                  const int* Q, double* x, double* wdet, double* JinvT, int* bad, cudaStream_t st) {
    long long Nq = 1;
    for (int l = 0; l < g.d; ++l) Nq *= Q[l];
    const int blocks = grid_for(Nq);
    const double* n[3] = {qnode[0], g.d > 1 ? qnode[1] : nullptr, g.d > 2 ? qnode[2] : nullptr};
    const double* w[3] = {qweight[0], g.d > 1 ? qweight[1] : nullptr, g.d > 2 ? qweight[2] : nullptr};
    const int q1 = g.d > 1 ? Q[1] : 1, q2 = g.d > 2 ? Q[2] : 1;
    switch (g.d) {
        case 1: qgrid_geometry_kernel<1><<<blocks, 256, 0, st>>>(g, n[0], n[1], n[2], w[0], w[1], w[2], Q[0], q1, q2, x, wdet, JinvT, bad); break;
        case 2: qgrid_geometry_kernel<2><<<blocks, 256, 0, st>>>(g, n[0], n[1], n[2], w[0], w[1], w[2], Q[0], q1, q2, x, wdet, JinvT, bad); break;
        case 3: qgrid_geometry_kernel<3><<<blocks, 256, 0, st>>>(g, n[0], n[1], n[2], w[0], w[1], w[2], Q[0], q1, q2, x, wdet, JinvT, bad); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_rhs_eval(int d, int kind, long long Nq, const double* x, const double* wdet, const double* tnode,
                            const double* tweight, int nb, double T, double* F, cudaStream_t st) {
    const int blocks = grid_for(Nq * nb);
    switch (d) {
        case 1: rhs_eval_kernel<1><<<blocks, 256, 0, st>>>(kind, Nq, x, wdet, tnode, tweight, nb, T, F); break;
        case 2: rhs_eval_kernel<2><<<blocks, 256, 0, st>>>(kind, Nq, x, wdet, tnode, tweight, nb, T, F); break;
        case 3: rhs_eval_kernel<3><<<blocks, 256, 0, st>>>(kind, Nq, x, wdet, tnode, tweight, nb, T, F); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_colloc(long long L, int nin, long long R, int nout, const int* first, const double* tab, int p1,
                          const int* tlo, const int* thi, int qoff, bool transpose, double beta, const double* in,
                          double* out, cudaStream_t st) {
    const int blocks = grid_for(L * nout * R);
    if (transpose)
        colloc_tr_kernel<<<blocks, 256, 0, st>>>(L, nin, R, nout, first, tab, p1, tlo, thi, qoff, beta, in, out);
    else
        colloc_fwd_kernel<<<blocks, 256, 0, st>>>(L, nin, R, nout, first, tab, p1, qoff, in, out);
    return cudaGetLastError();
}

cudaError_t launch_error_terms(int d, int kind, long long Nq, int nb, const double* x, const double* wdet,
                               const double* JinvT, const double* V, const double* G0, const double* G1,
                               const double* G2, const double* Vt, const double* tnode, const double* tweight,
                               double T, double wt_dt, double nu, double* partial, int nblocks, cudaStream_t st) {
    switch (d) {
        case 1: error_terms_kernel<1><<<nblocks, 256, 0, st>>>(kind, Nq, nb, x, wdet, JinvT, V, G0, G1, G2, Vt, tnode, tweight, T, wt_dt, nu, partial); break;
        case 2: error_terms_kernel<2><<<nblocks, 256, 0, st>>>(kind, Nq, nb, x, wdet, JinvT, V, G0, G1, G2, Vt, tnode, tweight, T, wt_dt, nu, partial); break;
        case 3: error_terms_kernel<3><<<nblocks, 256, 0, st>>>(kind, Nq, nb, x, wdet, JinvT, V, G0, G1, G2, Vt, tnode, tweight, T, wt_dt, nu, partial); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace stiga
