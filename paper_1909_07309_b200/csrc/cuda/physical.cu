// Physical spatial stiffness / mass assembly (one CTA per element, geometry evaluated in-kernel)
// and the stencil SpMM of the space-time system mat-vec.  See physical.cuh.
#include "physical.cuh"

#include <algorithm>

namespace stiga {
namespace gpu {

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr int kMaxP = 8;

__device__ __forceinline__ double field(int kind, const double* x) {
    switch (kind) {
        case kFieldSeparableNu: return 50.5 + 49.5 * x[1] / hypot(x[0], x[1]);                       // problems.cpp:224-227
        case kFieldDeformedKappa: return 1.0 + 0.5 * sin(2.0 * kPi * x[0]) * cos(2.0 * kPi * x[1]);   // BASELINE c4
        case kFieldDeformedC: return 1.0 + 0.25 * x[2];                                               // BASELINE c4
        default: return 1.0;
    }
}

// Knot t_i of the uniform open knot vector of degree p with ne elements.
__device__ __forceinline__ double uknot(int i, int p, int ne) {
    const int k = i - p;
    return k <= 0 ? 0.0 : (k >= ne ? 1.0 : static_cast<double>(k) / ne);
}

// Cox-De Boor values of the deg+1 functions non-zero on span k (bspline.cpp:14-29).
__device__ __forceinline__ void cox(int k, int deg, int p, int ne, double x, double* N) {
    double left[kMaxP + 1], right[kMaxP + 1];
    N[0] = 1.0;
    for (int j = 1; j <= deg; ++j) {
        left[j] = x - uknot(k + 1 - j, p, ne);
        right[j] = uknot(k + j, p, ne) - x;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            const double den = right[r + 1] + left[j - r];
            const double temp = den != 0.0 ? N[r] / den : 0.0;
            N[r] = saved + right[r + 1] * temp;
            saved = left[j - r] * temp;
        }
        N[j] = saved;
    }
}

// Values and first derivatives of the p+1 B-splines at x (bspline.cpp:100-130); returns first index.
__device__ __forceinline__ int basis(double x, int p, int ne, double* val, double* der) {
    int e = static_cast<int>(floor(x * ne));
    e = min(max(e, 0), ne - 1);
    const int k = e + p;
    cox(k, p, p, ne, x, val);
    double low[kMaxP + 1];
    if (p == 1) low[0] = 1.0;
    else cox(k, p - 1, p, ne, x, low);
    for (int r = 0; r <= p; ++r) {
        const int i = k - p + r;
        double dv = 0.0;
        if (r > 0) {
            const double den = uknot(i + p, p, ne) - uknot(i, p, ne);
            if (den != 0.0) dv += low[r - 1] / den;
        }
        if (r < p) {
            const double den = uknot(i + p + 1, p, ne) - uknot(i + 1, p, ne);
            if (den != 0.0) dv -= low[r] / den;
        }
        der[r] = p * dv;
    }
    return k - p;
}

// F(eta) and J = dF/deta (geometry.cpp:41-97) of the uniform-knot spline map.
template <int D>
__device__ void geometry_eval(const PhysicalDesc& g, const double* eta, double* x, double* J) {
    double val[D][kMaxP + 1], der[D][kMaxP + 1];
    int first[D];
    for (int l = 0; l < D; ++l) first[l] = basis(eta[l], g.pg, g.neg, val[l], der[l]);
    for (int c = 0; c < D; ++c) x[c] = 0.0;
    for (int i = 0; i < D * D; ++i) J[i] = 0.0;
    const int m = g.neg + g.pg;  // basis functions per direction
    int idx[D];
    for (int l = 0; l < D; ++l) idx[l] = 0;
    while (true) {
        long long row = 0, stride = 1;
        for (int l = 0; l < D; ++l) {
            row += (first[l] + idx[l]) * stride;
            stride *= m;
        }
        double w = 1.0;
        for (int l = 0; l < D; ++l) w *= val[l][idx[l]];
        for (int r = 0; r < D; ++r) x[r] += w * g.cp[row + g.ncp * r];
        for (int c = 0; c < D; ++c) {
            double wc = 1.0;
            for (int l = 0; l < D; ++l) wc *= (l == c) ? der[l][idx[l]] : val[l][idx[l]];
            for (int r = 0; r < D; ++r) J[r + D * c] += wc * g.cp[row + g.ncp * r];
        }
        int l = 0;
        while (l < D && ++idx[l] > g.pg) idx[l++] = 0;
        if (l == D) break;
    }
}

template <int D>
__device__ __forceinline__ double det_inv(const double* J, double* Ji) {
    if (D == 1) {
        Ji[0] = 1.0 / J[0];
        return J[0];
    } else if (D == 2) {
        const double det = J[0] * J[3] - J[2] * J[1];
        Ji[0] = J[3] / det;
        Ji[3] = J[0] / det;
        Ji[2] = -J[2] / det;
        Ji[1] = -J[1] / det;
        return det;
    } else {
        auto a = [&](int r, int c) { return J[r + 3 * c]; };
        const double det = a(0, 0) * (a(1, 1) * a(2, 2) - a(2, 1) * a(1, 2)) -
                           a(0, 1) * (a(1, 0) * a(2, 2) - a(2, 0) * a(1, 2)) +
                           a(0, 2) * (a(1, 0) * a(2, 1) - a(2, 0) * a(1, 1));
        Ji[0 + 3 * 0] = (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) / det;
        Ji[0 + 3 * 1] = -(a(0, 1) * a(2, 2) - a(0, 2) * a(2, 1)) / det;
        Ji[0 + 3 * 2] = (a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1)) / det;
        Ji[1 + 3 * 0] = -(a(1, 0) * a(2, 2) - a(1, 2) * a(2, 0)) / det;
        Ji[1 + 3 * 1] = (a(0, 0) * a(2, 2) - a(0, 2) * a(2, 0)) / det;
        Ji[1 + 3 * 2] = -(a(0, 0) * a(1, 2) - a(0, 2) * a(1, 0)) / det;
        Ji[2 + 3 * 0] = (a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0)) / det;
        Ji[2 + 3 * 1] = -(a(0, 0) * a(2, 1) - a(0, 1) * a(2, 0)) / det;
        Ji[2 + 3 * 2] = (a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0)) / det;
        return det;
    }
}

// One CTA per element: quadrature-point geometry factors G = w det nu J^-1 J^-T and w det gamma in
// smem, then every (a, b) pair of local functions, atomically added into the stencil rows.
template <int D>
__global__ void __launch_bounds__(256) physical_assembly_kernel(PhysicalDesc g, double* Kst, double* Mst) {
    constexpr int NG = D * (D + 1) / 2 + 1;  // unique G entries + mass weight
    extern __shared__ double sm[];
    const int q = g.q, P1 = g.p + 1;
    int QD = 1, LD = 1;
    for (int l = 0; l < D; ++l) {
        QD *= q;
        LD *= P1;
    }
    double* gq = sm;                     // QD x NG
    double* tv = gq + QD * NG;           // D x q x P1 values
    double* td = tv + D * q * P1;        // D x q x P1 derivatives
    int* firstl = reinterpret_cast<int*>(td + D * q * P1);  // D
    int e[D];
    {
        long long rem = blockIdx.x;
        for (int l = 0; l < D; ++l) {
            e[l] = static_cast<int>(rem % g.n_el);
            rem /= g.n_el;
        }
    }
    for (int i = threadIdx.x; i < D * q * P1; i += blockDim.x) {
        const int l = i / (q * P1), r = i % (q * P1);
        const int src = (e[l] * q) * P1 + r;
        tv[i] = g.bval[src];
        td[i] = g.bder[src];
    }
    if (threadIdx.x < D) firstl[threadIdx.x] = g.bfirst[e[threadIdx.x] * q];
    for (int qi = threadIdx.x; qi < QD; qi += blockDim.x) {
        double eta[D], w = 1.0;
        int rem = qi;
        for (int l = 0; l < D; ++l) {
            const int jl = rem % q;
            rem /= q;
            eta[l] = g.qnode[e[l] * q + jl];
            w *= g.qweight[e[l] * q + jl];
        }
        double x[D], J[D * D], Ji[D * D];
        geometry_eval<D>(g, eta, x, J);
        const double det = det_inv<D>(J, Ji);
        const double nu = field(g.nu_kind, x), gam = field(g.gamma_kind, x);
        int k = 0;
        for (int r = 0; r < D; ++r)
            for (int c = r; c < D; ++c) {
                double s = 0.0;  // (J^-1 J^-T)_{rc} = sum_m Ji[r][m] Ji[c][m]
                for (int m = 0; m < D; ++m) s += Ji[r + D * m] * Ji[c + D * m];
                gq[qi * NG + k++] = w * det * nu * s;
            }
        gq[qi * NG + NG - 1] = w * det * gam;
    }
    __syncthreads();
    const int W = 2 * g.p + 1;
    long long ostride[D], nstride[D];
    {
        long long o = 1, s = 1;
        for (int l = 0; l < D; ++l) {
            ostride[l] = o;
            nstride[l] = s;
            o *= W;
            s *= g.n;
        }
    }
    const long long S = ostride[D - 1] * W;
    for (int pair = threadIdx.x; pair < LD * LD; pair += blockDim.x) {
        const int ia = pair % LD, ib = pair / LD;
        int a[D], b[D], ga[D], gb[D];
        bool ok = true;
        {
            int ra = ia, rb = ib;
            for (int l = 0; l < D; ++l) {
                a[l] = ra % P1;
                ra /= P1;
                b[l] = rb % P1;
                rb /= P1;
                ga[l] = firstl[l] + a[l];
                gb[l] = firstl[l] + b[l];
                ok = ok && ga[l] >= 0 && ga[l] < g.n && gb[l] >= 0 && gb[l] < g.n;
            }
        }
        if (!ok) continue;
        double kab = 0.0, mab = 0.0;
        for (int qi = 0; qi < QD; ++qi) {
            int j[D];
            int rem = qi;
            for (int l = 0; l < D; ++l) {
                j[l] = rem % q;
                rem /= q;
            }
            double va = 1.0, vb = 1.0, da[D], db[D];
            for (int c = 0; c < D; ++c) da[c] = db[c] = 1.0;
            for (int l = 0; l < D; ++l) {
                const double vla = tv[(l * q + j[l]) * P1 + a[l]], dla = td[(l * q + j[l]) * P1 + a[l]];
                const double vlb = tv[(l * q + j[l]) * P1 + b[l]], dlb = td[(l * q + j[l]) * P1 + b[l]];
                va *= vla;
                vb *= vlb;
                for (int c = 0; c < D; ++c) {
                    da[c] *= (c == l) ? dla : vla;
                    db[c] *= (c == l) ? dlb : vlb;
                }
            }
            const double* G = gq + qi * NG;
            double s = 0.0;
            int k = 0;
            for (int r = 0; r < D; ++r)
                for (int c = r; c < D; ++c) {
                    const double gv = G[k++];
                    s += (r == c) ? gv * da[r] * db[r] : gv * (da[r] * db[c] + da[c] * db[r]);
                }
            kab += s;
            mab += G[NG - 1] * va * vb;
        }
        long long row = 0, off = 0;
        for (int l = 0; l < D; ++l) {
            row += ga[l] * nstride[l];
            off += (gb[l] - ga[l] + g.p) * ostride[l];
        }
        atomicAdd(Kst + row * S + off, kab);
        atomicAdd(Mst + row * S + off, mab);
    }
}

// y[i, t] = sum_o Mst[i][o] P[j(i,o), t] + Kst[i][o] Q[j(i,o), t] for TB time columns per thread.
template <int D, int TB>
__global__ void __launch_bounds__(128) stencil_spmm2_kernel(PhysicalDesc g, const double* __restrict__ Mst,
                                                            const double* __restrict__ P, const double* __restrict__ Kst,
                                                            const double* __restrict__ Q, double* __restrict__ y,
                                                            long long n_t) {
    long long Ns = 1;
    for (int l = 0; l < D; ++l) Ns *= g.n;
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long t0 = static_cast<long long>(blockIdx.y) * TB;
    if (i >= Ns) return;
    const int W = 2 * g.p + 1;
    int il[D], lo[D], hi[D];
    long long nstride[D], ostride[D];
    {
        long long rem = i, s = 1, o = 1;
        for (int l = 0; l < D; ++l) {
            il[l] = static_cast<int>(rem % g.n);
            rem /= g.n;
            lo[l] = max(0, il[l] - g.p) - il[l] + g.p;
            hi[l] = min(g.n - 1, il[l] + g.p) - il[l] + g.p;
            nstride[l] = s;
            ostride[l] = o;
            s *= g.n;
            o *= W;
        }
    }
    const long long S = ostride[D - 1] * W;
    const int tb = static_cast<int>(min(static_cast<long long>(TB), n_t - t0));
    double acc[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) acc[k] = 0.0;
    const double* mrow = Mst + i * S;
    const double* krow = Kst + i * S;
    int o[D];
    for (int l = 0; l < D; ++l) o[l] = lo[l];
    while (true) {
        long long off = 0, j = 0;
        for (int l = 0; l < D; ++l) {
            off += o[l] * ostride[l];
            j += (il[l] + o[l] - g.p) * nstride[l];
        }
        const double mv = __ldg(mrow + off), kv = __ldg(krow + off);
        const double* pc = P + j + Ns * t0;
        const double* qc = Q + j + Ns * t0;
        if (tb == TB) {
#pragma unroll
            for (int k = 0; k < TB; ++k) acc[k] += mv * __ldg(pc + Ns * k) + kv * __ldg(qc + Ns * k);
        } else {
#pragma unroll
            for (int k = 0; k < TB; ++k)
                if (k < tb) acc[k] += mv * __ldg(pc + Ns * k) + kv * __ldg(qc + Ns * k);
        }
        int l = 0;
        while (l < D && ++o[l] > hi[l]) {
            o[l] = lo[l];
            ++l;
        }
        if (l == D) break;
    }
#pragma unroll
    for (int k = 0; k < TB; ++k)
        if (k < tb) y[i + Ns * (t0 + k)] = acc[k];
}

template <int D>
__global__ void stencil_diag_kernel(PhysicalDesc g, const double* Kst, const double* Mst, double* dK, double* dM) {
    long long Ns = 1, S = 1, c = 0, o = 1;
    for (int l = 0; l < D; ++l) {
        Ns *= g.n;
        c += g.p * o;
        o *= 2 * g.p + 1;
    }
    S = o;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < Ns;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        dK[i] = Kst[i * S + c];
        dM[i] = Mst[i * S + c];
    }
}

template <int D>
cudaError_t assembly_d(const PhysicalDesc& g, double* Kst, double* Mst, cudaStream_t st) {
    long long elems = 1;
    int QD = 1;
    for (int l = 0; l < D; ++l) {
        elems *= g.n_el;
        QD *= g.q;
    }
    constexpr int NG = D * (D + 1) / 2 + 1;
    const size_t smem = sizeof(double) * (QD * NG + 2 * D * g.q * (g.p + 1)) + sizeof(int) * D;
    cudaError_t e = cudaFuncSetAttribute(physical_assembly_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    physical_assembly_kernel<D><<<static_cast<unsigned>(elems), 256, smem, st>>>(g, Kst, Mst);
    return cudaGetLastError();
}

template <int D>
cudaError_t spmm_d(const PhysicalDesc& g, const double* Mst, const double* P, const double* Kst, const double* Q,
                   double* y, long long n_t, cudaStream_t st) {
    constexpr int TB = 24;
    long long Ns = 1;
    for (int l = 0; l < D; ++l) Ns *= g.n;
    dim3 grid(static_cast<unsigned>((Ns + 127) / 128), static_cast<unsigned>((n_t + TB - 1) / TB));
    stencil_spmm2_kernel<D, TB><<<grid, 128, 0, st>>>(g, Mst, P, Kst, Q, y, n_t);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_physical_assembly(const PhysicalDesc& g, double* Kst, double* Mst, cudaStream_t st) {
    if (g.p > kMaxP || g.pg > kMaxP) return cudaErrorInvalidValue;
    switch (g.d) {
        case 1: return assembly_d<1>(g, Kst, Mst, st);
        case 2: return assembly_d<2>(g, Kst, Mst, st);
        case 3: return assembly_d<3>(g, Kst, Mst, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_stencil_spmm2(const PhysicalDesc& g, const double* Mst, const double* P, const double* Kst,
                                 const double* Q, double* y, long long n_t, cudaStream_t st) {
    switch (g.d) {
        case 1: return spmm_d<1>(g, Mst, P, Kst, Q, y, n_t, st);
        case 2: return spmm_d<2>(g, Mst, P, Kst, Q, y, n_t, st);
        case 3: return spmm_d<3>(g, Mst, P, Kst, Q, y, n_t, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_stencil_diag(const PhysicalDesc& g, const double* Kst, const double* Mst, double* dK, double* dM,
                                cudaStream_t st) {
    const unsigned blocks = 148 * 8;
    switch (g.d) {
        case 1: stencil_diag_kernel<1><<<blocks, 256, 0, st>>>(g, Kst, Mst, dK, dM); break;
        case 2: stencil_diag_kernel<2><<<blocks, 256, 0, st>>>(g, Kst, Mst, dK, dM); break;
        case 3: stencil_diag_kernel<3><<<blocks, 256, 0, st>>>(g, Kst, Mst, dK, dM); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace stiga
