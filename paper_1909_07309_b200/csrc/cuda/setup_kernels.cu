// Device half of the preconditioner setup.  See setup_kernels.cuh.
#include "setup_kernels.cuh"

namespace stiga {
namespace gpu {

namespace {

constexpr int kMaxTerms = 8;

struct KronDiag {
    int D = 0, nterms = 0;
    int dims[kSetupMaxDim + 1] = {};
    double c[kMaxTerms] = {};
    const double* dg[kMaxTerms][kSetupMaxDim + 1] = {};
};

int blocks_for(long long n) {
    const long long b = (n + 255) / 256;
    return static_cast<int>(b < 148 * 32 ? (b < 1 ? 1 : b) : 148 * 32);
}

// fdsolve.cpp:91-136 per spatial index s, in the host's operation order (host/fdsetup.cpp)
__global__ void __launch_bounds__(256) schur_inv_kernel(SchurArgs a, long long Ns, double* __restrict__ S_inv,
                                                         int* flag) {
    for (long long s = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; s < Ns;
         s += static_cast<long long>(gridDim.x) * blockDim.x) {
        // Lambda_s = ((0 + lambda_1) + lambda_2) + lambda_3 (kron_sum_eigenvalues, fdsolve.cpp:91-99)
        long long rem = s;
        double ls = 0.0;
        for (int l = 0; l < a.d; ++l) {
            const long long i = rem % a.n[l];
            rem /= a.n[l];
            ls = __dadd_rn(ls, a.lam[l][i]);
        }
        if (!(ls > 0.0)) atomicOr(flag, 1);
        const double li = __ddiv_rn(1.0, ls);
        double S = __dadd_rn(a.gs, __dmul_rn(a.nu, ls));
        const double nls = __dmul_rn(a.nu, ls);
        const double lin = __ddiv_rn(li, a.nu);
        const double li2 = __dmul_rn(li, li);
        for (int j = 0; j < a.npairs; ++j) {
            const double c = a.pc[4 * j], c1sq = a.pc[4 * j + 1], ga2 = a.pc[4 * j + 2], gb2 = a.pc[4 * j + 3];
            const double rinv = __ddiv_rn(1.0, __dadd_rn(nls, __dmul_rn(c, li)));
            const double Pd = __dsub_rn(lin, __dmul_rn(c1sq, __dmul_rn(li2, rinv)));
            S = __dadd_rn(S, __dmul_rn(a.gg, __dadd_rn(__dmul_rn(ga2, Pd), __dmul_rn(gb2, rinv))));
        }
        if (a.zero_block) S = __dadd_rn(S, __dmul_rn(a.cz, li));
        if (S == 0.0) atomicOr(flag, 2);
        S_inv[s] = __ddiv_rn(1.0, S);
    }
}

__global__ void __launch_bounds__(256) dinv_sqrt_kernel(const double* __restrict__ D, double* __restrict__ out,
                                                         long long n, int* flag) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double v = D[i];
        if (!(v > 0.0)) atomicOr(flag, 1);
        out[i] = __ddiv_rn(1.0, __dsqrt_rn(v));
    }
}

__global__ void __launch_bounds__(256) kron_diag_kernel(KronDiag k, const double* num, double* out, long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        long long idx[kSetupMaxDim + 1];
        long long rem = i;
        for (int l = 0; l < k.D; ++l) {
            idx[l] = rem % k.dims[l];
            rem /= k.dims[l];
        }
        double acc = 0.0;
        for (int t = 0; t < k.nterms; ++t) {
            double v = 1.0;
            for (int l = 0; l < k.D; ++l) v = __dmul_rn(k.dg[t][l][idx[l]], v);
            acc = t == 0 ? __dmul_rn(k.c[t], v) : __dadd_rn(acc, __dmul_rn(k.c[t], v));
        }
        out[i] = num ? __ddiv_rn(num[i], acc) : acc;
    }
}

__global__ void __launch_bounds__(256) physical_diag_kernel(const double* __restrict__ dM, const double* __restrict__ dK,
                                                            const double* __restrict__ W, const double* __restrict__ M,
                                                            long long Ns, int nt, const double* den, double* out) {
    const long long n = Ns * nt;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long t = i / Ns, s = i - t * Ns;
        const double v = __dadd_rn(__dmul_rn(dM[s], W[t]), __dmul_rn(dK[s], M[t]));
        out[i] = den ? __ddiv_rn(v, den[i]) : v;
    }
}

}  // namespace

cudaError_t launch_schur_inv(const SchurArgs& a, long long Ns, double* S_inv, int* flag, cudaStream_t st) {
    if (a.d < 1 || a.d > kSetupMaxDim) return cudaErrorInvalidValue;
    schur_inv_kernel<<<blocks_for(Ns), 256, 0, st>>>(a, Ns, S_inv, flag);
    return cudaGetLastError();
}

cudaError_t launch_dinv_sqrt(const double* D, double* out, long long n, int* flag, cudaStream_t st) {
    dinv_sqrt_kernel<<<blocks_for(n), 256, 0, st>>>(D, out, n, flag);
    return cudaGetLastError();
}

cudaError_t launch_kron_diag(int D, const int* dims, int nterms, const double* coeffs, const double* const* diags,
                             const double* num, double* out, long long n, cudaStream_t st) {
    if (D < 1 || D > kSetupMaxDim + 1 || nterms < 1 || nterms > kMaxTerms) return cudaErrorInvalidValue;
    KronDiag k;
    k.D = D;
    k.nterms = nterms;
    for (int l = 0; l < D; ++l) k.dims[l] = dims[l];
    for (int t = 0; t < nterms; ++t) {
        k.c[t] = coeffs[t];
        for (int l = 0; l < D; ++l) k.dg[t][l] = diags[t * D + l];
    }
    kron_diag_kernel<<<blocks_for(n), 256, 0, st>>>(k, num, out, n);
    return cudaGetLastError();
}

cudaError_t launch_physical_diag(const double* dM, const double* dK, const double* W, const double* M, long long Ns,
                                 int nt, const double* den, double* out, cudaStream_t st) {
    physical_diag_kernel<<<blocks_for(Ns * nt), 256, 0, st>>>(dM, dK, W, M, Ns, nt, den, out);
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace stiga
