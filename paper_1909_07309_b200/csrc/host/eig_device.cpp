// cuSOLVER backend of sym_eig for the preconditioner setup ("GPU-side setup"): the
// symmetric eigenproblems behind spd_generalized_eig (pencil.cpp:12-21, after the host Cholesky
// reduction), the split half-pencils of the folded directions and the Hermitian embedding of the
// time pencil (pencil.cpp:23-95) run as cusolverDnDsyevd on the current device.  The contract is the
// host solver's (ascending eigenvalues, orthonormal eigenvectors); the FD apply is invariant to the
// basis inside eigenvalue clusters, and the setup still refines the spatial eigenvalues by Rayleigh
// quotients (host/fdsetup.cpp).
#include "eig_device.hpp"

#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <stdexcept>
#include <string>

namespace stiga {

namespace {

void cs(cusolverStatus_t s, const char* what) {
    if (s != CUSOLVER_STATUS_SUCCESS) throw std::runtime_error(std::string("cuSOLVER ") + what + " failed (status " +
                                                               std::to_string(static_cast<int>(s)) + ")");
}
void cu(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Handle {
    cusolverDnHandle_t h = nullptr;
    Handle() { cs(cusolverDnCreate(&h), "create"); }
    ~Handle() {
        if (h) cusolverDnDestroy(h);
    }
};

template <typename T>
struct Dev {
    T* p = nullptr;
    explicit Dev(size_t n) { cu(cudaMalloc(&p, sizeof(T) * (n ? n : 1)), "cudaMalloc"); }
    ~Dev() {
        if (p) cudaFree(p);
    }
};

}  // namespace

void sym_eig_cusolver(const DenseMatrix& A, Vector& w, DenseMatrix& Q) {
    const Index n = A.rows;
    if (A.cols != n) throw std::invalid_argument("sym_eig: matrix not square");
    w.assign(static_cast<size_t>(n), 0.0);
    Q = DenseMatrix(n, n);
    if (n == 0) return;
    // symmetrize as the host solver does (lower triangle is what syevd reads)
    DenseMatrix T = A;
    for (Index j = 0; j < n; ++j)
        for (Index i = j + 1; i < n; ++i) {
            const double s = 0.5 * (T(i, j) + T(j, i));
            T(i, j) = s;
            T(j, i) = s;
        }
    static thread_local Handle handle;
    const int ni = static_cast<int>(n);
    Dev<double> dA(static_cast<size_t>(n) * n), dW(static_cast<size_t>(n));
    Dev<int> dInfo(1);
    cu(cudaMemcpy(dA.p, T.a.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice), "upload");
    int lwork = 0;
    cs(cusolverDnDsyevd_bufferSize(handle.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, ni, dA.p, ni, dW.p,
                                   &lwork),
       "syevd_bufferSize");
    Dev<double> work(static_cast<size_t>(lwork));
    cs(cusolverDnDsyevd(handle.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, ni, dA.p, ni, dW.p, work.p, lwork,
                        dInfo.p),
       "syevd");
    int info = 0;
    cu(cudaMemcpy(&info, dInfo.p, sizeof(int), cudaMemcpyDeviceToHost), "download");
    if (info != 0) throw std::runtime_error("sym_eig: cuSOLVER syevd did not converge (info " + std::to_string(info) + ")");
    cu(cudaMemcpy(w.data(), dW.p, sizeof(double) * n, cudaMemcpyDeviceToHost), "download");
    cu(cudaMemcpy(Q.a.data(), dA.p, sizeof(double) * n * n, cudaMemcpyDeviceToHost), "download");
}

}  // namespace stiga
