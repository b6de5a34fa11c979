// Banded Kronecker passes for the space-time system mat-vec (KronSumOperator::apply,
// kronop.cpp:108-115, applied sum-factorized over the kron_sum_terms structure of
// solver.cpp:10-30), GMRES BLAS-1 kernels (gmres.cpp:76-85,121) and the FP64 peak probe.
// All of these are HBM-bound streaming kernels: grid-stride loops, coalesced along the
// fastest tensor index, 148 SMs x 8 resident blocks.
#include "aux_kernels.cuh"

#include <algorithm>
#include <chrono>

namespace stiga {
namespace gpu {

namespace {

constexpr int kThreads = 256;
constexpr int kDotBlocks = 148 * 4;

inline unsigned grid_for(long long n) {
    const long long b = (n + kThreads - 1) / kThreads;
    return static_cast<unsigned>(std::max(1LL, std::min(b, 148LL * 16)));
}

__device__ __forceinline__ double band_row(const Band& B, const double* __restrict__ in, long long base, long long L,
                                           int i, int n) {
    const int w = 2 * B.p + 1;
    const double* row = B.band + static_cast<long long>(i) * w;
    const int jlo = max(0, i - B.p), jhi = min(n - 1, i + B.p);
    double s = 0.0;
    for (int j = jlo; j <= jhi; ++j) s += __ldg(row + (j - i + B.p)) * __ldg(in + base + L * j);
    return s;
}

__global__ void banded_pass_kernel(ModeGeom g, const double* __restrict__ in0, const double* __restrict__ in1,
                                   double* __restrict__ out0, double* __restrict__ out1, Band A, Band B, Band C,
                                   Band D, double beta0) {
    const long long total = g.ncols * g.n;
    const long long Ln = g.L * g.n;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = e / Ln;
        const long long rem = e - r * Ln;
        const int i = static_cast<int>(rem / g.L);
        const long long l = rem - static_cast<long long>(i) * g.L;
        const long long base = l + Ln * r;
        double s0 = 0.0;
        if (A.band) s0 += band_row(A, in0, base, g.L, i, g.n);
        if (B.band) s0 += band_row(B, in1, base, g.L, i, g.n);
        if (beta0 != 0.0) s0 += beta0 * out0[e];
        out0[e] = s0;
        if (out1) {
            double s1 = 0.0;
            if (C.band) s1 += band_row(C, in0, base, g.L, i, g.n);
            if (D.band) s1 += band_row(D, in1, base, g.L, i, g.n);
            out1[e] = s1;
        }
    }
}

// Time-banded pass on a time slab with halos (sharded system mat-vec):
// y[s, r] = sum_j A[t0 + r][j] a[s, j - t0 + hl] + B[t0 + r][j] b[s, j - t0 + hl], |j - (t0 + r)| <= p.
__global__ void time_band_slab_kernel(long long Ns, int nt, long long t0, long long ntl, int hl,
                                      const double* __restrict__ a, const double* __restrict__ b,
                                      double* __restrict__ y, Band A, Band B) {
    const long long total = Ns * ntl;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = e / Ns;
        const long long s = e - r * Ns;
        const int i = static_cast<int>(t0 + r);
        const long long base = s + Ns * (hl - t0);  // a[s, j - t0 + hl] = a[base + Ns j]
        double v = 0.0;
        if (A.band) v += band_row(A, a, base, Ns, i, nt);
        if (B.band) v += band_row(B, b, base, Ns, i, nt);
        y[e] = v;
    }
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void dot_partial_kernel(const double* __restrict__ x, const double* __restrict__ y, long long n,
                                   double* __restrict__ partials) {
    __shared__ double ws[32];
    double s = 0.0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        s += x[i] * y[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) partials[blockIdx.x] = v;
    }
}

__global__ void dot_finish_kernel(const double* __restrict__ partials, int np, double* __restrict__ result) {
    __shared__ double ws[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) s += partials[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) *result = v;
    }
}

__global__ void axpy_kernel(double alpha, const double* __restrict__ x, double* __restrict__ y, long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        y[i] += alpha * x[i];
}

__global__ void scal_kernel(double alpha, const double* __restrict__ x, double* __restrict__ y, long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        y[i] = alpha * x[i];
}

__global__ void sub_kernel(const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ z,
                           long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        z[i] = x[i] - y[i];
}

__global__ void peak_dfma_kernel(double* out, int iters, double a, double b) {
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.678) out[0] = s;
}

__global__ void peak_dmma_kernel(double* out, int iters) {
    const double a = threadIdx.x * 1e-3, b = 0.5;
    double c[8][2];
    for (int i = 0; i < 8; ++i) {
        c[i][0] = i;
        c[i][1] = -i;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[i][0]), "+d"(c[i][1])
                             : "d"(a), "d"(b));
    }
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

}  // namespace

cudaError_t launch_banded_pass(const ModeGeom& g, const double* in0, const double* in1, double* out0, double* out1,
                               Band A, Band B, Band C, Band D, double beta0, cudaStream_t st) {
    const long long total = g.ncols * g.n;
    if (total <= 0) return cudaSuccess;
    banded_pass_kernel<<<grid_for(total), kThreads, 0, st>>>(g, in0, in1, out0, out1, A, B, C, D, beta0);
    return cudaGetLastError();
}

cudaError_t launch_time_band_slab(long long Ns, int nt, long long t0, long long ntl, int hl, const double* a,
                                  const double* b, double* y, Band A, Band B, cudaStream_t st) {
    const long long total = Ns * ntl;
    if (total <= 0) return cudaSuccess;
    time_band_slab_kernel<<<grid_for(total), kThreads, 0, st>>>(Ns, nt, t0, ntl, hl, a, b, y, A, B);
    return cudaGetLastError();
}

int dot_partials_size() { return kDotBlocks; }

cudaError_t launch_dot(const double* x, const double* y, long long n, double* d_partials, double* d_result,
                       cudaStream_t st) {
    dot_partial_kernel<<<kDotBlocks, kThreads, 0, st>>>(x, y, n, d_partials);
    dot_finish_kernel<<<1, 1024, 0, st>>>(d_partials, kDotBlocks, d_result);
    return cudaGetLastError();
}

cudaError_t launch_axpy(double alpha, const double* x, double* y, long long n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    axpy_kernel<<<grid_for(n), kThreads, 0, st>>>(alpha, x, y, n);
    return cudaGetLastError();
}

cudaError_t launch_scal(double alpha, const double* x, double* y, long long n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    scal_kernel<<<grid_for(n), kThreads, 0, st>>>(alpha, x, y, n);
    return cudaGetLastError();
}

cudaError_t launch_sub(const double* x, const double* y, double* z, long long n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    sub_kernel<<<grid_for(n), kThreads, 0, st>>>(x, y, z, n);
    return cudaGetLastError();
}

cudaError_t fp64_peak_probe(double ms, double* tf_dmma, double* tf_dfma) {
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(double));
    if (e != cudaSuccess) return e;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int tpb = 256, bps = 2;
    float t = 0.f;
    // calibrate iterations to ~ms
    int it = 200;
    peak_dmma_kernel<<<sms * bps, tpb>>>(d, it);
    cudaEventRecord(e0);
    peak_dmma_kernel<<<sms * bps, tpb>>>(d, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t, e0, e1);
    it = std::max(1, static_cast<int>(it * ms / std::max(t, 1e-3f)));
    cudaEventRecord(e0);
    peak_dmma_kernel<<<sms * bps, tpb>>>(d, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t, e0, e1);
    *tf_dmma = 2.0 * 256 * 32 * it * (tpb / 32.0) * sms * bps / (t * 1e-3) / 1e12;
    int itf = std::max(1, it * 2);
    cudaEventRecord(e0);
    peak_dfma_kernel<<<sms * bps, tpb>>>(d, itf, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t, e0, e1);
    *tf_dfma = 2.0 * 128 * static_cast<double>(itf) * tpb * sms * bps / (t * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace stiga
