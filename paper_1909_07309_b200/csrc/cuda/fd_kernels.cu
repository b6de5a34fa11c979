// Elementwise kernels of the FD apply: the standalone block-arrowhead solve (split time variant),
// the D^-1/2 scale pass and the block copies of the sharded transposes.  The mode products live in
// fd_mode*.cu, the time-fused kernel in fd_time*.cu (shared helpers: fd_common.cuh).
#include "fd_common.cuh"

namespace stiga {
namespace gpu {

namespace {

// Standalone block-arrowhead solve (fdsolve.cpp:24-65) between two time-mode products.  Block =
// 32 consecutive spatial indices (one per lane, coalesced) x P warps; warp w handles pairs
// j = w mod P.  Forward pass: pair eliminations accumulate the Schur right-hand side (reduced over
// the P warps in smem); second pass recomputes y_j from Z instead of storing it (24 B/DoF of HBM
// traffic instead of 32) and writes x_j = y_j - H_j^-1 B_j x_last.
template <int P>
__global__ void __launch_bounds__(32 * P) arrowhead_kernel(const double* __restrict__ Z, double* __restrict__ Xo,
                                                           long long Ns, ArrowParams ap) {
    __shared__ double part_s[P][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long s0 = static_cast<long long>(blockIdx.x) * 32 + lane;
    const bool valid = s0 < Ns;
    const long long s = valid ? s0 : Ns - 1;
    double lam = 0.0;  // ((0 + lambda_1) + lambda_2) + ... (fdsolve.cpp:91-99)
    long long rem = s + ap.s_off;  // global spatial index (slab offset in the sharded apply)
    for (int l = 0; l < ap.d; ++l) {
        const long long q = rem / ap.n[l];
        lam = lam + __ldg(ap.lam[l] + (rem - q * ap.n[l]));
        rem = q;
    }
    const double linv = 1.0 / lam;
    const double nu = ap.nu, inv_nu = ap.inv_nu, gam = ap.gamma;
    const double nulam = nu * lam;
    const int nt = ap.n_t;
    const double* zc = Z + s;
    double part = 0.0;
#pragma unroll 4
    for (int j = w; j < ap.npairs; j += P) {
        double xa, xb;
        const double rinv = pair_rinv(nulam, linv, __ldg(ap.pair_c + j));
        pair_apply(rinv, linv, inv_nu, __ldg(ap.pair_c1 + j), __ldg(ap.pair_c1sq + j), __ldg(zc + (2 * j) * Ns),
                   __ldg(zc + (2 * j + 1) * Ns), xa, xb);
        part = fma(__ldg(ap.pair_gg + 2 * j), xa, fma(__ldg(ap.pair_gg + 2 * j + 1), xb, part));
    }
    double xz = 0.0;
    const int z = nt - 2;
    if (ap.zero_count && w == P - 1) {
        xz = linv * __ldg(zc + z * Ns) * inv_nu;
        part += gam * __ldg(ap.g + z) * xz;
    }
    part_s[w][lane] = part;
    __syncthreads();
    double srhs = __ldg(zc + (nt - 1) * Ns);
#pragma unroll
    for (int k = 0; k < P; ++k) srhs += part_s[k][lane];
    const double xlast = __ldg(ap.S_inv + ap.s_off + s) * srhs;
    if (!valid) return;
    double* xo = Xo + s;
#pragma unroll 4
    for (int j = w; j < ap.npairs; j += P) {
        const double c1 = __ldg(ap.pair_c1 + j), c1sq = __ldg(ap.pair_c1sq + j);
        const double rinv = pair_rinv(nulam, linv, __ldg(ap.pair_c + j));
        double ya, yb, ca, cb;
        pair_apply(rinv, linv, inv_nu, c1, c1sq, __ldg(zc + (2 * j) * Ns), __ldg(zc + (2 * j + 1) * Ns), ya, yb);
        pair_apply(rinv, linv, inv_nu, c1, c1sq, __ldg(ap.pair_gg + 2 * j) * xlast, __ldg(ap.pair_gg + 2 * j + 1) * xlast,
                   ca, cb);
        xo[(2 * j) * Ns] = ya - ca;
        xo[(2 * j + 1) * Ns] = yb - cb;
    }
    if (w == P - 1) {
        if (ap.zero_count) xo[z * Ns] = xz - (gam * __ldg(ap.g + z) * inv_nu) * (linv * xlast);
        xo[(nt - 1) * Ns] = xlast;
    }
}

__global__ void scale_kernel(const double* __restrict__ a, const double* __restrict__ x, double* __restrict__ y,
                             long long n) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    const long long i0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(x) |
                           reinterpret_cast<uintptr_t>(y)) & 15u) == 0;
    if (aligned) {  // 16-byte vector path (slab offsets of the sharded apply can be odd)
        const long long n2 = n >> 1;
        const double2* a2 = reinterpret_cast<const double2*>(a);
        const double2* x2 = reinterpret_cast<const double2*>(x);
        double2* y2 = reinterpret_cast<double2*>(y);
        for (long long i = i0; i < n2; i += stride) {
            const double2 av = a2[i], xv = x2[i];
            y2[i] = make_double2(av.x * xv.x, av.y * xv.y);
        }
        if (i0 == 0 && (n & 1)) y[n - 1] = a[n - 1] * x[n - 1];
    } else {
        for (long long i = i0; i < n; i += stride) y[i] = a[i] * x[i];
    }
}


}  // namespace

cudaError_t launch_arrowhead(const double* Z, double* X, long long Ns, const ArrowParams& ap, cudaStream_t st) {
    if (Ns <= 0) return cudaSuccess;
    constexpr int P = 8;
    const long long blocks = (Ns + 31) / 32;
    arrowhead_kernel<P><<<static_cast<unsigned>(blocks), 32 * P, 0, st>>>(Z, X, Ns, ap);
    return cudaGetLastError();
}

__global__ void copy_blocks_kernel(const double* __restrict__ src, long long sld, double* __restrict__ dst,
                                   long long dld, long long rows, long long cols) {
    const long long total = rows * cols;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = e / cols, c = e - r * cols;
        dst[r * dld + c] = src[r * sld + c];
    }
}

cudaError_t launch_copy_blocks(const double* src, long long sld, double* dst, long long dld, long long rows,
                               long long cols, cudaStream_t st) {
    const long long total = rows * cols;
    if (total <= 0) return cudaSuccess;
    const long long blocks = std::min<long long>((total + 255) / 256, 148LL * 16);
    copy_blocks_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(src, sld, dst, dld, rows, cols);
    return cudaGetLastError();
}

cudaError_t launch_scale(const double* a, const double* x, double* y, long long n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int threads = 256;
    const long long blocks = std::min<long long>((n / 2 + threads - 1) / threads + 1, 148LL * 8);
    scale_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(a, x, y, n);
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace stiga

