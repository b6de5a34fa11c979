// FP64 tensor-core kernels of the extended-FD apply (sm_100a).
//
// Every mode product is a batch of small GEMMs  Y_fiber = J * X_fiber  with J the n x n
// eigenvector factor (n = 16..260).  One CTA owns BN fibers and ALL n output rows: the fiber
// tile (n x BN doubles) is staged once in shared memory with cp.async, J is streamed from L2
// in 16-column chunks through a 2-stage cp.async pipeline, and the products run on the FP64
// tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4; measured 36.9 TF/s on B200 vs 34.0 for
// DFMA, profiles/r01_fp64_peak.txt).  Each warp owns MI 8-row strips x NI 8-column tiles.
//
// The time-fused kernel keeps the tile resident across U_t^T, the block-arrowhead solve of
// fdsolve.cpp:24-65 (forward pair eliminations, diagonal Schur, back substitution) and U_t,
// so the time direction costs one HBM round trip instead of three.
#include "fd_kernels.cuh"

#include <algorithm>
#include <mutex>

namespace stiga {
namespace gpu {

namespace {

constexpr int kBK = 16;        // J columns per pipeline stage
constexpr int kLDJ = kBK + 4;  // smem row stride of a J stage (20 == 4 mod 16 -> conflict-free A fragments)
constexpr int kStages = 2;
constexpr int kMaxThreads = 384;

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = valid ? 8 : 0;  // src-size 0 -> zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct KArgs {
    ModeGeom geo;
    int S, Mp, Kp, Xrows, BN, LDX, WM, WN;
};

struct Smem {
    double* Xs;       // Kp x LDX fiber tile (rows = mode index j, cols = fiber)
    double* Js;       // kStages x Mp x kLDJ
    long long* colbase;  // input fiber offsets (BN)
    long long* obase;    // output fiber offsets (BN)
};

__device__ __forceinline__ Smem carve(const KArgs& a) {
    extern __shared__ __align__(16) double smem_raw[];
    Smem s;
    s.Xs = smem_raw;
    s.Js = s.Xs + static_cast<size_t>(a.Xrows) * a.LDX;
    s.colbase = reinterpret_cast<long long*>(s.Js + static_cast<size_t>(kStages) * a.Mp * kLDJ);
    s.obase = s.colbase + a.BN;
    return s;
}

// Global offset of element 0 of each fiber of the tile (c -> l + L*n*r).
__device__ __forceinline__ void compute_colbase(const KArgs& a, long long c0, long long* colbase, long long* obase) {
    for (int c = threadIdx.x; c < a.BN; c += blockDim.x) {
        long long cc = c0 + c;
        if (cc >= a.geo.ncols) cc = a.geo.ncols - 1;
        const long long r = cc / a.geo.L;
        const long long l = cc - r * a.geo.L;
        colbase[c] = l + a.geo.L * static_cast<long long>(a.geo.n) * r;
        obase[c] = l + a.geo.L * static_cast<long long>(a.geo.m) * r;
    }
}

// Issues the cp.async copies of the fiber tile (rows >= n are zeroed with plain stores).
__device__ __forceinline__ void load_tile(const KArgs& a, const Smem& sm, long long c0, const double* __restrict__ X) {
    const int n = a.geo.n;
    const int bn = static_cast<int>(min(static_cast<long long>(a.BN), a.geo.ncols - c0));
    const int total = n * a.BN;
    if (a.geo.L == 1) {
        const double* src = X + c0 * n;  // fibers contiguous
        for (int e = threadIdx.x; e < total; e += blockDim.x) {
            const int c = e / n;
            const int j = e - c * n;
            const bool v = c < bn;
            cp_async8(sm.Xs + j * a.LDX + c, v ? src + e : X, v);
        }
    } else {
        for (int e = threadIdx.x; e < total; e += blockDim.x) {
            const int j = e / a.BN;
            const int c = e - j * a.BN;
            const bool v = c < bn;
            cp_async8(sm.Xs + j * a.LDX + c, v ? X + sm.colbase[c] + a.geo.L * j : X, v);
        }
    }
    const int ztotal = (a.Kp - n) * a.BN;
    for (int e = threadIdx.x; e < ztotal; e += blockDim.x) {
        const int j = n + e / a.BN;
        sm.Xs[j * a.LDX + (e % a.BN)] = 0.0;
    }
}

// Multiplies the tile elements this thread copied by the matching entries of `scale`.
__device__ __forceinline__ void scale_own_tile(const KArgs& a, const Smem& sm, long long c0,
                                               const double* __restrict__ scale) {
    const int n = a.geo.n;
    const int bn = static_cast<int>(min(static_cast<long long>(a.BN), a.geo.ncols - c0));
    const int total = n * a.BN;
    if (a.geo.L == 1) {
        for (int e = threadIdx.x; e < total; e += blockDim.x) {
            const int c = e / n;
            const int j = e - c * n;
            if (c < bn) sm.Xs[j * a.LDX + c] *= __ldg(scale + c0 * n + e);
        }
    } else {
        for (int e = threadIdx.x; e < total; e += blockDim.x) {
            const int j = e / a.BN;
            const int c = e - j * a.BN;
            if (c < bn) sm.Xs[j * a.LDX + c] *= __ldg(scale + sm.colbase[c] + a.geo.L * j);
        }
    }
}

__device__ __forceinline__ void load_j_chunk(const KArgs& a, const Smem& sm, const double* __restrict__ Jg, int kc,
                                             int stage) {
    const int k0 = kc * kBK;
    const int pieces = min(kBK, a.Kp - k0) / 2;  // 16-byte pieces per row
    double* dst = sm.Js + static_cast<size_t>(stage) * a.Mp * kLDJ;
    const int total = a.Mp * pieces;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int r = e / pieces;
        const int p = e - r * pieces;
        cp_async16(dst + r * kLDJ + 2 * p, Jg + static_cast<size_t>(r) * a.Kp + k0 + 2 * p);
    }
}

// Issues the first two J chunks (two commit groups, possibly empty).
__device__ __forceinline__ void gemm_prologue(const KArgs& a, const Smem& sm, const double* __restrict__ Jg) {
    const int nchunks = (a.Kp + kBK - 1) / kBK;
    load_j_chunk(a, sm, Jg, 0, 0);
    cp_commit();
    if (nchunks > 1) load_j_chunk(a, sm, Jg, 1, 1);
    cp_commit();
}

// acc[mi][ni] += sum_k J[row][k] * Xs[k][col] over the full padded contraction length.
template <int MI, int NI>
__device__ __forceinline__ void gemm_main(const KArgs& a, const Smem& sm, const double* __restrict__ Jg,
                                          double (&acc)[MI][NI][2]) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int warp_m = warp % a.WM;
    const int warp_n = warp / a.WM;
    const int g = lane >> 2, t = lane & 3;
    const int nchunks = (a.Kp + kBK - 1) / kBK;
    const double* xb = sm.Xs + t * a.LDX + warp_n * NI * 8 + g;
    for (int kc = 0; kc < nchunks; ++kc) {
        cp_wait<1>();
        __syncthreads();
        const double* js = sm.Js + static_cast<size_t>(kc & 1) * a.Mp * kLDJ + (warp_m * MI * 8 + g) * kLDJ + t;
        const int k0 = kc * kBK;
        const int ksteps = min(kBK, a.Kp - k0) >> 2;
#pragma unroll
        for (int kk = 0; kk < kBK / 4; ++kk) {
            if (kk < ksteps) {
                double av[MI], bv[NI];
#pragma unroll
                for (int mi = 0; mi < MI; ++mi) av[mi] = js[mi * 8 * kLDJ + kk * 4];
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) bv[ni] = xb[(k0 + kk * 4) * a.LDX + ni * 8];
#pragma unroll
                for (int mi = 0; mi < MI; ++mi) {
                    if (warp_m * MI + mi < a.S) {
#pragma unroll
                        for (int ni = 0; ni < NI; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
                    }
                }
            }
        }
        __syncthreads();
        if (kc + 2 < nchunks) load_j_chunk(a, sm, Jg, kc + 2, kc & 1);
        cp_commit();
    }
}

// Writes the accumulator rows < row_limit into Xs (row = J row, col = fiber).
template <int MI, int NI>
__device__ __forceinline__ void acc_to_smem(const KArgs& a, const Smem& sm, const double (&acc)[MI][NI][2],
                                            int row_limit) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int warp_m = warp % a.WM;
    const int warp_n = warp / a.WM;
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
        const int row = (warp_m * MI + mi) * 8 + g;
        if (warp_m * MI + mi < a.S && row < row_limit) {
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
                const int col = (warp_n * NI + ni) * 8 + 2 * t;
                sm.Xs[row * a.LDX + col] = acc[mi][ni][0];
                sm.Xs[row * a.LDX + col + 1] = acc[mi][ni][1];
            }
        }
    }
}

// Coalesced store of the m x BN staged output tile (optionally scaled elementwise).
__device__ __forceinline__ void store_tile(const KArgs& a, const Smem& sm, long long c0, double* __restrict__ Y,
                                           const double* __restrict__ post) {
    const int m = a.geo.m;
    const int bn = static_cast<int>(min(static_cast<long long>(a.BN), a.geo.ncols - c0));
    if (a.geo.L == 1) {
        const int total = m * bn;
        double* dst = Y + c0 * m;
        for (int e = threadIdx.x; e < total; e += blockDim.x) {
            const int c = e / m;
            const int i = e - c * m;
            double v = sm.Xs[i * a.LDX + c];
            if (post) v *= __ldg(post + c0 * m + e);
            dst[e] = v;
        }
    } else {
        const int total = m * a.BN;
        for (int e = threadIdx.x; e < total; e += blockDim.x) {
            const int i = e / a.BN;
            const int c = e - i * a.BN;
            if (c < bn) {
                const long long gi = sm.obase[c] + a.geo.L * i;
                double v = sm.Xs[i * a.LDX + c];
                if (post) v *= __ldg(post + gi);
                Y[gi] = v;
            }
        }
    }
}

template <int MI, int NI>
__global__ void __launch_bounds__(kMaxThreads, 1)
    mode_product_kernel(KArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ Jg,
                        const double* __restrict__ pre, const double* __restrict__ post) {
    const Smem sm = carve(a);
    const long long c0 = static_cast<long long>(blockIdx.x) * a.BN;
    if (a.geo.L != 1) {
        compute_colbase(a, c0, sm.colbase, sm.obase);
        __syncthreads();
    }
    load_tile(a, sm, c0, X);
    cp_commit();
    gemm_prologue(a, sm, Jg);
    if (pre) {
        cp_wait<2>();  // this thread's tile copies have landed
        scale_own_tile(a, sm, c0, pre);
    }
    double acc[MI][NI][2];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    gemm_main<MI, NI>(a, sm, Jg, acc);
    // gemm_main ends with a barrier: Xs is free for the output staging
    acc_to_smem<MI, NI>(a, sm, acc, a.geo.m);
    __syncthreads();
    store_tile(a, sm, c0, Y, post);
}

// apply_pair_inverse (fdsolve.cpp:11-20) with R_j^-1 recomputed from Lambda_s (fdsolve.cpp:114-119).
__device__ __forceinline__ void pair_inverse(double lam, double linv, double nu, double cj, double c1, double u,
                                             double w, double& xa, double& xb) {
    const double rinv = 1.0 / (nu * lam + cj * linv);
    const double luiu = linv * u;
    const double riluiu = rinv * luiu;
    xa = luiu / nu - (c1 * c1 / nu) * (linv * riluiu) - c1 * (linv * (rinv * w));
    xb = c1 * riluiu + rinv * w;
}

// Block-arrowhead solve (fdsolve.cpp:24-65) on the resident tile: column c = one spatial
// eigen-index, rows = time eigen-coordinates.  P threads share a column (pairs j = p mod P).
__device__ __forceinline__ void arrowhead_tile(const KArgs& a, const Smem& sm, long long c0, const ArrowParams& ap) {
    int P = 1;
    while (P < 32 && 2 * P * a.BN <= static_cast<int>(blockDim.x)) P *= 2;
    const int tid = threadIdx.x;
    if (tid >= P * a.BN) return;  // whole warps (P*BN is a multiple of 32)
    const int c = tid / P;
    const int p = tid - c * P;
    long long s = c0 + c;
    if (s >= a.geo.ncols) s = a.geo.ncols - 1;
    double lam = 0.0;  // ((0 + lambda_1) + lambda_2) + ... (fdsolve.cpp:91-99)
    long long rem = s;
    for (int l = 0; l < ap.d; ++l) {
        const long long q = rem / ap.n[l];
        lam = lam + __ldg(ap.lam[l] + (rem - q * ap.n[l]));
        rem = q;
    }
    const double linv = 1.0 / lam;
    const double nu = ap.nu, gam = ap.gamma;
    const int nt = ap.n_t;
    const int LDX = a.LDX;
    double* col = sm.Xs + c;
    const double slast = col[(nt - 1) * LDX];
    double part = 0.0;
    for (int j = p; j < ap.npairs; j += P) {
        double xa, xb;
        pair_inverse(lam, linv, nu, __ldg(ap.pair_c + j), __ldg(ap.pair_c1 + j), col[(2 * j) * LDX],
                     col[(2 * j + 1) * LDX], xa, xb);
        col[(2 * j) * LDX] = xa;
        col[(2 * j + 1) * LDX] = xb;
        part += gam * (__ldg(ap.g + 2 * j) * xa + __ldg(ap.g + 2 * j + 1) * xb);
    }
    if (ap.zero_count && p == 0) {
        const int z = nt - 2;
        const double xz = linv * col[z * LDX] / nu;
        col[z * LDX] = xz;
        part += gam * __ldg(ap.g + z) * xz;
    }
    for (int off = P >> 1; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    const double xlast = __ldg(ap.S_inv + s) * (slast + part);
    for (int j = p; j < ap.npairs; j += P) {
        double xa, xb;
        pair_inverse(lam, linv, nu, __ldg(ap.pair_c + j), __ldg(ap.pair_c1 + j),
                     (gam * __ldg(ap.g + 2 * j)) * xlast, (gam * __ldg(ap.g + 2 * j + 1)) * xlast, xa, xb);
        col[(2 * j) * LDX] -= xa;
        col[(2 * j + 1) * LDX] -= xb;
    }
    if (p == 0) {
        if (ap.zero_count) {
            const int z = nt - 2;
            col[z * LDX] -= (gam * __ldg(ap.g + z) / nu) * (linv * xlast);
        }
        col[(nt - 1) * LDX] = xlast;
    }
}

template <int MI, int NI>
__global__ void __launch_bounds__(kMaxThreads, 1)
    time_fused_kernel(KArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ Jt,
                      const double* __restrict__ J, ArrowParams ap) {
    const Smem sm = carve(a);
    const long long c0 = static_cast<long long>(blockIdx.x) * a.BN;
    compute_colbase(a, c0, sm.colbase, sm.obase);
    __syncthreads();
    load_tile(a, sm, c0, X);
    cp_commit();
    gemm_prologue(a, sm, Jt);
    double acc[MI][NI][2];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    gemm_main<MI, NI>(a, sm, Jt, acc);  // Z = U_t^T x
    gemm_prologue(a, sm, J);            // prefetch U_t while the arrowhead runs
    acc_to_smem<MI, NI>(a, sm, acc, a.Kp);
    __syncthreads();
    arrowhead_tile(a, sm, c0, ap);
    __syncthreads();
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    gemm_main<MI, NI>(a, sm, J, acc);  // y = U_t z
    acc_to_smem<MI, NI>(a, sm, acc, a.geo.m);
    __syncthreads();
    store_tile(a, sm, c0, Y, nullptr);
}

__global__ void scale_kernel(const double* __restrict__ a, const double* __restrict__ x, double* __restrict__ y,
                             long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        y[i] = a[i] * x[i];
}

KArgs make_args(const Tiling& t, const ModeGeom& g) {
    KArgs a;
    a.geo = g;
    a.S = t.S;
    a.Mp = t.Mp;
    a.Kp = t.Kp;
    a.Xrows = t.Xrows;
    a.BN = t.BN;
    a.LDX = t.LDX;
    a.WM = t.WM;
    a.WN = t.WN;
    return a;
}

template <typename K>
cudaError_t prepare(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}

template <int MI>
cudaError_t launch_mode_mi(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                           const double* pre, const double* post, cudaStream_t st) {
    auto k = mode_product_kernel<MI, 2>;
    cudaError_t e = prepare(k, t.smem);
    if (e != cudaSuccess) return e;
    const long long blocks = (g.ncols + t.BN - 1) / t.BN;
    k<<<static_cast<unsigned>(blocks), t.threads(), t.smem, st>>>(make_args(t, g), X, Y, J, pre, post);
    return cudaGetLastError();
}

template <int MI>
cudaError_t launch_time_mi(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt,
                           const double* J, const ArrowParams& ap, cudaStream_t st) {
    auto k = time_fused_kernel<MI, 2>;
    cudaError_t e = prepare(k, t.smem);
    if (e != cudaSuccess) return e;
    const long long blocks = (g.ncols + t.BN - 1) / t.BN;
    k<<<static_cast<unsigned>(blocks), t.threads(), t.smem, st>>>(make_args(t, g), X, Y, Jt, J, ap);
    return cudaGetLastError();
}

}  // namespace

Tiling choose_tiling(int m, int n) {
    Tiling t;
    t.S = (m + 7) / 8;
    t.WM = (t.S + 12) / 13;
    t.MI = (t.S + t.WM - 1) / t.WM;
    t.NI = 2;
    t.Mp = 8 * t.MI * t.WM;
    t.Kp = (n + 3) / 4 * 4;
    t.Xrows = std::max(t.Kp, (m + 3) / 4 * 4);
    const size_t max_smem = 227 * 1024;
    for (int wn : {4, 2, 1}) {
        if (t.WM * wn * 32 > kMaxThreads) continue;
        t.WN = wn;
        t.BN = 8 * t.NI * t.WN;
        t.LDX = t.BN + ((4 - t.BN % 16) + 16) % 16;
        t.smem = sizeof(double) * (static_cast<size_t>(t.Xrows) * t.LDX + static_cast<size_t>(kStages) * t.Mp * kLDJ) +
                 2 * sizeof(long long) * t.BN;
        if (t.smem <= max_smem) break;
    }
    return t;
}

#define STIGA_MI_SWITCH(MI_, CALL)                                                                   \
    switch (MI_) {                                                                                   \
        case 1: return CALL(1); case 2: return CALL(2); case 3: return CALL(3); case 4: return CALL(4); \
        case 5: return CALL(5); case 6: return CALL(6); case 7: return CALL(7); case 8: return CALL(8); \
        case 9: return CALL(9); case 10: return CALL(10); case 11: return CALL(11);                  \
        case 12: return CALL(12); case 13: return CALL(13);                                          \
        default: return cudaErrorInvalidValue;                                                       \
    }

cudaError_t launch_mode_product(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jpad,
                                const double* pre, const double* post, cudaStream_t st) {
    if (g.ncols <= 0) return cudaSuccess;
#define STIGA_CALL_MODE(M) launch_mode_mi<M>(t, g, X, Y, Jpad, pre, post, st)
    STIGA_MI_SWITCH(t.MI, STIGA_CALL_MODE)
#undef STIGA_CALL_MODE
}

cudaError_t launch_time_fused(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt_pad,
                              const double* J_pad, const ArrowParams& ap, cudaStream_t st) {
    if (g.ncols <= 0) return cudaSuccess;
#define STIGA_CALL_TIME(M) launch_time_mi<M>(t, g, X, Y, Jt_pad, J_pad, ap, st)
    STIGA_MI_SWITCH(t.MI, STIGA_CALL_TIME)
#undef STIGA_CALL_TIME
}

cudaError_t launch_scale(const double* a, const double* x, double* y, long long n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int threads = 256;
    const long long blocks = std::min<long long>((n + threads - 1) / threads, 148LL * 16);
    scale_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(a, x, y, n);
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace stiga
