// Fused sum-factorized space-time system mat-vec (KronSumOperator::apply, kronop.cpp:108-115, over the
// kron_sum_terms structure of solver.cpp:10-30):
//
//   y = gamma (W_t (x) M_d .. M_1) x + nu (M_t (x) sum_l M_d .. K_l .. M_1) x
//
// evaluated as spatial halves a = (M_d..M_1) x, b = sum_l (M_d..K_l..M_1) x and one banded time pass
// y = gamma W_t a + nu M_t b.  Two kernels instead of d+1 banded passes (48 instead of 16 d + 48 B/DoF
// of HBM traffic):
//
//  plane2_kernel   modes 0 and 1 of a tile of TR consecutive mode-1 rows (a contiguous chunk of the
//                  colex vector): x rows -> smem, mode 0 on every row (a = M_1 x, b = K_1 x, kept in
//                  smem), mode 1 on the TR - 2P interior rows (a2 = M_2 a, b2 = K_2 a + M_2 b) -> HBM.
//                  The P-row halos of neighbouring tiles are re-read (from L2) and mode 0 recomputed.
//  stream_kernel   [mode 2 (a3 = M_3 a2, b3 = K_3 a2 + M_3 b2) on a 32-column x 32-row tile, d = 3]
//                  then the time pass, streaming over the input time slices t' with a ring of 2P+1
//                  output accumulators per point in registers (every input slice is read once; y(t)
//                  is written when t' = t + P).
//
// Banded factors are in row band storage widened to 2P+1 taps (zeros outside each factor's band and
// outside the matrix), so tap loops are fully unrolled and branch free.  The tap coefficients are
// uniform across a warp (every lane of a warp works on the same row of the factor) and are read as
// broadcasts; the register windows along the contracted direction load every smem value once per
// R outputs.  Arithmetic is FP64 FMA in the reference's summation order per output (taps ascending).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "matvec_fused.cuh"

namespace stiga {
namespace gpu {

namespace {

__device__ __forceinline__ void cpa8(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int kTR = 32;  // tile rows of plane2_kernel (interior rows = kTR - 2P)
constexpr int kR0 = 4;   // mode-0 outputs per thread (register window along i0)

// smem pitch (in doubles) >= w, odd: 8-byte accesses of lanes at consecutive rows are conflict free
__host__ __device__ inline int odd_pitch(int w) { return w | 1; }

template <int P>
struct Plane2Smem {
    int xp, ap;  // pitches of the x tile (n0 + 2P zero-padded columns) and of the a, b tiles
    int nbuf;    // x buffers (2 = next tile prefetched with cp.async)
    __host__ __device__ size_t x_elems() const { return static_cast<size_t>(kTR) * xp; }
    __host__ __device__ size_t a_elems() const { return static_cast<size_t>(kTR) * ap; }
    __host__ __device__ size_t bytes() const { return sizeof(double) * (nbuf * x_elems() + 2 * a_elems()); }
};

template <int P>
__host__ __device__ inline Plane2Smem<P> plane2_smem(int n0, int nbuf) {
    Plane2Smem<P> s;
    s.xp = odd_pitch(n0 + 2 * P);
    s.ap = odd_pitch(n0);
    s.nbuf = nbuf;
    return s;
}

// Modes 0 and 1 of the colex tensor (n0, n1, R): x -> a2 = (M1 (x) M0) x, b2 = (K1 (x) M0 + M1 (x) K0) x.
// Bands (widened to 2P+1): m0/k0 rows of mode 0 (n0 rows), m1/k1 rows of mode 1 (n1 rows).
template <int P>
__global__ void __launch_bounds__(256) plane2_kernel(int n0, int n1, long long R, const double* __restrict__ x,
                                                     double* __restrict__ a2, double* __restrict__ b2,
                                                     const double* __restrict__ m0, const double* __restrict__ k0,
                                                     const double* __restrict__ m1, const double* __restrict__ k1,
                                                     int nbuf) {
    constexpr int W = 2 * P + 1;
    constexpr int B = kTR - 2 * P;      // interior (output) rows per tile
    constexpr int R1 = (B + 1) / 2;     // mode-1 output rows per warp task
    extern __shared__ double sm[];
    const Plane2Smem<P> L = plane2_smem<P>(n0, nbuf);
    double* xs[2] = {sm, sm + (nbuf > 1 ? L.x_elems() : 0)};
    double* as = sm + nbuf * L.x_elems();
    double* bs = as + L.a_elems();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const long long tiles_j = (n1 + B - 1) / B;
    const long long ntiles = tiles_j * R;

    // zero the P pad columns of the x buffers once (the copies never touch them)
    for (int e = threadIdx.x; e < nbuf * kTR * 2 * P; e += blockDim.x) {
        const int bb = e / (kTR * 2 * P), rem = e - bb * kTR * 2 * P;
        const int row = rem / (2 * P), c = rem - row * 2 * P;
        xs[bb][row * L.xp + (c < P ? c : n0 + c)] = 0.0;
    }
    // stage the x rows j0 - P .. j0 + B + P - 1 of tile `t` (zero rows outside [0, n1)) into buffer dst
    auto issue = [&](long long t, double* dst) {
        const long long r = t / tiles_j;
        const int j0 = static_cast<int>(t - r * tiles_j) * B;
        const double* src = x + static_cast<long long>(n0) * n1 * r;
        for (int e = threadIdx.x; e < kTR * n0; e += blockDim.x) {
            const int row = e / n0, i0 = e - row * n0;
            const int j = j0 - P + row;
            double* d = dst + row * L.xp + P + i0;
            if (j >= 0 && j < n1) cpa8(d, src + static_cast<long long>(n0) * j + i0);
            else *d = 0.0;
        }
        cpa_commit();
    };
    long long t = blockIdx.x;
    int cur = 0;
    if (t < ntiles) issue(t, xs[0]);
    for (; t < ntiles; t += gridDim.x) {
        const long long tn = t + gridDim.x;
        if (nbuf > 1 && tn < ntiles) {
            issue(tn, xs[cur ^ 1]);
            cpa_wait<1>();
        } else {
            cpa_wait<0>();
        }
        __syncthreads();
        const double* X = xs[cur];
        // ---- stage 1: mode 0 on all kTR rows; lane = row, warp = segments of kR0 consecutive i0 ----
        {
            const int row = lane;
            const int nseg = (n0 + kR0 - 1) / kR0;
            for (int sg = warp; sg < nseg; sg += nwarp) {
                const int i0s = sg * kR0;
                double xw[kR0 + 2 * P];
#pragma unroll
                for (int k = 0; k < kR0 + 2 * P; ++k) {
                    const int c = i0s + k;  // padded column (P pad on the left)
                    xw[k] = c < n0 + 2 * P ? X[row * L.xp + c] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < kR0; ++q) {
                    const int i0 = i0s + q;
                    if (i0 >= n0) break;
                    const double* mr = m0 + static_cast<long long>(i0) * W;
                    const double* kr = k0 + static_cast<long long>(i0) * W;
                    double sa = 0.0, sb = 0.0;
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        sa = fma(__ldg(mr + k), xw[q + k], sa);
                        sb = fma(__ldg(kr + k), xw[q + k], sb);
                    }
                    as[row * L.ap + i0] = sa;
                    bs[row * L.ap + i0] = sb;
                }
            }
        }
        __syncthreads();
        // ---- stage 2: mode 1 on the B interior rows; lane = column, task = (32-column block, row group) --
        {
            const long long r = t / tiles_j;
            const int j0 = static_cast<int>(t - r * tiles_j) * B;
            const int ncb = (n0 + 31) / 32;
            const int ngroups = (B + R1 - 1) / R1;
            for (int task = warp; task < ncb * ngroups; task += nwarp) {
                const int cb = task / ngroups, g = task - cb * ngroups;
                const int col = cb * 32 + lane;
                const int rs = g * R1;  // first interior row of the group (tile row P + rs)
                if (col < n0) {
                    double aw[R1 + 2 * P], bw[R1 + 2 * P];
#pragma unroll
                    for (int k = 0; k < R1 + 2 * P; ++k) {
                        const int row = rs + k;  // tile row of output rs - P + k ... (halo included)
                        aw[k] = row < kTR ? as[row * L.ap + col] : 0.0;
                        bw[k] = row < kTR ? bs[row * L.ap + col] : 0.0;
                    }
                    double* ya = a2 + static_cast<long long>(n0) * n1 * r;
                    double* yb = b2 + static_cast<long long>(n0) * n1 * r;
#pragma unroll
                    for (int q = 0; q < R1; ++q) {
                        const int j = j0 + rs + q;
                        if (rs + q >= B || j >= n1) break;
                        const double* mr = m1 + static_cast<long long>(j) * W;
                        const double* kr = k1 + static_cast<long long>(j) * W;
                        double sa = 0.0, sb = 0.0;
#pragma unroll
                        for (int k = 0; k < W; ++k) {
                            const double mk = __ldg(mr + k), kk = __ldg(kr + k);
                            sa = fma(mk, aw[q + k], sa);
                            sb = fma(kk, aw[q + k], sb);
                            sb = fma(mk, bw[q + k], sb);
                        }
                        ya[static_cast<long long>(n0) * j + col] = sa;
                        yb[static_cast<long long>(n0) * j + col] = sb;
                    }
                }
            }
        }
        __syncthreads();  // a/b tiles and x buffer `cur` are rewritten by the next tile
        if (nbuf == 1 && tn < ntiles) issue(tn, xs[0]);
        cur ^= (nbuf > 1 ? 1 : 0);
    }
}

// ---- stream kernel ----------------------------------------------------------------------------
constexpr int kSQ = 4;    // output rows (mode 2) or columns (time only) per thread
constexpr int kNS = 3;    // cp.async ring depth over time slices

// MODE2 = true: fields (L, n2, T) colex, tile = 32 consecutive l x 32 rows i2 (8 warps x kSQ rows).
// MODE2 = false: fields (L, T) (n2 = 1), tile = 256 * kSQ consecutive l (thread = kSQ columns, stride 256).
// Inputs a, b hold the time slices [ti0, ti0 + nti) (global indices), outputs y the slices
// [to0, to0 + nto) ⊂ [ti0, ti0 + nti) ... (the caller passes base pointers of those slices).
// cw / cm: band COLUMNS of gamma W_t and nu M_t: cw[t' * W + (d + P)] = gamma W_t(t' + d, t') (0 outside).
template <int P, bool MODE2>
__global__ void __launch_bounds__(256) stream_kernel(long long Lc, int n2, int ti0, int nti, int to0, int nto,
                                                     const double* __restrict__ a, const double* __restrict__ b,
                                                     double* __restrict__ y, const double* __restrict__ m2,
                                                     const double* __restrict__ k2, const double* __restrict__ cw,
                                                     const double* __restrict__ cm) {
    constexpr int W = 2 * P + 1;
    constexpr int ROWS_IN = MODE2 ? (8 * kSQ + 2 * P) : 1;   // staged rows per slice
    constexpr int COLS = MODE2 ? 32 : 256 * kSQ;             // staged columns per row
    constexpr int CP = MODE2 ? 33 : COLS;                    // column pitch
    constexpr int STAGE = 2 * ROWS_IN * CP;                  // a then b
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long slice = Lc * n2;  // entries per time slice
    const long long ncolb = (Lc + COLS - 1) / COLS;
    const int nrowb = MODE2 ? (n2 + 8 * kSQ - 1) / (8 * kSQ) : 1;
    const long long ntiles = ncolb * nrowb;
    const int te = ti0 + nti + P;  // streaming end (virtual zero slices finalize the last outputs)

    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long cb = tile % ncolb;
        const int rb = static_cast<int>(tile / ncolb);
        const long long l0 = cb * COLS;
        const int r0 = rb * 8 * kSQ;  // first output row (MODE2)
        auto issue = [&](int tp) {   // stage slice tp (global index) of a and b
            if (tp < ti0 + nti) {
                double* st = sm + (tp - ti0) % kNS * STAGE;
                const long long sbase = static_cast<long long>(tp - ti0) * slice;
                for (int e = threadIdx.x; e < ROWS_IN * COLS; e += blockDim.x) {
                    const int row = e / COLS, c = e - row * COLS;
                    const long long l = l0 + c;
                    const int i2 = MODE2 ? r0 - P + row : 0;
                    double* da = st + row * CP + c;
                    double* db = da + ROWS_IN * CP;
                    if (l < Lc && i2 >= 0 && i2 < n2) {
                        const long long off = sbase + l + Lc * i2;
                        cpa8(da, a + off);
                        cpa8(db, b + off);
                    } else {
                        *da = 0.0;
                        *db = 0.0;
                    }
                }
            }
            cpa_commit();
        };
        double acc[kSQ][W];
#pragma unroll
        for (int q = 0; q < kSQ; ++q)
#pragma unroll
            for (int s = 0; s < W; ++s) acc[q][s] = 0.0;
        __syncthreads();  // previous tile done with the ring
        for (int k = 0; k < kNS - 1; ++k) issue(ti0 + k);
        for (int base = ti0; base < te; base += W) {
#pragma unroll
            for (int u = 0; u < W; ++u) {
                const int tp = base + u;
                if (tp >= te) break;
                issue(tp + kNS - 1);
                cpa_wait<kNS - 1>();
                __syncthreads();
                double v3a[kSQ], v3b[kSQ];
                if (tp < ti0 + nti) {
                    const double* st = sm + (tp - ti0) % kNS * STAGE;
                    if (MODE2) {  // mode 2 on rows r0 + warp*kSQ + q, column lane
                        const int rw = warp * kSQ;
                        double aw[kSQ + 2 * P], bw[kSQ + 2 * P];
#pragma unroll
                        for (int k = 0; k < kSQ + 2 * P; ++k) {
                            aw[k] = st[(rw + k) * CP + lane];
                            bw[k] = st[ROWS_IN * CP + (rw + k) * CP + lane];
                        }
#pragma unroll
                        for (int q = 0; q < kSQ; ++q) {
                            const int i2 = min(r0 + rw + q, n2 - 1);  // rows past n2 are computed, not stored
                            const double* mr = m2 + static_cast<long long>(i2) * W;
                            const double* kr = k2 + static_cast<long long>(i2) * W;
                            double sa = 0.0, sb = 0.0;
#pragma unroll
                            for (int k = 0; k < W; ++k) {
                                const double mk = __ldg(mr + k), kk = __ldg(kr + k);
                                sa = fma(mk, aw[q + k], sa);
                                sb = fma(kk, aw[q + k], sb);
                                sb = fma(mk, bw[q + k], sb);
                            }
                            v3a[q] = sa;
                            v3b[q] = sb;
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < kSQ; ++q) {
                            v3a[q] = st[threadIdx.x + 256 * q];
                            v3b[q] = st[CP + threadIdx.x + 256 * q];
                        }
                    }
                    // time: output t = tp + dd receives cw(tp)[dd + P] a3 + cm(tp)[dd + P] b3
                    const double* cwr = cw + static_cast<long long>(tp) * W;
                    const double* cmr = cm + static_cast<long long>(tp) * W;
#pragma unroll
                    for (int dd = -P; dd <= P; ++dd) {
                        const double w = __ldg(cwr + dd + P), m = __ldg(cmr + dd + P);
                        constexpr int dummy = 0;
                        (void)dummy;
                        const int s = ((u + dd) % W + W) % W;
#pragma unroll
                        for (int q = 0; q < kSQ; ++q) acc[q][s] = fma(m, v3b[q], fma(w, v3a[q], acc[q][s]));
                    }
                }
                // output t = tp - P is complete
                {
                    const int tdone = tp - P;
                    const int s = ((u - P) % W + W) % W;
                    if (tdone >= to0 && tdone < to0 + nto) {
                        double* yt = y + static_cast<long long>(tdone - to0) * slice;
#pragma unroll
                        for (int q = 0; q < kSQ; ++q) {
                            if (MODE2) {
                                const int i2 = r0 + warp * kSQ + q;
                                const long long l = l0 + lane;
                                if (i2 < n2 && l < Lc) yt[l + Lc * i2] = acc[q][s];
                            } else {
                                const long long l = l0 + threadIdx.x + 256 * q;
                                if (l < Lc) yt[l] = acc[q][s];
                            }
                        }
                    }
#pragma unroll
                    for (int q = 0; q < kSQ; ++q) acc[q][s] = 0.0;
                }
                __syncthreads();  // stage (tp - ti0) % kNS is refilled by the next iteration's issue
            }
        }
        cpa_wait<0>();
    }
}

}  // namespace

// ---- host launchers ---------------------------------------------------------------------------

size_t plane2_smem_bytes(int n0, int P, int nbuf) {
    const size_t xp = odd_pitch(n0 + 2 * P), ap = odd_pitch(n0);
    return sizeof(double) * (nbuf * kTR * xp + 2 * kTR * ap);
}

cudaError_t launch_plane2(int n0, int n1, long long R, int P, const double* x, double* a2, double* b2,
                          const double* m0, const double* k0, const double* m1, const double* k1, cudaStream_t st) {
    if (R <= 0 || n0 <= 0 || n1 <= 0) return cudaSuccess;
    if (P < 1 || P > kMaxFusedP || kTR - 2 * P < 2) return cudaErrorInvalidValue;
    int nbuf = 2;
    size_t sm = plane2_smem_bytes(n0, P, nbuf);
    if (sm > 227 * 1024) {
        nbuf = 1;
        sm = plane2_smem_bytes(n0, P, nbuf);
    }
    if (sm > 227 * 1024) return cudaErrorInvalidValue;
    const int B = kTR - 2 * P;
    const long long ntiles = (n1 + B - 1) / B * R;
    const int per_sm = std::max(1, static_cast<int>((227 * 1024) / (sm + 1024)));
    const unsigned grid = static_cast<unsigned>(std::min<long long>(ntiles, 148LL * std::min(per_sm, 4)));
#define STIGA_P2(PP)                                                                                                 \
    case PP:                                                                                                         \
        cudaFuncSetAttribute(plane2_kernel<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)); \
        plane2_kernel<PP><<<grid, 256, sm, st>>>(n0, n1, R, x, a2, b2, m0, k0, m1, k1, nbuf);                        \
        break;
    switch (P) {
        STIGA_P2(1)
        STIGA_P2(2)
        STIGA_P2(3)
        STIGA_P2(4)
        STIGA_P2(5)
        STIGA_P2(6)
        default: return cudaErrorInvalidValue;
    }
#undef STIGA_P2
    return cudaGetLastError();
}

cudaError_t launch_stream(bool mode2, long long Lc, int n2, int ti0, int nti, int to0, int nto, int P, const double* a,
                          const double* b, double* y, const double* m2, const double* k2, const double* cw,
                          const double* cm, cudaStream_t st) {
    if (Lc <= 0 || nti <= 0 || nto <= 0) return cudaSuccess;
    if (P < 1 || P > kMaxFusedP || to0 < ti0 || to0 + nto > ti0 + nti) return cudaErrorInvalidValue;
    const int rows_in = mode2 ? 8 * kSQ + 2 * P : 1;
    const int cp = mode2 ? 33 : 256 * kSQ;
    const size_t sm = sizeof(double) * kNS * 2 * static_cast<size_t>(rows_in) * cp;
    const long long cols = mode2 ? 32 : 256 * kSQ;
    const long long ntiles = (Lc + cols - 1) / cols * (mode2 ? (n2 + 8 * kSQ - 1) / (8 * kSQ) : 1);
    const unsigned grid = static_cast<unsigned>(std::min<long long>(ntiles, 148LL * 4));
#define STIGA_ST(PP)                                                                                                  \
    case PP:                                                                                                          \
        if (mode2) {                                                                                                  \
            cudaFuncSetAttribute(stream_kernel<PP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                                 static_cast<int>(sm));                                                              \
            stream_kernel<PP, true><<<grid, 256, sm, st>>>(Lc, n2, ti0, nti, to0, nto, a, b, y, m2, k2, cw, cm);     \
        } else {                                                                                                      \
            cudaFuncSetAttribute(stream_kernel<PP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,             \
                                 static_cast<int>(sm));                                                              \
            stream_kernel<PP, false><<<grid, 256, sm, st>>>(Lc, 1, ti0, nti, to0, nto, a, b, y, m2, k2, cw, cm);     \
        }                                                                                                             \
        break;
    switch (P) {
        STIGA_ST(1)
        STIGA_ST(2)
        STIGA_ST(3)
        STIGA_ST(4)
        STIGA_ST(5)
        STIGA_ST(6)
        default: return cudaErrorInvalidValue;
    }
#undef STIGA_ST
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace stiga
