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
#include <cstdlib>

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

constexpr int kTR = 32;             // x rows per plane2 tile (outputs: the kTR - 2P interior rows)
constexpr int kPlaneThreads = 256;  // 8 warps, two CTAs per SM where the tiles fit (n0 <= ~170)
constexpr int kR1 = 6;              // mode-1 output rows per warp task (register window of kR1 + 2P rows)

__host__ __device__ inline int even_up(int w) { return (w + 1) & ~1; }

// smem layout of plane2_kernel (doubles): x tile [kTR][xp], the mode-1 results a1 = M1 x, b1 = K1 x of the
// B interior rows [B][ap] each (P zero columns on the left, >= P + 1 on the right, so mode 0 reads
// padded windows), the tile's mode-1 coefficient rows [B][wp] for M1 and K1.
struct Plane2Smem {
    int B, xp, ap, wp;
    __host__ __device__ Plane2Smem(int n0, int P)
        : B(kTR - 2 * P), xp(n0), ap(even_up(n0 + 2 * P + 1)), wp(even_up(2 * P + 1)) {}
    __host__ __device__ size_t x_elems() const { return static_cast<size_t>(kTR) * xp; }
    __host__ __device__ size_t a_elems() const { return static_cast<size_t>(B) * ap; }
    __host__ __device__ size_t c_elems() const { return static_cast<size_t>(B) * wp; }
    __host__ __device__ size_t bytes() const { return sizeof(double) * (x_elems() + 2 * a_elems() + 2 * c_elems()); }
};

// Modes 0 and 1 of the colex tensor (n0, n1, R): x -> a2 = (M1 (x) M0) x, b2 = (K1 (x) M0 + M1 (x) K0) x,
// evaluated as mode 1 first (a1 = M1 x, b1 = K1 x on the interior rows: no halo recomputation), then
// mode 0 (a2 = M0 a1, b2 = K0 a1 + M0 b1); Kronecker factors on distinct modes commute.
//  stage 1 (mode 1): lane = column, warp task = kR1 consecutive output rows of a 32-column block with a
//    register window of kR1 + 2P x rows; the coefficient rows (uniform per warp) are staged in smem.
//  stage 2 (mode 0): thread = a fixed pair of columns i0 = 2 pi, 2 pi + 1 (their four coefficient rows stay
//    in registers for the whole kernel) and rows g, g + G, ...; 16-byte window loads.
// dbuf: a second x-tile buffer (after the coefficient rows) receives the NEXT tile's rows while the
// current one is computed (cp.async groups: the wait before stage 1 leaves the prefetch in flight).
template <int P>
__global__ void __launch_bounds__(kPlaneThreads, 2) plane2_kernel(int n0, int n1, long long R,
                                                                  const double* __restrict__ x, double* __restrict__ a2,
                                                                  double* __restrict__ b2,
                                                                  const double* __restrict__ m0,
                                                                  const double* __restrict__ k0,
                                                                  const double* __restrict__ m1,
                                                                  const double* __restrict__ k1, int dbuf) {
    constexpr int W = 2 * P + 1;
    constexpr int B = kTR - 2 * P;
    constexpr int WP = (W + 1) & ~1;
    extern __shared__ __align__(16) double sm[];
    const Plane2Smem L(n0, P);
    double* xs = sm;
    double* as = xs + L.x_elems();
    double* bs = as + L.a_elems();
    double* cm = bs + L.a_elems();
    double* ck = cm + L.c_elems();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const long long tiles_j = (n1 + B - 1) / B;
    const long long ntiles = tiles_j * R;
    // stage-2 role and its coefficient rows (constant for the whole kernel)
    const int NP = (n0 + 1) / 2, G = max(1, static_cast<int>(blockDim.x) / NP);
    const int pi = threadIdx.x % NP, grp = threadIdx.x / NP;
    const bool s2 = grp < G;
    double cma[W], cmb[W], cka[W], ckb[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const int i0 = 2 * pi, i1 = 2 * pi + 1;
        cma[k] = s2 ? __ldg(m0 + static_cast<long long>(i0) * W + k) : 0.0;
        cka[k] = s2 ? __ldg(k0 + static_cast<long long>(i0) * W + k) : 0.0;
        cmb[k] = (s2 && i1 < n0) ? __ldg(m0 + static_cast<long long>(i1) * W + k) : 0.0;
        ckb[k] = (s2 && i1 < n0) ? __ldg(k0 + static_cast<long long>(i1) * W + k) : 0.0;
    }
    // zero the pad columns of the a1 / b1 tiles once (stage 1 writes only columns P .. P + n0 - 1)
    const int padw = L.ap - n0;
    for (int e = threadIdx.x; e < 2 * B * padw; e += blockDim.x) {
        const int f = e / (B * padw), rem = e - f * B * padw;
        const int row = rem / padw, c = rem - row * padw;
        (f ? bs : as)[row * L.ap + (c < P ? c : n0 + c)] = 0.0;
    }
    // x rows j0 - P .. j0 + B + P - 1 of tile tt (zero rows outside [0, n1)) into buffer dst (the tile's x
    // rows are one contiguous chunk of the colex vector; smem pitch = n0)
    auto issue_x = [&](long long tt, double* dst) {
        const long long rr = tt / tiles_j;
        const int jj = static_cast<int>(tt - rr * tiles_j) * B;
        const int jlo = max(jj - P, 0), jhi = min(jj + B + P, n1);  // rows that exist
        const int e0 = (jlo - (jj - P)) * n0, e1 = (jhi - (jj - P)) * n0;
        const double* src = x + static_cast<long long>(n0) * (n1 * rr + jlo) - e0;
        for (int e = threadIdx.x; e < kTR * n0; e += blockDim.x) {
            if (e >= e0 && e < e1) cpa8(dst + e, src + e);
            else dst[e] = 0.0;
        }
    };
    double* xbuf[2] = {xs, ck + L.c_elems()};
    int cur = 0;
    if (dbuf && blockIdx.x < ntiles) issue_x(blockIdx.x, xbuf[0]);
    cpa_commit();
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const long long r = t / tiles_j;
        const int j0 = static_cast<int>(t - r * tiles_j) * B;
        xs = dbuf ? xbuf[cur] : xbuf[0];
        if (dbuf) {
            if (t + gridDim.x < ntiles) issue_x(t + gridDim.x, xbuf[cur ^ 1]);
        } else {
            issue_x(t, xs);
        }
        cpa_commit();
        for (int e = threadIdx.x; e < B * WP; e += blockDim.x) {
            const int q = e / WP, k = e - q * WP;
            const int j = j0 + q;
            const bool ok = k < W && j < n1;
            cm[q * WP + k] = ok ? __ldg(m1 + static_cast<long long>(j) * W + k) : 0.0;
            ck[q * WP + k] = ok ? __ldg(k1 + static_cast<long long>(j) * W + k) : 0.0;
        }
        if (dbuf) cpa_wait<1>();  // this tile's rows landed; the next tile's stay in flight
        else cpa_wait<0>();
        __syncthreads();
        // ---- stage 1: mode 1 on the B interior rows ----
        {
            const int ncb = (n0 + 31) / 32;
            constexpr int ngroups = (B + kR1 - 1) / kR1;
            for (int task = warp; task < ncb * ngroups; task += nwarp) {
                const int cb = task / ngroups, g = task - cb * ngroups;
                const int col = min(cb * 32 + lane, n0 - 1);  // lanes past n0 recompute the last column
                const int rs = g * kR1;                       // first output row of the group (tile row P + rs)
                double xw[kR1 + 2 * P];
#pragma unroll
                for (int k = 0; k < kR1 + 2 * P; ++k) xw[k] = xs[min(rs + k, kTR - 1) * L.xp + col];
#pragma unroll
                for (int q = 0; q < kR1; ++q) {
                    if (rs + q >= B) break;
                    const double2* mr = reinterpret_cast<const double2*>(cm + (rs + q) * WP);
                    const double2* kr = reinterpret_cast<const double2*>(ck + (rs + q) * WP);
                    double sa = 0.0, sb = 0.0;
#pragma unroll
                    for (int k2 = 0; k2 < WP / 2; ++k2) {
                        const double2 mk = mr[k2], kk = kr[k2];
                        sa = fma(mk.x, xw[q + 2 * k2], sa);
                        sb = fma(kk.x, xw[q + 2 * k2], sb);
                        if (2 * k2 + 1 < W) {
                            sa = fma(mk.y, xw[q + 2 * k2 + 1], sa);
                            sb = fma(kk.y, xw[q + 2 * k2 + 1], sb);
                        }
                    }
                    as[(rs + q) * L.ap + P + col] = sa;
                    bs[(rs + q) * L.ap + P + col] = sb;
                }
            }
        }
        __syncthreads();
        // ---- stage 2: mode 0 on the B interior rows -> HBM ----
        if (s2) {
            double* ya = a2 + static_cast<long long>(n0) * n1 * r;
            double* yb = b2 + static_cast<long long>(n0) * n1 * r;
            for (int row = grp; row < B; row += G) {
                const int j = j0 + row;
                if (j >= n1) break;
                const double2* ar = reinterpret_cast<const double2*>(as + row * L.ap + 2 * pi);
                const double2* br = reinterpret_cast<const double2*>(bs + row * L.ap + 2 * pi);
                double aw[W + 1], bw[W + 1];
#pragma unroll
                for (int k = 0; k < (W + 1) / 2; ++k) {
                    const double2 va = ar[k], vb = br[k];
                    aw[2 * k] = va.x;
                    aw[2 * k + 1] = va.y;
                    bw[2 * k] = vb.x;
                    bw[2 * k + 1] = vb.y;
                }
                double sa0 = 0.0, sb0 = 0.0, sa1 = 0.0, sb1 = 0.0;
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    sa0 = fma(cma[k], aw[k], sa0);
                    sb0 = fma(cka[k], aw[k], sb0);
                    sb0 = fma(cma[k], bw[k], sb0);
                    sa1 = fma(cmb[k], aw[k + 1], sa1);
                    sb1 = fma(ckb[k], aw[k + 1], sb1);
                    sb1 = fma(cmb[k], bw[k + 1], sb1);
                }
                const long long o = static_cast<long long>(n0) * j + 2 * pi;
                ya[o] = sa0;
                yb[o] = sb0;
                if (2 * pi + 1 < n0) {
                    ya[o + 1] = sa1;
                    yb[o + 1] = sb1;
                }
            }
        }
        __syncthreads();  // x, a1/b1 tiles and coefficient rows are rewritten by the next tile
        cur ^= 1;
    }
    cpa_wait<0>();
}

// ---- stream kernel ----------------------------------------------------------------------------
// Threads and outputs per thread: mode 2 + time: 8 warps x 2 rows (a 16-row tile; the 2 P + 1 accumulators,
// the mode-2 coefficient rows and the row window live in registers, up to 255 of them); time only: 256
// columns per tile (one per thread), several CTAs per SM.
__host__ __device__ constexpr int st_threads(bool mode2) { return 256; }
__host__ __device__ constexpr int st_sq(bool mode2) { return mode2 ? 2 : 1; }
constexpr int kNS = 4;    // cp.async ring depth over time slices (kNS - 2 ahead of the consumed one)

struct StreamSmem {
    int rows_in, cols, cp, wp, nt;
    __host__ __device__ StreamSmem(bool mode2, int P, int nt_)
        : rows_in(mode2 ? (st_threads(true) / 32) * st_sq(true) + 2 * P : 1),
          cols(mode2 ? 32 : st_threads(false) * st_sq(false)), cp(mode2 ? 33 : st_threads(false) * st_sq(false)),
          wp(even_up(2 * P + 1)), nt(nt_) {}
    __host__ __device__ size_t stage() const { return 2 * static_cast<size_t>(rows_in) * cp; }
    __host__ __device__ size_t ring() const { return kNS * stage(); }
    __host__ __device__ size_t tcoef() const { return 2 * static_cast<size_t>(nt) * wp; }   // time columns
    // mode 2: the tile's coefficient rows (M_3, K_3 for the RPT output rows), read as warp broadcasts
    __host__ __device__ size_t ccoef() const { return rows_in > 1 ? 2 * static_cast<size_t>(rows_in) * wp : 0; }
    __host__ __device__ size_t bytes() const { return sizeof(double) * (ring() + tcoef() + ccoef()); }
};

// MODE2 = true: fields (L, n2, T) colex, tile = 32 consecutive l x 32 rows i2 (8 warps x kSQ rows).
// MODE2 = false: fields (L, T) (n2 = 1), tile = kST * kSQ consecutive l (thread = kSQ columns, stride kST).
// Inputs a, b hold the time slices [ti0, ti0 + nti) (global indices), outputs y the slices
// [to0, to0 + nto) inside them (the caller passes base pointers of those slices).
// cw / cm: band COLUMNS of gamma W_t and nu M_t, cw[t' * W + (d + P)] = gamma W_t(t' + d, t') (0 outside);
// nt = rows of the time factors.
template <int P, bool MODE2>
__global__ void __launch_bounds__(st_threads(MODE2), 2) stream_kernel(long long Lc, int n2, int nt, int ti0, int nti, int to0, int nto,
                                                     const double* __restrict__ a, const double* __restrict__ b,
                                                     double* __restrict__ y, const double* __restrict__ m2,
                                                     const double* __restrict__ k2, const double* __restrict__ cw,
                                                     const double* __restrict__ cm) {
    constexpr int W = 2 * P + 1;
    constexpr int kST = st_threads(MODE2), kSQ = st_sq(MODE2);
    constexpr int RPT = (kST / 32) * kSQ;  // mode-2 output rows per tile
    extern __shared__ __align__(16) double sm[];
    const StreamSmem S(MODE2, P, nt);
    const int ROWS_IN = S.rows_in, COLS = S.cols, CP = S.cp, WP = S.wp;
    const size_t STAGE = S.stage();
    double* tcw = sm + S.ring();
    double* tcm = tcw + static_cast<size_t>(nt) * WP;
    double* c2s = tcm + static_cast<size_t>(nt) * WP;  // MODE2: [RPT][2][WP] coefficient rows of the tile
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long slice = Lc * n2;  // entries per time slice
    const long long ncolb = (Lc + COLS - 1) / COLS;
    const int nrowb = MODE2 ? (n2 + RPT - 1) / RPT : 1;
    const long long ntiles = ncolb * nrowb;
    const int te = ti0 + nti + P;  // streaming end (virtual zero slices finalize the last outputs)
    // time band columns -> smem (padded to WP), once
    for (int e = threadIdx.x; e < nt * WP; e += blockDim.x) {
        const int tp = e / WP, k = e - tp * WP;
        tcw[e] = k < W ? __ldg(cw + static_cast<long long>(tp) * W + k) : 0.0;
        tcm[e] = k < W ? __ldg(cm + static_cast<long long>(tp) * W + k) : 0.0;
    }

    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long cb = tile % ncolb;
        const int rb = static_cast<int>(tile / ncolb);
        const long long l0 = cb * COLS;
        const int r0 = rb * RPT;  // first output row (MODE2)
        // staged elements of this thread: e = tid + kST k (row = e / COLS with COLS a power of two)
        constexpr int kLogCols = MODE2 ? 5 : 8;  // COLS = 32 (mode 2) or kST * kSQ = 256 (time only)
        static_assert((1 << kLogCols) == (MODE2 ? 32 : kST * kSQ), "COLS must be a power of two");
        auto issue = [&](int tp) {  // stage slice tp (global index) of a and b
            if (tp < ti0 + nti) {
                double* st = sm + static_cast<size_t>((tp - ti0) % kNS) * STAGE;
                const double* as_ = a + static_cast<long long>(tp - ti0) * slice + l0;
                const double* bs_ = b + static_cast<long long>(tp - ti0) * slice + l0;
                for (int e = threadIdx.x; e < ROWS_IN * COLS; e += kST) {
                    const int row = e >> kLogCols, c = e & (COLS - 1);
                    const int i2 = MODE2 ? r0 - P + row : 0;
                    double* da = st + row * CP + c;
                    double* db = da + ROWS_IN * CP;
                    if (l0 + c < Lc && i2 >= 0 && i2 < n2) {
                        const long long off = c + Lc * i2;
                        cpa8(da, as_ + off);
                        cpa8(db, bs_ + off);
                    } else {
                        *da = 0.0;
                        *db = 0.0;
                    }
                }
            }
            cpa_commit();
        };
        __syncthreads();  // previous tile done with the ring
        // mode-2 coefficient rows of the tile's output rows -> smem (warp-uniform rows: broadcast reads;
        // in registers they cost 4 P + 2 doubles per thread and halved the occupancy); visible after the
        // first streaming barrier
        if (MODE2) {
            for (int e = threadIdx.x; e < RPT * 2 * WP; e += blockDim.x) {
                const int q = e / (2 * WP), rem = e - q * 2 * WP, f = rem / WP, k = rem - f * WP;
                const int i2 = min(r0 + q, n2 - 1);  // rows past n2 are computed, not stored
                c2s[e] = k < W ? __ldg((f ? k2 : m2) + static_cast<long long>(i2) * W + k) : 0.0;
            }
        }
        double acc[kSQ][W];
#pragma unroll
        for (int q = 0; q < kSQ; ++q)
#pragma unroll
            for (int s = 0; s < W; ++s) acc[q][s] = 0.0;
        for (int k = 0; k < kNS - 1; ++k) issue(ti0 + k);
        // Modular accumulator ring: at stream step tau = tp - ti0, output t = tp + kk - P accumulates into
        // slot (tau + kk) mod W; the loop is unrolled by W so every slot index is a compile-time constant
        // (no register shifting).  One barrier per step: stage (tau - 1) mod kNS is refilled only after it.
        const int tot = te - ti0;
#pragma unroll 1
        for (int base = 0; base < tot; base += W) {
#pragma unroll
            for (int ph = 0; ph < W; ++ph) {
                const int tau = base + ph;
                if (tau >= tot) break;
                const int tp = ti0 + tau;
                cpa_wait<kNS - 2>();
                __syncthreads();  // stage tau landed for all; everyone is done with step tau - 1
                issue(tp + kNS - 1);
                if (tp < ti0 + nti) {
                    double v3a[kSQ], v3b[kSQ];
                    const double* st = sm + static_cast<size_t>(tau % kNS) * STAGE;
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
                            double sa = 0.0, sb = 0.0;
                            const double* cmq = c2s + (rw + q) * 2 * WP;
#pragma unroll
                            for (int k = 0; k < W; ++k) {
                                const double cmk = cmq[k], ckk = cmq[WP + k];
                                sa = fma(cmk, aw[q + k], sa);
                                sb = fma(ckk, aw[q + k], sb);
                                sb = fma(cmk, bw[q + k], sb);
                            }
                            v3a[q] = sa;
                            v3b[q] = sb;
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < kSQ; ++q) {
                            v3a[q] = st[threadIdx.x + kST * q];
                            v3b[q] = st[CP + threadIdx.x + kST * q];
                        }
                    }
                    // time: output t = tp + kk - P receives cw(tp)[kk] a3 + cm(tp)[kk] b3 (slot (ph + kk) mod W)
                    const double2* cwr = reinterpret_cast<const double2*>(tcw + static_cast<size_t>(tp) * WP);
                    const double2* cmr = reinterpret_cast<const double2*>(tcm + static_cast<size_t>(tp) * WP);
#pragma unroll
                    for (int k2 = 0; k2 < (W + 1) / 2; ++k2) {
                        const double2 w2 = cwr[k2], m2v = cmr[k2];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int kk = 2 * k2 + h;
                            if (kk < W) {
                                const double w = h ? w2.y : w2.x, m = h ? m2v.y : m2v.x;
                                const int slot = (ph + kk) % W;
#pragma unroll
                                for (int q = 0; q < kSQ; ++q)
                                    acc[q][slot] = fma(m, v3b[q], fma(w, v3a[q], acc[q][slot]));
                            }
                        }
                    }
                }
                // output t = tp - P is complete in slot ph
                const int tdone = tp - P;
                if (tdone >= to0 && tdone < to0 + nto) {
                    double* yt = y + static_cast<long long>(tdone - to0) * slice;
#pragma unroll
                    for (int q = 0; q < kSQ; ++q) {
                        if (MODE2) {
                            const int i2 = r0 + warp * kSQ + q;
                            const long long l = l0 + lane;
                            if (i2 < n2 && l < Lc) yt[l + Lc * i2] = acc[q][ph];
                        } else {
                            const long long l = l0 + threadIdx.x + kST * q;
                            if (l < Lc) yt[l] = acc[q][ph];
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < kSQ; ++q) acc[q][ph] = 0.0;
            }
        }
        cpa_wait<0>();
    }
}

}  // namespace

// ---- host launchers ---------------------------------------------------------------------------

size_t plane2_smem_bytes(int n0, int P) { return Plane2Smem(n0, P).bytes(); }

cudaError_t launch_plane2(int n0, int n1, long long R, int P, const double* x, double* a2, double* b2,
                          const double* m0, const double* k0, const double* m1, const double* k1, cudaStream_t st) {
    if (R <= 0 || n0 <= 0 || n1 <= 0) return cudaSuccess;
    if (P < 1 || P > kMaxFusedP || kTR - 2 * P < 2 || (n0 + 1) / 2 > kPlaneThreads) return cudaErrorInvalidValue;
    const size_t sm1 = plane2_smem_bytes(n0, P);
    if (sm1 > 227 * 1024) return cudaErrorInvalidValue;
    // STIGA_PLANE2_DBUF=1: double-buffer the x tile when two CTAs per SM still fit (measured no faster:
    // c3 1.95 vs 1.90 ms -- the two co-resident CTAs already overlap one tile's load with the other's work)
    static const bool want_dbuf = std::getenv("STIGA_PLANE2_DBUF") != nullptr;
    const size_t sm2 = sm1 + sizeof(double) * Plane2Smem(n0, P).x_elems();
    const int dbuf = (want_dbuf && 2 * (sm2 + 1024) <= 228 * 1024) ? 1 : 0;
    const size_t sm = dbuf ? sm2 : sm1;
    const int B = kTR - 2 * P;
    const long long ntiles = (n1 + B - 1) / B * R;
    const int per_sm = std::max(1, static_cast<int>((227 * 1024) / (sm + 1024)));
    const unsigned grid = static_cast<unsigned>(std::min<long long>(ntiles, 148LL * std::min(per_sm, 2)));
#define STIGA_P2(PP)                                                                                                 \
    case PP:                                                                                                         \
        cudaFuncSetAttribute(plane2_kernel<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)); \
        plane2_kernel<PP><<<grid, kPlaneThreads, sm, st>>>(n0, n1, R, x, a2, b2, m0, k0, m1, k1, dbuf);              \
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

cudaError_t launch_stream(bool mode2, long long Lc, int n2, int nt, int ti0, int nti, int to0, int nto, int P,
                          const double* a, const double* b, double* y, const double* m2, const double* k2,
                          const double* cw, const double* cm, cudaStream_t st) {
    if (Lc <= 0 || nti <= 0 || nto <= 0) return cudaSuccess;
    if (P < 1 || P > kMaxFusedP || to0 < ti0 || to0 + nto > ti0 + nti || ti0 < 0 || ti0 + nti > nt)
        return cudaErrorInvalidValue;
    const StreamSmem S(mode2, P, nt);
    const size_t sm = S.bytes();
    if (sm > 227 * 1024) return cudaErrorInvalidValue;
    const int rpt = (st_threads(true) / 32) * st_sq(true);
    const long long ntiles = (Lc + S.cols - 1) / S.cols * (mode2 ? (n2 + rpt - 1) / rpt : 1);
    // mode 2: two CTAs per SM (<= 128 registers); time only: up to four
    const int per_sm = std::max(1, std::min(mode2 ? 2 : 4, static_cast<int>((227 * 1024) / (sm + 1024))));
    const unsigned grid = static_cast<unsigned>(std::min<long long>(ntiles, 148LL * per_sm));
#define STIGA_ST(PP)                                                                                                  \
    case PP:                                                                                                          \
        if (mode2) {                                                                                                  \
            cudaFuncSetAttribute(stream_kernel<PP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                                 static_cast<int>(sm));                                                              \
            stream_kernel<PP, true><<<grid, st_threads(true), sm, st>>>(Lc, n2, nt, ti0, nti, to0, nto, a, b, y, m2, k2, cw, cm);  \
        } else {                                                                                                      \
            cudaFuncSetAttribute(stream_kernel<PP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,             \
                                 static_cast<int>(sm));                                                              \
            stream_kernel<PP, false><<<grid, st_threads(false), sm, st>>>(Lc, 1, nt, ti0, nti, to0, nto, a, b, y, m2, k2, cw, cm);  \
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
