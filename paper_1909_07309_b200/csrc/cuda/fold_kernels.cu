// Folded (centrosymmetric) mode products: half the FP64 work of a dense mode product.
//
// On uniform open knots with both spatial end functions dropped and constant coefficients (the
// identity-geometry configs c1, c2, c3, c5) the 1D pencil (K_l, M_l) is centrosymmetric,
// J K_l J = K_l and J M_l J = M_l with J the exchange matrix.  Its eigenvectors then split into
// symmetric and skew ones (host/fdsetup.cpp builds them that way): with n = 2h + o (o = n mod 2) and
// F = h + o,
//   U = Q blockdiag(W_e, W_o),   Q^T x = [ (x_top + J x_bot)/sqrt2 ; x_mid (o = 1) ; (x_top - J x_bot)/sqrt2 ],
// so the forward product y = U^T x of a fiber is
//   y[r]     = sum_k A_e[r][k] (x[k] + x[n-1-k])   r < F    (A_e = W_e^T / sqrt2, middle column / 2)
//   y[F + r] = sum_k A_o[r][k] (x[k] - x[n-1-k])   r < h    (A_o = W_o^T / sqrt2)
// and the backward product x = U y is
//   p[i] = sum_c A_p[i][c] y[c],  q[i] = sum_c A_q[i][c] y[F + c],
//   x[i] = p[i] + q[i],  x[n-1-i] = p[i] - q[i]  (i < h),  x[h] = p[h] (o = 1).
// Two F x F products instead of one n x n product: 2 F^2 ~ n^2 / 2 multiply-adds per fiber.
//
// Kernel structure follows mode_product_kernel (fd_kernels.cu): a CTA owns a row block of both
// folded matrices (MI 8-row strips each) and BN = 16 WN fibers; two 16-row fiber chunks (forward:
// rows k0.. and the mirrored rows n-k0-16..; backward: rows k0.. and F+k0..) and the two matrix
// chunks stream through a cp.async pipeline; the fold (x_k +- x_{n-1-k}) is formed while the
// B fragments are read from shared memory; DMMA.8x8x4 on the FP64 tensor cores; register epilogue.
#include "fd_kernels.cuh"

#include <algorithm>
#include <cstdlib>
#include <utility>
#include <vector>

namespace stiga {
namespace gpu {

namespace {

constexpr int kBK = 16;
constexpr int kLDJ = kBK + 4;  // == 4 mod 16 doubles: conflict-free A fragments
constexpr size_t kSmemPerSM = 228 * 1024;
constexpr size_t kSmemPerCTA = 227 * 1024;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp8z(unsigned s, const double* g, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "r"(valid ? 8 : 0));
}

__device__ __forceinline__ void cp16(unsigned s, const double* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}

__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void wait_n() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

struct FArgs {
    ModeGeom geo;
    int F, h;      // folded length F = h + (n mod 2), h = n / 2
    int Kp;        // round4(F): padded contraction of both folded matrices
    int RB, nstage;
    int S;         // live 8-row strips of the first matrix (ceil(F / 8))
    long long A2;  // offset (doubles) of the second folded matrix after the first (Mp * Kp)
};

template <int MI_, int WN_, int NI_, bool PS_ = false, int WM_ = 1>
struct FShape {
    static constexpr int MI = MI_, WN = WN_, NI = NI_;
    static constexpr bool PS = PS_;  // forward only: D^-1/2 pre-scale chunks staged beside both fiber chunks
    // WM = 1: every warp accumulates both folded products; WM = 2: warp row 0 the first, warp row 1
    // the second (half the accumulators per thread: larger row blocks at the same occupancy)
    static constexpr int WM = WM_;
    static constexpr int NTHR = 32 * WM * WN;
    static constexpr int BN = 8 * NI * WN;
    static constexpr int LDX = BN + 4;            // == 4 mod 16 doubles: conflict-free B fragments
    static constexpr int MPB = 8 * MI;
    static constexpr int XCNT = kBK * BN / NTHR;  // fiber-chunk elements per thread and buffer (4 NI)
    static constexpr int JPIECES = MPB * (kBK / 2);
    static constexpr int JROWSTEP = NTHR / 8;
    static constexpr int JCNT = (JPIECES + NTHR - 1) / NTHR;
    static constexpr int XROWSTEP = NTHR / BN;    // L > 1: chunk rows between a thread's elements
    static constexpr int XCOLSTEP = NTHR / 16;    // L == 1: fibers between a thread's elements
    // stage: Xa (16 x LDX), Xb (16 x LDX), J1 (MPB x LDJ), J2 (MPB x LDJ)
    static constexpr int XB = kBK * LDX;
    static constexpr int J1 = 2 * kBK * LDX;
    static constexpr int J2 = J1 + MPB * kLDJ;
    static constexpr int DA = J2 + MPB * kLDJ;       // PS: D chunk of Xa's rows (then Xb's at DA + XB)
    static constexpr int STAGE = DA + (PS ? 2 * kBK * LDX : 0);
};

__device__ __forceinline__ long long fbase(long long cc, long long L, int n) {
    if (L == 1) return cc * n;
    const long long r = cc / L;
    return (cc - r * L) + L * static_cast<long long>(n) * r;
}

// Per-thread loader state, computed once per tile (mirrors Prod in fd_common.cuh).  Element u of a
// fiber chunk: L == 1: fiber tid/16 + u*XCOLSTEP, chunk row tid%16; L > 1: fiber tid%BN, chunk row
// tid/BN + u*XROWSTEP.  Global address of (element u, fiber row r) = xg + u*xstep + L*r.
struct FProd {
    const double* xg;  // element u = 0, fiber row 0
    long long xstep;   // between elements u
    long long L;       // between fiber rows
    unsigned xs;       // smem byte offset of element u = 0 (Xa; Xb adds XB)
    unsigned xsstep;   // smem bytes between elements u
    int jr0, jrstep;   // chunk row of element u = jr0 + u*jrstep
    unsigned colmask;  // element u's fiber inside the tensor
    bool full_tile;
    const double* jg;  // J1 row piece for chunk 0
    unsigned js;
    int jp2;
};

template <class SH>
__device__ __forceinline__ FProd make_fprod(const FArgs& a, long long c0, const double* X, const double* Jg) {
    FProd p;
    const int tid = threadIdx.x;
    p.L = a.geo.L;
    p.full_tile = c0 + SH::BN <= a.geo.ncols;
    p.colmask = 0;
    if (a.geo.L == 1) {
        const int j = tid & (kBK - 1), cf = tid >> 4;
        p.jr0 = j;
        p.jrstep = 0;
        p.xs = 8u * (j * SH::LDX + cf);
        p.xsstep = 8u * SH::XCOLSTEP;
        p.xg = X + (c0 + cf) * a.geo.n;
        p.xstep = static_cast<long long>(SH::XCOLSTEP) * a.geo.n;
#pragma unroll
        for (int u = 0; u < SH::XCNT; ++u)
            if (c0 + cf + u * SH::XCOLSTEP < a.geo.ncols) p.colmask |= 1u << u;
    } else {
        const int c = tid % SH::BN, j0 = tid / SH::BN;
        const long long cc = c0 + c;
        const bool cv = cc < a.geo.ncols;
        p.jr0 = j0;
        p.jrstep = SH::XROWSTEP;
        p.xs = 8u * (j0 * SH::LDX + c);
        p.xsstep = 8u * SH::XROWSTEP * SH::LDX;
        p.xg = X + fbase(cv ? cc : 0, a.geo.L, a.geo.n);
        p.xstep = 0;  // the element's chunk row carries the stride
        p.colmask = cv ? 0xffffffffu : 0u;
    }
    p.jp2 = 2 * (tid & 7);
    p.js = 8u * ((tid >> 3) * kLDJ + p.jp2);
    p.jg = Jg + static_cast<size_t>(tid >> 3) * a.Kp + p.jp2;
    return p;
}

// Chunk q: matrix columns [16q, 16q+16) of both folded matrices; fiber rows ra0 + r (Xa) and
// rb0 + r (Xb), r = 0..15, zero-filled outside [0, n).  Interior chunks of full tiles take the
// unpredicated path.
template <class SH, bool FWD>
__device__ __forceinline__ void fissue(const FArgs& a, const FProd& p, unsigned st, int q, const double* X,
                                       const double* Dp = nullptr) {
    const int k0 = q * kBK;
    const int kw = min(kBK, a.Kp - k0);
    if (p.jp2 < kw) {
#pragma unroll
        for (int u = 0; u < SH::JCNT; ++u) {
            if ((u + 1) * SH::NTHR <= SH::JPIECES || (threadIdx.x >> 3) + u * SH::JROWSTEP < SH::MPB) {
                const double* g = p.jg + k0 + static_cast<size_t>(u) * SH::JROWSTEP * a.Kp;
                const unsigned s = st + p.js + 8u * u * SH::JROWSTEP * kLDJ;
                cp16(s + 8u * SH::J1, g);
                cp16(s + 8u * SH::J2, g + a.A2);
            }
        }
    }
    const int n = a.geo.n;
    const int ra0 = k0, rb0 = FWD ? n - k0 - kBK : a.F + k0;
    const double* xa = p.xg + p.L * ra0;
    const double* xb = p.xg + p.L * rb0;
    const unsigned sa = st + p.xs, sb = st + 8u * SH::XB + p.xs;
    const long long dofs = SH::PS ? Dp - X : 0;  // D^-1/2 element = X element + dofs
    const unsigned dsa = 8u * (SH::DA - 0), dsb = 8u * SH::DA;  // D chunks: Xa's at DA, Xb's at DA + XB
    if (p.full_tile && ra0 + kBK <= n && rb0 >= 0 && rb0 + kBK <= n) {
#pragma unroll
        for (int u = 0; u < SH::XCNT; ++u) {
            const long long o = u * p.xstep + p.L * (p.jr0 + u * p.jrstep);
            cp8z(sa + u * p.xsstep, xa + o, true);
            cp8z(sb + u * p.xsstep, xb + o, true);
            if constexpr (SH::PS) {
                cp8z(sa + dsa + u * p.xsstep, xa + o + dofs, true);
                cp8z(sb + dsb + u * p.xsstep, xb + o + dofs, true);
            }
        }
    } else {
#pragma unroll
        for (int u = 0; u < SH::XCNT; ++u) {
            const int jr = p.jr0 + u * p.jrstep;
            const bool fv = (p.colmask >> u) & 1u;
            const bool va = fv && ra0 + jr < n, vb = fv && rb0 + jr >= 0 && rb0 + jr < n;
            const long long o = u * p.xstep + p.L * jr;
            cp8z(sa + u * p.xsstep, va ? xa + o : X, va);
            cp8z(sb + u * p.xsstep, vb ? xb + o : X, vb);
            if constexpr (SH::PS) {
                cp8z(sa + dsa + u * p.xsstep, va ? xa + o + dofs : Dp, va);
                cp8z(sb + dsb + u * p.xsstep, vb ? xb + o + dofs : Dp, vb);
            }
        }
    }
}

template <class SH, bool FWD, bool FULL = false>
__device__ __forceinline__ void fload(const double* ja, const double* xa, const double* xb, int kk, int mact,
                                      double (&a1)[SH::MI], double (&a2)[SH::MI], double (&b1)[SH::NI],
                                      double (&b2)[SH::NI]) {
#pragma unroll
    for (int mi = 0; mi < SH::MI; ++mi) {
        a1[mi] = (FULL || mi < mact) ? ja[mi * 8 * kLDJ + kk * 4] : 0.0;
        a2[mi] = (FULL || mi < mact) ? ja[(SH::J2 - SH::J1) + mi * 8 * kLDJ + kk * 4] : 0.0;
    }
#pragma unroll
    for (int ni = 0; ni < SH::NI; ++ni) {
        double u = xa[kk * 4 * SH::LDX + ni * 8];
        if (SH::PS) u *= xa[SH::DA + kk * 4 * SH::LDX + ni * 8];
        if (FWD) {  // xb points at mirrored row 15 - t; rows run backwards
            double w = xb[-kk * 4 * SH::LDX + ni * 8];
            if (SH::PS) w *= xb[SH::DA - kk * 4 * SH::LDX + ni * 8];
            b1[ni] = u + w;
            b2[ni] = u - w;
        } else {
            b1[ni] = u;
            b2[ni] = xb[kk * 4 * SH::LDX + ni * 8];
        }
    }
}

// WM = 2: one folded product per warp (matrix m = warp row): A fragments from J1 or J2, B fragments
// x_k + x_{n-1-k} (m = 0) / x_k - x_{n-1-k} (m = 1) forward, the first / second half backward.
template <class SH, bool FWD, bool FULL = false>
__device__ __forceinline__ void fload1(const double* ja, const double* xa, const double* xb, int kk, int mact,
                                       double sgn, double (&a)[SH::MI], double (&b)[SH::NI]) {
#pragma unroll
    for (int mi = 0; mi < SH::MI; ++mi) a[mi] = (FULL || mi < mact) ? ja[mi * 8 * kLDJ + kk * 4] : 0.0;
#pragma unroll
    for (int ni = 0; ni < SH::NI; ++ni) {
        if (FWD) {
            double u = xa[kk * 4 * SH::LDX + ni * 8];
            double w = xb[-kk * 4 * SH::LDX + ni * 8];
            if (SH::PS) {
                u *= xa[SH::DA + kk * 4 * SH::LDX + ni * 8];
                w *= xb[SH::DA - kk * 4 * SH::LDX + ni * 8];
            }
            b[ni] = fma(sgn, w, u);  // exact: sgn = +-1
        } else {
            b[ni] = xa[kk * 4 * SH::LDX + ni * 8];  // xa already points at this warp's half
        }
    }
}

template <class SH, bool FWD, int KS, bool FULL = false>
__device__ __forceinline__ void fmma1(const double* ja, const double* xa, const double* xb, int mact, double sgn,
                                      double (&c)[SH::MI][SH::NI][2]) {
    constexpr int MI = SH::MI, NI = SH::NI;
    double a[2][MI], b[2][NI];
    fload1<SH, FWD, FULL>(ja, xa, xb, 0, mact, sgn, a[0], b[0]);
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int cur = kk & 1, nxt = cur ^ 1;
        if (kk + 1 < KS) fload1<SH, FWD, FULL>(ja, xa, xb, kk + 1, mact, sgn, a[nxt], b[nxt]);
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
                if (FULL || mi < mact) dmma(c[mi][ni][0], c[mi][ni][1], a[cur][mi], b[cur][ni]);
    }
}

// Both folded products over KS k-steps of 4, fragments double-buffered in registers.
template <class SH, bool FWD, int KS, bool FULL = false>
__device__ __forceinline__ void fmma(const double* ja, const double* xa, const double* xb, int mact,
                                     double (&c1)[SH::MI][SH::NI][2], double (&c2)[SH::MI][SH::NI][2]) {
    constexpr int MI = SH::MI, NI = SH::NI;
    double a1[2][MI], a2[2][MI], b1[2][NI], b2[2][NI];
    fload<SH, FWD, FULL>(ja, xa, xb, 0, mact, a1[0], a2[0], b1[0], b2[0]);
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int cur = kk & 1, nxt = cur ^ 1;
        if (kk + 1 < KS) fload<SH, FWD, FULL>(ja, xa, xb, kk + 1, mact, a1[nxt], a2[nxt], b1[nxt], b2[nxt]);
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
                if (FULL || mi < mact) {
                    dmma(c1[mi][ni][0], c1[mi][ni][1], a1[cur][mi], b1[cur][ni]);
                    dmma(c2[mi][ni][0], c2[mi][ni][1], a2[cur][mi], b2[cur][ni]);
                }
    }
}

template <int MI, int WN, int NI, bool FWD, bool POST, bool PS>
__global__ void __launch_bounds__(32 * WN)
    fold_mode_kernel(FArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ J,
                     const double* __restrict__ post, const double* __restrict__ pre) {
    using SH = FShape<MI, WN, NI, PS>;
    extern __shared__ __align__(16) double smem[];
    const int rb = blockIdx.x % a.RB;
    const long long c0 = static_cast<long long>(blockIdx.x / a.RB) * SH::BN;
    const int strip0 = rb * MI;
    const FProd p = make_fprod<SH>(a, c0, X, J + static_cast<size_t>(rb) * SH::MPB * a.Kp);
    double c1[MI][NI][2], c2[MI][NI][2];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) c1[mi][ni][0] = c1[mi][ni][1] = c2[mi][ni][0] = c2[mi][ni][1] = 0.0;

    const int nchunks = (a.Kp + kBK - 1) / kBK;
    const int ns = a.nstage;
    const int lane = threadIdx.x & 31, wn = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int mact = min(MI, max(0, a.S - strip0));
    const unsigned st0 = smem_u32(smem);
    for (int s = 0; s < ns - 1; ++s) {
        if (s < nchunks) fissue<SH, FWD>(a, p, st0 + 8u * s * SH::STAGE, s, X, pre);
        commit();
    }
    const int ja_off = SH::J1 + g * kLDJ + t;
    const int xa_off = t * SH::LDX + wn * NI * 8 + g;
    const int xb_off = SH::XB + (FWD ? (kBK - 1 - t) : t) * SH::LDX + wn * NI * 8 + g;
    int stage = 0;
    for (int q = 0; q < nchunks; ++q) {
        if (ns >= 3) wait_n<1>();
        else wait_n<0>();
        __syncthreads();
        const int nq = q + ns - 1;
        if (nq < nchunks) {
            int nst = stage + ns - 1;
            if (nst >= ns) nst -= ns;
            fissue<SH, FWD>(a, p, st0 + 8u * nst * SH::STAGE, nq, X, pre);
        }
        commit();
        const double* sb = smem + stage * SH::STAGE;
        const int ks = min(kBK, a.Kp - q * kBK) >> 2;
        if (mact == MI) {  // all strips live: unpredicated MMAs (no WARPSYNC per DMMA)
            if (ks == 4) fmma<SH, FWD, 4, true>(sb + ja_off, sb + xa_off, sb + xb_off, mact, c1, c2);
            else if (ks == 3) fmma<SH, FWD, 3, true>(sb + ja_off, sb + xa_off, sb + xb_off, mact, c1, c2);
            else if (ks == 2) fmma<SH, FWD, 2, true>(sb + ja_off, sb + xa_off, sb + xb_off, mact, c1, c2);
            else fmma<SH, FWD, 1, true>(sb + ja_off, sb + xa_off, sb + xb_off, mact, c1, c2);
        } else if (ks == 4) fmma<SH, FWD, 4>(sb + ja_off, sb + xa_off, sb + xb_off, mact, c1, c2);
        else if (ks == 3) fmma<SH, FWD, 3>(sb + ja_off, sb + xa_off, sb + xb_off, mact, c1, c2);
        else if (ks == 2) fmma<SH, FWD, 2>(sb + ja_off, sb + xa_off, sb + xb_off, mact, c1, c2);
        else fmma<SH, FWD, 1>(sb + ja_off, sb + xa_off, sb + xb_off, mact, c1, c2);
        if (++stage == ns) stage = 0;
    }

    // register epilogue
    const int n = a.geo.n;
    const long long L = a.geo.L;
    long long ob[NI][2];
    bool cv[NI][2];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const long long cc = c0 + (wn * NI + ni) * 8 + 2 * t + v;
            cv[ni][v] = cc < a.geo.ncols;
            ob[ni][v] = fbase(cv[ni][v] ? cc : 0, L, n);
        }
    if constexpr (!FWD && POST) {  // D^-1/2 post-scale: every scale load issued before the first store
        double plo[MI][NI][2], phi[MI][NI][2];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
            const int i = (strip0 + mi) * 8 + g;
            const int ilo = i < a.F ? i : 0, ihi = i < a.h ? n - 1 - i : 0;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    plo[mi][ni][v] = cv[ni][v] ? __ldg(post + ob[ni][v] + L * ilo) : 0.0;
                    phi[mi][ni][v] = cv[ni][v] ? __ldg(post + ob[ni][v] + L * ihi) : 0.0;
                }
        }
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
            const int i = (strip0 + mi) * 8 + g;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    if (!cv[ni][v]) continue;
                    double* y = Y + ob[ni][v];
                    if (i < a.h) {
                        y[L * i] = plo[mi][ni][v] * (c1[mi][ni][v] + c2[mi][ni][v]);
                        y[L * (n - 1 - i)] = phi[mi][ni][v] * (c1[mi][ni][v] - c2[mi][ni][v]);
                    } else if (i < a.F) {  // middle row (odd n)
                        y[L * i] = plo[mi][ni][v] * c1[mi][ni][v];
                    }
                }
        }
        return;
    }
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
        const int i = (strip0 + mi) * 8 + g;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                if (!cv[ni][v]) continue;
                double* y = Y + ob[ni][v];
                if (FWD) {
                    if (i < a.F) y[L * i] = c1[mi][ni][v];
                    if (i < a.h) y[L * (a.F + i)] = c2[mi][ni][v];
                } else if (i < a.h) {
                    y[L * i] = c1[mi][ni][v] + c2[mi][ni][v];
                    y[L * (n - 1 - i)] = c1[mi][ni][v] - c2[mi][ni][v];
                } else if (i < a.F) {  // middle row (odd n)
                    y[L * i] = c1[mi][ni][v];
                }
            }
    }
}


// WM = 2 variant: warp row 0 accumulates the first folded product, warp row 1 the second; each thread
// holds MI x NI accumulator tiles of ONE matrix, so a CTA covers twice the rows per register budget.
// Backward, the q half goes through shared memory to the warp that holds p (x = p +- q).
template <int MI, int WN, int NI, bool FWD, bool POST, bool PS, bool SC = false>
__global__ void __launch_bounds__(64 * WN)
    fold_ms_kernel(FArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ J,
                   const double* __restrict__ post, const double* __restrict__ pre,
                   const __grid_constant__ Scatter sc) {
    using SH = FShape<MI, WN, NI, PS, 2>;
    extern __shared__ __align__(16) double smem[];
    const int rb = blockIdx.x % a.RB;
    const long long c0 = static_cast<long long>(blockIdx.x / a.RB) * SH::BN;
    const int strip0 = rb * MI;
    const FProd p = make_fprod<SH>(a, c0, X, J + static_cast<size_t>(rb) * SH::MPB * a.Kp);
    double c[MI][NI][2];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) c[mi][ni][0] = c[mi][ni][1] = 0.0;

    const int nchunks = (a.Kp + kBK - 1) / kBK;
    const int ns = a.nstage;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wn = warp % WN, wm = warp / WN;
    const int g = lane >> 2, t = lane & 3;
    const int mact = min(MI, max(0, a.S - strip0));
    const unsigned st0 = smem_u32(smem);
    for (int s = 0; s < ns - 1; ++s) {
        if (s < nchunks) fissue<SH, FWD>(a, p, st0 + 8u * s * SH::STAGE, s, X, pre);
        commit();
    }
    const int ja_off = SH::J1 + wm * (SH::J2 - SH::J1) + g * kLDJ + t;
    const int xa_off = (FWD ? 0 : wm * SH::XB) + t * SH::LDX + wn * NI * 8 + g;
    const int xb_off = SH::XB + (kBK - 1 - t) * SH::LDX + wn * NI * 8 + g;
    const double sgn = wm ? -1.0 : 1.0;
    int stage = 0;
    for (int q = 0; q < nchunks; ++q) {
        if (ns >= 3) wait_n<1>();
        else wait_n<0>();
        __syncthreads();
        const int nq = q + ns - 1;
        if (nq < nchunks) {
            int nst = stage + ns - 1;
            if (nst >= ns) nst -= ns;
            fissue<SH, FWD>(a, p, st0 + 8u * nst * SH::STAGE, nq, X, pre);
        }
        commit();
        const double* sb = smem + stage * SH::STAGE;
        const int ks = min(kBK, a.Kp - q * kBK) >> 2;
        if (mact == MI) {  // all strips live: unpredicated MMAs (no WARPSYNC per DMMA)
            if (ks == 4) fmma1<SH, FWD, 4, true>(sb + ja_off, sb + xa_off, sb + xb_off, mact, sgn, c);
            else if (ks == 3) fmma1<SH, FWD, 3, true>(sb + ja_off, sb + xa_off, sb + xb_off, mact, sgn, c);
            else if (ks == 2) fmma1<SH, FWD, 2, true>(sb + ja_off, sb + xa_off, sb + xb_off, mact, sgn, c);
            else fmma1<SH, FWD, 1, true>(sb + ja_off, sb + xa_off, sb + xb_off, mact, sgn, c);
        } else if (ks == 4) fmma1<SH, FWD, 4>(sb + ja_off, sb + xa_off, sb + xb_off, mact, sgn, c);
        else if (ks == 3) fmma1<SH, FWD, 3>(sb + ja_off, sb + xa_off, sb + xb_off, mact, sgn, c);
        else if (ks == 2) fmma1<SH, FWD, 2>(sb + ja_off, sb + xa_off, sb + xb_off, mact, sgn, c);
        else fmma1<SH, FWD, 1>(sb + ja_off, sb + xa_off, sb + xb_off, mact, sgn, c);
        if (++stage == ns) stage = 0;
    }

    const int n = a.geo.n;
    const long long L = a.geo.L;
    long long ob[NI][2];
    bool cv[NI][2];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const long long cc = c0 + (wn * NI + ni) * 8 + 2 * t + v;
            cv[ni][v] = cc < a.geo.ncols;
            ob[ni][v] = fbase(cv[ni][v] ? cc : 0, L, n);
        }
    if constexpr (FWD && SC) {
        // scatter epilogue (fd_kernels.cuh Scatter, forward): output element (fiber l + L r, row) of
        // the time slab is spatial index a = l + L row at local time b = r; it goes to the rank that
        // owns a, at (a - off[q]) + ld[q] (b + b_shift) -- the fused all-to-all of the sharded apply
        const int row0 = wm ? a.F : 0, rows = wm ? a.h : a.F;
        long long fl[NI][2], fr[NI][2];
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const long long cc = c0 + (wn * NI + ni) * 8 + 2 * t + v;
                fr[ni][v] = cc / L;
                fl[ni][v] = cc - fr[ni][v] * L;
            }
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
            const int i = (strip0 + mi) * 8 + g;
            if (i >= rows) continue;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    if (!cv[ni][v]) continue;
                    const long long ca = fl[ni][v] + L * (row0 + i);
                    double* base = sc.ptr[0];
                    long long o = 0, ld = sc.ld[0];
#pragma unroll
                    for (int k = 1; k < kMaxRanks; ++k)
                        if (k < sc.G && ca >= sc.off[k]) {
                            base = sc.ptr[k];
                            o = sc.off[k];
                            ld = sc.ld[k];
                        }
                    base[ca - o + sc.a_shift + ld * (fr[ni][v] + sc.b_shift)] = c[mi][ni][v];
                }
        }
    } else if constexpr (FWD) {
        const int row0 = wm ? a.F : 0, rows = wm ? a.h : a.F;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
            const int i = (strip0 + mi) * 8 + g;
            if (i >= rows) continue;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (cv[ni][v]) Y[ob[ni][v] + L * (row0 + i)] = c[mi][ni][v];
        }
    } else {
        cp_wait_all();
        __syncthreads();  // every warp is done with the pipeline stages: reuse them for q
        double* Qs = smem;  // MPB x LDX
        if (wm == 1) {
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                    for (int v = 0; v < 2; ++v) Qs[(mi * 8 + g) * SH::LDX + (wn * NI + ni) * 8 + 2 * t + v] = c[mi][ni][v];
        }
        __syncthreads();
        if (wm == 1) return;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
            const int i = (strip0 + mi) * 8 + g;
            double plo[NI][2], phi[NI][2];
            if constexpr (POST) {  // this strip's scale loads issued before its stores
                const int ilo = i < a.F ? i : 0, ihi = i < a.h ? n - 1 - i : 0;
#pragma unroll
                for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        plo[ni][v] = cv[ni][v] ? __ldg(post + ob[ni][v] + L * ilo) : 0.0;
                        phi[ni][v] = cv[ni][v] ? __ldg(post + ob[ni][v] + L * ihi) : 0.0;
                    }
            }
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    if (!cv[ni][v]) continue;
                    const double pv = c[mi][ni][v];
                    const double qv = Qs[(mi * 8 + g) * SH::LDX + (wn * NI + ni) * 8 + 2 * t + v];
                    double* y = Y + ob[ni][v];
                    if (i < a.h) {
                        double lo = pv + qv, hi = pv - qv;
                        if constexpr (POST) {
                            lo *= plo[ni][v];
                            hi *= phi[ni][v];
                        }
                        y[L * i] = lo;
                        y[L * (n - 1 - i)] = hi;
                    } else if (i < a.F) {  // middle row (odd n)
                        double m = pv;
                        if constexpr (POST) m *= plo[ni][v];
                        y[L * i] = m;
                    }
                }
        }
    }
}

template <typename K>
int occ_of(K kernel, int threads, size_t smem) {
    int n = 0;
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) ==
            cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) == cudaSuccess)
        return n;
    cudaGetLastError();
    return std::max(0, std::min(static_cast<int>(kSmemPerSM / (smem + 1024)), 2048 / threads));
}

FArgs make_fargs(const Tiling& t, const ModeGeom& g) {
    FArgs a;
    a.geo = g;
    a.h = g.n / 2;
    a.F = g.n - a.h;
    a.Kp = t.Kp;
    a.RB = t.RB;
    a.nstage = t.nstage;
    a.S = (a.F + 7) / 8;
    a.A2 = static_cast<long long>(t.Mp) * t.Kp;
    return a;
}

template <int MI, int WN, int NI>
cudaError_t fold_launch_t(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                          const double* post, const double* pre, bool fwd, cudaStream_t st, int* occ) {
    auto k = fwd ? (pre ? fold_mode_kernel<MI, WN, NI, true, false, true>
                        : fold_mode_kernel<MI, WN, NI, true, false, false>)
                 : (post ? fold_mode_kernel<MI, WN, NI, false, true, false>
                         : fold_mode_kernel<MI, WN, NI, false, false, false>);
    const size_t smem = pre ? fold_prescale_smem(t) : t.smem;
    if (occ) {
        *occ = occ_of(k, 32 * WN, smem);
        return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const long long blocks = (g.ncols + t.BN - 1) / t.BN * t.RB;
    k<<<static_cast<unsigned>(blocks), 32 * WN, smem, st>>>(make_fargs(t, g), X, Y, J, post, pre);
    return cudaGetLastError();
}

template <int MI, int WN>
cudaError_t fold_ms_launch_t(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                             const double* post, const double* pre, bool fwd, cudaStream_t st, int* occ,
                             const Scatter* sc = nullptr) {
    auto k = fwd ? (sc ? fold_ms_kernel<MI, WN, 2, true, false, false, true>
                       : (pre ? fold_ms_kernel<MI, WN, 2, true, false, true>
                              : fold_ms_kernel<MI, WN, 2, true, false, false>))
                 : (post ? fold_ms_kernel<MI, WN, 2, false, true, false>
                         : fold_ms_kernel<MI, WN, 2, false, false, false>);
    const size_t smem = pre ? fold_prescale_smem(t) : t.smem;
    if (occ) {
        *occ = occ_of(k, 64 * WN, smem);
        return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const long long blocks = (g.ncols + t.BN - 1) / t.BN * t.RB;
    k<<<static_cast<unsigned>(blocks), 64 * WN, smem, st>>>(make_fargs(t, g), X, Y, J, post, pre,
                                                              sc ? *sc : Scatter{});
    return cudaGetLastError();
}

template <int WN>
cudaError_t fold_ms_dispatch_wn(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                                const double* post, const double* pre, bool fwd, cudaStream_t st, int* occ,
                                const Scatter* sc = nullptr) {
    switch (t.MI) {
        case 1: return fold_ms_launch_t<1, WN>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        case 2: return fold_ms_launch_t<2, WN>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        case 3: return fold_ms_launch_t<3, WN>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        case 4: return fold_ms_launch_t<4, WN>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        case 5: return fold_ms_launch_t<5, WN>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        case 6: return fold_ms_launch_t<6, WN>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        case 7: return fold_ms_launch_t<7, WN>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        case 8: return fold_ms_launch_t<8, WN>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        case 9: return fold_ms_launch_t<9, WN>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        default: return cudaErrorInvalidValue;
    }
}

template <int WN, int NI>
cudaError_t fold_dispatch_wn(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                             const double* post, const double* pre, bool fwd, cudaStream_t st, int* occ) {
    if constexpr (NI == 4) {  // 16 MI accumulators: spills beyond MI = 3
        switch (t.MI) {
            case 1: return fold_launch_t<1, WN, NI>(t, g, X, Y, J, post, pre, fwd, st, occ);
            case 2: return fold_launch_t<2, WN, NI>(t, g, X, Y, J, post, pre, fwd, st, occ);
            case 3: return fold_launch_t<3, WN, NI>(t, g, X, Y, J, post, pre, fwd, st, occ);
            default: return cudaErrorInvalidValue;
        }
    } else {
        switch (t.MI) {
            case 1: return fold_launch_t<1, WN, NI>(t, g, X, Y, J, post, pre, fwd, st, occ);
            case 2: return fold_launch_t<2, WN, NI>(t, g, X, Y, J, post, pre, fwd, st, occ);
            case 3: return fold_launch_t<3, WN, NI>(t, g, X, Y, J, post, pre, fwd, st, occ);
            case 4: return fold_launch_t<4, WN, NI>(t, g, X, Y, J, post, pre, fwd, st, occ);
            case 5: return fold_launch_t<5, WN, NI>(t, g, X, Y, J, post, pre, fwd, st, occ);
            case 6: return fold_launch_t<6, WN, NI>(t, g, X, Y, J, post, pre, fwd, st, occ);
            case 7: return fold_launch_t<7, WN, NI>(t, g, X, Y, J, post, pre, fwd, st, occ);
            default: return cudaErrorInvalidValue;
        }
    }
}

cudaError_t fold_dispatch(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                          const double* post, const double* pre, bool fwd, cudaStream_t st, int* occ,
                          const Scatter* sc = nullptr) {
    if (t.WM == 2) {
        if (t.NI != 2) return cudaErrorInvalidValue;
        if (t.WN == 4) return fold_ms_dispatch_wn<4>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        if (t.WN == 2) return fold_ms_dispatch_wn<2>(t, g, X, Y, J, post, pre, fwd, st, occ, sc);
        return cudaErrorInvalidValue;
    }
    if (sc) return cudaErrorInvalidValue;  // scatter epilogue: WM = 2 layout only
    if (t.NI == 2 && t.WN == 4) return fold_dispatch_wn<4, 2>(t, g, X, Y, J, post, pre, fwd, st, occ);
    if (t.NI == 2 && t.WN == 2) return fold_dispatch_wn<2, 2>(t, g, X, Y, J, post, pre, fwd, st, occ);
    if (t.NI == 4 && t.WN == 2) return fold_dispatch_wn<2, 4>(t, g, X, Y, J, post, pre, fwd, st, occ);
    if (t.NI == 4 && t.WN == 4) return fold_dispatch_wn<4, 4>(t, g, X, Y, J, post, pre, fwd, st, occ);
    return cudaErrorInvalidValue;
}

}  // namespace

std::vector<Tiling> fold_tiling_candidates(int n) {
    std::vector<std::pair<double, Tiling>> c;
    const int h = n / 2, F = n - h;
    if (h < 1) return {};
    const int S = (F + 7) / 8;
    const int Kp = (F + 3) / 4 * 4;
    for (int WM : {1, 2})
    for (int MI = 1; MI <= (WM == 2 ? 9 : 7); ++MI) {
        const int RB = (S + MI - 1) / MI;
        if ((S + RB - 1) / RB != MI) continue;  // a smaller MI covers the strips with as many row blocks
        for (int WN : {4, 2})
        for (int NI : {2, 4}) {
            if (NI == 4 && (MI > 3 || WM == 2)) continue;  // 16 MI accumulators
            for (int ns : {3, 2}) {
                Tiling t;
                t.fold = 1;
                t.MI = MI;
                t.WM = WM;
                t.NI = NI;
                t.WN = WN;
                t.S = S;
                t.RB = RB;
                t.MpB = 8 * MI;
                t.Mp = RB * t.MpB;
                t.Kp = Kp;
                t.BN = 8 * NI * WN;
                t.LDX = t.BN + 4;
                t.nstage = ns;
                t.smem = sizeof(double) * static_cast<size_t>(ns) * (2 * kBK * t.LDX + 2 * t.MpB * kLDJ);
                if (t.smem > kSmemPerCTA) continue;
                int occ = 0;
                fold_dispatch(t, ModeGeom{}, nullptr, nullptr, nullptr, nullptr, nullptr, true, nullptr, &occ);
                t.ctas_per_sm = occ;
                if (occ < 1) continue;
                const double eff = 0.85 + 0.15 * static_cast<double>(S) / (RB * MI);
                c.emplace_back(std::min(occ * WM * WN, 16) * eff - 0.05 * RB + 0.02 * WN + 0.01 * ns + 0.03 * NI -
                                   0.04 * WM,
                               t);
            }
        }
    }
    std::stable_sort(c.begin(), c.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<Tiling> out;
    if (!std::getenv("STIGA_NO_FOLD_RES")) out = fold_res_candidates(n, 0);  // resident-factor kernels first
    for (auto& e : c) out.push_back(e.second);
    return out;
}

cudaError_t launch_fold_product(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jfold,
                                bool forward, const double* post_scale, cudaStream_t st, const double* pre_scale,
                                const Scatter* sc) {
    if (g.ncols <= 0) return cudaSuccess;
    if (t.fold == 2) {
        if (sc) return cudaErrorInvalidValue;
        return launch_fold_res(t, g, X, Y, Jfold, forward, post_scale, st, pre_scale);
    }
    if (!t.fold || g.m != g.n || g.n < 2 || (forward && post_scale) || (!forward && pre_scale))
        return cudaErrorInvalidValue;
    // the folded epilogue picks the owner from the spatial index: only by_time = 0 descriptors
    if (sc && (!forward || pre_scale || t.WM != 2 || sc->G < 1 || sc->G > kMaxRanks || sc->by_time != 0))
        return cudaErrorInvalidValue;
    if (pre_scale && fold_prescale_smem(t) > kSmemPerCTA) return cudaErrorInvalidValue;
    return fold_dispatch(t, g, X, Y, Jfold, post_scale, pre_scale, forward, st, nullptr, sc);
}

size_t fold_prescale_smem(const Tiling& t) {
    if (t.fold == 2) return fold_res_prescale_smem(t);
    return t.smem + sizeof(double) * static_cast<size_t>(t.nstage) * 2 * kBK * t.LDX;
}

}  // namespace gpu
}  // namespace stiga
