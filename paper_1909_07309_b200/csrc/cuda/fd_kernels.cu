// FP64 tensor-core kernels of the extended-FD apply (sm_100a).
//
// Every mode product is a batch of small GEMMs  Y_fiber = J * X_fiber  with J the n x n
// eigenvector factor (n = 16..260).  A CTA owns a row block of J (MI*WM 8-row strips) and
// BN = 16*WN fibers.  Both operands stream through a 2-3 stage cp.async pipeline in 16-wide
// contraction chunks (J chunk: rows x 16 from L2, fiber chunk: 16 x BN from HBM), the products
// run on the FP64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4; 36.9 TF/s measured on
// B200 vs 34.0 TF/s for DFMA, profiles/r01_fp64_peak.txt) with fragments double-buffered in
// registers, and the accumulators are stored straight from registers (no smem epilogue), so
// several CTAs per SM overlap one tile's epilogue with another's main loop.  All per-chunk
// producer work is compile-time unrolled (element counts follow from MI/WM/WN) so the issue
// slots go to LDS + DMMA.
//
// The time-fused kernel keeps the whole n_t x BN tile of one CTA: Z = U_t^T X lands in shared
// memory, the block-arrowhead solve of fdsolve.cpp:24-65 (forward pair eliminations, diagonal
// Schur, back substitution) runs in place, and Z is the resident B operand of y = U_t Z; the
// time direction costs one HBM round trip instead of three.
#include "fd_kernels.cuh"

#include <algorithm>
#include <cmath>
#include <utility>
#include <vector>
#include <cstdio>
#include <cstdlib>

namespace stiga {
namespace gpu {

namespace {

constexpr int kBK = 16;        // contraction chunk per pipeline stage
constexpr int kLDJ = kBK + 4;  // smem row stride of a J chunk (20 == 4 mod 16: conflict-free A fragments)
constexpr size_t kSmemPerSM = 228 * 1024;
constexpr size_t kSmemPerCTA = 227 * 1024;

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async8(unsigned s, const double* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void cp_async8_zfill(unsigned s, const double* gmem, bool valid) {
    const int sz = valid ? 8 : 0;  // src-size 0 -> zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async16(unsigned s, const double* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_wait_n() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct KArgs {
    ModeGeom geo;
    int Kp, RB, Zrows, nstage;
    int S;  // 8-row strips holding output rows (ceil(rows/8)); strips past S are skipped
};

// Compile-time shape of a CTA.
template <int MI_, int WM_, int WN_, bool PS_ = false>
struct Shape {
    static constexpr int MI = MI_, WM = WM_, WN = WN_, NI = 2;
    static constexpr bool PS = PS_;  // fused D^-1/2 pre-scale: a D chunk is staged beside each fiber chunk
    static constexpr int NTHR = 32 * WM * WN;
    static constexpr int BN = 16 * WN;
    static constexpr int LDX = BN + 4;  // == 4 mod 16
    static constexpr int MPB = 8 * MI * WM;
    static constexpr int XCNT = kBK * BN / NTHR;       // fiber-chunk elements per thread (8/WM)
    static constexpr int JPIECES = MPB * (kBK / 2);    // 16-byte J pieces per chunk
    static constexpr int JROWSTEP = NTHR / 8;          // J rows between a thread's pieces
    static constexpr int JCNT = (JPIECES + NTHR - 1) / NTHR;
    static constexpr int XROWSTEP = NTHR / BN;         // fiber-chunk rows between elements (L > 1)
    static constexpr int XCOLSTEP = NTHR / 16;         // fibers between elements (L == 1)
    static constexpr int DOFF = kBK * LDX + MPB * kLDJ;  // D chunk offset within a stage (PS)
    static constexpr int STAGE = DOFF + (PS ? kBK * LDX : 0);  // doubles per pipeline stage
    static_assert(kBK * BN % NTHR == 0, "fiber chunk must split evenly over the CTA");
};

// Global offset of element 0 of fiber cc (colex: l + L*n*r).
__device__ __forceinline__ long long fiber_base(long long cc, long long L, int n) {
    if (L == 1) return cc * n;
    const long long r = cc / L;
    return (cc - r * L) + L * static_cast<long long>(n) * r;
}

// Per-thread producer state, computed once per tile.
//  fiber chunk, L == 1 (fibers contiguous): row j = tid % 16, fiber c = tid/16 + u*NTHR/16;
//  fiber chunk, L  > 1 (fibers strided):    fiber c = tid % BN, row j = tid/BN + u*NTHR/BN;
//  J chunk: piece tid % 8 of rows tid/8 + u*NTHR/8.
struct Prod {
    const double* xg;    // global address of element u = 0 for chunk 0
    long long xstep;     // global stride between elements u (elements)
    long long xkstep;    // global stride between chunks (elements)
    unsigned xs;         // smem byte offset (within a stage) of element u = 0
    int xrow0;           // chunk row of element u = 0 (row check for the tail chunk)
    unsigned colmask;    // element u belongs to a fiber inside the tensor
    bool full_tile;
    bool contiguous;     // L == 1
    const double* dg;    // PS: D^-1/2 address of element u = 0 for chunk 0 (same offsets as xg)
    const double* jg;    // J global address of this thread's piece u = 0 for chunk 0
    unsigned js;         // smem byte offset (within a stage) of piece u = 0
    int jp2;             // 2 * piece index (column offset within the chunk)
};

template <class SH>
__device__ __forceinline__ Prod make_prod(const KArgs& a, long long c0, const double* X, const double* Jg) {
    Prod p;
    const int tid = threadIdx.x;
    p.colmask = 0;
    p.full_tile = c0 + SH::BN <= a.geo.ncols;
    p.contiguous = a.geo.L == 1;
    if (p.contiguous) {
        const int j = tid & (kBK - 1), cf = tid >> 4;
        p.xrow0 = j;
        p.xs = 8u * (j * SH::LDX + cf);
        p.xg = X + (c0 + cf) * a.geo.n + j;
        p.xstep = static_cast<long long>(SH::XCOLSTEP) * a.geo.n;
        p.xkstep = kBK;
#pragma unroll
        for (int u = 0; u < SH::XCNT; ++u)
            if (c0 + cf + u * SH::XCOLSTEP < a.geo.ncols) p.colmask |= 1u << u;
    } else {
        const int c = tid & (SH::BN - 1), j0 = tid / SH::BN;
        const long long cc = c0 + c;
        const bool cv = cc < a.geo.ncols;
        p.xrow0 = j0;
        p.xs = 8u * (j0 * SH::LDX + c);
        p.xg = X + fiber_base(cv ? cc : 0, a.geo.L, a.geo.n) + a.geo.L * j0;
        p.xstep = a.geo.L * SH::XROWSTEP;
        p.xkstep = a.geo.L * kBK;
        p.colmask = cv ? 0xffffffffu : 0u;
    }
    p.jp2 = 2 * (tid & 7);
    p.js = 8u * ((tid >> 3) * kLDJ + p.jp2);
    p.jg = Jg + static_cast<size_t>(tid >> 3) * a.Kp + p.jp2;
    return p;
}

// Issues the J (and optionally fiber) copies of chunk q into the stage at smem byte address st.
template <class SH>
__device__ __forceinline__ void issue_chunk(const KArgs& a, const Prod& p, unsigned st, int q, bool load_x,
                                            const double* X) {
    const int k0 = q * kBK;
    const int kw = min(kBK, a.Kp - k0);
    if (p.jp2 < kw) {
        const double* jg = p.jg + k0;
        const unsigned js = st + 8u * kBK * SH::LDX + p.js;
#pragma unroll
        for (int u = 0; u < SH::JCNT; ++u) {
            if ((u + 1) * SH::NTHR <= SH::JPIECES || (threadIdx.x >> 3) + u * SH::JROWSTEP < SH::MPB)
                cp_async16(js + 8u * u * SH::JROWSTEP * kLDJ, jg + static_cast<size_t>(u) * SH::JROWSTEP * a.Kp);
        }
    }
    if (!load_x) return;
    auto copy_chunk = [&](const double* xg, unsigned xs) {
        if (p.contiguous) {
            if (p.full_tile && k0 + kBK <= a.geo.n) {
#pragma unroll
                for (int u = 0; u < SH::XCNT; ++u) cp_async8(xs + 8u * u * SH::XCOLSTEP, xg + u * p.xstep);
            } else {
                const bool rowv = k0 + p.xrow0 < a.geo.n;
#pragma unroll
                for (int u = 0; u < SH::XCNT; ++u) {
                    const bool v = rowv && ((p.colmask >> u) & 1u);
                    cp_async8_zfill(xs + 8u * u * SH::XCOLSTEP, v ? xg + u * p.xstep : X, v);
                }
            }
        } else {
            if (p.full_tile && k0 + kBK <= a.geo.n) {
#pragma unroll
                for (int u = 0; u < SH::XCNT; ++u) cp_async8(xs + 8u * u * SH::XROWSTEP * SH::LDX, xg + u * p.xstep);
            } else {
                const bool colv = p.colmask != 0u;
#pragma unroll
                for (int u = 0; u < SH::XCNT; ++u) {
                    const bool v = colv && (k0 + p.xrow0 + u * SH::XROWSTEP < a.geo.n);
                    cp_async8_zfill(xs + 8u * u * SH::XROWSTEP * SH::LDX, v ? xg + u * p.xstep : X, v);
                }
            }
        }
    };
    copy_chunk(p.xg + q * p.xkstep, st + p.xs);
    if constexpr (SH::PS) copy_chunk(p.dg + q * p.xkstep, st + 8u * SH::DOFF + p.xs);
}

// acc += J_chunk * B_chunk over KS k-steps of 4.  A fragments from the J stage (ja), B fragments
// from bb (row stride LDX).  Fragments double-buffered in registers.  Only the warp's first mact
// strips are computed (warp-uniform predicate): strips wholly past the output rows are skipped, so
// a row block that overhangs the matrix costs only its live strips; padded rows inside a live
// strip are zero J rows and produce zeros that are never stored.
template <class SH, int KS>
__device__ __forceinline__ void mma_chunk(const double* ja, const double* bb, int mact,
                                          double (&acc)[SH::MI][SH::NI][2]) {
    constexpr int MI = SH::MI, NI = SH::NI;
    double av[2][MI], bv[2][NI];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) av[0][mi] = mi < mact ? ja[mi * 8 * kLDJ] : 0.0;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) bv[0][ni] = SH::PS ? bb[ni * 8] * bb[SH::DOFF + ni * 8] : bb[ni * 8];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int cur = kk & 1, nxt = cur ^ 1;
        if (kk + 1 < KS) {
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) av[nxt][mi] = mi < mact ? ja[mi * 8 * kLDJ + (kk + 1) * 4] : 0.0;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
                bv[nxt][ni] = SH::PS ? bb[(kk + 1) * 4 * SH::LDX + ni * 8] * bb[SH::DOFF + (kk + 1) * 4 * SH::LDX + ni * 8]
                                     : bb[(kk + 1) * 4 * SH::LDX + ni * 8];
        }
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
                if (mi < mact) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], av[cur][mi], bv[cur][ni]);
    }
}

// Register epilogue: acc rows (< m) of the CTA's row block straight to global memory.
template <class SH>
__device__ __forceinline__ void store_acc(const KArgs& a, const double (&acc)[SH::MI][SH::NI][2], long long c0,
                                          int strip0, double* __restrict__ Y, const double* __restrict__ post) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wm = warp % SH::WM, wn = warp / SH::WM;
    const int g = lane >> 2, t = lane & 3;
    const int m = a.geo.m;
    long long ob[SH::NI][2];
    bool cv[SH::NI][2];
#pragma unroll
    for (int ni = 0; ni < SH::NI; ++ni)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const long long cc = c0 + (wn * SH::NI + ni) * 8 + 2 * t + v;
            cv[ni][v] = cc < a.geo.ncols;
            ob[ni][v] = fiber_base(cv[ni][v] ? cc : 0, a.geo.L, m);
        }
    if (post) {  // fused D^-1/2 post-scale: all scale loads issued before the first store
        double sc[SH::MI][SH::NI][2];
#pragma unroll
        for (int mi = 0; mi < SH::MI; ++mi) {
            const int i = (strip0 + wm * SH::MI + mi) * 8 + g;
            const long long off = a.geo.L * i;
#pragma unroll
            for (int ni = 0; ni < SH::NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v) sc[mi][ni][v] = (i < m && cv[ni][v]) ? __ldg(post + ob[ni][v] + off) : 0.0;
        }
#pragma unroll
        for (int mi = 0; mi < SH::MI; ++mi) {
            const int i = (strip0 + wm * SH::MI + mi) * 8 + g;
            if (i < m) {
                const long long off = a.geo.L * i;
#pragma unroll
                for (int ni = 0; ni < SH::NI; ++ni)
#pragma unroll
                    for (int v = 0; v < 2; ++v)
                        if (cv[ni][v]) Y[ob[ni][v] + off] = sc[mi][ni][v] * acc[mi][ni][v];
            }
        }
        return;
    }
#pragma unroll
    for (int mi = 0; mi < SH::MI; ++mi) {
        const int i = (strip0 + wm * SH::MI + mi) * 8 + g;
        if (i < m) {
            const long long off = a.geo.L * i;
#pragma unroll
            for (int ni = 0; ni < SH::NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (cv[ni][v]) Y[ob[ni][v] + off] = acc[mi][ni][v];
        }
    }
}

template <class SH>
__device__ __forceinline__ void zero_acc(double (&acc)[SH::MI][SH::NI][2]) {
#pragma unroll
    for (int mi = 0; mi < SH::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < SH::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
}

__device__ __forceinline__ void cp_wait_stage(int nstage) {
    if (nstage >= 3) cp_wait_n<1>();
    else cp_wait_n<0>();
}

// Multistage GEMM over the full contraction.  X_STREAM: the fiber operand streams through the
// stages with J; otherwise it is resident in smem at Bres (row stride LDX) and only J streams.
template <class SH, bool X_STREAM>
__device__ __forceinline__ void gemm(const KArgs& a, double* stages, const Prod& p, const double* X, const double* Bres,
                                     bool prologue_issued, int strip0, double (&acc)[SH::MI][SH::NI][2]) {
    const int nchunks = (a.Kp + kBK - 1) / kBK;
    const int ns = a.nstage;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp % SH::WM, wn = warp / SH::WM;
    const int g = lane >> 2, t = lane & 3;
    const int ja_off = kBK * SH::LDX + (wm * SH::MI * 8 + g) * kLDJ + t;  // within a stage
    const int bb_off = t * SH::LDX + wn * SH::NI * 8 + g;
    const int mact = min(SH::MI, max(0, a.S - (strip0 + wm * SH::MI)));
    const unsigned st0 = smem_u32(stages);
    if (!prologue_issued) {
        for (int s = 0; s < ns - 1; ++s) {
            if (s < nchunks) issue_chunk<SH>(a, p, st0 + 8u * s * SH::STAGE, s, X_STREAM, X);
            cp_commit();
        }
    }
    int stage = 0;
    for (int q = 0; q < nchunks; ++q) {
        cp_wait_stage(ns);
        __syncthreads();
        const int nq = q + ns - 1;
        if (nq < nchunks) {
            int nst = stage + ns - 1;
            if (nst >= ns) nst -= ns;
            issue_chunk<SH>(a, p, st0 + 8u * nst * SH::STAGE, nq, X_STREAM, X);
        }
        cp_commit();
        const double* st = stages + stage * SH::STAGE;
        const double* ja = st + ja_off;
        const double* bb = X_STREAM ? st + bb_off : Bres + q * kBK * SH::LDX + bb_off;
        const int ksteps = min(kBK, a.Kp - q * kBK) >> 2;
        if (ksteps == 4) {
            mma_chunk<SH, 4>(ja, bb, mact, acc);
        } else if (ksteps == 3) {
            mma_chunk<SH, 3>(ja, bb, mact, acc);
        } else if (ksteps == 2) {
            mma_chunk<SH, 2>(ja, bb, mact, acc);
        } else {
            mma_chunk<SH, 1>(ja, bb, mact, acc);
        }
        if (++stage == ns) stage = 0;
    }
}

// PS: Y = (I (x) J (x) I)(pre .* X) -- the D^-1/2 pre-scale of the apply fused into the first forward
// mode product: each fiber chunk's D^-1/2 chunk is staged beside it by the same cp.async pattern
// and B fragments are scaled as they are read (two DMULs per k-step on the FP64 pipe, against the
// separate 24 B/DoF HBM pass of scale_kernel).
template <int MI, int WN, bool PS>
__global__ void __launch_bounds__(32 * WN)
    mode_product_kernel(KArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ J,
                        const double* __restrict__ post, const double* __restrict__ pre) {
    using SH = Shape<MI, 1, WN, PS>;
    extern __shared__ __align__(16) double smem[];
    const int rb = blockIdx.x % a.RB;  // row blocks of one fiber tile are adjacent -> X tile reused from L2
    const long long c0 = static_cast<long long>(blockIdx.x / a.RB) * SH::BN;
    const double* Jg = J + static_cast<size_t>(rb) * SH::MPB * a.Kp;
    Prod p = make_prod<SH>(a, c0, X, Jg);
    if constexpr (PS) p.dg = pre + (p.xg - X);
    double acc[SH::MI][SH::NI][2];
    zero_acc<SH>(acc);
    gemm<SH, true>(a, smem, p, X, nullptr, false, rb * MI, acc);
    store_acc<SH>(a, acc, c0, rb * MI, Y, post);
}

// 1/x to ~1 ulp: MUFU double-precision reciprocal seed (rcp.approx.ftz.f64, full exponent range,
// no float conversions on the FP64 pipe) + two Newton steps.  The IEEE division subroutine would
// cost ~10x more FP64 issue slots, and in the arrowhead passes those slots are shared with DMMA.
__device__ __forceinline__ double rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// apply_pair_inverse (fdsolve.cpp:11-20) with R_j^-1 = 1/(nu Lambda_s + c_j Lambda_s^-1) recomputed
// from Lambda_s (fdsolve.cpp:114-119).  Same expression tree as the reference, with x/nu evaluated
// as x*(1/nu) (exact at nu = 1, within 1 ulp otherwise) and c1*c1/nu precomputed per pair.
__device__ __forceinline__ double pair_rinv(double nulam, double linv, double cj) {
    return rcp(fma(cj, linv, nulam));  // nulam = nu * Lambda_s, hoisted out of the pair loops
}

__device__ __forceinline__ void pair_apply(double rinv, double linv, double inv_nu, double c1, double c1sq_nu,
                                           double u, double w, double& xa, double& xb) {
    const double luiu = linv * u;
    const double riluiu = rinv * luiu;
    xa = luiu * inv_nu - c1sq_nu * (linv * riluiu) - c1 * (linv * (rinv * w));
    xb = c1 * riluiu + rinv * w;
}

// Block-arrowhead solve (fdsolve.cpp:24-65) on the resident tile: column c = one spatial
// eigen-index, rows = time eigen-coordinates.  P = NTHR/BN = 2*WM threads share a column
// (pairs j = p mod P, Schur right-hand side reduced with shuffles).
// Pair constants staged in smem once per CTA (the 8-byte cp.async fiber copies go through L1 and
// evict them, and the arrowhead is otherwise latency-bound on their reloads):
// cs[k * NP + j], k = 0..6: c_j, c1_j, c1_j^2/nu, g[2j], g[2j+1], gamma g[2j], gamma g[2j+1].
__device__ __forceinline__ int arrow_np(const ArrowParams& ap) { return ap.n_t / 2 + 1; }

// Per-column constants of the tile (staged during the GEMM prologue, so the arrowhead never waits on
// global loads): ccol[c] = Lambda_s, ccol[BN + c] = 1/Lambda_s (one IEEE division per column instead
// of one per thread), ccol[2 BN + c] = S^-1.
__device__ __forceinline__ void stage_column_consts(const ArrowParams& ap, long long c0, long long ncols, int BN,
                                                    double* ccol) {
    for (int c = threadIdx.x; c < BN; c += blockDim.x) {
        long long s = c0 + c;
        if (s >= ncols) s = ncols - 1;
        double lam = 0.0;  // ((0 + lambda_1) + lambda_2) + ... (fdsolve.cpp:91-99)
        long long rem = s + ap.s_off;  // global spatial index (slab offset in the sharded apply)
        for (int l = 0; l < ap.d; ++l) {
            const long long q = rem / ap.n[l];
            lam = lam + __ldg(ap.lam[l] + (rem - q * ap.n[l]));
            rem = q;
        }
        ccol[c] = lam;
        ccol[BN + c] = 1.0 / lam;
        ccol[2 * BN + c] = __ldg(ap.S_inv + ap.s_off + s);
    }
}

__device__ __forceinline__ void stage_arrow_consts(const ArrowParams& ap, double* cs) {
    const int NP = arrow_np(ap);
    for (int j = threadIdx.x; j < ap.npairs; j += blockDim.x) {
        cs[j] = __ldg(ap.pair_c + j);
        cs[NP + j] = __ldg(ap.pair_c1 + j);
        cs[2 * NP + j] = __ldg(ap.pair_c1sq + j);
        cs[3 * NP + j] = __ldg(ap.g + 2 * j);
        cs[4 * NP + j] = __ldg(ap.g + 2 * j + 1);
        cs[5 * NP + j] = __ldg(ap.pair_gg + 2 * j);
        cs[6 * NP + j] = __ldg(ap.pair_gg + 2 * j + 1);
    }
}

template <class SH>
__device__ __forceinline__ void arrowhead_tile(const KArgs& a, double* Zs, long long c0, const ArrowParams& ap,
                                               const double* cs, const double* ccol) {
    const int NP = arrow_np(ap);
    constexpr int P = SH::NTHR / SH::BN;
    static_assert(P >= 1 && P <= 32 && (P & (P - 1)) == 0, "threads per column must be a power of two <= 32");
    const int tid = threadIdx.x;
    const int c = tid / P;
    const int p = tid - c * P;
    const double lam = ccol[c], linv = ccol[SH::BN + c];
    const double nu = ap.nu, inv_nu = ap.inv_nu, gam = ap.gamma;
    const double nulam = nu * lam;
    const int nt = ap.n_t;
    double* col = Zs + c;
    const double slast = col[(nt - 1) * SH::LDX];
    // Forward sweep: Schur right-hand side sum_j gamma g_j . H_j^-1 z_j (fdsolve.cpp:31-47) without
    // storing H_j^-1 z_j; the back sweep then forms x_j = H_j^-1 (z_j - gamma g_j x_last) from the
    // untouched z_j -- equal to the reference's y_j - H_j^-1 (gamma g_j x_last) (fdsolve.cpp:52-63)
    // by linearity, with fewer FP64 instructions (which share the pipe with the DMMAs) and no stores.
    double part = 0.0;
    for (int j = p; j < ap.npairs; j += P) {
        double xa, xb;
        const double rinv = pair_rinv(nulam, linv, cs[j]);
        pair_apply(rinv, linv, inv_nu, cs[NP + j], cs[2 * NP + j], col[(2 * j) * SH::LDX], col[(2 * j + 1) * SH::LDX], xa,
                   xb);
        part = fma(cs[5 * NP + j], xa, fma(cs[6 * NP + j], xb, part));  // gamma g[2j] x_a + gamma g[2j+1] x_b
    }
    double xz = 0.0;
    if (ap.zero_count && p == 0) {
        xz = linv * col[(nt - 2) * SH::LDX] * inv_nu;
        part += gam * __ldg(ap.g + nt - 2) * xz;
    }
#pragma unroll
    for (int off = P >> 1; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    const double xlast = ccol[2 * SH::BN + c] * (slast + part);
    for (int j = p; j < ap.npairs; j += P) {
        double xa, xb;
        const double rinv = pair_rinv(nulam, linv, cs[j]);
        const double u = fma(-cs[5 * NP + j], xlast, col[(2 * j) * SH::LDX]);
        const double w = fma(-cs[6 * NP + j], xlast, col[(2 * j + 1) * SH::LDX]);
        pair_apply(rinv, linv, inv_nu, cs[NP + j], cs[2 * NP + j], u, w, xa, xb);
        col[(2 * j) * SH::LDX] = xa;
        col[(2 * j + 1) * SH::LDX] = xb;
    }
    if (p == 0) {
        if (ap.zero_count) col[(nt - 2) * SH::LDX] = xz - (gam * __ldg(ap.g + nt - 2) * inv_nu) * (linv * xlast);
        col[(nt - 1) * SH::LDX] = xlast;
    }
}

template <int MI, int WM, int WN>
__global__ void __launch_bounds__(32 * WM * WN)
    time_fused_kernel(KArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ Jt,
                      const double* __restrict__ J, ArrowParams ap) {
    using SH = Shape<MI, WM, WN>;
    extern __shared__ __align__(16) double smem[];
    double* Zs = smem;                                               // Zrows x LDX, resident
    double* stages = smem + static_cast<size_t>(a.Zrows) * SH::LDX;  // nstage x stage
    double* cs = stages + static_cast<size_t>(a.nstage) * SH::STAGE;    // 7 x (n_t/2 + 1) pair constants
    double* ccol = cs + 7 * arrow_np(ap);                               // 3 x BN column constants
    const long long c0 = static_cast<long long>(blockIdx.x) * SH::BN;
    stage_arrow_consts(ap, cs);  // visible after the GEMM's first barrier
    stage_column_consts(ap, c0, a.geo.ncols, SH::BN, ccol);
    Prod p = make_prod<SH>(a, c0, X, Jt);
    double acc[SH::MI][SH::NI][2];
    zero_acc<SH>(acc);
    gemm<SH, true>(a, stages, p, X, nullptr, false, 0, acc);  // Z = U_t^T x
    // Z -> smem (rows < Kp; padded rows are exact zeros because the padded J rows are zero)
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int wm = warp % WM, wn = warp / WM;
        const int g = lane >> 2, t = lane & 3;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
            const int row = (wm * MI + mi) * 8 + g;
            if (row < a.Zrows) {
#pragma unroll
                for (int ni = 0; ni < SH::NI; ++ni) {
                    const int col = (wn * SH::NI + ni) * 8 + 2 * t;
                    Zs[row * SH::LDX + col] = acc[mi][ni][0];
                    Zs[row * SH::LDX + col + 1] = acc[mi][ni][1];
                }
            }
        }
    }
    __syncthreads();  // Z visible; every warp is done with the GEMM-1 stages
    // U_t chunks stream in while the arrowhead runs
    p.jg = J + (p.jg - Jt);
    {
        const int nchunks = (a.Kp + kBK - 1) / kBK;
        const unsigned st0 = smem_u32(stages);
        for (int s = 0; s < a.nstage - 1; ++s) {
            if (s < nchunks) issue_chunk<SH>(a, p, st0 + 8u * s * SH::STAGE, s, false, X);
            cp_commit();
        }
    }
    if (!(ap.debug & 1)) arrowhead_tile<SH>(a, Zs, c0, ap, cs, ccol);
    __syncthreads();
    zero_acc<SH>(acc);
    gemm<SH, false>(a, stages, p, X, Zs, true, 0, acc);  // y = U_t z
    store_acc<SH>(a, acc, c0, 0, Y, nullptr);
}

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

KArgs make_args(const Tiling& t, const ModeGeom& g) {
    KArgs a;
    a.geo = g;
    a.Kp = t.Kp;
    a.RB = t.RB;
    a.Zrows = t.Zrows;
    a.nstage = t.nstage;
    a.S = (g.m + 7) / 8;
    return a;
}

// Resident CTAs per SM of an instantiation (exact occupancy query; smem/thread bound when no
// device is current).
template <typename K>
int occupancy(K kernel, int threads, size_t smem) {
    int n = 0;
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) ==
            cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) == cudaSuccess)
        return n;
    cudaGetLastError();
    return std::max(0, std::min(static_cast<int>(kSmemPerSM / (smem + 1024)), 2048 / threads));
}

// ---- instantiation dispatch --------------------------------------------------------------------
template <int MI, int WN>
cudaError_t launch_mode_t(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                          const double* post, const double* pre, cudaStream_t st, int* occ) {
    auto k = pre ? mode_product_kernel<MI, WN, true> : mode_product_kernel<MI, WN, false>;
    const size_t smem = pre ? prescale_smem(t) : t.smem;
    if (occ) {
        *occ = occupancy(k, 32 * WN, smem);
        return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const long long blocks = (g.ncols + t.BN - 1) / t.BN * t.RB;
    k<<<static_cast<unsigned>(blocks), 32 * WN, smem, st>>>(make_args(t, g), X, Y, J, post, pre);
    return cudaGetLastError();
}

template <int MI, int WM, int WN>
cudaError_t launch_time_t(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt,
                          const double* J, const ArrowParams& ap, cudaStream_t st, int* occ) {
    auto k = time_fused_kernel<MI, WM, WN>;
    if (occ) {
        *occ = occupancy(k, 32 * WM * WN, t.smem);
        return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(t.smem));
    if (e != cudaSuccess) return e;
    const long long blocks = (g.ncols + t.BN - 1) / t.BN;
    k<<<static_cast<unsigned>(blocks), 32 * WM * WN, t.smem, st>>>(make_args(t, g), X, Y, Jt, J, ap);
    return cudaGetLastError();
}

#define STIGA_MI_SWITCH(MI_, CALL)                                                                   \
    switch (MI_) {                                                                                   \
        case 1: return CALL(1); case 2: return CALL(2); case 3: return CALL(3); case 4: return CALL(4); \
        case 5: return CALL(5); case 6: return CALL(6); case 7: return CALL(7); case 8: return CALL(8); \
        case 9: return CALL(9); case 10: return CALL(10); case 11: return CALL(11);                  \
        case 12: return CALL(12); case 13: return CALL(13);                                          \
        default: return cudaErrorInvalidValue;                                                       \
    }

template <int WN>
cudaError_t dispatch_mode_wn(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                             const double* post, const double* pre, cudaStream_t st, int* occ) {
#define STIGA_CALL_MODE(M) launch_mode_t<M, WN>(t, g, X, Y, J, post, pre, st, occ)
    STIGA_MI_SWITCH(t.MI, STIGA_CALL_MODE)
#undef STIGA_CALL_MODE
}

cudaError_t dispatch_mode(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                          const double* post, const double* pre, cudaStream_t st, int* occ) {
    if (t.WM != 1) return cudaErrorInvalidValue;
    if (t.WN == 4) return dispatch_mode_wn<4>(t, g, X, Y, J, post, pre, st, occ);
    if (t.WN == 2) return dispatch_mode_wn<2>(t, g, X, Y, J, post, pre, st, occ);
    return cudaErrorInvalidValue;
}

template <int WM, int WN>
cudaError_t dispatch_time_w(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt,
                            const double* J, const ArrowParams& ap, cudaStream_t st, int* occ) {
#define STIGA_CALL_TIME(M) launch_time_t<M, WM, WN>(t, g, X, Y, Jt, J, ap, st, occ)
    STIGA_MI_SWITCH(t.MI, STIGA_CALL_TIME)
#undef STIGA_CALL_TIME
}

cudaError_t dispatch_time(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt,
                          const double* J, const ArrowParams& ap, cudaStream_t st, int* occ) {
    if (t.WN == 2) {
        if (t.WM == 1) return dispatch_time_w<1, 2>(t, g, X, Y, Jt, J, ap, st, occ);
        if (t.WM == 2) return dispatch_time_w<2, 2>(t, g, X, Y, Jt, J, ap, st, occ);
        if (t.WM == 4) return dispatch_time_w<4, 2>(t, g, X, Y, Jt, J, ap, st, occ);
    } else if (t.WN == 4) {
        if (t.WM == 1) return dispatch_time_w<1, 4>(t, g, X, Y, Jt, J, ap, st, occ);
        if (t.WM == 2) return dispatch_time_w<2, 4>(t, g, X, Y, Jt, J, ap, st, occ);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

std::vector<Tiling> mode_tiling_candidates(int m, int n) {
    std::vector<std::pair<double, Tiling>> c;
    const int S = (m + 7) / 8;
    const int Kp = (n + 3) / 4 * 4;
    const int rb0 = (S + 12) / 13;
    for (int RB = rb0; RB <= std::min(S, rb0 + 3); ++RB) {
        const int MI = (S + RB - 1) / RB;
        if (MI > 13 || MI < 1) continue;
        if (RB > rb0 && (S + rb0 - 1) / rb0 == MI) continue;  // same MI as a smaller RB
        for (int WN : {4, 2}) {
            Tiling t;
            t.MI = MI;
            t.WM = 1;
            t.NI = 2;
            t.WN = WN;
            t.S = S;
            t.RB = RB;
            t.MpB = 8 * MI;
            t.Mp = RB * t.MpB;
            t.Kp = Kp;
            t.BN = 16 * WN;
            t.LDX = t.BN + 4;
            t.nstage = 3;
            t.smem = sizeof(double) * static_cast<size_t>(t.nstage) * (kBK * t.LDX + t.MpB * kLDJ);
            if (t.smem > kSmemPerCTA) continue;
            int occ = 0;
            dispatch_mode(t, ModeGeom{}, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &occ);
            t.ctas_per_sm = occ;
            if (occ < 1) continue;
            // strips past S are skipped, so padding costs only imbalance; each extra row block
            // re-stages the fiber tile
            const double eff = 0.85 + 0.15 * static_cast<double>(S) / (RB * MI);
            c.emplace_back(std::min(occ * t.WN, 16) * eff + 0.02 * WN - 0.05 * RB, t);
        }
    }
    std::stable_sort(c.begin(), c.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<Tiling> out;
    for (auto& e : c) out.push_back(e.second);
    return out;
}

Tiling choose_mode_tiling(int m, int n, bool prescale) {
    (void)prescale;  // the D^-1/2 pre-scale is a separate elementwise pass
    const std::vector<Tiling> c = mode_tiling_candidates(m, n);
    if (c.empty()) {
        Tiling t;
        t.MI = 0;
        return t;
    }
    return c.front();
}

std::vector<Tiling> time_tiling_candidates(int nt) {
    std::vector<std::pair<double, Tiling>> c;
    int force_wm = 0, force_wn = 0, force_ns = 0;  // debugging aid: STIGA_FORCE_TIME_TILING="WM,WN,NS"
    if (const char* f = std::getenv("STIGA_FORCE_TIME_TILING"))
        std::sscanf(f, "%d,%d,%d", &force_wm, &force_wn, &force_ns);
    const int S = (nt + 7) / 8;
    const int Kp = (nt + 3) / 4 * 4;
    for (int WM : {1, 2, 4}) {
        const int MI = (S + WM - 1) / WM;
        if (MI > 13 || MI < 1) continue;
        for (int WN : {4, 2}) {
            if (WM == 4 && WN == 4) continue;
            if ((force_wm && WM != force_wm) || (force_wn && WN != force_wn)) continue;
            for (int ns : {3, 2}) {
                if (force_ns && ns != force_ns) continue;
                Tiling t;
                t.MI = MI;
                t.WM = WM;
                t.NI = 2;
                t.WN = WN;
                t.S = S;
                t.RB = 1;
                t.MpB = 8 * MI * WM;
                t.Mp = t.MpB;
                t.Kp = Kp;
                t.BN = 16 * WN;
                t.LDX = t.BN + 4;
                t.Zrows = Kp;
                t.nstage = ns;
                t.smem = sizeof(double) * (static_cast<size_t>(Kp) * t.LDX +
                                           static_cast<size_t>(ns) * (kBK * t.LDX + t.MpB * kLDJ) +
                                           7 * static_cast<size_t>(nt / 2 + 1) + 3 * static_cast<size_t>(t.BN));
                if (t.smem > kSmemPerCTA) continue;
                int occ = 0;
                ArrowParams ap;
                dispatch_time(t, ModeGeom{}, nullptr, nullptr, nullptr, nullptr, ap, nullptr, &occ);
                t.ctas_per_sm = occ;
                if (occ < 1) continue;
                const double eff = 0.85 + 0.15 * static_cast<double>(S) / (WM * MI);
                c.emplace_back(std::min(occ * WM * WN, 16) * eff + 0.01 * ns + 0.02 * WN, t);
            }
        }
    }
    std::stable_sort(c.begin(), c.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<Tiling> out;
    for (auto& e : c) out.push_back(e.second);
    return out;
}

Tiling choose_time_tiling(int nt) {
    const std::vector<Tiling> c = time_tiling_candidates(nt);
    if (c.empty()) {
        Tiling t;
        t.MI = 0;
        return t;
    }
    return c.front();
}

size_t prescale_smem(const Tiling& t) {
    return t.smem + sizeof(double) * static_cast<size_t>(t.nstage) * kBK * t.LDX;
}

bool prescale_fits(const Tiling& t) { return t.WM == 1 && prescale_smem(t) <= kSmemPerCTA; }

cudaError_t launch_mode_product(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jpad,
                                const double* post_scale, cudaStream_t st, const double* pre_scale) {
    if (g.ncols <= 0) return cudaSuccess;
    if (pre_scale && !prescale_fits(t)) return cudaErrorInvalidValue;
    return dispatch_mode(t, g, X, Y, Jpad, post_scale, pre_scale, st, nullptr);
}

cudaError_t launch_time_fused(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt_pad,
                              const double* J_pad, const ArrowParams& ap, cudaStream_t st) {
    if (g.ncols <= 0) return cudaSuccess;
    return dispatch_time(t, g, X, Y, Jt_pad, J_pad, ap, st, nullptr);
}

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
