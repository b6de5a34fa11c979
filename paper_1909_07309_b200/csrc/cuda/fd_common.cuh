// Shared device helpers of the FD-apply kernels (fd_mode.cu, fd_mode_sc.cu, fd_time.cu,
// fd_time_sc.cu, fd_kernels.cu): cp.async staging, the DMMA chunk loop, register epilogues (plain,
// D^-1/2-scaled, peer-memory scatter) and the block-arrowhead helpers.  Split over several
// translation units only so that nvcc compiles the kernel instantiations in parallel.
#pragma once
#include "fd_kernels.cuh"

#include <algorithm>
#include <cmath>
#include <utility>
#include <vector>
#include <cstdio>
#include <cstdlib>


namespace stiga {
namespace gpu {

// Scatter variants live in their own translation units (fd_mode_sc.cu / fd_time_sc.cu).
cudaError_t dispatch_mode_scatter(const Tiling& t, const ModeGeom& g, const double* X, const double* J,
                                  cudaStream_t st, int* occ, const Scatter* sc);
cudaError_t dispatch_time_scatter(const Tiling& t, const ModeGeom& g, const double* X, const double* Jt,
                                  const double* J, const ArrowParams& ap, cudaStream_t st, int* occ,
                                  const Scatter* sc);

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
    static constexpr bool EXACT = (kBK * BN) % NTHR == 0;  // false for WM = 3: the last copy round is guarded
    static constexpr int XCNT = (kBK * BN + NTHR - 1) / NTHR;  // fiber-chunk elements per thread (8/WM)
    static constexpr int JPIECES = MPB * (kBK / 2);    // 16-byte J pieces per chunk
    static constexpr int JROWSTEP = NTHR / 8;          // J rows between a thread's pieces
    static constexpr int JCNT = (JPIECES + NTHR - 1) / NTHR;
    static constexpr int XROWSTEP = NTHR / BN;         // fiber-chunk rows between elements (L > 1)
    static constexpr int XCOLSTEP = NTHR / 16;         // fibers between elements (L == 1)
    static constexpr int DOFF = kBK * LDX + MPB * kLDJ;  // D chunk offset within a stage (PS)
    static constexpr int STAGE = DOFF + (PS ? kBK * LDX : 0);  // doubles per pipeline stage
    static_assert(NTHR % BN == 0 && NTHR % 16 == 0, "fiber-chunk copy rounds must be whole rows / fibers");
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
            if (c0 + cf + u * SH::XCOLSTEP < a.geo.ncols && (SH::EXACT || cf + u * SH::XCOLSTEP < SH::BN))
                p.colmask |= 1u << u;
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
                for (int u = 0; u < SH::XCNT; ++u)
                    if (SH::EXACT || ((p.colmask >> u) & 1u)) cp_async8(xs + 8u * u * SH::XCOLSTEP, xg + u * p.xstep);
            } else {
                const bool rowv = k0 + p.xrow0 < a.geo.n;
#pragma unroll
                for (int u = 0; u < SH::XCNT; ++u) {
                    const bool v = rowv && ((p.colmask >> u) & 1u);
                    if (SH::EXACT || static_cast<int>(threadIdx.x >> 4) + u * SH::XCOLSTEP < SH::BN)
                        cp_async8_zfill(xs + 8u * u * SH::XCOLSTEP, v ? xg + u * p.xstep : X, v);
                }
            }
        } else {
            if (p.full_tile && k0 + kBK <= a.geo.n) {
#pragma unroll
                for (int u = 0; u < SH::XCNT; ++u)
                    if (SH::EXACT || p.xrow0 + u * SH::XROWSTEP < kBK)
                        cp_async8(xs + 8u * u * SH::XROWSTEP * SH::LDX, xg + u * p.xstep);
            } else {
                const bool colv = p.colmask != 0u;
#pragma unroll
                for (int u = 0; u < SH::XCNT; ++u) {
                    const bool v = colv && (k0 + p.xrow0 + u * SH::XROWSTEP < a.geo.n);
                    if (SH::EXACT || p.xrow0 + u * SH::XROWSTEP < kBK)
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
template <class SH, int KS, bool FULL = false>
__device__ __forceinline__ void mma_chunk(const double* ja, const double* bb, int mact,
                                          double (&acc)[SH::MI][SH::NI][2]) {
    constexpr int MI = SH::MI, NI = SH::NI;
    double av[2][MI], bv[2][NI];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) av[0][mi] = (FULL || mi < mact) ? ja[mi * 8 * kLDJ] : 0.0;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) bv[0][ni] = SH::PS ? bb[ni * 8] * bb[SH::DOFF + ni * 8] : bb[ni * 8];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int cur = kk & 1, nxt = cur ^ 1;
        if (kk + 1 < KS) {
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) av[nxt][mi] = (FULL || mi < mact) ? ja[mi * 8 * kLDJ + (kk + 1) * 4] : 0.0;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
                bv[nxt][ni] = SH::PS ? bb[(kk + 1) * 4 * SH::LDX + ni * 8] * bb[SH::DOFF + (kk + 1) * 4 * SH::LDX + ni * 8]
                                     : bb[(kk + 1) * 4 * SH::LDX + ni * 8];
        }
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
                if (FULL || mi < mact) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], av[cur][mi], bv[cur][ni]);
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

// Scatter epilogue (Scatter in fd_kernels.cuh): each output element goes straight to the receive
// buffer of its owner rank (peer memory over NVLink, or a virtual rank's local buffer).  The owner
// search is a warp-divergence-free compare chain over the G partition offsets (integer pipe only).
template <class SH>
__device__ __forceinline__ void store_acc_scatter(const KArgs& a, const double (&acc)[SH::MI][SH::NI][2], long long c0,
                                                  int strip0, const Scatter& sc) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wm = warp % SH::WM, wn = warp / SH::WM;
    const int g = lane >> 2, t = lane & 3;
    const int m = a.geo.m;
    const long long L = a.geo.L;
    long long fl[SH::NI][2], fr[SH::NI][2];
    bool cv[SH::NI][2];
#pragma unroll
    for (int ni = 0; ni < SH::NI; ++ni)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const long long cc = c0 + (wn * SH::NI + ni) * 8 + 2 * t + v;
            cv[ni][v] = cc < a.geo.ncols;
            fr[ni][v] = cc / L;
            fl[ni][v] = cc - fr[ni][v] * L;
        }
#pragma unroll
    for (int mi = 0; mi < SH::MI; ++mi) {
        const int i = (strip0 + wm * SH::MI + mi) * 8 + g;
        if (i >= m) continue;
#pragma unroll
        for (int ni = 0; ni < SH::NI; ++ni)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                if (!cv[ni][v]) continue;
                long long ca, cb;
                if (sc.by_time) {
                    ca = fl[ni][v];
                    cb = i;
                } else {
                    ca = fl[ni][v] + L * i;
                    cb = fr[ni][v];
                }
                const long long key = sc.by_time ? cb : ca;
                // owner = last rank whose offset <= key; static indices only (parameters stay in the
                // constant bank, no local-memory copy of the descriptor)
                double* base = sc.ptr[0];
                long long o = 0, ld = sc.ld[0];
#pragma unroll
                for (int k = 1; k < kMaxRanks; ++k)
                    if (k < sc.G && key >= sc.off[k]) {
                        base = sc.ptr[k];
                        o = sc.off[k];
                        ld = sc.ld[k];
                    }
                const long long da = ca - (sc.by_time ? 0 : o) + sc.a_shift;
                const long long db = cb - (sc.by_time ? o : 0) + sc.b_shift;
                base[da + ld * db] = acc[mi][ni][v];
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
        // all strips live (the usual case): the unpredicated chunk -- a runtime-predicated mma.sync
        // costs a WARPSYNC + NOP per DMMA (folded-kernel analysis)
        if (mact == SH::MI) {
            if (ksteps == 4) mma_chunk<SH, 4, true>(ja, bb, mact, acc);
            else if (ksteps == 3) mma_chunk<SH, 3, true>(ja, bb, mact, acc);
            else if (ksteps == 2) mma_chunk<SH, 2, true>(ja, bb, mact, acc);
            else mma_chunk<SH, 1, true>(ja, bb, mact, acc);
        } else if (ksteps == 4) {
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


// 1/x to ~1 ulp: MUFU double-precision reciprocal seed (rcp.approx.ftz.f64, full exponent range,
// no float conversions on the FP64 pipe) + two Newton steps.  The IEEE division subroutine would
// cost ~10x more FP64 issue slots, and in the arrowhead passes those slots are shared with DMMA.
__device__ __forceinline__ double rcp(double x) {
#ifdef STIGA_RCP_IEEE
    return 1.0 / x;
#endif
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
#ifdef STIGA_ARROW_NOFMA
    const double luiu = __dmul_rn(linv, u);
    const double riluiu = __dmul_rn(rinv, luiu);
    xa = __dsub_rn(__dsub_rn(__dmul_rn(luiu, inv_nu), __dmul_rn(c1sq_nu, __dmul_rn(linv, riluiu))),
                   __dmul_rn(c1, __dmul_rn(linv, __dmul_rn(rinv, w))));
    xb = __dadd_rn(__dmul_rn(c1, riluiu), __dmul_rn(rinv, w));
#else
    const double luiu = linv * u;
    const double riluiu = rinv * luiu;
    xa = luiu * inv_nu - c1sq_nu * (linv * riluiu) - c1 * (linv * (rinv * w));
    xb = c1 * riluiu + rinv * w;
#endif
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
                                               const double* cs, const double* ccol, double* red = nullptr) {
    const int NP = arrow_np(ap);
    constexpr int P = SH::NTHR / SH::BN;
    constexpr bool POW2 = (P & (P - 1)) == 0;  // WM = 3: P = 6, the Schur sum is reduced through smem (red)
    static_assert(P >= 1 && P <= 32, "threads per column");
    const int tid = threadIdx.x;
    const int c = POW2 ? tid / P : tid % SH::BN;
    const int p = POW2 ? tid - c * P : tid / SH::BN;
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
    if constexpr (POW2) {
#pragma unroll
        for (int off = P >> 1; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    } else {  // the P partial sums of a column live in different warps: fixed-order sum through smem
        red[p * SH::BN + c] = part;
        __syncthreads();
        part = 0.0;
#pragma unroll
        for (int q = 0; q < P; ++q) part += red[q * SH::BN + c];
    }
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


#define STIGA_MI_SWITCH(MI_, CALL)                                                                   \
    switch (MI_) {                                                                                   \
        case 1: return CALL(1); case 2: return CALL(2); case 3: return CALL(3); case 4: return CALL(4); \
        case 5: return CALL(5); case 6: return CALL(6); case 7: return CALL(7); case 8: return CALL(8); \
        case 9: return CALL(9); case 10: return CALL(10); case 11: return CALL(11);                  \
        case 12: return CALL(12); case 13: return CALL(13);                                          \
        default: return cudaErrorInvalidValue;                                                       \
    }

}  // namespace
}  // namespace gpu
}  // namespace stiga
