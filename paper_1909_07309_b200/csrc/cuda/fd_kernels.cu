// FP64 tensor-core kernels of the extended-FD apply (sm_100a).
//
// Every mode product is a batch of small GEMMs  Y_fiber = J * X_fiber  with J the n x n
// eigenvector factor (n = 16..260).  A CTA owns a row block of J (MI*WM 8-row strips) and BN
// fibers.  Both operands stream through an `nstage`-deep cp.async pipeline in 16-wide
// contraction chunks (J chunk: rows x 16 from L2, fiber chunk: 16 x BN from HBM), the products
// run on the FP64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4; 36.9 TF/s measured on
// B200 vs 34.0 TF/s for DFMA, profiles/r01_fp64_peak.txt) with fragments double-buffered in
// registers, and the accumulators are stored straight from registers (no smem epilogue), so
// several CTAs per SM overlap one tile's epilogue with another's main loop.
//
// The time-fused kernel keeps the whole n_t x BN tile of one CTA: Z = U_t^T X lands in shared
// memory, the block-arrowhead solve of fdsolve.cpp:24-65 (forward pair eliminations, diagonal
// Schur, back substitution) runs in place, and Z is the resident B operand of y = U_t Z; the
// time direction costs one HBM round trip instead of three.
#include "fd_kernels.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace stiga {
namespace gpu {

namespace {

constexpr int kBK = 16;        // contraction chunk per pipeline stage
constexpr int kLDJ = kBK + 4;  // smem row stride of a J chunk (20 == 4 mod 16: conflict-free A fragments)
constexpr int kMaxThreads = 256;
constexpr size_t kSmemPerSM = 228 * 1024;
constexpr size_t kSmemPerCTA = 227 * 1024;

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
__device__ __forceinline__ void cp_wait_n() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// wait until at most (nstage - 2) groups are pending
__device__ __forceinline__ void cp_wait_stage(int nstage) {
    if (nstage >= 4) cp_wait_n<2>();
    else if (nstage == 3) cp_wait_n<1>();
    else cp_wait_n<0>();
}

struct KArgs {
    ModeGeom geo;
    int S, MpB, Kp, BN, bn_log2, LDX, WM, WN, nstage, RB, Zrows;
    int prescale;
};

__device__ __forceinline__ int stage_doubles(const KArgs& a) {
    return kBK * a.LDX + a.MpB * kLDJ + (a.prescale ? kBK * a.LDX : 0);
}

// Global offset of element 0 of fiber cc (colex: l + L*n*r).
__device__ __forceinline__ long long fiber_base(long long cc, long long L, int n) {
    if (L == 1) return cc * n;
    const long long r = cc / L;
    return (cc - r * L) + L * static_cast<long long>(n) * r;
}

// Per-thread producer state of the fiber-chunk copies (precomputed once per tile, so a chunk
// costs a handful of integer ops per element).  Element u of this thread:
//   L == 1 (fibers contiguous): row j = tid % 16 (fixed), fiber c = tid/16 + u*nthr/16;
//   L  > 1 (fibers strided):    fiber c = tid % BN (fixed), row j = tid/BN + u*nthr/BN.
struct XProd {
    int cnt;               // elements per thread per chunk
    unsigned emask;        // element u exists (lies inside the 16 x BN chunk)
    unsigned umask;        // ... and its fiber is inside the tensor
    int row0, row_step;    // row of element u within a chunk = row0 + u*row_step
    int s_off, s_step;     // smem offsets (doubles) within a chunk
    long long g_off, g_step, g_kstep;  // global element offsets
};

__device__ __forceinline__ XProd make_xprod(const KArgs& a, long long c0) {
    XProd x;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int total = kBK * a.BN;
    x.cnt = (total + nthr - 1) / nthr;
    x.umask = 0;
    x.emask = 0;
    if (a.geo.L == 1) {
        const int j = tid & (kBK - 1), cf = tid >> 4, cstep = nthr >> 4;
        x.row0 = j;
        x.row_step = 0;
        x.s_off = j * a.LDX + cf;
        x.s_step = cstep;
        x.g_off = (c0 + cf) * a.geo.n + j;
        x.g_step = static_cast<long long>(cstep) * a.geo.n;
        x.g_kstep = kBK;
        for (int u = 0; u < x.cnt; ++u) {
            const int c = cf + u * cstep;
            if (c < a.BN) x.emask |= 1u << u;
            if (c < a.BN && c0 + c < a.geo.ncols) x.umask |= 1u << u;
        }
    } else {
        const int c = tid & (a.BN - 1), j0 = tid >> a.bn_log2, jstep = nthr >> a.bn_log2;
        x.row0 = j0;
        x.row_step = jstep;
        x.s_off = j0 * a.LDX + c;
        x.s_step = jstep * a.LDX;
        const long long cc = c0 + c;
        const bool cv = cc < a.geo.ncols;
        x.g_off = fiber_base(cv ? cc : 0, a.geo.L, a.geo.n) + a.geo.L * j0;
        x.g_step = a.geo.L * jstep;
        x.g_kstep = a.geo.L * kBK;
        for (int u = 0; u < x.cnt; ++u) {
            if (j0 + u * jstep < kBK) x.emask |= 1u << u;
            if (cv && j0 + u * jstep < kBK) x.umask |= 1u << u;
        }
    }
    return x;
}

struct JProd {
    int cnt;          // 16-byte pieces per thread per chunk
    int p2;           // 2 * (piece index within the row) (fixed per thread)
    int r0, rstep;    // row of piece u = r0 + u*rstep
};

__device__ __forceinline__ JProd make_jprod(const KArgs& a) {
    JProd j;
    const int tid = threadIdx.x, nthr = blockDim.x;
    j.cnt = (a.MpB * 8 + nthr - 1) / nthr;
    j.p2 = 2 * (tid & 7);
    j.r0 = tid >> 3;
    j.rstep = nthr >> 3;
    return j;
}

__device__ __forceinline__ void issue_x(const KArgs& a, const XProd& x, double* Xc, double* Dc,
                                        const double* __restrict__ X, const double* __restrict__ D, int q) {
    const int k0 = q * kBK;
    const long long gq = x.g_off + q * x.g_kstep;
    for (int u = 0; u < x.cnt; ++u) {
        if (!((x.emask >> u) & 1u)) continue;  // outside the chunk: must not touch smem
        const bool v = ((x.umask >> u) & 1u) && (k0 + x.row0 + u * x.row_step < a.geo.n);
        const long long gi = gq + u * x.g_step;
        const int so = x.s_off + u * x.s_step;
        cp_async8(Xc + so, v ? X + gi : X, v);
        if (Dc) cp_async8(Dc + so, v ? D + gi : D, v);
    }
}

__device__ __forceinline__ void prescale_own(const XProd& x, double* Xc, const double* Dc) {
    for (int u = 0; u < x.cnt; ++u) {
        const int so = x.s_off + u * x.s_step;
        if ((x.umask >> u) & 1u) Xc[so] *= Dc[so];
    }
}

__device__ __forceinline__ void issue_j(const KArgs& a, const JProd& jp, double* Jc, const double* __restrict__ Jg,
                                        int q) {
    const int k0 = q * kBK;
    const int kw = min(kBK, a.Kp - k0);
    if (jp.p2 >= kw) return;
    const double* src = Jg + k0 + jp.p2;
    for (int u = 0; u < jp.cnt; ++u) {
        const int r = jp.r0 + u * jp.rstep;
        if (r < a.MpB) cp_async16(Jc + r * kLDJ + jp.p2, src + static_cast<size_t>(r) * a.Kp);
    }
}

// acc += J_chunk * B_chunk over KS k-steps of 4.  A fragments from the J stage (ja), B fragments
// from bb (row stride ldb).  Fragments double-buffered in registers; no predicates (padded J
// rows are zero, so padded strips just produce zeros that are never stored).
template <int MI, int NI, int KS>
__device__ __forceinline__ void mma_chunk(const double* ja, const double* bb, int ldb, double (&acc)[MI][NI][2]) {
    double av[2][MI], bv[2][NI];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) av[0][mi] = ja[mi * 8 * kLDJ];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) bv[0][ni] = bb[ni * 8];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int cur = kk & 1, nxt = cur ^ 1;
        if (kk + 1 < KS) {
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) av[nxt][mi] = ja[mi * 8 * kLDJ + (kk + 1) * 4];
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) bv[nxt][ni] = bb[(kk + 1) * 4 * ldb + ni * 8];
        }
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], av[cur][mi], bv[cur][ni]);
    }
}

template <int MI, int NI>
__device__ __forceinline__ void mma_chunk_any(int ksteps, const double* ja, const double* bb, int ldb,
                                              double (&acc)[MI][NI][2]) {
    switch (ksteps) {
        case 4: mma_chunk<MI, NI, 4>(ja, bb, ldb, acc); break;
        case 3: mma_chunk<MI, NI, 3>(ja, bb, ldb, acc); break;
        case 2: mma_chunk<MI, NI, 2>(ja, bb, ldb, acc); break;
        default: mma_chunk<MI, NI, 1>(ja, bb, ldb, acc); break;
    }
}

// Register epilogue: acc rows (< m) of the CTA's row block straight to global memory.
template <int MI, int NI>
__device__ __forceinline__ void store_acc(const KArgs& a, const double (&acc)[MI][NI][2], long long c0, int strip0,
                                          double* __restrict__ Y) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wm = warp % a.WM, wn = warp / a.WM;
    const int g = lane >> 2, t = lane & 3;
    const int m = a.geo.m;
    long long ob[NI][2];
    bool cv[NI][2];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const long long cc = c0 + (wn * NI + ni) * 8 + 2 * t + v;
            cv[ni][v] = cc < a.geo.ncols;
            ob[ni][v] = fiber_base(cv[ni][v] ? cc : 0, a.geo.L, m);
        }
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
        const int i = (strip0 + wm * MI + mi) * 8 + g;
        if (i < m) {
            const long long off = a.geo.L * i;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (cv[ni][v]) Y[ob[ni][v] + off] = acc[mi][ni][v];
        }
    }
}

template <int MI, int NI>
__device__ __forceinline__ void zero_acc(double (&acc)[MI][NI][2]) {
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
}

// Multistage GEMM over the full contraction.  X_STREAM: the fiber operand streams through the
// stages with J; otherwise it is resident in smem at Bres (row stride a.LDX) and only J streams.
template <int MI, int NI, bool X_STREAM>
__device__ __forceinline__ void gemm(const KArgs& a, double* stages, const double* __restrict__ Jg,
                                     const double* __restrict__ X, const double* __restrict__ D, const double* Bres,
                                     const XProd& xp, const JProd& jp, bool prologue_issued, double (&acc)[MI][NI][2]) {
    const int nchunks = (a.Kp + kBK - 1) / kBK;
    const int sd = stage_doubles(a);
    const int ns = a.nstage;
    const int LDX = a.LDX;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp % a.WM, wn = warp / a.WM;
    const int g = lane >> 2, t = lane & 3;
    const int ja_off = kBK * LDX + (wm * MI * 8 + g) * kLDJ + t;  // within a stage
    const int bb_off = t * LDX + wn * NI * 8 + g;
    const int dc_off = kBK * LDX + a.MpB * kLDJ;
    if (!prologue_issued) {
        for (int s = 0; s < ns - 1; ++s) {
            if (s < nchunks) {
                double* st = stages + static_cast<size_t>(s) * sd;
                issue_j(a, jp, st + kBK * LDX, Jg, s);
                if (X_STREAM) issue_x(a, xp, st, D ? st + dc_off : nullptr, X, D, s);
            }
            cp_commit();
        }
    }
    int stage = 0;
    for (int q = 0; q < nchunks; ++q) {
        cp_wait_stage(ns);
        double* st = stages + static_cast<size_t>(stage) * sd;
        if (X_STREAM && D) prescale_own(xp, st, st + dc_off);
        __syncthreads();
        const int nq = q + ns - 1;
        if (nq < nchunks) {
            int nst = stage + ns - 1;
            if (nst >= ns) nst -= ns;
            double* sn = stages + static_cast<size_t>(nst) * sd;
            issue_j(a, jp, sn + kBK * LDX, Jg, nq);
            if (X_STREAM) issue_x(a, xp, sn, D ? sn + dc_off : nullptr, X, D, nq);
        }
        cp_commit();
        const double* ja = st + ja_off;
        const double* bb = X_STREAM ? st + bb_off : Bres + q * kBK * LDX + bb_off;
        const int ksteps = min(kBK, a.Kp - q * kBK) >> 2;
        if (ksteps == 4)
            mma_chunk<MI, NI, 4>(ja, bb, LDX, acc);
        else
            mma_chunk_any<MI, NI>(ksteps, ja, bb, LDX, acc);
        if (++stage == ns) stage = 0;
    }
}

// Issues the GEMM prologue (J chunks only) so it overlaps work done before gemm<..., false>.
__device__ __forceinline__ void gemm_prologue_j(const KArgs& a, double* stages, const double* __restrict__ Jg,
                                                const JProd& jp) {
    const int nchunks = (a.Kp + kBK - 1) / kBK;
    const int sd = stage_doubles(a);
    for (int s = 0; s < a.nstage - 1; ++s) {
        if (s < nchunks) issue_j(a, jp, stages + static_cast<size_t>(s) * sd + kBK * a.LDX, Jg, s);
        cp_commit();
    }
}

template <int MI, int NI>
__global__ void __launch_bounds__(kMaxThreads)
    mode_product_kernel(KArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ J,
                        const double* __restrict__ D) {
    extern __shared__ __align__(16) double smem[];
    const int rb = blockIdx.x % a.RB;  // row blocks of one fiber tile are adjacent -> X tile reused from L2
    const long long c0 = static_cast<long long>(blockIdx.x / a.RB) * a.BN;
    const int strip0 = rb * MI * a.WM;
    const double* Jg = J + static_cast<size_t>(rb) * a.MpB * a.Kp;
    const XProd xp = make_xprod(a, c0);
    const JProd jp = make_jprod(a);
    double acc[MI][NI][2];
    zero_acc(acc);
    gemm<MI, NI, true>(a, smem, Jg, X, D, nullptr, xp, jp, false, acc);
    store_acc(a, acc, c0, strip0, Y);
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
__device__ __forceinline__ void arrowhead_tile(const KArgs& a, double* Zs, long long c0, const ArrowParams& ap) {
    int P = 1;
    while (P < 32 && 2 * P * a.BN <= static_cast<int>(blockDim.x)) P *= 2;
    const int tid = threadIdx.x;
    if (tid >= P * a.BN) return;  // whole warps (P*BN is a multiple of 16; BN >= 16)
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
    const int LD = a.LDX;
    double* col = Zs + c;
    const double slast = col[(nt - 1) * LD];
    double part = 0.0;
    for (int j = p; j < ap.npairs; j += P) {
        double xa, xb;
        pair_inverse(lam, linv, nu, __ldg(ap.pair_c + j), __ldg(ap.pair_c1 + j), col[(2 * j) * LD],
                     col[(2 * j + 1) * LD], xa, xb);
        col[(2 * j) * LD] = xa;
        col[(2 * j + 1) * LD] = xb;
        part += gam * (__ldg(ap.g + 2 * j) * xa + __ldg(ap.g + 2 * j + 1) * xb);
    }
    if (ap.zero_count && p == 0) {
        const int z = nt - 2;
        const double xz = linv * col[z * LD] / nu;
        col[z * LD] = xz;
        part += gam * __ldg(ap.g + z) * xz;
    }
    const unsigned mask = (P * a.BN >= 32) ? 0xffffffffu : ((1u << (P * a.BN)) - 1u);
    for (int off = P >> 1; off > 0; off >>= 1) part += __shfl_xor_sync(mask, part, off);
    const double xlast = __ldg(ap.S_inv + s) * (slast + part);
    for (int j = p; j < ap.npairs; j += P) {
        double xa, xb;
        pair_inverse(lam, linv, nu, __ldg(ap.pair_c + j), __ldg(ap.pair_c1 + j),
                     (gam * __ldg(ap.g + 2 * j)) * xlast, (gam * __ldg(ap.g + 2 * j + 1)) * xlast, xa, xb);
        col[(2 * j) * LD] -= xa;
        col[(2 * j + 1) * LD] -= xb;
    }
    if (p == 0) {
        if (ap.zero_count) {
            const int z = nt - 2;
            col[z * LD] -= (gam * __ldg(ap.g + z) / nu) * (linv * xlast);
        }
        col[(nt - 1) * LD] = xlast;
    }
}

template <int MI, int NI>
__global__ void __launch_bounds__(kMaxThreads)
    time_fused_kernel(KArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ Jt,
                      const double* __restrict__ J, ArrowParams ap) {
    extern __shared__ __align__(16) double smem[];
    double* Zs = smem;                                             // Zrows x LDX, resident
    double* stages = smem + static_cast<size_t>(a.Zrows) * a.LDX;  // nstage x stage
    const long long c0 = static_cast<long long>(blockIdx.x) * a.BN;
    const XProd xp = make_xprod(a, c0);
    const JProd jp = make_jprod(a);
    double acc[MI][NI][2];
    zero_acc(acc);
    gemm<MI, NI, true>(a, stages, Jt, X, nullptr, nullptr, xp, jp, false, acc);  // Z = U_t^T x
    // Z -> smem (rows < Kp; padded rows are exact zeros because the padded J rows are zero)
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int wm = warp % a.WM, wn = warp / a.WM;
        const int g = lane >> 2, t = lane & 3;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
            const int row = (wm * MI + mi) * 8 + g;
            if (row < a.Zrows) {
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) {
                    const int col = (wn * NI + ni) * 8 + 2 * t;
                    Zs[row * a.LDX + col] = acc[mi][ni][0];
                    Zs[row * a.LDX + col + 1] = acc[mi][ni][1];
                }
            }
        }
    }
    __syncthreads();  // Z visible; every warp is done with the GEMM-1 stages
    gemm_prologue_j(a, stages, J, jp);  // U_t chunks stream in while the arrowhead runs
    if (!(ap.debug & 1)) arrowhead_tile(a, Zs, c0, ap);
    __syncthreads();
    zero_acc(acc);
    gemm<MI, NI, false>(a, stages, J, nullptr, nullptr, Zs, xp, jp, true, acc);  // y = U_t z
    store_acc(a, acc, c0, 0, Y);
}

__global__ void scale_kernel(const double* __restrict__ a, const double* __restrict__ x, double* __restrict__ y,
                             long long n) {
    const long long n2 = n >> 1;
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const double2* x2 = reinterpret_cast<const double2*>(x);
    double2* y2 = reinterpret_cast<double2*>(y);
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n2;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double2 av = a2[i], xv = x2[i];
        y2[i] = make_double2(av.x * xv.x, av.y * xv.y);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) y[n - 1] = a[n - 1] * x[n - 1];
}

KArgs make_args(const Tiling& t, const ModeGeom& g) {
    KArgs a;
    a.geo = g;
    a.S = t.S;
    a.MpB = t.MpB;
    a.Kp = t.Kp;
    a.BN = t.BN;
    a.bn_log2 = 0;
    while ((1 << a.bn_log2) < t.BN) ++a.bn_log2;
    a.LDX = t.LDX;
    a.WM = t.WM;
    a.WN = t.WN;
    a.nstage = t.nstage;
    a.RB = t.RB;
    a.Zrows = t.Zrows;
    a.prescale = t.prescale ? 1 : 0;
    return a;
}

// Resident CTAs per SM of an instantiation (exact occupancy query; falls back to a smem/thread
// bound with a register estimate when no device is current).
template <typename K>
int occupancy(K kernel, int threads, size_t smem, int MI) {
    int n = 0;
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) ==
            cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) == cudaSuccess)
        return n;
    cudaGetLastError();
    const int regs = std::min(255, 16 * MI + 40);
    const int by_smem = static_cast<int>(kSmemPerSM / (smem + 1024));
    const int by_regs = 65536 / (threads * ((regs + 7) / 8 * 8));
    return std::max(0, std::min({by_smem, 2048 / threads, by_regs}));
}

#define STIGA_MI_CASES(MI_, EXPR)                                                                    \
    switch (MI_) {                                                                                   \
        case 1: return EXPR(1); case 2: return EXPR(2); case 3: return EXPR(3); case 4: return EXPR(4); \
        case 5: return EXPR(5); case 6: return EXPR(6); case 7: return EXPR(7); case 8: return EXPR(8); \
        case 9: return EXPR(9); case 10: return EXPR(10); case 11: return EXPR(11);                  \
        case 12: return EXPR(12); case 13: return EXPR(13);                                          \
        default: return 0;                                                                           \
    }

int mode_occupancy(int MI, int threads, size_t smem) {
#define STIGA_OCC_MODE(M) occupancy(mode_product_kernel<M, 2>, threads, smem, M)
    STIGA_MI_CASES(MI, STIGA_OCC_MODE)
#undef STIGA_OCC_MODE
}

int time_occupancy(int MI, int threads, size_t smem) {
#define STIGA_OCC_TIME(M) occupancy(time_fused_kernel<M, 2>, threads, smem, M)
    STIGA_MI_CASES(MI, STIGA_OCC_TIME)
#undef STIGA_OCC_TIME
}

template <int MI>
cudaError_t launch_mode_mi(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                           const double* pre, cudaStream_t st) {
    auto k = mode_product_kernel<MI, 2>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(t.smem));
    if (e != cudaSuccess) return e;
    const long long blocks = (g.ncols + t.BN - 1) / t.BN * t.RB;
    k<<<static_cast<unsigned>(blocks), t.threads(), t.smem, st>>>(make_args(t, g), X, Y, J, pre);
    return cudaGetLastError();
}

template <int MI>
cudaError_t launch_time_mi(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt,
                           const double* J, const ArrowParams& ap, cudaStream_t st) {
    auto k = time_fused_kernel<MI, 2>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(t.smem));
    if (e != cudaSuccess) return e;
    const long long blocks = (g.ncols + t.BN - 1) / t.BN;
    k<<<static_cast<unsigned>(blocks), t.threads(), t.smem, st>>>(make_args(t, g), X, Y, Jt, J, ap);
    return cudaGetLastError();
}

}  // namespace

Tiling choose_mode_tiling(int m, int n, bool prescale) {
    Tiling best;
    double best_score = -1.0;
    const int S = (m + 7) / 8;
    const int Kp = (n + 3) / 4 * 4;
    const int rb0 = (S + 12) / 13;
    for (int RB = rb0; RB <= rb0 + 1; ++RB) {
        const int MI = (S + RB - 1) / RB;
        if (MI > 13 || MI < 1) continue;
        for (int WN : {4, 2}) {
            for (int ns : {3, 2}) {
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
                t.nstage = ns;
                t.prescale = prescale;
                t.smem = sizeof(double) * static_cast<size_t>(ns) *
                         (kBK * t.LDX + t.MpB * kLDJ + (prescale ? kBK * t.LDX : 0));
                if (t.smem > kSmemPerCTA) continue;
                t.ctas_per_sm = mode_occupancy(MI, t.threads(), t.smem);
                if (t.ctas_per_sm < 1) continue;
                const double eff = static_cast<double>(S) / (RB * MI);
                const double score = std::min(t.ctas_per_sm * t.WM * t.WN, 16) * eff + 0.01 * ns + 0.02 * WN;
                if (score > best_score) {
                    best_score = score;
                    best = t;
                }
            }
        }
    }
    return best;
}

Tiling choose_time_tiling(int nt) {
    Tiling best;
    double best_score = -1.0;
    int force_wm = 0, force_wn = 0, force_ns = 0;  // debugging aid: STIGA_FORCE_TIME_TILING="WM,WN,NS"
    if (const char* f = std::getenv("STIGA_FORCE_TIME_TILING")) std::sscanf(f, "%d,%d,%d", &force_wm, &force_wn, &force_ns);
    const int S = (nt + 7) / 8;
    const int Kp = (nt + 3) / 4 * 4;
    const int wm0 = (S + 12) / 13;
    for (int WM = wm0; WM <= wm0 + (force_wm ? 8 : 2); ++WM) {
        const int MI = (S + WM - 1) / WM;
        if (MI > 13 || MI < 1) continue;
        for (int WN : {4, 2, 1}) {
            if (32 * WM * WN > kMaxThreads) continue;
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
                                           static_cast<size_t>(ns) * (kBK * t.LDX + t.MpB * kLDJ));
                if (t.smem > kSmemPerCTA) continue;
                t.ctas_per_sm = time_occupancy(MI, t.threads(), t.smem);
                if (t.ctas_per_sm < 1) continue;
                const double eff = static_cast<double>(S) / (WM * MI);
                const double score = std::min(t.ctas_per_sm * WM * WN, 16) * eff + 0.01 * ns + 0.02 * WN;
                if (score > best_score) {
                    best_score = score;
                    best = t;
                }
            }
        }
    }
    return best;
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
                                const double* pre, cudaStream_t st) {
    if (g.ncols <= 0) return cudaSuccess;
    if (pre && !t.prescale) return cudaErrorInvalidValue;
#define STIGA_CALL_MODE(M) launch_mode_mi<M>(t, g, X, Y, Jpad, pre, st)
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
    const long long blocks = std::min<long long>((n / 2 + threads - 1) / threads + 1, 148LL * 8);
    scale_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(a, x, y, n);
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace stiga
